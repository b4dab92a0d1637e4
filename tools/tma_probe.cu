// NVLink write/read efficiency of bulk-async (TMA engine) copies vs 16-byte
// LDG/STG to peer memory (design probe, not product).  One process, two GPUs
// with peer access; kernels on both GPUs never wait on each other.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tools/tma_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) {                                                            \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));   \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// bulk store: smem tile -> global (peer) via the TMA engine; STAGES tiles in flight
template <int TILE, int STAGES>
__global__ void bulk_store(char* dst, long bytes) {
  extern __shared__ __align__(128) char sm[];
  // fill smem once (content irrelevant)
  for (int i = threadIdx.x * 16; i < TILE * STAGES; i += blockDim.x * 16) *(int4*)(sm + i) = make_int4(1, 2, 3, 4);
  __syncthreads();
  if (threadIdx.x != 0) return;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  long ntiles = bytes / TILE;
  int s = 0;
  for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + t * TILE),
                 "r"(smem_addr(sm + s * TILE)), "n"(TILE)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(STAGES - 1) : "memory");
    s = (s + 1) % STAGES;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// bulk load: global (peer) -> smem via the TMA engine, mbarrier completion
template <int TILE, int STAGES>
__global__ void bulk_load(const char* src, long bytes, int* sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[i])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  long ntiles = bytes / TILE;
  uint32_t phase[STAGES] = {0};
  int issued = 0;
  long t = blockIdx.x;
  long tdone = blockIdx.x;
  int acc = 0;
  // prologue
  for (int s = 0; s < STAGES && t < ntiles; ++s, t += gridDim.x, ++issued) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar[s])), "n"(TILE) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(sm + s * TILE)),
                 "l"(src + t * TILE), "n"(TILE), "r"(smem_addr(&bar[s]))
                 : "memory");
  }
  int s = 0;
  while (tdone < ntiles) {
    // wait stage s
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(ok)
          : "r"(smem_addr(&bar[s])), "r"(phase[s])
          : "memory");
    }
    phase[s] ^= 1;
    acc += sm[s * TILE];
    tdone += gridDim.x;
    if (t < ntiles) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar[s])), "n"(TILE) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_addr(sm + s * TILE)),
                   "l"(src + t * TILE), "n"(TILE), "r"(smem_addr(&bar[s]))
                   : "memory");
      t += gridDim.x;
    }
    s = (s + 1) % STAGES;
  }
  if (acc == 12345) *sink = acc;
}

__global__ void stg_store(int4* dst, long n) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    dst[i] = make_int4(1, 2, 3, (int)i);
}
__global__ void ldg_load(const int4* src, long n, int* sink) {
  int acc = 0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x * 4) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      long j = i + (long)u * gridDim.x * blockDim.x;
      v[u] = j < n ? __ldcg(src + j) : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u].x;
  }
  if (acc == 12345) *sink = acc;
}

int main() {
  int nd;
  CK(cudaGetDeviceCount(&nd));
  if (nd < 2) return 0;
  const long bytes = 256l << 20;
  char* buf[2];
  int* sink[2];
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&buf[d], bytes));
    CK(cudaMalloc(&sink[d], 64));
    CK(cudaStreamCreate(&st[d]));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  auto run = [&](const char* name, auto launch, bool bidi) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      for (int d = 0; d < (bidi ? 2 : 1); ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventRecord(e0[d], st[d]));
        launch(d);
        CK(cudaGetLastError());
        CK(cudaEventRecord(e1[d], st[d]));
      }
      float worst = 0;
      for (int d = 0; d < (bidi ? 2 : 1); ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(e1[d]));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
        worst = ms > worst ? ms : worst;
      }
      if (r && worst < best) best = worst;
    }
    std::printf("%-44s %s %8.1f GB/s per direction\n", name, bidi ? "bidi" : "1dir", bytes / (best * 1e-3) / 1e9);
  };
  for (int bidi = 0; bidi < 2; ++bidi) {
    run("STG.128 to peer (592x512)", [&](int d) { stg_store<<<592, 512, 0, st[d]>>>((int4*)buf[1 - d], bytes / 16); }, bidi);
    run("LDG.128 from peer (592x512, 4 in flight)",
        [&](int d) { ldg_load<<<592, 512, 0, st[d]>>>((const int4*)buf[1 - d], bytes / 16, sink[d]); }, bidi);
#define BS(TILE, ST, G)                                                                                          \
  {                                                                                                              \
    CK(cudaSetDevice(0));                                                                                        \
    CK(cudaFuncSetAttribute(bulk_store<TILE, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE * ST));      \
    CK(cudaSetDevice(1));                                                                                        \
    CK(cudaFuncSetAttribute(bulk_store<TILE, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE * ST));      \
    run("bulk store tile=" #TILE " stages=" #ST " grid=" #G,                                                    \
        [&](int d) { bulk_store<TILE, ST><<<G, 128, TILE * ST, st[d]>>>(buf[1 - d], bytes); }, bidi);          \
  }
#define BL(TILE, ST, G)                                                                                          \
  {                                                                                                              \
    CK(cudaSetDevice(0));                                                                                        \
    CK(cudaFuncSetAttribute(bulk_load<TILE, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE * ST));       \
    CK(cudaSetDevice(1));                                                                                        \
    CK(cudaFuncSetAttribute(bulk_load<TILE, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE * ST));       \
    run("bulk load  tile=" #TILE " stages=" #ST " grid=" #G,                                                    \
        [&](int d) { bulk_load<TILE, ST><<<G, 128, TILE * ST, st[d]>>>(buf[1 - d], bytes, sink[d]); }, bidi);  \
  }
    BS(4096, 4, 148) BS(16384, 4, 148) BS(32768, 4, 148) BS(16384, 8, 148) BS(16384, 4, 296)
    BL(4096, 4, 148) BL(16384, 4, 148) BL(32768, 4, 148) BL(16384, 8, 148) BL(16384, 4, 296)
  }
  return 0;
}
