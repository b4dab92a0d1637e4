// Launch-prologue probe (design probe, not product): what does the first
// remote flag store of a launch cost, with and without an L2-flushing kernel
// in front of it, and what do the sys-scope fences cost at exit?  One process,
// two GPUs, peer access; only GPU 0 runs kernels (stores to GPU 1 memory need
// no kernel there).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o entry_probe tools/entry_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      std::exit(1);                                                                  \
    }                                                                                \
  } while (0)

__device__ __forceinline__ unsigned long long now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void st_rlx_sys(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rel_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_rlx_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// t[0] start, t[1] after remote relaxed store #1, t[2] after remote load (round
// trip), t[3] after remote relaxed store #2, t[4] after local store + remote
// load, t[5] after st.release.sys remote, t[6] after fence.acq_rel.gpu,
// t[7] after fence.sc.sys
__global__ void prologue(unsigned* remote, unsigned* local, unsigned long long* out, unsigned e) {
  const int b = blockIdx.x;
  unsigned long long t[8];
  __shared__ unsigned s;
  t[0] = now();
  if (threadIdx.x == 0) st_rlx_sys(remote + b, e);
  t[1] = now();
  if (threadIdx.x == 0) s = ld_rlx_sys(remote + 4096 + b);
  __syncthreads();
  t[2] = now();
  if (threadIdx.x == 0) st_rlx_sys(remote + 8192 + b, e);
  t[3] = now();
  if (threadIdx.x == 0) {
    local[b] = e;
    s += ld_rlx_sys(remote + 4096 + b);
  }
  __syncthreads();
  t[4] = now();
  if (threadIdx.x == 0) st_rel_sys(remote + 12288 + b, e + s);
  __syncthreads();
  t[5] = now();
  if (threadIdx.x == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  __syncthreads();
  t[6] = now();
  if (threadIdx.x == 0) asm volatile("fence.sc.sys;" ::: "memory");
  __syncthreads();
  t[7] = now();
  if (threadIdx.x == 0 && (b == 0 || b == gridDim.x - 1))
    for (int i = 0; i < 8; ++i) out[(b == 0 ? 0 : 8) + i] = t[i];
}

__global__ void flush(int4* p, long n16, int v) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n16; i += (long)gridDim.x * blockDim.x)
    p[i] = make_int4(v, v, v, v);
}
__global__ void spin(long long ns) {
  unsigned long long t0 = now();
  while ((long long)(now() - t0) < ns) {}
}

__global__ void k_empty() {}
__global__ void k_remote_store(unsigned* remote) {
  if (threadIdx.x == 0) st_rlx_sys(remote + blockIdx.x, 1u);
}
__global__ void k_remote_store_fence(unsigned* remote) {
  if (threadIdx.x == 0) {
    st_rlx_sys(remote + blockIdx.x, 1u);
    asm volatile("fence.sc.sys;" ::: "memory");
  }
}
__global__ void k_remote_load(unsigned* remote, unsigned* out) {
  if (threadIdx.x == 0) out[blockIdx.x] = ld_rlx_sys(remote + blockIdx.x);
}
__global__ void k_smem(unsigned* out) {
  extern __shared__ unsigned sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = sm[5];
}

// event-timed launches with the host far ahead (a spin kernel in front)
template <typename F>
double event_us(F launch) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  std::vector<double> v;
  for (int it = 0; it < 25; ++it) {
    spin<<<1, 1>>>(200000);
    CK(cudaEventRecord(a));
    launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (it >= 5) v.push_back(ms * 1e3);
  }
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

int main() {
  int nd = 0;
  CK(cudaGetDeviceCount(&nd));
  if (nd < 2) return 0;
  unsigned *remote, *local;
  unsigned long long* out;
  int4* fb;
  const long fbytes = 256l << 20;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&remote, 1 << 20));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&local, 1 << 20));
  CK(cudaMalloc(&out, 16 * 8));
  CK(cudaMalloc(&fb, fbytes));
  const char* names[] = {"remote st.relaxed #1", "remote ld round trip", "remote st.relaxed #2",
                         "local st + remote ld", "st.release.sys remote", "fence.acq_rel.gpu", "fence.sc.sys"};
  for (int variant = 0; variant < 3; ++variant) {
    std::vector<std::vector<double>> d(7);
    for (int it = 0; it < 30; ++it) {
      if (variant >= 1) flush<<<592, 512>>>(fb, fbytes / 16, it);
      if (variant == 2) spin<<<1, 1>>>(50000);
      prologue<<<148, 512>>>(remote, local, out, (unsigned)it);
      CK(cudaDeviceSynchronize());
      unsigned long long h[16];
      CK(cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost));
      if (it < 5) continue;
      for (int i = 0; i < 7; ++i) d[i].push_back((h[i + 1] - h[i]) / 1e3);
    }
    std::printf("variant %s\n", variant == 0 ? "back-to-back" : variant == 1 ? "after L2 flush" : "after flush+spin");
    for (int i = 0; i < 7; ++i) {
      std::sort(d[i].begin(), d[i].end());
      std::printf("  %-24s median %.3f us  min %.3f  max %.3f\n", names[i], d[i][d[i].size() / 2], d[i][0], d[i].back());
    }
  }
  std::printf("launch cost, CUDA events with the host ahead (median us):\n");
  std::printf("  empty 16x512            %.2f\n", event_us([&] { k_empty<<<16, 512>>>(); }));
  std::printf("  empty 148x512           %.2f\n", event_us([&] { k_empty<<<148, 512>>>(); }));
  std::printf("  remote store 16x512     %.2f\n", event_us([&] { k_remote_store<<<16, 512>>>(remote); }));
  std::printf("  remote st+fence 16x512  %.2f\n", event_us([&] { k_remote_store_fence<<<16, 512>>>(remote); }));
  std::printf("  remote load 16x512      %.2f\n", event_us([&] { k_remote_load<<<16, 512>>>(remote, local); }));
  std::printf("  40KB smem 16x512        %.2f\n", event_us([&] { k_smem<<<16, 512, 40 * 1024>>>(local); }));
  return 0;
}
