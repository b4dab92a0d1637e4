// Kernel-completion probe (design probe, not product): which kinds of peer
// memory access make a kernel's launch + completion expensive?  One process,
// two GPUs with peer access; GPU 0 runs every kernel.  For each variant:
//   single: CUDA events around ONE launch (median of 200), the number a
//           collective call pays;
//   b2b:    200 launches between one event pair, per launch.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o completion_probe tools/completion_probe.cu
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
__device__ __forceinline__ unsigned ld_acq_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// variant:
//  0 nothing
//  1 one relaxed.sys store per CTA to the peer
//  2 one relaxed.sys load per CTA from the peer
//  3 one weak (ld.global) load per CTA from the peer
//  4 one acquire.sys load per CTA from the peer
//  5 one release.sys store per CTA to LOCAL memory
//  6 pull `bytes` from the peer (LDG.128), store locally
//  7 push `bytes` (local LDG.128, STG.128 to the peer)
//  8 local copy of `bytes`
//  9 one relaxed.sys store per CTA to the peer, then fence.sc.sys
// 10 pull `bytes` from the peer, store locally, relaxed.sys store to LOCAL flag
// 11 one relaxed.sys store per CTA to LOCAL memory
__global__ void __launch_bounds__(512) probe(int variant, unsigned* remote, unsigned* local, const int4* src,
                                             int4* dst, long n16, unsigned e, int active) {
  const int b = blockIdx.x;
  __shared__ unsigned s;
  if (variant >= 1 && variant <= 4 && b >= active) return;  // only the first `active` CTAs touch the peer
  if (variant == 1) {
    if (threadIdx.x == 0) st_rlx_sys(remote + b * 32, e);
  } else if (variant == 2) {
    if (threadIdx.x == 0) s = ld_rlx_sys(remote + b * 32);
  } else if (variant == 3) {
    if (threadIdx.x == 0) s = *(volatile unsigned*)(remote + b * 32);
  } else if (variant == 4) {
    if (threadIdx.x == 0) s = ld_acq_sys(remote + b * 32);
  } else if (variant == 5) {
    if (threadIdx.x == 0) st_rel_sys(local + b * 32, e);
  } else if (variant == 6 || variant == 7 || variant == 8 || variant == 10) {
    for (long i = b * (long)blockDim.x + threadIdx.x; i < n16; i += (long)gridDim.x * blockDim.x) dst[i] = src[i];
    if (variant == 10) {
      __syncthreads();
      if (threadIdx.x == 0) st_rlx_sys(local + b * 32, e);
    }
  } else if (variant == 9) {
    if (threadIdx.x == 0) {
      st_rlx_sys(remote + b * 32, e);
      asm volatile("fence.sc.sys;" ::: "memory");
    }
  } else if (variant == 11) {
    if (threadIdx.x == 0) st_rlx_sys(local + b * 32, e);
  }
  if (variant >= 2 && variant <= 4 && threadIdx.x == 0 && s == 0xdeadbeefu) local[1 << 20] = s;
}

int main(int argc, char** argv) {
  int nd = 0;
  CK(cudaGetDeviceCount(&nd));
  if (nd < 2) {
    std::printf("{\"skip\": \"needs 2 GPUs\"}\n");
    return 0;
  }
  CK(cudaSetDevice(1));
  unsigned* remote;
  int4* rbuf;
  const long maxbytes = 64l << 20;
  CK(cudaMalloc(&remote, 1 << 22));
  CK(cudaMemset(remote, 0, 1 << 22));
  CK(cudaMalloc(&rbuf, maxbytes));
  CK(cudaMemset(rbuf, 1, maxbytes));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  unsigned* local;
  int4 *lbuf, *lbuf2;
  CK(cudaMalloc(&local, 1 << 23));
  CK(cudaMemset(local, 0, 1 << 23));
  CK(cudaMalloc(&lbuf, maxbytes));
  CK(cudaMalloc(&lbuf2, maxbytes));
  CK(cudaMemset(lbuf, 2, maxbytes));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t a, z;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&z));
  const char* names[] = {"nothing",          "remote st.relaxed.sys x1/CTA", "remote ld.relaxed.sys x1/CTA",
                         "remote ld.weak x1/CTA", "remote ld.acquire.sys x1/CTA", "local st.release.sys x1/CTA",
                         "pull bytes",       "push bytes",                    "local copy bytes",
                         "remote st.relaxed.sys + fence.sc.sys", "pull bytes + local st.relaxed.sys",
                         "local st.relaxed.sys x1/CTA"};
  const int nvar = 12;
  const long sizes[] = {4096, 1 << 20, 16 << 20};
  unsigned e = 1;
  for (int grid : {148, 296}) {
    for (int v = 0; v < nvar; ++v) {
      for (long bytes : sizes) for (int act : {1, 4, 16, 64, 148, 296}) {
        const bool data = v == 6 || v == 7 || v == 8 || v == 10;
        if (!data && bytes != sizes[0]) continue;
        if (act > grid || ((v < 1 || v > 4) && act != grid) || (v >= 3 && v <= 4 && act != grid)) continue;
        const int4* src = v == 6 || v == 10 ? rbuf : lbuf;
        int4* dst = v == 7 ? rbuf : lbuf2;
        const long n16 = bytes / 16;
        for (int w = 0; w < 20; ++w) probe<<<grid, 512, 0, st>>>(v, remote, local, src, dst, n16, e++, act);
        CK(cudaStreamSynchronize(st));
        std::vector<float> one;
        for (int i = 0; i < 200; ++i) {
          CK(cudaEventRecord(a, st));
          probe<<<grid, 512, 0, st>>>(v, remote, local, src, dst, n16, e++, act);
          CK(cudaEventRecord(z, st));
          CK(cudaEventSynchronize(z));
          float ms;
          CK(cudaEventElapsedTime(&ms, a, z));
          one.push_back(ms * 1e3f);
        }
        std::sort(one.begin(), one.end());
        CK(cudaEventRecord(a, st));
        for (int i = 0; i < 200; ++i) probe<<<grid, 512, 0, st>>>(v, remote, local, src, dst, n16, e++, act);
        CK(cudaEventRecord(z, st));
        CK(cudaEventSynchronize(z));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, z));
        std::printf(
            "{\"grid\": %d, \"active\": %d, \"variant\": %d, \"what\": \"%s\", \"bytes\": %ld, \"single_us_p50\": %.2f, "
            "\"single_us_p10\": %.2f, \"b2b_us\": %.2f}\n",
            grid, act, v, names[v], data ? bytes : 0, one[one.size() / 2], one[one.size() / 10], ms * 1e3f / 200);
        std::fflush(stdout);
      }
    }
  }
  CK(cudaGetLastError());
  return 0;
}
