// Cross-GPU flag latency probe (design probe, not product): two GPUs play
// ping-pong through flags in each other's memory, one thread each, with
// different store/load/fence flavours; plus the cost of a system fence after
// remote stores.  Kernels on different GPUs wait on each other (allowed: one
// kernel per GPU).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o flag_probe tools/flag_probe.cu
#include <cuda_runtime.h>

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

__device__ __forceinline__ unsigned ld_acq_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_vol(const unsigned* p) { return *(volatile const unsigned*)p; }
__device__ __forceinline__ void st_rel_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rlx_sys(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// variant: 0 rel/acq sys, 1 relaxed.sys both, 2 volatile both, 3 fence.sc.sys + relaxed, 4 fence.acq_rel.sys + relaxed
template <int V>
__global__ void pingpong(unsigned* mine, unsigned* theirs, int iters, int leader, unsigned long long* out) {
  unsigned long long t0 = now();
  for (int i = 1; i <= iters; ++i) {
    if (leader) {
      if (V == 0) st_rel_sys(theirs, i);
      else if (V == 1) st_rlx_sys(theirs, i);
      else if (V == 2) *(volatile unsigned*)theirs = i;
      else if (V == 3) { asm volatile("fence.sc.sys;" ::: "memory"); st_rlx_sys(theirs, i); }
      else { asm volatile("fence.acq_rel.sys;" ::: "memory"); st_rlx_sys(theirs, i); }
      while ((V == 0 ? ld_acq_sys(mine) : V == 2 ? ld_vol(mine) : ld_rlx_sys(mine)) < (unsigned)i) {}
    } else {
      while ((V == 0 ? ld_acq_sys(mine) : V == 2 ? ld_vol(mine) : ld_rlx_sys(mine)) < (unsigned)i) {}
      if (V == 0) st_rel_sys(theirs, i);
      else if (V == 1) st_rlx_sys(theirs, i);
      else if (V == 2) *(volatile unsigned*)theirs = i;
      else if (V == 3) { asm volatile("fence.sc.sys;" ::: "memory"); st_rlx_sys(theirs, i); }
      else { asm volatile("fence.acq_rel.sys;" ::: "memory"); st_rlx_sys(theirs, i); }
    }
  }
  out[0] = now() - t0;
}

// cost of a fence after `nbytes` of remote 16B stores by one CTA
template <int F>
__global__ void store_then_fence(int4* remote, long n16, unsigned long long* out) {
  for (long i = threadIdx.x; i < n16; i += blockDim.x) remote[i] = make_int4(1, 2, 3, 4);
  __syncthreads();
  unsigned long long t0 = now();
  if (threadIdx.x == 0) {
    if (F == 0) asm volatile("fence.sc.sys;" ::: "memory");
    else if (F == 1) asm volatile("fence.acq_rel.sys;" ::: "memory");
    else if (F == 2) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    else __threadfence_system();
  }
  __syncthreads();
  if (threadIdx.x == 0) out[0] = now() - t0;
}

int main() {
  int nd = 0;
  CK(cudaGetDeviceCount(&nd));
  if (nd < 2) return 0;
  unsigned* flag[2];
  unsigned long long* out[2];
  int4* buf[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&flag[d], 256));
    CK(cudaMalloc(&out[d], 64));
    CK(cudaMalloc(&buf[d], 64 << 20));
  }
  const int iters = 2000;
  const char* names[] = {"st.release.sys/ld.acquire.sys", "st.relaxed.sys/ld.relaxed.sys", "volatile/volatile",
                         "fence.sc.sys+relaxed", "fence.acq_rel.sys+relaxed"};
  for (int v = 0; v < 5; ++v) {
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaMemset(flag[d], 0, 256));
      CK(cudaDeviceSynchronize());
    }
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      void (*k)(unsigned*, unsigned*, int, int, unsigned long long*) =
          v == 0 ? pingpong<0> : v == 1 ? pingpong<1> : v == 2 ? pingpong<2> : v == 3 ? pingpong<3> : pingpong<4>;
      k<<<1, 1>>>(flag[d], flag[1 - d], iters, d == 0, out[d]);
    }
    unsigned long long ns = 0;
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaDeviceSynchronize());
    }
    CK(cudaSetDevice(0));
    CK(cudaMemcpy(&ns, out[0], 8, cudaMemcpyDeviceToHost));
    std::printf("%-32s round trip %.3f us\n", names[v], ns / 1e3 / iters);
  }
  const char* fn[] = {"fence.sc.sys", "fence.acq_rel.sys", "fence.acq_rel.gpu", "__threadfence_system"};
  long sizes[] = {0, 16, 4096, 65536, 1 << 20};
  for (int f = 0; f < 4; ++f)
    for (long s : sizes) {
      CK(cudaSetDevice(0));
      unsigned long long best = ~0ull;
      for (int r = 0; r < 5; ++r) {
        if (f == 0) store_then_fence<0><<<1, 512>>>(buf[1], s / 16, out[0]);
        else if (f == 1) store_then_fence<1><<<1, 512>>>(buf[1], s / 16, out[0]);
        else if (f == 2) store_then_fence<2><<<1, 512>>>(buf[1], s / 16, out[0]);
        else store_then_fence<3><<<1, 512>>>(buf[1], s / 16, out[0]);
        unsigned long long ns;
        CK(cudaMemcpy(&ns, out[0], 8, cudaMemcpyDeviceToHost));
        if (ns < best) best = ns;
      }
      std::printf("%-22s after %8ld B remote stores: %.3f us\n", fn[f], s, best / 1e3);
    }
  return 0;
}
