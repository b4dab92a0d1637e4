// Launch-latency probe (design probe, not product): how long from a 1-thread
// "stamp" kernel's %globaltimer to the first CTA of the next kernel starting,
// and what does the launch shape change?  One GPU.  Variants:
//   tiny      1 x 32 threads, 8 B of parameters
//   grid      148 x 512, 8 B of parameters
//   params4k  148 x 512, 4 KB __grid_constant__ parameters (the fused kernel carries ~0.7 KB,
//             the 16-segment form ~5 KB)
//   regs128   148 x 512, __launch_bounds__(512, 1), ~128 registers and a large body (not executed)
//   regs128+pdl  the same launched with programmatic stream serialization (cudaLaunchKernelEx)
// Printed: median / p10 of (first CTA start - stamp) and of CUDA-event time around the launch.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_probe tools/launch_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
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

__global__ void stamp(unsigned long long* out) { *out = now(); }

// every CTA records its start; the host takes the minimum
__global__ void k_small(unsigned long long* starts) {
  const unsigned long long t = now();
  if (threadIdx.x == 0) starts[blockIdx.x] = t;
}

template <int PADW>
struct Big {
  unsigned long long* starts;
  int pad[PADW];
};
template <int PADW>
__global__ void k_params(const __grid_constant__ Big<PADW> a) {
  const unsigned long long t = now();
  if (threadIdx.x == 0) a.starts[blockIdx.x] = t + (unsigned long long)a.pad[blockIdx.x % PADW] * 0ull;
}
// the same 4 KB of arguments in device memory, staged into shared memory by the CTA
__global__ void k_params_dev(const Big<1020>* __restrict__ g) {
  const unsigned long long t = now();
  __shared__ Big<1020> a;
  const int* src = reinterpret_cast<const int*>(g);
  int* dst = reinterpret_cast<int*>(&a);
  for (int i = threadIdx.x; i < (int)(sizeof(a) / 4); i += blockDim.x) dst[i] = src[i];
  __syncthreads();
  if (threadIdx.x == 0) a.starts[blockIdx.x] = t + (unsigned long long)a.pad[blockIdx.x % 1020] * 0ull;
}

// a large, register-hungry body behind a flag that is never set
__global__ void __launch_bounds__(512, 1) k_regs(unsigned long long* starts, const float4* src, float4* dst, int flag) {
  const unsigned long long t = now();
  if (threadIdx.x == 0) starts[blockIdx.x] = t;
  if (flag) {
    float4 v[24];
#pragma unroll
    for (int i = 0; i < 24; ++i) v[i] = src[threadIdx.x + i * 512];
#pragma unroll 1
    for (int it = 0; it < flag; ++it) {
#pragma unroll
      for (int i = 0; i < 24; ++i) {
        v[i].x = v[i].x * v[(i + 1) % 24].y + v[(i + 7) % 24].z;
        v[i].y = v[i].y * v[(i + 3) % 24].w + v[(i + 5) % 24].x;
        v[i].z = v[i].z * v[(i + 11) % 24].x + v[(i + 13) % 24].y;
        v[i].w = v[i].w * v[(i + 17) % 24].z + v[(i + 19) % 24].w;
      }
    }
#pragma unroll
    for (int i = 0; i < 24; ++i) dst[threadIdx.x + i * 512] = v[i];
  }
}

int main() {
  unsigned long long *ts, *starts;
  float4 *src, *dst;
  CK(cudaMalloc(&ts, 8));
  CK(cudaMalloc(&starts, 4096 * 8));
  CK(cudaMalloc(&src, 24 * 512 * 16));
  CK(cudaMalloc(&dst, 24 * 512 * 16));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t a, z;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&z));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, k_regs));
  std::printf("{\"k_regs_registers\": %d, \"k_regs_binary_bytes_approx\": %d}\n", fa.numRegs, (int)fa.maxThreadsPerBlock);
  Big<1020> big;
  std::memset(&big, 0, sizeof(big));
  big.starts = starts;
  Big<14> b64;
  Big<126> b512;
  Big<254> b1k;
  Big<510> b2k;
  Big<2046> b8k;
  std::memset(&b64, 0, sizeof(b64));
  std::memset(&b512, 0, sizeof(b512));
  std::memset(&b1k, 0, sizeof(b1k));
  std::memset(&b2k, 0, sizeof(b2k));
  std::memset(&b8k, 0, sizeof(b8k));
  b64.starts = b512.starts = b1k.starts = b2k.starts = b8k.starts = starts;
  Big<1020>* dbig;
  CK(cudaMalloc(&dbig, sizeof(big)));
  CK(cudaMemcpy(dbig, &big, sizeof(big), cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(k_params<2046>, cudaFuncAttributeMaxDynamicSharedMemorySize, 0));
  const char* names[] = {"tiny 1x32", "grid 148x512", "params4k 148x512", "regs128 148x512", "regs128+pdl 148x512",
                         "params64 148x512", "params512 148x512", "params1k 148x512", "params2k 148x512",
                         "params8k 148x512", "args4k in device memory, staged to smem 148x512"};
  for (int v = 0; v < 11; ++v) {
    std::vector<double> lat, ev;
    for (int i = 0; i < 220; ++i) {
      CK(cudaMemsetAsync(starts, 0xff, 4096 * 8, st));
      CK(cudaEventRecord(a, st));
      stamp<<<1, 1, 0, st>>>(ts);
      int nb = 148;
      if (v == 0) {
        nb = 1;
        k_small<<<1, 32, 0, st>>>(starts);
      } else if (v == 1) {
        k_small<<<148, 512, 0, st>>>(starts);
      } else if (v == 2) {
        k_params<<<148, 512, 0, st>>>(big);
      } else if (v == 3) {
        k_regs<<<148, 512, 0, st>>>(starts, src, dst, 0);
      } else if (v == 5) {
        k_params<<<148, 512, 0, st>>>(b64);
      } else if (v == 6) {
        k_params<<<148, 512, 0, st>>>(b512);
      } else if (v == 7) {
        k_params<<<148, 512, 0, st>>>(b1k);
      } else if (v == 8) {
        k_params<<<148, 512, 0, st>>>(b2k);
      } else if (v == 9) {
        k_params<<<148, 512, 0, st>>>(b8k);
      } else if (v == 10) {
        k_params_dev<<<148, 512, 0, st>>>(dbig);
      } else {
        cudaLaunchConfig_t cfg;
        std::memset(&cfg, 0, sizeof(cfg));
        cfg.gridDim = dim3(148);
        cfg.blockDim = dim3(512);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int zero = 0;
        CK(cudaLaunchKernelEx(&cfg, k_regs, starts, (const float4*)src, dst, zero));
      }
      CK(cudaEventRecord(z, st));
      CK(cudaEventSynchronize(z));
      unsigned long long h_ts, h_st[148];
      CK(cudaMemcpy(&h_ts, ts, 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(h_st, starts, nb * 8, cudaMemcpyDeviceToHost));
      unsigned long long first = *std::min_element(h_st, h_st + nb);
      unsigned long long last = *std::max_element(h_st, h_st + nb);
      float ms;
      CK(cudaEventElapsedTime(&ms, a, z));
      if (i >= 20) {
        lat.push_back((double)(first - h_ts) / 1e3);
        ev.push_back(ms * 1e3 + 0.0 * (double)(last - first));
      }
    }
    std::sort(lat.begin(), lat.end());
    std::sort(ev.begin(), ev.end());
    std::printf(
        "{\"variant\": \"%s\", \"stamp_to_first_cta_us_p50\": %.2f, \"p10\": %.2f, \"event_us_stamp_plus_kernel_p50\": %.2f}\n",
        names[v], lat[lat.size() / 2], lat[lat.size() / 10], ev[ev.size() / 2]);
    std::fflush(stdout);
  }
  // parameter-size sweep (bytes = 8 + 4 * PADW)
  auto sweep = [&](auto tag, int bytes) {
    constexpr int W = decltype(tag)::value;
    Big<W> b;
    std::memset(&b, 0, sizeof(b));
    b.starts = starts;
    std::vector<double> lat, ev;
    for (int i = 0; i < 220; ++i) {
      CK(cudaEventRecord(a, st));
      stamp<<<1, 1, 0, st>>>(ts);
      k_params<W><<<148, 512, 0, st>>>(b);
      CK(cudaEventRecord(z, st));
      CK(cudaEventSynchronize(z));
      unsigned long long h_ts, h_st[148];
      CK(cudaMemcpy(&h_ts, ts, 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(h_st, starts, 148 * 8, cudaMemcpyDeviceToHost));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, z));
      if (i >= 20) {
        lat.push_back((double)(*std::min_element(h_st, h_st + 148) - h_ts) / 1e3);
        ev.push_back(ms * 1e3);
      }
    }
    std::sort(lat.begin(), lat.end());
    std::sort(ev.begin(), ev.end());
    std::printf("{\"param_bytes\": %d, \"stamp_to_first_cta_us_p50\": %.2f, \"event_us_stamp_plus_kernel_p50\": %.2f}\n",
                bytes, lat[lat.size() / 2], ev[ev.size() / 2]);
    std::fflush(stdout);
  };
#define SWEEP(W) sweep(std::integral_constant<int, W>{}, 8 + 4 * W);
  SWEEP(638) SWEEP(766) SWEEP(894) SWEEP(1000) SWEEP(1020) SWEEP(1022) SWEEP(1024) SWEEP(1150) SWEEP(1238)
  SWEEP(1284) SWEEP(1534) SWEEP(2046) SWEEP(4094)
  return 0;
}
