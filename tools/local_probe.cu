// HBM probe for the 1-GPU local-reduce pattern (design probe, not product):
// V=8 source buffers, one owned region per "rank", every element read from all
// 8 buffers and the folded value written to all 8.  Compares cache-operator
// variants against a plain copy (the MEASURED_PEAKS denominator).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o local_probe tools/local_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));       \
      std::exit(1);                                                                        \
    }                                                                                      \
  } while (0)

struct Ptrs {
  float4* b[8];
};

template <int LD, int ST>
__device__ __forceinline__ float4 ld(const float4* p) {
  if (LD == 0) return __ldcg(p);
  if (LD == 1) return *p;
  if (LD == 2) return __ldcs(p);
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
template <int ST>
__device__ __forceinline__ void st(float4* p, float4 v) {
  if (ST == 0) __stcg(p, v);
  else if (ST == 1) *p = v;
  else __stcs(p, v);
}

template <int LD, int ST, bool TILED>
__global__ void __launch_bounds__(512) fold8(Ptrs P, long nvec) {
  const long nthr = (long)gridDim.x * blockDim.x;
  const long tile = 1024;
  auto body = [&](long i) {
    float4 x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = ld<LD, ST>(P.b[j] + i);
    float4 a = x[0], c = x[2], e = x[4], g = x[6];
    a.x += x[1].x; a.y += x[1].y; a.z += x[1].z; a.w += x[1].w;
    c.x += x[3].x; c.y += x[3].y; c.z += x[3].z; c.w += x[3].w;
    e.x += x[5].x; e.y += x[5].y; e.z += x[5].z; e.w += x[5].w;
    g.x += x[7].x; g.y += x[7].y; g.z += x[7].z; g.w += x[7].w;
    a.x += c.x; a.y += c.y; a.z += c.z; a.w += c.w;
    e.x += g.x; e.y += g.y; e.z += g.z; e.w += g.w;
    a.x += e.x; a.y += e.y; a.z += e.z; a.w += e.w;
#pragma unroll
    for (int j = 0; j < 8; ++j) st<ST>(P.b[j] + i, a);
  };
  if (TILED) {
    for (long t = blockIdx.x; t * tile < nvec; t += gridDim.x)
      for (long i = t * tile + threadIdx.x; i < (t + 1) * tile && i < nvec; i += blockDim.x) body(i);
  } else {
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += nthr) body(i);
  }
}

__global__ void copyk(float4* d, const float4* s, long n) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) d[i] = s[i];
}

int main() {
  const long n = 25600000;  // floats per rank
  const long nvec = n / 4;
  Ptrs P;
  for (int j = 0; j < 8; ++j) {
    CK(cudaMalloc(&P.b[j], n * 4));
    CK(cudaMemset(P.b[j], 0, n * 4));
  }
  float* flush;
  CK(cudaMalloc(&flush, 256 << 20));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto timeit = [&](auto fn, double bytes, const char* name) {
    float best = 1e9, sum = 0;
    for (int r = 0; r < 12; ++r) {
      CK(cudaMemset(flush, r, 256 << 20));
      CK(cudaEventRecord(a));
      fn();
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      if (r >= 2) {
        sum += ms;
        if (ms < best) best = ms;
      }
    }
    std::printf("%-34s best %8.1f us  mean %8.1f us  %7.1f GB/s (best)\n", name, best * 1e3, sum / 10 * 1e3,
                bytes / (best * 1e-3) / 1e9);
  };
  const double bytes = 16.0 * n * 4;
  int grids[] = {148, 296, 592, 1184};
  for (int g : grids) {
    char nm[64];
    std::snprintf(nm, 64, "copy grid=%d", g);
    timeit([&] { copyk<<<g, 512>>>(P.b[1], P.b[0], nvec); }, 2.0 * n * 4, nm);
  }
  for (int g : grids) {
    char nm[64];
    std::snprintf(nm, 64, "fold8 cg/cg grid=%d", g);
    timeit([&] { fold8<0, 0, false><<<g, 512>>>(P, nvec); }, bytes, nm);
    std::snprintf(nm, 64, "fold8 cg/cg tiled grid=%d", g);
    timeit([&] { fold8<0, 0, true><<<g, 512>>>(P, nvec); }, bytes, nm);
    std::snprintf(nm, 64, "fold8 def/def grid=%d", g);
    timeit([&] { fold8<1, 1, false><<<g, 512>>>(P, nvec); }, bytes, nm);
    std::snprintf(nm, 64, "fold8 cg/cs grid=%d", g);
    timeit([&] { fold8<0, 2, false><<<g, 512>>>(P, nvec); }, bytes, nm);
    std::snprintf(nm, 64, "fold8 nc/cs grid=%d", g);
    timeit([&] { fold8<3, 2, false><<<g, 512>>>(P, nvec); }, bytes, nm);
    std::snprintf(nm, 64, "fold8 cs/cs grid=%d", g);
    timeit([&] { fold8<2, 2, false><<<g, 512>>>(P, nvec); }, bytes, nm);
  }
  return 0;
}
