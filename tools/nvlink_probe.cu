// NVLink 5 peer-memory micro-benchmark (design probe, not part of the product).
// One process, two GPUs with peer access; kernels on both devices run
// concurrently (they never wait on each other).  Reports GB/s per direction
// for pull (remote LDG -> local STG), push (local LDG -> remote STG), both
// directions at once, and the fused N=2 pattern (remote+local LDG, add,
// local+remote STG), for several CTA counts / unroll depths.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvlink_probe tools/nvlink_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e = (x);                                                                  \
    if (e != cudaSuccess) {                                                               \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      std::exit(1);                                                                       \
    }                                                                                     \
  } while (0)

template <int U, int MODE>
__global__ void copy_k(int4* __restrict__ dst, const int4* __restrict__ src, long n) {
  // MODE 0: ld.cg ; MODE 1: default ld ; MODE 2: ld.nc.L1::no_allocate
  const long stride = (long)gridDim.x * blockDim.x * U;
  for (long base = (long)blockIdx.x * blockDim.x * U + threadIdx.x; base < n; base += stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long i = base + (long)u * blockDim.x;
      if (i < n) {
        if (MODE == 0)
          v[u] = __ldcg(src + i);
        else if (MODE == 1)
          v[u] = src[i];
        else
          asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                       : "l"(src + i));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long i = base + (long)u * blockDim.x;
      if (i < n) dst[i] = v[u];
    }
  }
}

// fused N=2: out = a(local) + b(remote) written to local and remote
template <int U>
__global__ void fold2_k(float4* la, const float4* rb, float4* rdst, long n) {
  const long stride = (long)gridDim.x * blockDim.x * U;
  for (long base = (long)blockIdx.x * blockDim.x * U + threadIdx.x; base < n; base += stride) {
    float4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long i = base + (long)u * blockDim.x;
      if (i < n) {
        a[u] = __ldcg(la + i);
        b[u] = __ldcg(rb + i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long i = base + (long)u * blockDim.x;
      if (i < n) {
        float4 r = make_float4(b[u].x + a[u].x, b[u].y + a[u].y, b[u].z + a[u].z, b[u].w + a[u].w);
        la[i] = r;
        rdst[i] = r;
      }
    }
  }
}

typedef void (*launcher)(int4*, const int4*, long, int, int, cudaStream_t);

template <int U, int MODE>
void launch_copy(int4* d, const int4* s, long n, int blocks, int threads, cudaStream_t st) {
  copy_k<U, MODE><<<blocks, threads, 0, st>>>(d, s, n);
}

int main(int argc, char** argv) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    std::printf("need 2 GPUs\n");
    return 0;
  }
  const size_t bytes = (argc > 1) ? std::atol(argv[1]) : (size_t)51200000;
  const long n = bytes / 16;
  int4 *buf[2], *buf2[2];
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&buf[d], bytes));
    CK(cudaMalloc(&buf2[d], bytes));
    CK(cudaMemset(buf[d], 1, bytes));
    CK(cudaMemset(buf2[d], 2, bytes));
    CK(cudaStreamCreate(&st[d]));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  struct Cfg {
    const char* name;
    launcher fn;
  };
  Cfg cfgs[] = {{"cg_U1", launch_copy<1, 0>}, {"cg_U4", launch_copy<4, 0>}, {"cg_U8", launch_copy<8, 0>},
                {"def_U4", launch_copy<4, 1>}, {"nc_U4", launch_copy<4, 2>}, {"nc_U8", launch_copy<8, 2>}};
  int grids[] = {148, 296, 592};
  int threads_opts[] = {256, 512, 1024};
  std::printf("bytes=%zu\n", bytes);
  std::printf("%-8s %-6s %-7s %-5s  %10s %10s %10s %10s\n", "kernel", "grid", "threads", "", "pull_1dir", "push_1dir",
              "pull_bidi", "push_bidi");
  for (auto& c : cfgs)
    for (int g : grids)
      for (int t : threads_opts) {
        float res[4];
        for (int pat = 0; pat < 4; ++pat) {
          const bool push = pat & 1, bidi = pat & 2;
          float best = 1e30f;
          for (int rep = 0; rep < 4; ++rep) {
            for (int d = 0; d < (bidi ? 2 : 1); ++d) {
              CK(cudaSetDevice(d));
              int4* dst = push ? buf[1 - d] : buf2[d];
              const int4* src = push ? buf2[d] : buf[1 - d];
              CK(cudaEventRecord(e0[d], st[d]));
              c.fn(dst, src, n, g, t, st[d]);
              CK(cudaEventRecord(e1[d], st[d]));
            }
            float worst = 0;
            for (int d = 0; d < (bidi ? 2 : 1); ++d) {
              CK(cudaSetDevice(d));
              CK(cudaEventSynchronize(e1[d]));
              float ms;
              CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
              if (ms > worst) worst = ms;
            }
            if (rep && worst < best) best = worst;
          }
          res[pat] = bytes / (best * 1e-3) / 1e9;
        }
        std::printf("%-8s %-6d %-7d %-5s  %10.1f %10.1f %10.1f %10.1f\n", c.name, g, t, "", res[0], res[1], res[2],
                    res[3]);
      }
  // fused N=2 pattern on both GPUs simultaneously
  for (int g : grids)
    for (int t : threads_opts) {
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        const long half = n / 2;
        for (int d = 0; d < 2; ++d) {
          CK(cudaSetDevice(d));
          float4* la = (float4*)buf[d] + d * half;
          const float4* rb = (const float4*)buf[1 - d] + d * half;
          float4* rd = (float4*)buf[1 - d] + d * half;
          CK(cudaEventRecord(e0[d], st[d]));
          fold2_k<2><<<g, t, 0, st[d]>>>(la, rb, rd, half);
          CK(cudaEventRecord(e1[d], st[d]));
        }
        float worst = 0;
        for (int d = 0; d < 2; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventSynchronize(e1[d]));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
          if (ms > worst) worst = ms;
        }
        if (rep && worst < best) best = worst;
      }
      // bus bytes per GPU for an N=2 allreduce of `bytes`: S
      std::printf("fold2    %-6d %-7d busbw=%8.1f GB/s (%.1f us)\n", g, t, bytes / (best * 1e-3) / 1e9, best * 1e3);
    }
  return 0;
}
