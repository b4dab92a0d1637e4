// NVLink 5 payload ceiling on this box (design probe, not product).
//
// What a bit-exact allreduce needs from the links: every GPU must bring in
// 2(N-1)/N * S bytes of peer data (raw inputs for its fold + the peers'
// results) and, symmetrically, send as much.  So its bus bandwidth is capped
// by the per-direction PAYLOAD rate the links sustain while both directions
// are busy.  This probe measures that rate for every way the SMs / TMA / copy
// engines can move the bytes, at sizes large enough that launch costs vanish:
//
//   pattern   1dir  : GPU 0 moves B bytes to/from its peers, the others idle
//             bidi  : every GPU moves B bytes (spread over its G-1 peers)
//   engine    ldg   : remote LDG.128 -> local STG.128            (pull)
//             stg   : local LDG.128 -> remote STG.128            (push)
//             mix   : half of B pulled, half pushed               (FUSED pattern, no math)
//             bulk_ld / bulk_st : cp.async.bulk (TMA engine) peer->smem->local / local->smem->peer
//             ce    : cudaMemcpyPeerAsync on one stream per peer  (copy engines)
//
// Output: one JSON line per (engine, pattern, bytes, launch shape); GB/s is
// B / max-over-GPUs event time, i.e. payload per direction per GPU.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvlink_ceiling tools/nvlink_ceiling.cu
//   tools/nvlink_ceiling [ngpus] [MiB...]
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e = (x);                                                                  \
    if (e != cudaSuccess) {                                                               \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      std::exit(1);                                                                       \
    }                                                                                     \
  } while (0)

constexpr int MAXG = 8;

struct Pairs {  // per GPU: G-1 (src, dst) pointer pairs of `n` int4 each
  const int4* src[MAXG];
  int4* dst[MAXG];
  long n;
  int np;
};

__device__ __forceinline__ int4 ldcg(const int4* p) {
  int4 v;
  asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// grid-stride copy over all pairs, U 16-byte loads in flight per thread.  The pairs are
// INTERLEAVED (vector i of the job belongs to pair i % np): at every moment every CTA
// talks to every peer, as the allreduce kernels do.  (A blocked layout, pair = i / n,
// makes all SMs of every GPU target the same peer at once: with 4 GPUs three of them
// then converge on one destination and the measured rate halves.)
template <int U>
__global__ void __launch_bounds__(512) copy_pairs(const __grid_constant__ Pairs P) {
  const long np = P.np;
  const long total = P.n * np;
  const long stride = (long)gridDim.x * blockDim.x * U;
  for (long base = (long)blockIdx.x * blockDim.x * U + threadIdx.x; base < total; base += stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long i = base + (long)u * blockDim.x;
      if (i < total) v[u] = ldcg(P.src[i % np] + i / np);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long i = base + (long)u * blockDim.x;
      if (i < total) __stcg(P.dst[i % np] + i / np, v[u]);
    }
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// TMA bulk copy src -> smem -> dst, TILE bytes per stage, STAGES in flight, one
// issuing thread per CTA; tiles dealt round-robin over CTAs across all pairs
template <int TILE, int STAGES>
__global__ void bulk_pairs(const __grid_constant__ Pairs P) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < STAGES; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const long tiles_per = P.n * 16 / TILE;
  const long total = tiles_per * P.np;
  uint32_t phase = 0;  // bit s = parity of stage s
  long t = blockIdx.x;
  int s = 0;
  for (; t < total; t += gridDim.x) {
    const int p = (int)(t % P.np);  // interleaved over the peers (see copy_pairs)
    const long off = (t / P.np) * TILE;
    // stage s free once its previous store has read it
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(STAGES - 1) : "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "n"(TILE) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sm + s * TILE)),
                 "l"(reinterpret_cast<const char*>(P.src[p]) + off), "n"(TILE), "r"(smem_u32(&bar[s]))
                 : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
                   : "=r"(ok)
                   : "r"(smem_u32(&bar[s])), "r"((phase >> s) & 1u)
                   : "memory");
    phase ^= 1u << s;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                     reinterpret_cast<char*>(P.dst[p]) + off),
                 "r"(smem_u32(sm + s * TILE)), "n"(TILE)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    s = (s + 1) % STAGES;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  int nd = 0;
  CK(cudaGetDeviceCount(&nd));
  int G = argc > 1 ? std::atoi(argv[1]) : nd;
  if (G > nd) G = nd;
  if (G < 2) {
    std::printf("{\"error\": \"needs 2 GPUs\"}\n");
    return 0;
  }
  std::vector<long> sizes_mib;
  for (int i = 2; i < argc; ++i) sizes_mib.push_back(std::atol(argv[i]));
  if (sizes_mib.empty()) sizes_mib = {256, 1024};
  const long maxB = sizes_mib.back() << 20;
  // per GPU: `in` (what peers read), `out` (where peers write / local results)
  char *in[MAXG], *out[MAXG];
  cudaStream_t st[MAXG][MAXG];
  cudaEvent_t e0[MAXG], e1[MAXG];
  for (int d = 0; d < G; ++d) {
    CK(cudaSetDevice(d));
    for (int q = 0; q < G; ++q)
      if (q != d) {
        const cudaError_t pe = cudaDeviceEnablePeerAccess(q, 0);
        if (pe == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError(); else CK(pe);
      }
    CK(cudaMalloc(&in[d], maxB));
    CK(cudaMalloc(&out[d], 2 * maxB));  // [0, maxB): pulled into; [maxB, 2 maxB): pushed into
    CK(cudaMemset(in[d], 1, maxB));
    CK(cudaMemset(out[d], 2, 2 * maxB));
    for (int q = 0; q < G; ++q) CK(cudaStreamCreateWithFlags(&st[d][q], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
    CK(cudaFuncSetAttribute(bulk_pairs<16384, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 8));
    CK(cudaFuncSetAttribute(bulk_pairs<32768, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 4));
    CK(cudaFuncSetAttribute(bulk_pairs<65536, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 * 3));
  }
  for (int d = 0; d < G; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceSynchronize());
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));

  // pairs of GPU d moving B bytes: pull = peers' `in` -> own `out`; push = own `in` -> peers' `out`
  // (regions disjoint per (reader, writer) so nothing is written twice)
  auto pairs = [&](int d, long B, bool push, long lo_frac_num, long lo_frac_den) {
    Pairs P;
    P.np = G - 1;
    const long per = B / (G - 1) / 16 / 1024 * 1024;  // int4, multiple of 1024 vectors
    P.n = per * lo_frac_num / lo_frac_den / 1024 * 1024;
    int k = 0;
    for (int q = 0; q < G; ++q) {
      if (q == d) continue;
      const long slot = (long)k * per * 16;
      if (!push) {
        P.src[k] = reinterpret_cast<const int4*>(in[q] + slot);
        P.dst[k] = reinterpret_cast<int4*>(out[d] + slot);
      } else {
        const int kk = d < q ? d : d - 1;  // d's slot index as seen from q
        P.src[k] = reinterpret_cast<const int4*>(in[d] + slot);
        P.dst[k] = reinterpret_cast<int4*>(out[q] + maxB + (long)kk * per * 16);
      }
      ++k;
    }
    return P;
  };

  auto time_it = [&](bool all, const std::function<void(int)>& go) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      const int act = all ? G : 1;
      for (int d = 0; d < act; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventRecord(e0[d], st[d][0]));
        for (int q = 1; q < G; ++q) CK(cudaStreamWaitEvent(st[d][q], e0[d], 0));
      }
      for (int d = 0; d < act; ++d) {
        CK(cudaSetDevice(d));
        go(d);
        CK(cudaGetLastError());
      }
      float worst = 0;
      for (int d = 0; d < act; ++d) {
        CK(cudaSetDevice(d));
        for (int q = 1; q < G; ++q) {  // join the per-peer streams
          cudaEvent_t j;
          CK(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
          CK(cudaEventRecord(j, st[d][q]));
          CK(cudaStreamWaitEvent(st[d][0], j, 0));
          CK(cudaEventDestroy(j));
        }
        CK(cudaEventRecord(e1[d], st[d][0]));
      }
      for (int d = 0; d < act; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(e1[d]));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
        worst = ms > worst ? ms : worst;
      }
      if (rep && worst < best) best = worst;
    }
    return best;
  };

  auto emit = [&](const char* engine, const char* pattern, long B, const std::string& shape, float ms) {
    std::printf("{\"probe\": \"nvlink_ceiling\", \"gpus\": %d, \"engine\": \"%s\", \"pattern\": \"%s\", \"bytes_per_dir\": %ld, "
                "\"shape\": \"%s\", \"ms\": %.4f, \"gbs_per_dir\": %.1f}\n",
                G, engine, pattern, B, shape.c_str(), ms, B / (ms * 1e-3) / 1e9);
    std::fflush(stdout);
  };

  for (long mib : sizes_mib) {
    const long B = mib << 20;
    for (int all = 0; all < 2; ++all) {
      const char* pat = all ? "bidi" : "1dir";
      // SM engines: grid x threads, U loads in flight
      // PROBE_FEW_CTAS=1: small grids (how much one SM can move: collectives overlapping compute)
      const bool few = std::getenv("PROBE_FEW_CTAS") != nullptr;
      std::vector<int> grids = few ? std::vector<int>{16, 32, 64} : std::vector<int>{sms, 2 * sms, 4 * sms};
      for (int g : grids) {
        for (int mode = 0; mode < 3; ++mode) {  // 0 pull, 1 push, 2 mix
          const char* eng = mode == 0 ? "ldg" : mode == 1 ? "stg" : "mix";
          float ms = time_it(all, [&](int d) {
            if (mode < 2) {
              Pairs P = pairs(d, B, mode == 1, 1, 1);
              copy_pairs<8><<<g, 512, 0, st[d][0]>>>(P);
            } else {  // half pulled, half pushed, concurrently on two streams
              Pairs A = pairs(d, B, false, 1, 2), Bp = pairs(d, B, true, 1, 2);
              copy_pairs<8><<<g / 2, 512, 0, st[d][0]>>>(A);
              copy_pairs<8><<<g / 2, 512, 0, st[d][1]>>>(Bp);
            }
          });
          emit(eng, pat, B, std::to_string(g) + "x512 U8", ms);
        }
      }
      // TMA bulk
      for (int push = 0; push < 2; ++push) {
        struct BC { int tile, stages, grid; };
        std::vector<BC> bcs = few ? std::vector<BC>{{32768, 4, 16}, {65536, 3, 16}, {32768, 4, 32}, {65536, 3, 32},
                                                    {32768, 4, 64}}
                                  : std::vector<BC>{{16384, 8, sms}, {32768, 4, sms}, {65536, 3, sms}, {32768, 4, 2 * sms}};
        for (const BC& c : bcs) {
          float ms = time_it(all, [&](int d) {
            Pairs P = pairs(d, B, push, 1, 1);
            const size_t smem = (size_t)c.tile * c.stages;
            if (c.tile == 16384) bulk_pairs<16384, 8><<<c.grid, 32, smem, st[d][0]>>>(P);
            else if (c.tile == 32768) bulk_pairs<32768, 4><<<c.grid, 32, smem, st[d][0]>>>(P);
            else bulk_pairs<65536, 3><<<c.grid, 32, smem, st[d][0]>>>(P);
          });
          emit(push ? "bulk_st" : "bulk_ld", pat, B,
               "tile " + std::to_string(c.tile) + " x" + std::to_string(c.stages) + " grid " + std::to_string(c.grid), ms);
        }
      }
      // copy engines: one stream per peer, pull (dst local) and push (dst peer)
      for (int push = 0; push < 2; ++push) {
        float ms = time_it(all, [&](int d) {
          Pairs P = pairs(d, B, push, 1, 1);
          for (int k = 0; k < P.np; ++k)
            CK(cudaMemcpyAsync(P.dst[k], P.src[k], P.n * 16, cudaMemcpyDeviceToDevice, st[d][k == 0 ? 0 : k]));
        });
        emit(push ? "ce_push" : "ce_pull", pat, B, "1 stream per peer", ms);
      }
    }
  }
  return 0;
}
