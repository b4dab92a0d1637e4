/*
 * rbx.h -- C ABI of the B200-native multi-ring allreduce (librbx.so).
 *
 * This is the drop-in boundary for the reference `ringbox` hot path
 * (/root/reference/pkg/src/ringbox).  The reference exposes a Python API and no
 * FFI; each entry point below states which reference interface it replaces.
 * Plain pointers and sizes only: no torch types cross this ABI.  Every
 * function returns an rbx status code, never throws, and records a
 * thread-local message readable with rbx_last_error().
 *
 * Device buffers passed to the collectives must be SYMMETRIC: registered on
 * every rank with rbx_register_buffer() (or allocated with
 * rbx_alloc_symmetric() and registered), used at the same byte offset and
 * element count on every rank.  There is no host or NCCL fallback: an
 * unregistered buffer is an error.
 */
#ifndef RBX_H_
#define RBX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RBX_ABI_VERSION 1

/* status codes */
#define RBX_OK 0
#define RBX_ERR_INVALID 1     /* bad argument: maps to ValueError (multiring.py:165-166, runtime.py:74-77) */
#define RBX_ERR_CUDA 2        /* CUDA runtime failure */
#define RBX_ERR_COLLECTIVE 3  /* peer lost / timeout: maps to CollectiveError(rank, phase) (runtime.py:42-48) */
#define RBX_ERR_UNSUPPORTED 4 /* dtype/mode combination not implemented */

/* dtypes: the reference's {f32, f64, i64} (runtime.py:37) plus bf16/f16 (fp32 accumulate) and i32 */
#define RBX_F32 0
#define RBX_F64 1
#define RBX_I64 2
#define RBX_BF16 3
#define RBX_F16 4
#define RBX_I32 5

/* execution modes (all produce bit-identical results) */
#define RBX_MODE_AUTO 0       /* LL for a whole-buffer allreduce of <= RBX_LL_AUTO_BYTES (env, default
                                 1 MiB) on a multi-GPU communicator, else FUSED */
#define RBX_MODE_RING_DIMS 1  /* one reduce-scatter / all-gather stage per grid dimension (the paper's rings) */
#define RBX_MODE_FUSED 2      /* all dims folded in one pass (nested order), result pushed to every peer */
#define RBX_MODE_FUSED_PULL 3 /* like FUSED, but the all-gather pulls the peers' owned chunks */
#define RBX_MODE_LOCAL 4      /* virtual ranks on one GPU, no synchronisation (1-GPU roofline) */
#define RBX_MODE_PUSH 5       /* two-shot, NVLink writes only: inputs pushed to the owners' inboxes
                                 (rbx_set_inbox), results pushed back to every rank */
#define RBX_MODE_LL 6         /* low latency, allreduce of <= 1 MiB per rank: 8-byte {data, epoch} words
                                 pushed into the communicator's LL area, no flags or fences */

/* collective ops */
#define RBX_OP_ALLREDUCE 0
#define RBX_OP_REDUCE_SCATTER 1
#define RBX_OP_ALLGATHER 2
#define RBX_OP_BARRIER 3

typedef struct rbx_comm rbx_comm_t;
typedef struct {
  unsigned char bytes[64]; /* cudaIpcMemHandle_t */
} rbx_ipc_handle_t;

int rbx_version(void);
/* Message of the last failed call on this thread; *rank / *stage receive the
 * failing peer rank and plan step for RBX_ERR_COLLECTIVE (else -1). */
const char *rbx_last_error(int *rank, int *stage);

/* ---- host-only planning (no GPU needed) ---- */
/* ring.chunk_bounds -- pkg/src/ringbox/ring.py:57-70 */
int rbx_chunk_bounds(int64_t count, int64_t n_chunks, int64_t index, int64_t *off, int64_t *len);
/* runtime.owned_region -- pkg/src/ringbox/runtime.py:187-196 */
int rbx_owned_region(const int *dims, int ndims, int rank, int64_t count, int64_t *off, int64_t *len);
/* Rank order in which the reference schedule (multiring.py:170-211) folds `rank`'s owned region. */
int rbx_fold_order(const int *dims, int ndims, int rank, int *order_out);
/* Flattened step table of `rank` for inspection (see paper_1708_02188_b200/_native.py). Returns the
 * number of int64 words (may exceed cap; nothing is written past cap), or -1. */
int64_t rbx_plan_describe(const int *dims, int ndims, int rank, int64_t count, int op, int mode, int dtype,
                          int64_t *out, int64_t cap);

/* ---- devices and symmetric memory ---- */
int rbx_device_count(int *n);
/* Single-process use of several GPUs (virtual ranks on distinct devices, profiling harnesses):
 * lets `device` load/store `peer`'s memory directly over NVLink. */
int rbx_enable_peer_access(int device, int peer);
/* PlacedBuffer(memory="device") storage (runtime.py:51-69): cudaMalloc + IPC export. */
int rbx_alloc_symmetric(int device, size_t bytes, void **ptr, rbx_ipc_handle_t *handle);
int rbx_free(void *ptr);
/* IPC handle + byte offset of any cudaMalloc'd pointer (e.g. a torch tensor). */
int rbx_export_buffer(void *ptr, rbx_ipc_handle_t *handle, uint64_t *offset);

/* ---- communicator: replaces RankContext + peer sockets (runtime.py:159-184, 348-386) ---- */
/* Phase 1: allocate this rank's signal area; returns its IPC handle for exchange. */
int rbx_comm_create(rbx_comm_t **comm, int rank, int nranks, const int *dims, int ndims, int device,
                    int nblocks, int threads, rbx_ipc_handle_t *signal_handle);
/* Phase 2: map every peer's signal area (handles indexed by rank). */
int rbx_comm_connect(rbx_comm_t *comm, const rbx_ipc_handle_t *signal_handles);
int rbx_comm_destroy(rbx_comm_t *comm);
int rbx_comm_set_timeout(rbx_comm_t *comm, double seconds);
int rbx_comm_info(rbx_comm_t *comm, int *rank, int *nranks, int *nblocks, int *threads, uint64_t *launches);
/* Fault injection (the reference's Workload.crash_rank/crash_phase, runtime.py:393-394, 429-432): the
 * NEXT collective launch of this communicator processes only `fraction` of its first data step (for
 * MODE_LL: fraction > 0 = the scatter half) and then returns without signalling, as a rank that dies
 * mid-collective with part of its data pushed.  The caller then exits; peers' watchdogs report it. */
int rbx_comm_inject_fault(rbx_comm_t *comm, double fraction);
/* Timeline of the last launch (RBX_TRACE=1 at create): %globaltimer ns of the first (words 0..31) and
 * last (32..63) CTA: 0 start, 1 plan staged, 2 entry signalled, 3+3s/4+3s/5+3s step s waited/worked/
 * signalled, 30 steps done, 31 exit.  Tracing / profiling subsystem. */
int rbx_comm_trace(rbx_comm_t *comm, uint64_t *out, int cap);
/* Which kernel ran this communicator's last collective (RBX_KERNEL_*): the evidence that a call took a
 * specialised path and not the generic step interpreter. */
#define RBX_KERNEL_NONE 0
#define RBX_KERNEL_STEP 1   /* rbx_step_kernel: the generic step-table interpreter */
#define RBX_KERNEL_FUSED 2  /* rbx_fused_kernel: FUSED allreduce / reduce-scatter / all-gather */
#define RBX_KERNEL_RINGS 3  /* rbx_rings_kernel: RING_DIMS / PUSH with per-CTA matched stages */
#define RBX_KERNEL_LL 4     /* rbx_ll_kernel: small messages, {data, epoch} words */
#define RBX_KERNEL_LOCAL 5  /* rbx_local_kernel: all ranks on one GPU (MODE_LOCAL) */
int rbx_comm_last_kernel(rbx_comm_t *comm, int *kind);
/* Page-lock host memory in place (PlacedBuffer(numpy) staging, hoststage.py): copies from / to it then
 * run at the host link's DMA rate.  Memory that is already page-locked is not an error; *registered
 * (optional) is 1 only if this call registered it (then rbx_host_unregister releases it). */
int rbx_host_register(void *ptr, size_t bytes, int *registered);
int rbx_host_unregister(void *ptr);
/* Diagnostic: a 1-thread kernel on `stream` that writes the device's %globaltimer (ns, the clock of
 * rbx_comm_trace) to the device word *dst -- brackets a collective on the device clock. */
int rbx_stamp(uint64_t *dst, void *stream);
/* Profiling harness: `rank`'s share of a FUSED allreduce of bufs[0..N) (any GPUs with peer access from
 * the current device) through the specialised kernel with the flag protocol off, on the current device.
 * Single process, no peer ever waits: ncu can replay it (it must never wrap a multi-rank run). */
int rbx_fused_harness(const int *dims, int ndims, int rank, void *const *bufs, size_t count, int dtype, int nblocks,
                      int threads, void *stream);
/* Collective registration: every rank passes its own (ptr, bytes) and all ranks' handles/offsets. */
int rbx_register_buffer(rbx_comm_t *comm, void *ptr, size_t bytes, const rbx_ipc_handle_t *handles,
                        const uint64_t *offsets, int *buf_id);

/* This process's mapping of `rank`'s copy of the registered buffer that contains `buf` (same byte
 * offset): the symmetric-memory view, for callers that move data between ranks themselves (e.g. the
 * bench's copy-engine ceiling measurement). */
int rbx_peer_pointer(rbx_comm_t *comm, const void *buf, int rank, void **out);

/* MODE_PUSH scratch: bytes of symmetric inbox the given buffers need (host-only), and the collective
 * registration of this rank's inbox (handles/offsets of every rank, like rbx_register_buffer). */
int64_t rbx_inbox_bytes(const int *dims, int ndims, const size_t *counts, int nbufs, int dtype);
int rbx_set_inbox(rbx_comm_t *comm, void *ptr, size_t bytes, const rbx_ipc_handle_t *handles,
                  const uint64_t *offsets);

/* ---- collectives (asynchronous on `stream`, a cudaStream_t or NULL) ---- */
/* runtime.allreduce(ctx, obj) -- pkg/src/ringbox/runtime.py:295-297 */
int rbx_allreduce(rbx_comm_t *comm, void *buf, size_t count, int dtype, int mode, void *stream);
/* runtime.reduce_scatter(ctx, obj) -> owned view -- runtime.py:278-284 */
int rbx_reduce_scatter(rbx_comm_t *comm, void *buf, size_t count, int dtype, int mode, void *stream,
                       int64_t *owned_off, int64_t *owned_len);
/* runtime.allgather(ctx, obj) -- runtime.py:287-292 */
int rbx_allgather(rbx_comm_t *comm, void *buf, size_t count, int dtype, int mode, void *stream);
/* One launch over a bucket list; Workload.lengths semantics (runtime.py:82-91, 390-398), buckets concurrent. */
int rbx_allreduce_buckets(rbx_comm_t *comm, void *const *bufs, const size_t *counts, int nbufs, int dtype,
                          int mode, void *stream);
/* Allreduce of the element window [lo, hi) of a count-element buffer with the FULL buffer's chunk
 * geometry and reduction order (bit-identical to those elements of rbx_allreduce). Lets callers
 * pipeline H2D / reduce / D2H or reduce a bucket as its gradients become ready. */
int rbx_allreduce_window(rbx_comm_t *comm, void *buf, size_t count, size_t lo, size_t hi, int dtype, int mode,
                         void *stream);
/* Device-side flag barrier across all ranks (no data). */
int rbx_barrier(rbx_comm_t *comm, void *stream);
/* After the stream has been synchronised: RBX_ERR_COLLECTIVE if a watchdog fired. */
int rbx_check(rbx_comm_t *comm);

/* ---- virtual ranks on ONE GPU (single launch; cooperative when ranks synchronise) ---- */
int rbx_vcomm_create(rbx_comm_t **comm, int nranks, const int *dims, int ndims, int device, int nblocks_per_rank,
                     int threads);
/* bufs[r] = rank r's device buffer.  mode RBX_MODE_LOCAL = the 1-GPU local reduce (no flags). */
int rbx_vcollective(rbx_comm_t *comm, void *const *bufs, size_t count, int dtype, int op, int mode, void *stream);
int rbx_vcollective_window(rbx_comm_t *comm, void *const *bufs, size_t count, size_t lo, size_t hi, int dtype, int op,
                           int mode, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* RBX_H_ */
