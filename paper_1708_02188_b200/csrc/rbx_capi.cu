// C ABI (include/rbx.h): communicators, IPC-mapped symmetric memory, plan
// caching and kernel launch for the sm_100a multi-ring allreduce.
//
// Reference mapping (pkg/src/ringbox/runtime.py):
//   RankContext (159-184)         -> rbx_comm: rank, grid, peer signal areas, plan cache
//   peer sockets + handshake      -> cudaIpc-mapped peer buffers + signal areas (348-386)
//   schedule_for (174-177)        -> per (buffer, count, dtype, op, mode) device plan cache
//   _run_phases (199-267)         -> one launch of rbx_step_kernel<T>
//   CollectiveError (42-48)       -> RBX_ERR_COLLECTIVE + (rank, step) from the device watchdog
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "rbx.h"
#include "rbx_kernel.cuh"
#include "rbx_plan.h"

#include "rbx_fused.cuh"
#include "rbx_rings.cuh"
#include "rbx_local.cuh"
#include "rbx_ll.cuh"

namespace rbx {
const void* local_kernel_f32(int v, int nlev);
const void* local_kernel_f64(int v, int nlev);
const void* local_kernel_i64(int v, int nlev);
const void* local_kernel_bf16(int v, int nlev);
const void* local_kernel_f16(int v, int nlev);
const void* local_kernel_i32(int v, int nlev);
const void* step_kernel_f32();
const void* step_kernel_f64();
const void* step_kernel_i64();
const void* step_kernel_bf16();
const void* step_kernel_f16();
const void* step_kernel_i32();
const void* ll_kernel_f32(int maxv);
const void* ll_kernel_f64(int maxv);
const void* ll_kernel_i64(int maxv);
const void* ll_kernel_bf16(int maxv);
const void* ll_kernel_f16(int maxv);
const void* ll_kernel_i32(int maxv);
const void* fused_kernel_f32(int nsrc, int nlev, int ndst, int maxseg);
const void* fused_kernel_f64(int nsrc, int nlev, int ndst, int maxseg);
const void* fused_kernel_i64(int nsrc, int nlev, int ndst, int maxseg);
const void* fused_kernel_bf16(int nsrc, int nlev, int ndst, int maxseg);
const void* fused_kernel_f16(int nsrc, int nlev, int ndst, int maxseg);
const void* fused_kernel_i32(int nsrc, int nlev, int ndst, int maxseg);
const void* rings_kernel_f32();
const void* rings_kernel_f64();
const void* rings_kernel_i64();
const void* rings_kernel_bf16();
const void* rings_kernel_f16();
const void* rings_kernel_i32();
}  // namespace rbx

namespace {

// %globaltimer into *dst (diagnostic: brackets a collective on the device clock)
__global__ void stamp_kernel(uint64_t* dst) { *dst = rbx::global_ns(); }

thread_local std::string g_err;
thread_local int g_err_rank = -1, g_err_stage = -1;

int fail(int code, const std::string& msg, int rank = -1, int stage = -1) {
  g_err = msg;
  g_err_rank = rank;
  g_err_stage = stage;
  return code;
}

#define RBX_CUDA(call)                                                                          \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess) return fail(RBX_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

int dtype_size(int dt) {
  switch (dt) {
    case RBX_F32: return 4;
    case RBX_F64: return 8;
    case RBX_I64: return 8;
    case RBX_BF16: return 2;
    case RBX_F16: return 2;
    case RBX_I32: return 4;
    default: return 0;
  }
}

struct RegBuf {
  char* base = nullptr;  // local pointer as registered
  size_t bytes = 0;
  std::vector<char*> at;  // per rank: pointer to that rank's copy, valid in this process
};

struct CachedPlan {
  rbx::Plan* dev = nullptr;  // nplans contiguous plans
  void** ptrs = nullptr;
  int nplans = 0;
  int plan_bytes = 0;  // staged into shared memory by every CTA
  bool uses_inbox = false;
  const void* local_fn = nullptr;  // specialised MODE_LOCAL kernel (rbx_local.cuh), if the shape has one
  std::shared_ptr<rbx::LocalArgs> local_args;
  int local_grid = 0;
  // specialised FUSED allreduce kernel (rbx_fused.cuh), if the shape has one: arguments for
  // one segment (fused1) or a bucket list of up to RBX_FUSED_MAXSEG (fusedN)
  const void* fused_fn = nullptr;
  std::shared_ptr<rbx::FusedArgsT<1>> fused1;
  std::shared_ptr<rbx::FusedArgsT<RBX_FUSED_MAXSEG>> fusedN;
  // specialised RING_DIMS kernel (rbx_rings.cuh): one stage per grid dimension, matched waits
  const void* rings_fn = nullptr;
  std::shared_ptr<rbx::RingsArgs> rings;
};

struct LLKey {  // cached MODE_LL launch arguments: buffers, count, dtype
  std::vector<void*> bufs;
  size_t count;
  int dtype;
  bool operator<(const LLKey& o) const {
    if (count != o.count) return count < o.count;
    if (dtype != o.dtype) return dtype < o.dtype;
    return bufs < o.bufs;
  }
};

struct OpenedHandle {
  void* ptr = nullptr;
  int refs = 0;
};

}  // namespace

struct rbx_comm {
  int rank = 0, nranks = 1, device = 0, nblocks = 0, threads = 512;
  int nvirtual = 0;  // >0: all ranks hosted by this process on one GPU
  rbx::Geometry geo;
  uint32_t* sig_local = nullptr;     // own signal area(s)
  std::vector<uint32_t*> sig;        // per rank, mapped
  std::vector<void*> opened;  // base pointers of every IPC mapping this communicator opened (one ref each)
  rbx::ErrRecord* err_host = nullptr;
  rbx::ErrRecord* err_dev = nullptr;
  uint64_t timeout_ns = 30ull * 1000000000ull;  // runtime.py:39 DEFAULT_TIMEOUT_S
  std::vector<RegBuf> bufs;
  std::map<std::string, CachedPlan> plans;
  // Plans replaced while a CUDA graph may still reference them (a capture has used this
  // communicator): kept alive until rbx_comm_destroy instead of freed.
  std::vector<CachedPlan> retired;
  bool captured = false;  // some launch of this communicator was recorded into a CUDA graph
  std::vector<char*> retired_inboxes;  // virtual comms' own inboxes replaced after a capture
  bool warned_misalign = false;
  uint64_t launches = 0;
  bool connected = false;
  int sm_count = 148;
  int max_coresident = 0;  // co-resident CTAs of the step kernel
  // work tile in 16-byte vectors (0: contiguous range per CTA); env RBX_TILE.  -1 = default:
  // pass_tile() with dynamic tiles; with static tiles 1024 for 4/8-byte types and 2048 for bf16/f16, whose
  // heavier fold needs more vectors in flight per call (profiles/r01_tile_by_dtype.txt)
  int tile = -1;
  // dynamic work tiles (claimed from a per-step counter); env RBX_DYN.  With 2048-vector tiles
  // N=2 581 -> 595 GB/s, N=4 578 -> 597 GB/s busbw at 102.4 MB fp32 (profiles/r01_dyn_tiles_4gpu.txt)
  int dyn_tiles = 1;
  int tail_split = 1;
  int fence_every = 0;  // env RBX_FENCE_EVERY: fence.sys every this many dynamic tiles (experiment)  // env RBX_TAIL_SPLIT: finer tiles for the last nb tiles' worth of a step
  int local_tile = 2048;   // same for the HBM-bound local mode (measured best of 0/512/2048/4096/8192/32768); env RBX_LOCAL_TILE
  size_t bytes_per_cta = 32 * 1024;   // adaptive CTA count per call; env RBX_BYTES_PER_CTA
  int min_blocks = 16;                // env RBX_MIN_BLOCKS
  unsigned long long* trace_dev = nullptr;  // 64-word kernel timeline when RBX_TRACE is set
  // specialised local kernel: CTAs per SM (0 = occupancy limit); env RBX_LOCAL_CTAS_PER_SM.
  // 1 x 512 threads per SM measured 0.967-0.972 of the copy peak vs 0.925-0.928 at the
  // occupancy limit (2 per SM) on config 2 (profiles/r01_local_ctas_per_sm.txt).
  int local_ctas_per_sm = 1;
  bool local_specialised = true;
  int local_hint = 0;  // cache policy of the local kernel's streams (rbx_local.cuh LocalArgs::hint); env RBX_LOCAL_HINT  // MODE_LOCAL uses rbx_local_kernel where the shape has one; env RBX_LOCAL_GENERIC=1
  // MODE_PUSH inboxes: this rank's (registered, symmetric) and every rank's mapping
  char* inbox_local = nullptr;
  size_t inbox_bytes = 0;
  std::vector<char*> inbox_at;
  bool inbox_owned = false;  // virtual comms allocate their own
  // MODE_LL: every rank's LL area (rbx_ll.cuh), carved from the signal allocation
  std::vector<unsigned long long*> ll_at;
  size_t ll_auto_bytes = RBX_LL_MAX_BYTES;  // AUTO picks LL up to this many bytes per rank; env RBX_LL_AUTO_BYTES
  int ll_threads = 512;
  // one-shot LL up to this many bytes; env RBX_LL_ONESHOT_BYTES.  Off by default: on B200 it
  // measured slower than two-shot at every size (4 KB: 21 vs 13 us event time at N=2,
  // profiles/r01_ll_*), the launch/teardown floor dominates and it folds N x the elements.
  int64_t ll_oneshot_bytes = 0;
  int ll_words_per_thread = 2;        // CTAs per LL call = words / (threads * this); env RBX_LL_WPT (2 vs 4: 16 KB-256 KB 7-10 % faster at N=2, profiles/r02_ll_wpt_2gpu.jsonl)
  int ll_coresident = 0;              // co-resident CTAs of the LL kernel
  std::map<LLKey, std::unique_ptr<rbx::LLArgs>> ll_cache;  // per (buffers, count, dtype)
  // Launches of one communicator share a device epoch, so they must not overlap:
  // a launch on a different stream than the previous one waits for it.
  cudaEvent_t order_ev = nullptr;
  cudaStream_t last_stream = nullptr;
  bool has_last = false;
  // one-shot fault injection for the next launch (rbx_comm_inject_fault); -1 = off
  int fault_milli = -1;
  // FUSED allreduce through the specialised kernel (rbx_fused.cuh) where the grid shape has one;
  // env RBX_FUSED_KERNEL=0 forces the generic step interpreter
  bool fused_specialised = true;
  int pdl = 1;  // programmatic dependent launch for the fused kernel; env RBX_PDL
  int last_kernel = RBX_KERNEL_NONE;  // rbx_comm_last_kernel
  int fused_dbg = 0;  // env RBX_FUSED_DBG: experiment knobs of the fused kernel (rbx_fused.cuh FusedArgsT::dbg)
  bool plain_launch = false;  // env RBX_PLAIN_LAUNCH=1: fused kernel through cudaLaunchKernel (no launch attributes)
  bool rings_specialised = true;  // RING_DIMS through rbx_rings_kernel where possible; env RBX_RINGS_KERNEL=0: generic
  bool rings_gpu_fence = true;    // local-only stages signal after a GPU-scope fence; env RBX_RINGS_GPU_FENCE=0: sys release
  bool push_specialised = true;   // MODE_PUSH allreduce through the matched-stage kernel; env RBX_PUSH_KERNEL=0: generic
};

namespace {

// IPC mappings are per process (cudaIpcOpenMemHandle fails on a second open of
// the same handle), so they are shared by every communicator of the process and
// reference-counted.  ctypes releases the GIL, so calls may come from several
// threads at once: the table has a lock.
std::map<std::string, OpenedHandle>& opened_handles() {
  static std::map<std::string, OpenedHandle> m;
  return m;
}
std::mutex& opened_lock() {
  static std::mutex mu;
  return mu;
}

int open_handle(rbx_comm* c, const rbx_ipc_handle_t& h, void** out) {
  std::string key(reinterpret_cast<const char*>(h.bytes), sizeof(h.bytes));
  std::lock_guard<std::mutex> lock(opened_lock());
  auto& m = opened_handles();
  auto it = m.find(key);
  if (it != m.end()) {
    it->second.refs++;
    *out = it->second.ptr;
    c->opened.push_back(it->second.ptr);
    return RBX_OK;
  }
  cudaIpcMemHandle_t ch;
  std::memcpy(&ch, h.bytes, sizeof(ch));
  void* p = nullptr;
  RBX_CUDA(cudaIpcOpenMemHandle(&p, ch, cudaIpcMemLazyEnablePeerAccess));
  m[key] = OpenedHandle{p, 1};
  *out = p;
  c->opened.push_back(p);
  return RBX_OK;
}

// Drop this communicator's references; unmap what no communicator uses any more.
void close_handles(rbx_comm* c) {
  std::lock_guard<std::mutex> lock(opened_lock());
  auto& m = opened_handles();
  for (void* p : c->opened) {
    for (auto it = m.begin(); it != m.end(); ++it) {
      if (it->second.ptr != p) continue;
      if (--it->second.refs <= 0) {
        cudaIpcCloseMemHandle(p);
        m.erase(it);
      }
      break;
    }
  }
  c->opened.clear();
}

const void* kernel_for(int dtype) {
  switch (dtype) {
    case RBX_F32: return rbx::step_kernel_f32();
    case RBX_F64: return rbx::step_kernel_f64();
    case RBX_I64: return rbx::step_kernel_i64();
    case RBX_BF16: return rbx::step_kernel_bf16();
    case RBX_F16: return rbx::step_kernel_f16();
    case RBX_I32: return rbx::step_kernel_i32();
    default: return nullptr;
  }
}

const void* ll_kernel_for(int dtype, int maxv) {
  switch (dtype) {
    case RBX_F32: return rbx::ll_kernel_f32(maxv);
    case RBX_F64: return rbx::ll_kernel_f64(maxv);
    case RBX_I64: return rbx::ll_kernel_i64(maxv);
    case RBX_BF16: return rbx::ll_kernel_bf16(maxv);
    case RBX_F16: return rbx::ll_kernel_f16(maxv);
    case RBX_I32: return rbx::ll_kernel_i32(maxv);
    default: return nullptr;
  }
}

// One allocation per rank holds the signal area and, 256-byte aligned after
// it, the LL area; both are exported with one IPC handle.
constexpr size_t ll_offset() { return ((size_t)rbx::SigLayout::bytes + 255) / 256 * 256; }
size_t sig_alloc_bytes(int nranks) { return ll_offset() + (size_t)rbx::ll_area_bytes(nranks); }
unsigned long long* ll_area_of(uint32_t* sig) {
  return reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(sig) + ll_offset());
}

const void* fused_kernel_for(int dtype, int nsrc, int nlev, int ndst, int maxseg) {
  switch (dtype) {
    case RBX_F32: return rbx::fused_kernel_f32(nsrc, nlev, ndst, maxseg);
    case RBX_F64: return rbx::fused_kernel_f64(nsrc, nlev, ndst, maxseg);
    case RBX_I64: return rbx::fused_kernel_i64(nsrc, nlev, ndst, maxseg);
    case RBX_BF16: return rbx::fused_kernel_bf16(nsrc, nlev, ndst, maxseg);
    case RBX_F16: return rbx::fused_kernel_f16(nsrc, nlev, ndst, maxseg);
    case RBX_I32: return rbx::fused_kernel_i32(nsrc, nlev, ndst, maxseg);
    default: return nullptr;
  }
}

// Shape of a plan the specialised FUSED kernel runs: step 0 (after the entry wait)
// does every segment with the same (sources, nesting, destinations), step 1 is the
// exit wait.  Allreduce: fold all N buffers, store into all N; reduce-scatter: fold
// all N, store into mine; all-gather: copy mine into the N-1 peers.
bool fused_shape(const rbx::Plan& p, int N, int* nsrc, int* nlev, int* ndst) {
  if (p.nsteps != 2 || p.steps[1].nseg != 0 || p.nentry != N - 1) return false;
  const rbx::Step& st = p.steps[0];
  if (st.nseg < 1) return false;
  const rbx::Seg& s0 = p.segs[st.seg0];
  const bool fold = s0.nsrc == N && (s0.ndst == N || s0.ndst == 1);
  const bool copy = s0.nsrc == 1 && s0.ndst == N - 1 && s0.nlev == 1;
  if (!fold && !copy) return false;
  for (int k = 0; k < st.nseg; ++k) {
    const rbx::Seg& sg = p.segs[st.seg0 + k];
    if (sg.nsrc != s0.nsrc || sg.ndst != s0.ndst || sg.acc || sg.nlev != s0.nlev) return false;
    for (int j = 0; j < sg.nsrc; ++j)
      if (sg.ctrl[j] != s0.ctrl[j]) return false;
  }
  *nsrc = s0.nsrc;
  *nlev = s0.nlev;
  *ndst = s0.ndst;
  return true;
}

// Arguments of the specialised FUSED kernel from a plan of fused_shape().
template <int MAXSEG>
bool fused_args_from_plan(const rbx_comm* c, const rbx::Plan& p, const std::vector<void*>& table,
                          rbx::FusedArgsT<MAXSEG>* a) {
  std::memset(a, 0, sizeof(*a));
  const int N = c->nranks;
  int nsrc, nlev, ndst;
  if (!fused_shape(p, N, &nsrc, &nlev, &ndst)) return false;
  const rbx::Step& st = p.steps[0];
  if (st.nseg > MAXSEG) return false;
  a->nseg = st.nseg;
  a->me = c->rank;
  a->npeers = N - 1;
  a->total_vec = st.total_vec;
  a->my_sig = c->sig[c->rank];
  for (int i = 0, q = 0; q < N; ++q) {
    if (q == c->rank) continue;
    a->peer_rank[i] = (uint8_t)q;
    a->peer_sig[i++] = c->sig[q];
  }
  const rbx::Seg& s0 = p.segs[st.seg0];
  for (int j = 0; j < nsrc; ++j) a->ctrl[j] = s0.ctrl[j];
  for (int k = 0; k < st.nseg; ++k) {
    const rbx::Seg& sg = p.segs[st.seg0 + k];
    rbx::FusedSeg& fs = a->seg[k];
    fs.vec_begin = sg.vec_begin;
    fs.nvec = sg.nvec;
    fs.body_off = sg.body_off;
    fs.off = sg.off;
    fs.head = sg.head;
    fs.tail = sg.tail;
    for (int j = 0; j < nsrc; ++j) fs.src[j] = static_cast<const char*>(table[sg.tbl + sg.src[j]]);
    for (int j = 0; j < ndst; ++j) fs.dst[j] = static_cast<char*>(table[sg.tbl + sg.dst[j]]);
  }
  return true;
}

const void* rings_kernel_for(int dtype) {
  switch (dtype) {
    case RBX_F32: return rbx::rings_kernel_f32();
    case RBX_F64: return rbx::rings_kernel_f64();
    case RBX_I64: return rbx::rings_kernel_i64();
    case RBX_BF16: return rbx::rings_kernel_bf16();
    case RBX_F16: return rbx::rings_kernel_f16();
    case RBX_I32: return rbx::rings_kernel_i32();
    default: return nullptr;
  }
}

// Arguments of the matched-stage kernel (rbx_rings.cuh) from a RING_DIMS or PUSH allreduce
// plan (rbx_plan.cpp): every plan step becomes one kernel stage per segment (a PUSH scatter
// step has one segment per peer); the step's waits go to its first stage, its signals to its
// last; slots are the plan's.  Every wait becomes a MATCHED wait (rbx_rings.cuh explains why
// that is sufficient).  The last plan step is the exit wait.
bool rings_args_from_plan(const rbx_comm* c, const rbx::Plan& p, const std::vector<void*>& table, rbx::RingsArgs* a) {
  std::memset(a, 0, sizeof(*a));
  const int nsteps = p.nsteps - 1;  // data steps
  if (nsteps < 1 || p.steps[nsteps].nseg != 0) return false;
  a->me = c->rank;
  a->my_sig = c->sig[c->rank];
  for (int q = 0; q < c->nranks; ++q) a->sig[q] = c->sig[q];
  a->nentry = p.nentry;
  for (int i = 0; i < p.nentry; ++i) a->entry_peer[i] = p.entry_peers[i];
  int ns = 0;
  for (int s = 0; s <= nsteps; ++s) {
    const rbx::Step& st = p.steps[s];
    for (int w = 1; w < st.nwait; ++w)
      if (p.waits[st.wait0 + w].slot != p.waits[st.wait0].slot) return false;
    if (s == nsteps) {
      a->nexit = st.nwait;
      a->exit_slot = st.nwait ? p.waits[st.wait0].slot : 0;
      for (int w = 0; w < st.nwait; ++w) a->exit_peer[w] = p.waits[st.wait0 + w].peer;
      break;
    }
    if (st.nseg < 1 || ns + st.nseg > RBX_RINGS_MAX_STAGES) return false;
    if (st.nseg > 1 && a->group_count == 0) {  // one step, several segments: independent stages
      a->group_first = ns;
      a->group_count = st.nseg;
    }
    for (int k = 0; k < st.nseg; ++k) {
      const rbx::Seg& sg = p.segs[st.seg0 + k];
      const bool shape_ok = (sg.nlev == 1 && (sg.nsrc == 1 || sg.nsrc == 2 || sg.nsrc == 4 || sg.nsrc == 8)) ||
                            (sg.nlev == 2 && (sg.nsrc == 4 || sg.nsrc == 8)) || (sg.nlev == 3 && sg.nsrc == 8);
      if (sg.acc || !shape_ok) return false;
      rbx::RingStage& R = a->st[ns++];
      R.off = sg.off;
      R.len = sg.len;
      R.nsrc = sg.nsrc;
      R.ndst = sg.ndst;
      R.nlev = sg.nlev;
      for (int j = 0; j < sg.nsrc; ++j) {
        R.src[j] = static_cast<const char*>(table[sg.tbl + sg.src[j]]);
        R.ctrl[j] = sg.ctrl[j];
      }
      for (int d = 0; d < sg.ndst; ++d) R.dst[d] = static_cast<char*>(table[sg.tbl + sg.dst[d]]);
      // stage 0 of a plan with an entry handshake waits on the entry flags instead
      const bool first = k == 0 && !(s == 0 && p.nentry);
      R.nwait = first ? (uint8_t)st.nwait : 0;
      R.wait_slot = st.nwait ? p.waits[st.wait0].slot : 0;
      for (int w = 0; first && w < st.nwait; ++w) R.wait_peer[w] = p.waits[st.wait0 + w].peer;
      const bool last = k == st.nseg - 1;
      R.nsig = last ? (uint8_t)st.nsig : 0;
      R.sig_slot = (uint8_t)(s + 1);
      for (int j = 0; last && j < st.nsig; ++j) R.sig_peer[j] = p.sigs[st.sig0 + j];
      R.local_only = (uint8_t)(c->rings_gpu_fence && sg.ndst == 1 && sg.dst[0] == c->rank);
    }
  }
  a->nstages = ns;
  return true;
}

const void* local_kernel_for(int dtype, int v, int nlev) {
  switch (dtype) {
    case RBX_F32: return rbx::local_kernel_f32(v, nlev);
    case RBX_F64: return rbx::local_kernel_f64(v, nlev);
    case RBX_I64: return rbx::local_kernel_i64(v, nlev);
    case RBX_BF16: return rbx::local_kernel_bf16(v, nlev);
    case RBX_F16: return rbx::local_kernel_f16(v, nlev);
    case RBX_I32: return rbx::local_kernel_i32(v, nlev);
    default: return nullptr;
  }
}

// Kernel arguments of the specialised local kernel from a MODE_LOCAL plan
// (one step, one segment per owned region, all V buffers as destinations).
bool local_args_from_plan(const rbx::Plan& p, const std::vector<void*>& bufs, rbx::LocalArgs* a) {
  std::memset(a, 0, sizeof(*a));
  if (p.nsteps != 1) return false;
  const rbx::Step& st = p.steps[0];
  if (st.nseg > RBX_LOCAL_MAX_SEGS) return false;
  a->nseg = st.nseg;
  a->total_vec = st.total_vec;
  for (size_t d = 0; d < bufs.size(); ++d) a->dst[d] = static_cast<char*>(bufs[d]);
  for (int k = 0; k < st.nseg; ++k) {
    const rbx::Seg& sg = p.segs[st.seg0 + k];
    rbx::LocalSeg& ls = a->seg[k];
    ls.vec_begin = sg.vec_begin;
    ls.nvec = sg.nvec;
    ls.body_off = sg.body_off;
    for (int j = 0; j < sg.nsrc; ++j) {
      ls.src[j] = static_cast<const char*>(bufs[sg.src[j]]);
      ls.ctrl[j] = sg.ctrl[j];
    }
    for (int i = 0; i < sg.head + sg.tail; ++i) {
      if (a->nscalar >= (int)(sizeof(a->scalar_elem) / sizeof(a->scalar_elem[0]))) return false;
      a->scalar_elem[a->nscalar] = i < sg.head ? sg.off + i : sg.body_off + sg.nvec * p.vec + (i - sg.head);
      a->scalar_seg[a->nscalar] = (uint8_t)k;
      a->nscalar++;
    }
  }
  return true;
}

int coresident_blocks(int device, int threads, int* out) {
  int sms = 0;
  RBX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  int worst = 1 << 30;
  const size_t max_smem = (rbx::plan_smem_bytes(RBX_MAX_SEGS) + 15) / 16 * 16;
  static_assert((rbx::plan_smem_bytes(RBX_MAX_SEGS) + 15) / 16 * 16 + 1024 <= 48 * 1024,
                "staged plan must fit the default dynamic shared memory window");
  for (int dt = RBX_F32; dt <= RBX_I32; ++dt) {
    int per_sm = 0;
    RBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel_for(dt), threads, max_smem));
    if (per_sm * sms < worst) worst = per_sm * sms;
  }
  *out = worst;
  return RBX_OK;
}

// Every kernel of the library asks for the same L1 / shared-memory split, so
// consecutive launches of ours (barrier -> collective, bucket -> bucket) never
// make the SMs drain and reconfigure the carveout between them.  env
// RBX_CARVEOUT: percent of the unified L1 given to shared memory (-1: leave
// each kernel's default).
int set_carveouts(int device, int pct) {
  static std::mutex mu;
  static std::map<int, int> done;  // device -> carveout applied
  std::lock_guard<std::mutex> lock(mu);
  if (pct < 0) return RBX_OK;
  auto hit = done.find(device);
  if (hit != done.end() && hit->second == pct) return RBX_OK;
  std::vector<const void*> fns;
  for (int dt = RBX_F32; dt <= RBX_I32; ++dt) {
    fns.push_back(kernel_for(dt));
    fns.push_back(ll_kernel_for(dt, 1));
    fns.push_back(ll_kernel_for(dt, RBX_MAX_RANKS));
    for (int n : {1, 2, 4, 8})
      for (int l = 1; l <= 3; ++l)
        for (int d : {1, 3, 7, n})
          for (int ms : {1, RBX_FUSED_MAXSEG}) fns.push_back(fused_kernel_for(dt, n, l, d, ms));
    for (int v : {2, 4, 8})
      for (int l = 1; l <= 3; ++l) fns.push_back(local_kernel_for(dt, v, l));
    fns.push_back(rings_kernel_for(dt));
  }
  for (const void* f : fns)
    if (f) RBX_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
  done[device] = pct;
  return RBX_OK;
}

int common_init(rbx_comm* c, const int* dims, int ndims, int device, int threads) {
  std::string err;
  if (!c->geo.init(dims, ndims, &err)) return fail(RBX_ERR_INVALID, err);
  if (threads <= 0) threads = 512;
  if (threads % 32 || threads > 512) return fail(RBX_ERR_INVALID, "threads must be a multiple of 32 and <= 512");
  c->threads = threads;
  c->ll_threads = threads;
  c->device = device;
  if (const char* t = std::getenv("RBX_TILE")) c->tile = std::atoi(t);
  if (const char* t = std::getenv("RBX_LOCAL_TILE")) c->local_tile = std::atoi(t);
  if (const char* t = std::getenv("RBX_DYN")) c->dyn_tiles = std::atoi(t);
  if (const char* t = std::getenv("RBX_TAIL_SPLIT")) c->tail_split = std::max(1, std::atoi(t));
  if (const char* t = std::getenv("RBX_FENCE_EVERY")) c->fence_every = std::max(0, std::atoi(t));
  if (const char* t = std::getenv("RBX_LOCAL_GENERIC")) c->local_specialised = std::atoi(t) == 0;
  if (const char* t = std::getenv("RBX_LOCAL_HINT")) c->local_hint = std::atoi(t);
  if (const char* t = std::getenv("RBX_FUSED_KERNEL")) c->fused_specialised = std::atoi(t) != 0;
  if (const char* t = std::getenv("RBX_PDL")) c->pdl = std::atoi(t) != 0;
  if (const char* t = std::getenv("RBX_FUSED_DBG")) c->fused_dbg = std::atoi(t);
  if (const char* t = std::getenv("RBX_PLAIN_LAUNCH")) c->plain_launch = std::atoi(t) != 0;
  if (const char* t = std::getenv("RBX_RINGS_KERNEL")) c->rings_specialised = std::atoi(t) != 0;
  if (const char* t = std::getenv("RBX_RINGS_GPU_FENCE")) c->rings_gpu_fence = std::atoi(t) != 0;
  if (const char* t = std::getenv("RBX_PUSH_KERNEL")) c->push_specialised = std::atoi(t) != 0;
  if (const char* t = std::getenv("RBX_LOCAL_CTAS_PER_SM")) c->local_ctas_per_sm = std::atoi(t);
  if (const char* t = std::getenv("RBX_BYTES_PER_CTA")) c->bytes_per_cta = (size_t)std::max(1L, std::atol(t));
  if (const char* t = std::getenv("RBX_MIN_BLOCKS")) c->min_blocks = std::max(1, std::atoi(t));
  if (const char* t = std::getenv("RBX_LL_AUTO_BYTES"))
    c->ll_auto_bytes = std::min((size_t)std::max(0L, std::atol(t)), (size_t)RBX_LL_MAX_BYTES);
  if (const char* t = std::getenv("RBX_LL_WPT")) c->ll_words_per_thread = std::max(1, std::atoi(t));
  if (const char* t = std::getenv("RBX_LL_ONESHOT_BYTES")) c->ll_oneshot_bytes = std::atol(t);
  RBX_CUDA(cudaSetDevice(device));
  RBX_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
  int carveout = 50;  // 114 KB of shared memory: covers the step kernel's staged plan at 2 CTAs per SM
  if (const char* t = std::getenv("RBX_CARVEOUT")) carveout = std::atoi(t);
  if (int rc2 = set_carveouts(device, carveout)) return rc2;
  int rc = coresident_blocks(device, threads, &c->max_coresident);
  if (rc) return rc;
  if (const char* t = std::getenv("RBX_TRACE")) {
    if (std::atoi(t)) {
      RBX_CUDA(cudaMalloc(reinterpret_cast<void**>(&c->trace_dev), 64 * sizeof(unsigned long long)));
      RBX_CUDA(cudaMemset(c->trace_dev, 0, 64 * sizeof(unsigned long long)));
    }
  }
  RBX_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->err_host), sizeof(rbx::ErrRecord), cudaHostAllocMapped));
  std::memset(c->err_host, 0, sizeof(rbx::ErrRecord));
  RBX_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->err_dev), c->err_host, 0));
  return RBX_OK;
}

std::string plan_key(int op, int mode, int dtype, const std::vector<const void*>& ptrs, const std::vector<size_t>& counts) {
  std::string k = std::to_string(op) + ":" + std::to_string(mode) + ":" + std::to_string(dtype);
  char buf[64];
  for (size_t i = 0; i < ptrs.size(); ++i) {
    std::snprintf(buf, sizeof(buf), "|%p#%zu", ptrs[i], counts.empty() ? 0 : counts[i % counts.size()]);
    k += buf;
  }
  return k;
}

// Default work tile of step s with dynamic tiles: one pass of the fold loop, i.e. threads x U
// vectors, where U is fold_body's unroll for the step's widest fold (rbx_kernel.cuh; 8 for a
// copy step).  A smaller tile leaves loads of the pass unissued (N=2, tile 512: 503 vs 595
// GB/s); a larger one coarsens the tail.  fp32 FUSED: N=2 -> 2048, (2,2) -> 1024, (2,2,2) -> 512.
int pass_tile(const rbx::Plan& p, int s, int threads) {
  int u = 0;
  for (int k = 0; k < p.steps[s].nseg; ++k) {
    const rbx::Seg& sg = p.segs[p.steps[s].seg0 + k];
    if (sg.acc) continue;
    int us;
    if (sg.nsrc < 2) {
      us = 8;  // copy (REPLACE): fold_body<T,1,L> keeps 8 loads in flight per thread
    } else {
      const int B = sg.nsrc < 8 ? sg.nsrc : 8;
      const int u_ld = std::max(1, RBX_LD_DEPTH / B);
      const int u_acc = std::max(1, 32 / (std::max(1, (int)sg.nlev) * p.vec));
      us = std::min(u_ld, u_acc);
    }
    u = std::max(u, us);
  }
  return u ? threads * u : 2048;
}

// tables: one pointer table shared by every plan, or one per plan (MODE_PUSH
// tables depend on the rank: own inbox slots, this rank's slot in the peers').
int upload(rbx_comm* c, std::vector<rbx::Plan>& host, const std::vector<std::vector<void*>>& tables,
           CachedPlan* out, int dtype) {
  std::vector<void*> flat;
  std::vector<size_t> base;
  for (const auto& t : tables) {
    base.push_back(flat.size());
    flat.insert(flat.end(), t.begin(), t.end());
  }
  RBX_CUDA(cudaMalloc(reinterpret_cast<void**>(&out->ptrs), sizeof(void*) * (flat.size() ? flat.size() : 1)));
  if (!flat.empty())
    RBX_CUDA(cudaMemcpy(out->ptrs, flat.data(), sizeof(void*) * flat.size(), cudaMemcpyHostToDevice));
  int maxsegs = 0;
  for (size_t i = 0; i < host.size(); ++i) {
    rbx::Plan& p = host[i];
    p.ptrs = out->ptrs + (tables.size() == host.size() ? base[i] : 0);
    if (p.nosync)
      p.tile = c->local_tile;
    else if (c->tile >= 0)
      p.tile = c->tile;
    else
      p.tile = dtype_size(dtype) == 2 ? 2048 : 1024;
    for (int s = 0; s < p.nsteps; ++s)  // dynamic tiles: one fold pass of each step's widest fold
      p.steps[s].tile = (!p.nosync && c->tile < 0 && c->dyn_tiles) ? pass_tile(p, s, c->threads) : 0;
    p.dyn = (!p.nosync && p.tile > 0) ? c->dyn_tiles : 0;
    p.tail_split = c->tail_split;
    p.fence_every = c->fence_every;
    int segs = 0;
    for (int s = 0; s < p.nsteps; ++s) segs += p.steps[s].nseg;
    if (segs > maxsegs) maxsegs = segs;
  }
  out->plan_bytes = (int)rbx::plan_smem_bytes(maxsegs);
  RBX_CUDA(cudaMalloc(reinterpret_cast<void**>(&out->dev), sizeof(rbx::Plan) * host.size()));
  RBX_CUDA(cudaMemcpy(out->dev, host.data(), sizeof(rbx::Plan) * host.size(), cudaMemcpyHostToDevice));
  out->nplans = (int)host.size();
  return RBX_OK;
}

void free_plan(CachedPlan& cp) {
  cudaFree(cp.dev);
  cudaFree(cp.ptrs);
}

// Drop cached plans (all, or only those using the inbox).  Plans a captured CUDA graph
// may replay are retired (freed at destroy); otherwise they are freed after the
// device is idle.
int drop_plans(rbx_comm* c, bool inbox_only) {
  if (!c->captured) RBX_CUDA(cudaDeviceSynchronize());
  for (auto it = c->plans.begin(); it != c->plans.end();) {
    if (inbox_only && !it->second.uses_inbox) {
      ++it;
      continue;
    }
    if (c->captured)
      c->retired.push_back(it->second);
    else
      free_plan(it->second);
    it = c->plans.erase(it);
  }
  return RBX_OK;
}

// Bound the plan cache (one entry per distinct buffer pointer / window / count: DDP
// bucket rebuilds or fresh tensors would otherwise grow device memory without limit).
constexpr size_t kMaxPlans = 512;
int bound_plans(rbx_comm* c) { return c->plans.size() >= kMaxPlans ? drop_plans(c, false) : RBX_OK; }

// Serialise launches of one communicator across streams (outside stream
// capture; inside a graph the capture order is the user's contract).
int order_before(rbx_comm* c, cudaStream_t stream, bool* capturing) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  RBX_CUDA(cudaStreamIsCapturing(stream, &st));
  *capturing = st != cudaStreamCaptureStatusNone;
  if (*capturing) {
    c->captured = true;
    return RBX_OK;
  }
  if (!c->order_ev) RBX_CUDA(cudaEventCreateWithFlags(&c->order_ev, cudaEventDisableTiming));
  if (c->has_last && stream != c->last_stream) RBX_CUDA(cudaStreamWaitEvent(stream, c->order_ev, 0));
  return RBX_OK;
}

int order_after(rbx_comm* c, cudaStream_t stream, bool capturing) {
  if (capturing) return RBX_OK;
  RBX_CUDA(cudaEventRecord(c->order_ev, stream));
  c->last_stream = stream;
  c->has_last = true;
  return RBX_OK;
}

int launch(rbx_comm* c, const CachedPlan& cp, int dtype, cudaStream_t stream, bool cooperative, int nblocks) {
  const void* fn = kernel_for(dtype);
  if (!fn) return fail(RBX_ERR_INVALID, "unknown dtype");
  rbx::KernelArgs a;
  a.plans = cp.dev;
  a.nblocks = nblocks;
  a.timeout_ns = c->timeout_ns;
  a.err = c->err_dev;
  a.plan_bytes = cp.plan_bytes;
  a.trace = c->trace_dev;
  a.fault_milli = c->fault_milli;
  c->fault_milli = -1;
  void* params[] = {&a};
  dim3 grid((unsigned)(nblocks * cp.nplans)), block((unsigned)c->threads);
  const size_t smem = (size_t)((cp.plan_bytes + 15) / 16 * 16);
  bool capturing = false;
  if (int rc = order_before(c, stream, &capturing)) return rc;
  if (cooperative) {
    RBX_CUDA(cudaLaunchCooperativeKernel(fn, grid, block, params, smem, stream));
  } else {
    RBX_CUDA(cudaLaunchKernel(fn, grid, block, params, smem, stream));
  }
  c->launches++;
  c->last_kernel = RBX_KERNEL_STEP;
  return order_after(c, stream, capturing);
}

// Launch of the specialised FUSED kernel (rbx_fused.cuh) with programmatic
// dependent launch: its CTAs may become resident while the previous kernel on
// the stream drains (griddepcontrol.wait guards every memory read).
int fused_launch(rbx_comm* c, CachedPlan& cp, cudaStream_t stream, int nb) {
  void* argp;
  if (cp.fused1) {
    cp.fused1->timeout_ns = c->timeout_ns;
    cp.fused1->trace = c->trace_dev;
    cp.fused1->fault_milli = c->fault_milli;
    cp.fused1->dbg = c->fused_dbg;
    argp = cp.fused1.get();
  } else {
    cp.fusedN->timeout_ns = c->timeout_ns;
    cp.fusedN->trace = c->trace_dev;
    cp.fusedN->fault_milli = c->fault_milli;
    cp.fusedN->dbg = c->fused_dbg;
    argp = cp.fusedN.get();
  }
  c->fault_milli = -1;
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)nb);
  cfg.blockDim = dim3((unsigned)c->threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = c->pdl;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* params[] = {argp};
  bool capturing = false;
  if (int rc = order_before(c, stream, &capturing)) return rc;
  if (c->plain_launch)
    RBX_CUDA(cudaLaunchKernel(cp.fused_fn, cfg.gridDim, cfg.blockDim, params, 0, stream));
  else
    RBX_CUDA(cudaLaunchKernelExC(&cfg, cp.fused_fn, params));
  c->launches++;
  c->last_kernel = RBX_KERNEL_FUSED;
  return order_after(c, stream, capturing);
}

int rings_launch(rbx_comm* c, CachedPlan& cp, cudaStream_t stream, int nb) {
  cp.rings->timeout_ns = c->timeout_ns;
  cp.rings->trace = c->trace_dev;
  cp.rings->fault_milli = c->fault_milli;
  c->fault_milli = -1;
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)nb);
  cfg.blockDim = dim3((unsigned)c->threads);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = c->pdl;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* params[] = {cp.rings.get()};
  bool capturing = false;
  if (int rc = order_before(c, stream, &capturing)) return rc;
  RBX_CUDA(cudaLaunchKernelExC(&cfg, cp.rings_fn, params));
  c->launches++;
  c->last_kernel = RBX_KERNEL_RINGS;
  return order_after(c, stream, capturing);
}

// Every (mode, dtype) pair is supported: RING_DIMS keeps bf16/f16 stage
// partials in fp32 workspaces (ws_table), LL folds in fp32 registers.
int check_mode_dtype(int mode, int dtype) {
  (void)dtype;
  if (mode < RBX_MODE_AUTO || mode > RBX_MODE_LL) return fail(RBX_ERR_INVALID, "unknown mode");
  return RBX_OK;
}

// MODE_LL launch (rbx_ll.cuh): ranks[0..nhosted) are the ranks this launch
// plays (1 for a per-rank communicator, V for a virtual one).
int ll_launch(rbx_comm* c, const std::vector<int>& ranks, void* const* bufs, size_t count, int dtype,
              cudaStream_t stream, bool cooperative) {
  const int V = (int)ranks.size();
  const void* fn = ll_kernel_for(dtype, V == 1 ? 1 : RBX_MAX_RANKS);
  if (!fn) return fail(RBX_ERR_INVALID, "unknown dtype");
  const int es = dtype_size(dtype);
  if (count * (size_t)es > (size_t)RBX_LL_MAX_BYTES)
    return fail(RBX_ERR_INVALID, "MODE_LL handles at most " + std::to_string(RBX_LL_MAX_BYTES) + " bytes per rank");
  if (c->ll_coresident == 0) {
    int per_sm = 0;
    RBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, c->ll_threads, 0));
    c->ll_coresident = std::max(1, per_sm) * c->sm_count;
  }
  LLKey key{std::vector<void*>(bufs, bufs + V), count, dtype};
  auto it = c->ll_cache.find(key);
  if (it == c->ll_cache.end()) {
    const rbx::Geometry& g = c->geo;
    const int m = (int)g.active_dims().size();
    // LL words per rank (rbx_ll.cuh LLFmt): 2-byte types pack two elements per word
    const int64_t words = es == 2 ? ((int64_t)count + 1) / 2 : (es == 8 ? 2 * (int64_t)count : (int64_t)count);
    int nb = (int)std::min<int64_t>((words + (int64_t)c->ll_threads * c->ll_words_per_thread - 1) /
                                        ((int64_t)c->ll_threads * c->ll_words_per_thread),
                                    (int64_t)c->nblocks);
    if (nb < 1) nb = 1;
    if ((int64_t)nb * V > c->ll_coresident) nb = std::max(1, c->ll_coresident / V);
    std::unique_ptr<rbx::LLArgs> a(new rbx::LLArgs);
    std::memset(a.get(), 0, sizeof(rbx::LLArgs));
    a->nranks = c->nranks;
    a->nlev = m;
    a->nb = nb;
    a->nhosted = V;
    a->cap = rbx::ll_cap_words(c->nranks);
    a->err = c->err_dev;
    a->trace = c->trace_dev;
    const int64_t bytes = (int64_t)count * es;
    a->oneshot = bytes <= c->ll_oneshot_bytes && bytes <= RBX_LL_ONESHOT_MAX_BYTES;
    for (int q = 0; q < c->nranks; ++q) {
      const std::vector<int> o = rbx::fold_order(g, q);
      for (int k = 0; k < c->nranks; ++k) a->orders.of[q][k] = (uint8_t)o[k];
    }
    const std::vector<uint8_t> ctrl = rbx::fold_ctrl(g);
    for (int v = 0; v < V; ++v) {
      rbx::LLRank& R = a->rank[v];
      const int me = ranks[v];
      R.me = me;
      R.buf = static_cast<char*>(bufs[v]);
      R.my_sig = c->sig[me];
      for (int q = 0; q < c->nranks; ++q) {
        R.area[q] = c->ll_at[q];
        rbx::region_after(g, q, (int64_t)count, m, &R.off[q], &R.len[q]);
      }
      const std::vector<int> order = rbx::fold_order(g, me);
      for (int k = 0; k < c->nranks; ++k) {
        R.order[k] = (uint8_t)order[k];
        R.ctrl[k] = ctrl[k];
      }
    }
    if (c->ll_cache.size() >= 4096) c->ll_cache.clear();  // bound host memory (~8 KB per entry)
    it = c->ll_cache.emplace(std::move(key), std::move(a)).first;
  }
  rbx::LLArgs* a = it->second.get();
  a->timeout_ns = c->timeout_ns;
  a->fault = c->fault_milli < 0 ? -1 : (c->fault_milli == 0 ? 0 : 1);
  c->fault_milli = -1;
  const int nb = a->nb;
  void* params[] = {a};
  rbx::LLArgsT<1> a1;  // per-rank form: the same fields with one hosted rank
  if (V == 1) {
    std::memcpy(&a1, a, offsetof(rbx::LLArgs, rank));
    a1.rank[0] = a->rank[0];
    params[0] = &a1;
  }
  dim3 grid((unsigned)(nb * V)), block((unsigned)c->ll_threads);
  bool capturing = false;
  if (int rc = order_before(c, stream, &capturing)) return rc;
  if (cooperative) {
    RBX_CUDA(cudaLaunchCooperativeKernel(fn, grid, block, params, 0, stream));
  } else {  // per-rank form: programmatic dependent launch, like the specialised kernels
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = c->pdl;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    RBX_CUDA(cudaLaunchKernelExC(&cfg, fn, params));
  }
  c->launches++;
  c->last_kernel = RBX_KERNEL_LL;
  return order_after(c, stream, capturing);
}

// MODE_PUSH pointer-table entries of rank `me` for one buffer (rbx_plan.h
// table_entries): buffers, own inbox slots, own slot in every peer's inbox.
// Inbox pointers are biased by -off*itemsize so the plan's element offsets
// address them directly, and padded so that element `off` sits at the same
// 16-byte phase as in the buffer (one head/body/tail split fits both).
std::vector<void*> push_table(const rbx::Geometry& g, int me, int64_t count, int es, int mis,
                              const std::vector<char*>& bufs, const std::vector<char*>& inbox, int64_t inbox_off) {
  const int R = g.nranks;
  const int m = (int)g.active_dims().size();
  const int vec = 16 / es;
  const int64_t slot = rbx::inbox_slot_bytes(g, count, es);
  std::vector<void*> t(3 * R, nullptr);
  for (int q = 0; q < R; ++q) t[q] = bufs[q];
  auto biased = [&](int owner, int slot_idx) -> void* {
    int64_t o, l;
    rbx::region_after(g, owner, count, m, &o, &l);
    const int64_t pad = mis >= 0 ? ((mis + o) % vec) * es : 0;
    const uintptr_t a = reinterpret_cast<uintptr_t>(inbox[owner]) + inbox_off + slot_idx * slot + pad - o * es;
    return reinterpret_cast<void*>(a);
  };
  for (int p = 0; p < R; ++p) t[R + p] = biased(me, p);
  for (int q = 0; q < R; ++q) t[2 * R + q] = biased(q, me);
  return t;
}

// RING_DIMS bf16/f16 pointer table: buffers, then every rank's fp32 partial
// workspace (carved from its inbox), biased so the plan's element offsets
// address it and element vectors stay 32-byte aligned like in the buffer.
std::vector<void*> ws_table(const rbx::Geometry& g, int64_t count, int es, int mis, const std::vector<char*>& bufs,
                            const std::vector<char*>& inbox, int64_t inbox_off) {
  const int R = g.nranks;
  const int vec = 16 / es;
  std::vector<void*> t(2 * R, nullptr);
  for (int q = 0; q < R; ++q) {
    t[q] = bufs[q];
    int64_t o, l;
    rbx::region_after(g, q, count, 1, &o, &l);  // region after the first ring dimension
    const int64_t pad = mis >= 0 ? (mis + o) % vec : 0;
    t[R + q] = reinterpret_cast<void*>(reinterpret_cast<uintptr_t>(inbox[q]) + inbox_off + (pad - o) * 4);
  }
  return t;
}

bool needs_fp32_partials(const rbx::Geometry& g, int mode, int dtype, int op) {
  return mode == RBX_MODE_RING_DIMS && (dtype == RBX_BF16 || dtype == RBX_F16) && g.active_dims().size() > 1 &&
         (op == RBX_OP_ALLREDUCE || op == RBX_OP_REDUCE_SCATTER);
}

// Elements between the previous 16-byte boundary and element 0, if identical
// for every rank's copy (then the scalar head/tail peel is the same
// everywhere); -1 if the copies are differently aligned (scalar path only).
int misalign(const std::vector<void*>& ptrs, int es) {
  int m = -1;
  for (void* p : ptrs) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    if (a % es) return -1;
    const int mm = (int)((a % 16) / es);
    if (m >= 0 && mm != m) return -1;
    m = mm;
  }
  return m < 0 ? 0 : m;
}

int find_buffer(rbx_comm* c, const void* p, size_t bytes, int* id, size_t* off) {
  for (size_t i = 0; i < c->bufs.size(); ++i) {
    const RegBuf& b = c->bufs[i];
    const char* q = static_cast<const char*>(p);
    if (q >= b.base && q + bytes <= b.base + b.bytes) {
      *id = (int)i;
      *off = (size_t)(q - b.base);
      return RBX_OK;
    }
  }
  return fail(RBX_ERR_INVALID, "buffer is not registered with this communicator (use rbx_register_buffer / "
                               "PlacedBuffer.device(); there is no unregistered fallback)");
}

int real_collective(rbx_comm* c, void* const* bufs, const size_t* counts, int nbufs, int dtype, int op, int mode,
                    cudaStream_t stream, int64_t lo = 0, int64_t hi = -1) {
  if (!c || c->nvirtual) return fail(RBX_ERR_INVALID, "not a per-rank communicator");
  if (!c->connected) return fail(RBX_ERR_INVALID, "communicator is not connected");
  const int es = dtype_size(dtype);
  if (!es) return fail(RBX_ERR_INVALID, "unknown dtype");
  if (mode == RBX_MODE_LOCAL) return fail(RBX_ERR_INVALID, "MODE_LOCAL needs a virtual communicator");
  if (int rc = check_mode_dtype(mode, dtype)) return rc;
  if (c->err_host->code) return fail(RBX_ERR_COLLECTIVE, "communicator is in an error state", c->err_host->peer, c->err_host->step);
  size_t total = 0;
  for (int k = 0; k < nbufs; ++k) total += counts[k];
  if (total == 0 && op != RBX_OP_BARRIER) return RBX_OK;  // empty collective: nothing moves on any rank
  const bool whole = lo == 0 && (hi < 0 || hi == (int64_t)total);
  const bool ll = mode == RBX_MODE_LL || (mode == RBX_MODE_AUTO && op == RBX_OP_ALLREDUCE && nbufs == 1 && whole &&
                                          c->nranks > 1 && total * (size_t)es <= c->ll_auto_bytes);
  if (ll) {
    if (op != RBX_OP_ALLREDUCE || nbufs != 1 || !whole)
      return fail(RBX_ERR_INVALID, "MODE_LL supports a whole-buffer single allreduce only");
    // LL never maps the buffer into peers, but the contract is the same for every
    // mode: collectives run on registered (symmetric) buffers only
    int id;
    size_t off;
    if (int rc = find_buffer(c, bufs[0], counts[0] * es, &id, &off)) return rc;
    return ll_launch(c, {c->rank}, bufs, counts[0], dtype, stream, false);
  }
  std::vector<const void*> kp(bufs, bufs + nbufs);
  std::vector<size_t> kc(counts, counts + nbufs);
  const std::string key = plan_key(op, mode, dtype, kp, kc) + "@" + std::to_string(lo) + ":" + std::to_string(hi);
  auto it = c->plans.find(key);
  if (it == c->plans.end()) {
    if (int rc = bound_plans(c)) return rc;
    std::vector<rbx::Plan> host(1);
    std::vector<void*> ptrs;
    rbx::PlanSpec spec;
    spec.op = (rbx::Op)op;
    spec.mode = (rbx::Mode)mode;
    spec.vec = 16 / es;
    spec.nblocks = c->nblocks;
    spec.lo = lo;
    spec.hi = hi;
    const bool push = mode == RBX_MODE_PUSH && (op == RBX_OP_ALLREDUCE || op == RBX_OP_REDUCE_SCATTER);
    const bool ws = needs_fp32_partials(c->geo, mode, dtype, op);
    spec.partials_fp32 = ws;
    // pointer-table entries per buffer
    const int E = push ? 3 * c->nranks : (ws ? 2 * c->nranks : c->nranks);
    int64_t inbox_off = 0;
    std::string err;
    for (int k = 0; k < nbufs; ++k) {
      int id;
      size_t off;
      if (op != RBX_OP_BARRIER && counts[k] == 0) {
        for (int q = 0; q < E; ++q) ptrs.push_back(nullptr);  // empty bucket: never dereferenced
      } else if (op != RBX_OP_BARRIER) {
        int rc = find_buffer(c, bufs[k], counts[k] * es, &id, &off);
        if (rc) return rc;
        std::vector<char*> mine;
        for (int q = 0; q < c->nranks; ++q) mine.push_back(c->bufs[id].at[q] + off);
        spec.mis = misalign(std::vector<void*>(mine.begin(), mine.end()), es);
        if (spec.mis < 0 && !c->warned_misalign) {
          // correct, but every element goes through the scalar path (one CTA per segment)
          std::fprintf(stderr, "librbx: rank %d: buffer copies are differently aligned across ranks (16-byte phase); "
                               "this collective runs element by element -- allocate symmetric buffers at equal offsets\n",
                       c->rank);
          c->warned_misalign = true;
        }
        if (push || ws) {
          const int64_t need = rbx::inbox_buffer_bytes(c->geo, (int64_t)counts[k], es);
          if (inbox_off + need > (int64_t)c->inbox_bytes)
            return fail(RBX_ERR_INVALID, "inbox too small for this mode: need " + std::to_string(inbox_off + need) +
                                             " bytes, have " + std::to_string(c->inbox_bytes) +
                                             " (rbx_set_inbox; size with rbx_inbox_bytes)");
          std::vector<void*> t = push ? push_table(c->geo, c->rank, (int64_t)counts[k], es, spec.mis, mine,
                                                   c->inbox_at, inbox_off)
                                      : ws_table(c->geo, (int64_t)counts[k], es, spec.mis, mine, c->inbox_at, inbox_off);
          ptrs.insert(ptrs.end(), t.begin(), t.end());
          inbox_off += need;
        } else {
          ptrs.insert(ptrs.end(), mine.begin(), mine.end());
        }
      }
      if (!rbx::build_plan(c->geo, c->rank, (int64_t)counts[k], spec, k * E, &host[0], k == 0, &err))
        return fail(RBX_ERR_INVALID, err);
    }
    for (int q = 0; q < c->nranks; ++q) host[0].sig[q] = c->sig[q];
    host[0].my_sig = c->sig[c->rank];
    CachedPlan cp;
    cp.uses_inbox = push || ws;
    int rc = upload(c, host, {ptrs}, &cp, dtype);
    if (rc) return rc;
    // RING_DIMS over a one-dimensional grid is the same single ring fold as FUSED (same
    // order, same pushes): both go through the specialised kernel
    const bool one_ring = mode == RBX_MODE_RING_DIMS && c->geo.active_dims().size() == 1;
    // reduce-scatter / all-gather alone: the same kernel with one destination / one source
    const bool fused = ((mode == RBX_MODE_FUSED || mode == RBX_MODE_AUTO || one_ring) && op == RBX_OP_ALLREDUCE &&
                        !push && !ws) ||
                       ((mode == RBX_MODE_FUSED || mode == RBX_MODE_AUTO) &&
                        (op == RBX_OP_REDUCE_SCATTER || op == RBX_OP_ALLGATHER) && !ws);
    int f_nsrc = 0, f_nlev = 0, f_ndst = 0;
    if (fused && c->fused_specialised && fused_shape(host[0], c->nranks, &f_nsrc, &f_nlev, &f_ndst)) {
      const int nseg = host[0].steps[0].nseg;
      const int maxseg = nseg <= 1 ? 1 : RBX_FUSED_MAXSEG;
      const void* fn = fused_kernel_for(dtype, f_nsrc, f_nlev, f_ndst, maxseg);
      int per_sm = 0;
      if (fn) RBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, c->threads, 0));
      if (fn && per_sm * c->sm_count >= c->nblocks) {
        bool ok;
        if (maxseg == 1) {
          cp.fused1 = std::make_shared<rbx::FusedArgsT<1>>();
          ok = fused_args_from_plan(c, host[0], ptrs, cp.fused1.get());
          if (!ok) cp.fused1.reset();
        } else {
          cp.fusedN = std::make_shared<rbx::FusedArgsT<RBX_FUSED_MAXSEG>>();
          ok = fused_args_from_plan(c, host[0], ptrs, cp.fusedN.get());
          if (!ok) cp.fusedN.reset();
        }
        if (ok) cp.fused_fn = fn;
      }
    }
    // the paper's per-dimension rings through the specialised kernel: whole aligned buffer,
    // 4/8-byte types (16-bit types keep fp32 stage partials in workspaces: generic kernel)
    const bool matched_stages = (mode == RBX_MODE_RING_DIMS && !one_ring && !ws) || (push && c->push_specialised);
    if (matched_stages && (op == RBX_OP_ALLREDUCE || op == RBX_OP_REDUCE_SCATTER) && nbufs == 1 && whole &&
        spec.mis == 0 && c->rings_specialised) {
      const void* fn = rings_kernel_for(dtype);
      int per_sm = 0;
      if (fn) RBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, c->threads, 0));
      if (fn && per_sm * c->sm_count >= c->nblocks) {
        cp.rings = std::make_shared<rbx::RingsArgs>();
        if (rings_args_from_plan(c, host[0], ptrs, cp.rings.get()))
          cp.rings_fn = fn;
        else
          cp.rings.reset();
      }
    }
    it = c->plans.emplace(key, cp).first;
  }
  // CTAs per call: enough to cover the bytes (bandwidth), few for small
  // messages (each CTA costs flag traffic and launch spread).  Every rank
  // derives the same value from the same counts.
  int nb = c->nblocks;
  if (op == RBX_OP_BARRIER) {
    nb = c->min_blocks;
  } else {
    const int64_t want = (int64_t)((total * (size_t)es + c->bytes_per_cta - 1) / c->bytes_per_cta);
    if (want < nb) nb = (int)(want < c->min_blocks ? c->min_blocks : want);
  }
  if (nb > c->nblocks) nb = c->nblocks;
  if (it->second.fused_fn) return fused_launch(c, it->second, stream, nb);
  if (it->second.rings_fn) return rings_launch(c, it->second, stream, nb);
  return launch(c, it->second, dtype, stream, false, nb);
}

}  // namespace

extern "C" {

int rbx_version(void) { return RBX_ABI_VERSION; }

const char* rbx_last_error(int* rank, int* stage) {
  if (rank) *rank = g_err_rank;
  if (stage) *stage = g_err_stage;
  return g_err.c_str();
}

int rbx_chunk_bounds(int64_t count, int64_t n_chunks, int64_t index, int64_t* off, int64_t* len) {
  if (n_chunks < 1) return fail(RBX_ERR_INVALID, "n_chunks must be >= 1, got " + std::to_string(n_chunks));
  if (index < 0 || index >= n_chunks)
    return fail(RBX_ERR_INVALID, "chunk index " + std::to_string(index) + " out of range");
  rbx::chunk_bounds(count, n_chunks, index, off, len);
  return RBX_OK;
}

int rbx_owned_region(const int* dims, int ndims, int rank, int64_t count, int64_t* off, int64_t* len) {
  rbx::Geometry g;
  std::string err;
  if (!g.init(dims, ndims, &err)) return fail(RBX_ERR_INVALID, err);
  if (rank < 0 || rank >= g.nranks) return fail(RBX_ERR_INVALID, "rank out of range");
  rbx::region_after(g, rank, count, (int)g.active_dims().size(), off, len);
  return RBX_OK;
}

int rbx_fold_order(const int* dims, int ndims, int rank, int* order_out) {
  rbx::Geometry g;
  std::string err;
  if (!g.init(dims, ndims, &err)) return fail(RBX_ERR_INVALID, err);
  if (rank < 0 || rank >= g.nranks) return fail(RBX_ERR_INVALID, "rank out of range");
  std::vector<int> o = rbx::fold_order(g, rank);
  for (size_t i = 0; i < o.size(); ++i) order_out[i] = o[i];
  return RBX_OK;
}

int64_t rbx_plan_describe(const int* dims, int ndims, int rank, int64_t count, int op, int mode, int dtype,
                          int64_t* out, int64_t cap) {
  rbx::Geometry g;
  std::string err;
  if (!g.init(dims, ndims, &err)) return fail(RBX_ERR_INVALID, err), -1;
  const int es = dtype_size(dtype);
  if (!es) return fail(RBX_ERR_INVALID, "unknown dtype"), -1;
  std::unique_ptr<rbx::Plan> p(new rbx::Plan);
  bool ok;
  if (mode == RBX_MODE_LOCAL)
    ok = rbx::build_local_plan(g, count, 16 / es, 0, 148, p.get(), &err);
  else {
    if (rank < 0 || rank >= g.nranks) return fail(RBX_ERR_INVALID, "rank out of range"), -1;
    rbx::PlanSpec spec;
    spec.op = (rbx::Op)op;
    spec.mode = (rbx::Mode)mode;
    spec.vec = 16 / es;
    ok = rbx::build_plan(g, rank, count, spec, 0, p.get(), true, &err);
  }
  if (!ok) return fail(RBX_ERR_INVALID, err), -1;
  return rbx::describe_plan(*p, out, cap);
}

int rbx_device_count(int* n) {
  RBX_CUDA(cudaGetDeviceCount(n));
  return RBX_OK;
}

int rbx_enable_peer_access(int device, int peer) {
  RBX_CUDA(cudaSetDevice(device));
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    (void)cudaGetLastError();
    return RBX_OK;
  }
  RBX_CUDA(e);
  return RBX_OK;
}

int rbx_alloc_symmetric(int device, size_t bytes, void** ptr, rbx_ipc_handle_t* handle) {
  RBX_CUDA(cudaSetDevice(device));
  RBX_CUDA(cudaMalloc(ptr, bytes ? bytes : 256));
  if (handle) {
    cudaIpcMemHandle_t h;
    RBX_CUDA(cudaIpcGetMemHandle(&h, *ptr));
    std::memcpy(handle->bytes, &h, sizeof(h));
  }
  return RBX_OK;
}

int rbx_free(void* ptr) {
  RBX_CUDA(cudaFree(ptr));
  return RBX_OK;
}

int rbx_export_buffer(void* ptr, rbx_ipc_handle_t* handle, uint64_t* offset) {
  // base of the allocation via the driver entry point (no link-time libcuda dependency)
  typedef CUresult (*range_fn)(CUdeviceptr*, size_t*, CUdeviceptr);
  static range_fn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    RBX_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !f) return fail(RBX_ERR_CUDA, "cuMemGetAddressRange unavailable");
    fn = reinterpret_cast<range_fn>(f);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) return fail(RBX_ERR_CUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  RBX_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle->bytes, &h, sizeof(h));
  *offset = (uint64_t)((CUdeviceptr)ptr - base);
  return RBX_OK;
}

int rbx_comm_create(rbx_comm_t** comm, int rank, int nranks, const int* dims, int ndims, int device, int nblocks,
                    int threads, rbx_ipc_handle_t* signal_handle) {
  std::unique_ptr<rbx_comm> c(new rbx_comm);
  int rc = common_init(c.get(), dims, ndims, device, threads);
  if (rc) return rc;
  if (c->geo.nranks != nranks)
    return fail(RBX_ERR_INVALID, "dims product " + std::to_string(c->geo.nranks) + " != nranks " + std::to_string(nranks));
  if (rank < 0 || rank >= nranks) return fail(RBX_ERR_INVALID, "rank out of range");
  c->rank = rank;
  c->nranks = nranks;
  if (nblocks <= 0) nblocks = c->sm_count;
  if (nblocks > RBX_MAX_BLOCKS) nblocks = RBX_MAX_BLOCKS;
  if (nblocks > c->max_coresident) nblocks = c->max_coresident;  // deadlock freedom: all CTAs resident
  c->nblocks = nblocks;
  RBX_CUDA(cudaMalloc(reinterpret_cast<void**>(&c->sig_local), sig_alloc_bytes(nranks)));
  RBX_CUDA(cudaMemset(c->sig_local, 0, sig_alloc_bytes(nranks)));
  cudaIpcMemHandle_t h;
  RBX_CUDA(cudaIpcGetMemHandle(&h, c->sig_local));
  std::memcpy(signal_handle->bytes, &h, sizeof(h));
  c->sig.assign(nranks, nullptr);
  c->sig[rank] = c->sig_local;
  c->ll_at.assign(nranks, nullptr);
  c->ll_at[rank] = ll_area_of(c->sig_local);
  RBX_CUDA(cudaDeviceSynchronize());
  *comm = c.release();
  return RBX_OK;
}

int rbx_comm_connect(rbx_comm_t* c, const rbx_ipc_handle_t* handles) {
  if (!c || c->nvirtual) return fail(RBX_ERR_INVALID, "not a per-rank communicator");
  RBX_CUDA(cudaSetDevice(c->device));
  for (int q = 0; q < c->nranks; ++q) {
    if (q == c->rank) continue;
    void* p = nullptr;
    int rc = open_handle(c, handles[q], &p);
    if (rc) return rc;
    c->sig[q] = static_cast<uint32_t*>(p);
    c->ll_at[q] = ll_area_of(c->sig[q]);
  }
  c->connected = true;
  return RBX_OK;
}

int rbx_comm_destroy(rbx_comm_t* c) {
  if (!c) return RBX_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (auto& kv : c->plans) free_plan(kv.second);
  for (auto& cp : c->retired) free_plan(cp);
  close_handles(c);
  if (c->sig_local) cudaFree(c->sig_local);
  if (c->trace_dev) cudaFree(c->trace_dev);
  if (c->order_ev) cudaEventDestroy(c->order_ev);
  if (c->inbox_owned && c->inbox_local) cudaFree(c->inbox_local);
  for (char* p : c->retired_inboxes) cudaFree(p);
  if (c->err_host) cudaFreeHost(c->err_host);
  delete c;
  return RBX_OK;
}

int rbx_comm_set_timeout(rbx_comm_t* c, double seconds) {
  if (!c || seconds <= 0) return fail(RBX_ERR_INVALID, "timeout must be > 0");
  c->timeout_ns = (uint64_t)(seconds * 1e9);
  return RBX_OK;
}

int rbx_comm_inject_fault(rbx_comm_t* c, double fraction) {
  if (!c) return fail(RBX_ERR_INVALID, "null communicator");
  if (!(fraction >= 0.0 && fraction <= 1.0)) return fail(RBX_ERR_INVALID, "fault fraction must be in [0, 1]");
  c->fault_milli = (int)(fraction * 1000.0 + 0.5);
  return RBX_OK;
}

int rbx_comm_trace(rbx_comm_t* c, uint64_t* out, int cap) {
  if (!c) return fail(RBX_ERR_INVALID, "null communicator");
  if (!c->trace_dev) return fail(RBX_ERR_INVALID, "tracing is off (set RBX_TRACE=1 before creating the communicator)");
  uint64_t buf[64];
  RBX_CUDA(cudaMemcpy(buf, c->trace_dev, sizeof(buf), cudaMemcpyDeviceToHost));
  for (int i = 0; i < cap && i < 64; ++i) out[i] = buf[i];
  return RBX_OK;
}

int rbx_comm_last_kernel(rbx_comm_t* c, int* kind) {
  if (!c || !kind) return fail(RBX_ERR_INVALID, "null argument");
  *kind = c->last_kernel;
  return RBX_OK;
}

int rbx_comm_info(rbx_comm_t* c, int* rank, int* nranks, int* nblocks, int* threads, uint64_t* launches) {
  if (!c) return fail(RBX_ERR_INVALID, "null communicator");
  if (rank) *rank = c->rank;
  if (nranks) *nranks = c->nranks;
  if (nblocks) *nblocks = c->nblocks;
  if (threads) *threads = c->threads;
  if (launches) *launches = c->launches;
  return RBX_OK;
}

int64_t rbx_inbox_bytes(const int* dims, int ndims, const size_t* counts, int nbufs, int dtype) {
  rbx::Geometry g;
  std::string err;
  if (!g.init(dims, ndims, &err)) return fail(RBX_ERR_INVALID, err), -1;
  const int es = dtype_size(dtype);
  if (!es) return fail(RBX_ERR_INVALID, "unknown dtype"), -1;
  int64_t total = 0;
  for (int k = 0; k < nbufs; ++k)
    if (counts[k]) total += rbx::inbox_buffer_bytes(g, (int64_t)counts[k], es);
  return total;
}

int rbx_set_inbox(rbx_comm_t* c, void* ptr, size_t bytes, const rbx_ipc_handle_t* handles, const uint64_t* offsets) {
  if (!c || c->nvirtual) return fail(RBX_ERR_INVALID, "not a per-rank communicator");
  RBX_CUDA(cudaSetDevice(c->device));
  RBX_CUDA(cudaDeviceSynchronize());  // no launch may still use the previous inbox
  std::vector<char*> at(c->nranks, nullptr);
  for (int q = 0; q < c->nranks; ++q) {
    if (q == c->rank) {
      at[q] = static_cast<char*>(ptr);
      continue;
    }
    void* p = nullptr;
    int rc = open_handle(c, handles[q], &p);
    if (rc) return rc;
    at[q] = static_cast<char*>(p) + offsets[q];
  }
  // cached MODE_PUSH / fp32-workspace plans point into the old inbox (retired, not freed,
  // if a captured graph may still replay them; the caller keeps the old inbox alive)
  if (int rc = drop_plans(c, true)) return rc;
  c->inbox_local = static_cast<char*>(ptr);
  c->inbox_bytes = bytes;
  c->inbox_at = at;
  return RBX_OK;
}

int rbx_register_buffer(rbx_comm_t* c, void* ptr, size_t bytes, const rbx_ipc_handle_t* handles,
                        const uint64_t* offsets, int* buf_id) {
  if (!c || c->nvirtual) return fail(RBX_ERR_INVALID, "not a per-rank communicator");
  RBX_CUDA(cudaSetDevice(c->device));
  RegBuf b;
  b.base = static_cast<char*>(ptr);
  b.bytes = bytes;
  b.at.assign(c->nranks, nullptr);
  for (int q = 0; q < c->nranks; ++q) {
    if (q == c->rank) {
      b.at[q] = b.base;
      continue;
    }
    void* p = nullptr;
    int rc = open_handle(c, handles[q], &p);
    if (rc) return rc;
    b.at[q] = static_cast<char*>(p) + offsets[q];
  }
  c->bufs.push_back(b);
  *buf_id = (int)c->bufs.size() - 1;
  return RBX_OK;
}

int rbx_fused_harness(const int* dims, int ndims, int rank, void* const* bufs, size_t count, int dtype, int nblocks,
                      int threads, void* stream) {
  // profiling harness: rank `rank`'s share of a FUSED allreduce through the specialised
  // kernel, with the flag protocol switched off (no entry/exit waits), so a profiler can
  // replay it without a peer; bufs[q] may live on any GPU with peer access
  rbx_comm tmp;
  std::string err;
  if (!tmp.geo.init(dims, ndims, &err)) return fail(RBX_ERR_INVALID, err);
  const int es = dtype_size(dtype);
  if (!es) return fail(RBX_ERR_INVALID, "unknown dtype");
  if (rank < 0 || rank >= tmp.geo.nranks) return fail(RBX_ERR_INVALID, "rank out of range");
  int dev = 0;
  RBX_CUDA(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::map<int, uint32_t*> scratch;  // per device: a signal area nobody else uses
  static std::map<int, rbx::ErrRecord*> errs;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!scratch.count(dev)) {
      uint32_t* p = nullptr;
      RBX_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), rbx::SigLayout::bytes));
      RBX_CUDA(cudaMemset(p, 0, rbx::SigLayout::bytes));
      scratch[dev] = p;
      rbx::ErrRecord* e = nullptr;
      RBX_CUDA(cudaMalloc(reinterpret_cast<void**>(&e), sizeof(rbx::ErrRecord)));
      RBX_CUDA(cudaMemset(e, 0, sizeof(rbx::ErrRecord)));
      errs[dev] = e;
    }
  }
  tmp.rank = rank;
  tmp.nranks = tmp.geo.nranks;
  tmp.threads = threads > 0 ? threads : 512;
  tmp.sig.assign(tmp.nranks, scratch[dev]);
  std::vector<void*> table(bufs, bufs + tmp.nranks);
  std::unique_ptr<rbx::Plan> plan(new rbx::Plan);
  rbx::PlanSpec spec;
  spec.op = rbx::OP_ALLREDUCE;
  spec.mode = rbx::MODE_FUSED;
  spec.vec = 16 / es;
  spec.mis = misalign(table, es);
  if (!rbx::build_plan(tmp.geo, rank, (int64_t)count, spec, 0, plan.get(), true, &err)) return fail(RBX_ERR_INVALID, err);
  const void* fn = fused_kernel_for(dtype, tmp.nranks, (int)tmp.geo.active_dims().size(), tmp.nranks, 1);
  if (!fn) return fail(RBX_ERR_UNSUPPORTED, "no specialised fused kernel for this grid");
  rbx::FusedArgsT<1> a;
  if (!fused_args_from_plan(&tmp, *plan, table, &a)) return fail(RBX_ERR_UNSUPPORTED, "plan shape");
  a.timeout_ns = 1000000000ull;
  a.err = errs[dev];
  a.trace = nullptr;
  a.fault_milli = -1;
  a.dbg = 1 | 2 | 8;  // relaxed exit flag into the scratch area, no exit wait, no entry handshake
  void* params[] = {&a};
  RBX_CUDA(cudaLaunchKernel(fn, dim3((unsigned)(nblocks > 0 ? nblocks : 148)), dim3((unsigned)tmp.threads), params, 0,
                            (cudaStream_t)stream));
  return RBX_OK;
}

int rbx_host_register(void* ptr, size_t bytes, int* registered) {
  if (registered) *registered = 0;
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, ptr) == cudaSuccess && attr.type == cudaMemoryTypeHost)
    return RBX_OK;  // already page-locked (cudaHostAlloc / pinned allocator): nothing to do
  (void)cudaGetLastError();
  const cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterDefault);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();  // not sticky: do not leave it for the next caller's error check
    if (e == cudaErrorHostMemoryAlreadyRegistered) return RBX_OK;
    return fail(RBX_ERR_CUDA, std::string("cudaHostRegister: ") + cudaGetErrorString(e));
  }
  if (registered) *registered = 1;
  return RBX_OK;
}

int rbx_host_unregister(void* ptr) {
  const cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return fail(RBX_ERR_CUDA, std::string("cudaHostUnregister: ") + cudaGetErrorString(e));
  }
  return RBX_OK;
}

int rbx_stamp(uint64_t* dst, void* stream) {
  stamp_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(dst);
  RBX_CUDA(cudaGetLastError());
  return RBX_OK;
}

int rbx_peer_pointer(rbx_comm_t* c, const void* buf, int rank, void** out) {
  if (!c || c->nvirtual) return fail(RBX_ERR_INVALID, "not a per-rank communicator");
  if (rank < 0 || rank >= c->nranks) return fail(RBX_ERR_INVALID, "rank out of range");
  int id;
  size_t off;
  if (int rc = find_buffer(c, buf, 1, &id, &off)) return rc;
  *out = c->bufs[id].at[rank] + off;
  return RBX_OK;
}

int rbx_allreduce(rbx_comm_t* c, void* buf, size_t count, int dtype, int mode, void* stream) {
  void* bufs[1] = {buf};
  size_t counts[1] = {count};
  return real_collective(c, bufs, counts, 1, dtype, RBX_OP_ALLREDUCE, mode, (cudaStream_t)stream);
}

int rbx_reduce_scatter(rbx_comm_t* c, void* buf, size_t count, int dtype, int mode, void* stream, int64_t* owned_off,
                       int64_t* owned_len) {
  void* bufs[1] = {buf};
  size_t counts[1] = {count};
  int rc = real_collective(c, bufs, counts, 1, dtype, RBX_OP_REDUCE_SCATTER, mode, (cudaStream_t)stream);
  if (rc) return rc;
  int64_t o, l;
  rbx::region_after(c->geo, c->rank, (int64_t)count, (int)c->geo.active_dims().size(), &o, &l);
  if (owned_off) *owned_off = o;
  if (owned_len) *owned_len = l;
  return RBX_OK;
}

int rbx_allgather(rbx_comm_t* c, void* buf, size_t count, int dtype, int mode, void* stream) {
  void* bufs[1] = {buf};
  size_t counts[1] = {count};
  return real_collective(c, bufs, counts, 1, dtype, RBX_OP_ALLGATHER, mode, (cudaStream_t)stream);
}

int rbx_allreduce_buckets(rbx_comm_t* c, void* const* bufs, const size_t* counts, int nbufs, int dtype, int mode,
                          void* stream) {
  if (!c) return fail(RBX_ERR_INVALID, "null communicator");
  if (nbufs < 1) return fail(RBX_ERR_INVALID, "empty bucket list");
  if ((int64_t)nbufs * c->nranks > 4096) return fail(RBX_ERR_INVALID, "bucket list too long");
  return real_collective(c, bufs, counts, nbufs, dtype, RBX_OP_ALLREDUCE, mode, (cudaStream_t)stream);
}

int rbx_barrier(rbx_comm_t* c, void* stream) {
  void* bufs[1] = {nullptr};
  size_t counts[1] = {0};
  return real_collective(c, bufs, counts, 1, RBX_F32, RBX_OP_BARRIER, RBX_MODE_FUSED, (cudaStream_t)stream);
}

int rbx_check(rbx_comm_t* c) {
  if (!c) return fail(RBX_ERR_INVALID, "null communicator");
  if (c->err_host->code) {
    return fail(RBX_ERR_COLLECTIVE,
                "collective watchdog: rank " + std::to_string(c->err_host->rank) + " timed out at plan step " +
                    std::to_string(c->err_host->step) + " waiting for rank " + std::to_string(c->err_host->peer),
                c->err_host->peer, c->err_host->step);
  }
  return RBX_OK;
}

int rbx_vcomm_create(rbx_comm_t** comm, int nranks, const int* dims, int ndims, int device, int nblocks_per_rank,
                     int threads) {
  std::unique_ptr<rbx_comm> c(new rbx_comm);
  int rc = common_init(c.get(), dims, ndims, device, threads);
  if (rc) return rc;
  if (c->geo.nranks != nranks)
    return fail(RBX_ERR_INVALID, "dims product " + std::to_string(c->geo.nranks) + " != nranks " + std::to_string(nranks));
  c->nranks = nranks;
  c->nvirtual = nranks;
  int nb = nblocks_per_rank > 0 ? nblocks_per_rank : c->max_coresident / nranks;
  if (nb < 1) nb = 1;
  if (nb > RBX_MAX_BLOCKS) nb = RBX_MAX_BLOCKS;
  c->nblocks = nb;
  const size_t stride = sig_alloc_bytes(nranks);  // per virtual rank: signal area + LL area
  RBX_CUDA(cudaMalloc(reinterpret_cast<void**>(&c->sig_local), stride * nranks));
  RBX_CUDA(cudaMemset(c->sig_local, 0, stride * nranks));
  c->sig.resize(nranks);
  c->ll_at.resize(nranks);
  for (int q = 0; q < nranks; ++q) {
    c->sig[q] = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(c->sig_local) + stride * q);
    c->ll_at[q] = ll_area_of(c->sig[q]);
  }
  c->connected = true;
  RBX_CUDA(cudaDeviceSynchronize());
  *comm = c.release();
  return RBX_OK;
}

int rbx_vcollective(rbx_comm_t* c, void* const* bufs, size_t count, int dtype, int op, int mode, void* stream) {
  return rbx_vcollective_window(c, bufs, count, 0, count, dtype, op, mode, stream);
}

int rbx_allreduce_window(rbx_comm_t* c, void* buf, size_t count, size_t lo, size_t hi, int dtype, int mode,
                         void* stream) {
  if (lo > hi || hi > count) return fail(RBX_ERR_INVALID, "window must satisfy lo <= hi <= count");
  void* bufs[1] = {buf};
  size_t counts[1] = {count};
  return real_collective(c, bufs, counts, 1, dtype, RBX_OP_ALLREDUCE, mode, (cudaStream_t)stream, (int64_t)lo,
                         (int64_t)hi);
}

int rbx_vcollective_window(rbx_comm_t* c, void* const* bufs, size_t count, size_t lo, size_t hi, int dtype, int op,
                           int mode, void* stream) {
  if (lo > hi || hi > count) return fail(RBX_ERR_INVALID, "window must satisfy lo <= hi <= count");
  if (!c || !c->nvirtual) return fail(RBX_ERR_INVALID, "not a virtual communicator");
  const int es = dtype_size(dtype);
  if (!es) return fail(RBX_ERR_INVALID, "unknown dtype");
  if (c->err_host->code) return fail(RBX_ERR_COLLECTIVE, "communicator is in an error state", c->err_host->peer, c->err_host->step);
  if (int rc = check_mode_dtype(mode, dtype)) return rc;
  const int V = c->nvirtual;
  if (mode == RBX_MODE_LL) {
    if (op != RBX_OP_ALLREDUCE || lo != 0 || hi != count)
      return fail(RBX_ERR_INVALID, "MODE_LL supports a whole-buffer single allreduce only");
    if (count == 0) return RBX_OK;
    std::vector<int> ranks;
    for (int r = 0; r < V; ++r) ranks.push_back(r);
    return ll_launch(c, ranks, bufs, count, dtype, (cudaStream_t)stream, true);
  }
  std::vector<const void*> kp(bufs, bufs + V);
  const std::string key =
      plan_key(op, mode, dtype, kp, {count}) + "@" + std::to_string(lo) + ":" + std::to_string(hi);
  auto it = c->plans.find(key);
  const bool local = (mode == RBX_MODE_LOCAL);
  if (local && op != RBX_OP_ALLREDUCE) return fail(RBX_ERR_INVALID, "MODE_LOCAL supports allreduce only");
  int nb = c->nblocks;
  if (local) nb = c->max_coresident > 0 ? c->max_coresident : c->sm_count;
  if (nb > RBX_MAX_BLOCKS) nb = RBX_MAX_BLOCKS;
  const bool push = mode == RBX_MODE_PUSH && (op == RBX_OP_ALLREDUCE || op == RBX_OP_REDUCE_SCATTER);
  const bool ws = needs_fp32_partials(c->geo, mode, dtype, op);
  if (push || ws) {  // virtual ranks share this process: one local allocation holds every rank's inbox
    const int64_t need = rbx::inbox_buffer_bytes(c->geo, (int64_t)count, es);
    if ((int64_t)c->inbox_bytes < need) {
      RBX_CUDA(cudaSetDevice(c->device));
      RBX_CUDA(cudaDeviceSynchronize());
      if (c->captured) {  // a captured graph may replay plans that address the old inbox
        if (c->inbox_local) c->retired_inboxes.push_back(c->inbox_local);
      } else if (c->inbox_local) {
        cudaFree(c->inbox_local);
      }
      c->inbox_local = nullptr;
      c->inbox_bytes = 0;
      if (int rc = drop_plans(c, true)) return rc;
      RBX_CUDA(cudaMalloc(reinterpret_cast<void**>(&c->inbox_local), (size_t)need * V));
      c->inbox_owned = true;
      c->inbox_bytes = (size_t)need;
      c->inbox_at.assign(V, nullptr);
      for (int r = 0; r < V; ++r) c->inbox_at[r] = c->inbox_local + (size_t)need * r;
      it = c->plans.find(key);
    }
  }
  if (it == c->plans.end()) {
    if (int rc = bound_plans(c)) return rc;
    std::string err;
    std::vector<void*> ptrs(bufs, bufs + V);
    std::vector<rbx::Plan> host(local ? 1 : V);
    std::vector<std::vector<void*>> tables{ptrs};
    const int mis = misalign(ptrs, es);
    if (local) {
      if (!rbx::build_local_plan(c->geo, (int64_t)count, 16 / es, mis, nb, &host[0], &err, (int64_t)lo, (int64_t)hi))
        return fail(RBX_ERR_INVALID, err);
    } else {
      rbx::PlanSpec spec;
      spec.op = (rbx::Op)op;
      spec.mode = (rbx::Mode)mode;
      spec.vec = 16 / es;
      spec.mis = mis;
      spec.nblocks = nb;
      spec.lo = (int64_t)lo;
      spec.hi = (int64_t)hi;
      spec.partials_fp32 = ws;
      if (push) tables.clear();
      if (ws) {
        std::vector<char*> cb;
        for (void* p : ptrs) cb.push_back(static_cast<char*>(p));
        tables = {ws_table(c->geo, (int64_t)count, es, mis, cb, c->inbox_at, 0)};
      }
      for (int r = 0; r < V; ++r) {
        if (!rbx::build_plan(c->geo, r, (int64_t)count, spec, 0, &host[r], true, &err)) return fail(RBX_ERR_INVALID, err);
        for (int q = 0; q < V; ++q) host[r].sig[q] = c->sig[q];
        host[r].my_sig = c->sig[r];
        if (push) {
          std::vector<char*> cb;
          for (void* p : ptrs) cb.push_back(static_cast<char*>(p));
          tables.push_back(push_table(c->geo, r, (int64_t)count, es, mis, cb, c->inbox_at, 0));
        }
      }
    }
    CachedPlan cp;
    cp.uses_inbox = push || ws;
    int rc = upload(c, host, tables, &cp, dtype);
    if (rc) return rc;
    if (local && c->local_specialised) {
      const void* fn = local_kernel_for(dtype, V, (int)c->geo.active_dims().size());
      auto args = std::make_shared<rbx::LocalArgs>();
      if (fn && local_args_from_plan(host[0], ptrs, args.get())) {
        args->hint = c->local_hint;
        int per_sm = 0;
        RBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, c->threads, 0));
        cp.local_fn = fn;
        cp.local_args = args;
        if (c->local_ctas_per_sm > 0) per_sm = std::min(per_sm, c->local_ctas_per_sm);
        cp.local_grid = std::max(1, per_sm) * c->sm_count;
      }
    }
    it = c->plans.emplace(key, cp).first;
  }
  if (it->second.local_fn) {  // specialised local-reduce kernel (no step table, no flags)
    void* params[] = {it->second.local_args.get()};
    bool capturing = false;
    if (int rc = order_before(c, (cudaStream_t)stream, &capturing)) return rc;
    RBX_CUDA(cudaLaunchKernel(it->second.local_fn, dim3((unsigned)it->second.local_grid), dim3((unsigned)c->threads),
                              params, 0, (cudaStream_t)stream));
    c->launches++;
    c->last_kernel = RBX_KERNEL_LOCAL;
    return order_after(c, (cudaStream_t)stream, capturing);
  }
  if (!local && (int64_t)nb * V > c->max_coresident)
    return fail(RBX_ERR_INVALID, "virtual ranks x blocks exceed co-resident CTAs");
  return launch(c, it->second, dtype, (cudaStream_t)stream, !local, nb);
}

}  // extern "C"
