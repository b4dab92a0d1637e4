/*
 * CPU ORACLE (plain C) for the multi-ring allreduce -- TEST INFRASTRUCTURE ONLY.
 *
 * A C restatement of the reference `ringbox` hot path
 * (/root/reference/pkg/src/ringbox, v0.1.0) used as
 *   (1) a fast checker for the GPU results (tests/), and
 *   (2) the CPU baseline / `bench.py --impl reference` arm ("kind": "port"):
 *       the reference runtime's per-rank phase loop with the TCP socket
 *       replaced by an in-memory mailbox, one thread per rank.
 * The product library (paper_1708_02188_b200/librbx.so) never links this.
 *
 * Restated reference functions:
 *   orc_chunk_bounds  -- pkg/src/ringbox/ring.py:57-70
 *   orc_schedule      -- pkg/src/ringbox/multiring.py:170-211 built from
 *                        ring_pass_transfers pkg/src/ringbox/ring.py:73-103 and
 *                        Grid.rings pkg/src/ringbox/multiring.py:48-55
 *   orc_replay        -- pkg/src/ringbox/ring.py:172-192 (phase-synchronous,
 *                        payloads staged from the pre-phase state)
 *   orc_runtime_port  -- pkg/src/ringbox/runtime.py:199-267 (_run_phases):
 *                        per phase each rank sends one chunk to its ring
 *                        successor and ADDs/REPLACEs the chunk received from its
 *                        predecessor; synchronisation is pairwise (dataflow),
 *                        not a global barrier, exactly like the socket runtime.
 * Pinned against the reference's golden digests in tests/test_oracle.py.
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <sched.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define ORC_MAX_RANKS 64
#define ORC_MAX_DIMS 8

enum { ORC_F32 = 0, ORC_F64 = 1, ORC_I64 = 2 };

typedef struct {
  int32_t src, dst, chunk, add;
  int64_t off, len;
} orc_transfer;

static size_t dtype_size(int dt) { return dt == ORC_F32 ? 4 : 8; }

int orc_chunk_bounds(int64_t count, int64_t n, int64_t i, int64_t *off, int64_t *len) {
  if (n < 1 || i < 0 || i >= n) return -1;
  int64_t q = count / n, r = count % n;
  if (i < r) {
    *off = i * (q + 1);
    *len = q + 1;
  } else {
    *off = r * (q + 1) + (i - r) * q;
    *len = q;
  }
  return 0;
}

static void coords_of(const int *dims, int nd, int rank, int *c) {
  for (int i = 0; i < nd; ++i) {
    c[i] = rank % dims[i];
    rank /= dims[i];
  }
}

static int rank_of(const int *dims, int nd, const int *c) {
  int r = 0, s = 1;
  for (int i = 0; i < nd; ++i) {
    r += c[i] * s;
    s *= dims[i];
  }
  return r;
}

/* Ring of `rank` along `dim`, ordered by the coordinate (Grid.rings). */
static void ring_members(const int *dims, int nd, int rank, int dim, int *members) {
  int c[ORC_MAX_DIMS];
  coords_of(dims, nd, rank, c);
  for (int j = 0; j < dims[dim]; ++j) {
    c[dim] = j;
    members[j] = rank_of(dims, nd, c);
  }
}

/* Emit the transfers of one ring pass (ring_pass_transfers) into phases
 * [phase0, phase0+d-1) of `out`; each phase row holds `n` transfers. */
static void ring_pass(const int *members, int d, int64_t off, int64_t len, int rs, orc_transfer *out,
                      int n, int phase0, int *fill) {
  for (int j = 0; j < d - 1; ++j) {
    for (int p = 0; p < d; ++p) {
      int c = rs ? ((p - j) % d + d) % d : ((p + 1 - j) % d + d) % d;
      int64_t o, l;
      orc_chunk_bounds(len, d, c, &o, &l);
      orc_transfer *t = &out[(size_t)(phase0 + j) * n + fill[phase0 + j]++];
      t->src = members[p];
      t->dst = members[(p + 1) % d];
      t->chunk = c;
      t->add = rs;
      t->off = off + o;
      t->len = l;
    }
  }
}

/* Build the composite schedule.  `out` must hold nphases*n transfers where
 * nphases = 2*sum(d_i - 1).  Returns the number of phases (or -1). */
int orc_schedule(const int *dims, int nd, int64_t count, orc_transfer *out, int max_phases) {
  int n = 1, nph = 0;
  if (nd < 1 || nd > ORC_MAX_DIMS) return -1;
  for (int i = 0; i < nd; ++i) {
    if (dims[i] < 1) return -1;
    n *= dims[i];
    nph += 2 * (dims[i] - 1);
  }
  if (n > ORC_MAX_RANKS || nph > max_phases) return -1;
  int *fill = calloc((size_t)nph + 1, sizeof(int));
  int64_t *roff = malloc(sizeof(int64_t) * n), *rlen = malloc(sizeof(int64_t) * n);
  int64_t *soff = malloc(sizeof(int64_t) * n * nd), *slen = malloc(sizeof(int64_t) * n * nd);
  for (int r = 0; r < n; ++r) {
    roff[r] = 0;
    rlen[r] = count;
  }
  int members[ORC_MAX_RANKS], c[ORC_MAX_DIMS];
  int phase = 0;
  for (int dim = 0; dim < nd; ++dim) {
    for (int r = 0; r < n; ++r) {
      soff[r * nd + dim] = roff[r];
      slen[r * nd + dim] = rlen[r];
    }
    int d = dims[dim];
    if (d == 1) continue;
    /* one ring per rank whose coord[dim] == 0 (multiring.py:182-197) */
    int64_t *noff = malloc(sizeof(int64_t) * n), *nlen = malloc(sizeof(int64_t) * n);
    memcpy(noff, roff, sizeof(int64_t) * n);
    memcpy(nlen, rlen, sizeof(int64_t) * n);
    for (int r = 0; r < n; ++r) {
      coords_of(dims, nd, r, c);
      if (c[dim] != 0) continue;
      ring_members(dims, nd, r, dim, members);
      int64_t off = roff[members[0]], len = rlen[members[0]];
      ring_pass(members, d, off, len, 1, out, n, phase, fill);
      for (int p = 0; p < d; ++p) {
        int64_t o, l;
        orc_chunk_bounds(len, d, (p + 1) % d, &o, &l);
        noff[members[p]] = off + o;
        nlen[members[p]] = l;
      }
    }
    memcpy(roff, noff, sizeof(int64_t) * n);
    memcpy(rlen, nlen, sizeof(int64_t) * n);
    free(noff);
    free(nlen);
    phase += d - 1;
  }
  for (int dim = nd - 1; dim >= 0; --dim) {
    int d = dims[dim];
    if (d == 1) continue;
    for (int r = 0; r < n; ++r) {
      coords_of(dims, nd, r, c);
      if (c[dim] != 0) continue;
      ring_members(dims, nd, r, dim, members);
      ring_pass(members, d, soff[members[0] * nd + dim], slen[members[0] * nd + dim], 0, out, n, phase,
                fill);
    }
    phase += d - 1;
  }
  free(fill);
  free(roff);
  free(rlen);
  free(soff);
  free(slen);
  return phase;
}

static void apply(int dt, int add, void *dst, const void *src, int64_t len) {
  if (!add) {
    memcpy(dst, src, (size_t)len * dtype_size(dt));
    return;
  }
  if (dt == ORC_F32) {
    float *a = dst;
    const float *b = src;
    for (int64_t i = 0; i < len; ++i) a[i] = a[i] + b[i];
  } else if (dt == ORC_F64) {
    double *a = dst;
    const double *b = src;
    for (int64_t i = 0; i < len; ++i) a[i] = a[i] + b[i];
  } else {
    uint64_t *a = dst; /* wrapping int64 add, as numpy */
    const uint64_t *b = src;
    for (int64_t i = 0; i < len; ++i) a[i] = a[i] + b[i];
  }
}

static int nphases_of(const int *dims, int nd, int *n) {
  int p = 0;
  *n = 1;
  for (int i = 0; i < nd; ++i) {
    p += 2 * (dims[i] - 1);
    *n *= dims[i];
  }
  return p;
}

/* replay(multiring_schedule(Grid(dims), count), bufs) in place. */
int orc_replay(const int *dims, int nd, int64_t count, int dt, void **bufs) {
  int n, nph = nphases_of(dims, nd, &n);
  orc_transfer *sched = malloc(sizeof(orc_transfer) * ((size_t)nph * n + 1));
  if (orc_schedule(dims, nd, count, sched, nph) < 0) {
    free(sched);
    return -1;
  }
  size_t es = dtype_size(dt);
  int64_t maxlen = 0;
  for (size_t i = 0; i < (size_t)nph * n; ++i)
    if (sched[i].len > maxlen) maxlen = sched[i].len;
  char **stage = malloc(sizeof(char *) * n);
  for (int i = 0; i < n; ++i) stage[i] = malloc((size_t)maxlen * es + 64);
  for (int p = 0; p < nph; ++p) {
    orc_transfer *row = &sched[(size_t)p * n];
    for (int t = 0; t < n; ++t)
      memcpy(stage[t], (char *)bufs[row[t].src] + row[t].off * es, (size_t)row[t].len * es);
    for (int t = 0; t < n; ++t) apply(dt, row[t].add, (char *)bufs[row[t].dst] + row[t].off * es, stage[t], row[t].len);
  }
  for (int i = 0; i < n; ++i) free(stage[i]);
  free(stage);
  free(sched);
  return 0;
}

/* ---------------- runtime port: one thread per rank, mailbox "sockets" ---------------- */

typedef struct {
  const orc_transfer *sched;
  int n, nph, dt;
  void **bufs;
  char **outbox;               /* per-rank staging = the serialised frame payload */
  volatile int64_t *sent;      /* sent[r] = phases whose payload rank r has posted */
  volatile int64_t *consumed;  /* consumed[r] = phases of rank r's payload applied by its receiver */
  volatile int *go;
} port_ctx;

typedef struct {
  port_ctx *ctx;
  int rank;
} port_arg;

static void spin_until(volatile int64_t *v, int64_t target) {
  int spins = 0;
  while (__atomic_load_n(v, __ATOMIC_ACQUIRE) < target)
    if (++spins > 64) {
      sched_yield();
      spins = 0;
    }
}

static void *port_worker(void *p) {
  port_arg *a = p;
  port_ctx *c = a->ctx;
  int me = a->rank;
  size_t es = dtype_size(c->dt);
  while (!__atomic_load_n(c->go, __ATOMIC_ACQUIRE)) sched_yield();
  for (int ph = 0; ph < c->nph; ++ph) {
    const orc_transfer *row = &c->sched[(size_t)ph * c->n];
    const orc_transfer *snd = NULL, *rcv = NULL;
    for (int t = 0; t < c->n; ++t) { /* runtime.py:205-209 */
      if (row[t].src == me) snd = &row[t];
      if (row[t].dst == me) rcv = &row[t];
    }
    if (snd) { /* do_send: tobytes + sendall (runtime.py:213-220) */
      spin_until(&c->consumed[me], ph);
      memcpy(c->outbox[me], (char *)c->bufs[me] + snd->off * es, (size_t)snd->len * es);
      __atomic_store_n(&c->sent[me], ph + 1, __ATOMIC_RELEASE);
    }
    if (rcv) { /* recv + view += payload / view[:] = payload (runtime.py:228-251) */
      spin_until(&c->sent[rcv->src], ph + 1);
      apply(c->dt, rcv->add, (char *)c->bufs[me] + rcv->off * es, c->outbox[rcv->src], rcv->len);
      __atomic_store_n(&c->consumed[rcv->src], ph + 1, __ATOMIC_RELEASE);
    }
  }
  return NULL;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + ts.tv_nsec * 1e-9;
}

/* Runs the allreduce in place over `bufs` with one thread per rank; returns
 * the wall time of the collective (threads already created and parked). */
int orc_runtime_port(const int *dims, int nd, int64_t count, int dt, void **bufs, double *seconds) {
  int n, nph = nphases_of(dims, nd, &n);
  orc_transfer *sched = malloc(sizeof(orc_transfer) * ((size_t)nph * n + 1));
  if (orc_schedule(dims, nd, count, sched, nph) < 0) {
    free(sched);
    return -1;
  }
  size_t es = dtype_size(dt);
  int64_t maxlen = 0;
  for (size_t i = 0; i < (size_t)nph * n; ++i)
    if (sched[i].len > maxlen) maxlen = sched[i].len;
  port_ctx ctx;
  volatile int go = 0;
  ctx.sched = sched;
  ctx.n = n;
  ctx.nph = nph;
  ctx.dt = dt;
  ctx.bufs = bufs;
  ctx.outbox = malloc(sizeof(char *) * n);
  ctx.sent = calloc(n, sizeof(int64_t));
  ctx.consumed = calloc(n, sizeof(int64_t));
  ctx.go = &go;
  for (int r = 0; r < n; ++r) {
    ctx.outbox[r] = malloc((size_t)maxlen * es + 64);
    memset(ctx.outbox[r], 0, (size_t)maxlen * es + 64); /* fault pages in outside the timing */
  }
  pthread_t *th = malloc(sizeof(pthread_t) * n);
  port_arg *args = malloc(sizeof(port_arg) * n);
  for (int r = 0; r < n; ++r) {
    args[r].ctx = &ctx;
    args[r].rank = r;
    pthread_create(&th[r], NULL, port_worker, &args[r]);
  }
  double t0 = now_s();
  __atomic_store_n(&go, 1, __ATOMIC_RELEASE);
  for (int r = 0; r < n; ++r) pthread_join(th[r], NULL);
  double t1 = now_s();
  if (seconds) *seconds = t1 - t0;
  for (int r = 0; r < n; ++r) free(ctx.outbox[r]);
  free(ctx.outbox);
  free((void *)ctx.sent);
  free((void *)ctx.consumed);
  free(th);
  free(args);
  free(sched);
  return 0;
}
