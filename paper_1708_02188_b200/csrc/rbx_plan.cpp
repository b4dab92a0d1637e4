// Host-side plan builder: grid geometry, remainder-first chunking and the
// per-rank step tables executed by the sm_100a kernel (see rbx_plan.h).
//
// Semantics follow the reference exactly:
//   chunk_bounds       pkg/src/ringbox/ring.py:57-70
//   Grid coords/rings  pkg/src/ringbox/multiring.py:32-55 (dim 0 fastest)
//   region shrinking   pkg/src/ringbox/multiring.py:186-197, owned_region runtime.py:187-196
//   fold order         ring.py:73-103 RS phase j: position p forwards chunk (p-j) mod d, so
//                      chunk c is folded starting at ring position c and the owner
//                      (position c-1) adds last; nested over dims (multiring.py:180-197).
#include "rbx_plan.h"

#include <algorithm>
#include <cstring>

namespace rbx {

bool Geometry::init(const int* d, int nd, std::string* err) {
  dims.assign(d, d + nd);
  nranks = 1;
  if (nd < 1) {
    if (err) *err = "dims must not be empty";
    return false;
  }
  for (int x : dims) {
    if (x < 1) {
      if (err) *err = "dimension sizes must be >= 1";
      return false;
    }
    nranks *= x;
    if (nranks > RBX_MAX_RANKS) {
      if (err) *err = "at most 16 ranks per box are supported";
      return false;
    }
  }
  if ((int)active_dims().size() > RBX_MAX_LEVELS) {
    if (err) *err = "at most 4 non-singleton dimensions are supported";
    return false;
  }
  return true;
}

void Geometry::coords(int rank, int* c) const {
  for (size_t i = 0; i < dims.size(); ++i) {
    c[i] = rank % dims[i];
    rank /= dims[i];
  }
}

int Geometry::rank_of(const int* c) const {
  int r = 0, stride = 1;
  for (size_t i = 0; i < dims.size(); ++i) {
    r += c[i] * stride;
    stride *= dims[i];
  }
  return r;
}

std::vector<int> Geometry::ring(int rank, int dim) const {
  int c[16];
  coords(rank, c);
  std::vector<int> out;
  for (int j = 0; j < dims[dim]; ++j) {
    c[dim] = j;
    out.push_back(rank_of(c));
  }
  return out;
}

std::vector<int> Geometry::active_dims() const {
  std::vector<int> a;
  for (size_t i = 0; i < dims.size(); ++i)
    if (dims[i] > 1) a.push_back((int)i);
  return a;
}

void chunk_bounds(int64_t count, int64_t n, int64_t i, int64_t* off, int64_t* len) {
  const int64_t q = count / n, r = count % n;
  if (i < r) {
    *off = i * (q + 1);
    *len = q + 1;
  } else {
    *off = r * (q + 1) + (i - r) * q;
    *len = q;
  }
}

void region_after(const Geometry& g, int rank, int64_t count, int upto_active, int64_t* off, int64_t* len) {
  int c[16];
  g.coords(rank, c);
  int64_t o = 0, l = count;
  const std::vector<int> act = g.active_dims();
  for (int i = 0; i < upto_active && i < (int)act.size(); ++i) {
    const int dim = act[i], d = g.dims[dim];
    int64_t so, sl;
    chunk_bounds(l, d, (c[dim] + 1) % d, &so, &sl);
    o += so;
    l = sl;
  }
  *off = o;
  *len = l;
}

std::vector<int> fold_order(const Geometry& g, int rank) {
  const std::vector<int> act = g.active_dims();
  int c[16];
  g.coords(rank, c);
  int start[16];
  for (size_t i = 0; i < g.dims.size(); ++i) start[i] = (c[i] + 1) % g.dims[i];
  // mixed radix over the active dims, active[0] fastest; digit j_L of level L
  // maps to coordinate (start_L + j_L) mod d_L.
  std::vector<int> order;
  const int n = g.nranks;
  for (int j = 0; j < n; ++j) {
    int cc[16];
    std::memcpy(cc, c, sizeof(cc));
    int rem = j;
    for (int dim : act) {
      const int d = g.dims[dim];
      cc[dim] = (start[dim] + rem % d) % d;
      rem /= d;
    }
    order.push_back(g.rank_of(cc));
  }
  return order;
}

std::vector<uint8_t> fold_ctrl(const Geometry& g) {
  const std::vector<int> act = g.active_dims();
  const int m = (int)act.size();
  std::vector<uint8_t> ctrl;
  for (int j = 0; j < g.nranks; ++j) {
    uint8_t starts = 0;
    int ending = 0, rem = j;
    bool chain = true;
    for (int L = 0; L < m; ++L) {
      const int d = g.dims[act[L]], digit = rem % d;
      rem /= d;
      if (digit == 0) starts |= (uint8_t)(1u << L);
      if (chain && digit == d - 1)
        ++ending;
      else
        chain = false;
    }
    const int e = std::min(ending, std::max(m - 1, 0));
    ctrl.push_back((uint8_t)(starts | (e << 4)));
  }
  return ctrl;
}

namespace {

struct StepProto {
  std::vector<Wait> waits;
  std::vector<int> sigs;
};

std::vector<int> without(const std::vector<int>& v, int x) {
  std::vector<int> o;
  for (int y : v)
    if (y != x) o.push_back(y);
  return o;
}

// members rotated so the list starts after `me` (spreads peer traffic)
std::vector<int> rotated_after(const std::vector<int>& members, int me) {
  auto it = std::find(members.begin(), members.end(), me);
  std::vector<int> o;
  const size_t n = members.size();
  size_t p = (it == members.end()) ? 0 : (size_t)(it - members.begin()) + 1;
  for (size_t j = 0; j < n; ++j) o.push_back(members[(p + j) % n]);
  return o;
}

void add_waits(std::vector<Wait>& w, int slot, const std::vector<int>& peers, bool all) {
  for (int q : peers) w.push_back(Wait{(uint8_t)slot, (uint8_t)q, (uint8_t)(all ? 1 : 0), 0});
}

bool push_step(Plan* p, const StepProto& s, std::string* err) {
  if (p->nsteps >= RBX_MAX_STEPS) {
    if (err) *err = "plan has too many steps";
    return false;
  }
  Step& st = p->steps[p->nsteps];
  int wbase = p->nsteps ? p->steps[p->nsteps - 1].wait0 + p->steps[p->nsteps - 1].nwait : 0;
  int sbase = p->nsteps ? p->steps[p->nsteps - 1].sig0 + p->steps[p->nsteps - 1].nsig : 0;
  if (wbase + (int)s.waits.size() > RBX_MAX_WAITS || sbase + (int)s.sigs.size() > RBX_MAX_SIGS) {
    if (err) *err = "plan has too many waits/signals";
    return false;
  }
  st.wait0 = wbase;
  st.nwait = (int)s.waits.size();
  for (size_t i = 0; i < s.waits.size(); ++i) p->waits[wbase + i] = s.waits[i];
  st.sig0 = sbase;
  st.nsig = (int)s.sigs.size();
  for (size_t i = 0; i < s.sigs.size(); ++i) p->sigs[sbase + i] = (uint8_t)s.sigs[i];
  st.seg0 = 0;
  st.nseg = 0;
  st.total_vec = 0;
  p->nsteps++;
  return true;
}

struct SegProto {
  int step;
  int64_t off, len;
  std::vector<int> src;
  std::vector<uint8_t> ctrl;
  int nlev;
  std::vector<int> dst;
  int acc = 0;  // Seg::acc
};

std::vector<uint8_t> single_level_ctrl(size_t n) {
  std::vector<uint8_t> c(n, 0);
  if (n) c[0] = 1;
  return c;
}

}  // namespace

static bool add_segments(Plan* p, std::vector<SegProto>& segs, int tbl, int vec, int mis, int64_t lo, int64_t hi,
                         std::string* err) {
  // Segments are stored grouped by step; merge into the existing layout.
  std::vector<Seg> all;
  std::vector<int> owner;
  for (int s = 0; s < p->nsteps; ++s)
    for (int k = 0; k < p->steps[s].nseg; ++k) {
      all.push_back(p->segs[p->steps[s].seg0 + k]);
      owner.push_back(s);
    }
  for (const SegProto& sp : segs) {
    Seg sg;
    std::memset(&sg, 0, sizeof(sg));
    // restrict to the element window [lo, hi): every operation is
    // element-wise, so a window keeps the full-buffer chunk geometry and order
    int64_t a = sp.off > lo ? sp.off : lo, b = sp.off + sp.len < hi ? sp.off + sp.len : hi;
    if (b < a) b = a;
    sg.off = a;
    sg.len = b - a;
    // scalar head up to the first 16-byte aligned element (the base of the
    // buffer is `mis` elements past a 16-byte boundary on every rank)
    int64_t head = sg.len;
    if (mis >= 0) {
      const int64_t phase = (mis + sg.off) % vec;
      head = phase ? (vec - phase) : 0;
      if (head > sg.len) head = sg.len;
    }
    sg.head = (int32_t)(head < (1 << 30) ? head : (1 << 30));
    if (head >= (1 << 30)) {
      if (err) *err = "misaligned segment too long for the scalar path";
      return false;
    }
    sg.body_off = sg.off + head;
    sg.nvec = (sg.len - head) / vec;
    sg.tail = (int32_t)(sg.len - head - sg.nvec * vec);
    sg.tbl = tbl;
    sg.nsrc = (uint8_t)sp.src.size();
    sg.ndst = (uint8_t)sp.dst.size();
    sg.nlev = (uint8_t)sp.nlev;
    sg.acc = (uint8_t)sp.acc;
    for (size_t i = 0; i < sp.src.size(); ++i) {
      sg.src[i] = (uint8_t)sp.src[i];
      sg.ctrl[i] = sp.ctrl[i];
    }
    for (size_t i = 0; i < sp.dst.size(); ++i) sg.dst[i] = (uint8_t)sp.dst[i];
    all.push_back(sg);
    owner.push_back(sp.step);
  }
  if (all.size() > RBX_MAX_SEGS) {
    if (err) *err = "plan has too many segments (bucket list too long)";
    return false;
  }
  int pos = 0;
  for (int s = 0; s < p->nsteps; ++s) {
    Step& st = p->steps[s];
    st.seg0 = pos;
    st.nseg = 0;
    st.total_vec = 0;
    for (size_t i = 0; i < all.size(); ++i) {
      if (owner[i] != s) continue;
      Seg sg = all[i];
      sg.vec_begin = st.total_vec;
      st.total_vec += sg.nvec;
      p->segs[pos++] = sg;
      st.nseg++;
    }
  }
  return true;
}

bool build_plan(const Geometry& g, int me, int64_t count, const PlanSpec& spec, int tbl, Plan* p, bool first,
                std::string* err) {
  const std::vector<int> act = g.active_dims();
  const int m = (int)act.size();
  const int n = g.nranks;
  if (first) {
    std::memset(p, 0, sizeof(Plan));
    p->me = me;
    p->nranks = n;
    p->vec = spec.vec;
    p->nblocks = spec.nblocks;
  }
  if (m == 0) return true;  // single rank: allreduce is the identity (runtime.py launch(1,(1,)))

  std::vector<int> everyone;
  for (int q = 0; q < n; ++q) everyone.push_back(q);
  const std::vector<int> peers = without(everyone, me);
  std::vector<std::vector<int>> ring(m);
  std::vector<int> start(m);
  {
    int c[16];
    g.coords(me, c);
    for (int i = 0; i < m; ++i) {
      ring[i] = g.ring(me, act[i]);
      start[i] = (c[act[i]] + 1) % g.dims[act[i]];
    }
  }
  auto rot_src = [&](int i) {
    std::vector<int> s;
    const int d = (int)ring[i].size();
    for (int j = 0; j < d; ++j) s.push_back(ring[i][(start[i] + j) % d]);
    return s;
  };
  auto region = [&](int rank, int upto, int64_t* o, int64_t* l) { region_after(g, rank, count, upto, o, l); };

  std::vector<StepProto> steps;
  std::vector<SegProto> segs;
  std::vector<int> entry;
  int64_t o, l;

  Mode mode = spec.mode == MODE_AUTO ? MODE_FUSED : spec.mode;
  if (mode == MODE_PUSH && spec.op == OP_ALLGATHER) mode = MODE_FUSED;  // allgather is push-only already
  if (spec.op == OP_BARRIER) {
    entry = peers;
    StepProto s0;
    add_waits(s0.waits, 0, peers, false);
    steps.push_back(s0);
  } else if (mode == MODE_FUSED || mode == MODE_FUSED_PULL) {
    entry = peers;
    region(me, m, &o, &l);
    const std::vector<int> order = fold_order(g, me);
    const std::vector<uint8_t> ctrl = fold_ctrl(g);
    if (spec.op == OP_ALLGATHER) {
      StepProto s0;
      add_waits(s0.waits, 0, peers, false);
      s0.sigs = peers;
      if (mode == MODE_FUSED) {
        segs.push_back(SegProto{0, o, l, {me}, single_level_ctrl(1), 1, rotated_after(peers, me)});
      } else {
        for (int q : rotated_after(peers, me)) {
          int64_t qo, ql;
          region(q, m, &qo, &ql);
          segs.push_back(SegProto{0, qo, ql, {q}, single_level_ctrl(1), 1, {me}});
        }
      }
      StepProto exit;
      add_waits(exit.waits, 1, peers, false);
      steps = {s0, exit};
    } else {
      const bool push = (spec.op == OP_ALLREDUCE && mode == MODE_FUSED);
      StepProto s0;
      add_waits(s0.waits, 0, peers, false);
      s0.sigs = peers;
      segs.push_back(SegProto{0, o, l, order, ctrl, m, push ? rotated_after(everyone, me) : std::vector<int>{me}});
      steps.push_back(s0);
      if (spec.op == OP_ALLREDUCE && mode == MODE_FUSED_PULL) {
        StepProto s1;
        add_waits(s1.waits, 1, peers, true);
        s1.sigs = peers;
        for (int q : rotated_after(peers, me)) {
          int64_t qo, ql;
          region(q, m, &qo, &ql);
          segs.push_back(SegProto{1, qo, ql, {q}, single_level_ctrl(1), 1, {me}});
        }
        steps.push_back(s1);
      }
      StepProto exit;
      add_waits(exit.waits, (int)steps.size(), peers, false);
      steps.push_back(exit);
    }
  } else if (mode == MODE_PUSH && spec.op != OP_ALLGATHER) {
    // Two-shot, writes only.  Step 0: push my input of every peer's owned
    // region into that peer's inbox (slot `me`).  Step 1: once every peer has
    // pushed (ALL CTAs: the tile split of a region differs between the two
    // steps), fold my region from my buffer and my inbox slots in the
    // reference order and push the result into every buffer.  No peer ever
    // reads my buffer, so no ENTRY wait is needed; the exit wait also
    // guarantees peers are done reading their inboxes before my next call
    // writes into them again.
    const int R = n;
    StepProto s0;
    for (int q : rotated_after(peers, me)) {
      int64_t qo, ql;
      region(q, m, &qo, &ql);
      segs.push_back(SegProto{0, qo, ql, {me}, single_level_ctrl(1), 1, {2 * R + q}});
    }
    s0.sigs = peers;
    StepProto s1;
    add_waits(s1.waits, 1, peers, true);
    region(me, m, &o, &l);
    std::vector<int> src;
    for (int p : fold_order(g, me)) src.push_back(p == me ? me : R + p);
    const bool ar = spec.op == OP_ALLREDUCE;
    segs.push_back(SegProto{1, o, l, src, fold_ctrl(g), m, ar ? rotated_after(everyone, me) : std::vector<int>{me}});
    s1.sigs = peers;
    StepProto exit;
    add_waits(exit.waits, 2, peers, false);
    steps = {s0, s1, exit};
  } else if (mode == MODE_RING_DIMS) {
    std::vector<int> partners;
    for (int i = 0; i < m; ++i)
      for (int q : ring[i])
        if (q != me && std::find(partners.begin(), partners.end(), q) == partners.end()) partners.push_back(q);
    std::sort(partners.begin(), partners.end());
    entry = partners;
    auto fold_ctrl1 = [&](int i) { return single_level_ctrl(ring[i].size()); };
    if (spec.op == OP_ALLREDUCE || spec.op == OP_REDUCE_SCATTER) {
      const int last = m - 1;
      for (int i = 0; i < m; ++i) {
        StepProto s;
        if (i == 0)
          add_waits(s.waits, 0, without(ring[0], me), false);
        else
          add_waits(s.waits, (int)steps.size(), ring[i], true);  // previous step's slot
        region(me, i + 1, &o, &l);
        std::vector<int> dst = {me};
        if (i == last && spec.op == OP_ALLREDUCE) dst = rotated_after(ring[i], me);
        std::vector<int> src = rot_src(i);
        int acc = 0;
        if (spec.partials_fp32 && m > 1) {
          // stage partials stay fp32 in the workspaces (one RNE at the very end)
          if (i > 0) {
            for (int& q : src) q += n;
            acc |= 1;
          }
          if (i < last) {
            dst = {n + me};
            acc |= 2;
          }
        }
        SegProto sp{(int)steps.size(), o, l, src, fold_ctrl1(i), 1, dst};
        sp.acc = acc;
        segs.push_back(sp);
        if (i < last)
          s.sigs = ring[i + 1];
        else
          s.sigs = (spec.op == OP_ALLREDUCE) ? ring[i] : partners;
        steps.push_back(s);
      }
      if (spec.op == OP_ALLREDUCE) {
        for (int i = m - 2; i >= 0; --i) {
          StepProto s;
          add_waits(s.waits, (int)steps.size(), ring[i + 1], true);
          region(me, i + 1, &o, &l);
          segs.push_back(SegProto{(int)steps.size(), o, l, {me}, single_level_ctrl(1), 1,
                                  rotated_after(without(ring[i], me), me)});
          s.sigs = ring[i];
          steps.push_back(s);
        }
        StepProto exit;
        add_waits(exit.waits, (int)steps.size(), without(ring[0], me), false);
        steps.push_back(exit);
      } else {
        StepProto exit;
        add_waits(exit.waits, (int)steps.size(), partners, false);
        steps.push_back(exit);
      }
    } else {  // allgather, dims m-1 .. 0
      for (int i = m - 1; i >= 0; --i) {
        StepProto s;
        if (i < m - 1) add_waits(s.waits, (int)steps.size(), ring[i + 1], true);
        add_waits(s.waits, 0, without(ring[i], me), false);
        region(me, i + 1, &o, &l);
        segs.push_back(SegProto{(int)steps.size(), o, l, {me}, single_level_ctrl(1), 1,
                                rotated_after(without(ring[i], me), me)});
        s.sigs = ring[i];
        steps.push_back(s);
      }
      StepProto exit;
      add_waits(exit.waits, (int)steps.size(), without(ring[0], me), false);
      steps.push_back(exit);
    }
  } else {
    if (err) *err = "unsupported mode for a rank plan";
    return false;
  }

  if (first) {
    p->nentry = (int)entry.size();
    for (size_t i = 0; i < entry.size(); ++i) p->entry_peers[i] = (uint8_t)entry[i];
    for (const StepProto& s : steps)
      if (!push_step(p, s, err)) return false;
  } else if (p->nsteps != (int)steps.size()) {
    if (err) *err = "bucket plans disagree in structure";
    return false;
  }
  return add_segments(p, segs, tbl, spec.vec, spec.mis, spec.lo, spec.hi < 0 ? count : spec.hi, err);
}

bool build_local_plan(const Geometry& g, int64_t count, int vec, int mis, int nblocks, Plan* p, std::string* err,
                      int64_t lo, int64_t hi) {
  std::memset(p, 0, sizeof(Plan));
  p->me = 0;
  p->nranks = g.nranks;
  p->vec = vec;
  p->nblocks = nblocks;
  p->nosync = 1;
  const int m = (int)g.active_dims().size();
  if (m == 0) return true;
  StepProto s0;
  if (!push_step(p, s0, err)) return false;
  std::vector<SegProto> segs;
  const std::vector<uint8_t> ctrl = fold_ctrl(g);
  std::vector<int> everyone;
  for (int q = 0; q < g.nranks; ++q) everyone.push_back(q);
  for (int r = 0; r < g.nranks; ++r) {
    int64_t o, l;
    region_after(g, r, count, m, &o, &l);
    segs.push_back(SegProto{0, o, l, fold_order(g, r), ctrl, m, rotated_after(everyone, r)});
  }
  return add_segments(p, segs, 0, vec, mis, lo, hi < 0 ? count : hi, err);
}

int64_t inbox_slot_bytes(const Geometry& g, int64_t count, int itemsize) {
  const int m = (int)g.active_dims().size();
  int64_t maxlen = 0;
  for (int r = 0; r < g.nranks; ++r) {
    int64_t o, l;
    region_after(g, r, count, m, &o, &l);
    if (l > maxlen) maxlen = l;
  }
  const int64_t raw = maxlen * itemsize + 16;  // + phase pad (see rbx_capi.cu push_table)
  return (raw + 255) / 256 * 256;
}

int64_t describe_plan(const Plan& p, int64_t* out, int64_t cap) {
  std::vector<int64_t> v;
  v.push_back(p.nsteps);
  v.push_back(p.nentry);
  for (int i = 0; i < p.nentry; ++i) v.push_back(p.entry_peers[i]);
  for (int s = 0; s < p.nsteps; ++s) {
    const Step& st = p.steps[s];
    v.push_back(st.nwait);
    for (int w = 0; w < st.nwait; ++w) {
      const Wait& x = p.waits[st.wait0 + w];
      v.push_back(x.slot);
      v.push_back(x.peer);
      v.push_back(x.all);
    }
    v.push_back(st.nsig);
    for (int k = 0; k < st.nsig; ++k) v.push_back(p.sigs[st.sig0 + k]);
    v.push_back(st.nseg);
    for (int k = 0; k < st.nseg; ++k) {
      const Seg& sg = p.segs[st.seg0 + k];
      v.push_back(sg.off);
      v.push_back(sg.len);
      v.push_back(sg.nsrc);
      for (int i = 0; i < sg.nsrc; ++i) v.push_back(sg.src[i]);
      for (int i = 0; i < sg.nsrc; ++i) v.push_back(sg.ctrl[i]);
      v.push_back(sg.nlev);
      v.push_back(sg.ndst);
      for (int i = 0; i < sg.ndst; ++i) v.push_back(sg.dst[i]);
      v.push_back(sg.tbl);
      v.push_back(sg.head);
      v.push_back(sg.nvec);
      v.push_back(sg.tail);
      v.push_back(sg.acc);
    }
  }
  const int64_t n = (int64_t)v.size();
  for (int64_t i = 0; i < n && i < cap; ++i) out[i] = v[i];
  return n;
}

}  // namespace rbx
