"""Planner calibration on a B200 box.

The reference planner scores decompositions with a per-dimension bandwidth and
a per-phase latency read from the topology JSON (pkg/src/ringbox/multiring.py:
228-268, costmodel.py:92-147).  On a B200 box both are measured here, on the
device, with the communicator itself:

* latency L  = one device flag barrier across all ranks (the per-stage cost of
  a ring phase in RING_DIMS mode: signal + remote observe);
* bandwidth B = bus GB/s of a large allreduce (payload per direction per GPU).

`calibrated_topology(ctx)` returns the box in the reference's topology grammar
(topology.b200_box with measured B and L), so `plan()` picks dims from
measurements exactly as the reference picks them from its JSON.  With L > 0
every factorization ties on bandwidth and the fewest-phase grid wins (2x2x2 for
8 GPUs), matching SURVEY.md A.6.  Collective: call on every rank.
"""

from __future__ import annotations


def measure(ctx, big_elems: int = 64 * 1024 * 1024, iters: int = 10) -> dict:
    import torch
    import torch.distributed as dist

    dev = ctx.device
    stream = torch.cuda.current_stream(dev)
    # latency: device barrier
    ts = []
    for _ in range(iters + 2):
        torch.cuda._sleep(50_000)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        ctx.barrier()
        e.record(stream)
        torch.cuda.synchronize(dev)
        ts.append(s.elapsed_time(e) / 1e3)
    lat = sorted(ts[2:])[len(ts[2:]) // 2]
    # bandwidth: large allreduce
    work = ctx.empty(big_elems, "f32")
    work.fill_(1.0)
    bw = []
    for _ in range(iters + 2):
        ctx.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        ctx.collective("allreduce", work)
        e.record(stream)
        torch.cuda.synchronize(dev)
        work.fill_(1.0)
        t = s.elapsed_time(e) / 1e3
        n = ctx.grid.size
        bw.append(2 * (n - 1) / n * big_elems * 4 / t / 1e9)
    ctx.check()
    # every rank must feed the planner the same numbers: the worst latency and the
    # lowest median bandwidth over ranks
    med_bw = sorted(bw[2:])[len(bw[2:]) // 2]
    if dist.is_available() and dist.is_initialized():
        from .exchange import allgather_objects

        every = allgather_objects((lat, med_bw), ctx.group)
        lat, med_bw = max(x[0] for x in every), min(x[1] for x in every)
    return {"latency_s": float(lat), "bandwidth_gbps": float(med_bw)}


def calibrated_topology(ctx, **kw):
    from .topology import b200_box

    m = measure(ctx, **kw)
    return b200_box(ctx.grid.size, latency_s=m["latency_s"], bandwidth_gbps=m["bandwidth_gbps"]), m
