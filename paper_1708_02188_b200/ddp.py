"""DDP communication hook: gradient buckets reduced by the multi-ring kernel.

SURVEY.md section 8(f) item 1 / BASELINE config 5.  The reference has no
training integration (pkg/src/ringbox/bench.py:5-6 models compute + comm
without overlap).  Here every DDP gradient bucket is allreduced in the
reference's multi-ring order by librbx on a dedicated communication stream, so
the reduction of bucket k overlaps the backward computation of bucket k+1.

    ctx = RankContext(rank, Grid(dims), device=local_rank, blocking=False)
    model = DistributedDataParallel(model, device_ids=[local_rank])
    model.register_comm_hook(MultiringHookState(ctx), multiring_allreduce_hook)

Gradients are summed bit-exactly in the reference order, then divided by the
world size (DDP's averaging).  Bucket buffers are registered with the
communicator on first use (one collective IPC-handle exchange per bucket
buffer; DDP keeps them for the lifetime of the reducer).
"""

from __future__ import annotations

from dataclasses import dataclass, field


@dataclass
class MultiringHookState:
    ctx: object                      # runtime.RankContext (blocking=False)
    stream: object = None            # torch.cuda.Stream for communication (created lazily)
    mode: str | None = None          # execution mode override
    buckets: int = 0                 # statistics
    bytes: int = 0
    fast: bool = True                # cached per-bucket launch (no per-call Python bookkeeping)
    _fast: dict = field(default_factory=dict)


def _prepare(state: MultiringHookState, t):
    """First call on a bucket buffer (collective on every rank, in the same
    order): register it, agree on the shape, and cache the ctypes launch
    arguments so later calls cost one ctypes call plus stream bookkeeping."""
    import ctypes

    from . import _native
    from .runtime import _dtype_name

    ctx = state.ctx
    dt = _dtype_name(t)
    n = t.numel()
    m = _native.MODES[state.mode or ctx.mode]
    if n:
        ctx._ensure(t)
    ctx._agree_shape((t.data_ptr(), "allreduce", n, dt, m))
    ctx._ensure_inbox([n], dt, "allreduce", m)
    args = (ctx._comm, ctypes.c_void_p(t.data_ptr()), ctypes.c_size_t(n), ctypes.c_int(_native.DTYPE_CODES[dt]),
            ctypes.c_int(m), ctypes.c_void_p(state.stream.cuda_stream))
    traffic = ctx._rank_traffic(n, t.element_size(), "allreduce") if n else 0
    return args, traffic


def multiring_allreduce_hook(state: MultiringHookState, bucket):
    import torch

    ctx = state.ctx
    t = bucket.buffer()
    dev = t.device
    if state.stream is None:
        state.stream = torch.cuda.Stream(device=dev)
    comm = state.stream
    comm.wait_stream(torch.cuda.current_stream(dev))
    if state.fast:
        key = (t.data_ptr(), t.numel(), t.dtype)
        hit = state._fast.get(key)
        if hit is None:
            hit = state._fast[key] = _prepare(state, t)
        args, traffic = hit
        if t.numel():
            rc = ctx._L.rbx_allreduce(*args)
            if rc:
                from . import _native

                _native.check(rc)
        ctx.bytes_sent += traffic
    else:
        with torch.cuda.stream(comm):
            ctx.collective("allreduce", t, mode=state.mode)
    fut = torch.futures.Future(devices=[dev])
    with torch.cuda.stream(comm):
        t.div_(ctx.grid.size)
        fut.set_result(t)  # records an event on `comm`; DDP's wait() makes its stream wait on it
    state.buckets += 1
    state.bytes += t.numel() * t.element_size()
    return fut
