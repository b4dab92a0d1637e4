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
    _streams: dict = field(default_factory=dict)


def multiring_allreduce_hook(state: MultiringHookState, bucket):
    import torch

    ctx = state.ctx
    t = bucket.buffer()
    dev = t.device
    if state.stream is None:
        state.stream = torch.cuda.Stream(device=dev)
    comm = state.stream
    comm.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(comm):
        ctx.collective("allreduce", t, mode=state.mode)
        t.div_(ctx.grid.size)
        fut = torch.futures.Future(devices=[dev])
        fut.set_result(t)  # records an event on `comm`; DDP's wait() makes its stream wait on it
    t.record_stream(comm)
    state.buckets += 1
    state.bytes += t.numel() * t.element_size()
    return fut
