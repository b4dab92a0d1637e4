"""Rank-process body of `__graft_entry__.smoke()`'s per-rank check: a module of
its own (test infrastructure, next to the tests) so spawned processes can import
it by name however the entry module was loaded.  The oracle is only the checker."""

from __future__ import annotations

import os


def smoke_rank(rank: int, port: int, q) -> None:
    """One rank process of the per-rank path: RankContext (IPC-mapped peer
    buffers + signal areas) and one FUSED allreduce, the hot path of the bench."""
    try:
        import torch
        import torch.distributed as dist

        from oracle import ringbox_oracle as orc
        from paper_1708_02188_b200.multiring import Grid
        from paper_1708_02188_b200.runtime import RankContext

        os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
        dev = rank % torch.cuda.device_count()
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo", rank=rank, world_size=2)
        ctx = RankContext(rank, Grid((2,)), device=dev, mode="fused", nblocks=16, timeout_s=20.0)
        n = 100_003
        parts = [orc.generate_input(3, 0, r, n, "f32") for r in range(2)]
        t = ctx.empty(n, "f32")
        t.copy_(torch.from_numpy(parts[rank]))
        ctx.collective("allreduce", t)
        kernel = ctx.last_kernel()
        ok = orc.sha256(t.cpu().numpy()) == orc.sha256(orc.closed_form_allreduce(orc.Grid((2,)), parts))
        ok = ok and kernel == "fused"  # the specialised FUSED kernel, not the interpreter
        ctx.close()
        dist.destroy_process_group()
        q.put((rank, ok, f"(kernel {kernel})"))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, False, repr(exc)))
