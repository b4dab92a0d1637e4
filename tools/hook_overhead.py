"""Host (CPU) cost of one DDP comm-hook call, per variant, at N GPUs.

  torchrun --nproc-per-node 2 tools/hook_overhead.py

The autograd thread runs the hook between backward kernel launches, so every
microsecond here can starve the GPU queue during backward.  Diagnostic only.
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class FakeBucket:
    def __init__(self, t):
        self._t = t

    def buffer(self):
        return self._t


def main():
    import torch
    import torch.distributed as dist

    from paper_1708_02188_b200.ddp import MultiringHookState, multiring_allreduce_hook
    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import RankContext

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    gloo = dist.new_group(backend="gloo")
    ctx = RankContext(rank, Grid((world,)), group=gloo, device=rank, blocking=False)
    st = MultiringHookState(ctx)
    res = {}
    for n in (262_144, 6_553_600):  # a 1 MiB (LL) and a 25 MiB (FUSED) bucket
        t = torch.ones(n, device=dev)
        b = FakeBucket(t)
        multiring_allreduce_hook(st, b)  # registration, plan build
        torch.cuda.synchronize()
        dist.barrier()
        iters = 200
        for fast in (False, True):
            st.fast = fast
            multiring_allreduce_hook(st, b)
            torch.cuda.synchronize()
            torch.cuda._sleep(50_000_000)  # keep the GPU busy: the loop measures host time only
            t0 = time.perf_counter()
            for _ in range(iters):
                multiring_allreduce_hook(st, b)
            t1 = time.perf_counter()
            torch.cuda.synchronize()
            res[f"hook{'_fast' if fast else ''}_us_{n * 4 >> 20}MiB"] = round((t1 - t0) / iters * 1e6, 2)
        # NCCL through a Python hook, for comparison
        torch.cuda._sleep(50_000_000)
        t0 = time.perf_counter()
        for _ in range(iters):
            fut = dist.all_reduce(t, async_op=True).get_future()
            fut.then(lambda f: f.value()[0].div_(world))
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        res[f"nccl_hook_us_{n * 4 >> 20}MiB"] = round((t1 - t0) / iters * 1e6, 2)
    if rank == 0:
        print(json.dumps(res), flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
