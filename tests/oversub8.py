"""8 ranks (grid 2x2x2 / 2x4) as 8 processes on fewer GPUs (two contexts per
GPU, time-sliced): exercises the per-rank N=8 path -- 8-way IPC mapping,
flags, entry/exit handshakes, 7-peer FUSED folds, LL -- when the sandbox only
grants 4 GPUs.  Not a performance run (contexts on one GPU do not run
concurrently, every handshake waits for a context switch).

  torchrun --nproc-per-node 8 tests/oversub8.py

Checks every rank's result digest against the oracle's reference-order fold
(test infrastructure, used only as the checker).  Prints one JSON line per case.
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    from oracle import ringbox_oracle as orc
    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import RankContext

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    ngpu = torch.cuda.device_count()
    dev = rank % ngpu
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    ok_all = True
    for dims in ((2, 2, 2), (2, 4)):
        ctx = RankContext(rank, Grid(dims), device=dev, nblocks=8, timeout_s=20.0, blocking=False)
        for mode, n in (("auto", 1000), ("auto", 100_003), ("fused", 100_003), ("ring_dims", 100_003), ("ll", 4099)):
            parts = [orc.generate_input(7, 0, r, n, "f32") for r in range(world)]
            want = orc.sha256(orc.closed_form_allreduce(orc.Grid(dims), parts))
            t = ctx.empty(n, "f32")
            t.copy_(torch.from_numpy(parts[rank]))
            t0 = time.perf_counter()
            ctx.collective("allreduce", t, mode=mode)
            ctx.synchronize()
            dt = time.perf_counter() - t0
            got = orc.sha256(t.cpu().numpy())
            res = [None] * world
            dist.all_gather_object(res, got == want)
            ok_all = ok_all and all(res)
            if rank == 0:
                print(json.dumps({"dims": list(dims), "mode": mode, "n": n, "ranks": world, "gpus": ngpu,
                                  "bit_exact_all_ranks": all(res), "seconds": round(dt, 3)}), flush=True)
        ctx.close()
    dist.barrier()
    if rank == 0:
        print(json.dumps({"oversubscribed_8_rank_path_ok": ok_all}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
