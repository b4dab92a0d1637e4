"""Prologue study of the step kernel at N GPUs (RBX_TRACE=1): raw device
timelines of BOTH ranks (absolute %globaltimer ns) for a 1-element and a
config-sized fused allreduce, with and without an L2 flush before the call.

  torchrun --nproc-per-node 2 tools/entry_study.py
"""

import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import RankContext

    os.environ.setdefault("RBX_TRACE", "1")
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    dims = {2: (2,), 4: (2, 2), 8: (2, 2, 2)}[world]
    ctx = RankContext(rank, Grid(dims), device=rank, blocking=False)
    stream = torch.cuda.current_stream(dev)
    scratch = torch.empty(64 * 1024 * 1024, device=dev)
    for n in (1, 25_600_000):
        work = ctx.empty(n, "f32")
        for flush in (0, 1):
            rows = []
            for it in range(8):
                work.fill_(1.0)
                if flush:
                    scratch.fill_(1.0)
                    scratch.sum()
                torch.cuda._sleep(1_000_000)
                ctx.barrier()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(stream)
                ctx.collective("allreduce", work, mode="fused")
                e.record(stream)
                torch.cuda.synchronize()
                buf = (ctypes.c_uint64 * 64)()
                ctx._L.rbx_comm_trace(ctx._comm, buf, 64)
                rows.append({"event_us": round(s.elapsed_time(e) * 1e3, 2), "tr": list(buf)})
            allrows = [None] * world
            dist.all_gather_object(allrows, rows)
            if rank == 0:
                for it in range(3, 8):
                    t0 = min(allrows[r][it]["tr"][0] for r in range(world))
                    out = {"n": n, "flush": flush, "it": it}
                    for r in range(world):
                        tr = allrows[r][it]["tr"]
                        sl = {"start": 0, "staged_ld": 20, "staged": 21, "epoch": 22, "pre_entry": 1, "entry": 2,
                              "entry2": 23, "s0_wait": 3, "s0_work": 4, "s0_sig": 5, "s1_wait": 6, "s1_work": 7,
                              "s1_sig": 8, "steps_done": 30, "exit": 31}
                        out[f"r{r}"] = {"event_us": allrows[r][it]["event_us"],
                                        **{k: round((tr[v] - t0) / 1e3, 3) for k, v in sl.items() if tr[v]},
                                        "last_cta_exit": round((tr[32 + 31] - t0) / 1e3, 3) if tr[63] else None}
                    print(json.dumps(out), flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
