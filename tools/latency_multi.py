"""Latency breakdown of the multi-GPU kernel using the device timeline (RBX_TRACE=1).

  RBX_TRACE=1 torchrun --nproc-per-node N tools/latency_multi.py

Diagnostic only.  Prints, per size, the CUDA-event time of one allreduce and
the in-kernel timeline (microseconds since the first CTA started) of the first
and last CTA on rank 0.
"""

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
    sizes = [int(x) for x in os.environ.get("LAT_SIZES", "1,65536,1048576,25600000").split(",")]
    for n in sizes:
        work = ctx.empty(n, "f32")
        work.fill_(1.0)
        modes = os.environ.get("LAT_MODES", "fused,ring_dims,ll").split(",")
        for mode in [m for m in modes if m != "ll" or n * 4 <= (1 << 20)]:
            ts = []
            for it in range(12):
                torch.cuda._sleep(1_000_000)  # host runs ahead of the device
                ctx.barrier()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(stream)
                ctx.collective("allreduce", work, mode=mode)
                e.record(stream)
                torch.cuda.synchronize()
                ts.append(s.elapsed_time(e) * 1e3)
                work.fill_(1.0)
            tr = ctx.trace()
            t = torch.tensor(ts[2:], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if rank == 0:
                print(json.dumps({"n": n, "mode": mode, "event_us_median": round(t.median().item(), 2),
                                  "trace_rank0": tr}), flush=True)
    # barrier alone (host ahead: the spin before the start event hides Python launch cost)
    ts = []
    for it in range(12):
        torch.cuda._sleep(1_000_000)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        ctx.barrier()
        e.record(stream)
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    if rank == 0:
        print(json.dumps({"barrier_event_us": sorted(ts)[len(ts) // 2], "trace_rank0": ctx.trace()}), flush=True)
    # an empty torch kernel for the launch floor
    ts = []
    x = torch.empty(1, device=dev)
    for it in range(12):
        torch.cuda._sleep(1_000_000)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        x.fill_(0.0)
        e.record(stream)
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    if rank == 0:
        print(json.dumps({"tiny_torch_kernel_event_us": sorted(ts)[len(ts) // 2]}), flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
