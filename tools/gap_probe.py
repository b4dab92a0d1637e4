"""Where does a collective's fixed cost go?  Device-clock brackets around one
allreduce (diagnostic, not product).

  RBX_TRACE=1 torchrun --nproc-per-node 2 tools/gap_probe.py

Per size: rbx_stamp (a 1-thread %globaltimer kernel) immediately before and
after the collective on the same stream, CUDA events around the collective,
and the kernel's own timeline (first CTA start, first/last CTA exit).  Prints
medians on rank 0: launch gap (stamp -> first CTA start), in-kernel time,
completion gap (last CTA exit -> stamp), event time.
"""

import ctypes
import json
import os
import statistics
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
    L = ctx._L
    stream = torch.cuda.current_stream(dev)
    sp = ctypes.c_void_p(stream.cuda_stream)
    stamps = torch.zeros(2, dtype=torch.int64, device=dev)
    sizes = [int(x) for x in os.environ.get("GAP_SIZES", "1,1048576,25600000").split(",")]
    mode = os.environ.get("GAP_MODE", "fused")
    # calibration: two stamp kernels back to back (the stamp's own launch gap)
    cal = []
    for it in range(14):
        torch.cuda._sleep(1_000_000)
        L.rbx_stamp(ctypes.c_void_p(stamps.data_ptr()), sp)
        L.rbx_stamp(ctypes.c_void_p(stamps.data_ptr() + 8), sp)
        torch.cuda.synchronize()
        st = stamps.tolist()
        cal.append((st[1] - st[0]) / 1e3)
    if rank == 0:
        print(json.dumps({"stamp_to_stamp_us": round(statistics.median(cal[4:]), 3)}), flush=True)
    for n in sizes:
        work = ctx.empty(n, "f32")
        work.fill_(1.0)
        rows = []
        for it in range(14):
            torch.cuda._sleep(1_000_000)  # host runs ahead of the device
            ctx.barrier()
            L.rbx_stamp(ctypes.c_void_p(stamps.data_ptr()), sp)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            ctx.collective("allreduce", work, mode=mode)
            e.record(stream)
            L.rbx_stamp(ctypes.c_void_p(stamps.data_ptr() + 8), sp)
            torch.cuda.synchronize()
            buf = (ctypes.c_uint64 * 64)()
            L.rbx_comm_trace(ctx._comm, buf, 64)
            st = stamps.tolist()
            start = min(buf[0], buf[32])
            exit_ = max(buf[31], buf[63])
            rows.append({"event_us": s.elapsed_time(e) * 1e3, "stamp_us": (st[1] - st[0]) / 1e3,
                         "launch_gap_us": (start - st[0]) / 1e3, "kernel_us": (exit_ - start) / 1e3,
                         "completion_gap_us": (st[1] - exit_) / 1e3,
                         "prev_exit_to_start_us": (start - buf[29]) / 1e3 if buf[29] else None})
            work.fill_(1.0)
        rows = rows[4:]
        med = {k: round(statistics.median([r[k] for r in rows if r[k] is not None]), 3) for k in rows[0]
               if any(r[k] is not None for r in rows)}
        every = [None] * world
        dist.all_gather_object(every, med)
        if rank == 0:
            print(json.dumps({"n": n, "mode": mode, "carveout": os.environ.get("RBX_CARVEOUT", "default(50)"),
                              "per_rank": every}), flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
