"""Config 3: allreduce size sweep 4 KB - 1 GB, fp32 and bf16 (fp32 accumulate),
multi-ring kernel vs NCCL all_reduce, bus GB/s and % of 900 GB/s.

  torchrun --nproc-per-node N tools/sweep.py [--max-bytes 1073741824] [--out profiles/sweep_N.jsonl]

Each point: inputs restored + L2 flushed outside the timed region, host ~0.5 ms
ahead of the device, a device-side barrier of the arm's own kind (our flag
barrier / a 1-element NCCL allreduce), CUDA events around one collective, max
over ranks, trimmed mean (middle 80 %) of --iters.
One JSON line per (dtype, bytes, impl) on rank 0.
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-bytes", type=int, default=4096)
    ap.add_argument("--max-bytes", type=int, default=1 << 30)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--dtypes", default="f32,bf16")
    ap.add_argument("--mode", default="auto")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import RankContext

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    dims = {2: (2,), 4: (2, 2), 8: (2, 2, 2)}.get(world, (world,))
    ctx = RankContext(rank, Grid(dims), device=rank, blocking=False)
    scratch = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    out = open(args.out, "w") if (args.out and rank == 0) else None
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16}
    for dt in args.dtypes.split(","):
        esz = 4 if dt == "f32" else 2
        nbytes = args.min_bytes
        while nbytes <= args.max_bytes:
            n = nbytes // esz
            work = ctx.empty(n, dt)
            pristine = torch.randn(n, device=dev).to(tdt[dt])
            res = {}
            tiny = torch.zeros(1, device=dev)
            for impl in ("ours", "nccl"):
                ts = []
                for it in range(args.iters + 2):
                    work.copy_(pristine)
                    scratch.fill_(1.0)
                    scratch.sum()
                    if it == 0:
                        dist.barrier()
                    # both arms: the host runs ~0.5 ms ahead (Python launch cost hidden), then a
                    # device-side barrier of the arm's own kind aligns the GPUs before the start event
                    torch.cuda._sleep(1_000_000)
                    if impl == "ours":
                        ctx.barrier()
                    else:
                        dist.all_reduce(tiny)
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record(stream)
                    if impl == "ours":
                        ctx.collective("allreduce", work, mode=args.mode)
                    else:
                        dist.all_reduce(work)
                    e.record(stream)
                    torch.cuda.synchronize()
                    if it >= 2:
                        ts.append(s.elapsed_time(e))
                t = torch.tensor(ts, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                # events tick in ~2 us steps here: a trimmed mean (middle 80 %) resolves below that
                srt = t.sort().values
                k = len(srt) // 10
                sec = srt[k:len(srt) - k].mean().item() / 1e3
                bus = 2 * (world - 1) / world * nbytes / sec / 1e9
                res[impl] = (sec, bus)
            ctx.check()
            if rank == 0:
                line = {"n_gpus": world, "dims": list(dims), "dtype": dt, "bytes": nbytes,
                        "ours_us": round(res["ours"][0] * 1e6, 2), "ours_busbw_gbs": round(res["ours"][1], 2),
                        "ours_pct_of_900": round(100 * res["ours"][1] / 900, 2),
                        "nccl_us": round(res["nccl"][0] * 1e6, 2), "nccl_busbw_gbs": round(res["nccl"][1], 2),
                        "speedup_vs_nccl": round(res["nccl"][0] / res["ours"][0], 3)}
                print(json.dumps(line), flush=True)
                if out:
                    out.write(json.dumps(line) + "\n")
            nbytes *= 4
    if out:
        out.close()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
