"""Config 4: ResNet-101 (44,549,160 fp32 params) gradient allreduce in DDP-style
25 MB buckets (SURVEY.md A.9 bucket sizes).  Compares
  * ours, one launch over the whole bucket list (buckets in flight concurrently),
  * ours, one launch per bucket (the reference's sequential Workload.lengths
    semantics, pkg/src/ringbox/runtime.py:390-398),
  * NCCL all_reduce per bucket (comparison only).

  torchrun --nproc-per-node N tools/buckets.py

One JSON line per variant (rank 0): total time (CUDA events, max over ranks,
median of --iters) and bus GB/s over the 178.2 MB of gradients.
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

RESNET101_BUCKETS = [2_049_000, 7_875_584, 6_563_840, 6_965_760, 6_703_104, 6_703_104, 6_590_464, 1_098_304]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
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
    total = sum(RESNET101_BUCKETS)
    assert total == 44_549_160
    flat = ctx.empty(total, "f32")
    pristine = torch.randn(total, device=dev)
    views, off = [], 0
    for n in RESNET101_BUCKETS:
        views.append(flat[off:off + n])
        off += n
    scratch = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def run(variant):
        if variant == "ours_bucket_list_one_launch":
            ctx.allreduce_buckets(views)
        elif variant == "ours_per_bucket":
            for v in views:
                ctx.collective("allreduce", v)
        else:
            for v in views:
                dist.all_reduce(v)

    tiny = torch.zeros(1, device=dev)
    for variant in ("ours_bucket_list_one_launch", "ours_per_bucket", "nccl_per_bucket"):
        ts = []
        for it in range(args.iters + 2):
            flat.copy_(pristine)
            scratch.fill_(1.0)
            scratch.sum()
            if it == 0:
                dist.barrier()
            # both arms: host ~0.5 ms ahead, then a device-side barrier of the arm's own kind
            torch.cuda._sleep(1_000_000)
            if variant.startswith("ours"):
                ctx.barrier()
            else:
                dist.all_reduce(tiny)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            run(variant)
            e.record(stream)
            torch.cuda.synchronize()
            if it >= 2:
                ts.append(s.elapsed_time(e))
        ctx.check()
        t = torch.tensor(ts, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = t.median().item() / 1e3
        if rank == 0:
            print(json.dumps({"config": "config4: ResNet-101 44,549,160 fp32 params in 8 DDP buckets (25 MiB cap)",
                              "n_gpus": world, "dims": list(dims), "variant": variant,
                              "ms": round(sec * 1e3, 4),
                              "busbw_gbs": round(2 * (world - 1) / world * total * 4 / sec / 1e9, 2)}), flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
