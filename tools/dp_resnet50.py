"""Config 5 with MultiringDataParallel: ResNet-50 data-parallel training step
on synthetic ImageNet-shaped data (batch 32 per GPU, bf16 autocast), gradient
buckets allreduced from autograd hooks while backward runs, eager or with the
WHOLE step (forward, backward, bucket allreduces, SGD) in one CUDA graph.

  python tools/dp_resnet50.py --comm none [--graph 1]                 (N=1 reference step)
  torchrun --nproc-per-node N tools/dp_resnet50.py --comm multiring|nccl [--graph 0|1]

Prints one JSON line on rank 0: median step time (CUDA events, max over
ranks), images/s, and the reference's derived metrics
(pkg/src/ringbox/bench.py:45-56) when --t1-ms is given: efficiency t1/tN and
overhead tN - t1.  Random init, synthetic data (no network).
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--comm", choices=["multiring", "nccl", "none"], default="multiring")
    ap.add_argument("--graph", type=int, default=1)
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--nblocks", type=int, default=32, help="CTAs per allreduce (SMs left to backward)")
    ap.add_argument("--mode", default="auto", help="multi-ring mode (auto = fused; push: writes only, fewer SMs)")
    ap.add_argument("--t1-ms", type=float, default=None, help="N=1 step time for efficiency/overhead")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    import torchvision

    from paper_1708_02188_b200.dp import MultiringDataParallel
    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import RankContext

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    torch.backends.cudnn.benchmark = True
    torch.backends.cuda.matmul.allow_tf32 = True
    torch.backends.cudnn.allow_tf32 = True
    torch.manual_seed(0)
    model = torchvision.models.resnet50(num_classes=1000).to(dev).to(memory_format=torch.channels_last)
    nparams = sum(p.numel() for p in model.parameters())
    dp = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if args.comm != "none":
        assert world > 1, "--comm multiring/nccl needs torchrun with N > 1"
        ctx = None
        if args.comm == "multiring":
            dims = {2: (2,), 4: (2, 2), 8: (2, 2, 2)}.get(world, (world,))
            gloo = dist.new_group(backend="gloo")
            ctx = RankContext(rank, Grid(dims), group=gloo, device=local, nblocks=args.nblocks, blocking=False,
                              mode=args.mode)
        dp = MultiringDataParallel(model, ctx, comm=args.comm)
    opt = torch.optim.SGD(model.parameters(), lr=0.1, momentum=0.9, foreach=True)
    torch.manual_seed(1 + rank)
    x = torch.randn(args.batch, 3, 224, 224, device=dev).to(memory_format=torch.channels_last)
    y = torch.randint(0, 1000, (args.batch,), device=dev)
    lossf = torch.nn.CrossEntropyLoss()
    loss_buf = torch.zeros((), device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        if dp is not None:
            dp.zero_grad()
        else:
            opt.zero_grad(set_to_none=False)
        with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):
            loss = lossf(model(x), y)
        loss.backward()
        opt.step()
        loss_buf.copy_(loss.detach())

    if args.graph:
        if dp is not None:
            g = dp.capture(step, warmup=args.warmup)
        else:
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                for _ in range(args.warmup):
                    step()
            stream.wait_stream(side)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
        run = g.replay
    else:
        for _ in range(args.warmup):
            step()
        run = step
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ts = []
    for _ in range(args.iters):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        run()
        e.record(stream)
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    if dp is not None and dp.ctx is not None:
        dp.ctx.check()
    t = torch.tensor(ts, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = t.median().item()
    if rank == 0:
        line = {
            "config": "config5: ResNet-50 data-parallel step, synthetic 3x224x224, 1000 classes, bf16 autocast",
            "engine": "MultiringDataParallel" if dp is not None else "single GPU",
            "comm": args.comm, "graph": bool(args.graph), "n_gpus": world, "batch_per_gpu": args.batch,
            "nblocks": args.nblocks if args.comm == "multiring" else None, "params": nparams,
            "mode": args.mode if args.comm == "multiring" else None,
            "grad_bytes": nparams * 4, "buckets": len(dp.buckets) if dp is not None else None,
            "t_iter_ms": round(t_ms, 3), "images_per_s": round(world * args.batch / t_ms * 1e3, 1),
            "loss": float(loss_buf.item()),
        }
        if args.t1_ms:
            line["efficiency"] = round(args.t1_ms / t_ms, 4)  # bench.py:45-56
            line["overhead_ms"] = round(t_ms - args.t1_ms, 3)
        print(json.dumps(line), flush=True)
    if dp is not None:
        dp.close()
    if dp is not None and dp.ctx is not None:
        dp.ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
