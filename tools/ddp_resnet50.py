"""Config 5: ResNet-50 data-parallel training step on synthetic ImageNet-shaped
data, gradients allreduced by the multi-ring kernel (DDP comm hook, overlapped
with backward) or by NCCL (DDP default), at 1/2/4/8 GPUs.

  torchrun --nproc-per-node N tools/ddp_resnet50.py --comm ours|nccl [--iters 20]

Prints one JSON line (rank 0): per-iteration time (CUDA events, max over
ranks), images/s, the bytes of gradient reduced per step.  Scaling efficiency
and communication overhead follow the reference's definitions
(pkg/src/ringbox/bench.py:45-56): eff = t_1 / t_N, overhead = t_N - t_1.
Synthetic data, random init (no network access for ImageNet / checkpoints).
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--comm", choices=["ours", "nccl", "nccl_hook", "noop_hook"], default="ours")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=32)  # per GPU
    ap.add_argument("--amp", default="bf16", choices=["bf16", "none"])
    ap.add_argument("--nblocks", type=int, default=32, help="CTAs of the allreduce kernel (leave SMs to backward)")
    ap.add_argument("--bucket-view", type=int, default=1, help="gradient_as_bucket_view")
    ap.add_argument("--threads", type=int, default=512, help="threads per CTA of the allreduce kernels")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    import torchvision

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
    hook_state = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        model = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local], bucket_cap_mb=25,
                                                          gradient_as_bucket_view=bool(args.bucket_view))
        if args.comm == "ours":
            from paper_1708_02188_b200.ddp import MultiringHookState, multiring_allreduce_hook
            from paper_1708_02188_b200.multiring import Grid
            from paper_1708_02188_b200.runtime import RankContext

            dims = {2: (2,), 4: (2, 2), 8: (2, 2, 2)}.get(world, (world,))
            gloo = dist.new_group(backend="gloo")  # host plumbing for handle exchange
            ctx = RankContext(rank, Grid(dims), group=gloo, device=local, nblocks=args.nblocks,
                              threads=args.threads, blocking=False)
            hook_state = MultiringHookState(ctx)
            model.register_comm_hook(hook_state, multiring_allreduce_hook)
        elif args.comm == "nccl_hook":  # the same Python-hook machinery around NCCL: isolates hook cost
            def nccl_hook(_, bucket):
                t = bucket.buffer()
                fut = dist.all_reduce(t, async_op=True).get_future()
                return fut.then(lambda f: f.value()[0].div_(world))

            model.register_comm_hook(None, nccl_hook)
        elif args.comm == "noop_hook":  # hook machinery only, no communication at all (cost floor of any hook)
            def noop_hook(_, bucket):
                fut = torch.futures.Future(devices=[dev])
                fut.set_result(bucket.buffer())
                return fut

            model.register_comm_hook(None, noop_hook)
    opt = torch.optim.SGD(model.parameters(), lr=0.1, momentum=0.9)
    x = torch.randn(args.batch, 3, 224, 224, device=dev).to(memory_format=torch.channels_last)
    y = torch.randint(0, 1000, (args.batch,), device=dev)
    lossf = torch.nn.CrossEntropyLoss()
    stream = torch.cuda.current_stream(dev)

    def step():
        opt.zero_grad(set_to_none=True)
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=args.amp == "bf16"):
            loss = lossf(model(x), y)
        loss.backward()
        opt.step()
        return loss

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ts = []
    for _ in range(args.iters):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        loss = step()
        e.record(stream)
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    t = torch.tensor(ts, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = t.median().item()
    if rank == 0:
        print(json.dumps({
            "config": "config5: ResNet-50 DDP step, synthetic 3x224x224, 1000 classes",
            "comm": args.comm if world > 1 else "none", "n_gpus": world, "batch_per_gpu": args.batch,
            "nblocks": args.nblocks if args.comm == "ours" else None,
            "threads": args.threads if args.comm == "ours" else None, "bucket_view": bool(args.bucket_view),
            "amp": args.amp, "params": nparams, "grad_bytes": nparams * 4,
            "t_iter_ms": round(t_ms, 3), "images_per_s": round(world * args.batch / t_ms * 1e3, 1),
            "loss": float(loss.item()),
            "hook_buckets": hook_state.buckets if hook_state else None,
        }), flush=True)
    if hook_state is not None:
        hook_state.ctx.close()  # before the process-group teardown (close communicators first)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
