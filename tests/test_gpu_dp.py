"""MultiringDataParallel (paper_1708_02188_b200/dp.py) on 2 and 4 GPUs (grids
(2,) and (2,2)): gradients reduced bucket by bucket from autograd hooks, in the gradient arena, are
bit-identical to the reference's allreduce of every bucket (oracle closed form
over all ranks' local gradients, one allreduce per bucket as with
Workload.lengths, runtime.py:390-398) times 1/N; the same step captured into a
CUDA graph and replayed gives the same bits; NCCL through the same machinery
agrees to rounding.  Ranks share the GPUs round-robin on smaller boxes, with
gloo (on CUDA tensors) standing in for NCCL as the comparison backend."""

import os
import socket

import pytest

from conftest import cuda_count, host_backend, rank_device

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _model(dev):
    import torch

    torch.manual_seed(0)
    # 1.14 M parameters; at a 256 KiB first cap and 512 KiB caps: 3 buckets of 0.87, 2.6 and 1.05 MB
    # (the first goes through the LL kernel, the others through the step kernel)
    return torch.nn.Sequential(torch.nn.Linear(256, 1024), torch.nn.ReLU(), torch.nn.Linear(1024, 640),
                               torch.nn.ReLU(), torch.nn.Linear(640, 333), torch.nn.ReLU(),
                               torch.nn.Linear(333, 10)).to(dev)


def _main(rank, world, port, q):
    import numpy as np
    import torch
    import torch.distributed as dist

    from oracle import ringbox_oracle as orc
    from paper_1708_02188_b200.dp import MultiringDataParallel
    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import RankContext

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    d = rank_device(rank)
    torch.cuda.set_device(d)
    dev = torch.device("cuda", d)
    backend = host_backend(world)  # gloo when ranks share a GPU (NCCL refuses that)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gloo = dist.new_group(backend="gloo")
        torch.manual_seed(100 + rank)
        x = torch.randn(64, 256, device=dev)
        y = torch.randint(0, 10, (64,), device=dev)

        def loss_of(m):
            return torch.nn.functional.cross_entropy(m(x), y)

        # local gradients (no communication), accumulated into zeroed grads like the arena
        plain = _model(dev)
        for p in plain.parameters():
            p.grad = torch.zeros_like(p)
        loss_of(plain).backward()

        dims = {2: (2,), 4: (2, 2)}[world]
        ctx = RankContext(rank, Grid(dims), group=gloo, device=d, blocking=False)
        model = _model(dev)
        dp = MultiringDataParallel(model, ctx, bucket_cap_mb=0.5, first_bucket_mb=0.25)
        nb = len(dp.buckets)
        dp.zero_grad()
        loss_of(dp).backward()
        torch.cuda.synchronize()
        ctx.check()
        got = dp.arena.cpu().numpy().copy()
        launched = dp.launched

        # expected: every bucket allreduced on its own in the reference order, times 1/N
        name = {id(p): n for n, p in model.named_parameters()}
        pl = dict(plain.named_parameters())
        local = np.concatenate([pl[name[id(p)]].grad.detach().cpu().numpy().ravel()
                                for b in dp.buckets for p in b]).astype(np.float32)
        parts = [None] * world
        dist.all_gather_object(parts, local, group=gloo)
        want = np.empty_like(local)
        for lo, hi in dp.ranges:
            red = orc.closed_form_allreduce(orc.Grid(dims), [pt[lo:hi] for pt in parts])
            want[lo:hi] = red * np.float32(1.0 / world)
        exact = bool(np.array_equal(got.view(np.uint32), want.view(np.uint32)))

        # no_sync(): the first backward accumulates locally, the second reduces the sum
        # (2x every local gradient: exactly twice the reduced bits, x2 commutes with RNE)
        dp.zero_grad()
        with dp.no_sync():
            loss_of(dp).backward()
        loss_of(dp).backward()
        torch.cuda.synchronize()
        exact = exact and bool(np.array_equal(dp.arena.cpu().numpy().view(np.uint32),
                                              (got * np.float32(2)).view(np.uint32)))
        launched_twice = dp.launched == 2 * len(dp.buckets)

        # the same step captured into a CUDA graph and replayed
        def step():
            dp.zero_grad()
            loss_of(dp).backward()

        g = dp.capture(step, warmup=2)
        dp.arena.fill_(7.0)
        g.replay()
        torch.cuda.synchronize()
        ctx.check()
        graph_same = bool(np.array_equal(dp.arena.cpu().numpy().view(np.uint32), got.view(np.uint32)))
        dp.close()

        # NCCL through the same arena/hook machinery
        model2 = _model(dev)
        dp2 = MultiringDataParallel(model2, comm="nccl", bucket_cap_mb=0.5, first_bucket_mb=0.25)
        dp2.zero_grad()
        loss_of(dp2).backward()
        torch.cuda.synchronize()
        close = bool(np.allclose(dp2.arena.cpu().numpy(), got, rtol=1e-5, atol=1e-7))
        dp2.close()
        ctx.close()
        q.put((rank, "ok", exact, graph_same, close, nb, launched if launched_twice else -1))
    except Exception as exc:  # noqa: BLE001
        import traceback

        q.put((rank, "error", traceback.format_exc(), False, False, 0, 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_dp_buckets_bit_exact_and_graph_replay(world):
    if cuda_count() < 1:
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for rank, status, exact, graph_same, close, nb, launched in res:
        assert status == "ok", exact
        assert exact, f"rank {rank}: bucket gradients differ from the reference order"
        assert graph_same, f"rank {rank}: graph replay differs from the eager step"
        assert close, f"rank {rank}: NCCL through the same machinery differs beyond rounding"
        assert nb == 3, nb
        assert launched == nb
