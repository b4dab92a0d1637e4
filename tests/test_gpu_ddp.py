"""DDP communication hook on 2 GPUs (config 5 integration): gradients reduced
by the multi-ring kernel agree bitwise across ranks and match NCCL's average
to float rounding (NCCL, or gloo when the two ranks share one GPU)."""

import os
import socket

import pytest

from conftest import cuda_count, host_backend, rank_device

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _main(rank, world, port, q):
    import hashlib

    import torch
    import torch.distributed as dist

    from paper_1708_02188_b200.ddp import MultiringHookState, multiring_allreduce_hook
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
        results = {}
        for comm in ("ours", "nccl"):
            torch.manual_seed(0)
            model = torch.nn.Sequential(torch.nn.Linear(256, 512), torch.nn.ReLU(), torch.nn.Linear(512, 10)).to(dev)
            ddp = torch.nn.parallel.DistributedDataParallel(model, device_ids=[d], bucket_cap_mb=1)
            if comm == "ours":
                ctx = RankContext(rank, Grid((world,)), group=gloo, device=d, blocking=False)
                state = MultiringHookState(ctx)
                ddp.register_comm_hook(state, multiring_allreduce_hook)
            torch.manual_seed(100 + rank)
            x = torch.randn(64, 256, device=dev)
            y = torch.randint(0, 10, (64,), device=dev)
            for _ in range(3):
                ddp.zero_grad()
                torch.nn.functional.cross_entropy(ddp(x), y).backward()
            torch.cuda.synchronize()
            grads = torch.cat([p.grad.flatten() for p in model.parameters()])
            results[comm] = grads.cpu()
            if comm == "ours":
                results["buckets"] = state.buckets
                ctx.check()
        dig = hashlib.sha256(results["ours"].numpy().tobytes()).hexdigest()
        close = torch.allclose(results["ours"], results["nccl"], rtol=1e-5, atol=1e-7)
        q.put((rank, "ok", dig, bool(close), results["buckets"]))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, "error", repr(exc), False, 0))
    finally:
        dist.destroy_process_group()


def test_ddp_hook_two_gpus():
    if cuda_count() < 1:
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for rank, status, dig, close, buckets in res:
        assert status == "ok", dig
        assert close, "multi-ring hook gradients differ from NCCL beyond rounding"
        assert buckets > 0
    assert res[0][2] == res[1][2], "ranks disagree bitwise"
