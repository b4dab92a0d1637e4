"""The 8-rank per-process path (configs 1/2: grids 2x4 and 2x2x2) on whatever
GPUs the box has: 8 spawned processes, several per GPU (time-sliced contexts),
each with its own communicator, IPC mappings and flags, exactly as on an
8-GPU box.  Every rank's result must equal the reference-order fold bit for
bit (oracle closed form = reference replay, tests/test_oracle.py)."""

import os
import socket

import pytest

from conftest import cuda_count

pytestmark = pytest.mark.gpu

RANKS = 8


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _main(rank, port, q):
    import torch
    import torch.distributed as dist

    from oracle import ringbox_oracle as orc
    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import RankContext

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dev = rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=RANKS)
    out = []
    try:
        for dims in ((2, 2, 2), (2, 4)):
            ctx = RankContext(rank, Grid(dims), device=dev, nblocks=8, timeout_s=20.0, blocking=False)
            for mode, n in (("fused", 100_003), ("ring_dims", 4099), ("ll", 4099)):
                parts = [orc.generate_input(7, 0, r, n, "f32") for r in range(RANKS)]
                want = orc.sha256(orc.closed_form_allreduce(orc.Grid(dims), parts))
                t = ctx.empty(n, "f32")
                t.copy_(torch.from_numpy(parts[rank]))
                ctx.collective("allreduce", t, mode=mode)
                ctx.synchronize()
                out.append((dims, mode, n, orc.sha256(t.cpu().numpy()) == want))
            ctx.close()
        q.put((rank, "ok", out))
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, "error", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_eight_rank_processes_bit_exact():
    if cuda_count() < 1:
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_main, args=(r, port, q)) for r in range(RANKS)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(RANKS)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    for item in res:
        assert item[1] == "ok", item[2]
        for dims, mode, n, ok in item[2]:
            assert ok, f"rank {item[0]}: {dims} {mode} n={n} differs from the reference order"
