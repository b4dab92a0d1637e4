"""Multi-process host plumbing on CPU: world_size-2 gloo groups exercising the
handle exchange and shape agreement the GPU path uses at registration time
(reference: coordinator shape agreement, pkg/src/ringbox/runtime.py:528-543;
plan-hash handshake, runtime.py:374-386)."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1708_02188_b200.errors import CollectiveError
from paper_1708_02188_b200.exchange import agree, allgather_objects, plan_fingerprint


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, scenario, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if scenario == "handles":
            fake = bytes([rank]) * 64
            got = allgather_objects((fake, rank * 4096, 1024, "f32"))
            out.put((rank, "ok", [g[0][0] for g in got], [g[1] for g in got]))
        elif scenario == "agree":
            keys = agree(("allreduce", 1000, "f32", 2))
            out.put((rank, "ok", len(keys), None))
        elif scenario == "mismatch":
            try:
                agree(("allreduce", 1000 if rank == 0 else 999, "f32", 2), what="length")
                out.put((rank, "no-error", None, None))
            except CollectiveError as exc:
                out.put((rank, "error", exc.rank, str(exc)))
        elif scenario == "fingerprint":
            fp = plan_fingerprint((2, 2), "i64", (10,) if rank == 0 else (11,))
            try:
                agree(fp, what="plan hash")
                out.put((rank, "no-error", None, None))
            except CollectiveError as exc:
                out.put((rank, "error", exc.rank, str(exc)))
    finally:
        dist.destroy_process_group()


def _run(scenario, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scenario, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_handle_exchange_world2():
    res = _run("handles")
    for rank, status, firsts, offs in res:
        assert status == "ok" and firsts == [0, 1] and offs == [0, 4096]


def test_handle_exchange_world8():
    """The N=8 (2,2,2) bench/scale launch: every rank sees all 8 handles in rank order."""
    res = _run("handles", world=8)
    for rank, status, firsts, offs in res:
        assert status == "ok" and firsts == list(range(8)) and offs == [r * 4096 for r in range(8)]


def test_agreement_world2():
    assert all(r[1] == "ok" and r[2] == 2 for r in _run("agree"))


def test_length_mismatch_detected_on_every_rank():
    res = _run("mismatch")
    for rank, status, culprit, msg in res:
        assert status == "error" and culprit == 1 and "mismatch" in msg


def test_plan_fingerprint_mismatch_detected():
    res = _run("fingerprint")
    assert all(r[1] == "error" and r[2] == 1 for r in res)


def test_plan_fingerprint_sensitivity():
    base = plan_fingerprint((2, 2), "i64", (10,))
    assert plan_fingerprint((4,), "i64", (10,)) != base
    assert plan_fingerprint((2, 2), "f32", (10,)) != base
    assert plan_fingerprint((2, 2), "i64", (11,)) != base
    assert plan_fingerprint((2, 2), "i64", (10,)) == base


@pytest.mark.parametrize("world", [3])
def test_three_ranks(world):
    res = _run("handles", world)
    assert [r[2] for r in res] == [[0, 1, 2]] * 3
