"""The reference's in-process collective tests (pkg/tests/test_runtime.py:124-171),
restated over real GPUs: one process per GPU, the same PlacedBuffer /
allreduce / reduce_scatter / allgather calls, numpy buffers (staged through
the GPU, memory="host") and CUDA tensors (memory="device").

  * hand values [1,2,3,4] + [10,20,30,40] (125-133);
  * reduce_scatter returns a view that shares memory with the buffer (135-142);
  * allgather broadcasts the owned chunks (144-158);
  * a length mismatch raises CollectiveError (160-164);
  * bytes_sent counts the payload: 2 x 5 elements x 8 bytes for N=2, length 10 (166-171).
"""

import os
import socket

import numpy as np
import pytest

from conftest import cuda_count

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _main(rank, world, port, scenario, q):
    import torch
    import torch.distributed as dist

    from paper_1708_02188_b200.errors import CollectiveError
    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import (PlacedBuffer, RankContext, allgather, allreduce, owned_region,
                                                reduce_scatter)

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dev = rank % torch.cuda.device_count()  # up to 2 ranks per GPU on smaller boxes (time-sliced)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = RankContext(rank, Grid((world,)), device=dev)
        if scenario == "hand_values":
            out = {}
            for memory in ("host", "device"):
                x = np.array([1, 2, 3, 4], dtype=np.int64) * (10 if rank == 1 else 1)
                if memory == "device":
                    t = ctx.empty(4, "i64")
                    t.copy_(torch.from_numpy(x))
                    buf = PlacedBuffer(t, device=f"cuda:{dev}")
                else:
                    buf = PlacedBuffer(x)
                res = allreduce(ctx, buf)
                assert res is buf  # same object back (runtime.py:295-297)
                got = res.data if memory == "host" else res.data.cpu().numpy()
                out[memory] = got.tolist()
            q.put((rank, "ok", out))
        elif scenario == "owned_view":
            out = {}
            for memory in ("host", "device"):
                x = np.full(8, rank + 1, dtype=np.int64)
                if memory == "device":
                    t = ctx.empty(8, "i64")
                    t.copy_(torch.from_numpy(x))
                    buf = PlacedBuffer(t, device=f"cuda:{dev}")
                else:
                    buf = PlacedBuffer(x)
                view = reduce_scatter(ctx, buf)
                off, length = owned_region(ctx.grid, rank, 8)
                if memory == "host":
                    shares = bool(np.shares_memory(view, buf.data))
                    vals = view.tolist()
                else:
                    torch.cuda.synchronize()
                    shares = view.untyped_storage().data_ptr() == buf.data.untyped_storage().data_ptr()
                    vals = view.cpu().tolist()
                out[memory] = (vals, length, shares)
            q.put((rank, "ok", out))
        elif scenario == "allgather":
            n = 6
            data = np.zeros(n, dtype=np.int64)
            off, length = owned_region(ctx.grid, rank, n)
            data[off:off + length] = rank + 1
            buf = PlacedBuffer(data)
            allgather(ctx, buf)
            regions = [owned_region(ctx.grid, r, n) for r in range(world)]
            q.put((rank, "ok", (buf.data.tolist(), regions)))
        elif scenario == "mismatch":
            buf = PlacedBuffer(np.zeros(4 if rank == 0 else 6, np.int64))
            try:
                allreduce(ctx, buf)
                q.put((rank, "ok", "no error"))
            except CollectiveError as exc:
                q.put((rank, "ok", ("CollectiveError", str(exc))))
        elif scenario == "host_pipeline":
            # multi-window host path (hoststage: page-locked, 3 streams, tapered windows) on a
            # malloc'd array and on a runtime.host_empty array; results vs the reference order
            from oracle import ringbox_oracle as orc
            from paper_1708_02188_b200.runtime import host_empty

            n = 3_000_017  # 12 MB of f32: 11 windows, ragged
            out = []
            for kind in ("numpy", "host_empty"):
                x = orc.generate_input(31, 0, rank, n, "f32")
                arr = x.copy() if kind == "numpy" else host_empty(n, "f32")
                arr[...] = x
                allreduce(ctx, PlacedBuffer(arr, memory="host"))
                out.append((kind, orc.sha256(arr)))
            q.put((rank, "ok", out))
        elif scenario == "bytes_sent":
            buf = PlacedBuffer(np.arange(10, dtype=np.int64))
            allreduce(ctx, buf)
            q.put((rank, "ok", ctx.bytes_sent))
        ctx.close()
    except Exception as exc:  # noqa: BLE001
        q.put((rank, "error", repr(exc)))
    finally:
        dist.destroy_process_group()


def _run(world, scenario):
    import torch.multiprocessing as mp

    if cuda_count() < 1:
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_main, args=(r, world, port, scenario, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=300)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
    for v in res.values():
        assert v[1] == "ok", v
    return {r: v[2] for r, v in res.items()}


def test_allreduce_two_ranks_hand_values():
    for r, out in _run(2, "hand_values").items():
        assert out == {"host": [11, 22, 33, 44], "device": [11, 22, 33, 44]}, r


@pytest.mark.parametrize("world", [2, 4])
def test_reduce_scatter_returns_owned_view(world):
    for r, out in _run(world, "owned_view").items():
        for memory, (vals, length, shares) in out.items():
            want = world * (world + 1) // 2
            assert vals == [want] * length, (r, memory)
            assert shares, (r, memory)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_allgather_broadcasts_owned_chunks(world):
    res = _run(world, "allgather")
    _, regions = res[0]
    expect = np.zeros(6, dtype=np.int64)
    for r, (off, length) in enumerate(regions):
        expect[off:off + length] = r + 1
    for r, (data, _) in res.items():
        assert data == expect.tolist(), r


def test_length_mismatch_raises():
    for r, out in _run(2, "mismatch").items():
        assert out[0] == "CollectiveError", (r, out)


@pytest.mark.parametrize("world", [2, 4])
def test_host_buffer_pipeline_matches_reference(world):
    """PlacedBuffer(memory="host") through the windowed host pipeline equals the
    reference-order allreduce bit for bit, for plain and host_empty arrays."""
    from oracle import ringbox_oracle as orc

    n = 3_000_017
    parts = [orc.generate_input(31, 0, r, n, "f32") for r in range(world)]
    want = orc.sha256(orc.closed_form_allreduce(orc.Grid((world,)), parts))
    for r, out in _run(world, "host_pipeline").items():
        for kind, dig in out:
            assert dig == want, (r, kind)


def test_bytes_sent_counts_payload():
    # each rank sends half the buffer twice: 5 elements * 8 bytes * 2
    assert set(_run(2, "bytes_sent").values()) == {80}
