"""Multi-process parity: one process per rank, IPC-mapped peer buffers, real
IPC handles.  On a box with N >= world GPUs every rank has its own GPU and the
peer traffic crosses NVLink; with fewer GPUs the rank processes share them
round-robin (conftest.rank_device), so the whole per-process path -- handle
exchange, mappings, flags, watchdog -- runs on a 1-GPU box too.

Mirrors the reference's runtime tests (pkg/tests/test_runtime.py:174-228,
test_acceptance.py:41-73): digests equal the reference replay/runtime
digests bit-for-bit, traffic counters follow 2(N-1)/N, a crashed rank is
detected and attributed, a shape mismatch aborts cleanly."""

import hashlib
import os
import socket

import numpy as np
import pytest

from conftest import cuda_count, golden, rank_device
from oracle import ringbox_oracle as orc

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dkey(d):
    return "x".join(map(str, d))


def _rank_main(rank, world, port, cases, q):
    import torch
    import torch.distributed as dist

    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import PlacedBuffer, RankContext, allgather, allreduce, reduce_scatter

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dev = rank_device(rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    try:
        for case in cases:
            dims, mode, dtype, lengths, seed = case["dims"], case["mode"], case["dtype"], case["lengths"], case["seed"]
            ctx = RankContext(rank, Grid(tuple(dims)), device=dev, mode=mode)
            for it, length in enumerate(lengths):
                x = orc.generate_input(seed, it, rank, length, dtype)
                t = ctx.empty(length, dtype)
                t.copy_(torch.from_numpy(x))
                buf = PlacedBuffer(t, device=f"cuda:{dev}")
                op = case.get("op", "allreduce")
                if op == "allreduce":
                    allreduce(ctx, buf)
                else:
                    view = reduce_scatter(ctx, buf)
                    owned = view.clone()
                    t.fill_(float("nan") if dtype != "i64" else -7)
                    view.copy_(owned)
                    allgather(ctx, buf)
                torch.cuda.synchronize()
                out.append((tuple(dims), mode, dtype, it, length, op,
                            hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest(), ctx.bytes_sent))
            ctx.close()
        q.put((rank, "ok", out))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, "error", repr(exc)))
    finally:
        dist.destroy_process_group()


def _spawn(world, cases, timeout=600):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=timeout)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
    for r, v in res.items():
        assert v[1] == "ok", v
    return res


def _dims_for(world):
    return [d for d in orc.factorizations(world, 3)]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_all_decompositions_all_modes_bit_exact(world):
    if cuda_count() < 1:
        pytest.skip("no CUDA device")
    g = golden("replay_digests")
    lengths = [0, 1, 17, 1000, 4099]
    cases = []
    for dims in _dims_for(world):
        for mode in ("fused", "fused_pull", "ring_dims", "push", "ll"):
            for dtype in ("f32", "i64", "f64"):
                cases.append({"dims": dims, "mode": mode, "dtype": dtype, "lengths": lengths, "seed": world})
    res = _spawn(world, cases)
    for r in range(world):
        for dims, mode, dtype, it, length, op, dig, _ in res[r][2]:
            assert dig == g[f"{_dkey(dims)}:{dtype}:{it}:{length}"], (r, dims, mode, dtype, length)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_reference_runtime_digests_and_traffic(world):
    """Same inputs as the reference RUNTIME run (tests/golden/runtime_digests.json)."""
    if cuda_count() < 1:
        pytest.skip("no CUDA device")
    g = golden("runtime_digests")
    grids = {2: [(2,)], 4: [(2, 2), (4,)], 8: [(2, 4), (2, 2, 2), (8,)]}[world]
    cases = [{"dims": d, "mode": "auto", "dtype": dt, "lengths": [0, 1, 17, 1000], "seed": world}
             for d in grids for dt in ("f32", "i64")]
    res = _spawn(world, cases)
    for r in range(world):
        sent = {}
        for dims, mode, dtype, it, length, op, dig, bytes_sent in res[r][2]:
            assert dig == g[f"{_dkey(dims)}:{dtype}:{it}:{length}"]
            sent[(dims, dtype)] = bytes_sent
        for (dims, dtype), b in sent.items():
            assert b == g[f"{_dkey(dims)}:{dtype}:bytes_sent"][r]  # reference traffic counter


@pytest.mark.parametrize("world", [2, 4, 8])
def test_reduce_scatter_allgather_pair(world):
    if cuda_count() < 1:
        pytest.skip("no CUDA device")
    # fused / auto: reduce_scatter and allgather each through the specialised kernel
    # (fold N -> store 1, copy 1 -> store N-1), aligned bodies and scalar edges
    grids = _dims_for(world) if world < 8 else [(2, 4), (2, 2, 2), (8,)]
    cases = [{"dims": d, "mode": m, "dtype": "f32", "lengths": [10007, 1], "seed": 11, "op": "rs+ag"}
             for d in grids for m in ("fused", "ring_dims", "push")]
    cases += [{"dims": d, "mode": "auto", "dtype": dt, "lengths": [1_000_003, 4096], "seed": 12, "op": "rs+ag"}
              for d in grids for dt in (("f32", "f64", "i64") if world < 8 else ("f32", "i64"))]
    res = _spawn(world, cases)
    for r in range(world):
        for dims, mode, dtype, it, length, op, dig, _ in res[r][2]:
            seed = 11 if mode != "auto" else 12
            parts = [orc.generate_input(seed, it, q, length, dtype) for q in range(world)]
            want = orc.closed_form_allreduce(orc.Grid(dims), parts)
            assert dig == orc.sha256(want), (dims, mode, dtype, length)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_full_size_config(world):
    if cuda_count() < 1:
        pytest.skip("no CUDA device")
    n = 25_600_000
    cases = [{"dims": d, "mode": m, "dtype": "f32", "lengths": [n], "seed": 0}
             for d in ([(2, 4), (2, 2, 2)] if world == 8 else _dims_for(world)[:1]) for m in ("fused", "ring_dims", "push")]
    res = _spawn(world, cases)
    large = golden("large_digests")
    for r in range(world):
        for dims, mode, dtype, it, length, op, dig, _ in res[r][2]:
            key = f"{_dkey(dims)}:f32:seed0:{n}"
            if key in large:
                assert dig == large[key]
            else:
                parts = [orc.generate_input(0, 0, q, n, "f32") for q in range(world)]
                assert dig == orc.sha256(orc.closed_form_allreduce(orc.Grid(dims), parts))


def _bucket_main(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import RankContext

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dev = rank_device(rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sizes = [2049, 7875, 6563, 1, 0, 6965, 1098]
        ctx = RankContext(rank, Grid((world,) if world < 4 else (2, world // 2)), device=dev)
        flat = ctx.empty(sum(sizes), "f32")
        xs = [orc.generate_input(5, k, rank, s, "f32") for k, s in enumerate(sizes)]
        views, off = [], 0
        for s, x in zip(sizes, xs):
            v = flat[off:off + s]
            v.copy_(torch.from_numpy(x))
            views.append(v)
            off += s
        ctx.allreduce_buckets(views)
        torch.cuda.synchronize()
        q.put((rank, "ok", [hashlib.sha256(v.cpu().numpy().tobytes()).hexdigest() for v in views], ctx.launches))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, "error", repr(exc), None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_bucket_list_one_launch(world):
    """Config 4 semantics: a bucket list reduced in ONE launch, each bucket
    chunked on its own exactly like a Workload.lengths entry."""
    if cuda_count() < 1:
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_bucket_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    dims = (world,) if world < 4 else (2, world // 2)
    sizes = [2049, 7875, 6563, 1, 0, 6965, 1098]
    for rank, status, digs, launches in res:
        assert status == "ok", digs
        assert launches == 1
        for k, s in enumerate(sizes):
            parts = [orc.generate_input(5, k, q_, s, "f32") for q_ in range(world)]
            assert digs[k] == orc.sha256(orc.closed_form_allreduce(orc.Grid(dims), parts))


def _bf16_main(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import RankContext

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dev = rank_device(rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        dims = (2, world // 2) if world >= 4 else (world,)
        for mode in ("fused", "ring_dims", "push", "ll"):
            ctx = RankContext(rank, Grid(dims), device=dev, mode=mode)
            rng = np.random.default_rng(100 + rank)
            bits = orc.bf16_round(rng.standard_normal(30_011).astype(np.float32))
            t = ctx.empty(len(bits), "bf16")
            t.copy_(torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16))
            ctx.collective("allreduce", t)
            out.append((mode, hashlib.sha256(t.view(torch.int16).cpu().numpy().tobytes()).hexdigest()))
            ctx.close()
        q.put((rank, "ok", out))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, "error", repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_bf16_all_modes_match_policy(world):
    """bf16 (fp32 accumulate, one RNE): FUSED, RING_DIMS (fp32 partial
    workspaces between stages) and PUSH all equal the oracle policy."""
    if cuda_count() < 1:
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_bf16_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    dims = (2, world // 2) if world >= 4 else (world,)
    parts = [orc.bf16_round(np.random.default_rng(100 + r).standard_normal(30_011).astype(np.float32))
             for r in range(world)]
    want = orc.sha256(orc.bf16_allreduce(orc.Grid(dims), parts).view(np.int16))
    for rank, status, out in res:
        assert status == "ok", out
        for mode, dig in out:
            assert dig == want, (rank, mode)


def _calib_main(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1708_02188_b200.calibrate import calibrated_topology
    from paper_1708_02188_b200.multiring import Grid, plan
    from paper_1708_02188_b200.runtime import RankContext

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dev = rank_device(rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = RankContext(rank, Grid((world,)), device=dev, blocking=False)
        t, m = calibrated_topology(ctx, big_elems=16 * 1024 * 1024, iters=4)
        p = plan(t, t.devices(), 0.1024)
        # errors surface as the reference's exception types
        errs = []
        stray = torch.empty(1000, device=f"cuda:{dev}")
        try:
            import ctypes

            from paper_1708_02188_b200 import _native

            _native.check(ctx._L.rbx_allreduce(ctx._comm, ctypes.c_void_p(stray.data_ptr()), 1000, 0, 0, None))
        except ValueError as exc:
            errs.append("unregistered:" + str(exc)[:40])
        q.put((rank, "ok", m, p.grid.dims, errs))
        ctx.close()
    except Exception as exc:  # noqa: BLE001
        q.put((rank, "error", repr(exc), None, None))
    finally:
        dist.destroy_process_group()


def test_planner_calibration_and_abi_errors():
    """measured per-stage latency and bus bandwidth feed the
    reference planner through a B200 topology; unregistered buffers are refused."""
    if cuda_count() < 1:
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_calib_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    shared = cuda_count() < 2  # two time-sliced contexts on one GPU: a barrier costs a time slice
    for rank, status, m, dims, errs in res:
        assert status == "ok", m
        if shared:
            assert m["latency_s"] > 0 and m["bandwidth_gbps"] > 0
        else:
            assert 0 < m["latency_s"] < 1e-3 and m["bandwidth_gbps"] > 100
        assert m == res[0][2], "ranks must feed the planner the same calibration"
        assert dims == (2,)
        assert errs and errs[0].startswith("unregistered:buffer is not registered")


def test_launch_api_matches_reference_and_detects_faults():
    """`launch` (runtime.py:435-589): serial-oracle digests for i64, a crashed
    rank is attributed, a shape mismatch aborts."""
    if cuda_count() < 1:
        pytest.skip("no CUDA device")
    from paper_1708_02188_b200.runtime import Workload, generate_input, launch

    n, dims = 4, (2, 2)
    w = Workload(lengths=(0, 1, 17, 64), seed=11)
    rep = launch(n, dims, w, share_gpus=True)
    assert rep.ok, rep.error
    for it, length in enumerate(w.lengths):
        total = np.sum([generate_input(w, it, r, length) for r in range(n)], axis=0).astype(np.int64)
        want = hashlib.sha256(np.asarray(total, dtype=np.int64).tobytes()).hexdigest()
        assert {rep.results[r].digests[it] for r in range(n)} == {want}
    rep = launch(2, (2,), Workload(lengths=(50,), seed=1, length_overrides={1: 49}), share_gpus=True)
    assert not rep.ok and "mismatch" in rep.error
    rep = launch(n, (n,), Workload(lengths=(100,), seed=1, crash_rank=1, crash_phase=1), timeout_s=15,
                 share_gpus=True)
    assert not rep.ok and rep.failed_rank == 1


def _edge_main(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import RankContext

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dev = rank_device(rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    try:
        for dims in _dims_for(world):
            ctx = RankContext(rank, Grid(tuple(dims)), device=dev, mode="fused", nblocks=16)
            for dtype, n in (("f32", 100_003), ("i64", 33_335), ("f64", 4099)):
                x = orc.generate_input(21, 0, rank, n, dtype)
                # (1) a view 1 element past a 16-byte boundary on every rank: scalar head/tail peel
                base = ctx.empty(n + 3, dtype)
                t = base[1:1 + n]
                t.copy_(torch.from_numpy(x))
                ctx.collective("allreduce", t)
                out.append(("misaligned", tuple(dims), dtype, n, orc.sha256(t.cpu().numpy())))
                # (2) three element windows compose to the full allreduce
                w = ctx.empty(n, dtype)
                w.copy_(torch.from_numpy(x))
                for lo, hi in ((0, n // 3), (n // 3, n - 5), (n - 5, n)):
                    ctx.allreduce_window(w, lo, hi)
                out.append(("windows", tuple(dims), dtype, n, orc.sha256(w.cpu().numpy())))
            # (3) a bucket list (one launch; the multi-segment form of the kernel)
            sizes = [5000, 1, 0, 12_345, 777]
            flat = ctx.empty(sum(sizes) + 1, "f32")
            views, off = [], 1
            for k, s in enumerate(sizes):
                v = flat[off:off + s]
                v.copy_(torch.from_numpy(orc.generate_input(22, k, rank, s, "f32")))
                views.append(v)
                off += s
            l0 = ctx.launches
            ctx.allreduce_buckets(views)
            out.append(("buckets", tuple(dims), "f32", ctx.launches - l0,
                        [orc.sha256(v.cpu().numpy()) for v in views]))
            ctx.close()
        q.put((rank, "ok", out))
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, "error", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_fused_kernel_misaligned_windows_buckets(world):
    """The specialised FUSED kernel (rbx_fused.cuh) on the per-rank path: views
    whose element 0 is not 16-byte aligned (scalar edges), element windows
    (rbx_allreduce_window) and a bucket list with empty and 1-element buckets,
    every result equal to the reference-order fold bit for bit."""
    if cuda_count() < 1:
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_edge_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=900) for _ in range(world)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    for item in res:
        assert item[1] == "ok", item[2]
    sizes = [5000, 1, 0, 12_345, 777]
    for rank, _, out in res:
        for kind, dims, dtype, n, dig in out:
            g = orc.Grid(dims)
            if kind == "buckets":
                assert n == 1, "bucket list must be one launch"
                for k, s in enumerate(sizes):
                    parts = [orc.generate_input(22, k, r, s, "f32") for r in range(world)]
                    assert dig[k] == orc.sha256(orc.closed_form_allreduce(g, parts)), (rank, dims, k)
            else:
                parts = [orc.generate_input(21, 0, r, n, dtype) for r in range(world)]
                assert dig == orc.sha256(orc.closed_form_allreduce(g, parts)), (rank, kind, dims, dtype)


def _random_cases(world, seed=2024, count=10):
    """Seeded random cases for the specialised kernels: lengths that do not
    divide by the grid (ragged reference chunks), views 0-3 elements past a
    16-byte boundary, windows, every dtype, FUSED and RING_DIMS."""
    rng = np.random.default_rng(seed + world)
    grids = [tuple(d) for d in orc.factorizations(world, 3)]
    cases = []
    for k in range(count):
        dims = grids[int(rng.integers(len(grids)))]
        dtype = ["f32", "f64", "i64", "bf16"][int(rng.integers(4))]
        mode = ["fused", "ring_dims"][int(rng.integers(2))]
        n = int(rng.integers(1, 300_000))
        shift = int(rng.integers(0, 4)) if mode == "fused" else 0
        window = None
        if mode == "fused" and rng.random() < 0.4:
            lo = int(rng.integers(0, n))
            window = (lo, int(rng.integers(lo, n + 1)))
        cases.append({"dims": dims, "dtype": dtype, "mode": mode, "n": n, "shift": shift, "window": window, "seed": k})
    return cases


def _rand_input(case, rank):
    if case["dtype"] == "bf16":
        x = np.random.default_rng(1000 * case["seed"] + rank).standard_normal(case["n"]).astype(np.float32)
        return orc.bf16_round(x)
    return orc.generate_input(case["seed"], 1, rank, case["n"], case["dtype"])


def _rand_main(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import RankContext

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dev = rank_device(rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    try:
        for case in _random_cases(world):
            ctx = RankContext(rank, Grid(case["dims"]), device=dev, mode=case["mode"], nblocks=32)
            x = _rand_input(case, rank)
            base = ctx.empty(case["n"] + 4, case["dtype"])
            t = base[case["shift"]:case["shift"] + case["n"]]
            src = torch.from_numpy(x.view(np.int16)).view(torch.bfloat16) if case["dtype"] == "bf16" else torch.from_numpy(x)
            t.copy_(src)
            if case["window"]:
                ctx.allreduce_window(t, *case["window"])
            else:
                ctx.collective("allreduce", t)
            got = t.view(torch.int16).cpu().numpy() if case["dtype"] == "bf16" else t.cpu().numpy()
            out.append(orc.sha256(got))
            ctx.close()
        q.put((rank, "ok", out))
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, "error", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_specialised_kernels_randomised(world):
    """rbx_fused_kernel / rbx_rings_kernel on seeded random shapes: every grid of
    the world, f32/f64/i64/bf16, ragged lengths, misaligned views, windows --
    each rank's buffer equal to the reference-order fold (bf16: the fp32-
    accumulate policy) bit for bit; outside a window the input is untouched."""
    if cuda_count() < 1:
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rand_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=900) for _ in range(world)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    for item in res:
        assert item[1] == "ok", item[2]
    for k, case in enumerate(_random_cases(world)):
        g = orc.Grid(case["dims"])
        parts = [_rand_input(case, r) for r in range(world)]
        want = [orc.bf16_allreduce(g, parts)] * world if case["dtype"] == "bf16" else \
            [orc.closed_form_allreduce(g, parts)] * world
        for r in range(world):
            w = want[r].copy()
            if case["window"]:
                lo, hi = case["window"]
                w = parts[r].copy()
                w[lo:hi] = want[r][lo:hi]
            assert res[r][2][k] == orc.sha256(w), (r, case)


def _kernel_rank_main(rank, world, port, cases, q):
    import torch
    import torch.distributed as dist

    from paper_1708_02188_b200.multiring import Grid
    from paper_1708_02188_b200.runtime import RankContext

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dev = rank_device(rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    try:
        for dims, op, mode, dtype, n in cases:
            ctx = RankContext(rank, Grid(tuple(dims)), device=dev, mode=mode)
            x = orc.generate_input(5, 0, rank, n, "f32" if dtype == "bf16" else dtype)
            t = ctx.empty(n, dtype)
            t.copy_(torch.from_numpy(x))  # bf16: RNE of the fp32 inputs
            ctx.collective(op, t)
            torch.cuda.synchronize()
            out.append(((tuple(dims), op, mode, dtype, n), ctx.last_kernel()))
            ctx.close()
        q.put((rank, "ok", out))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, "error", repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_calls_take_the_specialised_kernels(world):
    """rbx_comm_last_kernel: each collective of the box's grids runs the kernel the
    design says it runs -- never a silent fallback to the
    generic step interpreter."""
    if cuda_count() < 1:
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    big, small = 1_000_000, 1000
    grid = (2,) if world == 2 else (2, 2)
    cases = [(grid, "allreduce", "auto", "f32", big), (grid, "reduce_scatter", "auto", "f32", big),
             (grid, "allgather", "auto", "f32", big), (grid, "allreduce", "auto", "f32", small),
             (grid, "allreduce", "auto", "bf16", big), (grid, "allreduce", "push", "f32", big),
             (grid, "allreduce", "fused_pull", "f32", big)]
    want = ["fused", "fused", "fused", "ll", "fused", "rings", "step"]
    if world == 4:
        cases += [(grid, "allreduce", "ring_dims", "f32", big), (grid, "reduce_scatter", "ring_dims", "f32", big),
                  ((4,), "allreduce", "auto", "i64", big)]
        want += ["rings", "rings", "fused"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_kernel_rank_main, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=600)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
    for r, v in res.items():
        assert v[1] == "ok", v
        got = [k for _, k in v[2]]
        assert got == want, list(zip([c for c, _ in v[2]], got, want))
