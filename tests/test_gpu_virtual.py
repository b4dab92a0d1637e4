"""GPU parity tests on ONE B200: every rank of a grid hosted by one launch.

* mode "local": the 1-GPU local-reduce kernel (bench N=1 path);
* modes "fused" / "fused_pull" / "ring_dims": the real multi-rank kernel (flags,
  epochs, NVLink-style pushes/pulls, per-dimension stages), each rank played
  by a CTA group of one cooperative launch.

Results must equal the reference replay digests bit-for-bit (tests/golden),
computed through the C ABI (librbx.so) -- the oracle is only the checker."""

import numpy as np
import pytest

from conftest import golden
from oracle import ringbox_oracle as orc

pytestmark = pytest.mark.gpu

RANK_COUNTS = (2, 3, 4, 6, 8, 12, 16)
LENGTHS = (0, 1, 17, 1000, 4099)


def _torch():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def all_dims():
    for n in RANK_COUNTS:
        for dims in orc.factorizations(n, 3):
            yield n, tuple(dims)
    yield 4, (1, 4)
    yield 6, (2, 1, 3)
    yield 16, (2, 2, 2, 2)


def dkey(dims):
    return "x".join(map(str, dims))


def run(vr, parts, op, mode, dtype_t):
    torch = _torch()
    ts = [torch.from_numpy(p.copy()).to("cuda") for p in parts]
    vr.collective(ts, op=op, mode=mode)
    torch.cuda.synchronize()
    vr.check()
    return [t.cpu().numpy() for t in ts]


@pytest.mark.parametrize("mode", ["local", "fused", "fused_pull", "ring_dims", "push", "ll"])
def test_all_decompositions_bit_exact(mode):
    """tests/golden/replay_digests.json: reference acceptance sweep
    (pkg/tests/test_acceptance.py:41-73) on the GPU, f32/f64/i64."""
    torch = _torch()
    from paper_1708_02188_b200.virtual import VirtualRanks

    g = golden("replay_digests")
    for n, dims in all_dims():
        vr = VirtualRanks(dims, nblocks_per_rank=0 if mode == "local" else 4)
        for dtype in ("i64", "f32", "f64"):
            for it, length in enumerate(LENGTHS):
                parts = [orc.generate_input(n, it, r, length, dtype) for r in range(n)]
                out = run(vr, parts, "allreduce", mode, None)
                want = g[f"{dkey(dims)}:{dtype}:{it}:{length}"]
                digs = {orc.sha256(o) for o in out}
                assert digs == {want}, (mode, dims, dtype, length)
        vr.close()
    del torch


@pytest.mark.parametrize("dims", [(2, 4), (2, 2, 2), (8,), (4, 2)])
@pytest.mark.parametrize("length", [25_600_000, 25_557_032])
@pytest.mark.parametrize("mode", ["local", "fused", "ring_dims", "push"])
def test_full_size_configs(dims, length, mode):
    """Configs 1/2 at full size (102.4 MB fp32 per rank) vs the reference digest."""
    torch = _torch()
    from paper_1708_02188_b200.virtual import VirtualRanks

    want = golden("large_digests")[f"{dkey(dims)}:f32:seed0:{length}"]
    parts = [orc.generate_input(0, 0, r, length, "f32") for r in range(8)]
    vr = VirtualRanks(dims)
    out = run(vr, parts, "allreduce", mode, None)
    assert {orc.sha256(o) for o in out} == {want}
    vr.close()
    del torch


@pytest.mark.parametrize("mode", ["fused", "ring_dims", "push"])
def test_reduce_scatter_then_allgather(mode):
    torch = _torch()
    from paper_1708_02188_b200.virtual import VirtualRanks

    for dims in [(2,), (2, 2), (3, 2), (2, 2, 2), (2, 4), (8,), (4, 4)]:
        n = int(np.prod(dims))
        grid = orc.Grid(dims)
        length = 10_007
        parts = [orc.generate_input(3, 0, r, length, "f32") for r in range(n)]
        want = orc.closed_form_allreduce(grid, parts)
        vr = VirtualRanks(dims, nblocks_per_rank=4)
        ts = [torch.from_numpy(p.copy()).cuda() for p in parts]
        vr.collective(ts, op="reduce_scatter", mode=mode)
        torch.cuda.synchronize()
        for r in range(n):
            off, ln = orc.owned_region(grid, r, length)
            assert np.array_equal(ts[r][off:off + ln].cpu().numpy(), want[off:off + ln])
            mask = torch.ones(length, dtype=torch.bool, device="cuda")
            mask[off:off + ln] = False
            ts[r][mask] = float("nan")  # non-owned regions are unspecified
        vr.collective(ts, op="allgather", mode=mode)
        torch.cuda.synchronize()
        vr.check()
        for r in range(n):
            assert np.array_equal(ts[r].cpu().numpy(), want)
        vr.close()


@pytest.mark.parametrize("mode", ["local", "fused", "ring_dims", "push", "ll"])
def test_bf16_f16_fp32_accumulate(mode):
    """bf16/f16: fold fp32-upcast inputs in the reference order, one RNE at the
    end (parity unpinned by the reference, which has no bf16: runtime.py:37)."""
    torch = _torch()
    from paper_1708_02188_b200.virtual import VirtualRanks

    for dims in [(2, 2, 2), (2, 4), (8,), (3, 2)]:
        n = int(np.prod(dims))
        grid = orc.Grid(dims)
        rng = np.random.default_rng(5)
        xs32 = [rng.standard_normal(33_333).astype(np.float32) for _ in range(n)]
        vr = VirtualRanks(dims, nblocks_per_rank=0 if mode == "local" else 4)
        bits = [orc.bf16_round(x) for x in xs32]
        ts = [torch.from_numpy(b.view(np.int16)).cuda().view(torch.bfloat16) for b in bits]
        vr.collective(ts, mode=mode)
        torch.cuda.synchronize()
        want = orc.bf16_allreduce(grid, bits)
        for t in ts:
            got = t.view(torch.int16).cpu().numpy().view(np.uint16)
            assert np.array_equal(got, want)
        h = [x.astype(np.float16) for x in xs32]
        ts = [torch.from_numpy(x).cuda() for x in h]
        vr.collective(ts, mode=mode)
        torch.cuda.synchronize()
        want = orc.f16_allreduce(grid, h)
        for t in ts:
            assert np.array_equal(t.cpu().numpy().view(np.uint16), want.view(np.uint16))
        vr.close()


def test_repeated_calls_epochs_and_launch_count():
    """Flags are epoch-tagged: many back-to-back calls on the same buffers stay
    correct without any reset, and each call is exactly one kernel launch."""
    torch = _torch()
    from paper_1708_02188_b200.virtual import VirtualRanks

    dims = (2, 2, 2)
    grid = orc.Grid(dims)
    vr = VirtualRanks(dims, nblocks_per_rank=8)
    base = vr.launches
    rng = np.random.default_rng(1)
    for k in range(12):
        length = int(rng.integers(1, 50_000))
        parts = [rng.integers(-1000, 1001, length).astype(np.int64) for _ in range(8)]
        ts = [torch.from_numpy(p).cuda() for p in parts]
        mode = ["fused", "ring_dims", "fused_pull", "push", "ll"][k % 5]
        vr.collective(ts, mode=mode)
        torch.cuda.synchronize()
        vr.check()
        want = np.sum(parts, axis=0)
        for t in ts:
            assert np.array_equal(t.cpu().numpy(), want)
    assert vr.launches - base == 12
    vr.close()


@pytest.mark.parametrize("oneshot_bytes", ["0", "65536"])
def test_ll_oneshot_and_twoshot_variants(oneshot_bytes, monkeypatch):
    """MODE_LL's two variants (RBX_LL_ONESHOT_BYTES=0 forces two-shot; 65536
    makes every size here one-shot) against the reference replay digests."""
    torch = _torch()
    from paper_1708_02188_b200.virtual import VirtualRanks

    monkeypatch.setenv("RBX_LL_ONESHOT_BYTES", oneshot_bytes)
    g = golden("replay_digests")
    for n, dims in all_dims():
        vr = VirtualRanks(dims, nblocks_per_rank=2)
        for dtype in ("i64", "f32", "f64"):
            for it, length in enumerate(LENGTHS):
                parts = [orc.generate_input(n, it, r, length, dtype) for r in range(n)]
                out = run(vr, parts, "allreduce", "ll", None)
                assert {orc.sha256(o) for o in out} == {g[f"{dkey(dims)}:{dtype}:{it}:{length}"]}, (dims, dtype, length)
        vr.close()
    del torch


def test_launches_on_different_streams_are_serialised():
    """Launches of one communicator share its device epoch; collectives issued
    back to back on different streams must not overlap (the library orders
    them), so alternating streams without any host sync stays correct."""
    torch = _torch()
    from paper_1708_02188_b200.virtual import VirtualRanks

    dims = (2, 2, 2)
    vr = VirtualRanks(dims, nblocks_per_rank=4)
    streams = [torch.cuda.Stream() for _ in range(3)]
    rng = np.random.default_rng(8)
    cases = []
    for k in range(18):
        length = int(rng.integers(1, 40_000))
        parts = [rng.integers(-1000, 1001, length).astype(np.int64) for _ in range(8)]
        ts = [torch.from_numpy(p).cuda() for p in parts]
        cases.append((parts, ts))
    torch.cuda.synchronize()
    for k, (parts, ts) in enumerate(cases):
        st = streams[k % 3]
        st.wait_stream(torch.cuda.current_stream())
        vr.collective(ts, mode=["ll", "fused", "ring_dims"][k % 3], stream=st)
    torch.cuda.synchronize()
    vr.check()
    for parts, ts in cases:
        want = np.sum(parts, axis=0)
        for t in ts:
            assert np.array_equal(t.cpu().numpy(), want)
    vr.close()


def test_ll_limits_and_large_ragged_inputs():
    """MODE_LL (8-byte {data, epoch} words, no flags): every size up to its
    1 MiB-per-rank cap is bit-exact, and a larger buffer is refused, not truncated."""
    torch = _torch()
    from paper_1708_02188_b200.virtual import VirtualRanks

    for dims in [(2,), (2, 2, 2), (4, 2), (3,)]:
        n = int(np.prod(dims))
        grid = orc.Grid(dims)
        vr = VirtualRanks(dims, nblocks_per_rank=8)
        for length in (262_144, 262_143, 99_991):
            parts = [orc.generate_input(6, 0, r, length, "f32") for r in range(n)]
            want = orc.closed_form_allreduce(grid, parts)
            ts = [torch.from_numpy(p.copy()).cuda() for p in parts]
            vr.collective(ts, mode="ll")
            torch.cuda.synchronize()
            vr.check()
            for t in ts:
                assert np.array_equal(t.cpu().numpy(), want), (dims, length)
        for length in (131_072, 65_537):
            parts = [orc.generate_input(7, 0, r, length, "f64") for r in range(n)]
            want = orc.closed_form_allreduce(grid, parts)
            ts = [torch.from_numpy(p.copy()).cuda() for p in parts]
            vr.collective(ts, mode="ll")
            torch.cuda.synchronize()
            for t in ts:
                assert np.array_equal(t.cpu().numpy(), want), (dims, length)
        for length in (524_288, 524_287, 77_777):  # bf16: two elements per LL word, odd regions
            rng = np.random.default_rng(length)
            bits = [orc.bf16_round(rng.standard_normal(length).astype(np.float32)) for _ in range(n)]
            want = orc.bf16_allreduce(grid, bits)
            ts = [torch.from_numpy(b.view(np.int16)).cuda().view(torch.bfloat16) for b in bits]
            vr.collective(ts, mode="ll")
            torch.cuda.synchronize()
            for t in ts:
                assert np.array_equal(t.view(torch.int16).cpu().numpy().view(np.uint16), want), (dims, length)
        too_big = [torch.zeros(262_145, device="cuda") for _ in range(n)]
        with pytest.raises(ValueError):
            vr.collective(too_big, mode="ll")
        with pytest.raises(ValueError):
            vr.collective([torch.zeros(100, device="cuda") for _ in range(n)], mode="ll", window=(0, 50))
        vr.close()


@pytest.mark.parametrize("mode,length,nblocks", [
    ("local", 50_001, 4), ("fused", 50_001, 4), ("push", 50_001, 4), ("ll", 50_001, 4),
    # more work tiles than CTAs: the dynamic-tile path (claim counters rewound at exit)
    ("fused", 400_003, 2), ("ring_dims", 400_003, 2), ("push", 400_003, 2),
])
def test_cuda_graph_replay(mode, length, nblocks):
    """Epochs and dynamic-tile counters live in device memory and are advanced /
    rewound by the kernel itself, so a captured launch replays correctly (CUDA
    graphs instead of per-call launches for static buffers)."""
    torch = _torch()
    from paper_1708_02188_b200.virtual import VirtualRanks

    dims = (2, 2, 2)
    grid = orc.Grid(dims)
    parts = [orc.generate_input(4, 0, r, length, "f32") for r in range(8)]
    want = orc.closed_form_allreduce(grid, parts)
    vr = VirtualRanks(dims, nblocks_per_rank=0 if mode == "local" else nblocks)
    src = [torch.from_numpy(p.copy()).cuda() for p in parts]
    ts = [s.clone() for s in src]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        vr.collective(ts, mode=mode, stream=s)  # warm-up: builds and uploads the plan
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        vr.collective(ts, mode=mode, stream=torch.cuda.current_stream())
    for _ in range(3):
        for t, x in zip(ts, src):
            t.copy_(x)
        g.replay()
        torch.cuda.synchronize()
        vr.check()
        for t in ts:
            assert np.array_equal(t.cpu().numpy(), want)
    vr.close()


@pytest.mark.parametrize("mode", ["local", "fused", "ring_dims", "push"])
def test_windows_compose_to_the_full_allreduce(mode):
    """rbx_vcollective_window: element windows keep the full buffer's chunk
    geometry and order, so any split reproduces the full result bit-for-bit."""
    torch = _torch()
    from paper_1708_02188_b200.virtual import VirtualRanks

    for dims in [(2, 2, 2), (2, 4), (3, 2)]:
        n = int(np.prod(dims))
        grid = orc.Grid(dims)
        length = 100_003
        parts = [orc.generate_input(9, 0, r, length, "f32") for r in range(n)]
        want = orc.closed_form_allreduce(grid, parts)
        vr = VirtualRanks(dims, nblocks_per_rank=0 if mode == "local" else 4)
        ts = [torch.from_numpy(p.copy()).cuda() for p in parts]
        cuts = [0, 1, 7777, 50_000, 50_001, 99_999, length]
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            vr.collective(ts, mode=mode, window=(lo, hi))
        torch.cuda.synchronize()
        vr.check()
        for t in ts:
            assert np.array_equal(t.cpu().numpy(), want)
        vr.close()


@pytest.mark.parametrize("windows", [1, 5, 12])
@pytest.mark.parametrize("n", [1, 4099, 1_000_003])
def test_allreduce_host_pipeline_bit_exact(n, windows):
    """VirtualRanks.allreduce_host (the bench's N=1 e2e call): page-locked numpy
    buffers streamed through equal, 64 KB-aligned windows on three streams;
    every window is a full-geometry allreduce of its elements, so the result
    equals the reference order over the whole buffer."""
    _torch()
    from paper_1708_02188_b200.runtime import host_empty
    from paper_1708_02188_b200.virtual import VirtualRanks

    dims = (2, 2, 2)
    grid = orc.Grid(dims)
    parts = [orc.generate_input(0, 0, r, n, "f32") for r in range(8)]
    want = orc.closed_form_allreduce(grid, parts)
    vr = VirtualRanks(dims, device=0, nblocks_per_rank=0)
    try:
        for kind in ("numpy", "host_empty"):
            arrays = [p.copy() if kind == "numpy" else host_empty(n, "f32") for p in parts]
            if kind == "host_empty":
                for a, p in zip(arrays, parts):
                    a[...] = p
            vr.allreduce_host(arrays, mode="local", windows=windows)
            for a in arrays:
                assert np.array_equal(a, want), (kind, n, windows)
    finally:
        vr.close()
