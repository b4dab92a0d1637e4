"""Host-side logic of round 2 on CPU: the host-buffer pipeline's window count,
the crash fraction of fault injection (the reference's crash_phase, runtime.py:
429-432), and the bench's per-GPU value definition in the reference arm."""

import numpy as np
import pytest

from paper_1708_02188_b200.hoststage import default_windows, window_bounds
from paper_1708_02188_b200.multiring import Grid
from paper_1708_02188_b200.runtime import _crash_fraction, multiring_schedule


def test_default_windows():
    assert default_windows(0) == 1
    assert default_windows(4096) == 1  # small buffers: one window (one launch, LL if eligible)
    assert default_windows(3 << 20) == 3
    assert default_windows(102_400_000) == 16  # the bench's 102.4 MB: capped
    assert default_windows(8 * 102_400_000, cap=8) == 8


class _Ctx:
    def __init__(self, dims):
        self.grid = Grid(dims)

    def schedule_for(self, n):
        return multiring_schedule(self.grid, n)


@pytest.mark.parametrize("dims,phases", [((4,), 6), ((2, 2), 4), ((2, 2, 2), 6), ((2, 4), 8)])
def test_crash_fraction_follows_the_reference_phase_count(dims, phases):
    ctx = _Ctx(dims)
    assert len(ctx.schedule_for(100).phases) == phases  # 2 * sum(d - 1), multiring.py:170-211
    assert _crash_fraction(ctx, 100, 1) == pytest.approx(1 / phases)
    assert _crash_fraction(ctx, 100, 0) == 0.0
    assert _crash_fraction(ctx, 100, None) == 0.0
    assert _crash_fraction(ctx, 100, 10 * phases) == 1.0  # past the end: the whole collective
    assert _crash_fraction(ctx, 0, 3) == 0.0  # empty buffer: nothing to move


def test_host_dtype_table_covers_the_reference_dtypes():
    from paper_1708_02188_b200.runtime import _NP_DTYPES

    for dt in ("f32", "f64", "i64"):  # runtime.py:37
        assert dt in _NP_DTYPES.values()
    assert _NP_DTYPES[np.dtype(np.float32)] == "f32"


@pytest.mark.parametrize("n,w", [(1, 8), (7, 3), (1000, 5), (102_400_000, 16), (25_600_000, 8), (13, 13)])
def test_window_bounds_tile_the_buffer(n, w):
    b = window_bounds(n, w)
    assert b[0][0] == 0 and b[-1][1] == n
    assert all(x[1] == y[0] for x, y in zip(b, b[1:]))
    assert all(hi > lo for lo, hi in b)
    if w >= 6 and n >= 1000:  # tapered ends: the unoverlapped first / last copies are the smallest
        sizes = [hi - lo for lo, hi in b]
        assert sizes[0] < sizes[1] < sizes[2] and sizes[-1] < sizes[-2] < sizes[-3]


@pytest.mark.parametrize("nbuf,lanes", [(1, 1), (1, 2), (1, 4), (8, 1), (8, 2), (8, 4), (3, 4), (2, 3)])
def test_pipeline_lanes_cover_every_window_once(nbuf, lanes):
    import torch

    from paper_1708_02188_b200.hoststage import HostPipeline

    pipe = HostPipeline.__new__(HostPipeline)  # no CUDA streams needed for the split
    pipe.lanes = lanes
    n = 1001
    hosts = [torch.zeros(n, dtype=torch.int32) for _ in range(nbuf)]
    devs = [torch.zeros(n, dtype=torch.int32) for _ in range(nbuf)]
    for lo, hi in window_bounds(n, 7, taper=False):
        pieces = pipe._pieces(hosts, devs, lo, hi)
        assert {lane for lane, _, _ in pieces} == set(range(min(lanes, len(pieces))))
        for _, h, d in pieces:
            h += 1
            d += 1
    for t in hosts + devs:
        assert torch.equal(t, torch.ones(n, dtype=torch.int32))  # every element in exactly one piece


@pytest.mark.parametrize("n,w,align", [(25_600_000, 12, 16384), (25_600_000, 16, 16384), (102_400_000, 16, 16384),
                                       (1_000_003, 5, 16384), (1000, 8, 16384), (5, 3, 4)])
def test_window_bounds_aligned_edges(n, w, align):
    """hoststage.HostPipeline rounds inner window edges to 64 KB (16384 fp32 elements):
    copies that start off such a boundary ran slower (profiles/r02_e2e_probe_align_1gpu.jsonl)."""
    b = window_bounds(n, w, taper=False, align=align)
    assert b[0][0] == 0 and b[-1][1] == n
    assert all(x[1] == y[0] for x, y in zip(b, b[1:]))
    assert all(hi > lo for lo, hi in b)
    assert all(lo % align == 0 for lo, _ in b)  # every window starts on the grid; only the last may end off it
    if n >= w * align:
        assert len(b) == w
        sizes = [hi - lo for lo, hi in b]
        assert max(sizes) - min(sizes) <= align + 1  # equal windows up to the rounding
