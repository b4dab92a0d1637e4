"""CPU tests of librbx.so: the library loads, exports the ABI, and its host-side
plan builder reproduces the reference schedule's chunking and reduction order
(checked against the oracle and the reference golden digests).  No GPU calls."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden
from oracle import ringbox_oracle as orc
from paper_1708_02188_b200 import _native
from plan_sim import simulate

RANK_COUNTS = (1, 2, 3, 4, 6, 8, 12, 16)


def all_dims():
    for n in RANK_COUNTS:
        for dims in orc.factorizations(n, 3):
            yield n, tuple(dims)
    yield 4, (1, 4)
    yield 6, (2, 1, 3)
    yield 16, (2, 2, 2, 2)


def test_library_exports_every_header_symbol():
    lib = _native.lib()
    header = open(os.path.join(ROOT, "include", "rbx.h")).read()
    declared = set(re.findall(r"\b(rbx_[a-z_]+)\s*\(", header))
    assert declared == set(_native.EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.rbx_version() == 1


def test_device_count_without_gpu_is_an_error_not_a_crash():
    n = ctypes.c_int(-1)
    rc = _native.lib().rbx_device_count(ctypes.byref(n))
    assert rc in (0, _native.ERR_CUDA)


def test_chunk_bounds_kats_native():
    for count, n, i, off, ln in golden("chunk_kats"):
        assert _native.chunk_bounds(count, n, i) == (off, ln)
    with pytest.raises(ValueError):
        _native.chunk_bounds(8, 4, 4)
    with pytest.raises(ValueError):
        _native.chunk_bounds(8, 0, 0)


def test_owned_regions_native():
    for key, regions in golden("owned_regions").items():
        dims_s, count = key.split(":")
        dims = tuple(int(x) for x in dims_s.split("x"))
        n = int(np.prod(dims))
        assert [list(_native.owned_region(dims, r, int(count))) for r in range(n)] == regions


def test_fold_order_native_matches_oracle():
    for n, dims in all_dims():
        grid = orc.Grid(dims)
        for r in range(n):
            assert _native.fold_order(dims, r) == orc.fold_order(grid, r)


def test_plan_rejects_bad_geometry():
    with pytest.raises(ValueError):
        _native.plan_describe((3, 7), 0, 10)  # 21 ranks > 16
    with pytest.raises(ValueError):
        _native.plan_describe((0,), 0, 10)


@pytest.mark.parametrize("mode", ["fused", "fused_pull", "ring_dims", "push"])
def test_plan_tables_reproduce_reference_allreduce(mode):
    """Simulate every rank's step table (3 CTAs/rank, random interleavings) and
    compare with the reference replay digests for all decompositions."""
    g = golden("replay_digests")
    lengths = (0, 1, 17, 1000, 4099)
    for n, dims in all_dims():
        for it, length in enumerate(lengths):
            if length > 1000 and n > 8:
                continue
            parts = [orc.generate_input(n, it, r, length, "f32") for r in range(n)]
            out = simulate(dims, parts, "allreduce", mode, nb=3, seed=it)
            want = g[f"{'x'.join(map(str, dims))}:f32:{it}:{length}"]
            assert {orc.sha256(b) for b in out} == {want}, (mode, dims, length)


@pytest.mark.parametrize("mode", ["fused", "ring_dims", "push"])
def test_plan_tables_reduce_scatter_and_allgather(mode):
    for n, dims in [(2, (2,)), (4, (2, 2)), (6, (3, 2)), (8, (2, 2, 2)), (8, (2, 4)), (8, (8,))]:
        grid = orc.Grid(dims)
        length = 1001
        parts = [orc.generate_input(7, 0, r, length, "f32") for r in range(n)]
        want = orc.closed_form_allreduce(grid, parts)
        rs = simulate(dims, parts, "reduce_scatter", mode, nb=2, seed=1)
        for r in range(n):
            off, ln = orc.owned_region(grid, r, length)
            assert np.array_equal(rs[r][off:off + ln], want[off:off + ln])
        # allgather from owned chunks only (other regions garbage)
        staged = []
        for r in range(n):
            b = np.full(length, np.nan, dtype=np.float32)
            off, ln = orc.owned_region(grid, r, length)
            b[off:off + ln] = want[off:off + ln]
            staged.append(b)
        ag = simulate(dims, staged, "allgather", mode, nb=2, seed=2)
        for r in range(n):
            assert np.array_equal(ag[r], want)


def test_local_plan_covers_every_element_once():
    for n, dims in all_dims():
        plan = _native.parse_plan(_native.plan_describe(dims, 0, 4099, "allreduce", "local"))
        if n == 1:
            assert plan["steps"] == []
            continue
        (step,) = plan["steps"]
        assert step["waits"] == [] and step["sigs"] == []
        covered = sorted((s["off"], s["len"]) for s in step["segs"])
        pos = 0
        for off, ln in covered:
            assert off == pos
            pos += ln
        assert pos == 4099


def test_vector_split_alignment():
    # exact ResNet-50 size: owned offsets not 16-byte aligned
    for r in range(8):
        plan = _native.parse_plan(_native.plan_describe((2, 4), r, 25_557_032, "allreduce", "fused"))
        sg = plan["steps"][0]["segs"][0]
        assert (sg["off"] + sg["head"]) % 4 == 0
        assert sg["head"] + sg["nvec"] * 4 + sg["tail"] == sg["len"]
        assert 0 <= sg["head"] < 4 and 0 <= sg["tail"] < 4
