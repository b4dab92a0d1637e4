"""Pin the oracle restatements (numpy + C) against the reference's own outputs.

The golden fixtures were produced by importing the reference `ringbox`
package (tests/golden/make_golden.py).  These tests run on CPU (no GPU).
"""

import numpy as np
import pytest

from conftest import golden
from oracle import oracle_c
from oracle import ringbox_oracle as orc

RANK_COUNTS = (1, 2, 3, 4, 6, 8, 12, 16)
LENGTHS = (0, 1, 17, 1000, 4099)
EXTRA_DIMS = {4: [(1, 4)], 6: [(2, 1, 3)], 16: [(2, 2, 2, 2)]}


def dkey(dims):
    return "x".join(map(str, dims))


def all_cases():
    for n in RANK_COUNTS:
        for dims in orc.factorizations(n, 3) + EXTRA_DIMS.get(n, []):
            yield n, tuple(dims)


def test_chunk_bounds_kats():
    for count, n, i, off, ln in golden("chunk_kats"):
        assert orc.chunk_bounds(count, n, i) == (off, ln)
        assert oracle_c.chunk_bounds(count, n, i) == (off, ln)


def test_generate_input_pinned():
    g = golden("input_digests")
    for dtype in ("i64", "f32", "f64"):
        for it, length in enumerate(LENGTHS):
            for r in range(8):
                assert orc.sha256(orc.generate_input(8, it, r, length, dtype)) == g[f"{dtype}:8:{it}:{r}"]


def test_owned_regions():
    g = golden("owned_regions")
    for key, regions in g.items():
        dims_s, count = key.split(":")
        grid = orc.Grid(tuple(int(x) for x in dims_s.split("x")))
        assert [list(orc.owned_region(grid, r, int(count))) for r in range(grid.size)] == regions


def _dump(phases):
    lines = []
    for i, ph in enumerate(phases):
        for (src, dst, c, off, ln, add) in ph:
            lines.append(f"{i} {src} {dst} {c} {off} {ln} {'add' if add else 'replace'}")
    return "\n".join(lines) + ("\n" if lines else "")


def test_schedule_dumps():
    g = golden("schedules")
    for key, text in g.items():
        if key.startswith("rs_"):
            continue
        dims_s, count = key.split(":")
        dims = tuple(int(x) for x in dims_s.split("x"))
        assert _dump(orc.multiring_schedule(orc.Grid(dims), int(count))) == text


@pytest.mark.parametrize("impl", ["numpy_replay", "closed_form", "c_replay"])
def test_replay_digests_all_decompositions(impl):
    """Reference acceptance sweep (pkg/tests/test_acceptance.py:41-73): every
    factorization of N in {1..16} x lengths x {i64,f32,f64} must reproduce the
    reference replay digest bit-for-bit."""
    g = golden("replay_digests")
    checked = 0
    for n, dims in all_cases():
        grid = orc.Grid(dims)
        for dtype in ("i64", "f32", "f64"):
            for it, length in enumerate(LENGTHS):
                parts = [orc.generate_input(n, it, r, length, dtype) for r in range(n)]
                if impl == "numpy_replay":
                    res = orc.replay(orc.multiring_schedule(grid, length), parts)
                    assert len({orc.sha256(x) for x in res}) == 1
                    out = res[0]
                elif impl == "closed_form":
                    out = orc.closed_form_allreduce(grid, parts)
                else:
                    out = oracle_c.replay(dims, parts, dtype)[0]
                assert orc.sha256(out) == g[f"{dkey(dims)}:{dtype}:{it}:{length}"], (dims, dtype, length)
                checked += 1
    assert checked == 450


def test_runtime_digests_match_replay_and_port():
    """The reference RUNTIME digests (forked TCP workers) equal the oracle, and
    the C runtime port (one thread per rank) reproduces them too."""
    g = golden("runtime_digests")
    for key, dig in g.items():
        if key.endswith("bytes_sent"):
            continue
        dims_s, dtype, it, length = key.split(":")
        dims = tuple(int(x) for x in dims_s.split("x"))
        n = int(np.prod(dims))
        parts = [orc.generate_input(n, int(it), r, int(length), dtype) for r in range(n)]
        assert orc.sha256(orc.closed_form_allreduce(orc.Grid(dims), parts)) == dig
        bufs = [p.copy() for p in parts]
        oracle_c.runtime_port(dims, bufs, dtype)
        assert {orc.sha256(b) for b in bufs} == {dig}


def test_small_vectors():
    for case in golden("small_vectors"):
        dt = orc.DTYPES[case["dtype"]]
        parts = [np.frombuffer(bytes.fromhex(h), dtype=dt).copy() for h in case["inputs_hex"]]
        out = orc.closed_form_allreduce(orc.Grid(tuple(case["dims"])), parts)
        assert out.tobytes().hex() == case["result_hex"]


def test_large_config_digests_c_oracle():
    """Configs 1/2 at full size (25.6 M fp32 x 8 ranks) -- C oracle vs reference digest."""
    g = golden("large_digests")
    length = 25_600_000
    parts = [orc.generate_input(0, 0, r, length, "f32") for r in range(8)]
    assert [orc.sha256(p) for p in parts] == g[f"inputs:f32:seed0:{length}"]
    for dims in [(2, 4), (2, 2, 2)]:
        out = orc.closed_form_allreduce(orc.Grid(dims), parts)
        assert orc.sha256(out) == g[f"{dkey(dims)}:f32:seed0:{length}"]


def test_fold_order_22x2_is_balanced_tree():
    # (2,2,2) == ((x0+x1)+(x2+x3))+((x4+x5)+(x6+x7)) for every element
    grid = orc.Grid((2, 2, 2))
    rng = np.random.default_rng(0)
    xs = [rng.standard_normal(4096).astype(np.float32) * 10.0 ** rng.integers(-3, 4) for _ in range(8)]
    want = ((xs[0] + xs[1]) + (xs[2] + xs[3])) + ((xs[4] + xs[5]) + (xs[6] + xs[7]))
    assert np.array_equal(orc.closed_form_allreduce(grid, xs), want)


def test_bf16_round_rne():
    x = np.array([1.0, 1.00390625, 1.005859375, -2.5, 3.0e38, np.inf], dtype=np.float32)
    bits = orc.bf16_round(x)
    back = orc.bf16_to_f32(bits)
    assert back[0] == 1.0 and back[1] == 1.0  # tie -> even
    assert back[2] == np.float32(1.0078125)
    assert back[3] == -2.5 and np.isinf(back[5])
