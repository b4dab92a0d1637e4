"""bench.py's output contract on CPU: the reference arm (`--impl reference`,
the reference runtime's phase loop ported to C, no GPU) prints ONE JSON line
with the keys the driver reads, for N=1 and for a multi-GPU launch shape;
plus the pure helpers the GPU arm uses (busbw, workload names, defaults)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config"}


def _run(*argv):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *argv], capture_output=True, text=True,
                         timeout=300, cwd=ROOT, env={**os.environ, "RANK": "0"})
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("gpus", [1, 8])
def test_reference_arm_line(gpus):
    d = _run("--impl", "reference", "--gpus", str(gpus), "--steps", "2", "--warmup", "1", "--elems", "40000")
    assert KEYS <= set(d)
    assert d["impl"] == "reference" and d["n_gpus"] == gpus and d["steps"] == 2 and d["warmup"] == 1
    assert d["metric"] == json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
    assert d["unit"] == "GB/s" and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["config"]["workload"].startswith("config2: 40000 f32/rank, 8 ranks")
    assert d["config"]["dims"] == [2, 2, 2]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["value"] == d["value"] and cb["cores"] >= 1 and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_busbw_and_workload_names():
    assert bench.busbw(2, 100, 1.0) == pytest.approx(100 / 1e9)
    assert bench.busbw(8, 8_000_000, 1e-3) == pytest.approx(2 * 7 / 8 * 8e6 / 1e-3 / 1e9)
    assert bench.workload_name(25_600_000, "f32", 8, (2, 2, 2)).startswith("config2: 25600000 f32/rank, 8 ranks")
    assert bench.DIMS_FOR == {1: (2, 2, 2), 2: (2,), 4: (2, 2), 8: (2, 2, 2)}


def test_default_arguments(monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = bench.parse_args()
    assert (a.gpus, a.steps, a.warmup, a.impl, a.elems, a.e2e_chunks) == (1, 20, 5, "ours", bench.N_ELEM, 12)
    assert a.warmup >= 3  # timing rules: W >= 3
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4"])
    assert bench.parse_args().e2e_chunks is None  # N>1: the runtime's default windows


def test_gpus_n_without_torchrun_self_launches(monkeypatch):
    """`python bench.py --gpus N` (no WORLD_SIZE) spawns N ranks through
    torch.distributed.run with the same arguments -- it never silently runs the
    1-GPU path for N > 1."""
    cmd = bench.self_launch_command(["--gpus", "4", "--steps", "3"], 4, 29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-4:] == [os.path.join(ROOT, "bench.py"), "--gpus", "4", "--steps", "3"][-4:]
    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2", "--steps", "3"])
    monkeypatch.setattr(bench.subprocess, "call", lambda c, env=None: calls.append(c) or 0)
    monkeypatch.setattr(bench, "main_single", lambda a: (_ for _ in ()).throw(AssertionError("N=1 path ran")))
    with pytest.raises(SystemExit) as ex:
        bench.main()
    assert ex.value.code == 0
    assert len(calls) == 1 and "--nproc-per-node=2" in calls[0] and calls[0][-4:] == ["--gpus", "2", "--steps", "3"]
