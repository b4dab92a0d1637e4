import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
for _p in (ROOT, TESTS):
    if _p not in sys.path:
        sys.path.insert(0, _p)
GOLDEN = os.path.join(ROOT, "tests", "golden")
TOPOLOGIES = os.path.join(ROOT, "paper_1708_02188_b200", "topologies")

_cache = {}


def golden(name):
    if name not in _cache:
        with open(os.path.join(GOLDEN, name + ".json"), encoding="utf-8") as fh:
            _cache[name] = json.load(fh)["data"]
    return _cache[name]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs in one box")


def cuda_count():
    try:
        import torch

        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


@pytest.fixture
def one_gpu():
    if cuda_count() < 1:
        pytest.skip("no CUDA device")


def need_gpus(n):
    return pytest.mark.skipif(cuda_count() < n, reason=f"needs {n} GPUs")


def rank_device(rank: int) -> int:
    """GPU of a rank process: one rank per GPU when the box has enough, else the
    ranks share the GPUs round-robin (time-sliced contexts: every rank keeps its
    own communicator, IPC mappings and flags, exactly as on a bigger box)."""
    import torch

    return rank % torch.cuda.device_count()


def host_backend(world: int) -> str:
    """torch.distributed backend for rank processes: NCCL refuses two ranks on
    one GPU, so a box with fewer GPUs than ranks uses gloo for the host side."""
    import torch

    return "nccl" if world <= torch.cuda.device_count() else "gloo"
