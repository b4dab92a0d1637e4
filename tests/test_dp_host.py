"""Host side of MultiringDataParallel (paper_1708_02188_b200/dp.py): the
bucket assignment reproduces DDP's 25 MiB bucketing of ResNet-50/101
(the config-4/5 bucket lists)."""

import pytest

from paper_1708_02188_b200.dp import ddp_bucket_assignment


def test_bucket_assignment_rules():
    mb = 1 << 20
    # first bucket closes at 1 MiB, later ones at the cap; a bucket closes once it reaches its cap
    assert ddp_bucket_assignment([mb // 2, mb // 2, mb, 3 * mb], mb, 2 * mb) == [[0, 1], [2, 3]]
    assert ddp_bucket_assignment([], mb, 2 * mb) == []
    assert ddp_bucket_assignment([10], mb, 2 * mb) == [[0]]


@pytest.mark.parametrize("name,want", [
    ("resnet50", [2_049_000, 7_875_584, 6_563_840, 6_637_568, 2_431_040]),
    ("resnet101", [2_049_000, 7_875_584, 6_563_840, 6_965_760, 6_703_104, 6_703_104, 6_590_464, 1_098_304]),
])
def test_resnet_buckets_match_ddp(name, want):
    torchvision = pytest.importorskip("torchvision")
    m = getattr(torchvision.models, name)(num_classes=1000)
    order = list(reversed(list(m.parameters())))
    got = [sum(order[i].numel() for i in b) for b in ddp_bucket_assignment([p.numel() * 4 for p in order])]
    assert got == want


def test_bucket_tracker_launch_order():
    """Any readiness order: every bucket launches once, in index order, never
    before all its parameters are ready; finish() releases the rest."""
    import random

    from paper_1708_02188_b200.dp import BucketTracker

    rng = random.Random(0)
    for _ in range(200):
        sizes = [rng.randint(1, 5) for _ in range(rng.randint(1, 8))]
        tr = BucketTracker(sizes)
        tr.start()
        events = [k for k, n in enumerate(sizes) for _ in range(n)]
        rng.shuffle(events)
        skip = rng.random() < 0.3  # some parameters get no gradient this pass
        if skip:
            events = events[: rng.randint(0, len(events))]
        seen = [0] * len(sizes)
        launched = []
        for k in events:
            seen[k] += 1
            for b in tr.ready(k):
                assert seen[b] == sizes[b], "launched before all its gradients were ready"
                launched.append(b)
        launched += tr.finish()
        assert launched == list(range(len(sizes)))
        assert not tr.active


def test_bucket_tracker_rejects_double_gradients():
    from paper_1708_02188_b200.dp import BucketTracker

    tr = BucketTracker([1, 1])
    tr.start()
    assert tr.ready(1) == []
    with pytest.raises(RuntimeError):
        tr.ready(1)
