"""Host planner (topology -> grid decomposition) vs the reference's outputs.

Golden values come from the reference itself (tests/golden/planner.json,
schedules.json); the rest mirrors pkg/tests/test_topology.py,
test_costmodel.py, test_multiring.py and test_ring.py."""

import itertools
import json
import os

import numpy as np
import pytest

from conftest import ROOT, golden
from paper_1708_02188_b200 import costmodel
from paper_1708_02188_b200.multiring import (
    Grid,
    Plan,
    build_grid,
    evaluate_decomposition,
    factorizations,
    multiring_schedule,
    plan,
    ring_partner_pairs,
)
from paper_1708_02188_b200.ring import (
    RingOrder,
    allgather_schedule,
    allreduce_schedule,
    chunk_bounds,
    dump_schedule,
    order_ranks_on_tree,
    reduce_scatter_schedule,
)
from paper_1708_02188_b200.topology import (
    TopologyError,
    b200_box,
    build_tree,
    load_topology,
    override_latency,
    parse_topology,
)

TOPO_DIR = os.path.join(ROOT, "paper_1708_02188_b200", "topologies")


def load(name):
    """Reference sample topologies are parsed from their golden serialization
    (tests/golden/planner.json, produced from pkg/sample_topologies); the B200
    box description ships with the package."""
    if name.startswith("b200"):
        return load_topology(os.path.join(TOPO_DIR, name))
    return parse_topology(golden("planner")[f"{name}:serialize"])


def doc_with(nodes, levels=None):
    levels = levels or [{"id": "l0", "bandwidth_gbps": 10.0, "latency_s": 0.0}]
    return json.dumps({"levels": levels, "nodes": nodes})


class TestTopology:
    def test_sample_topologies_roundtrip_reference_serialization(self):
        g = golden("planner")
        for name in ("host4.json", "two_switch_4dev.json", "cluster_4x16x4.json"):
            assert load(name).serialize() == g[f"{name}:serialize"]

    def test_cluster_shape(self):
        t = load("cluster_4x16x4.json")
        assert len(t.devices()) == 256
        assert [lv.bandwidth_gbps for lv in t.levels] == [20.0, 10.0, 9.5]

    @pytest.mark.parametrize("nodes,match", [
        ([{"id": "h", "kind": "host"}, {"id": "d", "kind": "device", "parent": "h", "link_level": "l0"},
          {"id": "d", "kind": "device", "parent": "h", "link_level": "l0"}], "duplicate node id 'd'"),
        ([{"id": "h", "kind": "host", "color": "blue"}], "unknown keys"),
        ([{"id": "d", "kind": "device", "parent": "nope", "link_level": "l0"}], "unknown parent"),
        ([{"id": "s", "kind": "switch"}, {"id": "d", "kind": "device", "parent": "s", "link_level": "l0"}],
         "not a host"),
        ([{"id": "a", "kind": "switch", "parent": "b", "link_level": "l0"},
          {"id": "b", "kind": "switch", "parent": "a", "link_level": "l0"}, {"id": "r", "kind": "host"}], "cycle"),
        ([{"id": "a", "kind": "host"}, {"id": "b", "kind": "host"}], "exactly one root"),
    ])
    def test_validation_errors(self, nodes, match):
        with pytest.raises(TopologyError, match=match):
            parse_topology(doc_with(nodes))

    def test_bad_json_and_bandwidth(self):
        with pytest.raises(TopologyError, match="invalid JSON"):
            parse_topology("{not json")
        with pytest.raises(TopologyError, match="bandwidth must be > 0"):
            parse_topology(doc_with([{"id": "h", "kind": "host"}],
                                    [{"id": "l0", "bandwidth_gbps": 0, "latency_s": 0.0}]))

    def test_routing(self):
        t = load("cluster_4x16x4.json")
        hops = t.route("host0.gpu0", "host63.gpu3")
        assert len(hops) == 6
        fwd = t.route("host0.gpu1", "host17.gpu2")
        rev = t.route("host17.gpu2", "host0.gpu1")
        assert [h.direction for h in fwd] == [(d, s) for s, d in reversed([h.direction for h in rev])]
        with pytest.raises(TopologyError, match="must differ"):
            t.route("host0.gpu0", "host0.gpu0")
        with pytest.raises(TopologyError, match="unknown node"):
            t.route("host0.gpu0", "ghost")
        assert t.min_bandwidth(["host0.gpu0", "host16.gpu0", "host32.gpu0", "host48.gpu0"]) == 9.5

    def test_override_latency(self):
        t = override_latency(load("host4.json"), 0.123)
        assert all(lv.latency_s == 0.123 for lv in t.levels)

    def test_b200_box_file_matches_builder(self):
        t = load("b200_nvswitch_8.json")
        assert t.devices() == [f"gpu{i}" for i in range(8)]
        assert t.serialize() == b200_box(8).serialize()
        assert all(h.link.bandwidth_gbps == 900.0 for h in t.route("gpu0", "gpu7"))


class TestCostModel:
    def test_reference_values(self):
        cm = golden("planner")["costmodel"]
        assert costmodel.allreduce_time(0.35, 256, 9.5, 0.0005).total == pytest.approx(cm["allreduce_time"], rel=1e-15)
        assert costmodel.multiring_time(0.35, [(4, 20.0), (16, 10.0), (4, 9.5)], 0.0005).total == pytest.approx(
            cm["multiring_time"], rel=1e-15)
        assert costmodel.multiring_time(0.1024, [(2, 900.0)] * 3).total == pytest.approx(
            cm["multiring_b200_2x2x2"], rel=1e-15)
        assert costmodel.parameter_server_time(0.35, 256, 10.0).seconds == pytest.approx(
            cm["parameter_server"], rel=1e-15)

    def test_acceptance_numbers(self):
        # pkg/tests/test_acceptance.py criteria 2, 3, 6
        assert abs(costmodel.allreduce_time(0.35, 256, 9.5, 0.0005).total - 0.329) < 1e-3
        assert abs(costmodel.multiring_time(0.35, [(4, 20.0), (16, 10.0), (4, 9.5)], 0.0005).total - 0.065) < 1e-3
        est = costmodel.parameter_server_time(0.35, 256, 10.0)
        assert 8.9 <= est.seconds <= 9.0 and abs(est.gathered_gb - 89.6) < 0.05

    def test_errors(self):
        with pytest.raises(ValueError):
            costmodel.multiring_time(-1.0, [(2, 1.0)])
        with pytest.raises(ValueError):
            costmodel.multiring_time(1.0, [])
        with pytest.raises(ValueError):
            costmodel.ring_reduction_time(1.0, 0, 1.0)


class TestGridAndSchedules:
    def test_factorizations(self):
        g = golden("planner")["factorizations"]
        for n, facs in g.items():
            assert [list(f) for f in factorizations(int(n), 3)] == facs

    @pytest.mark.parametrize("n", [2, 6, 12, 16, 36, 60])
    @pytest.mark.parametrize("max_dims", [1, 2, 3, 4])
    def test_factorizations_brute_force(self, n, max_dims):
        divs = [d for d in range(2, n + 1) if n % d == 0]
        want = {(n,)}
        for k in range(1, max_dims + 1):
            for tup in itertools.product(divs, repeat=k):
                if int(np.prod(tup)) == n:
                    want.add(tup)
        assert factorizations(n, max_dims) == sorted(want)

    def test_grid(self):
        g = build_grid(4, (2, 2))
        assert [g.coords(r) for r in range(4)] == [(0, 0), (1, 0), (0, 1), (1, 1)]
        for dims in [(2, 3, 4), (6,), (1, 2, 1, 3)]:
            gg = Grid(dims)
            assert {gg.rank_of(gg.coords(r)) for r in range(gg.size)} == set(range(gg.size))
        with pytest.raises(ValueError, match="product"):
            build_grid(5, (2, 2))

    def test_schedule_dumps_match_reference(self):
        for key, text in golden("schedules").items():
            if key == "rs_ring2:10":
                assert dump_schedule(reduce_scatter_schedule(RingOrder(("a", "b")), 10)) == text
                continue
            dims_s, count = key.split(":")
            dims = tuple(int(x) for x in dims_s.split("x"))
            assert dump_schedule(multiring_schedule(Grid(dims), int(count))) == text

    def test_phase_law_and_flat(self):
        for dims in [(2, 2), (4,), (2, 2, 2), (3, 4), (1, 4), (2, 1, 3)]:
            g = Grid(dims)
            assert len(multiring_schedule(g, 4 * g.size).phases) == 2 * sum(d - 1 for d in dims)
        flat = allreduce_schedule(RingOrder(tuple("abcde")), 20)
        assert multiring_schedule(Grid((5,)), 20).phases == flat.phases
        assert allgather_schedule(RingOrder(("x",)), 4).phases == ()

    def test_partner_pairs(self):
        g = golden("planner")["partner_pairs"]
        for key, pairs in g.items():
            dims = tuple(int(x) for x in key.split("x"))
            assert sorted(list(p) for p in ring_partner_pairs(Grid(dims))) == pairs

    def test_chunk_bounds(self):
        for count, n, i, off, ln in golden("chunk_kats"):
            assert chunk_bounds(count, n, i) == (off, ln)
        with pytest.raises(ValueError):
            chunk_bounds(8, 4, 4)


class TestPlanner:
    def _cmp(self, got: Plan, want: dict):
        doc = json.loads(got.to_json())
        assert doc["dims"] == want["dims"] or [
            {k: v for k, v in d.items() if k != "seconds"} for d in doc["dims"]
        ] == [{k: v for k, v in d.items() if k != "seconds"} for d in want["dims"]]
        for d, w in zip(doc["dims"], want["dims"]):
            assert d["seconds"] == pytest.approx(w["seconds"], rel=1e-12)
        assert doc["element_count"] == want["element_count"]
        assert doc["devices"] == want["devices"]
        assert doc["total_s"] == pytest.approx(want["total_s"], rel=1e-12)

    def test_sample_topology_plans_match_reference(self):
        g = golden("planner")
        for name in ("host4.json", "two_switch_4dev.json", "cluster_4x16x4.json"):
            t = load(name)
            devs = t.devices()
            self._cmp(plan(t, devs, 0.35), g[f"{name}:None:0.35"])
            if len(devs) >= 8:
                self._cmp(plan(t, devs[:8], 0.1024), g[f"{name}:first8:0.1024"])
                self._cmp(plan(t, devs[:8], 0.1024, dims=(2, 4)), g[f"{name}:first8:2x4:0.1024"])

    def test_b200_star_choices(self):
        g = golden("planner")
        for lat in (0.0, 5e-06, 0.0005):
            t = build_tree(8, bandwidths_gbps=(900.0,), latencies_s=(lat,))
            self._cmp(plan(t, t.devices(), 0.1024), g[f"b200star:{lat}"])
        # L=0 -> (2,4) (all tie); L>0 -> (2,2,2)
        t0 = b200_box(8, latency_s=0.0)
        assert plan(t0, t0.devices(), 0.1024).grid.dims == (2, 4)
        t5 = b200_box(8, latency_s=5e-6)
        assert plan(t5, t5.devices(), 0.1024).grid.dims == (2, 2, 2)

    def test_two_hosts_and_cluster(self):
        g = golden("planner")
        t = build_tree(4, 2, 1, (20.0, 10.0), (0.0005, 0.0005))
        self._cmp(plan(t, t.devices(), 0.1024), g["2hostx4"])
        self._cmp(plan(t, t.devices(), 0.1024, dims=(2, 4)), g["2hostx4:2x4"])
        t = build_tree(4, 16, 4, (20.0, 10.0, 9.5), (0.0005, 0.0005, 0.0005))
        self._cmp(plan(t, t.devices(), 0.35), g["cluster:auto:0.35"])

    def test_plan_json_roundtrip(self):
        t = build_tree(4, bandwidths_gbps=(20.0,), latencies_s=(0.0005,))
        p = plan(t, t.devices(), 0.001, latency_s=0.0005)
        again = Plan.from_json(p.to_json())
        assert again.grid.dims == p.grid.dims and again.schedule == p.schedule
        assert again.estimate.total == pytest.approx(p.estimate.total, rel=1e-12)

    def test_errors_and_dfs_order(self):
        t = build_tree(2, 2, 1, (10.0, 10.0), (0.001, 0.001))
        with pytest.raises(ValueError, match="must not be empty"):
            plan(t, [], 0.1)
        assert list(order_ranks_on_tree(t, ["host1.gpu1", "host0.gpu0"]).devices) == ["host0.gpu0", "host1.gpu1"]
        with pytest.raises(ValueError, match="not a device leaf"):
            order_ranks_on_tree(t, ["host0"])
        decomp, _ = evaluate_decomposition(build_tree(2, 2, 1, (20.0, 10.0), (0.0, 0.001)),
                                           order_ranks_on_tree(t, t.devices()), (2, 2), 0.01)
        assert [d.bandwidth_gbps for d in decomp.dims] == [20.0, 10.0]
