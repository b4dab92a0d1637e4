"""Topology description: the reference's JSON grammar, validated the same way.

Grammar and semantics follow pkg/src/ringbox/topology.py (parse_topology
192-288, Topology 65-179, build_tree 304-353): a rooted tree of `switch`,
`host` and `device` nodes; every non-root node has one uplink whose `level`
fixes its bandwidth (GB/s = 1e9 B/s per direction) and per-phase latency.
Devices are leaves whose parent is a host.

B200 addition: `b200_box(n)` / `topologies/b200_nvswitch_8.json` describe an
HGX B200 box in the same grammar -- the NVSwitch fabric is modelled as the host
node, every GPU hangs off it at NVLink-5 bandwidth (900 GB/s per direction),
so every pair of GPUs is one uniform, non-blocking hop.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

NODE_KINDS = ("device", "host", "switch")
B200_NVLINK_GBPS = 900.0


class TopologyError(ValueError):
    """Malformed or semantically invalid topology (carries a location string)."""

    def __init__(self, message: str, location: str | None = None):
        self.location = location
        super().__init__(message if location is None else f"{location}: {message}")


@dataclass(frozen=True)
class Level:
    id: str
    bandwidth_gbps: float
    latency_s: float


@dataclass(frozen=True)
class Node:
    id: str
    kind: str
    parent: str | None
    host_id: str | None = None


@dataclass(frozen=True)
class Link:
    """Uplink of `child` to `parent`."""

    child: str
    parent: str
    bandwidth_gbps: float
    level: str
    latency_s: float


@dataclass(frozen=True)
class Hop:
    src: str
    dst: str
    link: Link

    @property
    def direction(self) -> tuple[str, str]:
        return (self.src, self.dst)


class Topology:
    """Validated, immutable network tree."""

    def __init__(self, levels: list[Level], nodes: list[Node]):
        self.levels = tuple(levels)
        self._levels = {lv.id: lv for lv in self.levels}
        self.nodes = {nd.id: nd for nd in nodes}
        self._kids: dict[str, list[str]] = {nd.id: [] for nd in nodes}
        self._up: dict[str, Link] = {}
        roots = [nd.id for nd in nodes if nd.parent is None]
        for nd in nodes:
            if nd.parent is not None:
                self._kids[nd.parent].append(nd.id)
        if len(roots) != 1:
            raise TopologyError(f"expected exactly one root node, found {roots}")
        self.root = roots[0]

    # -- structure -------------------------------------------------------
    def level(self, level_id: str) -> Level:
        return self._levels[level_id]

    def uplink(self, node_id: str) -> Link | None:
        return self._up.get(node_id)

    def children(self, node_id: str) -> list[str]:
        return self._kids[node_id]

    def is_leaf(self, node_id: str) -> bool:
        return len(self._kids[node_id]) == 0

    def dfs_leaves(self) -> list[str]:
        """Leaves in depth-first (document) order."""
        out: list[str] = []
        stack = [self.root]
        while stack:
            nid = stack.pop()
            kids = self._kids[nid]
            if not kids:
                out.append(nid)
            else:
                stack.extend(kids[::-1])
        return out

    def devices(self) -> list[str]:
        return [n for n in self.dfs_leaves() if self.nodes[n].kind == "device"]

    def ancestry(self, node_id: str) -> list[str]:
        """node, parent, grandparent, ..., root (raises on cycles)."""
        chain = [node_id]
        seen = {node_id}
        parent = self.nodes[node_id].parent
        while parent is not None:
            if parent in seen:
                raise TopologyError(f"cycle through node '{chain[-1]}'")
            chain.append(parent)
            seen.add(parent)
            parent = self.nodes[parent].parent
        return chain

    def route(self, a: str, b: str) -> list[Hop]:
        """Directed link traversals on the unique tree path between two leaves."""
        for nid in (a, b):
            if nid not in self.nodes:
                raise TopologyError(f"unknown node '{nid}'")
            if not self.is_leaf(nid):
                raise TopologyError(f"route endpoints must be leaves, got '{nid}'")
        if a == b:
            raise TopologyError(f"route endpoints must differ, got '{a}' twice")
        up_a, up_b = self.ancestry(a), self.ancestry(b)
        on_b = set(up_b)
        meet = next(n for n in up_a if n in on_b)
        hops = [Hop(n, self._up[n].parent, self._up[n]) for n in up_a[: up_a.index(meet)]]
        down = up_b[: up_b.index(meet)]
        hops += [Hop(self._up[n].parent, n, self._up[n]) for n in reversed(down)]
        return hops

    def min_bandwidth(self, ring_order: list[str]) -> float:
        members = list(ring_order)
        if len(set(members)) < 2:
            raise TopologyError("ring needs at least 2 distinct devices")
        worst = float("inf")
        for i, a in enumerate(members):
            b = members[(i + 1) % len(members)]
            if a != b:
                worst = min([worst] + [h.link.bandwidth_gbps for h in self.route(a, b)])
        return worst

    def serialize(self) -> str:
        nodes = []
        for nd in self.nodes.values():
            entry: dict = {"id": nd.id, "kind": nd.kind}
            if nd.parent is not None:
                entry["parent"] = nd.parent
                entry["link_level"] = self._up[nd.id].level
            nodes.append(entry)
        levels = [{"id": lv.id, "bandwidth_gbps": lv.bandwidth_gbps, "latency_s": lv.latency_s} for lv in self.levels]
        return json.dumps({"levels": levels, "nodes": nodes}, indent=2, sort_keys=False)


class _Validator:
    """Turns a decoded JSON document into a Topology, or raises TopologyError."""

    def __init__(self, doc):
        if not isinstance(doc, dict):
            raise TopologyError("top level must be an object")
        self.doc = doc
        self.check_keys(doc, {"levels", "nodes"}, set(), "top level")

    @staticmethod
    def check_keys(obj: dict, required: set, optional: set, where: str) -> None:
        missing = sorted(required - set(obj))
        if missing:
            raise TopologyError(f"missing keys {missing}", where)
        extra = sorted(set(obj) - required - optional)
        if extra:
            raise TopologyError(f"unknown keys {extra}", where)

    def levels(self) -> list[Level]:
        out, seen = [], set()
        for i, raw in enumerate(self.doc["levels"]):
            where = f"levels[{i}]"
            if not isinstance(raw, dict):
                raise TopologyError("level must be an object", where)
            self.check_keys(raw, {"id", "bandwidth_gbps", "latency_s"}, set(), where)
            if raw["id"] in seen:
                raise TopologyError(f"duplicate level id '{raw['id']}'", where)
            seen.add(raw["id"])
            bw, lat = raw["bandwidth_gbps"], raw["latency_s"]
            if isinstance(bw, bool) or not isinstance(bw, (int, float)) or bw <= 0:
                raise TopologyError(f"bandwidth must be > 0, got {bw!r}", where)
            if isinstance(lat, bool) or not isinstance(lat, (int, float)) or lat < 0:
                raise TopologyError(f"latency must be >= 0, got {lat!r}", where)
            out.append(Level(raw["id"], float(bw), float(lat)))
        return out

    def build(self) -> Topology:
        levels = self.levels()
        by_level = {lv.id: lv for lv in levels}
        raws = []
        seen = set()
        for i, raw in enumerate(self.doc["nodes"]):
            where = f"nodes[{i}]"
            if not isinstance(raw, dict):
                raise TopologyError("node must be an object", where)
            self.check_keys(raw, {"id", "kind"}, {"parent", "link_level"}, where)
            nid = raw["id"]
            if not isinstance(nid, str) or not nid:
                raise TopologyError(f"node id must be a non-empty string, got {nid!r}", where)
            if nid in seen:
                raise TopologyError(f"duplicate node id '{nid}'", where)
            seen.add(nid)
            if raw["kind"] not in NODE_KINDS:
                raise TopologyError(f"kind must be one of {NODE_KINDS}, got {raw['kind']!r}", where)
            if ("parent" in raw) != ("link_level" in raw):
                raise TopologyError("'parent' and 'link_level' must appear together", where)
            raws.append((raw, where))
        kinds = {raw["id"]: raw["kind"] for raw, _ in raws}
        nodes = []
        for raw, where in raws:
            parent = raw.get("parent")
            host = None
            if parent is not None:
                if parent not in kinds:
                    raise TopologyError(f"unknown parent '{parent}'", where)
                if parent == raw["id"]:
                    raise TopologyError("node cannot be its own parent", where)
                if raw.get("link_level") not in by_level:
                    raise TopologyError(f"unknown level '{raw.get('link_level')}'", where)
            if raw["kind"] == "device":
                if parent is None:
                    raise TopologyError("device must have a host parent", where)
                if kinds[parent] != "host":
                    raise TopologyError(f"device parent '{parent}' is a {kinds[parent]}, not a host", where)
                host = parent
            nodes.append(Node(raw["id"], raw["kind"], parent, host))
        topo = Topology(levels, nodes)
        for raw, _ in raws:
            if raw.get("parent") is not None:
                lv = by_level[raw["link_level"]]
                topo._up[raw["id"]] = Link(raw["id"], raw["parent"], lv.bandwidth_gbps, lv.id, lv.latency_s)
        for nid in topo.nodes:
            topo.ancestry(nid)  # cycles / broken chains
        for raw, where in raws:
            if raw["kind"] == "device" and not topo.is_leaf(raw["id"]):
                raise TopologyError("device must be a leaf", where)
        return topo


def parse_topology(document: str) -> Topology:
    try:
        doc = json.loads(document)
    except json.JSONDecodeError as exc:
        raise TopologyError(f"invalid JSON: {exc}") from exc
    return _Validator(doc).build()


def load_topology(path: str) -> Topology:
    with open(path, encoding="utf-8") as fh:
        return parse_topology(fh.read())


def override_latency(t: Topology, latency_s: float) -> Topology:
    doc = json.loads(t.serialize())
    for lv in doc["levels"]:
        lv["latency_s"] = latency_s
    return parse_topology(json.dumps(doc))


def build_tree(
    devices_per_host: int,
    hosts_per_rack: int = 1,
    racks: int = 1,
    bandwidths_gbps: tuple = (20.0,),
    latencies_s: tuple = (0.0,),
) -> Topology:
    """Regular device/host[/rack[/director]] tree; levels innermost first."""
    has_rack = hosts_per_rack > 1 or racks > 1
    has_director = racks > 1
    tiers = 1 + int(has_rack) + int(has_director)
    if len(bandwidths_gbps) != tiers or len(latencies_s) != tiers:
        raise TopologyError(f"need {tiers} bandwidth/latency values for this geometry")
    names = ("intra-host", "intra-rack", "inter-rack")[:tiers]
    levels = [{"id": nm, "bandwidth_gbps": bw, "latency_s": lat} for nm, bw, lat in zip(names, bandwidths_gbps, latencies_s)]
    nodes: list[dict] = []
    if has_director:
        nodes.append({"id": "director", "kind": "switch"})
    for r in range(racks):
        tor = f"tor{r}"
        if has_director:
            nodes.append({"id": tor, "kind": "switch", "parent": "director", "link_level": "inter-rack"})
        elif has_rack:
            nodes.append({"id": tor, "kind": "switch"})
        for h in range(hosts_per_rack):
            host = f"host{r * hosts_per_rack + h}"
            hnode: dict = {"id": host, "kind": "host"}
            if has_rack:
                hnode.update(parent=tor, link_level="intra-rack")
            nodes.append(hnode)
            for d in range(devices_per_host):
                nodes.append({"id": f"{host}.gpu{d}", "kind": "device", "parent": host, "link_level": "intra-host"})
    return parse_topology(json.dumps({"levels": levels, "nodes": nodes}))


def b200_box(n_gpus: int = 8, latency_s: float = 0.0, bandwidth_gbps: float = B200_NVLINK_GBPS) -> Topology:
    """One HGX B200 box: all GPUs one NVSwitch hop apart at NVLink-5 bandwidth."""
    doc = {
        "levels": [{"id": "nvlink5", "bandwidth_gbps": bandwidth_gbps, "latency_s": latency_s}],
        "nodes": [{"id": "nvswitch", "kind": "host"}]
        + [{"id": f"gpu{i}", "kind": "device", "parent": "nvswitch", "link_level": "nvlink5"} for i in range(n_gpus)],
    }
    return parse_topology(json.dumps(doc))
