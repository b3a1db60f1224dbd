"""Plan documents as the executor sees them.

The drop-in boundary is the reference's persisted plan (`plan.json`, written by
planio.plan_to_json, reference pkg/src/meshplan/planio.py:73-121).  The
reference's own loader `runtime_from_json` (planio.py:128-156) rebuilds a
RuntimePlan but drops `op_specs`; this loader keeps them, because they are what
each device must actually compute.

Also restated here (pure integer arithmetic, parity-tested bit-exact against the
reference in tests/test_plan_parity.py):
  * spec strings           — sharding.py:102-133 (`R`, `S^0`, `S^{01}`)
  * local dims / bytes     — sharding.py:80-92
  * LogicalMesh coordinates — mesh.py:97-114 (row-major device ids)
  * shard boxes            — reshard.py:74-85 (mixed radix, first listed axis major)
"""
from __future__ import annotations

import json
import math
import re
from dataclasses import dataclass, field
from fractions import Fraction
from pathlib import Path
from typing import Iterable, Optional, Union

Box = tuple[tuple[int, int], ...]

KIND_INPUT = "input"
KIND_PARAM = "parameter"
KIND_MATMUL = "matmul"
KIND_BMM = "batched_matmul"
KIND_ELEM = "elementwise"
KIND_RED = "reduction"
KIND_RESHAPE = "reshape"
HEAVY = (KIND_MATMUL, KIND_BMM)


class PlanError(ValueError):
    """Rejected plan document (mirrors planio.PlanIOError, planio.py:23)."""


# --------------------------------------------------------------------------- specs

@dataclass(frozen=True)
class Spec:
    """Per-dimension tuple of mesh axes ('' = replicated)."""

    dims: tuple[tuple[int, ...], ...]

    @property
    def rank(self) -> int:
        return len(self.dims)

    def axes_used(self) -> tuple[int, ...]:
        return tuple(sorted(a for d in self.dims for a in d))

    def dim_of_axis(self, axis: int) -> Optional[int]:
        for i, d in enumerate(self.dims):
            if axis in d:
                return i
        return None

    def replicated_axes(self) -> tuple[int, ...]:
        used = set(self.axes_used())
        return tuple(a for a in (0, 1) if a not in used)

    def is_replicated(self) -> bool:
        return not any(self.dims)

    def permuted(self, order: Iterable[int]) -> "Spec":
        return Spec(tuple(self.dims[i] for i in order))

    def __str__(self) -> str:
        return format_spec(self)


_TOKEN = re.compile(r"R|S\^(\d|\{\d+\})")


def parse_spec(text: str) -> Spec:
    out = []
    pos = 0
    while pos < len(text):
        m = _TOKEN.match(text, pos)
        if m is None:
            raise PlanError(f"bad sharding spec {text!r} at offset {pos}")
        if m.group(0) == "R":
            out.append(())
        else:
            out.append(tuple(int(ch) for ch in m.group(1).strip("{}")))
        pos = m.end()
    if not out:
        raise PlanError("empty sharding spec")
    return Spec(tuple(out))


def format_spec(spec: Spec) -> str:
    parts = []
    for d in spec.dims:
        if not d:
            parts.append("R")
        elif len(d) == 1:
            parts.append(f"S^{d[0]}")
        else:
            parts.append("S^{" + "".join(map(str, d)) + "}")
    return "".join(parts)


def replicated(rank: int) -> Spec:
    return Spec(((),) * rank)


# --------------------------------------------------------------------------- meshes

@dataclass(frozen=True)
class Mesh:
    """2-D logical view (n_l, m_l) of a stage's devices, row-major ids."""

    n: int
    m: int
    device_ids: tuple[int, ...]

    def extent(self, axis: int) -> int:
        return self.n if axis == 0 else self.m

    def group_extent(self, axes: Iterable[int]) -> int:
        return math.prod(self.extent(a) for a in axes)

    @property
    def size(self) -> int:
        return self.n * self.m

    def device(self, i: int, j: int) -> int:
        return self.device_ids[i * self.m + j]

    def coords(self, device: int) -> tuple[int, int]:
        k = self.device_ids.index(device)
        return divmod(k, self.m)

    def axis_group(self, device: int, axes: tuple[int, ...]) -> tuple[int, ...]:
        """Devices that differ from `device` only along `axes` (sorted ids)."""
        i, j = self.coords(device)
        ii = range(self.n) if 0 in axes else (i,)
        jj = range(self.m) if 1 in axes else (j,)
        return tuple(sorted(self.device(a, b) for a in ii for b in jj))


def local_dims(dims: tuple[int, ...], spec: Spec, mesh: Mesh) -> tuple[int, ...]:
    return tuple(ext // mesh.group_extent(ax) for ext, ax in zip(dims, spec.dims))


def check_spec(dims: tuple[int, ...], spec: Spec, mesh: Mesh) -> None:
    if spec.rank != len(dims):
        raise PlanError(f"spec {spec} has rank {spec.rank}, tensor has rank {len(dims)}")
    for ext, ax in zip(dims, spec.dims):
        if any(a not in (0, 1) for a in ax):
            raise PlanError(f"unknown mesh axis in {spec}")
        if ext % mesh.group_extent(ax):
            raise PlanError(f"extent {ext} not divisible by mesh factor in {spec}")


def shard_box(dims: tuple[int, ...], spec: Spec, mesh: Mesh, coords: tuple[int, int]) -> Box:
    """Global half-open box held at logical coords (i, j): per dim, the block
    index is the mixed-radix number of the dim's axes in listed order."""
    out = []
    for ext, axes in zip(dims, spec.dims):
        idx, blocks = 0, 1
        for a in axes:
            idx = idx * mesh.extent(a) + coords[a]
            blocks *= mesh.extent(a)
        step = ext // blocks
        out.append((idx * step, idx * step + step))
    return tuple(out)


def device_box(dims, spec: Spec, mesh: Mesh, device: int) -> Box:
    return shard_box(dims, spec, mesh, mesh.coords(device))


def box_intersect(a: Box, b: Box) -> Optional[Box]:
    out = []
    for (a0, a1), (b0, b1) in zip(a, b):
        lo, hi = max(a0, b0), min(a1, b1)
        if hi <= lo:
            return None
        out.append((lo, hi))
    return tuple(out)


def box_numel(box: Box) -> int:
    return math.prod(hi - lo for lo, hi in box)


# --------------------------------------------------------------------------- graph

@dataclass(frozen=True)
class Node:
    id: int
    kind: str
    inputs: tuple[int, ...]
    dims: tuple[int, ...]
    elem_bytes: int
    flop: int
    reduce_axis: Optional[int] = None
    colocate_with: Optional[int] = None
    grad_of: Optional[int] = None

    @property
    def is_forward(self) -> bool:
        return self.colocate_with is None

    @property
    def nbytes(self) -> int:
        return math.prod(self.dims) * self.elem_bytes


@dataclass(frozen=True)
class Graph:
    nodes: tuple[Node, ...]
    outputs: tuple[int, ...]
    # images per microbatch of a convolutional graph when the graph itself cannot
    # tell (a stage sub-graph without the pooling head; plan config "image_batch")
    image_batch: Optional[int] = None

    def __len__(self) -> int:
        return len(self.nodes)

    def __getitem__(self, i: int) -> Node:
        return self.nodes[i]

    def consumers(self) -> dict[int, list[tuple[int, int]]]:
        """producer -> [(consumer, slot)]"""
        out: dict[int, list[tuple[int, int]]] = {n.id: [] for n in self.nodes}
        for n in self.nodes:
            for slot, p in enumerate(n.inputs):
                out[p].append((n.id, slot))
        return out

    @property
    def has_backward(self) -> bool:
        return any(n.colocate_with is not None for n in self.nodes)

    def matmul_flop(self, ids: Optional[Iterable[int]] = None) -> int:
        ids = range(len(self.nodes)) if ids is None else ids
        return sum(self.nodes[i].flop for i in ids if self.nodes[i].kind in HEAVY)


def graph_from_doc(doc: dict) -> Graph:
    """Graph JSON (graph.serialize, reference graph.py:393-414)."""
    if doc.get("version") != 1:
        raise PlanError("unsupported graph version")
    nodes = []
    for pos, d in enumerate(doc["nodes"]):
        kind = d["kind"]
        red = None
        if kind.startswith("reduction:"):
            kind, red = KIND_RED, int(kind.split(":", 1)[1])
        if d["id"] != pos:
            raise PlanError("graph ids must be dense")
        nodes.append(Node(
            id=d["id"], kind=kind, inputs=tuple(int(e[0]) for e in d["inputs"]),
            dims=tuple(d["shape"]["dims"]), elem_bytes=int(d["shape"]["elem_bytes"]),
            flop=int(d["flop"]), reduce_axis=red, colocate_with=d.get("colocate_with"),
            grad_of=d.get("grad_of")))
    return Graph(tuple(nodes), tuple(doc["outputs"]))


# --------------------------------------------------------------------------- plan

def _frac(v) -> Fraction:
    if isinstance(v, (list, tuple)):
        return Fraction(int(v[0]), int(v[1]))
    return Fraction(v)


@dataclass
class StagePlan:
    index: int
    op_ids: tuple[int, ...]
    mesh: Mesh
    op_specs: dict[int, Spec]          # every non-boundary member (planio.py:77-82)
    input_specs: dict[int, Spec]       # boundary inputs by producer id
    output_specs: dict[int, Spec]      # boundary outputs by original id
    t: Fraction
    mem_stage: int
    mem_act: int
    axis_bw: tuple[Fraction, Fraction] = (Fraction(1), Fraction(1))

    def spec_of(self, node_id: int) -> Spec:
        if node_id in self.op_specs:
            return self.op_specs[node_id]
        return self.input_specs[node_id]


@dataclass
class ExecPlan:
    graph: Graph
    cluster: dict
    stages: list[StagePlan]
    num_microbatches: int
    t_star: Fraction
    config: dict = field(default_factory=dict)
    doc: Optional[dict] = None

    @property
    def num_devices(self) -> int:
        return int(self.cluster["hosts"]) * int(self.cluster["devices_per_host"])

    @property
    def has_backward(self) -> bool:
        return self.graph.has_backward

    def stage_of_device(self, device: int) -> StagePlan:
        for s in self.stages:
            if device in s.mesh.device_ids:
                return s
        raise PlanError(f"device {device} is in no stage")

    def stage_of_op(self) -> dict[int, int]:
        return {oid: s.index for s in self.stages for oid in s.op_ids}


PLAN_KIND = "meshplan.plan"


def load_plan(src: Union[str, Path, dict]) -> ExecPlan:
    doc = src if isinstance(src, dict) else json.loads(Path(src).read_text())
    if doc.get("kind") != PLAN_KIND or doc.get("version") != 1:
        raise PlanError("not a meshplan plan document")
    graph = graph_from_doc(doc["graph"])
    if doc.get("config", {}).get("image_batch"):
        graph = Graph(graph.nodes, graph.outputs, int(doc["config"]["image_batch"]))
    stages = []
    for sd in doc["stages"]:
        mesh = Mesh(int(sd["logical_view"][0]), int(sd["logical_view"][1]),
                    tuple(int(d) for d in sd["device_ids"]))
        st = StagePlan(
            index=int(sd["index"]), op_ids=tuple(sd["op_ids"]), mesh=mesh,
            op_specs={int(k): parse_spec(v) for k, v in sd["op_specs"].items()},
            input_specs={int(k): parse_spec(v) for k, v in sd["boundary_inputs"].items()},
            output_specs={int(k): parse_spec(v) for k, v in sd["boundary_outputs"].items()},
            t=_frac(sd["t"]), mem_stage=int(sd["mem_stage"]), mem_act=int(sd["mem_act"]),
            axis_bw=(_frac(sd["axis_bw"][0]), _frac(sd["axis_bw"][1])))
        for oid, spec in st.op_specs.items():
            check_spec(graph[oid].dims, spec, mesh)
        stages.append(st)
    stages.sort(key=lambda s: s.index)
    seen: set[int] = set()
    for s in stages:
        ids = set(s.mesh.device_ids)
        if ids & seen:
            raise PlanError(f"stage {s.index} reuses devices of an earlier stage")
        seen |= ids
    n_dev = int(doc["cluster"]["hosts"]) * int(doc["cluster"]["devices_per_host"])
    if seen != set(range(n_dev)):
        raise PlanError("plan stages do not cover the cluster devices exactly")
    return ExecPlan(graph, dict(doc["cluster"]), stages, int(doc["num_microbatches"]),
                    _frac(doc["t_star"]), dict(doc.get("config", {})), doc)
