"""Cross-mesh resharding index plans (the paper's §7 / Fig. 8 orchestration).

Restates the reference's two-pass construction so the executor can derive the
exact Transfer / GatherOp lists on a box where the reference is not installed:

  * pass 1 (tile correspondence, reshard.py:97-108): for a destination piece,
    one transfer per distinct overlap with a source tile, sent by the lowest
    device id holding it, ordered by box;
  * pass 2 (reshard.py:111-157): destination devices needing the same tile form
    a replica group; the tile is cut along dim 0 at floor(span*r/g) so each
    member receives one slab over the inter-mesh link, then a local all-gather
    over the group (GatherOp) completes it.  optimize=False keeps pass 1 only.

Stage boundaries (reshard.py:276-328) aggregate per (producer, consumer) stage
pair; the executor keeps the per-tensor plans because it must move real data.
All outputs are compared bit-exactly with the reference (tests/test_plan_parity.py).
"""
from __future__ import annotations

from dataclasses import dataclass

from .plan import (Box, ExecPlan, Mesh, PlanError, Spec, box_intersect, box_numel,
                   check_spec, shard_box)


@dataclass(frozen=True)
class Transfer:
    src_device: int
    dst_device: int
    nbytes: int
    box: Box


@dataclass(frozen=True)
class Gather:
    devices: tuple[int, ...]
    axes: tuple[int, ...]
    nbytes: int
    box: Box                      # the tile the group completes
    pieces: tuple[Box, ...]       # per member (devices order): its slab (may be empty)


@dataclass(frozen=True)
class XPlan:
    transfers: tuple[Transfer, ...]
    gathers: tuple[Gather, ...]

    @property
    def inter_mesh_bytes(self) -> int:
        return sum(t.nbytes for t in self.transfers)


def _tiles(dims, spec: Spec, mesh: Mesh) -> list[tuple[int, Box]]:
    return [(mesh.device(i, j), shard_box(dims, spec, mesh, (i, j)))
            for i in range(mesh.n) for j in range(mesh.m)]


def _sources(piece: Box, src_tiles: list[tuple[int, Box]], dst: int,
             elem_bytes: int) -> list[Transfer]:
    owner: dict[Box, int] = {}
    for dev, tile in src_tiles:
        ov = box_intersect(piece, tile)
        if ov is not None and (ov not in owner or dev < owner[ov]):
            owner[ov] = dev
    return [Transfer(owner[b], dst, box_numel(b) * elem_bytes, b) for b in sorted(owner)]


def cross_mesh_plan(dims: tuple[int, ...], elem_bytes: int, src_spec: Spec, src_mesh: Mesh,
                    dst_spec: Spec, dst_mesh: Mesh, optimize: bool = True) -> XPlan:
    check_spec(dims, src_spec, src_mesh)
    check_spec(dims, dst_spec, dst_mesh)
    if set(src_mesh.device_ids) & set(dst_mesh.device_ids):
        raise PlanError("source and destination meshes share devices")
    src_tiles = _tiles(dims, src_spec, src_mesh)
    dst_tiles = _tiles(dims, dst_spec, dst_mesh)
    if not optimize:
        out: list[Transfer] = []
        for dev, tile in dst_tiles:
            out += _sources(tile, src_tiles, dev, elem_bytes)
        return XPlan(tuple(out), ())
    groups: dict[Box, list[int]] = {}
    for dev, tile in dst_tiles:
        groups.setdefault(tile, []).append(dev)
    rep_axes = dst_spec.replicated_axes()
    transfers: list[Transfer] = []
    gathers: list[Gather] = []
    for tile in sorted(groups):
        members = sorted(groups[tile])
        if len(members) == 1:
            transfers += _sources(tile, src_tiles, members[0], elem_bytes)
            continue
        g = len(members)
        (lo, hi), rest = tile[0], tile[1:]
        span = hi - lo
        pieces = []
        for r, dev in enumerate(members):
            a, b = lo + span * r // g, lo + span * (r + 1) // g
            piece = ((a, b),) + rest
            pieces.append(piece)
            if a < b:
                transfers += _sources(piece, src_tiles, dev, elem_bytes)
        gathers.append(Gather(tuple(members), rep_axes, box_numel(tile) * elem_bytes, tile,
                              tuple(pieces)))
    return XPlan(tuple(transfers), tuple(gathers))


@dataclass(frozen=True)
class BoundaryTensor:
    node: int                      # original producer id
    src_spec: Spec
    dst_spec: Spec
    xplan: XPlan


@dataclass(frozen=True)
class Boundary:
    producer: int
    consumer: int
    tensors: tuple[BoundaryTensor, ...]
    recv_bytes: int                # per-device bytes landing on the consumer

    @property
    def phase(self) -> str:
        return "fwd" if self.producer < self.consumer else "bwd"

    @property
    def tag_prefix(self) -> str:
        return "f" if self.phase == "fwd" else "b"

    @property
    def transfers(self) -> tuple[Transfer, ...]:
        return tuple(t for bt in self.tensors for t in bt.xplan.transfers)

    @property
    def gathers(self) -> tuple[Gather, ...]:
        return tuple(g for bt in self.tensors for g in bt.xplan.gathers)

    @property
    def inter_mesh_bytes(self) -> int:
        return sum(t.nbytes for t in self.transfers)


def stage_boundaries(plan: ExecPlan, optimize: bool = True) -> list[Boundary]:
    where = plan.stage_of_op()
    out = []
    for st in plan.stages:
        by_src: dict[int, list[int]] = {}
        for nid in sorted(st.input_specs):
            p = where.get(nid)
            if p is None or p == st.index:
                continue
            by_src.setdefault(p, []).append(nid)
        for p in sorted(by_src):
            src = plan.stages[p]
            tensors = []
            recv = 0
            for nid in by_src[p]:
                node = plan.graph[nid]
                sspec, dspec = src.output_specs[nid], st.input_specs[nid]
                xp = cross_mesh_plan(node.dims, node.elem_bytes, sspec, src.mesh, dspec,
                                     st.mesh, optimize)
                tensors.append(BoundaryTensor(nid, sspec, dspec, xp))
                recv += node.nbytes // st.mesh.group_extent(dspec.axes_used())
            out.append(Boundary(p, st.index, tuple(tensors), recv))
    return out


def sends_of(bd: Boundary, device: int) -> list[tuple[int, Transfer]]:
    """(tensor index, transfer) pairs `device` sends for boundary `bd`, in the
    order every rank derives (tensor order, then transfer order)."""
    return [(k, t) for k, bt in enumerate(bd.tensors) for t in bt.xplan.transfers
            if t.src_device == device]


def recvs_of(bd: Boundary, device: int) -> list[tuple[int, Transfer]]:
    return [(k, t) for k, bt in enumerate(bd.tensors) for t in bt.xplan.transfers
            if t.dst_device == device]
