"""Per-op layout contract inside a stage mesh.

For every op the executor needs (a) the spec each input must be in before the
local kernel runs and (b) the collective that finishes the op.  Both follow the
reference's strategy semantics:

  * matmul / bmm roots: the ParallelAlgorithm is recovered from the chosen
    output spec.  Every mesh axis of extent > 1 is used exactly once
    (sharding.py:264-273), so the axes not used by the output go to the
    contraction loop k; input specs follow the loop table _MATMUL_LOOPS
    (sharding.py:215-219) and a mapped k costs an all_reduce of partial sums
    (sharding.py:284-291).  Checked against enumerate_algorithms for every
    algorithm on every view of <= 8 devices (tests/test_plan_parity.py).
  * trivial members take their group's propagated spec and their operands are
    resharded to it (_required_spec, intra.py:241-248).
  * reshape members: transposes require the permuted spec; head split / merge
    are layout barriers evaluated on the replicated tensor (intra.py:149-160).

`relayout_moves` is the literal data movement between two specs on one mesh.
`resharding_cost` (sharding.py:322-350) is a cost model, not a recipe (it is
not literally executable on 2-D views with S^{01} dims, SURVEY §7 hard part 4),
so moves are derived from shard-box intersections, the same construction
cross_mesh_plan uses (reshard.py:97-108), restricted to one mesh.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

from .binding import Bound
from .plan import Box, Mesh, PlanError, Spec, box_intersect, device_box, replicated


@dataclass(frozen=True)
class MatmulAlgo:
    out_spec: Spec
    in_specs: tuple[Spec, Spec]
    k_axes: tuple[int, ...]          # all_reduce group axes (empty: no comm)


def _canon(axes, mesh: Mesh) -> tuple[int, ...]:
    return tuple(sorted(a for a in axes if mesh.extent(a) > 1))


def canonical(spec: Spec, mesh: Mesh) -> Spec:
    return Spec(tuple(_canon(d, mesh) for d in spec.dims))


def matmul_algo(kind_bmm: bool, out_spec: Spec, mesh: Mesh) -> MatmulAlgo:
    o = canonical(out_spec, mesh)
    used = set(o.axes_used())
    k = tuple(a for a in (0, 1) if mesh.extent(a) > 1 and a not in used)
    if kind_bmm:
        b, i, j = o.dims
        lhs, rhs = Spec((b, i, k)), Spec((b, k, j))
    else:
        i, j = o.dims
        lhs, rhs = Spec((i, k)), Spec((k, j))
    return MatmulAlgo(o, (lhs, rhs), k)


def reshape_required(bound: Bound, out_spec: Spec, in_rank: int) -> Spec:
    op = bound.op
    if op == "identity":
        return out_spec
    if op == "transpose":
        d = out_spec.dims
        return Spec(d[:-2] + (d[-1], d[-2]))
    # head split / merge (and their inverses): barrier through the replicated tensor
    return replicated(in_rank)


# --------------------------------------------------------------------------- relayout

@dataclass(frozen=True)
class Move:
    src: int
    dst: int
    box: Box            # global coordinates


def relayout_moves(dims: tuple[int, ...], src: Spec, dst: Spec, mesh: Mesh) -> list[Move]:
    """Every (src device -> dst device, global box) copy that materialises `dst`
    from `src` on one mesh.  A needed piece is taken from the device itself when
    it holds it, else from the lowest id holding it; a device's needed tile is
    covered exactly once.  Deterministic, so every rank derives the same list."""
    holders = [(d, device_box(dims, src, mesh, d)) for d in sorted(mesh.device_ids)]
    moves: list[Move] = []
    for d in sorted(mesh.device_ids):
        need = device_box(dims, dst, mesh, d)
        # source tiles partition the tensor (up to replication), so the distinct
        # overlaps partition `need`; pick the lowest holder, then prefer self.
        covered: dict[Box, int] = {}
        for e, tile in holders:
            ov = box_intersect(need, tile)
            if ov is not None and ov not in covered:
                covered[ov] = e
        mine = box_intersect(need, device_box(dims, src, mesh, d))
        if mine is not None:
            covered[mine] = d
        for box in sorted(covered):
            moves.append(Move(covered[box], d, box))
    return moves


def _contains(outer: Box, inner: Box) -> bool:
    return all(o0 <= i0 and i1 <= o1 for (o0, o1), (i0, i1) in zip(outer, inner))


def is_local_slice(dims, src: Spec, dst: Spec, mesh: Mesh, device: int) -> bool:
    return _contains(device_box(dims, src, mesh, device), device_box(dims, dst, mesh, device))


def all_local(dims, src: Spec, dst: Spec, mesh: Mesh) -> bool:
    return all(is_local_slice(dims, src, dst, mesh, d) for d in mesh.device_ids)


def allgather_axes(dims, have: Spec, req: Spec, mesh: Mesh, dim: int = 0) -> Optional[tuple[int, ...]]:
    """Mesh axes A such that, on every device, the `req` tile is the concatenation
    along `dim` (in device-id order, i.e. NCCL group rank order) of the `have`
    tiles of its A-axis group — then one all-gather realises the relayout (e.g.
    S^1R -> RR along dim 0 straight into the output; RS^1 -> RR along dim 1
    through a staging buffer and one permuting copy); None otherwise."""
    found = None
    for d in mesh.device_ids:
        need = device_box(dims, req, mesh, d)
        members = [e for e in sorted(mesh.device_ids)
                   if _contains(need, device_box(dims, have, mesh, e))]
        boxes = [device_box(dims, have, mesh, e) for e in members]
        if len(members) < 2 or any(b[:dim] + b[dim + 1:] != need[:dim] + need[dim + 1:]
                                   for b in boxes):
            return None
        cut = need[dim][0]
        step = (need[dim][1] - need[dim][0]) // len(members)
        for b in boxes:
            if b[dim] != (cut, cut + step):
                return None
            cut += step
        if cut != need[dim][1] or any(device_box(dims, req, mesh, e) != need for e in members):
            return None
        axes = next((ax for ax in ((0,), (1,), (0, 1)) if mesh.group_extent(ax) > 1
                     and mesh.axis_group(d, ax) == tuple(members)), None)
        if axes is None or (found is not None and axes != found):
            return None
        found = axes
    return found
