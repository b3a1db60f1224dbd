"""Communicators for one rank: NCCL over NVLink/NVSwitch through torch.distributed
(plumbing only; payloads are packed/unpacked by libmpexec kernels).

Groups are derived from the plan and created identically on every rank (the
torch.distributed rule for new_group):
  * per stage, per axis set {0}, {1}, {0,1}: the devices that differ from a
    device only along those axes (LogicalMesh.coord_device, mesh.py:111-114) —
    the k-group of an all_reduce (sharding.py:284-291) and the softmax row group;
  * per stage: all its devices (generic intra-mesh relayout P2P);
  * per cross-mesh boundary (reshard.py:276-328): the union of both stages'
    devices — one communicator per direction, so forward activations and
    backward gradients between the same stage pair never serialise on one
    NCCL stream (a 1F1B deadlock otherwise);
  * per GatherOp replica group (reshard.py:155-156): the local all-gather.
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist

from .plan import ExecPlan, Mesh
from .schedule import Program


class Comm:
    def __init__(self, plan: ExecPlan, program: Program, rank: int, world: int):
        self.rank = rank
        self.world = world
        self.enabled = world > 1
        self._groups: dict[tuple, object] = {}
        if not self.enabled:
            return
        if not dist.is_initialized():
            raise RuntimeError("multi-device plan needs torch.distributed initialised")
        keys: list[tuple] = []
        for st in plan.stages:
            m = st.mesh
            if m.size > 1:
                keys.append(("stage", st.index, tuple(sorted(m.device_ids))))
                for axes in ((0,), (1,), (0, 1)):
                    if m.group_extent(axes) <= 1:
                        continue
                    seen = set()
                    for d in m.device_ids:
                        grp = m.axis_group(d, axes)
                        if grp not in seen:
                            seen.add(grp)
                            keys.append(("axis", st.index, axes, grp))
        for bd in program.boundaries:
            ranks = tuple(sorted(set(plan.stages[bd.producer].mesh.device_ids)
                                 | set(plan.stages[bd.consumer].mesh.device_ids)))
            keys.append(("boundary", bd.producer, bd.consumer, ranks))
            for bt in bd.tensors:
                for g in bt.xplan.gathers:
                    keys.append(("gather", bd.producer, bd.consumer, g.devices))
        for k in keys:
            if k in self._groups:
                continue
            ranks = list(k[-1])
            # always a fresh communicator (never WORLD): directions must not share a stream
            self._groups[k] = dist.new_group(ranks=ranks)
        # a private world group for step-level reductions (loss, barrier)
        self.world_group = dist.new_group(ranks=list(range(world)))

    def stage_group(self, st_index: int, mesh: Mesh):
        return self._groups[("stage", st_index, tuple(sorted(mesh.device_ids)))]

    def axis_group(self, st_index: int, mesh: Mesh, axes: tuple[int, ...], device: int):
        return self._groups[("axis", st_index, axes, mesh.axis_group(device, axes))]

    def boundary_group(self, bd, plan: ExecPlan):
        ranks = tuple(sorted(set(plan.stages[bd.producer].mesh.device_ids)
                             | set(plan.stages[bd.consumer].mesh.device_ids)))
        return self._groups[("boundary", bd.producer, bd.consumer, ranks)]

    def gather_group(self, bd, devices: tuple[int, ...]):
        return self._groups[("gather", bd.producer, bd.consumer, devices)]

    # ------------------------------------------------------------------ ops
    def all_reduce(self, t: torch.Tensor, group, op=dist.ReduceOp.SUM) -> None:
        dist.all_reduce(t, op=op, group=group)

    def p2p(self, sends: list[tuple[torch.Tensor, int]], recvs: list[tuple[torch.Tensor, int]],
            group) -> list:
        ops = [dist.P2POp(dist.isend, t, peer, group=group) for t, peer in sends]
        ops += [dist.P2POp(dist.irecv, t, peer, group=group) for t, peer in recvs]
        if not ops:
            return []
        return dist.batch_isend_irecv(ops)

    def all_gather_into(self, out_flat: torch.Tensor, in_flat: torch.Tensor, group) -> None:
        dist.all_gather_into_tensor(out_flat, in_flat, group=group)
