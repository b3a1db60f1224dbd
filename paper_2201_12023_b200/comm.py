"""Communicators for one rank: NCCL communicators owned by libmpexec (mp_comm_*)
and driven on the caller's CUDA stream — no torch.distributed call on the hot
path (torch's process groups only bootstrap the unique ids and run step-level
barriers / scalar reductions).

Groups are derived from the plan and created identically on every rank:
  * per stage, per axis set {0}, {1}, {0,1}: the devices that differ from a
    device only along those axes (LogicalMesh.coord_device, mesh.py:111-114) —
    the k-group of an all_reduce (sharding.py:284-291) and the softmax row group;
  * per stage: all its devices (generic intra-mesh relayout P2P);
  * per cross-mesh boundary (reshard.py:276-328): the union of both stages'
    devices — one communicator per direction; the sender drives it on its send
    stream and the receiver on its compute stream, so forward activations and
    backward gradients between a stage pair never queue behind each other
    (with one stream, 1F1B deadlocks: stage i's blocked send of f_{b+1}
    precedes its recv of b_b);
  * per GatherOp replica group (reshard.py:155-156): the local all-gather.
Group ranks are ordered by global device id (= NCCL rank order).
"""
from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from . import native
from .plan import ExecPlan, Mesh
from .schedule import Program


@dataclass
class Group:
    key: tuple
    ranks: tuple[int, ...]
    comm: int = 0
    local: dict = field(default_factory=dict)

    def peer(self, global_rank: int) -> int:
        return self.local[global_rank]


PREFETCH = os.environ.get("MPEXEC_PREFETCH_RELAYOUT", "0") == "1"


class Comm:
    def __init__(self, plan: ExecPlan, program: Program, rank: int, world: int):
        self.rank = rank
        self.world = world
        self.enabled = world > 1
        self._groups: dict[tuple, Group] = {}
        if not self.enabled:
            return
        if not dist.is_initialized():
            raise RuntimeError("multi-device plan needs torch.distributed initialised")
        keys: list[tuple] = []
        for st in plan.stages:
            m = st.mesh
            if m.size > 1:
                # "pf": the same groups again for relayouts prefetched on the side
                # stream (NCCL must not see two streams driving one communicator)
                for tag in ("", "pf-") if PREFETCH else ("",):
                    keys.append((tag + "stage", st.index, tuple(sorted(m.device_ids))))
                    for axes in ((0,), (1,), (0, 1)):
                        if m.group_extent(axes) <= 1:
                            continue
                        seen = set()
                        for d in m.device_ids:
                            grp = m.axis_group(d, axes)
                            if grp not in seen:
                                seen.add(grp)
                                keys.append((tag + "axis", st.index, axes, grp))
        for bd in program.boundaries:
            ranks = tuple(sorted(set(plan.stages[bd.producer].mesh.device_ids)
                                 | set(plan.stages[bd.consumer].mesh.device_ids)))
            keys.append(("boundary", bd.producer, bd.consumer, ranks))
            for bt in bd.tensors:
                for g in bt.xplan.gathers:
                    keys.append(("gather", bd.producer, bd.consumer, g.devices))
        uniq = []
        for k in keys:
            if k not in self._groups:
                self._groups[k] = Group(k, tuple(k[-1]), 0,
                                        {r: i for i, r in enumerate(k[-1])})
                uniq.append(k)
        # one round of unique-id exchange: each group's lowest rank makes its id
        mine = {k: native.nccl_unique_id() for k in uniq if self._groups[k].ranks[0] == rank}
        allids: list = [None] * world
        dist.all_gather_object(allids, mine)
        ids = {}
        for part in allids:
            ids.update(part)
        # same global order on every rank -> no init deadlock
        for k in uniq:
            g = self._groups[k]
            if rank in g.local:
                g.comm = native.comm_init(ids[k], len(g.ranks), g.local[rank])
        self._connect(uniq)
        # torch group for step-level reductions (loss, barrier, max time)
        self.world_group = dist.new_group(ranks=list(range(world)))

    def _connect(self, keys) -> None:
        """Establish every P2P connection up front: one all-pairs exchange of
        one element per communicator, in the same global order on every rank.
        NCCL connects peers lazily, and the lazy handshake blocks the host in
        ncclGroupEnd until the peer posts its side; connected up front, a send
        that never comes is a device-side wait the watchdog can see (and the
        first timed step pays no connection setup)."""
        buf = torch.zeros(2 * self.world, dtype=torch.float32, device="cuda")
        for k in keys:
            g = self._groups[k]
            if self.rank not in g.local or len(g.ranks) < 2:
                continue
            me = g.local[self.rank]
            peers = [i for i in range(len(g.ranks)) if i != me]
            native.send_recv(g.comm, [(buf[i:i + 1], i) for i in peers],
                             [(buf[self.world + i:self.world + i + 1], i) for i in peers])
        torch.cuda.synchronize()

    def stage_group(self, st_index: int, mesh: Mesh, pf: bool = False) -> Group:
        return self._groups[("pf-stage" if pf else "stage", st_index,
                             tuple(sorted(mesh.device_ids)))]

    def axis_group(self, st_index: int, mesh: Mesh, axes: tuple[int, ...], device: int,
                   pf: bool = False) -> Group:
        return self._groups[("pf-axis" if pf else "axis", st_index, axes,
                             mesh.axis_group(device, axes))]

    def boundary_group(self, bd, plan: ExecPlan) -> Group:
        ranks = tuple(sorted(set(plan.stages[bd.producer].mesh.device_ids)
                             | set(plan.stages[bd.consumer].mesh.device_ids)))
        return self._groups[("boundary", bd.producer, bd.consumer, ranks)]

    def gather_group(self, bd, devices: tuple[int, ...]) -> Group:
        return self._groups[("gather", bd.producer, bd.consumer, devices)]

    # ------------------------------------------------------------------ ops
    # All ops are enqueued on the current CUDA stream (or `stream`).
    def all_reduce(self, t: torch.Tensor, group: Group, op=dist.ReduceOp.SUM, stream=None) -> None:
        native.allreduce(group.comm, t, 1 if op == dist.ReduceOp.MAX else 0, stream)

    def p2p(self, sends, recvs, group: Group, stream=None) -> list:
        """sends / recvs: [(tensor, global peer rank)] in one NCCL group."""
        if not sends and not recvs:
            return []
        native.send_recv(group.comm, [(t, group.peer(p)) for t, p in sends],
                         [(t, group.peer(p)) for t, p in recvs], stream)
        return []

    def all_to_all(self, out_flat: torch.Tensor, in_flat: torch.Tensor, group: Group,
                   stream=None) -> None:
        native.alltoall(group.comm, out_flat, in_flat, len(group.ranks), stream)

    def all_gather_into(self, out_flat: torch.Tensor, in_flat: torch.Tensor, group: Group,
                        stream=None) -> None:
        native.allgather(group.comm, out_flat, in_flat, stream)

    def reduce_scatter_into(self, out_flat: torch.Tensor, in_flat: torch.Tensor, group: Group,
                            stream=None) -> None:
        native.reduce_scatter(group.comm, out_flat, in_flat, stream)

    def async_errors(self) -> list[str]:
        """Groups whose communicator reports an asynchronous NCCL failure."""
        bad = []
        for k, g in self._groups.items():
            if g.comm:
                r = native.comm_async_error(g.comm)
                if r not in (0, 7):                   # ncclSuccess, ncclInProgress
                    bad.append(f"{k[0]} group {list(g.ranks)}: ncclResult {r}")
        return bad

    def abort(self, timeout: float = 60.0) -> bool:
        """Release every pending operation (watchdog path); the communicators
        are unusable afterwards.  All communicators are aborted concurrently:
        ncclCommAbort frees device memory, which waits for the device, so
        aborting an idle communicator while another one's kernel still spins
        would block until that kernel is aborted too.  Returns False when an
        abort has not returned within `timeout` seconds."""
        import threading
        comms = [g.comm for g in self._groups.values() if g.comm]
        for g in self._groups.values():
            g.comm = 0
        threads = [threading.Thread(target=native.comm_abort, args=(c,), daemon=True)
                   for c in comms]
        for t in threads:
            t.start()
        end = time.monotonic() + timeout
        for t in threads:
            t.join(max(0.0, end - time.monotonic()))
        return not any(t.is_alive() for t in threads)

    def close(self) -> None:
        for g in self._groups.values():
            if g.comm:
                native.comm_destroy(g.comm)
                g.comm = 0
