"""Static per-stage programs: the GPipe / 1F1B microbatch order and the
instruction lists the runtime interprets.

Restates reference reshard.py:331-424 (`_schedule_phases`, `emit_instructions`,
`_phase_durations`) so that the executor's program is identical, instruction by
instruction, to the one the reference simulator would run (checked against the
reference's `Program.to_json`, tests/test_plan_parity.py).  The runtime then
executes the same list for real: `compute` runs the stage's forward/backward
ops on the GPU instead of advancing a clock by `duration`.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction
from typing import Optional

from .plan import ExecPlan, PlanError
from .xmesh import Boundary, stage_boundaries

GPIPE = "gpipe"
ONE_F_ONE_B = "1f1b"
SCHEDULES = (GPIPE, ONE_F_ONE_B)


@dataclass(frozen=True)
class Instr:
    op: str                    # alloc|free|recv|compute|send|all_gather|sync
    stage: int
    microbatch: Optional[int] = None
    phase: Optional[str] = None
    buffer: Optional[str] = None
    nbytes: int = 0
    peer: Optional[int] = None
    tag: Optional[str] = None
    duration: Optional[Fraction] = None
    pairs: tuple = ()
    axes: tuple = ()
    boundary: Optional[Boundary] = field(default=None, compare=False, repr=False)
    gather_index: Optional[int] = None

    def to_json(self) -> dict:
        d: dict = {"op": self.op, "stage": self.stage}
        for k in ("microbatch", "phase", "buffer", "peer", "tag"):
            v = getattr(self, k)
            if v is not None:
                d[k] = v
        if self.nbytes:
            d["bytes"] = self.nbytes
        if self.duration is not None:
            d["duration"] = [self.duration.numerator, self.duration.denominator]
        if self.pairs:
            d["pairs"] = [list(p) for p in self.pairs]
        if self.axes:
            d["axes"] = list(self.axes)
        return d


@dataclass
class StageProgram:
    stage: int
    device_ids: tuple[int, ...]
    resident_bytes: int
    instructions: list[Instr]


@dataclass
class Program:
    stages: list[StageProgram]
    num_microbatches: int
    schedule: str
    has_backward: bool
    t_star: Fraction
    boundaries: list[Boundary]

    def to_json(self) -> dict:
        return {
            "schedule": self.schedule,
            "num_microbatches": self.num_microbatches,
            "has_backward": self.has_backward,
            "t_star": [self.t_star.numerator, self.t_star.denominator],
            "stages": [{"stage": sp.stage, "devices": list(sp.device_ids),
                        "resident_bytes": sp.resident_bytes,
                        "instructions": [i.to_json() for i in sp.instructions]}
                       for sp in self.stages],
        }


def phase_order(schedule: str, stage: int, num_stages: int, B: int,
                backward: bool) -> list[tuple[str, int]]:
    """(phase, microbatch) sequence of one stage."""
    if not backward:
        return [("fwd", b) for b in range(B)]
    if schedule == GPIPE:
        return [("fwd", b) for b in range(B)] + [("bwd", b) for b in range(B)]
    ahead = min(B, num_stages - stage)       # forwards in flight before the first backward
    seq = [("fwd", b) for b in range(ahead)]
    nxt = ahead
    for b in range(B):
        seq.append(("bwd", b))
        if nxt < B:
            seq.append(("fwd", nxt))
            nxt += 1
    return seq


def phase_durations(plan: ExecPlan) -> dict[int, tuple[Fraction, Fraction]]:
    out = {}
    g = plan.graph
    for st in plan.stages:
        if not plan.has_backward:
            out[st.index] = (st.t, Fraction(0))
            continue
        total = sum(g[o].flop for o in st.op_ids)
        fwd_flop = sum(g[o].flop for o in st.op_ids if g[o].colocate_with is None)
        fwd = st.t / 2 if total == 0 else st.t * Fraction(fwd_flop, total)
        out[st.index] = (fwd, st.t - fwd)
    return out


def build_program(plan: ExecPlan, schedule: str = GPIPE,
                  boundaries: Optional[list[Boundary]] = None) -> Program:
    if schedule not in SCHEDULES:
        raise PlanError(f"unknown schedule {schedule!r}; choose from {SCHEDULES}")
    B = plan.num_microbatches
    S = len(plan.stages)
    bwd = plan.has_backward
    bds = stage_boundaries(plan) if boundaries is None else boundaries
    durs = phase_durations(plan)
    incoming = {(st.index, ph): [b for b in bds if b.consumer == st.index and b.phase == ph]
                for st in plan.stages for ph in ("fwd", "bwd")}
    outgoing = {(st.index, ph): [b for b in bds if b.producer == st.index and b.phase == ph]
                for st in plan.stages for ph in ("fwd", "bwd")}
    progs = []
    for st in plan.stages:
        i = st.index
        ins: list[Instr] = []
        for ph, mb in phase_order(schedule, i, S, B, bwd):
            for bd in incoming[(i, ph)]:
                buf = f"{bd.tag_prefix}.{bd.producer}to{i}.{mb}"
                ins.append(Instr("alloc", i, mb, buffer=buf, nbytes=bd.recv_bytes))
                ins.append(Instr("recv", i, mb, buffer=buf, peer=bd.producer,
                                 nbytes=bd.inter_mesh_bytes,
                                 tag=f"{bd.tag_prefix}:{bd.producer}>{i}:{mb}", boundary=bd))
                for gi, g in enumerate(bd.gathers):
                    ins.append(Instr("all_gather", i, mb, nbytes=g.nbytes, axes=g.axes,
                                     boundary=bd, gather_index=gi))
            if ph == "fwd":
                ins.append(Instr("alloc", i, mb, buffer=f"act{i}.{mb}", nbytes=st.mem_act))
            ins.append(Instr("compute", i, mb, phase=ph,
                             duration=durs[i][0] if ph == "fwd" else durs[i][1]))
            for bd in outgoing[(i, ph)]:
                ins.append(Instr("send", i, mb, peer=bd.consumer, nbytes=bd.inter_mesh_bytes,
                                 tag=f"{bd.tag_prefix}:{i}>{bd.consumer}:{mb}",
                                 pairs=tuple((t.src_device, t.dst_device, t.nbytes)
                                             for t in bd.transfers), boundary=bd))
            if ph == "bwd" or not bwd:
                for pref, phx in (("f", "fwd"), ("b", "bwd")):
                    for bd in incoming[(i, phx)]:
                        ins.append(Instr("free", i, mb, buffer=f"{pref}.{bd.producer}to{i}.{mb}",
                                         nbytes=bd.recv_bytes))
                ins.append(Instr("free", i, mb, buffer=f"act{i}.{mb}", nbytes=st.mem_act))
        ins.append(Instr("sync", i))
        progs.append(StageProgram(i, tuple(st.mesh.device_ids), st.mem_stage, ins))
    return Program(progs, B, schedule, bwd, plan.t_star, bds)


def _frac_of(v) -> Fraction:
    return Fraction(v[0], v[1]) if isinstance(v, (list, tuple)) else Fraction(v)


def modeled_makespan(program: Program, plan: ExecPlan, zero_transfer: bool = False) -> Fraction:
    """The reference simulator's makespan for this program (sim.py:91-188 timing
    rules, exact rationals): per stage in instruction order; compute lasts its
    modeled duration; a send lasts its slowest pair's `transfer_time` (alpha +
    bytes / inter_bw, costs.py:88-92); a recv ends at max(now, its send's end);
    an all_gather costs alpha + (g-1)/g * bytes / min axis bandwidth
    (costs.py:63-73); sync is a barrier across the stages.  Memory accounting
    is not restated (the executor measures real memory).  This is the modeled
    comparator printed beside measured B200 times."""
    cl = plan.cluster
    alpha, inter_bw = _frac_of(cl["alpha"]), _frac_of(cl["inter_bw"])
    stages = program.stages
    n = len(stages)
    pc, now = [0] * n, [Fraction(0)] * n
    send_end: dict[str, Fraction] = {}

    def dur(ins: Instr) -> Fraction:
        if ins.op == "compute":
            return ins.duration or Fraction(0)
        if zero_transfer or ins.op in ("alloc", "free", "sync", "recv"):
            return Fraction(0)
        if ins.op == "send":
            return max((alpha + Fraction(b) / inter_bw for *_, b in ins.pairs), default=Fraction(0))
        if ins.op == "all_gather":
            st = plan.stages[ins.stage]
            g = st.mesh.group_extent(ins.axes)
            if g <= 1:
                return Fraction(0)
            bw = min(st.axis_bw[a] for a in ins.axes)
            return alpha + Fraction((g - 1) * ins.nbytes, g) / bw
        return Fraction(0)

    total = sum(len(sp.instructions) for sp in stages)
    done = 0
    while done < total:
        progressed = False
        at_sync = [pc[i] < len(stages[i].instructions) and
                   stages[i].instructions[pc[i]].op == "sync" for i in range(n)]
        fin = [pc[i] >= len(stages[i].instructions) for i in range(n)]
        if all(a or f for a, f in zip(at_sync, fin)) and not all(fin):
            barrier = max(now[i] for i in range(n) if at_sync[i])
            for i in range(n):
                if at_sync[i]:
                    now[i] = barrier
                    pc[i] += 1
                    done += 1
            continue
        for i in range(n):
            while pc[i] < len(stages[i].instructions):
                ins = stages[i].instructions[pc[i]]
                if ins.op == "sync":
                    break
                if ins.op == "recv":
                    if ins.tag not in send_end:
                        break
                    now[i] = max(now[i], send_end[ins.tag])
                else:
                    now[i] += dur(ins)
                    if ins.op == "send":
                        send_end[ins.tag] = now[i]
                pc[i] += 1
                done += 1
                progressed = True
        if not progressed:
            raise PlanError("deadlock in the instruction lists")
    return max(now) if now else Fraction(0)
