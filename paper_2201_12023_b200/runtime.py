"""The B200 plan executor: the drop-in for the reference's
`emit_instructions -> simulate` path (reshard.py:347-405, sim.py:91-188).

One process per GPU.  Each rank runs the instruction list of the stage that owns
its device, in order, for real:

  alloc / free      microbatch activation state (act{i}.{b}) and recv buffers
  recv / send       cross-mesh Transfers: sender-side box packing (mp_pack_box)
                    and NCCL P2P over NVLink on a per-boundary communicator,
                    receiver-side unpacking (mp_unpack_box)        reshard.py:97-157
  all_gather        the paper's local all-gather over a dst replica group
  compute fwd/bwd   the stage's ops on its logical mesh: each device runs its
                    local shard (tcgen05 GEMM / row kernels), inputs resharded
                    to the algorithm's input specs, k-split partials all-reduced
  sync              end of step: gradient reduction + fused Adam, barrier

The result mirrors SimResult (makespan, utilization, peak_bytes, events) with
measured times, plus the step loss and (optionally) the parameter gradients.
"""
from __future__ import annotations

import math
import os
import json
import time
import zlib
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Callable, Optional

import numpy as np
import torch
import torch.distributed as dist

from . import native
from .binding import Bound, bind
from .comm import Comm
from .layout import (all_local, allgather_axes, canonical, matmul_algo, relayout_moves,
                     reshape_required)
from .plan import (KIND_PARAM, ExecPlan, Mesh, PlanError, Spec, box_numel, device_box, load_plan,
                   local_dims, replicated)
from .schedule import GPIPE, Instr, Program, build_program, modeled_makespan
from .xmesh import recvs_of, sends_of


def stable_seed(*parts) -> int:
    """Process-independent 31-bit seed (Python's str hash is salted per process,
    so hash() would give every torchrun rank different synthetic weights)."""
    return zlib.crc32("/".join(str(p) for p in parts).encode()) & 0x7FFFFFFF


class ExecError(RuntimeError):
    """Executor failure naming rank and instruction (the SimError analogue,
    sim.py:26).  kind: "oom" (CUDA allocator, or the device_memory cap:
    sim.py:152-160), "deadlock" (watchdog timeout: sim.py:172-178), "nccl"
    (asynchronous communicator failure), "kernel" (a libmpexec call failed),
    "plan" (the plan cannot be executed as given)."""

    def __init__(self, msg: str, *, kind: str = "plan", rank: Optional[int] = None,
                 stage: Optional[int] = None, instruction: Optional[str] = None):
        super().__init__(msg)
        self.kind = kind
        self.rank = rank
        self.stage = stage
        self.instruction = instruction


@dataclass
class ExecEvent:
    stage: int
    op: str
    label: str
    start: float
    end: float


@dataclass
class ExecResult:
    makespan: float                               # seconds, measured (max over ranks)
    utilization: dict[int, float]                 # busy (compute/send/all_gather) / makespan
    peak_bytes: dict[int, int]                    # per device id (torch allocator peak)
    events: list[ExecEvent]
    loss: float                                   # sum over microbatches of 1/2 |y|^2
    step_times: list[float] = field(default_factory=list)
    grads: Optional[dict[int, np.ndarray]] = None  # global fp32 parameter gradients
    params: Optional[dict[int, np.ndarray]] = None
    outputs: Optional[dict] = None                  # (microbatch, node) -> global forward output
    gpu_launches: int = 0
    fused: dict = field(default_factory=dict)       # this rank's stage: fused clusters / epilogues
    # the reference simulator's modeled step for this program (schedule.modeled_makespan,
    # sim.py:91-188 timing rules) and the planner's T*, beside the measured makespan
    modeled_makespan: Optional[float] = None
    t_star: Optional[float] = None
    # MoE routing used (collect=True): (microbatch, gates node) -> int32 (T, 4)
    # {e1, pos1|-1, e2, pos2|-1}, the decisions the parity check replays
    routes: Optional[dict] = None

    def trace_json(self) -> str:
        """The reference's sim.json document (SimResult.trace_json, sim.py:46-57)
        with measured seconds: makespan as an exact [num, den] of whole
        nanoseconds, utilization per stage, peak bytes per device, every
        instruction's event.  Extra key: "measured": true."""
        ns = Fraction(round(self.makespan * 1e9), 10 ** 9)
        doc = {
            "makespan": [ns.numerator, ns.denominator],
            "makespan_seconds": float(self.makespan),
            "utilization": {str(k): float(v) for k, v in sorted(self.utilization.items())},
            "peak_bytes": {str(k): int(v) for k, v in sorted(self.peak_bytes.items())},
            "events": [{"stage": e.stage, "op": e.op, "label": e.label,
                        "start": float(e.start), "end": float(e.end)} for e in self.events],
            "measured": True,
        }
        return json.dumps(doc, sort_keys=True, indent=2)

    def gantt_rows(self, program) -> dict[str, list[list]]:
        """Per-device rows of [start, end, label] of the busy instructions
        (compute / send / all_gather) of the device's stage (sim.py:59-71)."""
        by_stage: dict[int, list[ExecEvent]] = {}
        for e in self.events:
            if e.op in BUSY_OPS:
                by_stage.setdefault(e.stage, []).append(e)
        rows: dict[str, list[list]] = {}
        for sp in program.stages:
            seq = [[float(e.start), float(e.end), e.label] for e in by_stage.get(sp.stage, [])]
            for dev in sp.device_ids:
                rows[str(dev)] = seq
        return rows


@dataclass
class AdamConfig:
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.0


BUSY_OPS = ("compute", "send", "all_gather")      # sim.py:23
# watchdog: a step whose device work has not finished after this many seconds
# is a deadlock (ExecError naming the first unfinished instruction)
STEP_TIMEOUT_S = float(os.environ.get("MPEXEC_STEP_TIMEOUT_S", "600"))

# Relayout prefetch on a side stream (StageRunner._prefetch).  Off by default:
# measured slower on both tensor-parallel bench plans (gpt13b_n4_tp 3149 -> 3011,
# moe24b_n4_ep 866 -> 801 TFLOP/s): the side-stream NCCL kernels take SMs from
# the persistent GEMMs that overlap them.
PREFETCH_RELAYOUT = os.environ.get("MPEXEC_PREFETCH_RELAYOUT", "0") == "1"
GATHER_ANY_DIM = os.environ.get("MPEXEC_GATHER_ANY_DIM", "1") != "0"
FUSE_BMM_EPI = os.environ.get("MPEXEC_FUSE_BMM_EPILOGUE", "1") == "1"


def _lo(box):
    return tuple(lo for lo, _ in box)


def _ext(box):
    return tuple(hi - lo for lo, hi in box)


def _rel(box, origin):
    return tuple((lo - o, hi - o) for (lo, hi), o in zip(box, origin))


class _Op:
    __slots__ = ("nid", "op", "bound", "ins", "out_spec", "algo", "grad_direct", "extra", "epi")

    def __init__(self, nid, op, bound, ins, out_spec, algo=None):
        self.nid = nid
        self.op = op
        self.bound = bound
        self.ins = ins                   # list of (producer id, required spec)
        self.out_spec = out_spec
        self.algo = algo
        self.grad_direct = False         # dW accumulated straight into the fp32 grad buffer
        self.extra = None
        self.epi = None                  # fused GEMM epilogue (kind, consumer, aux node)


class StageRunner:
    """Executes one stage's program on one device."""

    def __init__(self, plan: ExecPlan, program: Program, device_id: int, comm: Comm, *,
                 seed: int = 0, params: Optional[dict[int, np.ndarray]] = None,
                 inputs: Optional[Callable[[int, int], np.ndarray]] = None,
                 adam: Optional[AdamConfig] = None, input_scale: float = 1.0,
                 host_inputs: bool = False):
        self.plan = plan
        self.graph = plan.graph
        self.program = program
        self.me = device_id
        self.comm = comm
        self.st = plan.stage_of_device(device_id)
        self.mesh: Mesh = self.st.mesh
        self.sprog = program.stages[self.st.index]
        self.bound = bind(plan.graph)
        self.seed = seed
        self.adam = adam or AdamConfig()
        # GPT-2-style residual scaling: the IR has no LayerNorm, so every branch
        # weight gets std 0.02/sqrt(2*blocks) to keep the residual stream O(1)
        blocks = max(1, sum(1 for b in self.bound.values() if b.op in ("gelu", "softmax")) // 2)
        self.init_std = 0.02 / math.sqrt(2 * blocks)
        self.inputs_fn = inputs
        self.host_inputs = host_inputs
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.cons = plan.graph.consumers()
        self._moves_cache: dict = {}
        self._plans: dict = {}
        self.dw_stream = (torch.cuda.Stream() if os.environ.get("MPEXEC_DW_STREAM", "1") != "0"
                          else None)
        self.dw_pending = False
        self.g_fresh: set[int] = set()
        # MPEXEC_OP_TIMING=1: CUDA events around every op and relayout (analysis only)
        self.op_timer = [] if os.environ.get("MPEXEC_OP_TIMING") == "1" else None
        self.relayout_timer: list = []
        # relayout prefetch (see _prefetch): learned (node -> layouts its consumers
        # reshard it to), issued on a side stream as soon as the node is produced
        self._pf = False
        self.pf_stream = None
        self.pf_learn: dict[int, list] = {}
        self._compile()
        if self.mesh.size > 1 and PREFETCH_RELAYOUT:
            self.pf_stream = torch.cuda.Stream()
        self._init_params(params)
        self.step_count = 0
        self.vals: dict[int, dict[int, torch.Tensor]] = {}
        self.cache: dict[int, dict] = {}
        self.aux: dict[int, dict] = {}
        self.loss_acc = torch.zeros(1, dtype=torch.float32, device=self.dev)
        self.outputs: dict[int, torch.Tensor] = {}
        self.routes: dict[tuple[int, int], np.ndarray] = {}
        self.keep_outputs = False
        self._host_input_bufs: dict = {}
        self.h2d_bytes = 0
        self.send_stream = torch.cuda.Stream()
        self.sends_pending = False
        # CUDA graphs: one capture per (phase, slot); slots = in-flight bound
        self.use_graphs = os.environ.get("MPEXEC_CUDA_GRAPHS", "1") == "1"
        nst = len(plan.stages)
        B = plan.num_microbatches
        self.n_slots = (max(1, min(B, nst - self.st.index)) if program.schedule == "1f1b" or
                        not plan.has_backward else B)
        self.graphs: dict = {}
        self.cap_vals: dict = {}
        self.cap_aux: dict = {}
        self.static: dict = {}
        self.slot_send_ev: dict[int, torch.cuda.Event] = {}
        self.cap_out: dict = {}
        self.cap_routes: dict = {}
        self.graph_kernels: dict = {}
        self.capture_stream = None
        self.replayed_kernels = 0        # libmpexec kernels launched by graph replays
        self._cap_routes: list = []
        bwd = [i.microbatch for i in self.sprog.instructions
               if i.op == "compute" and i.phase == "bwd"]
        self.first_bwd_mb = bwd[0] if bwd else None

        self.input_mode = "host" if host_inputs else ("fn" if inputs is not None else "resident")
        self.h2d_stream = None
        self.h2d_ring: dict = {}
        self.h2d_ring_free: dict = {}
        self.h2d_ready: dict = {}
        self._resident_inputs: dict = {}

    # ------------------------------------------------------------------ compile
    def spec(self, nid: int) -> Spec:
        return canonical(self.st.spec_of(nid), self.mesh)

    def _compile(self):
        g = self.graph
        members = set(self.st.op_ids)
        self.fwd_ops: list[_Op] = []
        self.bwd_ops: list[_Op] = []
        self.param_ids: list[int] = []
        self.input_ids: list[int] = []
        # Parameters live with their consumers.  The planner's contiguous layer
        # cut can leave a weight node in one stage and its matmul in the next
        # (a boundary tensor of the plan); the executor keeps such a weight --
        # and its fp32 master / Adam state -- in the consuming stage, which also
        # owns its gradient, and the per-microbatch send/recv of it is elided.
        self.rehomed = {nid for nid in self.st.input_specs if g[nid].kind == KIND_PARAM}
        stage_of = self.plan.stage_of_op()
        for nid in sorted(set(self.st.op_ids) | self.rehomed):
            n = g[nid]
            b = self.bound[nid]
            out = self.spec(nid)
            if b.op == "param":
                users = {stage_of[c] for c, _ in self.cons[nid]}
                if len(users) > 1:
                    raise ExecError(f"parameter {nid} is consumed by stages {sorted(users)}; "
                                    "a weight shared across stages is not supported")
                if users and self.st.index not in users:
                    continue                          # moved to its consuming stage
                self.param_ids.append(nid)
                continue
            if b.op == "input":
                self.input_ids.append(nid)
                op = _Op(nid, "input", b, [], out)
                self.fwd_ops.append(op)
                continue
            if b.op in ("matmul", "bmm"):
                algo = matmul_algo(b.op == "bmm", out, self.mesh)
                ins = [(n.inputs[0], algo.in_specs[0]), (n.inputs[1], algo.in_specs[1])]
                op = _Op(nid, b.op, b, ins, out, algo)
                if n.grad_of is not None:
                    if self.cons[nid]:
                        raise ExecError(f"node {nid}: a consumed parameter gradient is not "
                                        "supported (builders never produce one)")
                    op.grad_direct = True
            elif n.kind == "reshape":
                req = reshape_required(b, out, len(g[n.inputs[0]].dims))
                ins = [(n.inputs[0], req)]
                if b.fwd_ref is not None:          # MoE routing gradients read the gates
                    ins.append((b.fwd_ref, replicated(len(g[b.fwd_ref].dims))))
                op = _Op(nid, b.op, b, ins, out)
            elif b.op == "reduce_sum":
                # operand replicated along the reduced axis, else in the output's layout
                ax = n.reduce_axis
                if len(g[n.inputs[0]].dims) != 3 or ax != 1:
                    raise ExecError(f"node {nid}: only (A, B, C) -> (A, C) reductions are bound")
                d = out.dims
                req = Spec(d[:ax] + ((),) + d[ax:])
                op = _Op(nid, b.op, b, [(n.inputs[0], req)], out)
            else:
                ins = [(p, out) for p in n.inputs]
                if b.fwd_ref is not None:
                    ins.append((b.fwd_ref, out))
                op = _Op(nid, b.op, b, ins, out)
            (self.fwd_ops if n.colocate_with is None else self.bwd_ops).append(op)
        # bmm outputs consumed only by a head merge are written in merged layout
        for op in self.fwd_ops + self.bwd_ops:
            if op.op != "bmm" or op.nid in self.st.output_specs:
                continue
            users = self.cons[op.nid]
            if len(users) != 1 or users[0][0] not in members:
                continue
            ub = self.bound[users[0][0]]
            if ub.op in ("merge", "merge_t") and op.out_spec.is_replicated() and \
                    self.spec(users[0][0]).is_replicated():
                op.extra = (ub.op, ub.heads)
        # stage outputs that other stages need
        self.out_ids = set(self.st.output_specs)
        self.grad_nodes = {g[n].grad_of: n for n in self.st.op_ids if g[n].grad_of is not None}
        # fwd output of the graph (for the loss seed / checks)
        self.seed_ids = [o.nid for o in self.bwd_ops if o.op == "seed"]
        self.members = members
        # values stored in a layout other than the plan's (fused-cluster outputs)
        self.actual: dict[int, Spec] = {}
        self.fuse_attention = os.environ.get("MPEXEC_FUSE_ATTENTION", "1") != "0"
        self.force_key_split = os.environ.get("MPEXEC_ATTN_KEY_SPLIT", "0") == "1"
        self.attn_clusters = self._fuse_attention() if self.fuse_attention else []
        self.fused_epilogues = (self._fuse_epilogues()
                                if os.environ.get("MPEXEC_FUSE_EPILOGUE", "1") != "0" else 0)
        self.tok_dw: dict[int, tuple[int, ...]] = {}
        if os.environ.get("MPEXEC_TOKEN_SPLIT_DW", "1") != "0":
            self._token_split_dw()
        self.local_conv = (self._local_conv()
                           if os.environ.get("MPEXEC_LOCAL_CONV", "1") != "0" else {})

    def have_spec(self, nid: int) -> Spec:
        """Layout the node's value is actually stored in."""
        return self.actual.get(nid) or self.spec(nid)

    def _token_split_dw(self) -> None:
        """dW = transpose(X) @ G with X and G both split over tokens the same
        way (data parallelism inside the stage): when the plan's algorithm
        would reshard X or G for it (e.g. a square transpose kept at S^aR, so X
        must go column-split), compute the local partial X_loc^T G_loc into a
        full-size fp32 buffer instead and all-reduce it over the token axes
        once per step (reduce_grads) — the same sum, no per-microbatch
        traffic.  The skipped transpose is dropped when nothing else reads it."""
        g = self.graph
        drop = set()
        for o in self.bwd_ops:
            if o.op != "matmul" or not o.grad_direct:
                continue
            (a, a_req), (bn, b_req) = o.ins
            if self.bound[a].op != "transpose" or a not in self.members:
                continue
            X = g[a].inputs[0]
            hx, hb = self.have_spec(X), self.have_spec(bn)
            if len(hx.dims) != 2 or hx.dims[1] or not hx.dims[0] or hb != hx:
                continue
            t_req = canonical(reshape_required(self.bound[a], self.spec(a), 2), self.mesh)
            costly = False
            for nid, have, req in ((X, hx, t_req), (a, self.have_spec(a), a_req),
                                   (bn, hb, b_req)):
                req = canonical(req, self.mesh)
                if have != req and self._relayout_plan(tuple(g[nid].dims), have, req)[0] != "local":
                    costly = True
            if not costly:
                continue
            o.extra = ("tok_dw", X)
            self.tok_dw[o.nid] = tuple(hx.dims[0])   # full-size buffer: _init_params
            if all(c == o.nid for c, _ in self.cons[a]) and a not in self.out_ids:
                drop.add(a)
        self.bwd_ops = [o for o in self.bwd_ops if o.nid not in drop]

    def _local_conv(self) -> dict[int, tuple[int, ...]]:
        """Wide-ResNet adapters on row-split activations.  The planner makes every
        im2col / subsample reshape (and its backward) a layout barrier: replicated
        in, replicated out (intra.py:149-160), i.e. an all-gather of the activation
        on every device.  When the operand's rows are split over mesh axes A in
        whole images (S^A on dim 0, N divisible by the A-group), each device's image
        block maps to a contiguous row block of the output, so the adapter runs on
        the local images and its value is kept row-split (`actual`); consumers
        that want it that way (the S^A R matmuls of data-parallel stages) read it
        with no communication, others reshard on demand."""
        out = {}
        for op in self.fwd_ops + self.bwd_ops:
            if op.op not in ("im2col", "col2im", "subsample", "subsample_grad") or \
                    op.nid in self.out_ids:
                continue
            sp = self.spec(op.ins[0][0])
            if len(sp.dims) != 2 or not sp.dims[0] or sp.dims[1]:
                continue
            A = tuple(sp.dims[0])
            if op.bound.conv[0] % self.mesh.group_extent(A) == 0:
                out[op.nid] = A
        return out

    def _fuse_epilogues(self) -> int:
        """Fold a matmul's single trivial consumer into its GEMM epilogue:
        gelu (dual output: pre-activation + activation), gelu_bwd (dX * gelu'),
        add (residual / gradient accumulation).  Only when no relayout or
        all-reduce sits between them (same spec, no k-split) and the matmul's
        own value is not needed elsewhere.  Returns the number fused."""
        refs = {op.bound.fwd_ref for op in self.fwd_ops + self.bwd_ops if op.bound.fwd_ref is not None}
        n = 0
        for name in ("fwd_ops", "bwd_ops"):
            ops = getattr(self, name)
            pos = {o.nid: i for i, o in enumerate(ops)}
            removed = set()
            for i, o in enumerate(ops):
                if o.op not in ("matmul", "bmm") or o.grad_direct or o.algo.k_axes \
                        or o.epi is not None or o.extra is not None \
                        or o.nid in self.st.output_specs:
                    continue
                users = self.cons[o.nid]
                if len(users) != 1 or users[0][0] not in pos or users[0][0] in removed:
                    continue
                u = users[0][0]
                uop = ops[pos[u]]
                if self.spec(u) != o.out_spec:
                    continue
                # epilogue aux rows must be 16-byte aligned (8 bf16 columns)
                if local_dims(self.graph[o.nid].dims, o.out_spec, self.mesh)[-1] % 8:
                    continue
                # bmm: the MoE expert FFN only (GPU time at K = 1024, graph-timed:
                # dual 306 us vs 227 + 87 us unfused; GeLU' 370 vs 227 + 174 us)
                if o.op == "bmm" and (uop.op not in ("gelu", "gelu_bwd") or not FUSE_BMM_EPI):
                    continue
                if uop.op == "gelu":
                    o.epi = ("dual", u, None)
                elif uop.op == "gelu_bwd" and o.nid not in refs:
                    x_ref = uop.bound.fwd_ref
                    if uop.ins[0][0] != o.nid or self.spec(x_ref) != o.out_spec:
                        continue
                    o.epi = ("gelu_grad", u, x_ref)
                elif uop.op == "add" and o.nid not in refs:
                    others = [p for p, _ in uop.ins if p != o.nid]
                    if len(others) != 1 or pos.get(others[0], -1) > i \
                            or self.spec(others[0]) != o.out_spec:
                        continue
                    o.epi = ("add", u, others[0])
                else:
                    continue
                removed.add(u)
                n += 1
            setattr(self, name, [o for o in ops if o.nid not in removed])
        return n

    # ------------------------------------------------------------------ fusion
    def _fuse_attention(self) -> list[dict]:
        """Replace each eligible attention cluster (graph.py:297-302 and its
        backward, graph.py:341-361) by the fused tcgen05 kernels (d = 64,
        s % 128 == 0).  The cluster's interior (head splits, scores, probs,
        their transposes and gradients) is never materialised, so the executor
        is free to pick how the work is split across the stage's devices; the
        values leaving the cluster are bit-for-bit the same tensors:

          local  q, k, v, dctx brought to one common (T, h) layout whose every
                 device tile is whole sequences x whole heads (batch split,
                 head split, or replicated): attention runs on the local tile
                 with no communication, and the head merges of ctx / dq / dk /
                 dv are produced directly in that layout (their consumers
                 reshard on demand, runtime.get)
          keys   the plan shards the key dim of scores / probs (RRS^A) over
                 replicated q, k, v: attention over the local key block, LSE
                 combine across A (see _run_attn_fwd)

        Returns the clusters fused."""
        g = self.graph
        b = self.bound
        cons = self.cons
        colo: dict[int, list[int]] = {}
        for nid in self.st.op_ids:
            c = g[nid].colocate_with
            if c is not None:
                colo.setdefault(c, []).append(nid)
        clusters = []
        for op in list(self.fwd_ops):
            S = op.nid
            if op.op != "bmm":
                continue
            qh, kh = g[S].inputs
            if b[qh].op != "split" or b[kh].op != "split_t":
                continue
            fwd_users = [c for c, _ in cons[S] if g[c].colocate_with is None]
            if len(fwd_users) != 1 or b[fwd_users[0]].op != "softmax":
                continue
            P = fwd_users[0]
            p_fwd = [c for c, _ in cons[P] if g[c].colocate_with is None]
            if len(p_fwd) != 1 or b[p_fwd[0]].op != "bmm" or g[p_fwd[0]].inputs[0] != P:
                continue
            C = p_fwd[0]
            vh = g[C].inputs[1]
            if b[vh].op != "split":
                continue
            Bn, H, sq, d = b[qh].heads
            if d != 64 or sq % 128 or b[kh].heads != (Bn, H, sq, d) or b[vh].heads != (Bn, H, sq, d):
                continue
            bwd = sorted(colo.get(C, []) + colo.get(P, []) + colo.get(S, []))
            try:
                dprobs = [n for n in colo.get(C, []) if b[n].op == "bmm" and g[n].inputs[0] != P
                          and b[g[n].inputs[1]].op == "transpose"][0]
                dvh = [n for n in colo.get(C, []) if b[n].op == "bmm" and n != dprobs][0]
                dS = [n for n in colo.get(P, []) if b[n].op == "softmax_bwd"][0]
                dqh = [n for n in colo.get(S, []) if b[n].op == "bmm" and g[n].inputs[0] == dS][0]
                dkh = [n for n in colo.get(S, []) if b[n].op == "bmm" and n != dqh][0]
            except IndexError:
                continue
            gC = g[dvh].inputs[1]                  # dL/dctx (a head split of dL/dctx2)
            if b[gC].op != "split" or g[dprobs].inputs[0] != gC:
                continue
            inner = set([S, P, C] + bwd)
            if any(n in self.st.output_specs for n in inner):
                continue
            # every cluster output consumed only by one head merge
            merges = {}
            for n, want in ((C, "merge"), (dqh, "merge"), (dkh, "merge_t"), (dvh, "merge")):
                users = [c for c, _ in cons[n] if c not in inner]
                if len(users) != 1 or b[users[0]].op != want or users[0] not in self.members:
                    break
                merges[n] = users[0]
            if len(merges) != 4:
                continue
            q, k, v = g[qh].inputs[0], g[kh].inputs[0], g[vh].inputs[0]
            dctx2 = g[gC].inputs[0]
            # head splits whose only consumers are inside the cluster are dropped
            splits = [x for x in (qh, kh, vh, gC)
                      if all(c in inner for c, _ in cons[x]) and x not in self.st.output_specs]
            cl = dict(S=S, P=P, C=C, qh=qh, kh=kh, vh=vh, gC=gC, dqh=dqh, dkh=dkh, dvh=dvh,
                      q=q, k=k, v=v, dctx2=dctx2, heads=(Bn, H, sq, d),
                      scale=b[P].softmax_scale, bwd=set(bwd), splits=set(splits),
                      merges=merges, key_axes=(), kv=(0, sq), local=None)
            local = self._attn_local_spec([q, k, v, dctx2], Bn, H, sq, d)
            if self.force_key_split and self.spec(S).dims[2]:
                local = None            # test hook: exercise the key-split path
            if local is not None and (not local.is_replicated() or self.mesh.size == 1 or
                                      all(self.spec(n).is_replicated()
                                          for n in [S, P, C, qh, kh, vh, gC] + bwd)):
                cl["local"] = local
            else:
                # keys sharded: scores / probs RRS^A over replicated q, k, v, dctx
                ss = self.spec(S)
                if (ss != self.spec(P) or ss.dims[0] or ss.dims[1] or not ss.dims[2]
                        or not all(self.spec(n).is_replicated() for n in (qh, kh, vh, gC))):
                    continue
                ok = True
                for dev in self._stage_devices():
                    k0, k1 = device_box(g[S].dims, ss, self.mesh, dev)[2]
                    ok &= k0 % 128 == 0 and (k1 - k0) % 128 == 0 and k1 > k0
                if not ok:
                    continue
                cl["key_axes"] = tuple(ss.dims[2])
                cl["kv"] = device_box(g[S].dims, ss, self.mesh, self.me)[2]
            clusters.append(cl)
        for cl in clusters:
            local = cl["local"] is not None
            drop_f = {cl["S"], cl["P"], cl["C"]} | (cl["splits"] & {cl["qh"], cl["kh"], cl["vh"]})
            drop_b = set(cl["bwd"]) | (cl["splits"] & {cl["gC"]})
            if local:
                drop_f.add(cl["merges"][cl["C"]])
                drop_b |= {cl["merges"][n] for n in (cl["dqh"], cl["dkh"], cl["dvh"])}
            fwd_ops = []
            for o in self.fwd_ops:
                if o.nid == cl["S"]:
                    nid = cl["merges"][cl["C"]] if local else cl["C"]
                    fo = _Op(nid, "attn_fwd", self.bound[nid], [], self.spec(nid))
                    fo.extra = cl
                    fwd_ops.append(fo)
                elif o.nid not in drop_f:
                    fwd_ops.append(o)
            self.fwd_ops = fwd_ops
            bwd_ops = []
            placed = False
            for o in self.bwd_ops:
                if o.nid in cl["bwd"] and not placed:
                    bo = _Op(cl["dqh"], "attn_bwd", self.bound[cl["dqh"]], [], self.spec(cl["dqh"]))
                    bo.extra = cl
                    bwd_ops.append(bo)
                    placed = True
                if o.nid not in drop_b:
                    bwd_ops.append(o)
            self.bwd_ops = bwd_ops
            if local:
                for n in (cl["C"], cl["dqh"], cl["dkh"], cl["dvh"]):
                    m = cl["merges"][n]
                    if m not in self.out_ids:
                        self.actual[m] = cl["local"]
        return clusters

    def _stage_devices(self) -> list[int]:
        return list(self.mesh.device_ids)

    def _attn_local_spec(self, nids, B: int, H: int, s: int, d: int) -> Optional[Spec]:
        """A (T, h) layout, taken from the attention inputs' own specs (most
        common first), in which every device of the stage holds whole sequences
        x whole heads; None if there is none."""
        specs = [self.spec(n) for n in nids]
        order = sorted(dict.fromkeys(specs), key=lambda sp: (-specs.count(sp), specs.index(sp)))
        dims = (B * s, H * d)
        for sp in order:
            if len(sp.dims) != 2:
                continue
            ok = True
            for dev in self._stage_devices():
                (r0, r1), (c0, c1) = device_box(dims, sp, self.mesh, dev)
                ok &= (r0 % s == 0 and (r1 - r0) % s == 0 and r1 > r0 and
                       c0 % d == 0 and (c1 - c0) % d == 0 and c1 > c0)
            if ok:
                return sp
        return None

    def _run_attn_fwd(self, mb: int, op: _Op):
        """Fused attention forward.  local: the device's tile of whole
        sequences x heads, no communication.  keys: each device attends over
        its own key block, then O and LSE are combined across the key axes A:
        M = max LSE, w = exp(LSE - M), O = sum(w O) / sum(w),
        LSE = M + log sum(w) (two all-reduces) — the plan's RRS^A scores /
        probs are never materialised."""
        cl = op.extra
        Bn, H, s, d = cl["heads"]
        if cl["local"] is not None:
            L = cl["local"]
            q = self._contig(self.get(mb, cl["q"], L))
            k = self._contig(self.get(mb, cl["k"], L))
            v = self._contig(self.get(mb, cl["v"], L))
            Bl, Hl = q.shape[0] // s, q.shape[1] // d
            o = torch.empty(q.shape, dtype=torch.bfloat16, device=self.dev)
            lse = torch.empty(Bl * Hl, s, dtype=torch.float32, device=self.dev)
            native.attn_fwd(q, k, v, o, lse, Bl, Hl, s, d, cl["scale"])
            self.aux.setdefault(mb, {})[cl["S"]] = (o, lse)
            m = cl["merges"][cl["C"]]
            if m in self.out_ids:
                return self._coerce(o, self.graph[m].dims, L, self.spec(m))
            return o
        rep = replicated(2)
        q = self._contig(self.get(mb, cl["q"], rep))
        k = self._contig(self.get(mb, cl["k"], rep))
        v = self._contig(self.get(mb, cl["v"], rep))
        o = torch.empty(Bn * s, H * d, dtype=torch.bfloat16, device=self.dev)
        lse = torch.empty(Bn * H, s, dtype=torch.float32, device=self.dev)
        k0, k1 = cl["kv"]
        native.attn_fwd(q, k, v, o, lse, Bn, H, s, d, cl["scale"], kv_range=(k0, k1 - k0))
        if cl["key_axes"]:
            axes = cl["key_axes"]
            m = lse.clone()
            self._allreduce(m, axes, dist.ReduceOp.MAX)
            w = torch.empty_like(lse)
            native.attn_combine_scale(o, lse, m, w, Bn, H, s, d)
            self._allreduce(o, axes)
            self._allreduce(w, axes)
            native.attn_combine_finish(o, w, m, lse, Bn, H, s, d)
        self.aux.setdefault(mb, {})[cl["S"]] = (o, lse)
        ctx = o.view(Bn, s, H, d).permute(0, 2, 1, 3)        # logical ctx (B*H, s, d)
        return self._coerce(ctx, self.graph[cl["C"]].dims, replicated(3), self.spec(cl["C"]))

    def _run_attn_bwd(self, mb: int, op: _Op):
        """Fused attention backward.  local: dq / dk / dv of the device's tile,
        written as the head merges' values.  keys: dQ partial sums over the
        local keys are all-reduced across the key axes; dK / dV come out for
        the local keys (RRS^A / RS^AR), then reach the nodes' own specs."""
        cl = op.extra
        Bn, H, s, d = cl["heads"]
        g = self.graph
        vals = self.vals[mb]
        o, lse = self.aux[mb][cl["S"]]
        L = cl["local"] if cl["local"] is not None else replicated(2)
        q = self._contig(self.get(mb, cl["q"], L))
        k = self._contig(self.get(mb, cl["k"], L))
        v = self._contig(self.get(mb, cl["v"], L))
        dout = self._contig(self.get(mb, cl["dctx2"], L))
        T, hdim = q.shape
        Bl, Hl = T // s, hdim // d
        k0, k1 = cl["kv"]
        dvec = torch.empty(Bl * Hl, s, dtype=torch.float32, device=self.dev)
        dq_acc = torch.empty(T, hdim, dtype=torch.float32, device=self.dev)   # zeroed by the pre pass
        dk = torch.empty(T, hdim, dtype=torch.bfloat16, device=self.dev)
        dv = torch.empty(T, hdim, dtype=torch.bfloat16, device=self.dev)
        native.attn_bwd(q, k, v, o, dout, lse, dvec, dq_acc, dk, dv, Bl, Hl, s, d, cl["scale"],
                        kv_range=(k0, k1 - k0))
        axes = cl["key_axes"] if cl["local"] is None else ()
        if axes:
            # sum the fp32 partials across the key groups, round to bf16 once
            self._allreduce(dq_acc, axes)
        dq = native.cast_f32_bf16(dq_acc, torch.empty(T, hdim, dtype=torch.bfloat16, device=self.dev))
        if cl["local"] is not None:
            for n, t in ((cl["dqh"], dq), (cl["dkh"], dk), (cl["dvh"], dv)):
                m = cl["merges"][n]
                vals[m] = (self._coerce(t, g[m].dims, L, self.spec(m)) if m in self.out_ids
                           else t)
            return None
        if axes:
            ks = Spec(((), (), axes))
            vs = Spec(((), axes, ()))
        else:
            ks = vs = replicated(3)
        vals[cl["dqh"]] = self._coerce(dq.view(Bn, s, H, d).permute(0, 2, 1, 3), g[cl["dqh"]].dims,
                                       replicated(3), self.spec(cl["dqh"]))
        dk4 = dk.view(Bn, s, H, d).permute(0, 2, 3, 1)
        dv4 = dv.view(Bn, s, H, d).permute(0, 2, 1, 3)
        if axes:
            dk4 = dk4.narrow(3, k0, k1 - k0)
            dv4 = dv4.narrow(2, k0, k1 - k0)
        vals[cl["dkh"]] = self._coerce(dk4, g[cl["dkh"]].dims, ks, self.spec(cl["dkh"]))
        vals[cl["dvh"]] = self._coerce(dv4, g[cl["dvh"]].dims, vs, self.spec(cl["dvh"]))
        return None

    def _coerce(self, v: torch.Tensor, dims, have: Spec, req: Spec) -> torch.Tensor:
        """A local value in layout `have` brought to layout `req` (no cache)."""
        have, req = canonical(have, self.mesh), canonical(req, self.mesh)
        if have == req:
            return v
        if self.op_timer is None:
            return self._coerce_impl(v, dims, have, req)
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        out = self._coerce_impl(v, dims, have, req)
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        kind, _ = self._relayout_plan(tuple(dims), have, req)
        self.relayout_timer.append((kind, math.prod(dims) * v.element_size(), e0, e1))
        return out

    def _coerce_impl(self, v, dims, have: Spec, req: Spec) -> torch.Tensor:
        kind, info = self._relayout_plan(tuple(dims), have, req)
        if kind == "local":
            return self._narrow(v, info)
        if kind == "allgather":
            out = torch.empty(local_dims(dims, req, self.mesh), dtype=v.dtype, device=self.dev)
            src = self._contig(self._as3(v))
            self.comm.all_gather_into(out.view(-1), src.view(-1),
                                      self.comm.axis_group(self.st.index, self.mesh, info, self.me,
                                                           pf=self._pf))
            return out
        if kind == "allgather_dim":
            # gather into a (g, *tile) staging buffer, then one copy that moves
            # the group dim next to `d` (member blocks concatenated along d)
            axes, d = info
            src = self._contig(v).view(*local_dims(dims, have, self.mesh))
            g = self.mesh.group_extent(axes)
            stage = torch.empty((g,) + tuple(src.shape), dtype=v.dtype, device=self.dev)
            self.comm.all_gather_into(stage.view(-1), src.view(-1),
                                      self.comm.axis_group(self.st.index, self.mesh, axes, self.me,
                                                           pf=self._pf))
            perm = stage.movedim(0, d)
            return native.pack_box(perm, (0,) * perm.dim(), tuple(perm.shape)).view(
                *local_dims(dims, req, self.mesh))
        return self._relayout(self._as3(v), tuple(dims), have, req)

    # ------------------------------------------------------------------ params
    def _zero_axes(self, pid: int) -> tuple[int, ...]:
        """Axes over which pid's gradient is all-reduced, when the plan's
        post_ilp_rewrite (intra.py:404-424) realises that all-reduce as
        reduce-scatter + all-gather: a grad root whose algorithm all-reduces
        over axes of extent > 1.  Only for gradients laid out like the parameter
        (or full-size token-split partials) and evenly divisible."""
        if os.environ.get("MPEXEC_ZERO", "1") == "0":
            return ()
        dw = self.grad_nodes.get(pid)
        if dw is None:
            return ()
        if dw in self.tok_dw:
            axes = self.tok_dw[dw]
            if not self.spec(pid).is_replicated():
                return ()
        else:
            if self.spec(dw) != self.spec(pid):
                return ()
            axes = matmul_algo(self.bound[dw].op == "bmm", self.spec(dw), self.mesh).k_axes
        gsz = self.mesh.group_extent(axes) if axes else 1
        if gsz <= 1:
            return ()
        n = math.prod(local_dims(self.graph[pid].dims, self.spec(pid), self.mesh))
        return tuple(axes) if n % gsz == 0 else ()

    def _init_params(self, init: Optional[dict[int, np.ndarray]]):
        """Resident local shards.  bf16 working copies of every parameter live in
        one flat buffer (wbf16).  fp32 master / Adam m, v live in flat buffers
        too: full local tiles for plain parameters, and for ZeRO parameters
        (replicated over the axes their gradient is reduced on) only this
        device's 1/g chunk — the optimizer state the post_ilp_rewrite shards.
        Gradients accumulate full-size in gradbuf (the dW GEMMs write there)."""
        g = self.graph
        self.zero: dict[int, tuple[int, ...]] = {}
        sizes = {}
        for pid in self.param_ids:
            sizes[pid] = math.prod(local_dims(g[pid].dims, self.spec(pid), self.mesh))
            ax = self._zero_axes(pid)
            if ax:
                self.zero[pid] = ax
        plain = [p for p in self.param_ids if p not in self.zero]
        zero = [p for p in self.param_ids if p in self.zero]
        total = sum(sizes.values())
        self.n_param = total
        self.wbf16 = torch.zeros(total, dtype=torch.bfloat16, device=self.dev)
        self.gradbuf = torch.zeros(total, dtype=torch.float32, device=self.dev)
        self.pviews: dict[int, tuple[int, tuple[int, ...]]] = {}
        off = 0
        for pid in plain + zero:                  # plain parameters first
            self.pviews[pid] = (off, tuple(local_dims(g[pid].dims, self.spec(pid), self.mesh)))
            off += sizes[pid]
        self.n_plain = sum(sizes[p] for p in plain)
        # ZeRO chunk of each parameter: (offset in the compact state, chunk, rank in group)
        self.zchunk: dict[int, tuple[int, int, int]] = {}
        zoff = 0
        for pid in zero:
            grp = self.comm.axis_group(self.st.index, self.mesh, self.zero[pid], self.me)
            gsz = len(grp.ranks)
            r = grp.peer(self.me)
            c = sizes[pid] // gsz
            self.zchunk[pid] = (zoff, c, r)
            zoff += c
        self.n_zero_state = zoff
        nstate = self.n_plain + zoff
        self.master = torch.zeros(nstate, dtype=torch.float32, device=self.dev)
        self.m = torch.zeros_like(self.master)
        self.v = torch.zeros_like(self.master)
        self.zgrad = torch.zeros(zoff, dtype=torch.float32, device=self.dev)
        self.zw = torch.zeros(zoff, dtype=torch.bfloat16, device=self.dev)
        full_init = torch.zeros(total, dtype=torch.float32, device=self.dev)
        for pid in self.param_ids:
            off, ld = self.pviews[pid]
            sz = sizes[pid]
            box = device_box(g[pid].dims, self.spec(pid), self.mesh, self.me)
            if init is not None:
                full = np.asarray(init[pid], dtype=np.float32)
                loc = full[tuple(slice(lo, hi) for lo, hi in box)]
                full_init[off:off + sz].copy_(torch.from_numpy(np.ascontiguousarray(loc)).reshape(-1))
            else:
                gen = torch.Generator(device=self.dev)
                gen.manual_seed(stable_seed(self.seed, "param", pid))
                # GPT-style init (std 0.02) keeps the 24-block residual stream O(1)
                full = torch.randn(g[pid].dims, generator=gen, device=self.dev) * self.init_std
                loc = full[tuple(slice(lo, hi) for lo, hi in box)]
                full_init[off:off + sz].copy_(loc.reshape(-1))
                del full
        if total:
            native.cast_f32_bf16(full_init, self.wbf16)
        if self.n_plain:
            self.master[:self.n_plain].copy_(full_init[:self.n_plain])
        for pid, (zo, c, r) in self.zchunk.items():
            off, _ = self.pviews[pid]
            self.master[self.n_plain + zo:self.n_plain + zo + c].copy_(
                full_init[off + r * c:off + (r + 1) * c])
        del full_init
        # gradient buffers of grad_of nodes are laid out in the dW node's own spec;
        # when that differs from the parameter spec a separate fp32 buffer is used.
        self.gviews: dict[int, torch.Tensor] = {}
        for pid in self.param_ids:
            dw = self.grad_nodes.get(pid)
            off, ld = self.pviews[pid]
            if dw is None:
                continue
            dws = self.spec(dw)
            if dw in self.tok_dw and pid not in self.zero:
                self.gviews[dw] = torch.zeros(g[dw].dims, dtype=torch.float32, device=self.dev)
            elif dws == self.spec(pid) or dw in self.tok_dw:
                self.gviews[dw] = self.gradbuf[off:off + math.prod(ld)].view(ld)
            else:
                dld = local_dims(g[dw].dims, dws, self.mesh)
                self.gviews[dw] = torch.zeros(dld, dtype=torch.float32, device=self.dev)

    def param_view(self, pid: int) -> torch.Tensor:
        off, ld = self.pviews[pid]
        return self.wbf16[off:off + math.prod(ld)].view(ld)

    # ------------------------------------------------------------------ values
    def value(self, mb: int, nid: int) -> torch.Tensor:
        if nid in self.pviews:
            return self.param_view(nid)
        try:
            return self.vals[mb][nid]
        except KeyError:
            raise ExecError(f"rank {self.me}: value of node {nid} for microbatch {mb} "
                            f"is not available") from None

    def get(self, mb: int, nid: int, req: Spec) -> torch.Tensor:
        """Local shard of node `nid` in layout `req` (reshard on demand)."""
        have = self.actual.get(nid) or self.spec(nid)
        v = self.value(mb, nid)
        if req == have:
            return v
        key = (nid, req)
        c = self.cache.setdefault(mb, {})
        hit = c.get(key)
        if hit is not None:
            if type(hit) is tuple:                 # prefetched on the side stream
                t, ev = hit
                cur = torch.cuda.current_stream()
                cur.wait_event(ev)
                t.record_stream(cur)
                c[key] = t
                return t
            return hit
        out = self._coerce(v, self.graph[nid].dims, have, req)
        c[key] = out
        if self.pf_stream is not None and not self.use_graphs:
            dims = tuple(self.graph[nid].dims)
            if self._relayout_plan(dims, canonical(have, self.mesh),
                                   canonical(req, self.mesh))[0] != "local":
                reqs = self.pf_learn.setdefault(nid, [])
                if req not in reqs:
                    reqs.append(req)
        return out

    def _prefetch(self, mb: int, nid: int) -> None:
        """Issue the relayouts node `nid`'s consumers needed last time (learned
        by get) right after it is produced, on the side stream with its own
        communicators, so the transfer overlaps the ops in between; get() then
        only waits on the event.  Every rank of the stage issues the same
        prefetches in the same order (same program, same learned table)."""
        v = self.vals[mb].get(nid)
        if v is None:
            return
        c = self.cache.setdefault(mb, {})
        have = self.have_spec(nid)
        dims = self.graph[nid].dims
        cur = torch.cuda.current_stream()
        for req in self.pf_learn[nid]:
            key = (nid, req)
            if key in c or req == have:
                continue
            self.pf_stream.wait_stream(cur)
            self._pf = True
            try:
                with torch.cuda.stream(self.pf_stream):
                    out = self._coerce(v, dims, have, req)
                    ev = torch.cuda.Event()
                    ev.record(self.pf_stream)
            finally:
                self._pf = False
            v.record_stream(self.pf_stream)
            c[key] = (out, ev)

    def _relayout_plan(self, dims, have: Spec, req: Spec):
        """How to realise `req` from `have` on this mesh (cached; decided from
        every device's boxes, so all ranks of the stage agree):
          local      every device's target box lies in its own tile: narrow
          allgather  every device's target is the dim-0 concatenation, in
                     device-id order, of the tiles of one axis group: one NCCL
                     all-gather straight into the output
          p2p        literal box moves (layout.relayout_moves) over NCCL P2P"""
        key = (dims, have, req)
        pl = self._plans.get(key)
        if pl is not None:
            return pl
        m = self.mesh
        if all_local(dims, have, req, m):
            mine = device_box(dims, have, m, self.me)
            want = device_box(dims, req, m, self.me)
            pl = ("local", [(lo - o, hi - lo) for (lo, hi), (o, _) in zip(want, mine)])
        else:
            axes = allgather_axes(dims, have, req, m)
            pl = ("allgather", axes) if axes is not None else None
            for d in range(1, len(dims)):
                if pl is None and GATHER_ANY_DIM:
                    axes = allgather_axes(dims, have, req, m, dim=d)
                    pl = ("allgather_dim", (axes, d)) if axes is not None else None
            if pl is None:
                pl = ("p2p", None)
        self._plans[key] = pl
        return pl

    def _narrow(self, v: torch.Tensor, cuts) -> torch.Tensor:
        """Slice a local value by logical (offset, length) per dim; head-split
        4-D views are narrowed on their batch dim when aligned to heads."""
        if v.dim() == len(cuts) + 1 and all(c[0] == 0 and c[1] == n
                                           for c, n in zip(cuts[1:], v.shape[2:])):
            H = v.shape[1]
            off, ln = cuts[0]
            if off % H == 0 and ln % H == 0:
                return v.narrow(0, off // H, ln // H)
        if v.dim() != len(cuts):
            v = self._as3(v)
        for d, (off, ln) in enumerate(cuts):
            if off != 0 or ln != v.shape[d]:
                v = v.narrow(d, off, ln)
        return v

    def _relayout(self, v: torch.Tensor, dims, have: Spec, req: Spec) -> torch.Tensor:
        key = (dims, have, req)
        moves = self._moves_cache.get(key)
        if moves is None:
            moves = relayout_moves(dims, have, req, self.mesh)
            self._moves_cache[key] = moves
        mine = _lo(device_box(dims, have, self.mesh, self.me))
        want = _lo(device_box(dims, req, self.mesh, self.me))
        out = torch.empty(local_dims(dims, req, self.mesh), dtype=v.dtype, device=self.dev)
        sends, recvs = [], []
        for mv in moves:
            if mv.src == self.me and mv.dst == self.me:
                buf = native.pack_box(v, _lo(_rel(mv.box, mine)), _ext(mv.box))
                native.unpack_box(buf, out, _lo(_rel(mv.box, want)), _ext(mv.box))
            elif mv.src == self.me:
                lo, ext = _lo(_rel(mv.box, mine)), _ext(mv.box)
                view = native.box_view(v, lo, ext)
                sends.append((view if view is not None else native.pack_box(v, lo, ext), mv.dst))
            elif mv.dst == self.me:
                lo, ext = _lo(_rel(mv.box, want)), _ext(mv.box)
                view = native.box_view(out, lo, ext)
                buf = view if view is not None else torch.empty(box_numel(mv.box), dtype=v.dtype,
                                                                device=self.dev)
                recvs.append((buf, mv.src, lo, ext, view is None))
        if sends or recvs:
            grp = self.comm.stage_group(self.st.index, self.mesh, pf=self._pf)
            works = self.comm.p2p(sends, [(b, s) for b, s, *_ in recvs], grp)
            for w in works:
                w.wait()
            for buf, _, lo, ext, packed in recvs:
                if packed:
                    native.unpack_box(buf, out, lo, ext)
        return out

    # ------------------------------------------------------------------ kernels
    def _contig(self, t: torch.Tensor) -> torch.Tensor:
        if t.is_contiguous():
            return t
        return native.pack_box(t, (0,) * t.dim(), tuple(t.shape)).view(t.shape)

    def _allreduce(self, t: torch.Tensor, axes: tuple[int, ...], op=dist.ReduceOp.SUM):
        if self.mesh.group_extent(axes) > 1:
            self.comm.all_reduce(t, self.comm.axis_group(self.st.index, self.mesh, axes, self.me), op)

    def _gemm_operands(self, a, b):
        """Bring two (possibly head-split 4-D) operands to a common batch form."""
        if a.dim() == b.dim():
            return a, b
        # splitting the batch dim is a view for any strides (no copy)
        if a.dim() == 4 and b.dim() == 3:
            return a, b.unflatten(0, (a.shape[0], a.shape[1]))
        if a.dim() == 3 and b.dim() == 4:
            return a.unflatten(0, (b.shape[0], b.shape[1])), b
        raise ExecError(f"gemm operand ranks {a.dim()} / {b.dim()}")

    def _run_matmul(self, mb: int, op: _Op) -> Optional[torch.Tensor]:
        if op.nid in self.tok_dw:
            X = op.extra[1]
            a = self.get(mb, X, self.have_spec(X)).transpose(0, 1)
            b = self.get(mb, op.ins[1][0], self.have_spec(op.ins[1][0]))
        else:
            a = self.get(mb, op.ins[0][0], op.ins[0][1])
            b = self.get(mb, op.ins[1][0], op.ins[1][1])
        a, b = self._gemm_operands(a, b)
        k_axes = op.algo.k_axes
        if op.grad_direct:
            # dW only feeds the step-end reduction: run it on a side stream so it
            # overlaps the dX chain and fills the other GEMMs' tail waves
            gv = self.gviews[op.nid]
            out_view = gv if a.dim() == 2 else gv.view(*a.shape[:-2], a.shape[-2], b.shape[-1])
            # the step's first contribution overwrites (beta = 0): no zero fill
            # of the fp32 gradient buffers between steps
            beta = 1.0
            if op.nid in self.g_fresh:
                self.g_fresh.discard(op.nid)
                beta = 0.0
            main = torch.cuda.current_stream()
            if self.dw_stream is None:
                self._gemm(a, b, out_view, beta=beta)
                return None
            self.dw_stream.wait_stream(main)
            with torch.cuda.stream(self.dw_stream):
                self._gemm(a, b, out_view, beta=beta)
            a.record_stream(self.dw_stream)
            b.record_stream(self.dw_stream)
            self.dw_pending = True
            return None
        shape = tuple(a.shape[:-2]) + (a.shape[-2], b.shape[-1])
        if op.epi is not None:
            kind, u, aux_nid = op.epi
            out = torch.empty(shape, dtype=torch.bfloat16, device=self.dev)
            vals = self.vals[mb]
            if kind == "dual":
                act = torch.empty_like(out)
                self._gemm(a, b, out, epilogue=native.EPI_GELU_DUAL, aux=act)
                vals[u] = act
                return out
            aux = self._contig(self._as3(self.get(mb, aux_nid, op.out_spec)))
            self._gemm(a, b, out, epilogue=native.EPI_GELU_GRAD if kind == "gelu_grad"
                       else native.EPI_ADD, aux=aux)
            vals[u] = out
            return None
        if op.extra is not None and not k_axes:
            # the only consumer is a head merge: write straight into (T, h) layout
            kind, (B, H, s, d) = op.extra
            buf = torch.empty(B * s, H * d, dtype=torch.bfloat16, device=self.dev)
            v4 = buf.view(B, s, H, d)
            out = v4.permute(0, 2, 1, 3) if kind == "merge" else v4.permute(0, 2, 3, 1)
            a4, b4 = a, b
            if a4.dim() == 3:
                a4, b4 = a4.unflatten(0, (B, H)), b4.unflatten(0, (B, H))
            self._gemm(a4, b4, out)
            return out
        out = torch.empty(shape, dtype=torch.bfloat16, device=self.dev)
        self._gemm(a, b, out)
        if k_axes:
            self._allreduce(out, k_axes)
        if out.dim() == 4:
            out = out.view(out.shape[0] * out.shape[1], *out.shape[2:])
        return out

    def _gemm(self, a, b, out, beta=0.0, epilogue=0, aux=None):
        if out.stride(-1) != 1 and out.stride(-2) == 1:
            if epilogue:
                raise ExecError("fused epilogues need a row-major output")
            native.gemm(b.transpose(-1, -2), a.transpose(-1, -2), out.transpose(-1, -2), beta=beta)
        else:
            native.gemm(a, b, out, beta=beta, epilogue=epilogue, aux=aux)

    def _run_reshape(self, mb: int, op: _Op) -> torch.Tensor:
        A = self.local_conv.get(op.nid)
        if A is not None:                     # row-split conv adapter (see _local_conv)
            rs = Spec((A, ()))
            x = self._contig(self.get(mb, op.ins[0][0], rs))
            N, H, W, C, k, s = op.bound.conv
            Nl = N // self.mesh.group_extent(A)
            if op.op == "im2col":
                y = native.im2col(x, Nl, H, W, C, k, s)
            elif op.op == "col2im":
                y = native.col2im(x, Nl, H, W, C, k, s)
            else:
                y = native.subsample(x, Nl, H, W, C, s, backward=op.op == "subsample_grad")
            self.actual[op.nid] = rs
            return y
        x = self.get(mb, op.ins[0][0], op.ins[0][1])
        kind = op.op
        if kind == "identity":
            y = x
        elif kind == "transpose":
            y = x.transpose(-1, -2)
        elif kind in ("dispatch", "combine"):
            G, S, E, C = op.bound.route
            gates = self._contig(x)
            route = native.moe_route(gates, S, C)
            y = native.moe_mask(route, gates, S, C, 0 if kind == "dispatch" else 1)
            if self.keep_outputs and kind == "dispatch":
                if torch.cuda.is_current_stream_capturing():
                    self._cap_routes.append((op.ins[0][0], route))   # copied after replays
                else:
                    self.routes[(mb, op.ins[0][0])] = route.cpu().numpy()
        elif kind in ("dispatch_grad", "combine_grad"):
            G, S, E, C = op.bound.route
            gates = self._contig(self.get(mb, op.ins[1][0], op.ins[1][1]))
            route = native.moe_route(gates, S, C)
            y = native.moe_mask_grad(route, self._contig(self._as3(x)), E, S, C,
                                     0 if kind == "dispatch_grad" else 1)
        elif kind in ("im2col", "col2im", "subsample", "subsample_grad"):
            N, H, W, C, k, s = op.bound.conv
            x2 = self._contig(x)
            if kind == "im2col":
                y = native.im2col(x2, N, H, W, C, k, s)
            elif kind == "col2im":
                y = native.col2im(x2, N, H, W, C, k, s)
            else:
                y = native.subsample(x2, N, H, W, C, s, backward=kind == "subsample_grad")
        elif kind == "broadcast":
            A, B, C = self.graph[op.nid].dims
            y = native.reduce_mid(self._contig(x).view(A, C), broadcast_b=B)
        elif kind == "regroup":
            A, P, C = op.bound.regroup
            x3 = self._as3(x)
            h = x3.shape[-1]
            y = self._contig(x3.view(A, P, C, h).permute(1, 0, 2, 3)).view(P, A * C, h)
        else:
            B, H, s, d = op.bound.heads
            if kind == "split":            # (T,h) -> (B,H,s,d)
                y = self._contig(x).view(B, s, H, d).permute(0, 2, 1, 3)
            elif kind == "split_t":        # (T,h) -> (B,H,d,s)
                y = self._contig(x).view(B, s, H, d).permute(0, 2, 3, 1)
            elif kind in ("merge", "merge_t"):
                x4 = x if x.dim() == 4 else self._contig(x).view(B, H, *x.shape[1:])
                perm = (0, 2, 1, 3) if kind == "merge" else (0, 3, 1, 2)
                y = self._contig(x4.permute(*perm)).view(B * s, H * d)
            else:
                raise ExecError(f"reshape op {kind}")
        if not op.out_spec.is_replicated() and kind not in ("identity", "transpose"):
            box = device_box(self.graph[op.nid].dims, op.out_spec, self.mesh, self.me)
            y = self._contig(y) if y.dim() == len(box) else self._contig(y).view(
                *self.graph[op.nid].dims)
            for d, (lo, hi) in enumerate(box):
                y = y.narrow(d, lo, hi - lo)
        return y

    def _split_axes(self, op: _Op) -> tuple[int, ...]:
        return tuple(a for a in op.out_spec.dims[-1] if self.mesh.extent(a) > 1)

    def _as3(self, t: torch.Tensor) -> torch.Tensor:
        return t if t.dim() != 4 else self._contig(t).view(-1, *t.shape[2:])

    def _run_elementwise(self, mb: int, op: _Op) -> torch.Tensor:
        k = op.op
        xs = [self._contig(self._as3(self.get(mb, p, r))) for p, r in op.ins]
        if k == "gelu":
            return native.gelu(xs[0])
        if k == "add":
            return native.add(xs[0], xs[1])
        if k == "identity":
            return xs[0]
        if k == "seed":
            y = xs[0]
            if self._is_representative(op.nid):
                native.sumsq(y, self.loss_acc)
            if self.keep_outputs:
                self.outputs[mb] = y.float().clone()
            return y
        if k == "gelu_bwd":
            g, x = xs
            return native.gelu_bwd(x, g)
        if k == "softmax":
            x = xs[0]
            split = self._split_axes(op)
            s = op.bound.softmax_scale
            if not split:
                return native.softmax(x, s)
            rows = x.numel() // x.shape[-1]
            stats = native.softmax_stats(x, s, torch.empty(3, rows, dtype=torch.float32, device=self.dev))
            self._allreduce(stats[0], split, dist.ReduceOp.MAX)
            native.softmax_rescale(stats, rows)
            self._allreduce(stats[1], split)
            return native.softmax_apply(x, stats, s)
        if k == "softmax_bwd":
            g, y = xs
            split = self._split_axes(op)
            s = op.bound.softmax_scale
            if not split:
                return native.softmax_bwd(y, g, s)
            rows = y.numel() // y.shape[-1]
            rd = native.softmax_rowdot(y, g, torch.empty(rows, dtype=torch.float32, device=self.dev))
            self._allreduce(rd, split)
            return native.softmax_bwd(y, g, s, rowdot=rd)
        raise ExecError(f"node {op.nid}: no kernel for elementwise op {k}")

    def _is_representative(self, nid: int) -> bool:
        """True on exactly one device per replica group of nid's spec."""
        i, j = self.mesh.coords(self.me)
        rep = set(self.spec(nid).replicated_axes())
        return (0 not in rep or i == 0) and (1 not in rep or j == 0)

    def _load_input(self, mb: int, op: _Op) -> torch.Tensor:
        """One microbatch of a graph input, local shard per its spec.
        fn: caller-provided global arrays (tests / oracle parity);
        resident: synthetic N(0,1) kept in HBM (two alternating microbatches);
        host: the same from pinned host memory, copied H2D every microbatch."""
        g = self.graph
        dims = g[op.nid].dims
        box = device_box(dims, op.out_spec, self.mesh, self.me)
        sl = tuple(slice(lo, hi) for lo, hi in box)
        if self.input_mode == "fn":
            full = np.asarray(self.inputs_fn(mb, op.nid), dtype=np.float32)
            return torch.from_numpy(np.ascontiguousarray(full[sl])).to(
                self.dev, dtype=torch.bfloat16)
        key = (op.nid, mb % 2)
        if self.input_mode == "host":
            hb = self._host_buf(op, mb)
            self.h2d_bytes += hb.numel() * hb.element_size()
            return hb.to(self.dev, non_blocking=True)
        t = self._resident_inputs.get(key)
        if t is None:
            gen = torch.Generator(device=self.dev)
            gen.manual_seed(stable_seed(self.seed, "input", op.nid, mb % 2))
            full = torch.randn(dims, generator=gen, device=self.dev, dtype=torch.float32)
            t = full[sl].to(torch.bfloat16).contiguous()
            self._resident_inputs[key] = t
        return t

    # ------------------------------------------------------------------ phases
    # ------------------------------------------------------------------ CUDA graphs
    def slot_of(self, mb: int) -> int:
        return mb % self.n_slots

    def _slot_guard(self, mb: int) -> None:
        """Graph mode: a slot's static buffers (captured outputs, staged inputs,
        received tensors) are rewritten when the slot is reused for microbatch
        mb; the compute stream first waits for the last send that read them."""
        ev = self.slot_send_ev.pop(self.slot_of(mb), None)
        if ev is not None:
            torch.cuda.current_stream().wait_event(ev)

    def _host_buf(self, op: _Op, mb: int) -> torch.Tensor:
        """Pinned host copy of this device's shard of a synthetic input (two
        alternating microbatches, like the resident inputs)."""
        key = (op.nid, mb % 2)
        hb = self._host_input_bufs.get(key)
        if hb is None:
            dims = self.graph[op.nid].dims
            box = device_box(dims, op.out_spec, self.mesh, self.me)
            gen = torch.Generator()
            gen.manual_seed(stable_seed(self.seed, "input", op.nid, mb % 2))
            full = torch.randn(dims, generator=gen)
            hb = full[tuple(slice(lo, hi) for lo, hi in box)].contiguous() \
                .to(torch.bfloat16).pin_memory()
            self._host_input_bufs[key] = hb
        return hb

    def _h2d_prefetch(self, mb: int) -> None:
        """Host inputs, graph mode: copy microbatch mb's inputs H2D on a copy
        stream into a two-deep staging ring while the previous microbatch
        computes; the ring slot is reused once the copy out of it (two
        microbatches earlier) has run on the compute stream."""
        if self.h2d_stream is None:
            self.h2d_stream = torch.cuda.Stream()
        r = mb % 2
        ev_free = self.h2d_ring_free.get(r)
        for op in self.fwd_ops:
            if op.op != "input":
                continue
            hb = self._host_buf(op, mb)
            dst = self.h2d_ring.get((r, op.nid))
            if dst is None:
                dst = self.h2d_ring[(r, op.nid)] = torch.empty(hb.shape, dtype=hb.dtype,
                                                               device=self.dev)
            if ev_free is not None:
                self.h2d_stream.wait_event(ev_free)
            with torch.cuda.stream(self.h2d_stream):
                dst.copy_(hb, non_blocking=True)
            self.h2d_bytes += hb.numel() * hb.element_size()
        ev = torch.cuda.Event()
        ev.record(self.h2d_stream)
        self.h2d_ready[mb] = (r, ev)

    def _graph_inputs(self, mb: int):
        """Graph mode: stage this microbatch's graph inputs into the slot's
        static buffers (outside the captured region).  Host inputs arrive
        through the prefetched H2D ring (_h2d_prefetch); the next microbatch's
        copy is issued here, so it overlaps this microbatch's compute."""
        vals = self.vals.setdefault(mb, {})
        k = self.slot_of(mb)
        host = self.input_mode == "host"
        if host:
            if mb not in self.h2d_ready:
                self._h2d_prefetch(mb)
            r, ev = self.h2d_ready.pop(mb)
            torch.cuda.current_stream().wait_event(ev)
        for op in self.fwd_ops:
            if op.op != "input":
                continue
            src = self.h2d_ring[(r, op.nid)] if host else self._load_input(mb, op)
            key = ("in", k, op.nid)
            buf = self.static.get(key)
            if buf is None:
                buf = torch.empty_like(src)
                self.static[key] = buf
            buf.copy_(src, non_blocking=True)
            vals[op.nid] = buf
        if host:
            free = torch.cuda.Event()
            free.record(torch.cuda.current_stream())
            self.h2d_ring_free[r] = free
            if mb + 1 < self.plan.num_microbatches:
                self._h2d_prefetch(mb + 1)

    def compute(self, phase: str, mb: int):
        """Run the stage's forward or backward ops for one microbatch: eagerly,
        or (graph mode) by replaying the CUDA graph captured for this
        (phase, slot) — slots = 1F1B in-flight bound, so a slot's activations
        are never live for two microbatches at once."""
        if not self.use_graphs:
            return self._compute_eager(phase, mb)
        self._slot_guard(mb)
        if phase == "fwd":
            self._graph_inputs(mb)
        # the step's first backward overwrites the fp32 gradient buffers (beta = 0)
        # and the others accumulate, so it replays a graph of its own
        first = phase == "bwd" and mb == self.first_bwd_mb
        key = (phase, self.slot_of(mb), first)
        vals = self.vals.setdefault(mb, {})
        g = self.graphs.get(key)
        if g is None:
            before = set(vals)
            g = torch.cuda.CUDAGraph()
            self.join_dw()
            had_out = mb in self.outputs
            self.g_fresh = set(self.gviews) if first else set()
            self._cap_routes = []
            l0 = native.launch_count()
            self._capture(g, lambda: (self._compute_eager(phase, mb, skip_inputs=True),
                                      self.join_dw()))
            # libmpexec kernels in the graph: every replay launches them again
            self.graph_kernels[key] = native.launch_count() - l0
            self.g_fresh = set()
            self.graphs[key] = g
            self.cap_vals[key] = {n: v for n, v in vals.items() if n not in before}
            self.cap_aux[key] = dict(self.aux.get(mb, {}))
            self.cap_routes[key] = self._cap_routes
            if self.keep_outputs and not had_out and mb in self.outputs:
                self.cap_out[key] = self.outputs[mb]      # the slot's static output buffer
            g.replay()
        else:
            vals.update(self.cap_vals[key])
            if self.cap_aux[key]:
                self.aux.setdefault(mb, {}).update(self.cap_aux[key])
            g.replay()
            self.replayed_kernels += self.graph_kernels[key]
        if key in self.cap_out:            # a replay rewrites the buffer: keep a copy
            self.outputs[mb] = self.cap_out[key].clone()
        for gid, route in self.cap_routes.get(key, ()):
            self.routes[(mb, gid)] = route.cpu().numpy()

    def _capture(self, g: "torch.cuda.CUDAGraph", fn) -> None:
        """Capture fn() into g on a side stream.  Unlike torch.cuda.graph() this
        does not synchronize the device first: a capture in a step whose
        peer never sends would otherwise block the host, and the step watchdog
        could not report the deadlock."""
        cur = torch.cuda.current_stream()
        if self.capture_stream is None:
            self.capture_stream = torch.cuda.Stream()
        cs = self.capture_stream
        cs.wait_stream(cur)
        with torch.cuda.stream(cs):
            g.capture_begin(capture_error_mode="thread_local")
            try:
                fn()
            finally:
                g.capture_end()
        cur.wait_stream(cs)

    def _compute_eager(self, phase: str, mb: int, skip_inputs: bool = False):
        vals = self.vals.setdefault(mb, {})
        timer = self.op_timer
        for op in (self.fwd_ops if phase == "fwd" else self.bwd_ops):
            if timer is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record()
                r0 = len(self.relayout_timer)
            n_before = len(vals)
            try:
                if op.op == "input":
                    if skip_inputs:
                        continue
                    out = self._load_input(mb, op)
                elif op.op == "attn_fwd":
                    out = self._run_attn_fwd(mb, op)
                elif op.op == "attn_bwd":
                    out = self._run_attn_bwd(mb, op)
                elif op.op in ("matmul", "bmm"):
                    out = self._run_matmul(mb, op)
                elif self.graph[op.nid].kind == "reshape":
                    out = self._run_reshape(mb, op)
                elif op.op == "reduce_sum":
                    out = native.reduce_mid(self._contig(self._as3(
                        self.get(mb, op.ins[0][0], op.ins[0][1]))))
                else:
                    out = self._run_elementwise(mb, op)
            except native.NativeError as e:
                raise ExecError(f"rank {self.me} stage {self.st.index} {phase}{mb} node "
                                f"{op.nid} ({op.op}): {e}", kind="kernel") from None
            if out is not None:
                vals[op.nid] = out
            if self.pf_learn and not skip_inputs and len(vals) > n_before:
                it = reversed(vals)
                for nid in [next(it) for _ in range(len(vals) - n_before)]:
                    if nid in self.pf_learn:
                        self._prefetch(mb, nid)
            if timer is not None:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record()
                timer.append((phase, op.op, e0, e1, self.relayout_timer[r0:]))

    def recv(self, ins: Instr):
        bd = ins.boundary
        mb = ins.microbatch
        vals = self.vals.setdefault(mb, {})
        outs = []
        for bt in bd.tensors:
            node = self.graph[bt.node]
            if node.kind == KIND_PARAM:               # re-homed weight: resident here
                outs.append(None)
                continue
            dspec = canonical(bt.dst_spec, self.mesh)
            shape = local_dims(node.dims, dspec, self.mesh)
            if self.use_graphs:
                self._slot_guard(mb)
                key = ("recv", self.slot_of(mb), bt.node)
                out = self.static.get(key)
                if out is None:
                    out = torch.empty(shape, dtype=torch.bfloat16, device=self.dev)
                    self.static[key] = out
            else:
                out = torch.empty(shape, dtype=torch.bfloat16, device=self.dev)
            vals[bt.node] = out
            outs.append((out, _lo(device_box(node.dims, dspec, self.mesh, self.me))))
        recvs = []
        for k, t in recvs_of(bd, self.me):
            if outs[k] is None:
                continue
            out, origin = outs[k]
            lo, ext = _lo(_rel(t.box, origin)), _ext(t.box)
            view = native.box_view(out, lo, ext)
            buf = view if view is not None else torch.empty(box_numel(t.box), dtype=torch.bfloat16,
                                                            device=self.dev)
            recvs.append((buf, t.src_device, out, lo, ext, view is None))
        if recvs:
            works = self.comm.p2p([], [(b, s) for b, s, *_ in recvs],
                                  self.comm.boundary_group(bd, self.plan))
            for w in works:
                w.wait()
            for buf, _, out, lo, ext, packed in recvs:
                if packed:
                    native.unpack_box(buf, out, lo, ext)

    def all_gather(self, ins: Instr):
        bd = ins.boundary
        mb = ins.microbatch
        gidx = ins.gather_index
        # locate the tensor owning the gather_index-th gather of this boundary
        k = gidx
        for bt in bd.tensors:
            if k < len(bt.xplan.gathers):
                ga = bt.xplan.gathers[k]
                break
            k -= len(bt.xplan.gathers)
        if self.me not in ga.devices or self.graph[bt.node].kind == KIND_PARAM:
            return
        out = self.vals[mb][bt.node]
        tile_lo = ga.box[0][0]
        rows = [p[0][1] - p[0][0] for p in ga.pieces]
        g = len(ga.devices)
        r = ga.devices.index(self.me)
        grp = self.comm.gather_group(bd, ga.devices)
        flat = out.view(-1)
        row_elems = out.numel() // out.shape[0]
        if all(x == rows[0] for x in rows):
            n = rows[0] * row_elems
            self.comm.all_gather_into(flat, flat[r * n:(r + 1) * n], grp)
        else:
            sends, recvs = [], []
            starts = [p[0][0] - tile_lo for p in ga.pieces]
            mine = flat[starts[r] * row_elems:(starts[r] + rows[r]) * row_elems]
            for q, dev in enumerate(ga.devices):
                if q == r:
                    continue
                if rows[r]:
                    sends.append((mine, dev))
                if rows[q]:
                    recvs.append((flat[starts[q] * row_elems:(starts[q] + rows[q]) * row_elems], dev))
            for w in self.comm.p2p(sends, recvs, grp):
                w.wait()

    def send(self, ins: Instr):
        """Cross-mesh sends run on a dedicated stream (after the compute that
        produced them) so a blocked send never stalls this stage's receives."""
        bd = ins.boundary
        mb = ins.microbatch
        sends = []
        for k, t in sends_of(bd, self.me):
            bt = bd.tensors[k]
            node = self.graph[bt.node]
            if node.kind == KIND_PARAM:               # re-homed to the consumer
                continue
            v = self._as3(self.value(mb, bt.node))
            mine = _lo(device_box(node.dims, self.spec(bt.node), self.mesh, self.me))
            lo, ext = _lo(_rel(t.box, mine)), _ext(t.box)
            view = native.box_view(v, lo, ext)
            sends.append((view if view is not None else native.pack_box(v, lo, ext), t.dst_device))
        if sends:
            self.send_stream.wait_stream(torch.cuda.current_stream())
            rec = getattr(self, "_recording", False)
            ea = torch.cuda.Event(enable_timing=rec)
            eb = torch.cuda.Event(enable_timing=rec)
            ea.record(self.send_stream)
            self.comm.p2p(sends, [], self.comm.boundary_group(bd, self.plan),
                          stream=self.send_stream)
            eb.record(self.send_stream)
            self._send_ev = (ea, eb)
            for buf, _ in sends:
                buf.record_stream(self.send_stream)
            if self.use_graphs:
                # record_stream does not protect graph-pool memory: the slot's
                # next replay waits on this event instead (_slot_guard)
                ev = torch.cuda.Event()
                ev.record(self.send_stream)
                self.slot_send_ev[self.slot_of(mb)] = ev
            self.sends_pending = True

    def free(self, ins: Instr):
        if ins.buffer and ins.buffer.startswith("act"):
            self.vals.pop(ins.microbatch, None)
            self.cache.pop(ins.microbatch, None)
            self.aux.pop(ins.microbatch, None)

    # ------------------------------------------------------------------ optimizer
    def join_dw(self):
        if self.dw_stream is not None and self.dw_pending:
            torch.cuda.current_stream().wait_stream(self.dw_stream)
            self.dw_pending = False

    def reduce_grads(self):
        """Finish the gradient of every parameter: reduce the k-split partial
        sums accumulated over the microbatches (sharding.py:284-291; one
        reduction per step instead of per microbatch, the sum is linear) and
        move them to the parameter's layout.  Gradient all-reduces the plan
        rewrites ZeRO-style (intra.py:404-424) become reduce-scatters into this
        device's optimizer chunk (apply_update all-gathers the new weights)."""
        g = self.graph
        self.join_dw()
        zs = [pid for pid in self.param_ids if pid in self.zero]
        if zs:
            native.group_start()
            try:
                for pid in zs:
                    off, ld = self.pviews[pid]
                    zo, c, _ = self.zchunk[pid]
                    grp = self.comm.axis_group(self.st.index, self.mesh, self.zero[pid], self.me)
                    self.comm.reduce_scatter_into(self.zgrad[zo:zo + c],
                                                  self.gradbuf[off:off + c * len(grp.ranks)], grp)
            finally:
                native.group_end()
        for pid in self.param_ids:
            dw = self.grad_nodes.get(pid)
            if dw is None or pid in self.zero:
                continue
            gv = self.gviews[dw]
            if dw in self.tok_dw:
                # full partial sums over the local tokens: reduce, keep the param's tile
                self._allreduce(gv, self.tok_dw[dw])
                off, ld = self.pviews[pid]
                box = device_box(g[pid].dims, self.spec(pid), self.mesh, self.me)
                native.pack_box(gv, tuple(lo for lo, _ in box), tuple(hi - lo for lo, hi in box),
                                out=self.gradbuf[off:off + math.prod(ld)])
                continue
            algo = matmul_algo(self.bound[dw].op == "bmm", self.spec(dw), self.mesh)
            if algo.k_axes:
                self._allreduce(gv, algo.k_axes)
            if self.spec(dw) != self.spec(pid):
                off, ld = self.pviews[pid]
                moved = self._relayout(gv, g[dw].dims, self.spec(dw), self.spec(pid))
                native.pack_box(moved, (0,) * moved.dim(), tuple(moved.shape),
                                out=self.gradbuf[off:off + math.prod(ld)])

    def apply_update(self):
        """Adam on the plain parameters' full tiles and on the ZeRO chunks, then
        the all-gather half of the rewrite refreshes the replicated bf16 weights."""
        self.step_count += 1
        if not self.n_param:
            return
        a = self.adam
        kw = dict(lr=a.lr, beta1=a.beta1, beta2=a.beta2, eps=a.eps, weight_decay=a.weight_decay,
                  grad_scale=1.0, step=self.step_count)
        n0 = self.n_plain
        if n0:
            native.adam_step(self.master[:n0], self.m[:n0], self.v[:n0], self.gradbuf[:n0],
                             self.wbf16[:n0], **kw)
        if self.n_zero_state:
            native.adam_step(self.master[n0:], self.m[n0:], self.v[n0:], self.zgrad, self.zw, **kw)
            native.group_start()
            try:
                for pid, (zo, c, _) in self.zchunk.items():
                    off, _ = self.pviews[pid]
                    grp = self.comm.axis_group(self.st.index, self.mesh, self.zero[pid], self.me)
                    self.comm.all_gather_into(self.wbf16[off:off + c * len(grp.ranks)],
                                              self.zw[zo:zo + c], grp)
            finally:
                native.group_end()

    def optimizer_step(self):
        self.reduce_grads()
        self.apply_update()

    def zero_grads(self):
        self.join_dw()
        # every dW GEMM's first launch of the step runs with beta = 0 (graph mode:
        # the first backward's own graph was captured that way); the gradbuf
        # regions no dW writes stay at their initial zeros
        self.g_fresh = set() if self.use_graphs else set(self.gviews)

    def local_grad(self, pid: int) -> torch.Tensor:
        """This device's tile of pid's reduced gradient (after reduce_grads)."""
        off, ld = self.pviews[pid]
        if pid in self.zero:
            zo, c, _ = self.zchunk[pid]
            grp = self.comm.axis_group(self.st.index, self.mesh, self.zero[pid], self.me)
            full = torch.empty(c * len(grp.ranks), dtype=torch.float32, device=self.dev)
            self.comm.all_gather_into(full, self.zgrad[zo:zo + c], grp)
            return full.view(ld)
        return self.gradbuf[off:off + math.prod(ld)].view(ld)

    # ------------------------------------------------------------------ step
    def _dispatch(self, ins: Instr, update: bool) -> None:
        if ins.op == "compute":
            self.compute(ins.phase, ins.microbatch)
        elif ins.op == "recv":
            self.recv(ins)
        elif ins.op == "send":
            self.send(ins)
        elif ins.op == "all_gather":
            self.all_gather(ins)
        elif ins.op == "free":
            self.free(ins)
        elif ins.op == "sync":
            if self.sends_pending:
                torch.cuda.current_stream().wait_stream(self.send_stream)
                self.sends_pending = False
            if update:
                self.optimizer_step()

    def run_step(self, *, record: bool = False, update: bool = True):
        """Enqueue the stage's instruction list once.  Returns (t0, t1, events,
        markers): step start / end events, with record=True a timing event pair
        per instruction (sends timed on the send stream), and one completion
        marker per instruction (the watchdog's progress record).  A failing
        instruction raises ExecError naming rank, stage and instruction."""
        self.zero_grads()
        self.loss_acc.zero_()
        events = []
        markers = []
        stream = torch.cuda.current_stream()
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        self._send_ev = None
        for ins in self.sprog.instructions:
            e0 = None
            if record:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            self._recording = record
            try:
                self._dispatch(ins, update)
            except torch.cuda.OutOfMemoryError as e:
                raise ExecError(
                    f"out of memory on device {self.me} (stage {self.st.index}) at {ins.op} "
                    f"{ins.buffer or _label(ins)}: {torch.cuda.memory_allocated(self.dev)} bytes "
                    f"allocated ({str(e).splitlines()[0]})", kind="oom", rank=self.me,
                    stage=self.st.index, instruction=_label(ins)) from None
            except ExecError as e:
                if e.rank is None:
                    e.rank, e.stage, e.instruction = self.me, self.st.index, _label(ins)
                raise
            except native.NativeError as e:
                raise ExecError(f"rank {self.me} stage {self.st.index} at {ins.op} "
                                f"{_label(ins)}: {e}", kind="kernel", rank=self.me,
                                stage=self.st.index, instruction=_label(ins)) from None
            if ins.op == "send" and self._send_ev is not None:
                a, b = self._send_ev
                self._send_ev = None
                if record:
                    events.append((ins, a, b))
                markers.append((ins, b))
                continue
            e1 = torch.cuda.Event(enable_timing=record)
            e1.record(stream)
            if record:
                events.append((ins, e0, e1))
            markers.append((ins, e1))
        self.join_dw()
        if self.pf_stream is not None:
            stream.wait_stream(self.pf_stream)
        t1 = torch.cuda.Event(enable_timing=True)
        t1.record(stream)
        return t0, t1, events, markers


def _label(ins: Instr) -> str:
    if ins.op == "compute":
        return f"{ins.phase}{ins.microbatch}@{ins.stage}"
    if ins.op in ("send", "recv"):
        return ins.tag or ins.op
    return ins.op


class Executor:
    """Public API: one rank's executor for a reference plan.

        ex = Executor("plan.json", schedule="1f1b")
        stats = ex.step()            # one training step (all microbatches + update)
        res = ex.result()            # SimResult-shaped summary of the last step

    Call on every rank (rank = device id of the (1,N) cluster)."""

    def __init__(self, plan, program: Optional[Program] = None, *, schedule: str = GPIPE,
                 params: Optional[dict[int, np.ndarray]] = None,
                 inputs: Optional[Callable[[int, int], np.ndarray]] = None, seed: int = 0,
                 adam: Optional[AdamConfig] = None, host_inputs: bool = False):
        if not torch.cuda.is_available():
            raise ExecError("the executor needs a CUDA device; there is no CPU execution path")
        native.load()
        native.preload_kernels()
        self.plan = plan if isinstance(plan, ExecPlan) else load_plan(plan)
        self.program = program or build_program(self.plan, schedule)
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        if self.world != self.plan.num_devices:
            raise ExecError(f"plan needs {self.plan.num_devices} devices, running on {self.world}")
        self.comm = Comm(self.plan, self.program, self.rank, self.world)
        try:
            self.runner = StageRunner(self.plan, self.program, self.rank, self.comm, seed=seed,
                                      params=params, inputs=inputs, adam=adam,
                                      host_inputs=host_inputs)
        except torch.cuda.OutOfMemoryError as e:
            st = self.plan.stage_of_device(self.rank).index
            raise ExecError(f"out of memory on device {self.rank} (stage {st}) at init "
                            f"(parameters and optimizer state): {str(e).splitlines()[0]}",
                            kind="oom", rank=self.rank, stage=st, instruction="init") from None
        self.step_times: list[float] = []
        self.last_events: list = []

    def barrier(self):
        if self.world > 1:
            dist.barrier(group=self.comm.world_group)

    def step(self, *, record: bool = False, update: bool = True,
             timeout: Optional[float] = None) -> float:
        """One step; returns this rank's device time (seconds).  The host waits
        for the device under a watchdog: past `timeout` seconds (default
        MPEXEC_STEP_TIMEOUT_S) the communicators are aborted and ExecError
        (kind "deadlock") names the first instruction that has not completed;
        an asynchronous NCCL failure raises ExecError (kind "nccl")."""
        t0, t1, evs, markers = self.runner.run_step(record=record, update=update)
        self._wait(t1, markers, STEP_TIMEOUT_S if timeout is None else timeout)
        dt = t0.elapsed_time(t1) * 1e-3
        self.step_times.append(dt)
        if record:
            self.last_events = [(ins, t0.elapsed_time(a) * 1e-3, t0.elapsed_time(b) * 1e-3)
                                for ins, a, b in evs]
        return dt

    def _wait(self, done: torch.cuda.Event, markers, timeout: float) -> None:
        if done.query():
            return
        start = time.monotonic()
        nap, last_poll = 5e-5, start
        while not done.query():
            time.sleep(nap)
            nap = min(nap * 2, 2e-3)
            now = time.monotonic()
            if self.comm.enabled and now - last_poll > 1.0:
                last_poll = now
                bad = self.comm.async_errors()
                if bad:
                    ins = self._first_pending(markers)
                    self.comm.abort()
                    raise ExecError(f"NCCL failure on rank {self.rank} (stage "
                                    f"{self.runner.st.index}) at {_describe(ins)}: "
                                    + "; ".join(bad), kind="nccl", rank=self.rank,
                                    stage=self.runner.st.index,
                                    instruction=_label(ins) if ins else None)
            if now - start > timeout:
                ins = self._first_pending(markers)
                self.comm.abort()
                raise ExecError(f"deadlock: rank {self.rank} stage {self.runner.st.index} "
                                f"waiting on {_describe(ins)} after {timeout:.0f} s",
                                kind="deadlock", rank=self.rank, stage=self.runner.st.index,
                                instruction=_label(ins) if ins else None)
        done.synchronize()

    @staticmethod
    def _first_pending(markers):
        for ins, ev in markers:
            if not ev.query():
                return ins
        return None

    def loss(self) -> float:
        loss = self.runner.loss_acc.clone()
        if self.world > 1:
            dist.all_reduce(loss, group=self.comm.world_group)
        return 0.5 * float(loss.item())

    def max_over_ranks(self, x: float) -> float:
        if self.world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=self.runner.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.comm.world_group)
        return float(t.item())

    def result(self, grads=None, outputs=None, launches: int = 0) -> ExecResult:
        """SimResult-shaped summary of the last step, gathered over all ranks
        (sim.py:39-44): utilization of every stage (its first device's busy
        compute / send / all_gather time over the makespan), the allocator
        peak of every device, and every stage's instruction events (measured
        from the step start, which a barrier aligns across ranks), sorted like
        the simulator's (start, stage, end, label)."""
        makespan = self.max_over_ranks(self.step_times[-1]) if self.step_times else 0.0
        evs = self.last_events
        st = self.runner.st
        mine = {"rank": self.rank, "stage": st.index,
                "leader": self.rank == min(st.mesh.device_ids),
                "events": [(ins.stage, ins.op, _label(ins), s, e) for ins, s, e in evs],
                "busy": sum(e - s for ins, s, e in evs if ins.op in BUSY_OPS),
                "peak": int(torch.cuda.max_memory_allocated())}
        parts = [mine]
        if self.world > 1:
            parts = [None] * self.world
            dist.all_gather_object(parts, mine, group=self.comm.world_group)
        util, peak, events = {}, {}, []
        for p in parts:
            peak[p["rank"]] = p["peak"]
            if p["leader"]:
                util[p["stage"]] = p["busy"] / makespan if makespan > 0 else 0.0
                events += [ExecEvent(*e) for e in p["events"]]
        events.sort(key=lambda e: (e.start, e.stage, e.end, e.label))
        r = self.runner
        return ExecResult(makespan=makespan, utilization=util, peak_bytes=peak, events=events,
                          modeled_makespan=float(modeled_makespan(self.program, self.plan)),
                          t_star=float(self.program.t_star),
                          loss=self.loss(), step_times=list(self.step_times), grads=grads,
                          outputs=outputs, gpu_launches=launches,
                          fused={"attention": len(r.attn_clusters),
                                 "attention_key_split": sum(1 for c in r.attn_clusters
                                                            if c["key_axes"]),
                                 "epilogues": r.fused_epilogues,
                                 "local_conv": len(r.local_conv),
                                 "token_split_dw": len(r.tok_dw)})


def _describe(ins: Optional[Instr]) -> str:
    if ins is None:
        return "the step's end"
    return f"{ins.op} {ins.tag or ins.buffer or _label(ins)}"


def execute(plan, program: Optional[Program] = None, *, schedule: str = GPIPE, steps: int = 1,
            params: Optional[dict[int, np.ndarray]] = None,
            inputs: Optional[Callable[[int, int], np.ndarray]] = None,
            seed: int = 0, adam: Optional[AdamConfig] = None, record: bool = True,
            collect: bool = False, update: bool = True, device_memory: Optional[int] = None,
            enforce_memory: bool = True, timeout: Optional[float] = None) -> ExecResult:
    """Run `steps` training steps of a reference plan on this process's GPU.

    The drop-in for `simulate(emit_instructions(plan, schedule), ...)`: call on
    every rank (torch.distributed initialised, rank = device id).  `params` /
    `inputs` (global fp32 arrays, identical on every rank) make runs reproducible
    against the CPU oracle; by default weights and inputs are synthetic (seeded).
    With collect=True the result carries the global parameter gradients of the
    last step (before its update) and the forward outputs.

    Errors (the simulator's contract, sim.py:152-178): device_memory (bytes;
    default: none beyond the GPU's own) caps this process's CUDA allocator when
    enforce_memory is set, and any allocation past it raises ExecError kind
    "oom" naming the device, stage and instruction; a step that does not finish
    within `timeout` seconds raises kind "deadlock" naming the instruction the
    stage is blocked on."""
    capped = device_memory is not None and enforce_memory and torch.cuda.is_available()
    if capped:
        total = torch.cuda.get_device_properties(torch.cuda.current_device()).total_memory
        torch.cuda.set_per_process_memory_fraction(min(1.0, device_memory / total))
    try:
        return _execute(plan, program, schedule, steps, params, inputs, seed, adam, record,
                        collect, update, timeout)
    finally:
        if capped:
            torch.cuda.set_per_process_memory_fraction(1.0)


def _execute(plan, program, schedule, steps, params, inputs, seed, adam, record, collect, update,
             timeout) -> ExecResult:
    ex = Executor(plan, program, schedule=schedule, params=params, inputs=inputs, seed=seed,
                  adam=adam)
    ex.runner.keep_outputs = collect
    launches0 = native.launch_count()
    grads = None
    for step in range(steps):
        last = step == steps - 1
        ex.barrier()
        torch.cuda.synchronize()
        ex.step(record=record and last, update=update and not (collect and last),
                timeout=timeout)
        if last and collect:
            ex.runner.reduce_grads()
            grads = _collect_grads(ex.runner, ex.comm, ex.world)
            if update:
                ex.runner.apply_update()
    outputs = _collect_outputs(ex.runner, ex.comm, ex.world) if collect else None
    res = ex.result(grads=grads, outputs=outputs, launches=native.launch_count() - launches0)
    if collect:
        parts = [ex.runner.routes]
        if ex.world > 1:
            parts = [None] * ex.world
            dist.all_gather_object(parts, ex.runner.routes, group=ex.comm.world_group)
        res.routes = {k: v for p in parts for k, v in p.items()}
    return res


def _gather_global(runner: StageRunner, comm: Comm, world: int, items: dict) -> dict:
    """items: key -> (global dims, local fp32 tensor, global box) on this rank.
    Returns key -> assembled global np array (on every rank)."""
    local = {k: (dims, t.detach().float().cpu().numpy(), box) for k, (dims, t, box) in items.items()}
    allparts = [local]
    if world > 1:
        allparts = [None] * world
        dist.all_gather_object(allparts, local, group=comm.world_group)
    out: dict = {}
    for part in allparts:
        for k, (dims, arr, box) in part.items():
            if k not in out:
                out[k] = np.zeros(dims, dtype=np.float32)
            out[k][tuple(slice(lo, hi) for lo, hi in box)] = arr
    return out


def _collect_grads(runner: StageRunner, comm: Comm, world: int) -> dict[int, np.ndarray]:
    """Global parameter gradients after reduce_grads (before the update)."""
    g = runner.graph
    items = {}
    for pid in runner.param_ids:
        if runner.grad_nodes.get(pid) is None:
            continue
        box = device_box(g[pid].dims, runner.spec(pid), runner.mesh, runner.me)
        items[pid] = (g[pid].dims, runner.local_grad(pid), box)
    return _gather_global(runner, comm, world, items)


def _collect_outputs(runner: StageRunner, comm: Comm, world: int) -> dict[int, np.ndarray]:
    items = {}
    for sid in runner.seed_ids:
        y = runner.graph[sid].inputs[0]
        dims = runner.graph[y].dims
        box = device_box(dims, runner.spec(sid), runner.mesh, runner.me)
        for mb, t in runner.outputs.items():
            items[(mb, y)] = (dims, t.view(*[hi - lo for lo, hi in box]), box)
    return _gather_global(runner, comm, world, items)
