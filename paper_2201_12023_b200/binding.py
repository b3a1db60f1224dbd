"""Numeric binding of the reference IR.

The reference IR carries no op semantics (SURVEY §7 hard part 1): ELEMENTWISE has
no function, RESHAPE need not preserve element counts (graph.py:240-245) and the
backward graph is a structural mirror (graph.py:317-366).  The executor fixes
one binding, derived only from graph structure, so any plan of any builder graph
gets a well-defined computation:

forward (colocate_with is None)
  input            graph input (one synthetic microbatch)
  parameter        weight
  matmul / bmm     y = a @ b                                    (graph.py:187-188)
  elementwise(a)   softmax(x / sqrt(d)) over the last dim when a is a bmm of
                   two activations (the attention probabilities, graph.py:300);
                   tanh-GeLU otherwise (the MLP activation, graph.py:262,308)
  elementwise(a,b) a + b                                        (residual, graph.py:305,311)
  reshape 2D->3D   attention head split (T,h) -> (B*H, s, d); when it feeds the
                   rhs of a bmm whose lhs is also a head split it is the
                   key-transposed split (B*H, d, s) (graph.py:297-299)
  reshape 3D->2D   head merge (B*H, s, d) -> (T, h)                (graph.py:302)
  reshape reversing dims: transpose; same dims: identity
  MoE layout adapters (builders.build_moe; no reference builder):
  elementwise(a) feeding them          softmax over the experts (the gates)
  reshape gates (T,E) -> (G, E*C, S)   dispatch mask: 1 at each token's routed
                                       (expert, slot), GShard top-2 routing in
                                       groups of S tokens, capacity C (csrc/moe.cu)
  reshape gates (T,E) -> (G, S, E*C)   combine weights: the gate at the same slots
  reshape of a bmm output, 3D -> 3D    regroup (A, B, h) -> (P, Q, h), C = B/P:
                                       out[p, a*C + c] = in[a, p*C + c]
                                       (group-major <-> expert-major, the all-to-all)
backward of the adapters
  combine                              (T,E) gradient = the incoming gradient at the
                                       routed slots (routing is piecewise constant)
  dispatch                             zero: the 0/1 mask is piecewise constant (the
                                       bmm producing its input still runs, as planned)
  regroup                              regroup back
Wide-ResNet adapters (builders.build_wide_resnet; N = images, from the pooling view):
  reshape (N*H*W, C) -> (N*Ho*Wo, k*k*C)   im2col, k x k window, stride s = H/Ho, pad k/2
  reshape (N*H*W, C) -> (N*Ho*Wo, C)       subsample (stride-s shortcut, stem pool)
  reduction                                sum over the axis (global pooling); its
                                           backward reshape broadcasts
  backward: col2im (the adjoint of im2col), subsample_grad (scatter into zeros)
backward (colocate_with = f)
  elementwise(out), colocated with out       loss seed dL/dy = y   (L = 1/2 |y|^2)
  elementwise(g) colocated with unary f       f'(x) * g (GeLU) / softmax backward
  elementwise(g) colocated with binary f      g (the add's grad, shared by both operands)
  elementwise(g1, g2)                         g1 + g2 (gradient accumulation, graph.py:328-332)
  reshape colocated with a matmul/bmm         operand transpose (graph.py:341-352)
  reshape colocated with a forward reshape r  inverse of r (graph.py:362-365)
  matmul / bmm                                dX = g @ W^T, dW = x^T @ g (grad_of tags dW)
The same table is restated independently in oracle/ (the CPU checker).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

from .plan import (Graph, HEAVY, KIND_BMM, KIND_ELEM, KIND_INPUT, KIND_MATMUL, KIND_PARAM,
                   KIND_RED, KIND_RESHAPE, PlanError)


@dataclass(frozen=True)
class Bound:
    op: str                       # semantic op code (see module doc)
    # head geometry for split / merge reshapes: (B, H, s, d)
    heads: Optional[tuple[int, int, int, int]] = None
    # node whose forward tensor the op reads besides its inputs (gelu_bwd / softmax_bwd)
    fwd_ref: Optional[int] = None
    softmax_scale: float = 1.0
    # MoE routing geometry (G, S, E, C) of dispatch / combine and their gradients
    route: Optional[tuple[int, int, int, int]] = None
    # regroup geometry (A, P, C): (A, P*C, h) -> (P, A*C, h)
    regroup: Optional[tuple[int, int, int]] = None
    # Wide-ResNet adapters (N, H, W, C, k, s): im2col / subsample of NHWC rows
    conv: Optional[tuple[int, int, int, int, int, int]] = None


def _head_geom(two_d: tuple[int, int], three_d: tuple[int, int, int],
               transposed: bool) -> tuple[int, int, int, int]:
    T, h = two_d
    X, Y, Z = three_d
    s, d = (Z, Y) if transposed else (Y, Z)
    if X * s * d != T * h or T % s or h % d:
        raise PlanError(f"reshape {two_d} <-> {three_d} is not a head split/merge")
    B, H = T // s, h // d
    if B * H != X:
        raise PlanError(f"reshape {two_d} <-> {three_d}: batch*heads mismatch")
    return (B, H, s, d)


def image_batch(graph: Graph) -> Optional[int]:
    """Images per microbatch of a convolutional graph: the leading dim of the
    (N, H*W, C) view its pooling reduction sums over (builders.build_wide_resnet),
    or the plan's `image_batch` hint for a stage sub-graph without the head."""
    if getattr(graph, "image_batch", None):
        return graph.image_batch
    for n in graph.nodes:
        if n.kind == KIND_RED and n.colocate_with is None:
            src = graph[n.inputs[0]]
            if len(src.dims) == 3:
                return src.dims[0]
    return None


def conv_geom(ind, outd, batch: Optional[int]):
    """(op, (N, H, W, C, k, s)) for a 2-D -> 2-D count-changing reshape of NHWC rows:
    im2col (columns x k*k, odd k) or subsample (same columns)."""
    if batch is None:
        return None
    (ri, ci), (ro, co) = ind, outd
    if ri % batch or ro % batch or co % ci:
        return None
    H, Ho = math.isqrt(ri // batch), math.isqrt(ro // batch)
    k = math.isqrt(co // ci)
    if H * H * batch != ri or Ho * Ho * batch != ro or k * k * ci != co or k % 2 == 0 or Ho > H:
        return None
    s = max(1, H // Ho)
    if (H + 2 * (k // 2) - k) // s + 1 != Ho:
        return None
    return ("subsample" if k == 1 else "im2col"), (batch, H, H, ci, k, s)


def bind(graph: Graph) -> dict[int, Bound]:
    out: dict[int, Bound] = {}
    cons = graph.consumers()
    batch = image_batch(graph)
    for n in graph.nodes:
        fwd = n.colocate_with is None
        if n.kind == KIND_INPUT:
            out[n.id] = Bound("input")
        elif n.kind == KIND_PARAM:
            out[n.id] = Bound("param")
        elif n.kind in HEAVY:
            out[n.id] = Bound("matmul" if n.kind == KIND_MATMUL else "bmm")
        elif n.kind == KIND_RED:
            out[n.id] = Bound("reduce_sum" if fwd else "broadcast")
        elif n.kind == KIND_ELEM:
            out[n.id] = _bind_elementwise(graph, n, out, cons)
        elif n.kind == KIND_RESHAPE:
            out[n.id] = _bind_reshape(graph, n, out, cons, batch)
        else:
            raise PlanError(f"node {n.id}: unknown kind {n.kind}")
    return out


def routing_geom(graph: Graph, r, cons) -> Optional[tuple[str, tuple[int, int, int, int]]]:
    """("dispatch" | "combine", (G, S, E, C)) when forward reshape `r` turns MoE
    gates (a unary forward elementwise of shape (T, E)) into a routing tensor."""
    if r.kind != KIND_RESHAPE or r.colocate_with is not None:
        return None
    src = graph[r.inputs[0]]
    if src.kind != KIND_ELEM or src.colocate_with is not None or len(src.inputs) != 1:
        return None
    if len(src.dims) != 2 or len(r.dims) != 3:
        return None
    if not any(graph[c].kind == KIND_BMM and slot == 0 for c, slot in cons[r.id]):
        return None
    T, E = src.dims
    X, Y, Z = r.dims
    disp = X * Z == T and Y % E == 0
    comb = X * Y == T and Z % E == 0
    if disp and comb:
        raise PlanError(f"node {r.id}: routing reshape {src.dims} -> {r.dims} is ambiguous")
    if disp:
        return "dispatch", (X, Z, E, Y // E)
    if comb:
        return "combine", (X, Y, E, Z // E)
    raise PlanError(f"node {r.id}: reshape of gates {src.dims} -> {r.dims} has no binding")


def _bind_elementwise(graph: Graph, n, bound: dict[int, Bound], cons) -> Bound:
    if n.colocate_with is None:
        if len(n.inputs) == 1:
            src = graph[n.inputs[0]]
            if any(routing_geom(graph, graph[c], cons) is not None for c, _ in cons[n.id]):
                return Bound("softmax", softmax_scale=1.0)       # MoE gates
            if src.kind == KIND_BMM and graph[src.inputs[1]].kind != KIND_PARAM:
                d = graph[src.inputs[0]].dims[-1]       # contraction length of q @ k^T
                return Bound("softmax", softmax_scale=1.0 / float(d) ** 0.5)
            return Bound("gelu")
        if len(n.inputs) == 2:
            return Bound("add")
        raise PlanError(f"node {n.id}: elementwise of arity {len(n.inputs)} has no binding")
    f = graph[n.colocate_with]
    if len(n.inputs) == 1 and n.inputs[0] == n.colocate_with and f.colocate_with is None:
        return Bound("seed")
    if len(n.inputs) == 2:
        return Bound("add")
    if len(n.inputs) != 1:
        raise PlanError(f"node {n.id}: backward elementwise arity {len(n.inputs)}")
    fb = bound[f.id]
    if fb.op == "gelu":
        return Bound("gelu_bwd", fwd_ref=f.inputs[0])
    if fb.op == "softmax":
        return Bound("softmax_bwd", fwd_ref=f.id, softmax_scale=fb.softmax_scale)
    if fb.op == "add":
        return Bound("identity")
    raise PlanError(f"node {n.id}: no backward binding for forward op {fb.op}")


def _bind_reshape(graph: Graph, n, bound: dict[int, Bound], cons, batch=None) -> Bound:
    src = graph[n.inputs[0]]
    ind, outd = src.dims, n.dims
    if n.colocate_with is not None:
        f = graph[n.colocate_with]
        if f.kind in HEAVY:
            return Bound("transpose")
        if f.kind == KIND_RESHAPE:
            fb = bound[f.id]
            if fb.op in ("dispatch", "combine"):
                return Bound(fb.op + "_grad", route=fb.route, fwd_ref=f.inputs[0])
            if fb.op == "regroup":
                A, P, C = fb.regroup
                return Bound("regroup", regroup=(P, A, C))
            if fb.op in ("im2col", "subsample"):
                return Bound("col2im" if fb.op == "im2col" else "subsample_grad", conv=fb.conv)
            inverse = {"split": "merge", "split_t": "merge_t", "merge": "split",
                       "merge_t": "split_t", "transpose": "transpose", "identity": "identity"}
            op = inverse[fb.op]
            return Bound(op, heads=fb.heads)
        if f.kind == KIND_RED:
            return Bound("broadcast")
        raise PlanError(f"node {n.id}: backward reshape colocated with {f.kind}")
    rg = routing_geom(graph, n, cons)
    if rg is not None:
        return Bound(rg[0], route=rg[1])
    if len(ind) == 3 and len(outd) == 3 and src.kind == KIND_BMM:
        A, B, h = ind
        P, Q, h2 = outd
        if h != h2 or B % P or Q != A * (B // P):
            raise PlanError(f"node {n.id}: reshape {ind} -> {outd} is not a regroup")
        return Bound("regroup", regroup=(A, P, B // P))
    if len(ind) == 2 and len(outd) == 3:
        transposed = False
        for c, slot in cons[n.id]:
            cn = graph[c]
            lhs = graph[cn.inputs[0]]
            if cn.kind == KIND_BMM and slot == 1 and lhs.kind == KIND_RESHAPE and \
                    routing_geom(graph, lhs, cons) is None:
                transposed = True
        return Bound("split_t" if transposed else "split",
                     heads=_head_geom(ind, outd, transposed))
    if len(ind) == 3 and len(outd) == 2:
        return Bound("merge", heads=_head_geom(outd, ind, False))
    if ind == outd:
        return Bound("identity")
    if len(ind) >= 2 and outd == ind[:-2] + (ind[-1], ind[-2]):
        return Bound("transpose")
    if len(ind) == 2 and len(outd) == 2:
        cg = conv_geom(ind, outd, batch)
        if cg is not None:
            return Bound(cg[0], conv=cg[1])
    raise PlanError(f"node {n.id}: reshape {ind} -> {outd} has no binding")
