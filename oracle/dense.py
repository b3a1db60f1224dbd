"""Dense single-device interpreter of a bound graph (test infrastructure only).

Every node is evaluated on the full (global) tensor in float64, in node-id
order (forward nodes precede the structural backward, graph.py:317-366).
"""
from __future__ import annotations

import numpy as np

from . import ir


def gelu(x):
    k0, k1 = 0.7978845608028654, 0.044715
    x2 = x * x
    return 0.5 * x * (1.0 + np.tanh(k0 * x * (1.0 + k1 * x2)))


def gelu_grad(x):
    k0, k1 = 0.7978845608028654, 0.044715
    x2 = x * x
    t = np.tanh(k0 * x * (1.0 + k1 * x2))
    return 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * k0 * (1 + 3 * k1 * x2)


def softmax(x, scale):
    z = scale * x
    z = z - z.max(axis=-1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=-1, keepdims=True)


def route(gates, G, S, E, C):
    """GShard top-2 routing per group of S tokens, capacity C (the rule in the
    product's csrc/moe.cu header, restated): list of (t, e, slot) kept pairs."""
    pairs = []
    g2 = np.asarray(gates, np.float64).reshape(G, S, E)
    for g in range(G):
        x = g2[g]
        e1 = x.argmax(axis=1)                      # first maximum = lowest index
        x2 = x.copy()
        x2[np.arange(S), e1] = -np.inf
        e2 = x2.argmax(axis=1)
        seen = np.zeros(E, np.int64)
        pos1 = np.empty(S, np.int64)
        for s in range(S):
            pos1[s] = seen[e1[s]]
            seen[e1[s]] += 1
        fill = np.minimum(seen, C)
        for s in range(S):
            if pos1[s] < C:
                pairs.append((g * S + s, int(e1[s]), int(pos1[s])))
        for s in range(S):
            p = fill[e2[s]]
            fill[e2[s]] += 1
            if p < C:
                pairs.append((g * S + s, int(e2[s]), int(p)))
    return pairs


def pairs_of(route_table):
    """(T, 4) {e1, pos1|-1, e2, pos2|-1} table (the executor's) -> kept pairs."""
    r = np.asarray(route_table)
    return [(t, int(r[t, 2 * k]), int(r[t, 2 * k + 1]))
            for k in (0, 1) for t in range(r.shape[0]) if r[t, 2 * k + 1] >= 0]


def routing_op(code, info, x, gates=None, pairs=None):
    """pairs: routing decisions to replay instead of deciding from the gates."""
    if code in ("dispatch", "combine"):
        G, S, E, C = info
        out = np.zeros((G, E * C, S) if code == "dispatch" else (G, S, E * C), x.dtype)
        for t, e, c in (route(x, G, S, E, C) if pairs is None else pairs):
            g, s = divmod(t, S)
            if code == "dispatch":
                out[g, e * C + c, s] = 1.0
            else:
                out[g, s, e * C + c] = x[t, e]
        return out
    (G, S, E, C), _ = info
    out = np.zeros((G * S, E), x.dtype)
    if code == "combine_grad":               # dispatch_grad: the 0/1 mask has none
        for t, e, c in (route(gates, G, S, E, C) if pairs is None else pairs):
            g, s = divmod(t, S)
            out[t, e] = x[g, s, e * C + c]
    return out


def regroup(info, x):
    A, P, C = info
    h = x.shape[-1]
    return x.reshape(A, P, C, h).transpose(1, 0, 2, 3).reshape(P, A * C, h)


def conv_op(code, info, x):
    """Wide-ResNet adapters on NHWC rows (restating csrc/conv.cu's contract)."""
    N, H, W, C, k, s = info
    p = k // 2
    Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    if code == "subsample":
        return x.reshape(N, H, W, C)[:, ::s, ::s][:, :Ho, :Wo].reshape(N * Ho * Wo, C)
    if code == "subsample_grad":
        out = np.zeros((N, H, W, C), x.dtype)
        out[:, ::s, ::s][:, :Ho, :Wo] = x.reshape(N, Ho, Wo, C)
        return out.reshape(N * H * W, C)
    if code == "im2col":
        xp = np.zeros((N, H + 2 * p, W + 2 * p, C), x.dtype)
        xp[:, p:p + H, p:p + W] = x.reshape(N, H, W, C)
        cols = np.empty((N, Ho, Wo, k, k, C), x.dtype)
        for ky in range(k):
            for kx in range(k):
                cols[:, :, :, ky, kx] = xp[:, ky:ky + s * Ho:s, kx:kx + s * Wo:s]
        return cols.reshape(N * Ho * Wo, k * k * C)
    # col2im: the adjoint of im2col
    d = x.reshape(N, Ho, Wo, k, k, C)
    xp = np.zeros((N, H + 2 * p, W + 2 * p, C), x.dtype)
    for ky in range(k):
        for kx in range(k):
            xp[:, ky:ky + s * Ho:s, kx:kx + s * Wo:s] += d[:, :, :, ky, kx]
    return xp[:, p:p + H, p:p + W].reshape(N * H * W, C)


def reshape_op(code, heads, x):
    if code == "identity":
        return x
    if code == "transpose":
        return np.swapaxes(x, -1, -2)
    B, H, s, d = heads
    if code == "split":
        return x.reshape(B, s, H, d).transpose(0, 2, 1, 3).reshape(B * H, s, d)
    if code == "split_t":
        return x.reshape(B, s, H, d).transpose(0, 2, 3, 1).reshape(B * H, d, s)
    if code == "merge":
        return x.reshape(B, H, s, d).transpose(0, 2, 1, 3).reshape(B * s, H * d)
    if code == "merge_t":
        return x.reshape(B, H, d, s).transpose(0, 3, 1, 2).reshape(B * s, H * d)
    raise ValueError(code)


def eval_node(code, info, n, args, val, pairs=None):
    """args: input values in slot order; val: all values (for forward refs);
    pairs: replayed MoE routing for routing ops (None: decide from the gates)."""
    if code in ("matmul", "batched_matmul"):
        return args[0] @ args[1]
    if code == "gelu":
        return gelu(args[0])
    if code == "softmax":
        return softmax(args[0], info)
    if code == "add":
        return args[0] + args[1]
    if code in ("seed", "identity"):
        return args[0]
    if code == "gelu_bwd":
        return gelu_grad(val[info]) * args[0]
    if code in ("dispatch", "combine"):
        return routing_op(code, info, args[0], pairs=pairs)
    if code in ("dispatch_grad", "combine_grad"):
        return routing_op(code, info, args[0], val[info[1]], pairs=pairs)
    if code == "regroup":
        return regroup(info, args[0])
    if code in ("im2col", "col2im", "subsample", "subsample_grad"):
        return conv_op(code, info, args[0])
    if code == "reduce_sum":
        return args[0].sum(axis=info)
    if code == "broadcast":
        shape = tuple(n["shape"]["dims"])
        return np.broadcast_to(np.expand_dims(args[0], 1), shape).copy()
    if code == "softmax_bwd":
        y = val[info[0]]
        g = args[0]
        return info[1] * y * (g - (g * y).sum(axis=-1, keepdims=True))
    return reshape_op(code, info, args[0])


def run(plan_doc, params, inputs, num_microbatches, dtype=np.float64, trace=None, routes=None):
    """-> (loss, grads{param id: array}, outputs{mb: array}) in `dtype`.
    trace: optional {node id: []}; each listed node's value is appended per
    microbatch.  routes: optional {(microbatch, gates node): (T, 4) table} of
    MoE routing decisions to replay (the executor's, see ExecResult.routes)."""
    doc, nodes, _ = ir.load(plan_doc)
    bound = ir.bind(nodes)
    grads = {}
    outputs = {}
    loss = 0.0
    for mb in range(num_microbatches):
        val = {}
        for n in nodes:
            nid = n["id"]
            code, info = bound[nid]
            if code == "input":
                val[nid] = np.asarray(inputs(mb, nid), dtype=dtype)
                continue
            if code == "parameter":
                val[nid] = np.asarray(params[nid], dtype=dtype)
                continue
            args = [val[p] for p in ir.node_inputs(n)]
            pairs = None
            if routes is not None and code in ("dispatch", "combine", "dispatch_grad",
                                               "combine_grad"):
                gid = ir.node_inputs(n)[0] if code in ("dispatch", "combine") else info[1]
                pairs = pairs_of(routes[(mb, gid)])
            val[nid] = eval_node(code, info, n, args, val, pairs)
            if trace is not None and nid in trace:
                trace[nid].append(val[nid])
            if code == "seed":
                y = val[nid]
                loss += 0.5 * float((y * y).sum())
                outputs[mb] = y
            g = n.get("grad_of")
            if g is not None:
                grads[g] = grads.get(g, 0.0) + val[nid]
    return loss, grads, outputs
