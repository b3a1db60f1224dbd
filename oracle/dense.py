"""Dense single-device interpreter of a bound graph (test infrastructure only).

Every node is evaluated on the full (global) tensor in float64, in node-id
order (forward nodes precede the structural backward, graph.py:317-366).
"""
from __future__ import annotations

import numpy as np

from . import ir


def gelu(x):
    k0, k1 = 0.7978845608028654, 0.044715
    return 0.5 * x * (1.0 + np.tanh(k0 * (x + k1 * x ** 3)))


def gelu_grad(x):
    k0, k1 = 0.7978845608028654, 0.044715
    t = np.tanh(k0 * (x + k1 * x ** 3))
    return 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * k0 * (1 + 3 * k1 * x * x)


def softmax(x, scale):
    z = scale * x
    z = z - z.max(axis=-1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=-1, keepdims=True)


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


def eval_node(code, info, n, args, val):
    """args: input values in slot order; val: all values (for forward refs)."""
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
    if code == "softmax_bwd":
        y = val[info[0]]
        g = args[0]
        return info[1] * y * (g - (g * y).sum(axis=-1, keepdims=True))
    return reshape_op(code, info, args[0])


def run(plan_doc, params, inputs, num_microbatches, dtype=np.float64):
    """-> (loss, grads{param id: array}, outputs{mb: array}) in `dtype`."""
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
            val[nid] = eval_node(code, info, n, args, val)
            if code == "seed":
                y = val[nid]
                loss += 0.5 * float((y * y).sum())
                outputs[mb] = y
            g = n.get("grad_of")
            if g is not None:
                grads[g] = grads.get(g, 0.0) + val[nid]
    return loss, grads, outputs
