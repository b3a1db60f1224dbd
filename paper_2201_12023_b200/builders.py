"""Graph builders for the models the reference cannot express yet.

The reference ships two builders (`build_mlp`, `build_transformer_blocks`,
graph.py:251-314).  Configs 3 and 4 of BASELINE.json (GShard MoE, Wide-ResNet)
have none, so they cannot be planned.  These builders extend the reference's
own IR with its own node constructors (`graph._Builder`, graph.py:191-245) and
its own structural backward (`graph._append_backward`, graph.py:317-366); they
emit the reference's graph JSON (`graph.serialize`, graph.py:397-416), which the
unmodified planner reads with `meshplan plan --graph FILE` (cli.py:76-84).

They are planner-side code: they import `meshplan` (the reference), which is
only needed where plans are made.  The executor consumes the resulting plans
like any other; `binding.py` gives every node below its numeric meaning.

GShard MoE block (`moe=1`), T = G*S tokens in G groups of S, E experts,
capacity C = 2*S/E (top-2 routing, capacity factor 1):

    logits = x @ Wg                      (T, E)            matmul
    gates  = elementwise(logits)         softmax over E
    dmask  = reshape(gates, (G, E*C, S)) dispatch mask     (layout adapter)
    cmask  = reshape(gates, (G, S, E*C)) combine weights   (layout adapter)
    xg     = reshape(x, (G, S, h))       group split
    xd     = bmm(dmask, xg)              (G, E*C, h)       dispatch einsum
    xe     = reshape(xd, (E, G*C, h))    group -> expert   (the all-to-all)
    h1     = bmm(xe, W1[E, h, F]); a = elementwise(h1); h2 = bmm(a, W2[E, F, h])
    yd     = reshape(h2, (G, E*C, h))    expert -> group   (the all-to-all back)
    y      = bmm(cmask, yd)              (G, S, h)         combine einsum
    out    = elementwise(reshape(y, (T, h)), x)            residual

This is GShard's dense-einsum formulation (arXiv 2006.16668 Alg. 1): dispatch
and combine are batched matmuls over groups, the experts a batched matmul
over E.  Reshape is the IR's free layout adapter whose element count need not
match (graph.py:241-243), so the masks are reshapes of the gates.
"""
from __future__ import annotations

import json
from typing import Optional


def _meshplan_graph():
    try:
        from meshplan import graph as G  # the reference planner's IR
    except ImportError as e:  # pragma: no cover - planner-side only
        raise ImportError("builders need the reference planner (meshplan) on sys.path; "
                          "plans are made where /root/reference is mounted") from e
    return G


def _attention(b, G, cur, batch: int, seq: int, hidden: int, heads: int, eb: int) -> int:
    """Self-attention + residual, node for node as build_transformer_blocks
    (graph.py:290-305)."""
    TS = G.TensorShape
    hd = hidden // heads
    tokens = batch * seq
    wq = b.parameter(TS((hidden, hidden), eb))
    wk = b.parameter(TS((hidden, hidden), eb))
    wv = b.parameter(TS((hidden, hidden), eb))
    q = b.matmul(cur, wq)
    k = b.matmul(cur, wk)
    v = b.matmul(cur, wv)
    qh = b.reshape(q, (batch * heads, seq, hd))
    kh = b.reshape(k, (batch * heads, hd, seq))
    vh = b.reshape(v, (batch * heads, seq, hd))
    scores = b.batched_matmul(qh, kh)
    probs = b.elementwise(scores)
    ctx = b.batched_matmul(probs, vh)
    ctx2 = b.reshape(ctx, (tokens, hidden))
    wo = b.parameter(TS((hidden, hidden), eb))
    proj = b.matmul(ctx2, wo)
    return b.elementwise(proj, cur)


def _dense_ffn(b, G, cur, hidden: int, ffn: int, eb: int) -> int:
    TS = G.TensorShape
    w1 = b.parameter(TS((hidden, ffn), eb))
    a = b.elementwise(b.matmul(cur, w1))
    w2 = b.parameter(TS((ffn, hidden), eb))
    return b.elementwise(b.matmul(a, w2), cur)


def _moe_ffn(b, G, cur, batch: int, seq: int, hidden: int, ffn: int, experts: int,
             group: int, eb: int) -> int:
    TS = G.TensorShape
    tokens = batch * seq
    if tokens % group:
        raise G.GraphError(f"tokens {tokens} not divisible by group size {group}")
    if (2 * group) % experts:
        raise G.GraphError(f"capacity 2*{group}/{experts} is not an integer")
    ng = tokens // group
    cap = 2 * group // experts
    wg = b.parameter(TS((hidden, experts), eb))
    gates = b.elementwise(b.matmul(cur, wg))
    dmask = b.reshape(gates, (ng, experts * cap, group))
    cmask = b.reshape(gates, (ng, group, experts * cap))
    xg = b.reshape(cur, (ng, group, hidden))
    xd = b.batched_matmul(dmask, xg)
    xe = b.reshape(xd, (experts, ng * cap, hidden))
    w1 = b.parameter(TS((experts, hidden, ffn), eb))
    a = b.elementwise(b.batched_matmul(xe, w1))
    w2 = b.parameter(TS((experts, ffn, hidden), eb))
    h2 = b.batched_matmul(a, w2)
    yd = b.reshape(h2, (ng, experts * cap, hidden))
    y = b.batched_matmul(cmask, yd)
    return b.elementwise(b.reshape(y, (tokens, hidden)), cur)


def build_moe(num_layers: int, batch: int, seq: int, hidden: int, heads: int, experts: int,
              *, group: Optional[int] = None, ffn_mult: int = 8, moe_every: int = 2,
              elem_bytes: int = 2, backward: bool = False):
    """GShard MoE language model body: `num_layers`
    transformer layers, every `moe_every`-th one (the 2nd, 4th, ...) with its MLP
    replaced by a top-2 MoE layer.  Like the reference's transformer builder it
    has no embedding, LayerNorm or vocabulary projection.  FFN width is
    `ffn_mult * hidden` (8h: the 2.4B configuration, h=1024, 16 layers, 16
    experts, has 2.39e9 parameters with it; see tests)."""
    G = _meshplan_graph()
    if min(num_layers, batch, seq, hidden, heads, experts) < 1 or hidden % heads:
        raise G.GraphError("build_moe: bad dimensions")
    group = seq if group is None else group
    ffn = ffn_mult * hidden
    b = G._Builder()
    cur = b.input(G.TensorShape((batch * seq, hidden), elem_bytes))
    for layer in range(num_layers):
        cur = _attention(b, G, cur, batch, seq, hidden, heads, elem_bytes)
        if (layer + 1) % moe_every == 0:
            cur = _moe_ffn(b, G, cur, batch, seq, hidden, ffn, experts, group, elem_bytes)
        else:
            cur = _dense_ffn(b, G, cur, hidden, ffn, elem_bytes)
    if backward:
        cur = G._append_backward(b, cur)
    return b.graph([cur])


def build_wide_resnet(batch: int, image: int = 224, base: int = 320, width: int = 2,
                      blocks=(3, 4, 6, 3), classes: int = 1024, *, elem_bytes: int = 2,
                      backward: bool = False):
    """Wide-ResNet-50 body: bottleneck blocks
    [3, 4, 6, 3], bottleneck width `base * width * 2**stage`, output channels
    4 * base * 2**stage.  Convolutions are not in the IR, so a
    k x k convolution is an im2col reshape (rows = output pixels, cols =
    k*k*C_in) followed by a matmul; stride-2 subsampling lives in the reshape.
    The stem is a 7x7/2 conv (3 -> base) and the 3x3/2 max-pool is folded into
    the first stage's reshape; the head is a global average pool (reduction over
    pixels) and a classifier matmul.  No BatchNorm (like the transformer
    builder's missing LayerNorm)."""
    G = _meshplan_graph()
    TS = G.TensorShape
    eb = elem_bytes
    b = G._Builder()
    hw = image // 2
    x = b.input(TS((batch * image * image, 3), eb))
    # stem: 7x7 stride-2 conv as im2col + matmul (3*49 = 147 columns)
    cols = b.reshape(x, (batch * hw * hw, 49 * 3))
    cur = b.elementwise(b.matmul(cols, b.parameter(TS((49 * 3, base), eb))))
    c_in = base
    hw //= 2                                         # 3x3/2 max-pool
    cur = b.reshape(cur, (batch * hw * hw, c_in))
    for stage, n in enumerate(blocks):
        mid = base * width * 2 ** stage
        c_out = 4 * base * 2 ** stage
        for i in range(n):
            stride = 2 if (i == 0 and stage > 0) else 1
            out_hw = hw // stride
            rows = batch * out_hw * out_hw
            t = b.elementwise(b.matmul(cur, b.parameter(TS((c_in, mid), eb))))      # 1x1
            t = b.reshape(t, (rows, 9 * mid))                                     # im2col 3x3/s
            t = b.elementwise(b.matmul(t, b.parameter(TS((9 * mid, mid), eb))))
            t = b.matmul(t, b.parameter(TS((mid, c_out), eb)))                    # 1x1
            if i == 0:
                sc = cur if stride == 1 else b.reshape(cur, (rows, c_in))         # subsample
                sc = b.matmul(sc, b.parameter(TS((c_in, c_out), eb)))             # projection
            else:
                sc = cur
            cur = b.elementwise(b.elementwise(t, sc))                             # add, act
            c_in, hw = c_out, out_hw
    pooled = b.reduction(b.reshape(cur, (batch, hw * hw, c_in)), 1)               # (batch, C)
    cur = b.matmul(pooled, b.parameter(TS((c_in, classes), eb)))
    if backward:
        cur = G._append_backward(b, cur)
    return b.graph([cur])


BUILDERS = {"moe": build_moe, "wresnet": build_wide_resnet}


def graph_json(name: str, **kwargs) -> bytes:
    G = _meshplan_graph()
    return G.serialize(BUILDERS[name](**kwargs))


def param_count(graph) -> int:
    return sum(n.out_shape.num_elements for n in graph.nodes if n.kind.value == "parameter")


if __name__ == "__main__":  # pragma: no cover
    import argparse
    import sys
    ap = argparse.ArgumentParser(description="write a builder graph as reference graph JSON")
    ap.add_argument("spec", help="e.g. moe:num_layers=16,batch=8,seq=1024,hidden=1024,"
                                 "heads=16,experts=16,backward=1")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    name, _, rest = a.spec.partition(":")
    kw = {k: int(v) for k, v in (it.split("=") for it in rest.split(",") if it)}
    if "backward" in kw:
        kw["backward"] = bool(kw["backward"])
    data = graph_json(name, **kw)
    with open(a.out, "wb") as f:
        f.write(data)
    g = json.loads(data)
    print(f"{name}: {len(g['nodes'])} nodes", file=sys.stderr)
