"""Oracle-side restatement of the reference IR, specs, boxes and the numeric
binding (test infrastructure only; see oracle/__init__.py)."""
from __future__ import annotations

import json
import re
from pathlib import Path

# ----------------------------------------------------------------- specs
# reference sharding.py:102-133:  R | S^a | S^{ab}
_TOK = re.compile(r"R|S\^(\d|\{\d+\})")


def spec_parse(text):
    dims, i = [], 0
    while i < len(text):
        m = _TOK.match(text, i)
        assert m, f"bad spec {text}"
        dims.append(() if m.group(0) == "R" else tuple(int(c) for c in m.group(1).strip("{}")))
        i = m.end()
    return tuple(dims)


def canon(spec, ext):
    """drop axes of extent 1 (reference _canon_axes, sharding.py:181-183)"""
    return tuple(tuple(sorted(a for a in d if ext[a] > 1)) for d in spec)


def box_of(dims, spec, ext, coords):
    """reference shard_box, reshard.py:74-85"""
    out = []
    for n, axes in zip(dims, spec):
        blocks, idx = 1, 0
        for a in axes:
            blocks *= ext[a]
            idx = idx * ext[a] + coords[a]
        step = n // blocks
        out.append((idx * step, (idx + 1) * step))
    return tuple(out)


def inter(a, b):
    out = []
    for (a0, a1), (b0, b1) in zip(a, b):
        lo, hi = max(a0, b0), min(a1, b1)
        if lo >= hi:
            return None
        out.append((lo, hi))
    return tuple(out)


def sl(box, origin=None):
    if origin is None:
        return tuple(slice(lo, hi) for lo, hi in box)
    return tuple(slice(lo - o, hi - o) for (lo, hi), o in zip(box, origin))


# ----------------------------------------------------------------- plan
class Stage:
    def __init__(self, d):
        self.index = d["index"]
        self.n, self.m = d["logical_view"]
        self.devices = tuple(d["device_ids"])
        self.ops = tuple(d["op_ids"])
        self.specs = {int(k): spec_parse(v) for k, v in d["op_specs"].items()}
        self.in_specs = {int(k): spec_parse(v) for k, v in d["boundary_inputs"].items()}
        self.out_specs = {int(k): spec_parse(v) for k, v in d["boundary_outputs"].items()}
        self.ext = (self.n, self.m)

    def coords(self, dev):
        return divmod(self.devices.index(dev), self.m)

    def spec(self, nid):
        s = self.specs.get(nid, self.in_specs.get(nid))
        return canon(s, self.ext)


def load(path_or_doc):
    doc = path_or_doc if isinstance(path_or_doc, dict) else json.loads(Path(path_or_doc).read_text())
    nodes = doc["graph"]["nodes"]
    stages = [Stage(d) for d in sorted(doc["stages"], key=lambda d: d["index"])]
    return doc, nodes, stages


def node_dims(n):
    return tuple(n["shape"]["dims"])


def node_inputs(n):
    return [e[0] for e in n["inputs"]]


# ----------------------------------------------------------------- binding
def _batch(nodes):
    """images per microbatch: leading dim of the pooling reduction's (N, HW, C) input"""
    for n in nodes:
        if n["kind"].startswith("reduction") and n.get("colocate_with") is None:
            d = node_dims(nodes[n["inputs"][0][0]])
            if len(d) == 3:
                return d[0]
    return None


def _conv(src, dst, batch):
    """NHWC im2col (k x k, stride s, pad k/2) or subsample reshape -> (code, (N,H,W,C,k,s))"""
    if batch is None:
        return None
    (ri, ci), (ro, co) = src, dst
    H = int(round((ri / batch) ** 0.5))
    Ho = int(round((ro / batch) ** 0.5))
    k = int(round((co / ci) ** 0.5))
    if batch * H * H != ri or batch * Ho * Ho != ro or k * k * ci != co or k % 2 == 0:
        return None
    s = max(1, H // Ho)
    if (H + 2 * (k // 2) - k) // s + 1 != Ho:
        return None
    return ("im2col" if k > 1 else "subsample", (batch, H, H, ci, k, s))


def bind(nodes):
    """node id -> (code, info).  Same rules as the product's binding, restated."""
    out = {}
    consumers = {n["id"]: [] for n in nodes}
    for n in nodes:
        for s, (p, _) in enumerate(n["inputs"]):
            consumers[p].append((n["id"], s))
    batch = _batch(nodes)
    for n in nodes:
        k, nid, ins = n["kind"], n["id"], node_inputs(n)
        co = n.get("colocate_with")
        if k in ("input", "parameter", "matmul", "batched_matmul"):
            out[nid] = (k, None)
        elif k.startswith("reduction"):
            out[nid] = ("reduce_sum", int(k.split(":")[1]))
        elif k == "elementwise":
            if co is None:
                if len(ins) == 2:
                    out[nid] = ("add", None)
                elif any(_routing(nodes, nodes[c], consumers) is not None
                         for c, _ in consumers[nid]):
                    out[nid] = ("softmax", 1.0)                      # MoE gates
                elif nodes[ins[0]]["kind"] == "batched_matmul" and \
                        nodes[nodes[ins[0]]["inputs"][1][0]]["kind"] != "parameter":
                    d = node_dims(nodes[nodes[ins[0]]["inputs"][0][0]])[-1]
                    out[nid] = ("softmax", 1.0 / d ** 0.5)
                else:
                    out[nid] = ("gelu", None)
            else:
                f = nodes[co]
                if len(ins) == 1 and ins[0] == co and f.get("colocate_with") is None:
                    out[nid] = ("seed", None)
                elif len(ins) == 2:
                    out[nid] = ("add", None)
                else:
                    fc, finfo = out[co]
                    if fc == "gelu":
                        out[nid] = ("gelu_bwd", node_inputs(f)[0])
                    elif fc == "softmax":
                        out[nid] = ("softmax_bwd", (co, finfo))
                    elif fc == "add":
                        out[nid] = ("identity", None)
                    else:
                        raise ValueError(f"no backward for {fc}")
        elif k == "reshape":
            src = node_dims(nodes[ins[0]])
            dst = node_dims(n)
            if co is not None:
                f = nodes[co]
                if f["kind"] in ("matmul", "batched_matmul"):
                    out[nid] = ("transpose", None)
                elif f["kind"].startswith("reduction"):
                    out[nid] = ("broadcast", None)
                elif out[co][0] in ("im2col", "subsample"):
                    out[nid] = ("col2im" if out[co][0] == "im2col" else "subsample_grad",
                                out[co][1])
                elif out[co][0] in ("dispatch", "combine"):
                    out[nid] = (out[co][0] + "_grad", (out[co][1], node_inputs(f)[0]))
                elif out[co][0] == "regroup":
                    A, P, C = out[co][1]
                    out[nid] = ("regroup", (P, A, C))
                else:
                    fc, heads = out[co]
                    inv = {"split": "merge", "split_t": "merge_t", "merge": "split",
                           "merge_t": "split_t", "transpose": "transpose", "identity": "identity"}
                    out[nid] = (inv[fc], heads)
            elif _routing(nodes, n, consumers) is not None:
                out[nid] = _routing(nodes, n, consumers)
            elif len(src) == 3 and len(dst) == 3 and nodes[ins[0]]["kind"] == "batched_matmul":
                A, B, _ = src
                out[nid] = ("regroup", (A, dst[0], B // dst[0]))
            elif len(src) == 2 and len(dst) == 3:
                tr = any(nodes[c]["kind"] == "batched_matmul" and s == 1
                         and nodes[nodes[c]["inputs"][0][0]]["kind"] == "reshape"
                         and _routing(nodes, nodes[nodes[c]["inputs"][0][0]], consumers) is None
                         for c, s in consumers[nid])
                T, h = src
                X, Y, Z = dst
                seq, d = (Z, Y) if tr else (Y, Z)
                out[nid] = ("split_t" if tr else "split", (T // seq, h // d, seq, d))
            elif len(src) == 3 and len(dst) == 2:
                T, h = dst
                X, seq, d = src
                out[nid] = ("merge", (T // seq, h // d, seq, d))
            elif src == dst:
                out[nid] = ("identity", None)
            elif src[::-1] == dst:
                out[nid] = ("transpose", None)
            else:
                cv = _conv(src, dst, batch)
                if cv is None:
                    raise ValueError(f"reshape {src} -> {dst}")
                out[nid] = cv
        else:
            raise ValueError(f"unsupported kind {k}")
    return out


def _routing(nodes, r, consumers):
    """MoE gates (T, E) -> dispatch (G, E*C, S) / combine (G, S, E*C): the
    product's binding.routing_geom, restated.  info = (G, S, E, C)."""
    if r["kind"] != "reshape" or r.get("colocate_with") is not None:
        return None
    src = nodes[r["inputs"][0][0]]
    if src["kind"] != "elementwise" or src.get("colocate_with") is not None \
            or len(src["inputs"]) != 1:
        return None
    sd, rd = node_dims(src), node_dims(r)
    if len(sd) != 2 or len(rd) != 3:
        return None
    if not any(nodes[c]["kind"] == "batched_matmul" and s == 0 for c, s in consumers[r["id"]]):
        return None
    T, E = sd
    X, Y, Z = rd
    if X * Z == T and Y % E == 0:
        return ("dispatch", (X, Z, E, Y // E))
    if X * Y == T and Z % E == 0:
        return ("combine", (X, Y, E, Z // E))
    raise ValueError(f"reshape of gates {sd} -> {rd}")
