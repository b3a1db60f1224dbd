"""Plan-faithful virtual-device executor (test infrastructure only).

Every device of every stage holds only its local shard of every tensor, in the
spec the plan assigns.  Per op and per device:
  * inputs are assembled into the op's required input spec from the shards the
    stage's devices hold (box intersections, reshard.py:64-71);
  * matmul/bmm: local product of the local operands; when the contraction loop
    k is mapped to mesh axes the partial sums are summed over the k-group
    (reference _matmul_algorithms, sharding.py:255-299);
  * trivial members compute locally on their propagated spec
    (intra.py:128-160); a softmax whose row is split is computed on the
    assembled full row and sliced (equal to the row-stat all-reduce);
  * reshapes follow the binding; head split/merge go through the replicated
    tensor (the planner's layout barrier, intra.py:149-160).
Stage boundaries move boxes per a restated cross_mesh_plan (reshard.py:97-157),
including the local all-gather over replica groups.  Parameter gradients are
accumulated unreduced over microbatches and summed over the k-group at the end
(the post_ilp_rewrite reduce-scatter + all-gather is a realisation of the same
sum, intra.py:404-424).
"""
from __future__ import annotations

import numpy as np

from . import dense, ir


def _tiles(dims, spec, st):
    return [(dev, ir.box_of(dims, spec, st.ext, st.coords(dev))) for dev in st.devices]


def xmesh(dims, sspec, sst, dspec, dst, optimize=True):
    """Restated cross_mesh_plan -> (transfers[(src, dst, box)], gathers[(devices, tile, pieces)])."""
    src = _tiles(dims, sspec, sst)

    def sources(piece, dev):
        best = {}
        for d, t in src:
            ov = ir.inter(piece, t)
            if ov is not None and (ov not in best or d < best[ov]):
                best[ov] = d
        return [(best[b], dev, b) for b in sorted(best)]

    dtiles = _tiles(dims, dspec, dst)
    if not optimize:
        return [t for dev, tile in dtiles for t in sources(tile, dev)], []
    groups = {}
    for dev, tile in dtiles:
        groups.setdefault(tile, []).append(dev)
    trans, gath = [], []
    for tile in sorted(groups):
        devs = sorted(groups[tile])
        if len(devs) == 1:
            trans += sources(tile, devs[0])
            continue
        g = len(devs)
        lo, hi = tile[0]
        pieces = []
        for r, dev in enumerate(devs):
            a, b = lo + (hi - lo) * r // g, lo + (hi - lo) * (r + 1) // g
            piece = ((a, b),) + tile[1:]
            pieces.append(piece)
            if a < b:
                trans += sources(piece, dev)
        gath.append((tuple(devs), tile, tuple(pieces)))
    return trans, gath


class ShardedRun:
    def __init__(self, plan_doc, params, inputs, num_microbatches, dtype=np.float64):
        self.doc, self.nodes, self.stages = ir.load(plan_doc)
        self.bound = ir.bind(self.nodes)
        self.params = params
        self.inputs = inputs
        self.B = num_microbatches
        self.dtype = dtype
        self.stage_of = {op: s.index for s in self.stages for op in s.ops}
        self.local = {}
        self.gacc = {}
        self.loss = 0.0
        self.outputs = {}

    # -------------------------------------------------------------- helpers
    def dims(self, nid):
        return ir.node_dims(self.nodes[nid])

    def key(self, dev, mb, nid):
        return (dev, None if self.bound[nid][0] == "parameter" else mb, nid)

    def fetch(self, st, dev, mb, nid, req):
        dims = self.dims(nid)
        need = ir.box_of(dims, req, st.ext, st.coords(dev))
        out = np.zeros([hi - lo for lo, hi in need], dtype=self.dtype)
        have_spec = st.spec(nid)
        for e in st.devices:
            have = ir.box_of(dims, have_spec, st.ext, st.coords(e))
            ov = ir.inter(need, have)
            if ov is not None:
                src = self.local[self.key(e, mb, nid)]
                out[ir.sl(ov, [b[0] for b in need])] = src[ir.sl(ov, [b[0] for b in have])]
        return out

    def assemble(self, st, mb, nid):
        dims = self.dims(nid)
        full = np.zeros(dims, dtype=self.dtype)
        for e in st.devices:
            box = ir.box_of(dims, st.spec(nid), st.ext, st.coords(e))
            full[ir.sl(box)] = self.local[self.key(e, mb, nid)]
        return full

    def kgroup(self, st, dev, k_axes):
        i, j = st.coords(dev)
        return [e for e in st.devices
                if all(st.coords(e)[a] == (i, j)[a] for a in (0, 1) if a not in k_axes)]

    # -------------------------------------------------------------- ops
    def run_op(self, st, mb, nid):
        n = self.nodes[nid]
        code, info = self.bound[nid]
        out_spec = st.spec(nid)
        dims = self.dims(nid)
        ins = ir.node_inputs(n)
        if code == "input":
            full = np.asarray(self.inputs(mb, nid), dtype=self.dtype)
            for dev in st.devices:
                self.local[(dev, mb, nid)] = full[ir.sl(ir.box_of(dims, out_spec, st.ext, st.coords(dev)))]
            return
        if code in ("matmul", "batched_matmul"):
            used = {a for d in out_spec for a in d}
            k = tuple(a for a in (0, 1) if st.ext[a] > 1 and a not in used)
            if code == "matmul":
                lhs, rhs = (out_spec[0], k), (k, out_spec[1])
            else:
                lhs, rhs = (out_spec[0], out_spec[1], k), (out_spec[0], k, out_spec[2])
            part = {dev: self.fetch(st, dev, mb, ins[0], lhs) @ self.fetch(st, dev, mb, ins[1], rhs)
                    for dev in st.devices}
            for dev in st.devices:
                red = sum(part[e] for e in self.kgroup(st, dev, k))
                self.local[(dev, mb, nid)] = red
                if n.get("grad_of") is not None:
                    key = (dev, n["grad_of"])
                    self.gacc[key] = self.gacc.get(key, 0.0) + part[dev]
            self.kaxes = getattr(self, "kaxes", {})
            self.kaxes[nid] = k
            return
        if n["kind"] == "reshape":
            if code == "identity":
                req = out_spec
            elif code == "transpose":
                req = out_spec[:-2] + (out_spec[-1], out_spec[-2])
            else:
                req = tuple(() for _ in self.dims(ins[0]))
            for dev in st.devices:
                x = self.fetch(st, dev, mb, ins[0], req)
                if code in ("identity", "transpose"):
                    self.local[(dev, mb, nid)] = dense.reshape_op(code, info, x)
                else:
                    val = {}
                    if code in ("dispatch_grad", "combine_grad"):
                        gid = info[1]
                        val[gid] = self.fetch(st, dev, mb, gid, tuple(() for _ in self.dims(gid)))
                    full = dense.eval_node(code, info, n, [x], val)
                    box = ir.box_of(dims, out_spec, st.ext, st.coords(dev))
                    self.local[(dev, mb, nid)] = full[ir.sl(box)]
            return
        if code == "reduce_sum":
            rep = tuple(() for _ in self.dims(ins[0]))
            for dev in st.devices:
                full = self.fetch(st, dev, mb, ins[0], rep).sum(axis=info)
                box = ir.box_of(dims, out_spec, st.ext, st.coords(dev))
                self.local[(dev, mb, nid)] = full[ir.sl(box)]
            return
        # elementwise members
        row_split = any(st.ext[a] > 1 for a in out_spec[-1])
        for dev in st.devices:
            box = ir.box_of(dims, out_spec, st.ext, st.coords(dev))
            if code in ("softmax", "softmax_bwd") and row_split:
                # compute on full rows, keep the local columns
                rows_spec = out_spec[:-1] + ((),)
                rbox = ir.box_of(dims, rows_spec, st.ext, st.coords(dev))
                args = [self.fetch(st, dev, mb, p, rows_spec) for p in ins]
                val = {}
                if code == "softmax_bwd":
                    val[info[0]] = self.fetch(st, dev, mb, info[0], rows_spec)
                y = dense.eval_node(code, info, n, args, val)
                self.local[(dev, mb, nid)] = y[..., box[-1][0] - rbox[-1][0]:box[-1][1] - rbox[-1][0]]
                continue
            args = [self.fetch(st, dev, mb, p, out_spec) for p in ins]
            val = {}
            if code == "gelu_bwd":
                val[info] = self.fetch(st, dev, mb, info, out_spec)
            if code == "softmax_bwd":
                val[info[0]] = self.fetch(st, dev, mb, info[0], out_spec)
            self.local[(dev, mb, nid)] = dense.eval_node(code, info, n, args, val)
        if code == "seed":
            y = self.assemble(st, mb, nid)
            self.loss += 0.5 * float((y * y).sum())
            self.outputs[mb] = y

    # -------------------------------------------------------------- boundaries
    def receive(self, st, mb, phase):
        for nid in sorted(st.in_specs):
            p = self.stage_of.get(nid)
            if p is None or p == st.index:
                continue
            if ("fwd" if p < st.index else "bwd") != phase:
                continue
            src = self.stages[p]
            dims = self.dims(nid)
            sspec = ir.canon(src.out_specs[nid], src.ext)
            dspec = st.spec(nid)
            trans, gath = xmesh(dims, sspec, src, dspec, st)
            for dev in st.devices:
                box = ir.box_of(dims, dspec, st.ext, st.coords(dev))
                self.local[self.key(dev, mb, nid)] = np.full([hi - lo for lo, hi in box], np.nan,
                                                             self.dtype)
            for s_dev, d_dev, box in trans:
                sbox = ir.box_of(dims, sspec, src.ext, src.coords(s_dev))
                dbox = ir.box_of(dims, dspec, st.ext, st.coords(d_dev))
                self.local[self.key(d_dev, mb, nid)][ir.sl(box, [b[0] for b in dbox])] = \
                    self.local[self.key(s_dev, mb, nid)][ir.sl(box, [b[0] for b in sbox])]
            for devs, tile, pieces in gath:
                for d in devs:
                    for owner, piece in zip(devs, pieces):
                        if owner == d or piece[0][0] >= piece[0][1]:
                            continue
                        self.local[self.key(d, mb, nid)][ir.sl(piece, [b[0] for b in tile])] = \
                            self.local[self.key(owner, mb, nid)][ir.sl(piece, [b[0] for b in tile])]

    # -------------------------------------------------------------- driver
    def run(self):
        for st in self.stages:
            for nid in st.ops:
                if self.bound[nid][0] == "parameter":
                    dims = self.dims(nid)
                    for dev in st.devices:
                        box = ir.box_of(dims, st.spec(nid), st.ext, st.coords(dev))
                        self.local[(dev, None, nid)] = np.asarray(self.params[nid], self.dtype)[ir.sl(box)]
        for mb in range(self.B):
            for phase in ("fwd", "bwd"):
                order = self.stages if phase == "fwd" else list(reversed(self.stages))
                for st in order:
                    self.receive(st, mb, phase)
                    for nid in sorted(st.ops):
                        n = self.nodes[nid]
                        is_fwd = n.get("colocate_with") is None
                        if is_fwd != (phase == "fwd") or self.bound[nid][0] == "parameter":
                            continue
                        self.run_op(st, mb, nid)
        grads = {}
        for st in self.stages:
            for nid in st.ops:
                pid = self.nodes[nid].get("grad_of")
                if pid is None:
                    continue
                dims = self.dims(nid)
                full = np.zeros(dims, self.dtype)
                for dev in st.devices:
                    red = sum(self.gacc[(e, pid)] for e in self.kgroup(st, dev, self.kaxes[nid]))
                    full[ir.sl(ir.box_of(dims, st.spec(nid), st.ext, st.coords(dev)))] = red
                grads[pid] = full
        return self.loss, grads, self.outputs


def run(plan_doc, params, inputs, num_microbatches, dtype=np.float64):
    return ShardedRun(plan_doc, params, inputs, num_microbatches, dtype).run()
