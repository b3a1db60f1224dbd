"""Profile-driven stage costs (the paper's Alg. 1 `Profile` step).

The reference planner prices a candidate stage (a contiguous layer range on a
submesh view, with the sharding its ILP chose) analytically: `t_compute =
flop / (devices * device_flops)` plus the ILP's modeled communication
(`intra.py:494-516`, `costs.py:83-92`).  Here the same candidate is executed on
B200s by this executor and its measured time per microbatch replaces the model:

  1. `stage_doc` turns one candidate into a self-contained single-stage plan
     document.  Tensors produced outside the range become graph inputs (as
     `extract_stage`, `intra.py:47-75`, does), but colocation and `grad_of` are
     kept so the stage runs its real forward and backward.
  2. `scripts/profile_stages.py run` executes every distinct document on its
     device count and records seconds per microbatch.
  3. `patch_reference(meshplan, table)` wraps the planner's `evaluate_stage`
     so each view's `StageCostReport` carries the measured time
     (`t_compute = measured`, `t_comm = 0`).  Every other step of the DP is the
     reference's own.

This changes plans by design, so it is opt-in and outside the bit-exact contract.
"""
from __future__ import annotations

import hashlib
import json
from fractions import Fraction
from typing import Iterable, Mapping, Optional

PLAN_KIND = "meshplan.plan"


def _rep(rank: int) -> str:
    return "R" * rank


def stage_doc(graph_doc: dict, op_ids: Iterable[int], view: tuple[int, int],
              specs: Mapping[int, str], num_microbatches: int = 2,
              cluster: Optional[dict] = None) -> dict:
    """Single-stage plan document for one candidate stage.

    graph_doc: the reference's serialized graph (`{"nodes": [...], "outputs": [...]}`).
    specs: original node id -> spec string (the ILP's node specs for the members).
    Externally produced tensors become `input` nodes, replicated."""
    nodes = graph_doc["nodes"]
    members = sorted(set(int(i) for i in op_ids))
    mset = set(members)
    externals = sorted({int(p) for i in members for p, _ in nodes[i]["inputs"]
                        if int(p) not in mset})
    local: dict[int, int] = {}
    out_nodes = []
    for p in externals:
        local[p] = len(out_nodes)
        out_nodes.append({"id": local[p], "kind": "input", "inputs": [],
                          "shape": dict(nodes[p]["shape"]), "flop": 0})
    for k, i in enumerate(members):
        local[i] = len(externals) + k
    for i in members:
        n = nodes[i]
        m = {"id": local[i], "kind": n["kind"],
             "inputs": [[local[int(p)], int(s)] for p, s in n["inputs"]],
             "shape": dict(n["shape"]), "flop": n.get("flop", 0)}
        for key in ("colocate_with", "grad_of"):
            if n.get(key) is not None and int(n[key]) in local:
                m[key] = local[int(n[key])]
        for key, val in n.items():
            if key not in m and key not in ("colocate_with", "grad_of"):
                m[key] = val
        out_nodes.append(m)
    outputs = [local[int(o)] for o in graph_doc.get("outputs", []) if int(o) in mset]
    n_dev = view[0] * view[1]
    op_specs = {}
    for p in externals:
        op_specs[str(local[p])] = _rep(len(nodes[p]["shape"]["dims"]))
    for i in members:
        op_specs[str(local[i])] = specs.get(i, _rep(len(nodes[i]["shape"]["dims"])))
    cl = dict(cluster or {})
    cl.update({"hosts": 1, "devices_per_host": n_dev})
    cl.setdefault("intra_bw", [900000000000, 1])
    cl.setdefault("inter_bw", [900000000000, 1])
    cl.setdefault("alpha", [1, 100000])
    cl.setdefault("device_flops", [1400000000000000, 1])
    cl.setdefault("device_memory", 180000000000)
    config = {"profile_stage": True}
    for n in nodes:      # convolutional graphs: keep the image count the binding needs
        if n["kind"].startswith("reduction") and "colocate_with" not in n:
            src = nodes[n["inputs"][0][0]]["shape"]["dims"]
            if len(src) == 3:
                config["image_batch"] = int(src[0])
    return {
        "version": 1, "kind": PLAN_KIND,
        "config": config,
        "cluster": cl,
        "graph": {"version": graph_doc.get("version", 1), "nodes": out_nodes, "outputs": outputs},
        "num_microbatches": int(num_microbatches),
        "t_star": [1, 1],
        "stages": [{
            "index": 0, "op_ids": list(range(len(out_nodes))),
            "logical_view": [int(view[0]), int(view[1])],
            "device_ids": list(range(n_dev)), "axis_bw": [[1, 1], [1, 1]],
            "op_specs": op_specs, "boundary_inputs": {}, "boundary_outputs": {},
            "t": [1, 1], "mem_stage": 0, "mem_act": 0,
        }],
    }


def doc_key(doc: dict) -> str:
    """Structural hash of a stage document (graph + specs + view): candidates
    that are the same computation (e.g. equal-length GPT layer ranges) share it."""
    st = doc["stages"][0]
    payload = json.dumps({"nodes": [[n["kind"], n["inputs"], n["shape"]["dims"],
                                     n.get("colocate_with"), n.get("grad_of")]
                                    for n in doc["graph"]["nodes"]],
                          "outputs": doc["graph"]["outputs"],
                          "view": st["logical_view"],
                          "specs": sorted(st["op_specs"].items(), key=lambda kv: int(kv[0]))},
                         sort_keys=True, separators=(",", ":"))
    return hashlib.sha256(payload.encode()).hexdigest()[:20]


def candidate_key(op_ids: Iterable[int], shape: tuple[int, int], view: tuple[int, int]) -> str:
    ops = sorted(int(i) for i in op_ids)
    h = hashlib.sha256(json.dumps(ops).encode()).hexdigest()[:16]
    return f"{h}|{shape[0]}x{shape[1]}|{view[0]}x{view[1]}"


def patch_reference(meshplan_pkg, index: Mapping[str, str], measured: Mapping[str, float],
                    strict: bool = True, missing: str = "model"):
    """Wrap `meshplan.inter.evaluate_stage` so every view report carries the
    measured seconds per microbatch of its candidate (index: candidate key ->
    doc key; measured: doc key -> seconds).  Unmeasured candidates raise (strict),
    keep the analytic cost (missing="model") or are priced out (missing="exclude").
    Returns the original function."""
    from dataclasses import replace
    inter = meshplan_pkg.inter
    orig = inter.evaluate_stage

    def evaluate_stage(graph, op_ids, shape, cluster, cost_model, *a, **kw):
        ev = orig(graph, op_ids, shape, cluster, cost_model, *a, **kw)
        views = []
        for vr in ev.views:
            ck = candidate_key(op_ids, (shape.n, shape.m), (vr.view.n_l, vr.view.m_l))
            dk = index.get(ck)
            if dk is None or dk not in measured:
                if strict:
                    raise KeyError(f"no measurement for candidate {ck}")
                if missing == "exclude":    # unmeasured candidates are never chosen
                    views.append(replace(vr, report=replace(
                        vr.report, t_compute=Fraction(10 ** 9), t_comm=Fraction(0))))
                else:
                    views.append(vr)
                continue
            t = Fraction(measured[dk]).limit_denominator(10**12)
            views.append(replace(vr, report=replace(vr.report, t_compute=t, t_comm=Fraction(0))))
        return type(ev)(ev.sub, tuple(views))

    inter.evaluate_stage = evaluate_stage
    return orig


def patch_cross_stage(meshplan_pkg):
    """SURVEY §8 f4 (the paper's stated limitation): the
    reference DP prices a stage by compute + intra-stage communication only
    (`intra.py:511-516`), so T* omits the cross-mesh transfers its own
    simulator charges (`sim.py:80-84`).  This wraps `evaluate_stage` so each
    view's t_comm also carries the receive time of the stage's external
    activations, one `transfer_time` (alpha + bytes / inter_bw, `costs.py:88-92`)
    per tensor.  Weights are excluded (parameter nodes of the original graph).
    Opt-in: it changes plans.  Returns the original function."""
    from dataclasses import replace
    inter = meshplan_pkg.inter
    orig = inter.evaluate_stage

    def evaluate_stage(graph_, op_ids, shape, cluster, cost_model, *a, **kw):
        ev = orig(graph_, op_ids, shape, cluster, cost_model, *a, **kw)
        params = {i for i, n in enumerate(graph_.nodes) if n.kind.value == "parameter"}
        views = []
        for vr in ev.views:
            specs = vr.plan.node_specs()
            extra = Fraction(0)
            for lid in ev.sub.boundary_inputs:
                if ev.sub.orig_of[lid] in params or lid not in specs:
                    continue
                nbytes = ev.sub.graph.node(lid).out_shape.byte_size // \
                    specs[lid].shard_factor(vr.view)
                extra += cost_model.transfer_time(nbytes)
            views.append(replace(vr, report=replace(vr.report, t_comm=vr.report.t_comm + extra)))
        return type(ev)(ev.sub, tuple(views))

    inter.evaluate_stage = evaluate_stage
    return orig
