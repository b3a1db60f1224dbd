"""Generate the golden fixtures that pin the executor's plan-level artifacts to
the live reference (run HERE, where /root/reference exists; the fixtures travel,
the reference does not):

  PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes (gzip JSON):
  xmesh.json.gz       cross_mesh_plan (reshard.py:111-157) Transfer / GatherOp
                      lists: the reference tests' meshes (test_reshard.py:16-107),
                      a randomized sweep, and the config-5 submesh pairs
                      (1,1)/(1,2)/(1,4) x every spec pair, optimize True/False
  boxes.json.gz       shard_box (reshard.py:74-85) for every spec of 2-D/3-D
                      tensors on every logical view of <= 8 devices
  algorithms.json.gz  enumerate_algorithms (sharding.py:222-299) for matmul and
                      batched matmul on every view of <= 8 devices
  programs/*.json.gz  Program.to_json() of emit_instructions (reshard.py:347-405)
                      for every committed plan x {gpipe, 1f1b}, and for the
                      reference tests' synthetic runtimes (test_reshard.py:112-151)
"""
from __future__ import annotations

import gzip
import itertools
import json
import random
import sys
from fractions import Fraction
from pathlib import Path

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.path.insert(0, str(REF.parent / "tests"))

from meshplan.graph import OpKind, OpNode, TensorShape  # noqa: E402
from meshplan.mesh import LogicalMesh  # noqa: E402
from meshplan.planio import runtime_from_json  # noqa: E402
from meshplan.reshard import (cross_mesh_plan, emit_instructions, shard_box)  # noqa: E402
from meshplan.sharding import enumerate_algorithms, enumerate_specs, format_spec  # noqa: E402

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
VIEWS = [(1, 1), (1, 2), (2, 1), (1, 4), (4, 1), (2, 2), (1, 8), (8, 1), (2, 4), (4, 2)]


def concrete(n, m, first):
    return LogicalMesh(n, m, (Fraction(10**9), Fraction(10**9)), tuple(range(first, first + n * m)))


def dump(path: Path, obj):
    path.parent.mkdir(parents=True, exist_ok=True)
    data = json.dumps(obj, sort_keys=True, separators=(",", ":")).encode()
    with open(path, "wb") as raw, gzip.GzipFile(fileobj=raw, mode="wb", mtime=0) as f:
        f.write(data)   # mtime=0: regenerating unchanged fixtures leaves them byte-identical


def xmesh_case(dims, eb, sv, ss, dv, ds, opt):
    shape = TensorShape(tuple(dims), eb)
    src, dst = concrete(*sv, 0), concrete(*dv, sv[0] * sv[1])
    p = cross_mesh_plan(shape, ss, src, ds, dst, optimize=opt)
    return {"dims": list(dims), "elem_bytes": eb, "src_view": list(sv), "dst_view": list(dv),
            "src_first": 0, "dst_first": sv[0] * sv[1],
            "src_spec": format_spec(ss), "dst_spec": format_spec(ds), "optimize": opt,
            "transfers": [[t.src_device, t.dst_device, t.nbytes, [list(b) for b in t.box]]
                          for t in p.transfers],
            "gathers": [[list(g.devices), list(g.axes), g.nbytes] for g in p.gathers],
            "inter_mesh_bytes": p.inter_mesh_bytes}


def make_xmesh():
    cases = []
    # reference test meshes (test_reshard.py): 8x8 on small views, exhaustive
    for sv, dv in itertools.product([(1, 2), (2, 2)], repeat=2):
        shape = TensorShape((8, 8))
        src, dst = concrete(*sv, 0), concrete(*dv, 16)
        for ss in enumerate_specs(shape, src):
            for ds in enumerate_specs(shape, dst):
                for opt in (True, False):
                    cases.append(xmesh_case((8, 8), 4, sv, ss, dv, ds, opt))
    # randomized sweep incl. uneven replica-group cuts (odd dim-0 extents)
    rng = random.Random(0)
    for _ in range(400):
        sv = rng.choice(VIEWS)
        dv = rng.choice(VIEWS)
        dims = tuple(rng.choice([6, 8, 12, 16, 24]) for _ in range(rng.choice([2, 3])))
        shape = TensorShape(dims, 2)
        ss = rng.choice(enumerate_specs(shape, concrete(*sv, 0)))
        ds = rng.choice(enumerate_specs(shape, concrete(*dv, 64)))
        cases.append(xmesh_case(dims, 2, sv, ss, dv, ds, rng.random() < 0.8))
    # config 5: (1,1)/(1,2)/(1,4) pairs, (rows, 8192) bf16 at a few sizes
    for sv, dv in itertools.product([(1, 1), (1, 2), (1, 4)], repeat=2):
        for rows in (64, 8192):
            shape = TensorShape((rows, 8192), 2)
            for ss in enumerate_specs(shape, concrete(*sv, 0)):
                for ds in enumerate_specs(shape, concrete(*dv, 8)):
                    for opt in (True, False):
                        cases.append(xmesh_case((rows, 8192), 2, sv, ss, dv, ds, opt))
    return cases


def make_boxes():
    out = []
    for v in VIEWS:
        mesh = concrete(*v, 0)
        for dims in ((8, 16), (16, 8, 24)):
            shape = TensorShape(dims, 2)
            for spec in enumerate_specs(shape, mesh):
                boxes = [[list(b) for b in shard_box(shape, spec, mesh, (i, j))]
                         for i in range(v[0]) for j in range(v[1])]
                out.append({"view": list(v), "dims": list(dims), "spec": format_spec(spec),
                            "boxes": boxes})
    return out


def make_algorithms():
    out = []
    for v in VIEWS:
        mesh = concrete(*v, 0)
        for kind, dims in ((OpKind.MATMUL, ((16, 32), (32, 8), (16, 8))),
                           (OpKind.BATCHED_MATMUL, ((8, 16, 32), (8, 32, 24), (8, 16, 24)))):
            a, b, c = (TensorShape(d, 2) for d in dims)
            node = OpNode(2, kind, ((0, 0), (1, 0)), c, 0)
            for alg in enumerate_algorithms(node, mesh, (a, b)):
                out.append({"view": list(v), "kind": kind.value, "out": format_spec(alg.output_spec),
                            "in": [format_spec(s) for s in alg.input_specs],
                            "comm": [[c.kind, c.bytes, list(c.axes)] for c in alg.comm]})
    return out


def make_programs():
    plans = sorted((ROOT / "plans").glob("*/plan.json"))
    for p in plans:
        doc = json.loads(p.read_text())
        rt = runtime_from_json(doc)
        for sched in ("gpipe", "1f1b"):
            prog = emit_instructions(rt, sched)
            dump(HERE / "programs" / f"{p.parent.name}.{sched}.json.gz", prog.to_json())
    # the reference tests' synthetic runtimes, serialized as plan documents
    from test_reshard import synthetic_runtime
    from meshplan.planio import cluster_to_json
    from meshplan import graph as graph_mod
    from meshplan.sharding import format_spec as fs
    cases = [([2, 2, 4, 2], 3, False), ([1, 2, 1], 3, True), ([4, 4, 4], 6, True),
             ([3, 3, 3, 3], 8, True), ([2, 3, 1], 5, True)]
    for k, (times, B, bwd) in enumerate(cases):
        rt = synthetic_runtime(times, B, backward=bwd, act_bytes=100)
        doc = {"version": 1, "kind": "meshplan.plan", "config": {},
               "cluster": cluster_to_json(rt.cluster),
               "graph": json.loads(graph_mod.serialize(rt.graph)),
               "num_microbatches": B, "t_star": [rt.t_star.numerator, rt.t_star.denominator],
               "stages": [{"index": s.index, "op_ids": list(s.op_ids),
                           "logical_view": [s.view.n_l, s.view.m_l],
                           "axis_bw": [[b.numerator, b.denominator] for b in s.view.axis_bandwidth],
                           "device_ids": list(s.view.device_ids),
                           "t": [s.t.numerator, s.t.denominator], "mem_stage": s.mem_stage,
                           "mem_act": s.mem_act, "op_specs": {},
                           "boundary_inputs": {str(k2): fs(v2) for k2, v2 in s.input_specs.items()},
                           "boundary_outputs": {str(k2): fs(v2) for k2, v2 in s.output_specs.items()}}
                          for s in rt.stages]}
        for sched in ("gpipe", "1f1b"):
            prog = emit_instructions(rt, sched)
            dump(HERE / "programs" / f"synthetic{k}.{sched}.json.gz",
                 {"plan": doc, "program": prog.to_json()})


def make_ilp_tables():
    """Random strategy tables (integer and rational costs, both edge
    orientations, tight and default budgets) with the reference solver's answer."""
    import sys as _sys
    _sys.path.insert(0, str(HERE.parent))
    from test_ilp_native import enc, rand_table
    from meshplan.intra import solve_ilp
    rng = random.Random(123)
    out = []
    for trial in range(48):
        t = rand_table(rng, rng.randint(1, 12), 7, rational=trial % 2 == 1, flip=trial % 3 == 0)
        budget = (3, 60, 200_000)[trial % 3]
        r = solve_ilp(t, budget)
        out.append({"table": enc(t), "budget": budget, "choice": list(r.choice),
                    "objective": [r.objective.numerator, r.objective.denominator],
                    "certified": bool(r.certified)})
    return out


if __name__ == "__main__":
    dump(HERE / "xmesh.json.gz", make_xmesh())
    dump(HERE / "boxes.json.gz", make_boxes())
    dump(HERE / "algorithms.json.gz", make_algorithms())
    make_programs()
    dump(HERE / "ilp_tables.json.gz", make_ilp_tables())
    print("golden fixtures written to", HERE)
