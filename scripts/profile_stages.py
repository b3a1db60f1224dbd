"""Profile-driven stage costs for the reference planner.

  # 1. here (needs the reference): enumerate the planner's stage candidates and
  #    write one single-stage plan document per distinct candidate
  python scripts/profile_stages.py emit --builder transformer:blocks=24,batch=8,seq=1024,\
hidden=2048,heads=32,elem_bytes=2,backward=1 --cluster plans/clusters/b200_1x4.json \
      --layers 4 --out exp/prof_gpt_n4

  # 2. on the GPU box: execute every document with this executor (one torchrun per
  #    device count), seconds per microbatch -> measured.json
  python scripts/profile_stages.py run exp/prof_gpt_n4          # launches torchrun itself

  # 3. here: plan with the measured costs in place of the analytic model
  python scripts/profile_stages.py plan exp/prof_gpt_n4 --out plans/gpt13b_n4_prof -- \
      --builder ... --cluster plans/clusters/b200_1x4.json --b 64 --layers 4 --epsilon 0

See paper_2201_12023_b200/profiling.py for what is measured and what is patched.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.dont_write_bytecode = True


def _ref(src):
    sys.path.insert(0, src)
    import meshplan  # noqa: F401
    import meshplan.intra  # noqa: F401
    import meshplan.inter  # noqa: F401
    return sys.modules["meshplan"]


def cmd_emit(a):
    mp = _ref(a.reference_src)
    from meshplan import cli
    from meshplan import graph as graph_mod
    from meshplan.inter import cluster_operators, DEFAULT_DELTA
    from meshplan.intra import evaluate_stage
    from meshplan.mesh import admissible_shapes
    from meshplan.costs import CostModel
    from meshplan.planio import cluster_from_json
    from meshplan.sharding import format_spec
    from paper_2201_12023_b200 import ilp, profiling
    ilp.patch_reference(mp)
    graph = (cli._parse_builder(a.builder) if a.builder
             else graph_mod.parse(Path(a.graph).read_bytes()))
    cdoc = json.loads(Path(a.cluster).read_text())
    cluster = cluster_from_json(cdoc)
    gdoc = json.loads(graph_mod.serialize(graph))
    clustering = cluster_operators(graph, a.layers, DEFAULT_DELTA)
    cm = CostModel(cluster)
    out = Path(a.out)
    (out / "docs").mkdir(parents=True, exist_ok=True)
    index, docs = {}, {}
    t0 = time.perf_counter()
    for lo in range(a.layers):
        for hi in range(lo + 1, a.layers + 1):
            ops = clustering.range_ops(lo, hi)
            for shape in admissible_shapes(cluster):
                if shape.num_devices > cluster.num_devices or shape.num_devices > a.max_devices:
                    continue
                ev = evaluate_stage(graph, ops, shape, cluster, cm)
                for vr in ev.views:
                    local = vr.plan.node_specs()
                    specs = {ev.sub.orig_of[k]: format_spec(v) for k, v in local.items()}
                    view = (vr.view.n_l, vr.view.m_l)
                    doc = profiling.stage_doc(gdoc, ops, view, specs, a.microbatches, cdoc)
                    dk = profiling.doc_key(doc)
                    ck = profiling.candidate_key(ops, (shape.n, shape.m), view)
                    index[ck] = dk
                    if dk not in docs:
                        docs[dk] = {"devices": view[0] * view[1], "layers": [lo, hi],
                                    "view": list(view), "modeled_s": float(vr.report.t_total)}
                        (out / "docs" / f"{dk}.json").write_text(json.dumps(doc))
    (out / "index.json").write_text(json.dumps({"candidates": index, "docs": docs}, indent=1))
    print(f"{len(index)} candidates, {len(docs)} distinct stage documents "
          f"({time.perf_counter() - t0:.1f} s) -> {out}")


def _run_rank(a):
    """Inside torchrun: execute every document for this world size."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2201_12023_b200.runtime import Executor
    d = Path(a.dir)
    idx = json.loads((d / "index.json").read_text())
    out = {}
    for dk, meta in sorted(idx["docs"].items()):
        if meta["devices"] != world:
            continue
        doc = json.loads((d / "docs" / f"{dk}.json").read_text())
        B = int(doc["num_microbatches"])
        ex = Executor(doc, schedule="1f1b", seed=7)
        for _ in range(a.warmup):
            ex.step()
        ts = []
        for _ in range(a.steps):
            ex.barrier()
            ts.append(ex.step())
        t = sorted(ts)[len(ts) // 2] / B
        out[dk] = t
        if rank == 0:
            print(json.dumps({"doc": dk, "layers": meta["layers"], "view": meta["view"],
                              "measured_s": t, "modeled_s": meta["modeled_s"]}), flush=True)
        ex.comm.close()
        del ex
        torch.cuda.empty_cache()
    if rank == 0:
        (d / f"measured_{world}.json").write_text(json.dumps(out, indent=1))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def cmd_run(a):
    if "WORLD_SIZE" in os.environ:
        return _run_rank(a)
    d = Path(a.dir)
    idx = json.loads((d / "index.json").read_text())
    import torch
    have = torch.cuda.device_count()
    sizes = sorted({m["devices"] for m in idx["docs"].values()})
    for n in sizes:
        if n > have:
            print(f"skip {n}-device documents: {have} GPUs", flush=True)
            continue
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
               "--master-port", str(29700 + n), __file__, "run", str(d),
               "--steps", str(a.steps), "--warmup", str(a.warmup)]
        subprocess.run(cmd, check=True, env={**os.environ, "PYTHONPATH": str(ROOT)})
    merged = {}
    for n in sizes:
        f = d / f"measured_{n}.json"
        if f.exists():
            merged.update(json.loads(f.read_text()))
    (d / "measured.json").write_text(json.dumps(merged, indent=1))
    print(f"{len(merged)} of {len(idx['docs'])} stage documents measured")


def cmd_plan(a):
    mp = _ref(a.reference_src)
    from meshplan import cli
    from paper_2201_12023_b200 import ilp, profiling
    ilp.patch_reference(mp)
    d = Path(a.dir)
    idx = json.loads((d / "index.json").read_text())
    measured = json.loads((d / "measured.json").read_text())
    profiling.patch_reference(mp, idx["candidates"], measured, strict=not (a.lenient or a.measured_only),
                              missing="exclude" if a.measured_only else "model")
    rest = a.rest[1:] if a.rest[:1] == ["--"] else a.rest
    return cli.main(["plan", *rest, "--out", a.out])


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    e = sub.add_parser("emit")
    e.add_argument("--builder", default=None)
    e.add_argument("--graph", default=None, help="reference graph JSON (e.g. from builders.py)")
    e.add_argument("--cluster", required=True)
    e.add_argument("--layers", type=int, required=True)
    e.add_argument("--microbatches", type=int, default=2)
    e.add_argument("--max-devices", type=int, default=1 << 30,
                   help="only candidates on submeshes of at most this many devices")
    e.add_argument("--out", required=True)
    e.add_argument("--reference-src", default="/root/reference/pkg/src")
    r = sub.add_parser("run")
    r.add_argument("dir")
    r.add_argument("--steps", type=int, default=3)
    r.add_argument("--warmup", type=int, default=1)
    p = sub.add_parser("plan")
    p.add_argument("dir")
    p.add_argument("--out", required=True)
    p.add_argument("--lenient", action="store_true",
                   help="keep the analytic cost for candidates without a measurement")
    p.add_argument("--measured-only", action="store_true",
                   help="candidates without a measurement are inadmissible (infinite cost)")
    p.add_argument("--reference-src", default="/root/reference/pkg/src")
    p.add_argument("rest", nargs=argparse.REMAINDER)
    a = ap.parse_args()
    return {"emit": cmd_emit, "run": cmd_run, "plan": cmd_plan}[a.cmd](a)


if __name__ == "__main__":
    sys.exit(main() or 0)
