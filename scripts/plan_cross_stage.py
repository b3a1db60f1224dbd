"""plan with cross-stage transfer time inside the reference DP
(profiling.patch_cross_stage) and compare with the plain planner: T* of each
plan next to the reference simulator's makespan with modeled transfers
(`simulate(..., zero_transfer=False)`, sim.py:91-188) -- the quantity T* is
meant to predict.  Run HERE (needs /root/reference).

  python scripts/plan_cross_stage.py --builder mlp:layers=2,batch=64,hidden=1024,backward=1 \\
      --cluster plans/clusters/b200_1x4.json --b 4 --out profiles/f4_cross_stage/cfg1
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.dont_write_bytecode = True


def _strip_cross_stage(doc):
    """The cross-stage plan's stage times include the receive term; remove it so
    the simulator (which models transfers itself) sees the plain stage costs."""
    from fractions import Fraction
    from math import prod
    from paper_2201_12023_b200.plan import Mesh, local_dims, parse_spec
    cl = doc["cluster"]
    frac = lambda v: Fraction(v[0], v[1]) if isinstance(v, list) else Fraction(v)  # noqa: E731
    alpha, bw = frac(cl["alpha"]), frac(cl["inter_bw"])
    nodes = doc["graph"]["nodes"]
    for st in doc["stages"]:
        mesh = Mesh(st["logical_view"][0], st["logical_view"][1], tuple(st["device_ids"]))
        extra = Fraction(0)
        for k, spec in st["boundary_inputs"].items():
            n = nodes[int(k)]
            if n["kind"] == "parameter":
                continue
            nbytes = prod(local_dims(tuple(n["shape"]["dims"]), parse_spec(spec), mesh)) * \
                n["shape"]["elem_bytes"]
            extra += alpha + Fraction(nbytes) / bw
        t = Fraction(st["t"][0], st["t"][1]) - extra
        st["t"] = [t.numerator, t.denominator]
    return doc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reference-src", default="/root/reference/pkg/src")
    ap.add_argument("--builder", default=None)
    ap.add_argument("--graph", default=None)
    ap.add_argument("--cluster", required=True)
    ap.add_argument("--b", type=int, required=True)
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--schedule", default="1f1b")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    sys.path.insert(0, a.reference_src)
    import meshplan
    import meshplan.inter  # noqa: F401
    from meshplan import cli
    from paper_2201_12023_b200 import ilp, profiling
    ilp.patch_reference(meshplan)
    out = Path(a.out)
    res = {}
    for mode in ("plain", "cross_stage"):
        orig = profiling.patch_cross_stage(meshplan) if mode == "cross_stage" else None
        d = out / mode
        argv = ["plan", "--cluster", a.cluster, "--b", str(a.b), "--epsilon", "0",
                "--schedule", a.schedule, "--out", str(d)]
        argv += ["--builder", a.builder] if a.builder else ["--graph", a.graph]
        if a.layers:
            argv += ["--layers", str(a.layers)]
        t0 = time.perf_counter()
        rc = cli.main(argv)
        dt = time.perf_counter() - t0
        if orig is not None:
            meshplan.inter.evaluate_stage = orig
        if rc != 0:
            raise SystemExit(f"planner failed ({mode}): {rc}")
        doc = json.loads((d / "plan.json").read_text())
        if mode == "cross_stage":
            doc = _strip_cross_stage(doc)     # simulate on the same compute times
        rt = meshplan.runtime_from_json(doc) if hasattr(meshplan, "runtime_from_json") \
            else meshplan.planio.runtime_from_json(doc)
        prog = meshplan.emit_instructions(rt, a.schedule)
        cm = meshplan.CostModel(rt.cluster)
        sim = meshplan.simulate(prog, cm)
        simz = meshplan.simulate(prog, cm, zero_transfer=True)
        t_star = float(doc["t_star"][0]) / float(doc["t_star"][1])
        res[mode] = {
            "stages": [{"devices": s["device_ids"], "view": s["logical_view"],
                        "ops": len(s["op_ids"])} for s in doc["stages"]],
            "t_star_s": t_star,
            "sim_makespan_s": float(sim.makespan),
            "sim_makespan_zero_transfer_s": float(simz.makespan),
            "t_star_error_vs_sim": float(sim.makespan) / t_star - 1.0,
            "planner_s": dt,
        }
        print(mode, json.dumps(res[mode]), flush=True)
    (out / "summary.json").write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
