"""Golden modeled makespans: the reference simulator (`simulate`, sim.py:91-188,
modeled and zero transfers, memory not enforced) on every committed plan x
schedule.  Run HERE (needs /root/reference); the output is committed.

  python tests/golden/make_sim_golden.py
"""
import glob
import gzip
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True


def main():
    import meshplan
    out = {}
    for f in sorted(glob.glob(str(ROOT / "plans/*/plan.json"))):
        doc = json.loads(Path(f).read_text())
        rt = meshplan.planio.runtime_from_json(doc)
        name = Path(f).parent.name
        out[name] = {}
        for sch in ("gpipe", "1f1b"):
            prog = meshplan.emit_instructions(rt, sch)
            cm = meshplan.CostModel(rt.cluster)
            for zero in (False, True):
                m = meshplan.simulate(prog, cm, zero_transfer=zero, enforce_memory=False).makespan
                out[name][f"{sch}{'_zero' if zero else ''}"] = [m.numerator, m.denominator]
    (ROOT / "tests/golden/sim_makespans.json").write_text(json.dumps(out, indent=0, sort_keys=True))
    print(len(out), "plans")
    # the reference's sim.json / gantt.json documents (cli.py:190-194) for two
    # plans: the executor's trace_json / gantt_rows must have their shape
    traces = {}
    for name in ("cfg1", "tiny_gpt_n2"):
        doc = json.loads((ROOT / "plans" / name / "plan.json").read_text())
        rt = meshplan.planio.runtime_from_json(doc)
        prog = meshplan.emit_instructions(rt, "1f1b")
        res = meshplan.simulate(prog, meshplan.CostModel(rt.cluster), enforce_memory=False)
        traces[name] = {"sim": json.loads(res.trace_json()), "gantt": res.gantt_rows(prog)}
    with gzip.open(ROOT / "tests/golden/sim_traces.json.gz", "wt") as f:
        json.dump(traces, f, sort_keys=True)


if __name__ == "__main__":
    main()
