"""Find the first node producing a non-finite value in an executor step."""
import json, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
from paper_2201_12023_b200.runtime import Executor

doc = json.loads((ROOT / (sys.argv[1] if len(sys.argv) > 1 else "plans/gpt13b_n1/plan.json")).read_text())
doc["num_microbatches"] = 1
ex = Executor(doc, schedule="1f1b")
r = ex.runner
orig = r.compute
def checked(phase, mb):
    vals = r.vals.setdefault(mb, {})
    for op in (r.fwd_ops if phase == "fwd" else r.bwd_ops):
        before = set(vals)
        # run a single op by temporarily narrowing the op list
        saved = (r.fwd_ops, r.bwd_ops)
        if phase == "fwd": r.fwd_ops = [op]
        else: r.bwd_ops = [op]
        orig(phase, mb)
        r.fwd_ops, r.bwd_ops = saved
        v = vals.get(op.nid)
        if v is not None:
            f = v.float()
            if not torch.isfinite(f).all():
                print("NONFINITE at", phase, op.nid, op.op, [ (p, str(s)) for p, s in op.ins], tuple(v.shape), flush=True)
                for p, s in op.ins:
                    x = r.value(mb, p).float()
                    print("   input", p, float(x.abs().max()), bool(torch.isfinite(x).all()))
                sys.exit(1)
    return None
r.compute = checked
for step in range(3):
    ex.step()
    print("step", step, "loss", ex.loss(), "gradnorm", float(r.gradbuf.norm()), "param absmax", float(r.master.abs().max()), flush=True)
