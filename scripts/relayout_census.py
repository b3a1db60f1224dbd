"""Which relayouts a stage pays per microbatch, decided on the host
exactly as the executor decides them (StageRunner._compile + _relayout_plan),
without a GPU:  python scripts/relayout_census.py plans/gpt13b_n4_tp/plan.json"""
import argparse
import json
import math
import sys
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2201_12023_b200 import runtime  # noqa: E402
from paper_2201_12023_b200.plan import format_spec, load_plan  # noqa: E402
from paper_2201_12023_b200.schedule import build_program  # noqa: E402


def census(plan_path, device):
    plan = load_plan(plan_path)
    prog = build_program(plan, "1f1b")
    r = runtime.StageRunner.__new__(runtime.StageRunner)
    r.plan, r.graph, r.program, r.me = plan, plan.graph, prog, device
    r.st = plan.stage_of_device(device)
    r.mesh = r.st.mesh
    r.sprog = prog.stages[r.st.index]
    r.bound = runtime.bind(plan.graph)
    r.cons = plan.graph.consumers()
    r._moves_cache, r._plans = {}, {}
    r.op_timer, r.relayout_timer = None, []
    r._pf, r.pf_stream, r.pf_learn = False, None, {}
    r._compile()
    rows = Counter()
    nbytes = Counter()
    for phase, ops in (("fwd", r.fwd_ops), ("bwd", r.bwd_ops)):
        for op in ops:
            for nid, req in op.ins:
                if nid in r.pviews if hasattr(r, "pviews") else False:
                    continue
                have = r.have_spec(nid)
                req = runtime.canonical(req, r.mesh)
                if have == req:
                    continue
                kind, _ = r._relayout_plan(tuple(r.graph[nid].dims), have, req)
                if kind == "local":
                    continue
                key = (phase, kind, r.bound[nid].op, r.bound[op.nid].op, format_spec(have),
                       format_spec(req), tuple(r.graph[nid].dims))
                rows[key] += 1
                nbytes[key] += math.prod(r.graph[nid].dims) * 2
    return r, rows, nbytes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("plan")
    ap.add_argument("--device", type=int, default=0)
    a = ap.parse_args()
    r, rows, nbytes = census(a.plan, a.device)
    print(f"stage {r.st.index} mesh {r.mesh} fused attention {len(r.attn_clusters)} "
          f"epilogues {r.fused_epilogues} token-split dW {len(r.tok_dw)}")
    tot = sum(nbytes.values())
    print(f"non-local relayouts per microbatch: {sum(rows.values())}, "
          f"{tot / 2**20:.0f} MiB of global tensors")
    for key, n in sorted(rows.items(), key=lambda kv: -nbytes[kv[0]]):
        print(f"{n:3d} x {nbytes[key] / n / 2**20:7.1f} MiB  {key}")


if __name__ == "__main__":
    main()
