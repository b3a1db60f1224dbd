"""Profile-driven stage costs: the single-stage documents that
`scripts/profile_stages.py` executes are valid plans of the same computation,
and the planner patch swaps in measured times.  CPU only."""
import json
import sys
import types
from fractions import Fraction
from pathlib import Path

import pytest

from paper_2201_12023_b200 import profiling
from paper_2201_12023_b200.binding import bind
from paper_2201_12023_b200.plan import load_plan
from paper_2201_12023_b200.schedule import build_program

ROOT = Path(__file__).resolve().parent.parent


def _stage_of(doc, idx):
    st = doc["stages"][idx]
    return [int(i) for i in st["op_ids"]], {int(k): v for k, v in st["op_specs"].items()}, \
        tuple(st["logical_view"])


@pytest.mark.parametrize("plan,idx", [("tiny_gpt_n2", 0), ("tiny_gpt_n2", 1),
                                      ("tiny_gpt_tp_n4", 1), ("mlp_n2", 0)])
def test_stage_doc_is_a_runnable_plan(plan, idx):
    doc = json.loads((ROOT / "plans" / plan / "plan.json").read_text())
    ops, specs, view = _stage_of(doc, idx)
    members = [i for i in ops if doc["graph"]["nodes"][i]["kind"] != "input"]
    sd = profiling.stage_doc(doc["graph"], members, view, specs, num_microbatches=2)
    p = load_plan(sd)
    prog = build_program(p, "1f1b")
    assert len(p.stages) == 1 and p.num_devices == view[0] * view[1]
    g = p.graph
    nodes = doc["graph"]["nodes"]
    n_ext = sum(1 for n in sd["graph"]["nodes"] if n["kind"] == "input")
    # every member kept with its kind, dims, colocation and grad_of structure
    assert len(g) == n_ext + len(members)
    for k, orig in enumerate(members):
        n = sd["graph"]["nodes"][n_ext + k]
        assert n["kind"] == nodes[orig]["kind"]
        assert n["shape"]["dims"] == nodes[orig]["shape"]["dims"]
        assert ("grad_of" in n) == (nodes[orig].get("grad_of") is not None)
    assert any(g[i].colocate_with is not None for i in range(len(g)))   # backward kept
    bind(g)                                                              # numerically bound
    assert prog.stages[0].instructions                                   # fwd + bwd program
    # same computation -> same key; a different view -> a different key
    assert profiling.doc_key(sd) == profiling.doc_key(
        profiling.stage_doc(doc["graph"], members, view, specs, num_microbatches=2))


def test_patch_reference_swaps_in_measured_times():
    from dataclasses import dataclass

    @dataclass(frozen=True)
    class Report:
        t_compute: Fraction
        t_comm: Fraction

        @property
        def t_total(self):
            return self.t_compute + self.t_comm

    @dataclass(frozen=True)
    class View:
        n_l: int
        m_l: int

    @dataclass(frozen=True)
    class VR:
        view: View
        report: Report

    @dataclass(frozen=True)
    class Ev:
        sub: object
        views: tuple

    @dataclass(frozen=True)
    class Shape:
        n: int
        m: int

    def evaluate_stage(graph, ops, shape, cluster, cm):
        return Ev(None, (VR(View(1, 2), Report(Fraction(1), Fraction(2))),
                         VR(View(2, 1), Report(Fraction(3), Fraction(4)))))
    inter = types.SimpleNamespace(evaluate_stage=evaluate_stage)
    pkg = types.SimpleNamespace(inter=inter)
    ops = [5, 6, 7]
    idx = {profiling.candidate_key(ops, (1, 2), (1, 2)): "a",
           profiling.candidate_key(ops, (1, 2), (2, 1)): "b"}
    profiling.patch_reference(pkg, idx, {"a": 0.25, "b": 0.5})
    ev = inter.evaluate_stage(None, ops, Shape(1, 2), None, None)
    assert [v.report.t_total for v in ev.views] == [Fraction(1, 4), Fraction(1, 2)]
    with pytest.raises(KeyError):
        profiling.patch_reference(pkg, {}, {})
        inter.evaluate_stage(None, [1], Shape(1, 1), None, None)


@pytest.mark.reference
def test_cross_stage_cost_in_dp(meshplan_ref, tmp_path):
    """with the cross-stage receive time inside the DP, config 1
    plans one (1,4) stage whose T* equals the reference simulator's makespan
    with modeled transfers (the plain planner's T* is 71% low)."""
    import subprocess
    import sys
    res = subprocess.run([sys.executable, str(ROOT / "scripts/plan_cross_stage.py"),
                          "--builder", "mlp:layers=2,batch=64,hidden=1024,backward=1",
                          "--cluster", str(ROOT / "plans/clusters/b200_1x4.json"), "--b", "4",
                          "--out", str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    s = json.loads((tmp_path / "summary.json").read_text())
    assert len(s["plain"]["stages"]) == 2 and s["plain"]["t_star_error_vs_sim"] > 1.0
    assert len(s["cross_stage"]["stages"]) == 1
    assert abs(s["cross_stage"]["t_star_error_vs_sim"]) < 1e-9
    assert s["cross_stage"]["sim_makespan_s"] < 0.6 * s["plain"]["sim_makespan_s"]
