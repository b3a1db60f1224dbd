"""Native intra-op ILP solver against the reference solver:
identical choice, exact objective and certified flag — on random tables with
integer and rational costs, with tight budgets (non-certified searches must stop
at the same node), edges in both orientations, and on real stage ILPs built by
the reference planner.  CPU only (the solver is host code in libmpexec)."""
import gzip
import json
import random
from fractions import Fraction
from pathlib import Path

import pytest

GOLD = Path(__file__).resolve().parent / "golden" / "ilp_tables.json.gz"


class Table:
    """Minimal StrategyTable stand-in (the fields solve_ilp reads)."""

    def __init__(self, c, d, edges):
        self.c, self.d, self.edges = c, d, edges

    @property
    def num_nodes(self):
        return len(self.c)

    def k(self, i):
        return len(self.c[i])

    def evaluate(self, choice):
        total = Fraction(0)
        for i, j in enumerate(choice):
            total += self.c[i][j] + self.d[i][j]
        for u, v, m in self.edges:
            total += m[choice[u]][choice[v]]
        return total


def rand_table(rng, n, max_k, edge_prob=0.6, rational=False, flip=False):
    ks = [rng.randint(1, max_k) for _ in range(n)]

    def val():
        if rational:
            return Fraction(rng.randint(0, 50), rng.choice([1, 3, 7, 900000000000, 100000]))
        return Fraction(rng.randint(0, 50))
    c = [[val() for _ in range(k)] for k in ks]
    d = [[Fraction(0)] * k for k in ks]
    edges = []
    for u in range(n):
        for v in range(u + 1, n):
            if rng.random() < edge_prob:
                a, b = (v, u) if flip and rng.random() < 0.5 else (u, v)
                edges.append((a, b, [[val() for _ in range(ks[b])] for _ in range(ks[a])]))
    return Table(c, d, edges)


def native_solve(table, budget):
    import sys
    import types
    from paper_2201_12023_b200 import ilp
    # the wrapper builds the reference's IntraPlan from the table's module
    mod = types.ModuleType("fake_intra")

    class IntraPlan:
        def __init__(self, table, choice, objective, certified):
            self.choice, self.objective, self.certified = choice, objective, certified
    mod.IntraPlan = IntraPlan
    sys.modules["fake_intra"] = mod
    Table.__module__ = "fake_intra"
    return ilp.solve_ilp(table, budget)


def enc(table):
    f = lambda x: [x.numerator, x.denominator]
    return {"c": [[f(x) for x in row] for row in table.c],
            "edges": [[u, v, [[f(x) for x in row] for row in m]] for u, v, m in table.edges]}


def dec(doc):
    f = lambda p: Fraction(p[0], p[1])
    c = [[f(x) for x in row] for row in doc["c"]]
    return Table(c, [[Fraction(0)] * len(r) for r in c],
                 [(u, v, [[f(x) for x in row] for row in m]) for u, v, m in doc["edges"]])


def test_native_matches_golden_reference_results():
    with gzip.open(GOLD, "rt") as fh:
        cases = json.load(fh)
    assert len(cases) >= 40
    for case in cases:
        t = dec(case["table"])
        got = native_solve(t, case["budget"])
        assert got.choice == case["choice"], case["budget"]
        assert got.objective == Fraction(*case["objective"])
        assert got.certified == case["certified"]


@pytest.mark.reference
@pytest.mark.parametrize("seed", range(12))
def test_native_matches_reference_random(meshplan_ref, seed):
    from meshplan.intra import solve_ilp
    rng = random.Random(seed)
    for trial in range(10):
        t = rand_table(rng, rng.randint(1, 12), 7, rational=trial % 2 == 1, flip=trial % 3 == 0)
        for budget in (3, 50, 200_000):
            ref = solve_ilp(t, budget)
            got = native_solve(t, budget)
            assert (got.choice, got.objective, got.certified) == \
                (ref.choice, ref.objective, ref.certified), (seed, trial, budget)


@pytest.mark.reference
def test_native_matches_reference_on_real_stage_ilps(meshplan_ref):
    """Stage ILPs the reference planner builds for a 1-block GPT on (1,4) views."""
    from meshplan.costs import CostModel
    from meshplan.graph import build_transformer_blocks
    from meshplan.intra import build_ilp, extract_stage, merge_trivial, solve_ilp
    from meshplan.mesh import ClusterMesh, SubmeshShape, logical_views
    from meshplan.sharding import SpecError
    import sys
    from paper_2201_12023_b200 import ilp
    g = build_transformer_blocks(1, 2, 32, 64, 4, elem_bytes=2, backward=True)
    cl = ClusterMesh(1, 4, 900 * 10**9, 900 * 10**9, Fraction(1, 100000), 14 * 10**14, 18 * 10**10)
    cm = CostModel(cl)
    merged = merge_trivial(extract_stage(g, range(len(g))))
    n_checked = 0
    for view in logical_views(SubmeshShape(1, 4), cl):
        try:
            table = build_ilp(merged, view, cm)
        except SpecError:
            continue
        for budget in (1000, 200_000):
            ref = solve_ilp(table, budget)
            got = ilp.solve_ilp(table, budget)
            assert got.choice == ref.choice and got.objective == ref.objective
            assert got.certified == ref.certified
            n_checked += 1
    assert n_checked >= 4


@pytest.mark.reference
def test_native_table_equals_reference_table(meshplan_ref):
    """ilp.build_ilp (int64 edge assembly, memoised algorithms / costs) builds the
    reference's strategy table entry for entry: same algorithms, node costs and
    exact edge-matrix Fractions on every view of a 1-block GPT on (1,2) and (1,4)."""
    from meshplan.costs import CostModel
    from meshplan.graph import build_transformer_blocks
    from meshplan.intra import build_ilp, extract_stage, merge_trivial, solve_ilp
    from meshplan.mesh import ClusterMesh, SubmeshShape, logical_views
    from meshplan.sharding import SpecError
    from paper_2201_12023_b200 import ilp
    g = build_transformer_blocks(1, 2, 32, 64, 4, elem_bytes=2, backward=True)
    checked = 0
    for m in (2, 4):
        cl = ClusterMesh(1, m, 900 * 10**9, 900 * 10**9, Fraction(1, 100000), 14 * 10**14,
                         18 * 10**10)
        cm = CostModel(cl)
        merged = merge_trivial(extract_stage(g, range(len(g))))
        for view in logical_views(SubmeshShape(1, m), cl):
            try:
                ref = build_ilp(merged, view, cm)
            except SpecError:
                continue
            got = ilp.build_ilp(merged, view, cm)
            assert got.algorithms == ref.algorithms and got.c == ref.c and got.d == ref.d
            assert [(u, v) for u, v, _ in got.edges] == [(u, v) for u, v, _ in ref.edges]
            for (_, _, gm), (_, _, rm) in zip(got.edges, ref.edges):
                assert [list(r) for r in gm] == [list(r) for r in rm]
            a, b = ilp.solve_ilp(got), solve_ilp(ref)
            assert (a.choice, a.objective, a.certified) == (b.choice, b.objective, b.certified)
            assert got.evaluate(a.choice) == ref.evaluate(b.choice)
            checked += 1
    assert checked >= 4


@pytest.mark.reference
@pytest.mark.parametrize("builder,cluster,b,layers", [
    ("mlp:layers=2,batch=64,hidden=1024,backward=1", "b200_1x4.json", 4, 2),
    ("transformer:blocks=1,batch=2,seq=32,hidden=64,heads=4,elem_bytes=2,backward=1",
     "b200_1x4.json", 3, 1),
])
def test_patched_planner_writes_identical_plans(meshplan_ref, tmp_path, builder, cluster, b,
                                                layers):
    """The whole reference planner with the native table + solver swapped in
    writes the same plan.json bytes as the untouched planner."""
    import subprocess
    import sys
    root = Path(__file__).resolve().parent.parent
    outs = {}
    for mode in ("native", "python"):
        cmd = [sys.executable, str(root / "scripts/plan_native.py")]
        if mode == "python":
            cmd.append("--python-solver")
        cmd += ["--", "plan", "--builder", builder, "--cluster",
                str(root / "plans/clusters" / cluster), "--b", str(b), "--layers", str(layers),
                "--epsilon", "0", "--schedule", "1f1b", "--out", str(tmp_path / mode)]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900,
                           env={**__import__("os").environ, "PYTHONPATH": str(root)})
        assert r.returncode == 0, r.stderr[-2000:]
        outs[mode] = (tmp_path / mode / "plan.json").read_bytes()
    assert outs["native"] == outs["python"]
