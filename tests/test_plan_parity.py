"""Plan-level parity (CPU): the executor's index plans, algorithms and programs
are bit-exact with the reference — pinned by the golden fixtures generated from
the live reference (tests/golden/make_golden.py), and re-checked live when
/root/reference is mounted.  The oracle's own restatements are pinned too."""
import gzip
import itertools
import json
import random
from pathlib import Path

import numpy as np
import pytest

from paper_2201_12023_b200.layout import matmul_algo, relayout_moves
from paper_2201_12023_b200.plan import (Mesh, load_plan, parse_spec, format_spec, shard_box,
                                        local_dims, device_box)
from paper_2201_12023_b200.schedule import build_program
from paper_2201_12023_b200.xmesh import cross_mesh_plan

GOLD = Path(__file__).resolve().parent / "golden"
ROOT = GOLD.parent.parent


def load(name):
    with gzip.open(GOLD / name, "rt") as f:
        return json.load(f)


def mesh(view, first):
    n, m = view
    return Mesh(n, m, tuple(range(first, first + n * m)))


XMESH = load("xmesh.json.gz")


def test_golden_xmesh_count():
    assert len(XMESH) > 800


@pytest.mark.parametrize("chunk", range(8))
def test_xmesh_matches_reference(chunk):
    for c in XMESH[chunk::8]:
        p = cross_mesh_plan(tuple(c["dims"]), c["elem_bytes"], parse_spec(c["src_spec"]),
                            mesh(c["src_view"], c["src_first"]), parse_spec(c["dst_spec"]),
                            mesh(c["dst_view"], c["dst_first"]), c["optimize"])
        got_t = [[t.src_device, t.dst_device, t.nbytes, [list(b) for b in t.box]]
                 for t in p.transfers]
        got_g = [[list(g.devices), list(g.axes), g.nbytes] for g in p.gathers]
        assert got_t == c["transfers"], c
        assert got_g == c["gathers"], c
        assert p.inter_mesh_bytes == c["inter_mesh_bytes"]


def test_oracle_xmesh_matches_reference():
    from oracle import ir, sharded

    class St:
        def __init__(self, view, first):
            self.n, self.m = view
            self.ext = tuple(view)
            self.devices = tuple(range(first, first + view[0] * view[1]))

        def coords(self, d):
            return divmod(self.devices.index(d), self.m)
    for c in XMESH[::3]:
        s, d = St(c["src_view"], c["src_first"]), St(c["dst_view"], c["dst_first"])
        ss = ir.canon(ir.spec_parse(c["src_spec"]), s.ext)
        ds = ir.canon(ir.spec_parse(c["dst_spec"]), d.ext)
        trans, gath = sharded.xmesh(tuple(c["dims"]), ss, s, ds, d, c["optimize"])
        assert [[a, b, [list(x) for x in box]] for a, b, box in trans] == \
            [[t[0], t[1], t[3]] for t in c["transfers"]]
        assert [list(g[0]) for g in gath] == [g[0] for g in c["gathers"]]


def test_shard_boxes_match_reference():
    from oracle import ir
    for c in load("boxes.json.gz"):
        m = mesh(c["view"], 0)
        spec = parse_spec(c["spec"])
        got = [[list(b) for b in shard_box(tuple(c["dims"]), spec, m, (i, j))]
               for i in range(m.n) for j in range(m.m)]
        assert got == c["boxes"]
        ospec = ir.spec_parse(c["spec"])
        got2 = [[list(b) for b in ir.box_of(tuple(c["dims"]), ospec, (m.n, m.m), (i, j))]
                for i in range(m.n) for j in range(m.m)]
        assert got2 == c["boxes"]


def test_matmul_algorithm_recovered_from_output_spec():
    """Every reference algorithm is determined by its output spec
    (sharding.py:264-291): same input specs, all_reduce over the k axes."""
    cases = load("algorithms.json.gz")
    assert len(cases) > 100
    seen = {}
    for c in cases:
        m = mesh(c["view"], 0)
        key = (tuple(c["view"]), c["kind"], c["out"])
        assert key not in seen, f"two algorithms share output spec {key}"
        seen[key] = c
        algo = matmul_algo(c["kind"] == "batched_matmul", parse_spec(c["out"]), m)
        assert [format_spec(s) for s in algo.in_specs] == c["in"]
        if c["comm"]:
            assert c["comm"][0][0] == "all_reduce"
            assert tuple(c["comm"][0][2]) == algo.k_axes
        else:
            assert algo.k_axes == ()


PROGRAMS = sorted((GOLD / "programs").glob("*.json.gz"))


@pytest.mark.parametrize("path", PROGRAMS, ids=[p.name for p in PROGRAMS])
def test_program_matches_reference(path):
    doc = load(f"programs/{path.name}")
    name, sched = path.name.split(".")[:2]
    if name.startswith("synthetic"):
        plan_doc, ref = doc["plan"], doc["program"]
    else:
        plan_doc, ref = json.loads((ROOT / "plans" / name / "plan.json").read_text()), doc
    prog = build_program(load_plan(plan_doc), sched)
    assert prog.to_json() == ref


@pytest.mark.parametrize("view", [(1, 2), (2, 1), (2, 2), (1, 4), (2, 4), (4, 2), (1, 8)])
def test_relayout_moves_materialise_every_spec_pair(view):
    """Applying the moves to a global arange gives every device exactly its
    destination tile (the literal realisation resharding_cost only costs)."""
    from oracle import ir
    m = mesh(view, 0)
    dims = (8, 16) if view != (2, 4) else (8, 8, 16)
    glob = np.arange(np.prod(dims)).reshape(dims)
    from paper_2201_12023_b200.plan import Spec
    specs = _all_specs(len(dims), m, dims)
    for src, dst in itertools.product(specs, repeat=2):
        held = {d: glob[ir.sl(device_box(dims, src, m, d))] for d in m.device_ids}
        got = {d: np.full(local_dims(dims, dst, m), -1) for d in m.device_ids}
        for mv in relayout_moves(dims, src, dst, m):
            sb = device_box(dims, src, m, mv.src)
            db = device_box(dims, dst, m, mv.dst)
            got[mv.dst][ir.sl(mv.box, [b[0] for b in db])] = held[mv.src][ir.sl(mv.box, [b[0] for b in sb])]
        for d in m.device_ids:
            assert np.array_equal(got[d], glob[ir.sl(device_box(dims, dst, m, d))]), (src, dst, d)


@pytest.mark.parametrize("view", [(1, 2), (2, 1), (2, 2), (1, 4), (2, 4), (4, 2), (1, 8)])
def test_allgather_fast_path_is_exact(view):
    """Whenever the all-gather fast path is taken, gathering the have-tiles of
    the axis group in device-id order reproduces exactly the target tile."""
    from oracle import ir
    from paper_2201_12023_b200.layout import allgather_axes
    m = mesh(view, 0)
    dims = (8, 16)
    glob = np.arange(np.prod(dims)).reshape(dims)
    hits = [0, 0]
    for src, dst in itertools.product(_all_specs(2, m, dims), repeat=2):
        for cdim in (0, 1):         # dim 0: straight into the output; dim 1: staged + permuted
            axes = allgather_axes(dims, src, dst, m, dim=cdim)
            if axes is None:
                continue
            hits[cdim] += 1
            for d in m.device_ids:
                grp = m.axis_group(d, axes)
                tiles = [glob[ir.sl(device_box(dims, src, m, e))] for e in grp]
                cat = np.concatenate(tiles, cdim)
                assert np.array_equal(cat, glob[ir.sl(device_box(dims, dst, m, d))])
                # the executor's staging: (g, *tile) -> move g next to cdim -> merge
                stage = np.stack(tiles, 0)
                perm = np.moveaxis(stage, 0, cdim)
                merged = perm.reshape(cat.shape)
                assert np.array_equal(merged, cat)
    assert hits[0] > 0 and hits[1] > 0


def _all_specs(rank, m, dims):
    from paper_2201_12023_b200.plan import Spec
    out = set()
    axes = [a for a in (0, 1) if m.extent(a) > 1]
    choices = [None] + list(range(rank))
    for assign in itertools.product(choices, repeat=len(axes)):
        for order in itertools.permutations(axes):
            d = [[] for _ in range(rank)]
            for a in order:
                k = assign[axes.index(a)]
                if k is not None:
                    d[k].append(a)
            sp = Spec(tuple(tuple(x) for x in d))
            if all(e % m.group_extent(ax) == 0 for e, ax in zip(dims, sp.dims)):
                out.add(sp)
    return sorted(out, key=format_spec)


# --------------------------------------------------------------- live reference
@pytest.mark.reference
def test_live_reference_programs_and_boundaries(meshplan_ref):
    from meshplan.planio import runtime_from_json
    from meshplan.reshard import _stage_boundaries, emit_instructions
    for p in sorted((ROOT / "plans").glob("*/plan.json")):
        doc = json.loads(p.read_text())
        rt = runtime_from_json(doc)
        plan = load_plan(doc)
        for sched in ("gpipe", "1f1b"):
            assert build_program(plan, sched).to_json() == emit_instructions(rt, sched).to_json()
        ref_b = _stage_boundaries(rt)
        mine = build_program(plan, "1f1b").boundaries
        assert [(b.producer, b.consumer, b.recv_bytes) for b in ref_b] == \
            [(b.producer, b.consumer, b.recv_bytes) for b in mine]
        for rb, mb in zip(ref_b, mine):
            assert [(t.src_device, t.dst_device, t.nbytes, t.box) for t in rb.plan.transfers] == \
                [(t.src_device, t.dst_device, t.nbytes, t.box) for t in mb.transfers]
            assert [(g.devices, g.axes, g.nbytes) for g in rb.plan.gathers] == \
                [(g.devices, g.axes, g.nbytes) for g in mb.gathers]


@pytest.mark.reference
def test_live_reference_random_xmesh(meshplan_ref):
    from fractions import Fraction
    from meshplan.graph import TensorShape
    from meshplan.mesh import LogicalMesh
    from meshplan.reshard import cross_mesh_plan as ref_xmesh
    from meshplan.sharding import enumerate_specs
    rng = random.Random(7)
    views = [(1, 1), (1, 2), (2, 1), (2, 2), (1, 4), (4, 1), (2, 4), (4, 2), (1, 8)]
    for _ in range(300):
        sv, dv = rng.choice(views), rng.choice(views)
        dims = tuple(rng.choice([8, 10, 12, 16]) for _ in range(rng.choice([2, 3])))
        shape = TensorShape(dims, 2)
        rs = LogicalMesh(*sv, (Fraction(1), Fraction(1)), tuple(range(sv[0] * sv[1])))
        rd = LogicalMesh(*dv, (Fraction(1), Fraction(1)), tuple(range(32, 32 + dv[0] * dv[1])))
        ss = rng.choice(enumerate_specs(shape, rs))
        ds = rng.choice(enumerate_specs(shape, rd))
        opt = rng.random() < 0.7
        r = ref_xmesh(shape, ss, rs, ds, rd, optimize=opt)
        p = cross_mesh_plan(dims, 2, parse_spec(format_spec_ref(ss)), Mesh(*sv, rs.device_ids),
                            parse_spec(format_spec_ref(ds)), Mesh(*dv, rd.device_ids), opt)
        assert [(t.src_device, t.dst_device, t.nbytes, t.box) for t in r.transfers] == \
            [(t.src_device, t.dst_device, t.nbytes, t.box) for t in p.transfers]
        assert [(g.devices, g.axes, g.nbytes) for g in r.gathers] == \
            [(g.devices, g.axes, g.nbytes) for g in p.gathers]


def format_spec_ref(spec):
    from meshplan.sharding import format_spec as f
    return f(spec)


def test_modeled_makespan_equals_reference_simulator():
    """schedule.modeled_makespan restates the reference simulator's timing rules
    (sim.py:91-188): exact rational equality with the reference's own makespan
    (golden, tests/golden/make_sim_golden.py) on every committed plan x schedule,
    modeled and zero transfers."""
    from fractions import Fraction
    from paper_2201_12023_b200.plan import load_plan
    from paper_2201_12023_b200.schedule import build_program, modeled_makespan
    gold = json.loads((ROOT / "tests/golden/sim_makespans.json").read_text())
    assert len(gold) >= 30
    for name, per in gold.items():
        plan = load_plan(ROOT / "plans" / name / "plan.json")
        for sch in ("gpipe", "1f1b"):
            prog = build_program(plan, sch)
            for zero in (False, True):
                want = Fraction(*per[f"{sch}{'_zero' if zero else ''}"])
                assert modeled_makespan(prog, plan, zero_transfer=zero) == want, (name, sch, zero)
