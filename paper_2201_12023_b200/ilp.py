"""Native drop-in for the reference's intra-op ILP solver.

`solve_ilp(table, budget)` has the signature and result of reference
intra.py:323-382: it takes the reference's StrategyTable and returns the
reference's IntraPlan (choice, exact Fraction objective, certified flag),
bit-identical to the Python branch-and-bound — the search runs in C++
(libmpexec mp_ilp_solve) on integers: every Fraction cost is scaled by the lcm
of all denominators, so every comparison is exact.  When the scaled values do
not fit the integer range, or the table has non-zero compute costs d (the
reference keeps them zero, intra.py:237), it falls back to the reference's own
solver.

`build_ilp(merged, mesh, cost_model)` is the drop-in for reference
intra.py:196-238 (the strategy table).  The same algorithms (enumerate_algorithms,
memoised per operator signature and logical view: it depends on nothing else),
the same node costs (collectives_time, memoised per collective list), and the
same edge matrices — but every matrix is assembled on int64 arrays: resharding
costs are computed once per distinct (src spec, dst spec, tensor) triple as exact
Fractions, scaled by the lcm D of all cost denominators, and each provenance
adds its [src spec of u's strategy i][dst spec of v's strategy j] gather to the
matrix.  The table keeps the reference's StrategyTable type; its edge matrices
are exact lazy views (entry [i][j] == Fraction(int, D)), so evaluate(), the
Python solver and export_lp see the same values, and solve_ilp hands the int64
arrays to the native branch and bound without any Fraction arithmetic.  Plans
stay byte-identical (tests/test_ilp_native.py).

`patch_reference(meshplan)` swaps both into a loaded reference planner so
`meshplan.cli plan` / `meshplan.plan` run unchanged but fast
(scripts/plan_native.py).
"""
from __future__ import annotations

import ctypes
import dataclasses
import math
import sys
from fractions import Fraction

import numpy as np

from . import native

_LIMIT = 1 << 62


def _scale(values):
    den = 1
    for v in values:
        den = den * v.denominator // math.gcd(den, v.denominator)
    return den


def _solve_scaled(table, budget, sc):
    """Native B&B on the table's int64 arrays (built by build_ilp)."""
    n = table.num_nodes
    k = np.asarray([len(row) for row in table.c], dtype=np.int32)
    u = np.asarray([e[0] for e in table.edges] or [0], dtype=np.int32)
    v = np.asarray([e[1] for e in table.edges] or [0], dtype=np.int32)
    costs, mats = sc["costs"], sc["mats"]
    choice = np.zeros(n, dtype=np.int32)
    obj = ctypes.c_int64()
    cert = ctypes.c_int()
    expl = ctypes.c_int64()
    ptr = lambda a, t: a.ctypes.data_as(ctypes.POINTER(t))          # noqa: E731
    rc = native.load().mp_ilp_solve(n, ptr(k, ctypes.c_int), ptr(costs, ctypes.c_int64),
                                    len(table.edges), ptr(u, ctypes.c_int), ptr(v, ctypes.c_int),
                                    ptr(mats, ctypes.c_int64), int(budget),
                                    ptr(choice, ctypes.c_int), ctypes.byref(obj),
                                    ctypes.byref(cert), ctypes.byref(expl))
    if rc != 0:
        raise native.NativeError(f"mp_ilp_solve failed (rc={rc})")
    intra = sys.modules[type(table).__module__]
    return intra.IntraPlan(table, [int(x) for x in choice], Fraction(obj.value, sc["den"]),
                           bool(cert.value))


def solve_ilp(table, budget: int = 200_000, _fallback=None):
    n = table.num_nodes
    if n == 0:
        raise ValueError("empty strategy table")
    sc = getattr(table, "_mp_scaled", None)
    if sc is not None:
        return _solve_scaled(table, budget, sc)
    if any(x != 0 for row in table.d for x in row):
        return _fallback(table, budget)
    flat_c = [Fraction(x) for row in table.c for x in row]
    flat_m = [Fraction(x) for _, _, m in table.edges for row in m for x in row]
    den = _scale(flat_c + flat_m)
    ints_c = [int(x * den) for x in flat_c]
    ints_m = [int(x * den) for x in flat_m]
    total = sum(max(abs(v) for v in row) for row in
                ([ints_c[i:i + 1] for i in range(len(ints_c))] or [[0]])) + sum(abs(v) for v in ints_m)
    if total >= _LIMIT or any(abs(v) >= _LIMIT for v in ints_c):
        return _fallback(table, budget)
    k = (ctypes.c_int * n)(*[len(row) for row in table.c])
    costs = (ctypes.c_int64 * len(ints_c))(*ints_c)
    ne = len(table.edges)
    u = (ctypes.c_int * max(ne, 1))(*[e[0] for e in table.edges])
    v = (ctypes.c_int * max(ne, 1))(*[e[1] for e in table.edges])
    mats = (ctypes.c_int64 * max(len(ints_m), 1))(*ints_m)
    choice = (ctypes.c_int * n)()
    obj = ctypes.c_int64()
    cert = ctypes.c_int()
    expl = ctypes.c_int64()
    rc = native.load().mp_ilp_solve(n, k, costs, ne, u, v, mats, int(budget), choice,
                                    ctypes.byref(obj), ctypes.byref(cert), ctypes.byref(expl))
    if rc != 0:
        raise native.NativeError(f"mp_ilp_solve failed (rc={rc})")
    intra = sys.modules[type(table).__module__]
    return intra.IntraPlan(table, list(choice), Fraction(obj.value, den), bool(cert.value))


# ----------------------------------------------------------------------------
# strategy table (reference intra.py:196-238)

class ScaledMatrix:
    """Exact lazy Fraction view of an int64 matrix in units of 1/den: row i,
    column j is Fraction(m[i, j], den) (what the reference's matrix holds)."""
    __slots__ = ("m", "den")

    def __init__(self, m, den):
        self.m, self.den = m, den

    def __len__(self):
        return self.m.shape[0]

    def __getitem__(self, i):
        return [Fraction(int(x), self.den) for x in self.m[i]]

    def __iter__(self):
        return (self[i] for i in range(len(self)))


_ALGS: dict = {}
_COLL: dict = {}
_RESH: dict = {}
_MESH_ID: dict = {}


class _SpecIds(dict):
    """ShardingSpec -> small int, with the inverse kept in _SPEC_OF.  Lookups
    go by object identity first (the memoised algorithms and propagated specs
    hand out the same objects again and again; hashing a spec is the slow part),
    by value otherwise; every object seen is kept alive so ids stay unique."""

    def setdefault(self, spec, n):
        sid = _SID_BY_OBJ.get(id(spec))
        if sid is not None:
            return sid
        sid = self.get(spec)
        if sid is None:
            sid = self[spec] = len(_SPEC_OF)
            _SPEC_OF.append(spec)
        _SID_BY_OBJ[id(spec)] = sid
        _KEEP.append(spec)
        return sid


_SID_BY_OBJ: dict = {}
_KEEP: list = []


_SPEC_OF: list = []
_SPEC_ID = _SpecIds()


def _algorithms(sh, node, mesh, in_shapes):
    """enumerate_algorithms (sharding.py:222-252) memoised: its result depends on
    the operator's kind, shapes, arity and reduce axis and on the view's extents
    only; ParallelAlgorithm carries the node id, so hits are re-labelled."""
    key = (node.kind, node.out_shape, in_shapes, len(node.inputs),
           getattr(node, "reduce_axis", None), mesh.n_l, mesh.m_l)
    hit = _ALGS.get((key, node.id))
    if hit is not None:
        return hit
    base = _ALGS.get(key)
    if base is None:
        base = _ALGS[key] = sh.enumerate_algorithms(node, mesh, in_shapes)
    hit = base if not base or base[0].node_id == node.id else \
        [dataclasses.replace(a, node_id=node.id) for a in base]
    _ALGS[(key, node.id)] = hit
    return hit


def _propagated(intra, merged, root, spec):
    """propagate_specs (intra.py:128-139) memoised on the stage's merged graph:
    the member specs depend only on the root and its output spec."""
    memo = merged.__dict__.setdefault("_mp_propagated", {})
    key = (root, _SPEC_ID.setdefault(spec, len(_SPEC_ID)))
    out = memo.get(key)
    if out is None:
        out = memo[key] = intra.propagate_specs(merged, root, spec)
    return out


def _lcm_den(values, den=1):
    for x in values:
        d = x.denominator
        den = den * d // math.gcd(den, d)
    return den


def build_ilp(merged, mesh, cost_model, _intra=None):
    intra = _intra or sys.modules["meshplan.intra"]
    sh = sys.modules["meshplan.sharding"]
    g = merged.sub.graph
    index = {r: i for i, r in enumerate(merged.roots)}
    vf = cost_model.volume_factors
    mkey = (mesh.n_l, mesh.m_l, tuple(mesh.axis_bandwidth), cost_model.cluster.alpha_latency,
            tuple(sorted(vf.items())) if vf else None)
    algorithms, specs_cache, c = [], [], []
    for r in merged.roots:
        node = g.node(r)
        in_shapes = tuple(g.node(pid).out_shape for pid, _ in node.inputs)
        algs = _algorithms(sh, node, mesh, in_shapes)
        if not algs:
            raise intra.PlannerError(f"no feasible strategy for node {r} "
                                     f"({node.kind.value}) on mesh {mesh.n_l}x{mesh.m_l}")
        algorithms.append(algs)
        specs_cache.append([_propagated(intra, merged, r, a.output_spec) for a in algs])
        row = []
        for a in algs:
            ck = (a.comm, mkey)
            t = _COLL.get(ck)
            if t is None:
                t = _COLL[ck] = cost_model.collectives_time(a.comm, mesh)
            row.append(t)
        c.append(row)
    # every resharding cost the edges need, once per distinct (src, dst, tensor):
    # specs are interned to ints once per occurrence (hashing a ShardingSpec is
    # the expensive part), cost keys are int tuples
    mid = _MESH_ID.setdefault(mkey, len(_MESH_ID))
    edge_plans = []
    needed = {}
    for (ur, vr), provenance in sorted(merged.edges.items()):
        u, v = index[ur], index[vr]
        terms = []
        for producer, consumer, slot in provenance:
            shape = g.node(producer).out_shape
            tkey = (shape.dims, shape.elem_bytes, mid)
            srcs, dsts = {}, {}
            si = [srcs.setdefault(_SPEC_ID.setdefault(specs_cache[u][i][producer], len(_SPEC_ID)),
                                  len(srcs))
                  for i in range(len(algorithms[u]))]
            di = [dsts.setdefault(_SPEC_ID.setdefault(
                      intra._required_spec(merged, algorithms[v][j], specs_cache[v][j], consumer,
                                           slot), len(_SPEC_ID)), len(dsts))
                  for j in range(len(algorithms[v]))]
            keys = [[(x, y) + tkey for y in dsts] for x in srcs]
            for row in keys:
                for k in row:
                    if k not in needed:
                        t = _RESH.get(k)
                        if t is None:
                            spec = _SPEC_OF
                            t = _RESH[k] = cost_model.collectives_time(
                                sh.resharding_cost(spec[k[0]], spec[k[1]], shape, mesh), mesh)
                        needed[k] = t
            terms.append((si, di, keys))
        edge_plans.append((u, v, terms))
    # one exact common unit for every cost, then integer matrices
    den = _lcm_den({x for row in c for x in row})
    den = _lcm_den(set(needed.values()), den)
    scaled = {k: t.numerator * (den // t.denominator) for k, t in needed.items()}
    c_int = [x.numerator * (den // x.denominator) for row in c for x in row]
    # every cost is >= 0: the objective is at most the sum of the per-node and
    # per-term maxima, which must fit the native solver's int64 range
    bound = 0
    o = 0
    for row in c:
        bound += max(c_int[o:o + len(row)])
        o += len(row)
    for _, _, terms in edge_plans:
        for _, _, keys in terms:
            bound += max(scaled[k] for row in keys for k in row)
    d = [[intra.ZERO] * len(a) for a in algorithms]
    if bound >= _LIMIT:
        # the scaled values would overflow the native solver: exact Fractions
        edges = []
        for u, v, terms in edge_plans:
            m = [[sum((Fraction(scaled[keys[si[i]][di[j]]], den) for si, di, keys in terms),
                      Fraction(0)) for j in range(len(algorithms[v]))]
                 for i in range(len(algorithms[u]))]
            edges.append((u, v, m))
        return intra.StrategyTable(merged, mesh, algorithms, c, d, edges)
    edges = []
    for u, v, terms in edge_plans:
        m = None
        for si, di, keys in terms:
            t = np.array([[scaled[k] for k in row] for row in keys], dtype=np.int64)
            g_ = t[np.asarray(si)[:, None], np.asarray(di)[None, :]]
            m = g_ if m is None else m + g_
        edges.append((u, v, np.ascontiguousarray(m)))
    st = intra.StrategyTable(merged, mesh, algorithms, c, d,
                             [(u, v, ScaledMatrix(m, den)) for u, v, m in edges])
    st._mp_scaled = {"den": den, "costs": np.asarray(c_int, dtype=np.int64),
                     "mats": (np.concatenate([m.ravel() for _, _, m in edges])
                              if edges else np.zeros(1, dtype=np.int64))}
    return st


def patch_reference(meshplan_module) -> None:
    """Route the loaded reference planner's stage ILPs through the native
    strategy table and solver."""
    intra = meshplan_module.intra
    original = intra.solve_ilp
    if getattr(original, "_mpexec_native", False):
        return

    def wrapped(table, budget=intra.DEFAULT_SOLVER_BUDGET):
        return solve_ilp(table, budget, _fallback=original)
    wrapped._mpexec_native = True
    intra.solve_ilp = wrapped

    def table(merged, mesh, cost_model):
        return build_ilp(merged, mesh, cost_model, intra)
    table._mpexec_native = True
    intra.build_ilp = table
