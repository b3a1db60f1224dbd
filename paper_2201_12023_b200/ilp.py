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

`patch_reference(meshplan)` swaps it into a loaded reference planner so
`meshplan.cli plan` / `meshplan.plan` run unchanged but fast
(scripts/plan_native.py).
"""
from __future__ import annotations

import ctypes
import math
import sys
from fractions import Fraction

from . import native

_LIMIT = 1 << 62


def _scale(values):
    den = 1
    for v in values:
        den = den * v.denominator // math.gcd(den, v.denominator)
    return den


def solve_ilp(table, budget: int = 200_000, _fallback=None):
    n = table.num_nodes
    if n == 0:
        raise ValueError("empty strategy table")
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


def patch_reference(meshplan_module) -> None:
    """Route the loaded reference planner's stage ILPs through the native solver."""
    intra = meshplan_module.intra
    original = intra.solve_ilp
    if getattr(original, "_mpexec_native", False):
        return

    def wrapped(table, budget=intra.DEFAULT_SOLVER_BUDGET):
        return solve_ilp(table, budget, _fallback=original)
    wrapped._mpexec_native = True
    intra.solve_ilp = wrapped
