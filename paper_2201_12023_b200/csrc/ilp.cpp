// Native branch-and-bound for the intra-op strategy ILP.
//
// Restates reference intra.py:323-401 (`solve_ilp`, `_greedy_assignment`) with
// identical semantics on exact integer costs (the Python wrapper scales every
// Fraction by the lcm of their denominators, so comparisons are exact):
//   * edges are charged when their later endpoint is assigned (matrix oriented
//     [earlier choice][later choice]);
//   * suffix lower bound = per-node minima + matrix minima of untouched edges;
//   * the incumbent starts from the greedy assignment (first strict minimum);
//   * DFS explores strategies in index order, prunes when acc + step +
//     suffix >= best (strict improvement only, so ties keep the lowest indices);
//   * `explored` counts dfs entries; at `budget` the search stops and the plan
//     is reported non-certified.
// Planning GPT-1.3B spends essentially all its time in this loop with Python
// Fractions; this is the same search on int128 arithmetic.
#include <stdint.h>
#include <string.h>
#include <algorithm>
#include <vector>

namespace {

typedef __int128 i128;

struct InEdge {
  int lo;
  const int64_t* m;   // [k_lo][k_hi] row-major, oriented (lo choice, hi choice)
  int k_hi;
};

struct Solver {
  int n;
  const int* k;
  std::vector<const int64_t*> c;     // node costs (c + d, scaled)
  std::vector<std::vector<InEdge>> in_edges;
  std::vector<i128> suffix;
  std::vector<int> choice, best_choice;
  i128 best_cost;
  int64_t explored = 0, budget;
  bool certified = true;

  i128 step_cost(int t, int j) const {
    i128 s = c[t][j];
    for (const InEdge& e : in_edges[t]) s += e.m[(int64_t)choice[e.lo] * e.k_hi + j];
    return s;
  }

  void dfs(int t, i128 acc) {
    if (explored >= budget) {
      certified = false;
      return;
    }
    ++explored;
    if (t == n) {
      if (acc < best_cost) {
        best_cost = acc;
        best_choice = choice;
      }
      return;
    }
    const int kt = k[t];
    // options are computed against the current prefix before iterating
    std::vector<i128> steps(kt);
    for (int j = 0; j < kt; ++j) steps[j] = step_cost(t, j);
    for (int j = 0; j < kt; ++j) {
      const i128 lb = acc + steps[j] + suffix[t + 1];
      if (lb >= best_cost) continue;
      choice[t] = j;
      dfs(t + 1, acc + steps[j]);
      if (explored >= budget) return;
    }
  }
};

}  // namespace

extern "C" {

// n nodes with k[t] strategies; node costs concatenated in `costs` (sum k);
// `n_edges` edges (u[e], v[e]) with matrices concatenated in `mats`
// (k[u] x k[v] row-major, original orientation).  All values are integers in a
// common unit.  Outputs: choice[n], *objective (int64, saturating), certified,
// explored.  Returns 0, or 2 on bad input.
int mp_ilp_solve(int n, const int* k, const int64_t* costs, int n_edges, const int* u,
                 const int* v, const int64_t* mats, int64_t budget, int* choice_out,
                 int64_t* objective_out, int* certified_out, int64_t* explored_out) {
  if (n <= 0 || !k || !costs || !choice_out || !objective_out) return 2;
  Solver s;
  s.n = n;
  s.k = k;
  s.budget = budget;
  s.c.resize(n);
  int64_t off = 0;
  for (int t = 0; t < n; ++t) {
    if (k[t] <= 0) return 2;
    s.c[t] = costs + off;
    off += k[t];
  }
  // transposed copies for edges whose later endpoint is u
  std::vector<std::vector<int64_t>> transposed;
  transposed.reserve(n_edges);
  s.in_edges.assign(n, {});
  const int64_t* m = mats;
  for (int e = 0; e < n_edges; ++e) {
    const int a = u[e], b = v[e];
    if (a < 0 || a >= n || b < 0 || b >= n) return 2;
    const int ka = k[a], kb = k[b];
    if (a < b) {
      s.in_edges[b].push_back(InEdge{a, m, kb});
    } else {
      transposed.emplace_back((size_t)ka * kb);
      std::vector<int64_t>& tr = transposed.back();
      for (int i = 0; i < ka; ++i)
        for (int j = 0; j < kb; ++j) tr[(size_t)j * ka + i] = m[(size_t)i * kb + j];
      s.in_edges[a].push_back(InEdge{b, tr.data(), ka});
    }
    m += (int64_t)ka * kb;
  }
  // suffix bounds
  s.suffix.assign(n + 1, 0);
  for (int t = n - 1; t >= 0; --t) {
    i128 mn = s.c[t][0];
    for (int j = 1; j < k[t]; ++j)
      if (s.c[t][j] < mn) mn = s.c[t][j];
    i128 acc = s.suffix[t + 1] + mn;
    for (const InEdge& ie : s.in_edges[t]) {
      const int rows = k[ie.lo];
      i128 mm = ie.m[0];
      for (int64_t q = 1; q < (int64_t)rows * ie.k_hi; ++q)
        if (ie.m[q] < mm) mm = ie.m[q];
      acc += mm;
    }
    s.suffix[t] = acc;
  }
  // greedy incumbent (first strict minimum per node, prefix-conditioned)
  s.choice.assign(n, 0);
  for (int t = 0; t < n; ++t) {
    int bj = 0;
    i128 bv = 0;
    for (int j = 0; j < k[t]; ++j) {
      const i128 val = s.step_cost(t, j);
      if (j == 0 || val < bv) {
        bv = val;
        bj = j;
      }
    }
    s.choice[t] = bj;
  }
  // incumbent cost = table.evaluate(greedy): node costs + every edge
  // (step_cost sums each node cost plus its in-edges against the greedy prefix,
  // so every edge is counted once, at its later endpoint)
  i128 g = 0;
  for (int t = 0; t < n; ++t) g += s.step_cost(t, s.choice[t]);
  s.best_cost = g;
  s.best_choice = s.choice;
  std::fill(s.choice.begin(), s.choice.end(), 0);
  s.dfs(0, 0);
  for (int t = 0; t < n; ++t) choice_out[t] = s.best_choice[t];
  const i128 lim = (i128)INT64_MAX;
  *objective_out = (int64_t)(s.best_cost > lim ? lim : s.best_cost);
  if (certified_out) *certified_out = s.certified ? 1 : 0;
  if (explored_out) *explored_out = s.explored;
  return 0;
}

}  // extern "C"
