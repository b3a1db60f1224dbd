"""GShard MoE: builder, binding, routing, oracle and executor.

CPU: the oracle's sharded run equals its dense run on the MoE plans; the dense
backward is the true gradient (finite differences, routing held fixed); the
product and oracle bindings agree; routing follows the stated rule on
hand-built cases (capacity overflow, top-2 fill behind top-1, ties).
GPU: the routing kernel and mask kernels are bit-exact against the oracle on
the same bf16 gates; the executor matches the oracle on MoE plans.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from parity_harness import ROOT, TOL, run_plan, synth

MOE_PLANS = ["moe_tiny_n1", "moe_tiny_n2", "moe_tiny_n4", "moe_tiny_tp_n4"]


def doc_of(name):
    return json.loads((ROOT / "plans" / name / "plan.json").read_text())


# ----------------------------------------------------------------- CPU

@pytest.mark.parametrize("name", MOE_PLANS)
def test_sharded_oracle_equals_dense_moe(name):
    from oracle import dense, sharded
    doc = doc_of(name)
    params, inputs = synth(doc, seed=3)
    B = doc["num_microbatches"]
    L, G, O = dense.run(doc, params, inputs, B)
    L2, G2, O2 = sharded.run(doc, params, inputs, B)
    assert abs(L - L2) <= 1e-9 * abs(L)
    for k in G:
        assert np.allclose(G[k], G2[k], rtol=1e-9, atol=1e-9 * np.abs(G[k]).max())


@pytest.mark.parametrize("name", MOE_PLANS + ["moe24b_n1", "moe24b_n4_ep"])
def test_product_binding_equals_oracle_binding_moe(name):
    from oracle import ir
    from paper_2201_12023_b200.binding import bind
    from paper_2201_12023_b200.plan import load_plan
    doc = doc_of(name)
    mine = bind(load_plan(doc).graph)
    ref = ir.bind(doc["graph"]["nodes"])
    names = {"input": "input", "parameter": "param", "matmul": "matmul", "batched_matmul": "bmm"}
    for nid, (code, info) in ref.items():
        assert mine[nid].op == names.get(code, code), (nid, mine[nid], code)
        if code in ("dispatch", "combine"):
            assert mine[nid].route == tuple(info)
        if code == "regroup":
            assert mine[nid].regroup == tuple(info)


def test_moe_binding_census():
    from paper_2201_12023_b200.binding import bind
    from paper_2201_12023_b200.plan import load_plan
    g = load_plan(doc_of("moe24b_n1")).graph
    ops = [b.op for b in bind(g).values()]
    # 16 layers, MoE every 2nd: 8 MoE layers, 16 attention softmaxes + 8 gate softmaxes
    assert ops.count("dispatch") == 8 and ops.count("combine") == 8
    assert ops.count("dispatch_grad") == 8 and ops.count("combine_grad") == 8
    assert ops.count("regroup") == 4 * 8            # 2 fwd + their 2 inverses per layer
    assert ops.count("softmax") == 16 + 8 and ops.count("gelu") == 16
    params = sum(int(np.prod(n.dims)) for n in g.nodes if n.kind == "parameter")
    assert params == 2_348_941_312                  # "2.4B" (ffn 8h)


def test_routing_rule_hand_cases():
    from oracle.dense import route
    # one group of 6 tokens, 3 experts, capacity 2
    g = np.array([[.7, .2, .1],     # e1=0 e2=1
                  [.6, .3, .1],     # e1=0 e2=1
                  [.5, .1, .4],     # e1=0 (dropped: 3rd top-1 of expert 0), e2=2
                  [.1, .8, .1],     # e1=1, e2=0 (tie 0/2 -> lowest index 0)
                  [.2, .2, .6],     # e1=2, e2=0 (tie -> 0)
                  [.3, .3, .4]])    # e1=2, e2=0
    pairs = sorted(route(g, 1, 6, 3, 2))
    # top-1: e0 <- t0@0, t1@1 (t2 dropped); e1 <- t3@0; e2 <- t4@0, t5@1
    # top-2 behind kept top-1 (fill e0=2, e1=1, e2=2): t0->e1@1, t1->e1@2 drop,
    # t2->e2@2 drop, t3->e0@2 drop, t4->e0@3 drop, t5->e0@4 drop
    assert pairs == [(0, 0, 0), (0, 1, 1), (1, 0, 1), (3, 1, 0), (4, 2, 0), (5, 2, 1)]


def test_moe_dense_backward_matches_finite_difference():
    """With the routing held fixed, the bound backward (combine gradient into
    the gates, zero through the 0/1 dispatch mask) is the true gradient."""
    from oracle import dense, ir
    doc = doc_of("moe_tiny_n1")
    params, inputs = synth(doc, seed=5)
    params = {k: v.astype(np.float64) for k, v in params.items()}
    nodes = doc["graph"]["nodes"]
    gid = [info[1] for code, info in ir.bind(nodes).values() if code == "combine_grad"][0]
    trace = {gid: []}
    L, G, _ = dense.run(doc, params, inputs, 1, trace=trace)
    routes = {}
    G_, S, E, C = [info for code, info in ir.bind(nodes).values() if code == "dispatch"][0]
    table = np.full((G_ * S, 4), -1, np.int64)
    for t, e, c in dense.route(trace[gid][0], G_, S, E, C):
        k = 0 if table[t, 0] < 0 else 1
        table[t, 2 * k], table[t, 2 * k + 1] = e, c
    routes[(0, gid)] = table
    wg = nodes[nodes[gid]["inputs"][0][0]]["inputs"][1][0]       # gating weight
    rng = np.random.default_rng(0)
    for pid in [wg] + list(G)[:5]:
        idx = tuple(rng.integers(0, s) for s in params[pid].shape)
        eps = 1e-6
        p2 = dict(params)
        p2[pid] = params[pid].copy()
        p2[pid][idx] += eps
        L2, _, _ = dense.run(doc, p2, inputs, 1, routes=routes)
        p2[pid][idx] -= 2 * eps
        L3, _, _ = dense.run(doc, p2, inputs, 1, routes=routes)
        fd = (L2 - L3) / (2 * eps)
        assert abs(fd - G[pid][idx]) <= 1e-4 * max(1.0, abs(fd)), (pid, fd, G[pid][idx])


@pytest.mark.reference
def test_builders_emit_reference_graphs(meshplan_ref):
    """The builders' graphs parse with the reference (graph.parse, validate_graph)
    and the committed MoE plans were planned from exactly these graphs."""
    from meshplan import graph as G
    from paper_2201_12023_b200 import builders
    g = builders.build_moe(16, 8, 1024, 1024, 16, 16, elem_bytes=2, backward=True)
    data = G.serialize(g)
    assert G.serialize(G.parse(data)) == data
    plan_graph = doc_of("moe24b_n1")["graph"]
    assert json.loads(data) == plan_graph
    w = builders.build_wide_resnet(8, backward=True)
    assert G.parse(G.serialize(w)).total_flop() == w.total_flop()


# ----------------------------------------------------------------- GPU

def _gates(T, E, seed, levels=None):
    import torch
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((T, E))
    if levels:                                   # coarse values: many exact ties
        x = np.round(x * levels) / levels
    g = np.exp(x) / np.exp(x).sum(1, keepdims=True)
    t = torch.tensor(g, dtype=torch.bfloat16, device="cuda")
    return t, t.float().cpu().numpy().astype(np.float64)


@pytest.mark.gpu
@pytest.mark.parametrize("T,S,E,C,levels", [(4096, 1024, 16, 128, None), (2048, 1024, 16, 16, 2),
                                            (3000, 1500, 8, 300, None), (96, 32, 4, 3, 1)])
def test_route_and_mask_kernels_exact(T, S, E, C, levels):
    import torch
    from oracle import dense
    from paper_2201_12023_b200 import native
    gates, g64 = _gates(T, E, seed=T + E, levels=levels)
    route = native.moe_route(gates, S, C)
    got = sorted(dense.pairs_of(route.cpu().numpy()))
    want = sorted(dense.route(g64, T // S, S, E, C))
    assert got == want
    for mode, code in ((0, "dispatch"), (1, "combine")):
        m = native.moe_mask(route, gates, S, C, mode).float().cpu().numpy()
        ref = dense.routing_op(code, (T // S, S, E, C), g64)
        assert np.array_equal(m, ref)
    d = torch.randn(T // S, S, E * C, device="cuda").to(torch.bfloat16)
    gg = native.moe_mask_grad(route, d, E, S, C, 1).float().cpu().numpy()
    ref = dense.routing_op("combine_grad", ((T // S, S, E, C), None), d.float().cpu().numpy(),
                           gates=g64)
    assert np.array_equal(gg, ref)
    z = native.moe_mask_grad(route, torch.ones(T // S, E * C, S, device="cuda",
                                               dtype=torch.bfloat16), E, S, C, 0)
    assert int(torch.count_nonzero(z)) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("schedule", ["1f1b", "gpipe"])
def test_moe_single_device_parity(schedule):
    errs = run_plan(ROOT / "plans/moe_tiny_n1/plan.json", schedule)
    print(json.dumps(errs, default=str))
    assert errs["ok"], errs
    assert errs["gpu_launches"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("plan,n", [("plans/moe_tiny_n2/plan.json", 2),
                                    ("plans/moe_tiny_n4/plan.json", 4),
                                    ("plans/moe_tiny_tp_n4/plan.json", 4)])
def test_moe_multi_device_parity(plan, n):
    import torch
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + n),
           str(ROOT / "scripts/parity_run.py"), str(ROOT / plan)]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900,
                         env={**os.environ, "PYTHONPATH": str(ROOT)})
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert res.returncode == 0 and lines, res.stdout[-3000:] + res.stderr[-3000:]
    errs = json.loads(lines[-1])
    assert errs["ok"], errs
