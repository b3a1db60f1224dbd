"""Wide-ResNet (BASELINE configs[3]): builder, conv adapters,
oracle and executor.

CPU: sharded oracle == dense oracle on the planner's WRN plans (incl. the
heterogeneous (1,2)+(1,2)+(1,4) plan for 8 GPUs, shrunk); product and oracle
bindings agree; col2im is the adjoint of im2col; the dense backward is the
true gradient (finite differences).
GPU: im2col / subsample / reduction kernels against the oracle restatement;
the executor matches the oracle on WRN plans.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from parity_harness import ROOT, run_plan, synth

WRN_PLANS = ["wresnet_tiny_n1", "wresnet_tiny_n2", "wresnet_tiny_n4", "wresnet_tiny_tp_n4",
             "wresnet_tiny_het_n8"]


def doc_of(name):
    return json.loads((ROOT / "plans" / name / "plan.json").read_text())


@pytest.mark.parametrize("name", WRN_PLANS)
def test_sharded_oracle_equals_dense_wrn(name):
    from oracle import dense, sharded
    doc = doc_of(name)
    params, inputs = synth(doc, seed=3)
    B = doc["num_microbatches"]
    L, G, O = dense.run(doc, params, inputs, B)
    L2, G2, O2 = sharded.run(doc, params, inputs, B)
    assert abs(L - L2) <= 1e-9 * abs(L)
    for k in G:
        assert np.allclose(G[k], G2[k], rtol=1e-9, atol=1e-9 * np.abs(G[k]).max())


@pytest.mark.parametrize("name", WRN_PLANS + ["wresnet1b_n1", "wresnet1b_n8"])
def test_product_binding_equals_oracle_binding_wrn(name):
    from oracle import ir
    from paper_2201_12023_b200.binding import bind
    from paper_2201_12023_b200.plan import load_plan
    doc = doc_of(name)
    mine = bind(load_plan(doc).graph)
    ref = ir.bind(doc["graph"]["nodes"])
    names = {"input": "input", "parameter": "param", "matmul": "matmul", "batched_matmul": "bmm"}
    for nid, (code, info) in ref.items():
        assert mine[nid].op == names.get(code, code), (nid, mine[nid], code)
        if code in ("im2col", "col2im", "subsample", "subsample_grad"):
            assert mine[nid].conv == tuple(info)


def test_wrn_binding_census():
    from paper_2201_12023_b200.binding import bind
    from paper_2201_12023_b200.plan import load_plan
    g = load_plan(doc_of("wresnet1b_n1")).graph
    ops = [b.op for b in bind(g).values()]
    assert ops.count("im2col") == 17 and ops.count("col2im") == 17      # stem + 16 blocks
    assert ops.count("subsample") == 4 and ops.count("reduce_sum") == 1
    params = sum(int(np.prod(n.dims)) for n in g.nodes if n.kind == "parameter")
    assert params == 1_679_448_000


@pytest.mark.parametrize("k,s,C", [(3, 1, 5), (3, 2, 8), (7, 2, 3)])
def test_col2im_is_adjoint_of_im2col(k, s, C):
    from oracle.dense import conv_op
    N, H = 2, 8
    rng = np.random.default_rng(0)
    x = rng.standard_normal((N * H * H, C))
    info = (N, H, H, C, k, s)
    cols = conv_op("im2col", info, x)
    y = rng.standard_normal(cols.shape)
    assert abs((cols * y).sum() - (x * conv_op("col2im", info, y)).sum()) < 1e-9
    sub = conv_op("subsample", (N, H, H, C, 1, s), x)
    z = rng.standard_normal(sub.shape)
    back = conv_op("subsample_grad", (N, H, H, C, 1, s), z)
    assert abs((sub * z).sum() - (x * back).sum()) < 1e-9


def test_wrn_dense_backward_matches_finite_difference():
    from oracle import dense
    doc = doc_of("wresnet_tiny_n1")
    params, inputs = synth(doc, seed=5)
    params = {k: v.astype(np.float64) for k, v in params.items()}
    L, G, _ = dense.run(doc, params, inputs, 1)
    rng = np.random.default_rng(0)
    for pid in [min(G)] + list(G)[-3:]:
        idx = tuple(rng.integers(0, s) for s in params[pid].shape)
        eps = 1e-4 * max(1e-3, abs(params[pid][idx]))
        p2 = dict(params)
        p2[pid] = params[pid].copy()
        p2[pid][idx] += eps
        L2, _, _ = dense.run(doc, p2, inputs, 1)
        p2[pid][idx] -= 2 * eps
        L3, _, _ = dense.run(doc, p2, inputs, 1)
        fd = (L2 - L3) / (2 * eps)
        assert abs(fd - G[pid][idx]) <= 1e-4 * max(abs(fd), 1e-3 * np.abs(G[pid]).max()), \
            (pid, fd, G[pid][idx])


# ----------------------------------------------------------------- GPU

@pytest.mark.gpu
@pytest.mark.parametrize("k,s,C", [(3, 1, 16), (3, 2, 8), (7, 2, 3), (1, 2, 24)])
def test_conv_adapter_kernels(k, s, C):
    import torch
    from oracle.dense import conv_op
    from paper_2201_12023_b200 import native
    N, H = 3, 14
    x = torch.randn(N * H * H, C, device="cuda").to(torch.bfloat16)
    x64 = x.float().cpu().numpy().astype(np.float64)
    info = (N, H, H, C, k, s)
    if k == 1:
        y = native.subsample(x, N, H, H, C, s)
        assert np.array_equal(y.float().cpu().numpy(), conv_op("subsample", info, x64))
        g = torch.randn_like(y)
        dx = native.subsample(g, N, H, H, C, s, backward=True)
        ref = conv_op("subsample_grad", info, g.float().cpu().numpy().astype(np.float64))
        assert np.array_equal(dx.float().cpu().numpy(), ref)
        return
    cols = native.im2col(x, N, H, H, C, k, s)
    assert np.array_equal(cols.float().cpu().numpy(), conv_op("im2col", info, x64))
    d = torch.randn_like(cols)
    dx = native.col2im(d, N, H, H, C, k, s).float().cpu().numpy()
    ref = conv_op("col2im", info, d.float().cpu().numpy().astype(np.float64))
    assert np.abs(dx - ref).max() <= 1e-2 * np.abs(ref).max()       # bf16 output rounding


@pytest.mark.gpu
def test_reduce_mid_and_broadcast():
    import torch
    from paper_2201_12023_b200 import native
    x = torch.randn(4, 49, 40, device="cuda").to(torch.bfloat16)
    r = native.reduce_mid(x).float()
    ref = x.float().sum(1)
    assert (r - ref).abs().max() <= 1e-2 * ref.abs().max()
    b = native.reduce_mid(r.to(torch.bfloat16), broadcast_b=49)
    assert torch.equal(b, r.to(torch.bfloat16)[:, None, :].expand(4, 49, 40))


@pytest.mark.gpu
@pytest.mark.parametrize("schedule", ["1f1b", "gpipe"])
def test_wrn_single_device_parity(schedule):
    errs = run_plan(ROOT / "plans/wresnet_tiny_n1/plan.json", schedule)
    print(json.dumps(errs, default=str))
    assert errs["ok"], errs
    assert errs["gpu_launches"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("plan,n", [("plans/wresnet_tiny_n2/plan.json", 2),
                                    ("plans/wresnet_tiny_n4/plan.json", 4),
                                    ("plans/wresnet_tiny_tp_n4/plan.json", 4),
                                    ("plans/wresnet_tiny_het_n8/plan.json", 8)])
def test_wrn_multi_device_parity(plan, n):
    import torch
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29540 + n),
           str(ROOT / "scripts/parity_run.py"), str(ROOT / plan)]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900,
                         env={**os.environ, "PYTHONPATH": str(ROOT)})
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert res.returncode == 0 and lines, res.stdout[-3000:] + res.stderr[-3000:]
    errs = json.loads(lines[-1])
    assert errs["ok"], errs
