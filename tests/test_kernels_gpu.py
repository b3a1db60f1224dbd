"""Numerics of every libmpexec kernel against a plain PyTorch fp32 reference of
the same op (on the GPU box).  Tolerances are stated per test: bf16 outputs are
compared with rtol/atol ~1e-2 scaled to the value range; fp32 outputs of the
tcgen05 GEMM with 2e-3 relative Frobenius error (bf16 inputs, fp32 accumulate)."""
import math

import pytest
import torch

from paper_2201_12023_b200 import native

pytestmark = pytest.mark.gpu


def rel_err(x, ref):
    x = x.float()
    ref = ref.float()
    return ((x - ref).norm() / ref.norm().clamp_min(1e-30)).item()


def rnd(*shape, scale=1.0, dtype=torch.bfloat16):
    return (torch.randn(*shape, device="cuda") * scale).to(dtype)


@pytest.fixture(autouse=True)
def _seed():
    torch.manual_seed(0)


GEMM_SHAPES = [(128, 256, 64), (256, 512, 128), (384, 256, 1024), (64, 1024, 1024),
               (1000, 520, 136), (512, 64, 512), (256, 128, 192), (2048, 2048, 2048),
               (8192, 2048, 128), (6144, 4096, 64)]   # last two: tail-wave split


@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_gemm_layouts(M, N, K, ta, tb):
    a = rnd(K, M).t() if ta else rnd(M, K)
    b = rnd(N, K).t() if tb else rnd(K, N)
    out = torch.empty(M, N, device="cuda", dtype=torch.float32)
    native.gemm(a, b, out)
    ref = a.float() @ b.float()
    assert rel_err(out, ref) < 2e-3


@pytest.mark.parametrize("M,N,K", [(256, 256, 256), (128, 512, 2048)])
def test_gemm_bf16_out_alpha_beta(M, N, K):
    a, b = rnd(M, K), rnd(K, N)
    c0 = rnd(M, N)
    out = c0.clone()
    native.gemm(a, b, out, alpha=0.5, beta=1.0)
    ref = 0.5 * (a.float() @ b.float()) + c0.float()
    assert rel_err(out, ref) < 1e-2
    acc = torch.randn(M, N, device="cuda")
    acc0 = acc.clone()
    native.gemm(a, b, acc, beta=1.0)
    assert rel_err(acc, a.float() @ b.float() + acc0) < 2e-3


def test_gemm_gelu_epilogue():
    a, b = rnd(256, 512), rnd(512, 768, scale=0.05)
    out = torch.empty(256, 768, device="cuda", dtype=torch.bfloat16)
    native.gemm(a, b, out, gelu=True)
    ref = torch.nn.functional.gelu(a.float() @ b.float(), approximate="tanh")
    assert rel_err(out, ref) < 1e-2


def test_gemm_batched_head_views():
    # head split / merge as strided views: q (T, h) -> (B, H, s, hd)
    B, s, H, hd = 2, 256, 4, 64
    T, h = B * s, H * hd
    q, k, v = rnd(T, h), rnd(T, h), rnd(T, h)
    qh = q.view(B, s, H, hd).permute(0, 2, 1, 3)          # (B,H,s,hd)
    kt = k.view(B, s, H, hd).permute(0, 2, 3, 1)          # (B,H,hd,s)  K-major B
    vh = v.view(B, s, H, hd).permute(0, 2, 1, 3)          # (B,H,s,hd)  MN-major B
    scores = torch.empty(B, H, s, s, device="cuda", dtype=torch.bfloat16)
    native.gemm(qh, kt, scores)
    ref = qh.float() @ kt.float()
    assert rel_err(scores, ref) < 1e-2
    ctx = torch.empty(T, h, device="cuda", dtype=torch.bfloat16)
    ctx_v = ctx.view(B, s, H, hd).permute(0, 2, 1, 3)     # write straight into merged layout
    native.gemm(scores, vh, ctx_v)
    ref2 = scores.float() @ vh.float()
    assert rel_err(ctx_v, ref2) < 1e-2
    # transposed batched operand (dK = Q^T-style)
    out = torch.empty(B, H, hd, s, device="cuda", dtype=torch.float32)
    native.gemm(qh.transpose(-1, -2), scores, out)
    assert rel_err(out, qh.float().transpose(-1, -2) @ scores.float()) < 2e-3


def test_gemm_misaligned_operands_are_repacked():
    """Odd inner extents (the Wide-ResNet stem's 147 im2col columns) go through
    zero-padded copies; a misaligned epilogue aux is still rejected."""
    a = rnd(128, 65)[:, :63]
    b = rnd(63, 128)
    out = torch.empty(128, 128, device="cuda")
    native.gemm(a, b, out)
    assert rel_err(out, a.float() @ b.float()) < 2e-3
    o2 = torch.empty(128, 147, device="cuda", dtype=torch.bfloat16)
    b2 = rnd(63, 147)
    native.gemm(a, b2, o2)
    assert rel_err(o2, a.float() @ b2.float()) < 1e-2
    aux = torch.empty(128, 135, device="cuda", dtype=torch.bfloat16)[:, :132]
    with pytest.raises(native.NativeError):
        native.gemm(rnd(128, 64), rnd(64, 132), torch.empty(128, 136, device="cuda",
                    dtype=torch.bfloat16)[:, :132], epilogue=native.EPI_ADD, aux=aux)


def test_elementwise_ops():
    x = rnd(4096 + 3, scale=2.0)
    y = native.gelu(x)
    assert rel_err(y, torch.nn.functional.gelu(x.float(), approximate="tanh")) < 1e-2
    dy = rnd(4096 + 3)
    dx = native.gelu_bwd(x, dy)
    xf = x.float().requires_grad_()
    torch.nn.functional.gelu(xf, approximate="tanh").backward(dy.float())
    assert rel_err(dx, xf.grad) < 1e-2
    z = native.add(x, dy)
    assert rel_err(z, x.float() + dy.float()) < 1e-2
    w = native.scale(x, 0.25)
    assert rel_err(w, 0.25 * x.float()) < 1e-2
    acc = torch.zeros(1, device="cuda")
    native.sumsq(x, acc)
    assert abs(acc.item() - (x.float() ** 2).sum().item()) / (x.float() ** 2).sum().item() < 1e-4


@pytest.mark.parametrize("rows,cols", [(512, 1024), (37, 200), (8, 4096)])
def test_softmax(rows, cols):
    x = rnd(rows, cols, scale=3.0)
    s = 1.0 / math.sqrt(64)
    y = native.softmax(x, s)
    ref = torch.softmax(s * x.float(), dim=-1)
    assert rel_err(y, ref) < 1e-2
    g = rnd(rows, cols)
    dx = native.softmax_bwd(y, g, s)
    xf = x.float().requires_grad_()
    torch.softmax(s * xf, dim=-1).backward(g.float())
    assert rel_err(dx, xf.grad) < 2e-2


def test_softmax_split_rows():
    rows, cols, parts = 64, 1024, 4
    s = 0.125
    x = rnd(rows, cols, scale=3.0)
    chunks = [c.contiguous() for c in x.chunk(parts, dim=1)]
    stats = [native.softmax_stats(c, s, torch.empty(3, rows, device="cuda")) for c in chunks]
    gmax = torch.stack([st[0] for st in stats]).max(0).values
    for st in stats:                      # emulate the MAX all-reduce
        st[0].copy_(gmax)
        native.softmax_rescale(st, rows)
    total = sum(st[1] for st in stats)    # emulate the SUM all-reduce
    for st in stats:
        st[1].copy_(total)
    y = torch.cat([native.softmax_apply(c, st, s) for c, st in zip(chunks, stats)], 1)
    assert rel_err(y, torch.softmax(s * x.float(), -1)) < 1e-2


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_pack_unpack_box(dtype):
    t = torch.randn(6, 40, 24, device="cuda").to(dtype)
    lo, ext = (1, 8, 8), (3, 16, 16)
    buf = native.pack_box(t, lo, ext)
    ref = t[1:4, 8:24, 8:24].reshape(-1)
    assert torch.equal(buf, ref)
    dst = torch.zeros_like(t)
    native.unpack_box(buf, dst, lo, ext)
    assert torch.equal(dst[1:4, 8:24, 8:24], t[1:4, 8:24, 8:24])
    assert dst.abs().sum() == t[1:4, 8:24, 8:24].abs().float().sum().to(dtype)
    # non-vectorisable box (odd inner extent) on a transposed view
    tv = t.transpose(0, 1)
    buf2 = native.pack_box(tv, (3, 1, 5), (7, 2, 3))
    assert torch.equal(buf2, tv[3:10, 1:3, 5:8].reshape(-1))


def test_adam_step():
    n = 10007
    master = torch.randn(n, device="cuda")
    m = torch.zeros(n, device="cuda")
    v = torch.zeros(n, device="cuda")
    g = torch.randn(n, device="cuda")
    p = torch.empty(n, device="cuda", dtype=torch.bfloat16)
    ref = master.clone().requires_grad_()
    opt = torch.optim.AdamW([ref], lr=1e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.0)
    for step in (1, 2):
        ref.grad = g.clone()
        opt.step()
        native.adam_step(master, m, v, g, p, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8,
                         weight_decay=0.0, grad_scale=1.0, step=step)
    assert rel_err(master, ref.detach()) < 1e-5
    assert rel_err(p, ref.detach()) < 1e-2


def test_launch_counter_advances():
    c0 = native.launch_count()
    native.gelu(rnd(64))
    assert native.launch_count() == c0 + 1


@pytest.mark.parametrize("M,N,K", [(256, 512, 256), (1000, 520, 136), (128, 256, 64)])
def test_gemm_fused_epilogues(M, N, K):
    a, b = rnd(M, K), rnd(K, N, scale=0.1)
    acc = a.float() @ b.float()
    aux = rnd(M, N)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    native.gemm(a, b, out, epilogue=native.EPI_ADD, aux=aux)
    assert rel_err(out, acc + aux.float()) < 1e-2
    native.gemm(a, b, out, epilogue=native.EPI_GELU_GRAD, aux=aux)
    xf = aux.float().requires_grad_()
    torch.nn.functional.gelu(xf, approximate="tanh").backward(acc)
    assert rel_err(out, xf.grad) < 1e-2
    act = torch.empty_like(out)
    native.gemm(a, b, out, epilogue=native.EPI_GELU_DUAL, aux=act)
    assert rel_err(out, acc) < 1e-2
    assert rel_err(act, torch.nn.functional.gelu(acc, approximate="tanh")) < 1e-2


@pytest.mark.parametrize("M,N,K,ta", [(1024, 1024, 8192, 1), (1024, 16, 8192, 1), (512, 512, 4096, 0)])
def test_gemm_split_k_accumulate(M, N, K, ta):
    """Few-tile fp32 += GEMMs (MoE attention / gating dW) take the split-K path:
    one batched launch into partials + an in-order sum; same result as the
    unsplit kernel to fp32 rounding, 2e-3 against torch fp32."""
    assert native._split_k(M, N, K) > 1
    a = rnd(K, M).t() if ta else rnd(M, K)
    b = rnd(K, N)
    base = torch.randn(M, N, device="cuda")
    out = base.clone()
    native.gemm(a, b, out, beta=1.0)
    native.SPLIT_K = False
    try:
        ref1 = base.clone()
        native.gemm(a, b, ref1, beta=1.0)
    finally:
        native.SPLIT_K = True
    ref = base + a.float() @ b.float()
    assert rel_err(out, ref) < 2e-3
    assert rel_err(out, ref1) < 1e-5


@pytest.mark.parametrize("batch,M,N,K,alpha", [(1, 1000, 520, 136, 1.0), (3, 384, 272, 64, 0.5),
                                               (1, 2048, 2048, 8192, 1.0), (2, 520, 1032, 256, 2.0)])
def test_gemm_f32_accumulate_reduce_epilogue(batch, M, N, K, alpha):
    """fp32 C += alpha * A B on the 2-CTA kernel leaves through TMA bulk reduce-adds
    (partial tiles clipped by the tensor map, batched C); same as torch fp32."""
    a = rnd(batch, K, M).transpose(-1, -2)      # the dW layout: X^T
    b = rnd(batch, K, N)
    c0 = torch.randn(batch, M, N, device="cuda")
    out = c0.clone()
    native.gemm(a if batch > 1 else a[0], b if batch > 1 else b[0],
                out if batch > 1 else out[0], alpha=alpha, beta=1.0)
    ref = c0 + alpha * (a.float() @ b.float())
    assert rel_err(out, ref) < 2e-3


@pytest.mark.parametrize("nb,M,N,K", [(3, 512, 768, 256), (2, 600, 520, 136)])
def test_gemm_fused_epilogues_batched(nb, M, N, K):
    """Batched 2-CTA tiles: bf16 C (and the dual epilogue's GeLU output) leave
    through TMA tensor stores from swizzled staging; the batched aux-reading
    epilogues keep direct stores.  Ragged M / N exercise the stores' clipping."""
    a, b = rnd(nb, M, K), rnd(nb, K, N, scale=0.1)
    acc = a.float() @ b.float()
    out = torch.full((nb, M, N), 7.0, device="cuda", dtype=torch.bfloat16)
    native.gemm(a, b, out)
    assert rel_err(out, acc) < 1e-2
    act = torch.full_like(out, 7.0)
    native.gemm(a, b, out, epilogue=native.EPI_GELU_DUAL, aux=act)
    assert rel_err(out, acc) < 1e-2
    assert rel_err(act, torch.nn.functional.gelu(acc, approximate="tanh")) < 1e-2
    aux = rnd(nb, M, N)
    native.gemm(a, b, out, epilogue=native.EPI_ADD, aux=aux)
    assert rel_err(out, acc + aux.float()) < 1e-2
    # an output view inside a wider buffer: stores must stay within the view
    big = torch.full((nb, M, N + 64), 5.0, device="cuda", dtype=torch.bfloat16)
    native.gemm(a, b, big[..., :N])
    assert rel_err(big[..., :N], acc) < 1e-2
    assert bool((big[..., N:] == 5.0).all())


@pytest.mark.parametrize("nb", [1, 4])
def test_gemm_gelu_epilogues_wide_range(nb):
    """Packed-pair GeLU / GeLU' epilogues over pre-activations far into both
    saturated tails (|x| up to 40, past the clamp at 16) against torch fp32."""
    M, N, K = 512, 512, 128
    a, b = rnd(nb, M, K), rnd(nb, K, N, scale=0.1)
    acc = a.float() @ b.float()
    pre = (torch.rand(nb, M, N, device="cuda") * 80 - 40).to(torch.bfloat16)
    out = torch.empty(nb, M, N, device="cuda", dtype=torch.bfloat16)
    native.gemm(a, b, out, epilogue=native.EPI_GELU_GRAD, aux=pre)
    xf = pre.float().requires_grad_()
    torch.nn.functional.gelu(xf, approximate="tanh").backward(acc)
    assert rel_err(out, xf.grad) < 1e-2
    assert torch.isfinite(out.float()).all()
    big = torch.empty_like(out)
    a2 = rnd(nb, M, K, scale=8.0)
    acc2 = a2.float() @ b.float()
    native.gemm(a2, b, out, epilogue=native.EPI_GELU_DUAL, aux=big)
    assert rel_err(big, torch.nn.functional.gelu(acc2, approximate="tanh")) < 1e-2


@pytest.mark.parametrize("nb", [1, 3])
def test_gemm_gelu_grad_epilogue_propagates_nan(nb):
    """A NaN pre-activation gives a NaN gradient in the fused GeLU' epilogue, as it
    does in the unfused gelu_bwd kernel (the |x| <= 16 clamp is NaN-propagating)."""
    M, N, K = 256, 512, 128
    a, b = rnd(nb, M, K), rnd(nb, K, N, scale=0.1)
    pre = rnd(nb, M, N)
    pre[:, 3, 7] = float("nan")
    pre[:, 100, 300] = float("inf")
    out = torch.empty(nb, M, N, device="cuda", dtype=torch.bfloat16)
    native.gemm(a, b, out, epilogue=native.EPI_GELU_GRAD, aux=pre)
    assert bool(torch.isnan(out[:, 3, 7]).all())
    fin = torch.isfinite(pre.float())
    xf = pre.float().where(fin, torch.zeros_like(pre.float())).requires_grad_()
    torch.nn.functional.gelu(xf, approximate="tanh").backward(a.float() @ b.float())
    assert rel_err(out.float()[fin], xf.grad[fin]) < 1e-2


@pytest.mark.parametrize("M,N,K", [(1024, 1024, 8192), (2048, 2048, 1024)])
def test_gemm_f32_overwrite_beta0(M, N, K):
    """The step's first dW launch overwrites the fp32 gradient buffer (beta = 0,
    no zero fill): garbage in C (NaN included) never leaks into the result, on the
    split-K path and the plain kernel."""
    a = rnd(K, M).t()
    b = rnd(K, N)
    out = torch.full((M, N), float("nan"), device="cuda")
    native.gemm(a, b, out, beta=0.0)
    assert rel_err(out, a.float() @ b.float()) < 2e-3


def test_gemm_rejects_misaligned_batch_strides():
    """16-byte C / aux accesses start at every batch base: an odd batch stride
    is an argument error (rc 2), never a device fault."""
    a, b = rnd(2, 256, 64), rnd(2, 64, 256)
    buf = torch.empty(2 * 256 * 256 + 3, device="cuda", dtype=torch.bfloat16)
    out = buf.as_strided((2, 256, 256), (256 * 256 + 3, 256, 1))
    aux = rnd(2, 256, 256)
    with pytest.raises(native.NativeError):
        native.gemm(a, b, out, epilogue=native.EPI_ADD, aux=aux)
    torch.cuda.synchronize()


def test_alltoall_two_ranks():
    """mp_alltoall (resharding_cost's all_to_all, sharding.py:346) on 2 GPUs:
    chunk i of each rank's input lands as chunk `rank` on rank i."""
    import os
    import subprocess
    import sys
    import textwrap
    from pathlib import Path
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    root = Path(__file__).resolve().parent.parent
    code = textwrap.dedent("""
        import os, torch, torch.distributed as dist
        from paper_2201_12023_b200 import native
        r = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(r)
        dist.init_process_group("nccl", device_id=torch.device("cuda", r))
        uid = [native.nccl_unique_id() if r == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = native.comm_init(uid[0], 2, r)
        x = (torch.arange(2 * 1000, device="cuda", dtype=torch.float32) + 10000 * r).to(torch.bfloat16)
        y = torch.empty_like(x)
        native.alltoall(comm, y, x, 2)
        torch.cuda.synchronize()
        want = torch.cat([(torch.arange(1000, device="cuda", dtype=torch.float32) + 1000 * r + 10000 * q)
                          .to(torch.bfloat16) for q in range(2)])
        assert torch.equal(y, want), (r, y[:4], want[:4])
        native.comm_destroy(comm)
        print("ok", r, flush=True)
        dist.destroy_process_group()
    """)
    script = root / "gpurun_out" / "_alltoall_probe.py"
    script.parent.mkdir(exist_ok=True)
    script.write_text(code)
    res = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node=2", "--master-addr", "127.0.0.1", "--master-port",
                          "29533", str(script)], capture_output=True, text=True, timeout=300,
                         env={**os.environ, "PYTHONPATH": str(root)})
    assert res.returncode == 0 and res.stdout.count("ok") == 2, res.stdout[-2000:] + res.stderr[-2000:]


@pytest.mark.parametrize("shape,lo,ext", [((8192, 1024), (4096, 512), (4096, 512)),
                                          ((8, 300, 96), (2, 7, 8), (5, 290, 80)),
                                          ((3, 4, 70, 64), (1, 0, 5, 8), (2, 4, 64, 56))])
def test_pack_unpack_box_rows(shape, lo, ext):
    """Row-form box copies (one warp per innermost row, >= 64 rows): exact on 2-, 3-
    and 4-D boxes of strided tiles, both directions."""
    t = torch.randn(*shape, device="cuda").to(torch.bfloat16)
    sl = tuple(slice(a, a + e) for a, e in zip(lo, ext))
    buf = native.pack_box(t, lo, ext)
    assert torch.equal(buf, t[sl].reshape(-1))
    dst = torch.zeros_like(t)
    native.unpack_box(buf, dst, lo, ext)
    assert torch.equal(dst[sl], t[sl])
    dst[sl] = 0
    assert not dst.any()


def test_gemm_bn512_pair_tiles():
    """256 x 512 pair tiles (MPEXEC_GEMM_BN512=1, one TMEM accumulator, two N = 256
    MMAs per k-step) on the wide GPT shapes, every B layout and the fused epilogues,
    against torch fp32 (run in a subprocess: the switch is read once per process)."""
    import os
    import subprocess
    import sys
    import textwrap
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    code = textwrap.dedent("""
        import torch
        from paper_2201_12023_b200 import native
        def rel(x, r):
            return float((x.float() - r).norm() / r.norm())
        torch.manual_seed(0)
        M, N, K = 8192, 8192, 512
        a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        for tb in (0, 1):
            b = (torch.randn(N, K, device="cuda").to(torch.bfloat16).t() if tb else
                 torch.randn(K, N, device="cuda").to(torch.bfloat16)) * 0.1
            acc = a.float() @ b.float()
            out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            native.gemm(a, b, out)
            assert rel(out, acc) < 1e-2, ("plain", tb)
            act = torch.empty_like(out)
            native.gemm(a, b, out, epilogue=native.EPI_GELU_DUAL, aux=act)
            assert rel(out, acc) < 1e-2 and rel(act, torch.nn.functional.gelu(acc, approximate="tanh")) < 1e-2
            aux = torch.randn(M, N, device="cuda").to(torch.bfloat16)
            native.gemm(a, b, out, epilogue=native.EPI_ADD, aux=aux)
            assert rel(out, acc + aux.float()) < 1e-2
            native.gemm(a, b, out, epilogue=native.EPI_GELU_GRAD, aux=aux)
            xf = aux.float().requires_grad_()
            torch.nn.functional.gelu(xf, approximate="tanh").backward(acc)
            assert rel(out, xf.grad) < 1e-2
            c = torch.randn(M, N, device="cuda")
            ref = c + acc
            native.gemm(a, b, c, beta=1.0)
            assert rel(c, ref) < 2e-3
        print("ok")
    """)
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                         cwd=root, env={**os.environ, "PYTHONPATH": str(root),
                                        "MPEXEC_GEMM_BN512": "1"})
    assert res.returncode == 0 and "ok" in res.stdout, res.stdout[-2000:] + res.stderr[-3000:]
