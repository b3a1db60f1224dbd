"""Throughput of the tcgen05 GEMM at the GPT-1.3B per-device shapes,
next to torch.matmul (cuBLAS) for context.  CUDA-event timing, warm-up, inputs
reused (these GEMMs are compute-bound; L2 residency does not change the bound)."""
import json
import os
import sys

import torch

from paper_2201_12023_b200 import native

SHAPES = [
    # name, M, N, K, ta, tb
    ("qkv_fwd", 8192, 2048, 2048, 0, 0),
    ("mlp_up_fwd", 8192, 8192, 2048, 0, 0),
    ("mlp_down_fwd", 8192, 2048, 8192, 0, 0),
    ("mlp_up_dX", 8192, 2048, 8192, 0, 1),
    ("mlp_up_dW", 2048, 8192, 8192, 1, 0),
    ("sq4096", 4096, 4096, 4096, 0, 0),
    ("sq8192", 8192, 8192, 8192, 0, 0),
]


def timeit(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3


def main():
    rows = []
    for name, M, N, K, ta, tb in SHAPES:
        a = torch.randn(K, M, device="cuda", dtype=torch.bfloat16).t() if ta else \
            torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16).t() if tb else \
            torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        t_mp = timeit(lambda: native.gemm(a, b, out))
        t_cb = timeit(lambda: torch.matmul(a, b, out=out))
        fl = 2.0 * M * N * K
        rows.append({"shape": name, "M": M, "N": N, "K": K, "ta": ta, "tb": tb,
                     "mp_tflops": fl / t_mp / 1e12, "cublas_tflops": fl / t_cb / 1e12,
                     "mp_us": t_mp * 1e6})
        print(json.dumps(rows[-1]), flush=True)
    # batched attention shapes (one 8-seq microbatch, 32 heads)
    B, H, s, hd = 8, 32, 1024, 64
    q = torch.randn(B * s, H * hd, device="cuda", dtype=torch.bfloat16)
    qh = q.view(B, s, H, hd).permute(0, 2, 1, 3)
    kt = q.view(B, s, H, hd).permute(0, 2, 3, 1)
    sc = torch.empty(B, H, s, s, device="cuda", dtype=torch.bfloat16)
    t = timeit(lambda: native.gemm(qh, kt, sc))
    print(json.dumps({"shape": "scores_bmm", "mp_tflops": 2.0 * B * H * s * s * hd / t / 1e12,
                      "mp_us": t * 1e6, "hbm_gbs": sc.numel() * 2 / t / 1e9}), flush=True)
    ctx = torch.empty(B * s, H * hd, device="cuda", dtype=torch.bfloat16)
    cv = ctx.view(B, s, H, hd).permute(0, 2, 1, 3)
    t = timeit(lambda: native.gemm(sc, qh, cv))
    print(json.dumps({"shape": "ctx_bmm", "mp_tflops": 2.0 * B * H * s * s * hd / t / 1e12,
                      "mp_us": t * 1e6}), flush=True)


if __name__ == "__main__" and not {"--attn", "--epi", "--layer", "--one"} & set(sys.argv):
    sys.exit(main())


def bench_attention():
    import math
    B, H, s, d = 8, 32, 1024, 64
    T = B * s
    q, k, v, do = (torch.randn(T, H * d, device="cuda", dtype=torch.bfloat16) for _ in range(4))
    o = torch.empty_like(q)
    lse = torch.empty(B * H, s, device="cuda")
    sc = 1 / math.sqrt(d)
    t = timeit(lambda: native.attn_fwd(q, k, v, o, lse, B, H, s, d, sc))
    fl = 4.0 * B * H * s * s * d
    print(json.dumps({"shape": "attn_fwd", "tflops": fl / t / 1e12, "us": t * 1e6}), flush=True)
    dvec = torch.empty(B * H, s, device="cuda")
    dq = torch.zeros(T, H * d, device="cuda")
    dk, dv = torch.empty_like(q), torch.empty_like(q)
    t = timeit(lambda: native.attn_bwd(q, k, v, o, do, lse, dvec, dq, dk, dv, B, H, s, d, sc))
    print(json.dumps({"shape": "attn_bwd", "tflops": 2.5 * fl / t / 1e12, "us": t * 1e6}), flush=True)


if __name__ == "__main__" and "--attn" in sys.argv:
    bench_attention()


def bench_epilogues():
    M, K = 8192, 2048
    for name, N, K2, epi in (("mlp_up+gelu_dual", 8192, 2048, native.EPI_GELU_DUAL),
                             ("proj+add", 2048, 2048, native.EPI_ADD),
                             ("mlp_down+add", 2048, 8192, native.EPI_ADD),
                             ("dX_mlp2+gelu_grad", 8192, 2048, native.EPI_GELU_GRAD),
                             ("mlp_up plain", 8192, 2048, 0)):
        a = torch.randn(M, K2, device="cuda", dtype=torch.bfloat16)
        b = torch.randn(K2, N, device="cuda", dtype=torch.bfloat16)
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        aux = torch.randn(M, N, device="cuda", dtype=torch.bfloat16)
        t = timeit(lambda: native.gemm(a, b, out, epilogue=epi, aux=aux if epi else None))
        print(json.dumps({"shape": name, "tflops": 2.0 * M * N * K2 / t / 1e12, "us": t * 1e6}), flush=True)


if __name__ == "__main__" and "--epi" in sys.argv:
    bench_epilogues()


def bench_layer():
    """Every GEMM of one GPT-1.3B block for one 8-sequence microbatch, in the
    form the executor issues it (layouts, fused epilogues, fp32 beta=1 dW)."""
    T, h, f = 8192, 2048, 8192
    bf = dict(device="cuda", dtype=torch.bfloat16)
    X = torch.randn(T, h, **bf)
    Hh = torch.randn(T, f, **bf)
    W = torch.randn(h, h, **bf)
    W1 = torch.randn(h, f, **bf)
    W2 = torch.randn(f, h, **bf)
    o_h = torch.empty(T, h, **bf)
    o_f = torch.empty(T, f, **bf)
    aux_h = torch.randn(T, h, **bf)
    aux_f = torch.randn(T, f, **bf)
    g_hh = torch.zeros(h, h, device="cuda")
    g_hf = torch.zeros(h, f, device="cuda")
    g_fh = torch.zeros(f, h, device="cuda")
    E = native
    cases = [
        ("fwd q/k/v/o (x4)", 4, lambda: E.gemm(X, W, o_h), T, h, h),
        ("fwd fc1 + gelu dual", 1, lambda: E.gemm(X, W1, o_f, epilogue=E.EPI_GELU_DUAL, aux=aux_f), T, f, h),
        ("fwd fc2 + add", 1, lambda: E.gemm(Hh, W2, o_h, epilogue=E.EPI_ADD, aux=aux_h), T, h, f),
        ("dX fc2: g W2^T + gelu'", 1, lambda: E.gemm(X, W2.t(), o_f, epilogue=E.EPI_GELU_GRAD, aux=aux_f), T, f, h),
        ("dX fc1: dH W1^T + add", 1, lambda: E.gemm(Hh, W1.t(), o_h, epilogue=E.EPI_ADD, aux=aux_h), T, h, f),
        ("dX o/q/k/v: g W^T (+add) (x4)", 4, lambda: E.gemm(X, W.t(), o_h, epilogue=E.EPI_ADD, aux=aux_h), T, h, h),
        ("dW fc2: a^T g (fp32 +=)", 1, lambda: E.gemm(Hh.t(), X, g_fh, beta=1.0), f, h, T),
        ("dW fc1: x^T dH (fp32 +=)", 1, lambda: E.gemm(X.t(), Hh, g_hf, beta=1.0), h, f, T),
        ("dW o/q/k/v: x^T g (fp32 +=) (x4)", 4, lambda: E.gemm(X.t(), X, g_hh, beta=1.0), h, h, T),
    ]
    tot_t = tot_f = 0.0
    for name, n, fn, M, N, K in cases:
        t = timeit(fn)
        fl = 2.0 * M * N * K
        tot_t += n * t
        tot_f += n * fl
        print(json.dumps({"gemm": name, "M": M, "N": N, "K": K, "us": t * 1e6,
                          "tflops": fl / t / 1e12}), flush=True)
    print(json.dumps({"layer_gemm_ms": tot_t * 1e3, "layer_tflops": tot_f / tot_t / 1e12}), flush=True)


if __name__ == "__main__" and "--layer" in sys.argv:
    bench_layer()


def bench_one(M, N, K, ta=0, tb=0, iters=5):
    """One GEMM shape, a few launches (for ncu: -k regex:gemm -s 2 -c 1).
    ta / tb: operand stored transposed (A MN-major / B K-major)."""
    a = (torch.randn(K, M, device="cuda", dtype=torch.bfloat16).t() if ta else
         torch.randn(M, K, device="cuda", dtype=torch.bfloat16))
    b = (torch.randn(N, K, device="cuda", dtype=torch.bfloat16).t() if tb else
         torch.randn(K, N, device="cuda", dtype=torch.bfloat16))
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    t = timeit(lambda: native.gemm(a, b, out), iters=iters, warm=2)
    print(json.dumps({"M": M, "N": N, "K": K, "ta": ta, "tb": tb,
                      "tflops": 2.0 * M * N * K / t / 1e12, "us": t * 1e6}))


if __name__ == "__main__" and "--one" in sys.argv:
    i = sys.argv.index("--one")
    bench_one(*(int(x) for x in sys.argv[i + 1:i + 6]), iters=int(os.environ.get("ITERS", "20")))
