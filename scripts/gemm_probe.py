"""Isolated timing of a few GEMM shapes/layouts (CUDA events, warm-up), with the
split-K path on and off.  python scripts/gemm_probe.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2201_12023_b200 import native  # noqa: E402


def t(fn, it=20):
    """GPU time per call: `it` calls captured in one CUDA graph (no host
    launch overhead in the measurement), replayed after a warm-up."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(it):
            fn()
    g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3


def mk(batch, M, N, K, ta, tb, f32):
    r = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16)  # noqa: E731
    a = r(batch, K, M).transpose(-1, -2) if ta else r(batch, M, K)
    b = r(batch, N, K).transpose(-1, -2) if tb else r(batch, K, N)
    if batch == 1:
        a, b = a[0], b[0]
    out = torch.zeros(*((batch,) if batch > 1 else ()), M, N, device="cuda",
                      dtype=torch.float32 if f32 else torch.bfloat16)
    return a, b, out


CASES = [  # batch, M, N, K, ta, tb, f32 (beta=1 accumulate), epilogue
    (1, 1024, 1024, 8192, 1, 0, 1, 0), (1, 1024, 16, 8192, 1, 0, 1, 0),
    (16, 1024, 8192, 1024, 1, 0, 1, 0), (16, 8192, 1024, 1024, 1, 0, 1, 0),
    (16, 1024, 8192, 1024, 0, 0, 0, 0), (16, 1024, 8192, 1024, 0, 0, 0, 4),
    (16, 1024, 8192, 1024, 0, 1, 0, 0), (16, 1024, 8192, 1024, 0, 1, 0, 3),
    (16, 1024, 1024, 8192, 0, 1, 0, 0), (16, 1024, 1024, 8192, 0, 0, 0, 0),
    (1, 8192, 1024, 1024, 0, 0, 0, 0), (1, 8192, 1024, 1024, 0, 1, 0, 0),
    (1, 8192, 8192, 1024, 0, 0, 0, 4), (1, 8192, 8192, 1024, 0, 1, 0, 3),
    (8, 2048, 1024, 1024, 0, 1, 0, 0), (8, 1024, 1024, 2048, 0, 0, 0, 0),
    (1, 8192, 2048, 2048, 0, 0, 0, 0), (1, 8192, 2048, 2048, 0, 0, 1, 0),
    (1, 8192, 8192, 2048, 0, 0, 0, 0), (1, 8192, 8192, 2048, 0, 0, 1, 0),
    (1, 8192, 8192, 2048, 0, 0, 0, 4), (1, 8192, 8192, 2048, 0, 1, 0, 3),
    (1, 2048, 2048, 8192, 1, 0, 1, 0),
    (1, 8192, 2048, 2048, 0, 0, 0, 2), (1, 8192, 2048, 8192, 0, 0, 0, 2),
    (16, 1024, 1024, 8192, 0, 0, 0, 2),
]
for batch, M, N, K, ta, tb, f32, epi in CASES:
    a, b, out = mk(batch, M, N, K, ta, tb, f32)
    aux = torch.empty_like(out, dtype=torch.bfloat16) if epi else None
    if epi in (2, 3):
        aux.normal_()
    fl = 2.0 * batch * M * N * K
    res = []
    for sk in ((True, False) if f32 else (True,)):
        native.SPLIT_K = sk
        us = t(lambda: native.gemm(a, b, out, beta=1.0 if f32 else 0.0, epilogue=epi, aux=aux))
        res.append(f"{'split' if sk else 'plain'} {us:8.1f} us {fl / us / 1e6:6.0f} TF/s")
    print(f"b{batch:<3d} {M:5d} {N:5d} {K:5d} {'T' if ta else 'N'}{'T' if tb else 'N'} "
          f"{'f32+=' if f32 else 'bf16 '} epi{epi}  " + " | ".join(res), flush=True)
native.SPLIT_K = True
