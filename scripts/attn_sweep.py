"""Fused attention throughput vs sequence length (fixed tokens per launch):
separates per-CTA fixed cost from the per-query-tile loop."""
import json
import math
import sys

import torch

from paper_2201_12023_b200 import native

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from bench_gemm import timeit  # noqa: E402

H, d = 32, 64
for B, s in ((16, 512), (8, 1024), (4, 2048), (2, 4096)):
    T = B * s
    q, k, v, do = (torch.randn(T, H * d, device="cuda", dtype=torch.bfloat16) for _ in range(4))
    o = torch.empty_like(q)
    lse = torch.empty(B * H, s, device="cuda")
    sc = 1 / math.sqrt(d)
    tf = timeit(lambda: native.attn_fwd(q, k, v, o, lse, B, H, s, d, sc))
    dvec = torch.empty(B * H, s, device="cuda")
    dq = torch.zeros(T, H * d, device="cuda")
    dk, dv = torch.empty_like(q), torch.empty_like(q)
    tb = timeit(lambda: native.attn_bwd(q, k, v, o, do, lse, dvec, dq, dk, dv, B, H, s, d, sc))
    fl = 4.0 * B * H * s * s * d
    print(json.dumps({"B": B, "s": s, "fwd_tflops": fl / tf / 1e12, "bwd_tflops": 2.5 * fl / tb / 1e12,
                      "fwd_us": tf * 1e6, "bwd_us": tb * 1e6}), flush=True)
