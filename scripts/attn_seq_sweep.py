"""fa_fwd / fa_bwd throughput against sequence length at a fixed token count (8192
tokens, 32 heads, d = 64): longer sequences mean more key tiles per CTA, so the
per-CTA start-up and drain cost shows up as the difference."""
import json
import math

import torch

from paper_2201_12023_b200 import native


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e-3


def main():
    H, d, T = 32, 64, 8192
    for s in (512, 1024, 2048, 4096):
        B = T // s
        q, k, v, do = (torch.randn(T, H * d, device="cuda", dtype=torch.bfloat16) for _ in range(4))
        o = torch.empty_like(q)
        lse = torch.empty(B * H, s, device="cuda")
        sc = 1 / math.sqrt(d)
        fl = 4.0 * B * H * s * s * d
        tf = timeit(lambda: native.attn_fwd(q, k, v, o, lse, B, H, s, d, sc))
        dvec = torch.empty(B * H, s, device="cuda")
        dq = torch.zeros(T, H * d, device="cuda")
        dk, dv = torch.empty_like(q), torch.empty_like(q)
        tb = timeit(lambda: native.attn_bwd(q, k, v, o, do, lse, dvec, dq, dk, dv, B, H, s, d, sc))
        print(json.dumps({"s": s, "fwd_tflops": fl / tf / 1e12, "bwd_tflops": 2.5 * fl / tb / 1e12}),
              flush=True)


if __name__ == "__main__":
    main()
