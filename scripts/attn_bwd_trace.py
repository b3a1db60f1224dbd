"""Where does fa_bwd's time go between query tiles?  Runs the backward at 8192 tokens
with MPEXEC_FA_BWD_TRACE set, so warp 2 stamps %globaltimer each time it publishes
P^T / dS^T for a query tile, and prints the median gap per position inside a work
tile.  Position 0 is the gap across a work-tile boundary.

The stamps are compiled in only with -DMP_FA_TRACE, so build a tracing library first:
    MPEXEC_NVCC_EXTRA=-DMP_FA_TRACE python -c \
        "from paper_2201_12023_b200 import build_native; build_native.build(force=True)"
(and rebuild without it afterwards).  Results: profiles/r2/fa_bwd_trace.jsonl."""
import json
import math
import os
import sys

import numpy as np

TRACE = "/tmp/fa_bwd_trace.bin"
os.environ["MPEXEC_FA_BWD_TRACE"] = TRACE

import torch  # noqa: E402

from paper_2201_12023_b200 import native  # noqa: E402


def main():
    H, d, T = 32, 64, 8192
    for s in (1024, 4096):
        B = T // s
        q, k, v, do = (torch.randn(T, H * d, device="cuda", dtype=torch.bfloat16) for _ in range(4))
        o = torch.empty_like(q)
        lse = torch.empty(B * H, s, device="cuda")
        sc = 1 / math.sqrt(d)
        native.attn_fwd(q, k, v, o, lse, B, H, s, d, sc)
        dvec = torch.empty(B * H, s, device="cuda")
        dq = torch.zeros(T, H * d, device="cuda")
        dk, dv = torch.empty_like(q), torch.empty_like(q)
        for _ in range(3):
            native.attn_bwd(q, k, v, o, do, lse, dvec, dq, dk, dv, B, H, s, d, sc)
        torch.cuda.synchronize()
        tr = np.fromfile(TRACE, dtype=np.int64).reshape(-1, 1024, 8)
        n_q = s // 128
        # per query tile g: stamps relative to the P warps' ps_full of g-1
        names = {"P:q_full": (0, 0), "P:st_full": (0, 1), "P:pbuf_free": (0, 2),
                 "P:ps_full": (0, 3), "MMA:S/dP issue": (0, 4), "MMA:acc(g-1) issue": (-1, 5),
                 "MMA:dQ(g-1) issue": (-1, 6), "dQ:dq_full(g-1)": (-1, 7),
                 "dQ:dq_full(g-2)": (-2, 7)}
        rel = {}
        for row in tr:
            n = int((row[:, 3] >= 0).sum())
            for g in range(2, n):
                pos = g % n_q
                base = row[g - 1, 3]
                for name, (dg, k) in names.items():
                    v_ = row[g + dg, k]
                    if v_ >= 0:
                        rel.setdefault(pos, {}).setdefault(name, []).append(v_ - base)
        out = {"s": s, "n_q": n_q, "span_us": float(tr[tr >= 0].max() - tr[tr >= 0].min()) / 1e3,
               "ns_after_prev_ps_full": {
                   p: {k: float(np.median(v_)) for k, v_ in d_.items()}
                   for p, d_ in sorted(rel.items()) if p < 4 or p == n_q - 1}}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    sys.exit(main())
