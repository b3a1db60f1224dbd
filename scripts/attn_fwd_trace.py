"""Where does the persistent fa_fwd spend its time between key tiles?  Runs the forward
at 8192 tokens with MPEXEC_FA_FWD_TRACE set, so the kernel stamps %globaltimer at fixed
points per key tile (softmax warp 2 and the MMA thread), and prints medians per position
of the key tile inside its work tile, relative to the softmax warps finishing P of the
previous key tile.

The stamps are compiled in only with -DMP_FA_TRACE:
    MPEXEC_NVCC_EXTRA=-DMP_FA_TRACE python -c \\
        "from paper_2201_12023_b200 import build_native; build_native.build(force=True)"
(rebuild without it afterwards).  Results: profiles/r2/fa_fwd_trace.jsonl."""
import json
import math
import os
import sys

import numpy as np

TRACE = "/tmp/fa_fwd_trace.bin"
os.environ["MPEXEC_FA_FWD_TRACE"] = TRACE

import torch  # noqa: E402

from paper_2201_12023_b200 import native  # noqa: E402

# slot -> (name, key-tile offset relative to J)
SLOTS = {7: ("MMA:S issued", 0), 0: ("SM:S seen", 0), 2: ("SM:o_done(prev tile)", -1),
         3: ("SM:epilogue done(prev tile)", -1), 4: ("MMA:PV begin (V ready)", 0),
         5: ("MMA:p_full seen", 0), 6: ("MMA:p_full1 seen", 0), 1: ("SM:P done", 0)}


def main():
    H, d, T = 32, 64, 8192
    for s in (1024, 4096):
        B = T // s
        q, k, v = (torch.randn(T, H * d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
        o = torch.empty_like(q)
        lse = torch.empty(B * H, s, device="cuda")
        for _ in range(3):
            native.attn_fwd(q, k, v, o, lse, B, H, s, d, 1 / math.sqrt(d))
        torch.cuda.synchronize()
        tr = np.fromfile(TRACE, dtype=np.int64).reshape(-1, 1024, 8)
        n_kv = s // 128
        rel = {}
        for row in tr:
            n = int((row[:, 1] >= 0).sum())
            for J in range(2, n):
                pos = J % n_kv
                base = row[J - 1, 1]
                for k_, (name, dj) in SLOTS.items():
                    v_ = row[J + dj, k_]
                    if v_ >= 0:
                        rel.setdefault(pos, {}).setdefault(name, []).append(int(v_ - base))
        out = {"s": s, "n_kv": n_kv,
               "ns_after_prev_P_done": {
                   p: {k_: float(np.median(v_)) for k_, v_ in d_.items()}
                   for p, d_ in sorted(rel.items()) if p < 3 or p == n_kv - 1}}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    sys.exit(main())
