"""One fused-attention forward + backward at the GPT-1.3B shape (8 x 1024 tokens,
32 heads, d = 64), for ncu captures of the two kernels."""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2201_12023_b200 import native  # noqa: E402

B, s, H, d = 8, 1024, 32, 64
T = B * s
q, k, v, do = (torch.randn(T, H * d, device="cuda", dtype=torch.bfloat16) for _ in range(4))
o = torch.empty_like(q)
lse = torch.empty(B * H, s, device="cuda")
dvec = torch.empty(B * H, s, device="cuda")
dq = torch.empty(T, H * d, device="cuda")
dk, dv = torch.empty_like(q), torch.empty_like(q)
for _ in range(2):
    native.attn_fwd(q, k, v, o, lse, B, H, s, d, 1 / math.sqrt(d))
    native.attn_bwd(q, k, v, o, do, lse, dvec, dq, dk, dv, B, H, s, d, 1 / math.sqrt(d))
torch.cuda.synchronize()
print("ok")
