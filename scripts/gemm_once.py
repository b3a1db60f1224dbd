"""One GEMM of a given shape/layout (for ncu captures): batch M N K ta tb f32acc [epilogue]."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2201_12023_b200 import native  # noqa: E402

batch, M, N, K, ta, tb, f32 = (int(x) for x in sys.argv[1:8])
epi = int(sys.argv[8]) if len(sys.argv) > 8 else 0
r = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16)  # noqa: E731
a = r(batch, K, M).transpose(-1, -2) if ta else r(batch, M, K)
b = r(batch, N, K).transpose(-1, -2) if tb else r(batch, K, N)
out = torch.zeros(batch, M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
aux = torch.randn_like(out, dtype=torch.bfloat16) if epi >= 2 else None
for _ in range(3):
    native.gemm(a, b, out, beta=1.0 if f32 else 0.0, epilogue=epi, aux=aux)
torch.cuda.synchronize()
print("ok")
