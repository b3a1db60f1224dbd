"""Fused tcgen05 attention vs a plain PyTorch fp32 reference of the same op
(non-causal softmax(q k^T / sqrt(d)) v on (B*s, H*d) tensors).
Tolerance: relative Frobenius error <= 1e-2 for O and LSE, <= 2e-2 for the grads."""
import math

import pytest
import torch

from paper_2201_12023_b200 import native

pytestmark = pytest.mark.gpu


def rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm()).item()


def ref_attention(q, k, v, B, H, s, d):
    def heads(t):
        return t.float().view(B, s, H, d).permute(0, 2, 1, 3)
    qh, kh, vh = heads(q), heads(k), heads(v)
    scale = 1.0 / math.sqrt(d)
    sc = scale * qh @ kh.transpose(-1, -2)
    lse = torch.logsumexp(sc, -1)
    o = torch.softmax(sc, -1) @ vh
    return o.permute(0, 2, 1, 3).reshape(B * s, H * d), lse.reshape(B * H, s)


# (3, 40, 1024, 64): 960 work tiles, so both persistent kernels loop over several tiles
# per CTA with an uneven last round (forward: 296 CTAs, backward: 148)
@pytest.mark.parametrize("B,H,s,extra", [(1, 1, 128, 0), (2, 4, 256, 0), (2, 4, 1024, 0),
                                         (1, 2, 384, 128), (3, 40, 1024, 64)])
def test_attention_forward_backward(B, H, s, extra):
    torch.manual_seed(0)
    d = 64
    ld = H * d + extra
    T = B * s
    base = torch.randn(4, T, ld, device="cuda", dtype=torch.bfloat16)
    q, k, v, do = (base[i, :, :H * d] for i in range(4))
    o = torch.empty(T, ld, device="cuda", dtype=torch.bfloat16)[:, :H * d]
    lse = torch.empty(B * H, s, device="cuda", dtype=torch.float32)
    scale = 1.0 / math.sqrt(d)
    native.attn_fwd(q, k, v, o, lse, B, H, s, d, scale)
    qf, kf, vf = (t.float().requires_grad_() for t in (q, k, v))
    ro, rlse = ref_attention(qf, kf, vf, B, H, s, d)
    assert rel(o, ro) < 1e-2
    assert rel(lse, rlse) < 1e-3
    ro.backward(do.float())
    dvec = torch.empty(B * H, s, device="cuda", dtype=torch.float32)
    dq = torch.zeros(T, ld, device="cuda", dtype=torch.float32)[:, :H * d]
    dk = torch.empty(T, ld, device="cuda", dtype=torch.bfloat16)[:, :H * d]
    dv = torch.empty(T, ld, device="cuda", dtype=torch.bfloat16)[:, :H * d]
    native.attn_bwd(q, k, v, o, do, lse, dvec, dq, dk, dv, B, H, s, d, scale)
    assert rel(dv, vf.grad) < 2e-2
    assert rel(dk, kf.grad) < 2e-2
    assert rel(dq, qf.grad) < 2e-2


def test_attention_rejects_bad_head_dim():
    x = torch.zeros(128, 128, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(1, 128, device="cuda")
    with pytest.raises(native.NativeError):
        native.attn_fwd(x, x, x, x, lse, 1, 1, 128, 128, 0.1)


def test_attention_forward_key_range():
    """kv_range=(kv0, len): O and LSE over that key slice only (the key-split path)."""
    torch.manual_seed(1)
    B, H, s, d = 2, 40, 1024, 64
    kv0, kvl = 256, 512
    q, k, v = (torch.randn(B * s, H * d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    o = torch.empty_like(q)
    lse = torch.empty(B * H, s, device="cuda", dtype=torch.float32)
    native.attn_fwd(q, k, v, o, lse, B, H, s, d, 1.0 / math.sqrt(d), kv_range=(kv0, kvl))

    def heads(t):
        return t.float().view(B, s, H, d).permute(0, 2, 1, 3)
    qh, kh, vh = heads(q), heads(k)[:, :, kv0:kv0 + kvl], heads(v)[:, :, kv0:kv0 + kvl]
    sc = qh @ kh.transpose(-1, -2) / math.sqrt(d)
    ro = (torch.softmax(sc, -1) @ vh).permute(0, 2, 1, 3).reshape(B * s, H * d)
    assert rel(o, ro) < 1e-2
    assert rel(lse, torch.logsumexp(sc, -1).reshape(B * H, s)) < 1e-3

