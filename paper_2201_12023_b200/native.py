"""ctypes binding of libmpexec.so (include/mp_exec.h) plus torch-tensor helpers.

This is the only door from the host runtime to device work.  There is no
fallback: if the library is missing or a call fails, a NativeError is raised
(the reference's errors are exceptions too, e.g. SimError at sim.py:26).
"""
from __future__ import annotations

import ctypes
import math
import os
from pathlib import Path
from typing import Optional

import torch

_LIB_PATH = Path(__file__).resolve().parent / "libmpexec.so"
_lib: Optional[ctypes.CDLL] = None

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_f32 = ctypes.c_float
c_vp = ctypes.c_void_p
c_i64p = ctypes.POINTER(ctypes.c_int64)

EXPORTS = {
    "mp_abi_version": ([], c_int),
    "mp_last_error": ([], ctypes.c_char_p),
    "mp_launch_count": ([], ctypes.c_uint64),
    "mp_gemm_bf16": ([c_vp, c_i64p, c_vp, c_i64p, c_vp, c_i64p, c_int, c_i64, c_i64,
                      c_f32, c_f32, c_int, c_vp], c_int),
    "mp_gemm_bf16_ex": ([c_vp, c_i64p, c_vp, c_i64p, c_vp, c_i64p, c_int, c_i64, c_i64,
                         c_f32, c_f32, c_int, c_vp, c_i64p, c_vp], c_int),
    "mp_gelu_fwd": ([c_vp, c_vp, c_i64, c_vp], c_int),
    "mp_gelu_bwd": ([c_vp, c_vp, c_vp, c_i64, c_vp], c_int),
    "mp_add": ([c_vp, c_vp, c_vp, c_i64, c_vp], c_int),
    "mp_scale": ([c_vp, c_vp, c_f32, c_i64, c_vp], c_int),
    "mp_sumsq": ([c_vp, c_vp, c_i64, c_vp], c_int),
    "mp_softmax_fwd": ([c_vp, c_vp, c_i64, c_i64, c_i64, c_f32, c_vp], c_int),
    "mp_softmax_stats": ([c_vp, c_vp, c_i64, c_i64, c_i64, c_f32, c_vp], c_int),
    "mp_softmax_rescale": ([c_vp, c_i64, c_vp], c_int),
    "mp_softmax_apply": ([c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_f32, c_vp], c_int),
    "mp_softmax_bwd": ([c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_f32, c_vp], c_int),
    "mp_softmax_rowdot": ([c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp], c_int),
    "mp_attn_fwd": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_f32,
                     c_vp], c_int),
    "mp_attn_bwd": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64,
                     c_i64, c_i64, c_i64, c_f32, c_vp], c_int),
    "mp_attn_fwd_kv": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_f32,
                        c_i64, c_i64, c_vp], c_int),
    "mp_attn_bwd_kv": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64,
                        c_i64, c_i64, c_i64, c_i64, c_f32, c_i64, c_i64, c_vp], c_int),
    "mp_attn_combine_scale": ([c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp],
                              c_int),
    "mp_attn_combine_finish": ([c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp],
                               c_int),
    "mp_nccl_version": ([], c_int),
    "mp_nccl_unique_id": ([c_vp], c_int),
    "mp_comm_init": ([c_vp, c_int, c_int, ctypes.POINTER(c_vp)], c_int),
    "mp_comm_destroy": ([c_vp], c_int),
    "mp_comm_abort": ([c_vp], c_int),
    "mp_preload_kernels": ([], c_int),
    "mp_comm_async_error": ([c_vp, ctypes.POINTER(c_int)], c_int),
    "mp_allreduce": ([c_vp, c_vp, c_i64, c_int, c_int, c_vp], c_int),
    "mp_allgather": ([c_vp, c_vp, c_vp, c_i64, c_int, c_vp], c_int),
    "mp_reduce_scatter": ([c_vp, c_vp, c_vp, c_i64, c_int, c_int, c_vp], c_int),
    "mp_group_start": ([], c_int),
    "mp_group_end": ([], c_int),
    "mp_alltoall": ([c_vp, c_vp, c_vp, c_i64, c_int, c_vp], c_int),
    "mp_send": ([c_vp, c_vp, c_i64, c_int, c_int, c_vp], c_int),
    "mp_recv": ([c_vp, c_vp, c_i64, c_int, c_int, c_vp], c_int),
    "mp_ilp_solve": ([c_int, ctypes.POINTER(c_int), c_i64p, c_int, ctypes.POINTER(c_int),
                      ctypes.POINTER(c_int), c_i64p, c_i64, ctypes.POINTER(c_int), c_i64p,
                      ctypes.POINTER(c_int), c_i64p], c_int),
    "mp_moe_route": ([c_vp, c_i64, c_i64, c_int, c_int, c_int, c_vp, c_vp], c_int),
    "mp_moe_mask": ([c_vp, c_vp, c_i64, c_vp, c_i64, c_int, c_int, c_int, c_int, c_vp], c_int),
    "mp_moe_mask_grad": ([c_vp, c_vp, c_vp, c_i64, c_int, c_int, c_int, c_int, c_vp], c_int),
    "mp_im2col": ([c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_int, c_int, c_int, c_vp], c_int),
    "mp_subsample": ([c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_int, c_int, c_vp], c_int),
    "mp_reduce_mid": ([c_vp, c_vp, c_i64, c_i64, c_i64, c_int, c_vp], c_int),
    "mp_pack_box": ([c_vp, c_i64p, c_i64p, c_i64p, c_int, c_int, c_vp, c_vp], c_int),
    "mp_unpack_box": ([c_vp, c_vp, c_i64p, c_i64p, c_i64p, c_int, c_int, c_vp], c_int),
    "mp_adam_step": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_f32, c_f32, c_f32, c_f32, c_f32,
                      c_f32, c_i64, c_vp], c_int),
    "mp_cast_f32_bf16": ([c_vp, c_vp, c_i64, c_vp], c_int),
    "mp_cast_bf16_f32": ([c_vp, c_vp, c_i64, c_vp], c_int),
    "mp_accum_bf16_f32": ([c_vp, c_vp, c_i64, c_vp], c_int),
    "mp_sum_parts_f32": ([c_vp, c_i64, c_i64, c_vp, c_f32, c_vp], c_int),
}


class NativeError(RuntimeError):
    """A libmpexec call failed (or the library is absent)."""


def lib_path() -> Path:
    return _LIB_PATH


def load(path: Optional[Path] = None) -> ctypes.CDLL:
    """Load libmpexec.so and bind every exported symbol; raises if anything is
    missing.  Never falls back to another implementation."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path or os.environ.get("MPEXEC_LIB", _LIB_PATH))
    if not p.exists():
        raise NativeError(f"{p} not built; run `python -m paper_2201_12023_b200.build_native`")
    lib = ctypes.CDLL(str(p))
    for name, (args, res) in EXPORTS.items():
        fn = getattr(lib, name, None)
        if fn is None:
            raise NativeError(f"{p} does not export {name}")
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().mp_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed (rc={rc}): {msg}")


def preload_kernels() -> None:
    _check(load().mp_preload_kernels(), "mp_preload_kernels")


def launch_count() -> int:
    return int(load().mp_launch_count())


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _arr(vals) -> ctypes.Array:
    return (ctypes.c_int64 * len(vals))(*[int(v) for v in vals])


def _require(t: torch.Tensor, dtype: torch.dtype, name: str) -> None:
    if not t.is_cuda:
        raise NativeError(f"{name} must be a CUDA tensor (no CPU path)")
    if t.dtype != dtype:
        raise NativeError(f"{name} must be {dtype}, got {t.dtype}")


# --------------------------------------------------------------------------- GEMM

def _split_batch(t: torch.Tensor, name: str):
    """(…, R, C) view -> (descriptor[6], batch extents (nb0, nb1)).  Up to two
    batch dims; a 1-batch-dim view uses (1, n)."""
    if t.dim() < 2 or t.dim() > 4:
        raise NativeError(f"{name}: rank {t.dim()} unsupported (2..4)")
    r, c = t.shape[-2], t.shape[-1]
    rs, cs = t.stride(-2), t.stride(-1)
    if r == 1:
        rs = cs * c if cs == 1 else 1
    if c == 1:
        cs = 1 if rs != 1 else r
    if t.dim() == 2:
        return [r, c, rs, cs, 0, 0], (1, 1)
    if t.dim() == 3:
        return [r, c, rs, cs, 0, t.stride(0)], (1, t.shape[0])
    return [r, c, rs, cs, t.stride(0), t.stride(1)], (t.shape[0], t.shape[1])


# Optional per-launch timing of the GEMM (bench.py roofline): list of
# (flops, start_event, end_event) recorded on the launching stream.
gemm_timer: Optional[list] = None


EPI_NONE, EPI_GELU, EPI_ADD, EPI_GELU_GRAD, EPI_GELU_DUAL = 0, 1, 2, 3, 4


def gemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, *, alpha: float = 1.0,
         beta: float = 0.0, gelu: bool = False, epilogue: int = 0,
         aux: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """out = epi(alpha * a @ b + beta * out) on the tcgen05 kernel.  a: (…, M, K),
    b: (…, K, N) bf16 views (any of K-/MN-major), out: (…, M, N) bf16 or fp32
    with unit column stride.  Batch dims must agree.  epilogue (see
    include/mp_exec.h): EPI_ADD / EPI_GELU_GRAD read `aux`, EPI_GELU_DUAL
    writes gelu(out) into `aux`; aux has out's shape, bf16, unit column stride."""
    _require(a, torch.bfloat16, "a")
    _require(b, torch.bfloat16, "b")
    if out.dtype not in (torch.bfloat16, torch.float32):
        raise NativeError("out must be bf16 or fp32")
    # TMA needs 16-byte aligned non-unit strides: operands / outputs with an odd
    # inner extent (the Wide-ResNet stem's 7*7*3 = 147 im2col columns, a 4-expert
    # gate) go through zero-padded copies
    a, b = _aligned(a), _aligned(b)
    if not _is_aligned(out) and epilogue == 0 and not gelu:
        tmp = _aligned(out, copy=beta != 0.0)
        gemm(a, b, tmp, alpha=alpha, beta=beta, stream=stream)
        out.copy_(tmp)
        return out
    ad, ab = _split_batch(a, "a")
    bd, bb = _split_batch(b, "b")
    cd, cb = _split_batch(out, "out")
    if not (ab == bb == cb):
        raise NativeError(f"batch mismatch {ab} {bb} {cb}")
    epi = 1 if gelu else int(epilogue)
    aux_ptr, aux_desc = None, None
    if epi >= 2:
        if aux is None:
            raise NativeError("epilogue needs aux")
        _require(aux, torch.bfloat16, "aux")
        xd, xb = _split_batch(aux, "aux")
        if xb != cb or xd[0] != cd[0] or xd[1] != cd[1] or xd[3] != 1:
            raise NativeError("aux must match out's shape with unit column stride")
        aux_ptr, aux_desc = aux.data_ptr(), _arr([xd[2], xd[4], xd[5]])
    if epi == 0 and out.dtype == torch.float32 and a.dim() == 2 and \
            b.dim() == 2 and out.is_contiguous():
        s = _split_k(ad[0], bd[1], ad[1])
        if s > 1:
            return _gemm_split_k(a, b, out, s, alpha, beta, stream)
    st = _stream(stream)
    timer = gemm_timer
    if timer is not None:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
    rc = load().mp_gemm_bf16_ex(a.data_ptr(), _arr(ad), b.data_ptr(), _arr(bd), out.data_ptr(),
                                _arr(cd), 1 if out.dtype == torch.float32 else 0, ab[0], ab[1],
                                float(alpha), float(beta), epi, aux_ptr, aux_desc, st)
    _check(rc, "mp_gemm_bf16_ex")
    if timer is not None:
        e1.record()
        timer.append((2.0 * ad[0] * ad[1] * bd[1] * ab[0] * ab[1], e0, e1))
    return out


def _is_aligned(t: torch.Tensor) -> bool:
    q = 16 // t.element_size()
    return t.data_ptr() % 16 == 0 and all(st % q == 0 for st, n in zip(t.stride(), t.shape)
                                          if st != 1 and n > 1)


def _aligned(t: torch.Tensor, copy: bool = True) -> torch.Tensor:
    """t itself when its strides suit TMA, else an equal-valued view into a buffer
    whose contiguous dim is padded to 16 bytes (zeros in the padding)."""
    if _is_aligned(t):
        return t
    q = 16 // t.element_size()
    inner = -1 if t.stride(-1) == 1 else -2
    shape = list(t.shape)
    if inner == -2:
        t2 = t.transpose(-1, -2)
        shape[-2], shape[-1] = shape[-1], shape[-2]
    else:
        t2 = t
    padded = shape[:-1] + [-(-shape[-1] // q) * q]
    buf = torch.zeros(padded, dtype=t.dtype, device=t.device)
    view = buf[..., :shape[-1]]
    if copy:
        view.copy_(t2)
    return view if inner == -1 else view.transpose(-1, -2)


SPLIT_K = os.environ.get("MPEXEC_SPLIT_K", "1") != "0"


def _split_k(M: int, N: int, K: int) -> int:
    """K splits for an accumulating fp32 GEMM whose output tiles fill at most half
    the machine (2-CTA pair tiles on 74 SM pairs, else 1-CTA tiles on 148 SMs):
    the largest power of two keeping tiles * splits within one wave and
    K / splits >= 512 in whole 64-deep k-blocks."""
    if not SPLIT_K:
        return 1
    if M >= 256 and N >= 256:
        tiles, cap = -(-M // 256) * -(-N // 256), 74
    else:
        bn = 256 if N > 128 else (128 if N > 64 else 64)
        tiles, cap = -(-M // 128) * -(-N // bn), 148
    s = 1
    while tiles * s * 2 <= cap and K % (64 * s * 2) == 0 and K // (s * 2) >= 512:
        s *= 2
    return s


def _gemm_split_k(a, b, out, s, alpha, beta, stream):
    """out = beta*out + alpha*a@b as s K-chunk GEMMs (one batched launch into fp32
    partials) plus an in-order sum (deterministic)."""
    M, K = a.shape
    N = b.shape[1]
    kc = K // s
    a3 = a.as_strided((s, M, kc), (kc * a.stride(1), a.stride(0), a.stride(1)))
    b3 = b.as_strided((s, kc, N), (kc * b.stride(0), b.stride(0), b.stride(1)))
    parts = torch.empty(s, M, N, dtype=torch.float32, device=out.device)
    gemm(a3, b3, parts, alpha=alpha, beta=0.0, stream=stream)
    _check(load().mp_sum_parts_f32(parts.data_ptr(), s, M * N, out.data_ptr(), float(beta),
                                   _stream(stream)), "mp_sum_parts_f32")
    if stream is not None:
        parts.record_stream(stream)
    return out


# --------------------------------------------------------------------------- elementwise

def _contig(t: torch.Tensor, name: str) -> None:
    if not t.is_contiguous():
        raise NativeError(f"{name} must be contiguous")


def gelu(x: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    _require(x, torch.bfloat16, "x")
    _contig(x, "x")
    out = torch.empty_like(x) if out is None else out
    _check(load().mp_gelu_fwd(x.data_ptr(), out.data_ptr(), x.numel(), _stream(stream)), "mp_gelu_fwd")
    return out


def gelu_bwd(x: torch.Tensor, dy: torch.Tensor, out: Optional[torch.Tensor] = None,
             stream=None) -> torch.Tensor:
    for t, n in ((x, "x"), (dy, "dy")):
        _require(t, torch.bfloat16, n)
        _contig(t, n)
    out = torch.empty_like(x) if out is None else out
    _check(load().mp_gelu_bwd(x.data_ptr(), dy.data_ptr(), out.data_ptr(), x.numel(),
                              _stream(stream)), "mp_gelu_bwd")
    return out


def add(a: torch.Tensor, b: torch.Tensor, out: Optional[torch.Tensor] = None,
        stream=None) -> torch.Tensor:
    for t, n in ((a, "a"), (b, "b")):
        _require(t, torch.bfloat16, n)
        _contig(t, n)
    if a.shape != b.shape:
        raise NativeError(f"add shape mismatch {tuple(a.shape)} {tuple(b.shape)}")
    out = torch.empty_like(a) if out is None else out
    _check(load().mp_add(a.data_ptr(), b.data_ptr(), out.data_ptr(), a.numel(), _stream(stream)),
           "mp_add")
    return out


def scale(x: torch.Tensor, s: float, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    _require(x, torch.bfloat16, "x")
    _contig(x, "x")
    out = torch.empty_like(x) if out is None else out
    _check(load().mp_scale(x.data_ptr(), out.data_ptr(), float(s), x.numel(), _stream(stream)),
           "mp_scale")
    return out


def sumsq(x: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
    _require(x, torch.bfloat16, "x")
    _contig(x, "x")
    _require(out, torch.float32, "out")
    _check(load().mp_sumsq(x.data_ptr(), out.data_ptr(), x.numel(), _stream(stream)), "mp_sumsq")
    return out


def _rows(x: torch.Tensor, name: str):
    if x.stride(-1) != 1:
        raise NativeError(f"{name}: last dim must be unit-stride")
    cols = x.shape[-1]
    rows = x.numel() // cols if cols else 0
    # rows of a (…, cols) tensor must be equally spaced
    ld = x.stride(-2) if x.dim() >= 2 else cols
    if x.dim() > 2:
        exp = ld * x.shape[-2]
        for d in range(x.dim() - 3, -1, -1):
            if x.stride(d) != exp:
                raise NativeError(f"{name}: rows not uniformly strided")
            exp *= x.shape[d]
    return rows, cols, ld


def softmax(x: torch.Tensor, s: float, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    _require(x, torch.bfloat16, "x")
    out = torch.empty_like(x) if out is None else out
    rows, cols, ld = _rows(x, "x")
    if _rows(out, "out")[2] != ld:
        raise NativeError("softmax out must share the input row stride")
    _check(load().mp_softmax_fwd(x.data_ptr(), out.data_ptr(), rows, cols, ld, float(s),
                                 _stream(stream)), "mp_softmax_fwd")
    return out


def softmax_stats(x: torch.Tensor, s: float, stats: torch.Tensor, stream=None) -> torch.Tensor:
    _require(x, torch.bfloat16, "x")
    _require(stats, torch.float32, "stats")
    rows, cols, ld = _rows(x, "x")
    _check(load().mp_softmax_stats(x.data_ptr(), stats.data_ptr(), rows, cols, ld, float(s),
                                   _stream(stream)), "mp_softmax_stats")
    return stats


def softmax_rescale(stats: torch.Tensor, rows: int, stream=None) -> torch.Tensor:
    _require(stats, torch.float32, "stats")
    _check(load().mp_softmax_rescale(stats.data_ptr(), rows, _stream(stream)), "mp_softmax_rescale")
    return stats


def softmax_apply(x: torch.Tensor, stats: torch.Tensor, s: float,
                  out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    _require(x, torch.bfloat16, "x")
    out = torch.empty_like(x) if out is None else out
    rows, cols, ld = _rows(x, "x")
    _check(load().mp_softmax_apply(x.data_ptr(), stats.data_ptr(), out.data_ptr(), rows, cols, ld,
                                   float(s), _stream(stream)), "mp_softmax_apply")
    return out


def softmax_rowdot(y: torch.Tensor, dy: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
    rows, cols, ld = _rows(y, "y")
    _check(load().mp_softmax_rowdot(y.data_ptr(), dy.data_ptr(), out.data_ptr(), rows, cols, ld,
                                    _stream(stream)), "mp_softmax_rowdot")
    return out


def softmax_bwd(y: torch.Tensor, dy: torch.Tensor, s: float, rowdot: Optional[torch.Tensor] = None,
                out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    _require(y, torch.bfloat16, "y")
    _require(dy, torch.bfloat16, "dy")
    out = torch.empty_like(y) if out is None else out
    rows, cols, ld = _rows(y, "y")
    if _rows(dy, "dy")[2] != ld or _rows(out, "out")[2] != ld:
        raise NativeError("softmax_bwd operands must share the row stride")
    _check(load().mp_softmax_bwd(y.data_ptr(), dy.data_ptr(), out.data_ptr(),
                                 rowdot.data_ptr() if rowdot is not None else None, rows, cols, ld,
                                 float(s), _stream(stream)), "mp_softmax_bwd")
    return out


# --------------------------------------------------------------------------- attention

def _heads_view(t: torch.Tensor, name: str):
    """(T, ld) bf16 with unit column stride -> (ptr, ld)."""
    _require(t, torch.bfloat16, name)
    if t.dim() != 2 or t.stride(1) != 1:
        raise NativeError(f"{name} must be a (tokens, hidden) row-major view")
    return t.data_ptr(), t.stride(0)


def attn_fwd(q, k, v, o, lse, B: int, H: int, s: int, d: int, scale: float, stream=None,
             kv_range=None):
    """Fused non-causal attention forward on (B*s, H*d) tensors; lse fp32 [B*H, s].
    kv_range=(kv0, kv_len) restricts the keys (O / lse then cover that range)."""
    ptrs = [_heads_view(t, n) for t, n in ((q, "q"), (k, "k"), (v, "v"), (o, "o"))]
    lds = {ld for _, ld in ptrs}
    if len(lds) != 1:
        raise NativeError("q/k/v/o must share the row stride")
    _require(lse, torch.float32, "lse")
    kv0, kvl = kv_range if kv_range is not None else (0, s)
    _check(load().mp_attn_fwd_kv(ptrs[0][0], ptrs[1][0], ptrs[2][0], ptrs[3][0], lse.data_ptr(),
                                 B, H, s, d, lds.pop(), float(scale), kv0, kvl, _stream(stream)),
           "mp_attn_fwd")


def attn_bwd(q, k, v, o, dout, lse, dvec, dq_acc, dk, dv, B: int, H: int, s: int, d: int,
             scale: float, stream=None, kv_range=None):
    ptrs = [_heads_view(t, n) for t, n in ((q, "q"), (k, "k"), (v, "v"), (o, "o"), (dout, "dout"),
                                            (dk, "dk"), (dv, "dv"))]
    lds = {ld for _, ld in ptrs} | {dq_acc.stride(0)}
    if len(lds) != 1:
        raise NativeError("attention operands must share the row stride")
    kv0, kvl = kv_range if kv_range is not None else (0, s)
    _check(load().mp_attn_bwd_kv(ptrs[0][0], ptrs[1][0], ptrs[2][0], ptrs[3][0], ptrs[4][0],
                                 lse.data_ptr(), dvec.data_ptr(), dq_acc.data_ptr(), ptrs[5][0],
                                 ptrs[6][0], B, H, s, d, lds.pop(), float(scale), kv0, kvl,
                                 _stream(stream)),
           "mp_attn_bwd")


def attn_combine_scale(o, lse, m, w, B: int, H: int, s: int, d: int, stream=None):
    """Key-split combine, step 1: w = exp(lse - m); o *= w (row-wise per head)."""
    p, ld = _heads_view(o, "o")
    for t, n in ((lse, "lse"), (m, "m"), (w, "w")):
        _require(t, torch.float32, n)
    _check(load().mp_attn_combine_scale(p, lse.data_ptr(), m.data_ptr(), w.data_ptr(), B, H, s, d,
                                        ld, _stream(stream)), "mp_attn_combine_scale")


def attn_combine_finish(o, wsum, m, lse, B: int, H: int, s: int, d: int, stream=None):
    """Key-split combine, step 2: o /= wsum; lse = m + log(wsum)."""
    p, ld = _heads_view(o, "o")
    for t, n in ((wsum, "wsum"), (m, "m"), (lse, "lse")):
        _require(t, torch.float32, n)
    _check(load().mp_attn_combine_finish(p, wsum.data_ptr(), m.data_ptr(), lse.data_ptr(), B, H, s,
                                         d, ld, _stream(stream)), "mp_attn_combine_finish")


# --------------------------------------------------------------------------- boxes

# --------------------------------------------------------------------------- MoE routing

def moe_route(gates: torch.Tensor, S: int, C: int, route: Optional[torch.Tensor] = None,
              stream=None) -> torch.Tensor:
    """GShard top-2 routing of (T, E) bf16 gates in groups of S tokens, capacity C
    -> int32 (T, 4) {e1, pos1|-1, e2, pos2|-1} (csrc/moe.cu)."""
    _require(gates, torch.bfloat16, "gates")
    T, E = gates.shape
    if gates.stride(1) != 1 or T % S:
        raise NativeError("moe_route: gates must be row-major (T, E) with T % S == 0")
    route = torch.empty(T, 4, dtype=torch.int32, device=gates.device) if route is None else route
    _check(load().mp_moe_route(gates.data_ptr(), gates.stride(0), T // S, S, E, C,
                               route.data_ptr(), _stream(stream)), "mp_moe_route")
    return route


def moe_mask(route: torch.Tensor, gates: torch.Tensor, S: int, C: int, mode: int,
             out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """mode 0: dispatch mask (G, E*C, S); mode 1: combine weights (G, S, E*C)."""
    _require(gates, torch.bfloat16, "gates")
    T, E = gates.shape
    G = T // S
    shape = (G, E * C, S) if mode == 0 else (G, S, E * C)
    out = torch.empty(shape, dtype=torch.bfloat16, device=gates.device) if out is None else out
    _contig(out, "out")
    _check(load().mp_moe_mask(route.data_ptr(), gates.data_ptr(), gates.stride(0), out.data_ptr(),
                              T, S, E, C, mode, _stream(stream)), "mp_moe_mask")
    return out


def moe_mask_grad(route: torch.Tensor, d: torch.Tensor, E: int, S: int, C: int, mode: int,
                  out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """(T, E) bf16: d at each token's routed slots (backward of moe_mask)."""
    _require(d, torch.bfloat16, "d")
    _contig(d, "d")
    T = route.shape[0]
    out = torch.empty(T, E, dtype=torch.bfloat16, device=d.device) if out is None else out
    _check(load().mp_moe_mask_grad(route.data_ptr(), d.data_ptr(), out.data_ptr(), T, S, E, C,
                                   mode, _stream(stream)), "mp_moe_mask_grad")
    return out


# --------------------------------------------------------------------------- conv adapters

def _conv_out(H: int, k: int, s: int) -> int:
    return (H + 2 * (k // 2) - k) // s + 1


def im2col(x: torch.Tensor, N: int, H: int, W: int, C: int, k: int, s: int,
           stream=None) -> torch.Tensor:
    """(N*H*W, C) NHWC -> (N*Ho*Wo, k*k*C) patches (csrc/conv.cu)."""
    _require(x, torch.bfloat16, "x")
    _contig(x, "x")
    Ho, Wo = _conv_out(H, k, s), _conv_out(W, k, s)
    out = torch.empty(N * Ho * Wo, k * k * C, dtype=torch.bfloat16, device=x.device)
    _check(load().mp_im2col(x.data_ptr(), out.data_ptr(), N, H, W, C, k, s, 0, _stream(stream)),
           "mp_im2col")
    return out


def col2im(d: torch.Tensor, N: int, H: int, W: int, C: int, k: int, s: int,
           stream=None) -> torch.Tensor:
    _require(d, torch.bfloat16, "d")
    _contig(d, "d")
    out = torch.empty(N * H * W, C, dtype=torch.bfloat16, device=d.device)
    _check(load().mp_im2col(d.data_ptr(), out.data_ptr(), N, H, W, C, k, s, 1, _stream(stream)),
           "mp_im2col")
    return out


def subsample(x: torch.Tensor, N: int, H: int, W: int, C: int, s: int, backward: bool = False,
              stream=None) -> torch.Tensor:
    """forward: (N*H*W, C) -> (N*Ho*Wo, C); backward: (N*Ho*Wo, C) -> (N*H*W, C)."""
    _require(x, torch.bfloat16, "x")
    _contig(x, "x")
    Ho, Wo = _conv_out(H, 1, s), _conv_out(W, 1, s)
    rows = N * H * W if backward else N * Ho * Wo
    out = torch.empty(rows, C, dtype=torch.bfloat16, device=x.device)
    _check(load().mp_subsample(x.data_ptr(), out.data_ptr(), N, H, W, C, s, int(backward),
                               _stream(stream)), "mp_subsample")
    return out


def reduce_mid(x: torch.Tensor, broadcast_b: Optional[int] = None, stream=None) -> torch.Tensor:
    """(A, B, C) -> (A, C) sum over B; with broadcast_b: (A, C) -> (A, B, C)."""
    _require(x, torch.bfloat16, "x")
    _contig(x, "x")
    if broadcast_b is None:
        A, B, C = x.shape
        out = torch.empty(A, C, dtype=torch.bfloat16, device=x.device)
    else:
        (A, C), B = x.shape, broadcast_b
        out = torch.empty(A, B, C, dtype=torch.bfloat16, device=x.device)
    _check(load().mp_reduce_mid(x.data_ptr(), out.data_ptr(), A, B, C,
                                int(broadcast_b is not None), _stream(stream)), "mp_reduce_mid")
    return out


def box_view(t: torch.Tensor, lo, ext) -> Optional[torch.Tensor]:
    """Flat zero-copy view of box [lo, lo+ext) when it is one contiguous run of
    a contiguous tensor (dims before the first partial dim have extent 1, dims
    after it are full); else None.  Lets P2P send/recv skip pack/unpack."""
    if not t.is_contiguous():
        return None
    shape = t.shape
    k = 0
    while k < len(shape) and ext[k] == 1:
        k += 1
    if any(ext[d] != shape[d] for d in range(k + 1, len(shape))):
        return None
    v = t
    for d in range(len(shape)):
        if lo[d] != 0 or ext[d] != shape[d]:
            v = v.narrow(d, lo[d], ext[d])
    return v.view(-1) if v.is_contiguous() else None


def pack_box(src: torch.Tensor, lo, ext, out: Optional[torch.Tensor] = None,
             stream=None) -> torch.Tensor:
    """Dense copy of src[lo:lo+ext] (src any strided view, rank <= 4)."""
    if not src.is_cuda:
        raise NativeError("pack_box: src must be CUDA")
    rank = src.dim()
    n = math.prod(ext)
    out = torch.empty(n, dtype=src.dtype, device=src.device) if out is None else out
    if n == 0:
        return out
    _check(load().mp_pack_box(src.data_ptr(), _arr(src.stride()), _arr(lo), _arr(ext), rank,
                              src.element_size(), out.data_ptr(), _stream(stream)), "mp_pack_box")
    return out


def unpack_box(buf: torch.Tensor, dst: torch.Tensor, lo, ext, stream=None) -> None:
    if not dst.is_cuda:
        raise NativeError("unpack_box: dst must be CUDA")
    if math.prod(ext) == 0:
        return
    _check(load().mp_unpack_box(buf.data_ptr(), dst.data_ptr(), _arr(dst.stride()), _arr(lo),
                                _arr(ext), dst.dim(), dst.element_size(), _stream(stream)),
           "mp_unpack_box")


# --------------------------------------------------------------------------- optimizer / casts

def adam_step(master, m, v, grad, param_bf16, *, lr, beta1, beta2, eps, weight_decay,
              grad_scale, step, stream=None) -> None:
    for t, n in ((master, "master"), (m, "m"), (v, "v"), (grad, "grad")):
        _require(t, torch.float32, n)
    _require(param_bf16, torch.bfloat16, "param")
    _check(load().mp_adam_step(master.data_ptr(), m.data_ptr(), v.data_ptr(), grad.data_ptr(),
                               param_bf16.data_ptr(), master.numel(), lr, beta1, beta2, eps,
                               weight_decay, grad_scale, int(step), _stream(stream)),
           "mp_adam_step")


def cast_f32_bf16(x: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
    _check(load().mp_cast_f32_bf16(x.data_ptr(), out.data_ptr(), x.numel(), _stream(stream)),
           "mp_cast_f32_bf16")
    return out


def cast_bf16_f32(x: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
    _check(load().mp_cast_bf16_f32(x.data_ptr(), out.data_ptr(), x.numel(), _stream(stream)),
           "mp_cast_bf16_f32")
    return out


def accum_bf16_f32(x: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
    _check(load().mp_accum_bf16_f32(x.data_ptr(), out.data_ptr(), x.numel(), _stream(stream)),
           "mp_accum_bf16_f32")
    return out


# --------------------------------------------------------------------------- NCCL

def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return 0
    if t.dtype == torch.float32:
        return 1
    raise NativeError(f"unsupported collective dtype {t.dtype}")


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().mp_nccl_unique_id(buf), "mp_nccl_unique_id")
    return buf.raw


def comm_init(uid: bytes, nranks: int, rank: int) -> int:
    out = c_vp()
    _check(load().mp_comm_init(ctypes.create_string_buffer(uid, 128), nranks, rank,
                               ctypes.byref(out)), "mp_comm_init")
    return out.value


def comm_destroy(comm: int) -> None:
    _check(load().mp_comm_destroy(comm), "mp_comm_destroy")


def comm_abort(comm: int) -> None:
    _check(load().mp_comm_abort(comm), "mp_comm_abort")


def comm_async_error(comm: int) -> int:
    """ncclResult_t of the communicator's asynchronous state (0 ok, 7 in progress)."""
    r = c_int(0)
    _check(load().mp_comm_async_error(comm, ctypes.byref(r)), "mp_comm_async_error")
    return int(r.value)


def allreduce(comm: int, t: torch.Tensor, op: int = 0, stream=None) -> None:
    if not t.is_contiguous():
        raise NativeError("allreduce needs a contiguous tensor")
    _check(load().mp_allreduce(comm, t.data_ptr(), t.numel(), _dt(t), op, _stream(stream)),
           "mp_allreduce")


def allgather(comm: int, out: torch.Tensor, inp: torch.Tensor, stream=None) -> None:
    _check(load().mp_allgather(comm, inp.data_ptr(), out.data_ptr(), inp.numel(), _dt(inp),
                               _stream(stream)), "mp_allgather")


def reduce_scatter(comm: int, out: torch.Tensor, inp: torch.Tensor, stream=None) -> None:
    """Sum-reduce `inp` (nranks * out.numel() elements) across the group; this
    rank receives its chunk in `out`."""
    _check(load().mp_reduce_scatter(comm, inp.data_ptr(), out.data_ptr(), out.numel(), _dt(out),
                                    0, _stream(stream)), "mp_reduce_scatter")


def group_start() -> None:
    _check(load().mp_group_start(), "mp_group_start")


def group_end() -> None:
    _check(load().mp_group_end(), "mp_group_end")


def alltoall(comm: int, out: torch.Tensor, inp: torch.Tensor, nranks: int, stream=None) -> None:
    """Equal-chunk all-to-all over a communicator of `nranks`: chunk i of inp goes to
    rank i, chunk i of out comes from rank i (contiguous tensors, same numel)."""
    if not (inp.is_contiguous() and out.is_contiguous()) or inp.numel() != out.numel() \
            or inp.numel() % nranks or inp.dtype != out.dtype:
        raise NativeError("alltoall needs equal contiguous tensors divisible by the group size")
    _check(load().mp_alltoall(comm, inp.data_ptr(), out.data_ptr(), inp.numel() // nranks,
                              _dt(inp), _stream(stream)), "mp_alltoall")


def send_recv(comm: int, sends, recvs, stream=None) -> None:
    """One NCCL group of sends [(tensor, peer)] and recvs [(tensor, peer)]."""
    lib = load()
    st = _stream(stream)
    _check(lib.mp_group_start(), "mp_group_start")
    try:
        for t, peer in sends:
            _check(lib.mp_send(comm, t.data_ptr(), t.numel(), _dt(t), peer, st), "mp_send")
        for t, peer in recvs:
            _check(lib.mp_recv(comm, t.data_ptr(), t.numel(), _dt(t), peer, st), "mp_recv")
    finally:
        _check(lib.mp_group_end(), "mp_group_end")
