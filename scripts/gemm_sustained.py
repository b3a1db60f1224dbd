"""Sustained (power-capped steady state) throughput of the tcgen05 GEMM against
cuBLAS (torch.matmul) on every GEMM shape of the GPT-1.3B step: each shape runs
back to back for ~2 s per implementation, CUDA-event timed over the last second,
SM clock sampled by NVML.  Tells whether a shape's in-step time is at the
library's level under the same power cap.

  python scripts/gemm_sustained.py [--secs 2]
"""
import argparse
import json
import threading
import time

import torch

from paper_2201_12023_b200 import native

# name, M, N, K, a transposed (K-major in memory as (K, M)), b transposed, fp32 += out
SHAPES = [
    ("qkv/out fwd", 8192, 2048, 2048, 0, 0, 0),
    ("mlp_up fwd", 8192, 8192, 2048, 0, 0, 0),
    ("mlp_down fwd", 8192, 2048, 8192, 0, 0, 0),
    ("dX 2048^2", 8192, 2048, 2048, 0, 1, 0),
    ("dX mlp_down", 8192, 8192, 2048, 0, 1, 0),
    ("dX mlp_up", 8192, 2048, 8192, 0, 1, 0),
    ("dW 2048^2", 2048, 2048, 8192, 1, 0, 1),
    ("dW mlp_down", 8192, 2048, 8192, 1, 0, 1),
    ("dW mlp_up", 2048, 8192, 8192, 1, 0, 1),
]


def clock_sampler(stop, out):
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    while not stop.is_set():
        out.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        time.sleep(0.05)


def sustained(fn, secs):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < secs / 2:          # heat up to the power cap
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        n += 10
    clocks, stop = [], threading.Event()
    th = threading.Thread(target=clock_sampler, args=(stop, clocks))
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = max(10, n)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    clocks.sort()
    return e0.elapsed_time(e1) * 1e-3 / iters, clocks[len(clocks) // 2] if clocks else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--secs", type=float, default=2.0)
    a = ap.parse_args()
    for name, M, N, K, ta, tb, acc in SHAPES:
        A = torch.randn(K, M, device="cuda", dtype=torch.bfloat16).t() if ta else \
            torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16).t() if tb else \
            torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
        fl = 2.0 * M * N * K
        if acc:
            C = torch.zeros(M, N, device="cuda", dtype=torch.float32)
            mine = lambda: native.gemm(A, B, C, beta=1.0)                     # noqa: E731
            # cuBLAS has no bf16 x bf16 -> fp32 += here: its bf16-out GEMM of the shape
            Cb16 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            lib = lambda: torch.matmul(A, B, out=Cb16)                       # noqa: E731
        else:
            C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            mine = lambda: native.gemm(A, B, C)                               # noqa: E731
            Cb16 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            lib = lambda: torch.matmul(A, B, out=Cb16)                       # noqa: E731
        tm, cm = sustained(mine, a.secs)
        tl, cl = sustained(lib, a.secs)
        print(json.dumps({"shape": name, "M": M, "N": N, "K": K, "fp32_acc": bool(acc),
                          "mine_tflops": fl / tm / 1e12, "mine_sm_mhz": cm,
                          "mine_flop_per_clk_sm": fl / tm / (cm * 1e6) / 148 if cm else None,
                          "cublas_bf16_tflops": fl / tl / 1e12, "cublas_sm_mhz": cl,
                          "cublas_flop_per_clk_sm": fl / tl / (cl * 1e6) / 148 if cl else None}),
              flush=True)


if __name__ == "__main__":
    main()
