"""Host cost of one libmpexec GEMM launch (Python wrapper + tensor-map encoding +
launch), measured with a tiny GEMM so the device never limits the loop."""
import json
import time

import torch

from paper_2201_12023_b200 import native


def per_call(fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / n * 1e6


def main():
    a = torch.randn(256, 64, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(64, 256, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(256, 256, device="cuda", dtype=torch.bfloat16)
    c32 = torch.zeros(256, 256, device="cuda")
    aux = torch.randn(256, 256, device="cuda", dtype=torch.bfloat16)
    x = torch.randn(1 << 16, device="cuda", dtype=torch.bfloat16)
    out = {
        "gemm_bf16_us": per_call(lambda: native.gemm(a, b, c)),
        "gemm_f32_acc_us": per_call(lambda: native.gemm(a.t().contiguous().t(), b, c32, beta=1.0)),
        "gemm_epi_add_us": per_call(lambda: native.gemm(a, b, c, epilogue=native.EPI_ADD, aux=aux)),
        "gelu_us": per_call(lambda: native.gelu(x)),
        "torch_empty_us": per_call(lambda: torch.empty(256, 256, device="cuda", dtype=torch.bfloat16)),
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
