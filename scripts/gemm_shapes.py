"""GEMM time by shape in one executor step (CUDA events around every launch),
plus the step's non-GEMM remainder.  For orientation; ncu is the evidence.

  python scripts/gemm_shapes.py plans/moe24b_n1/plan.json [--mb 4]
"""
import argparse
import json
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("plan")
    ap.add_argument("--mb", type=int, default=4)
    args = ap.parse_args()
    doc = json.loads(Path(args.plan).read_text())
    doc["num_microbatches"] = args.mb
    from paper_2201_12023_b200 import native
    from paper_2201_12023_b200.runtime import Executor
    ex = Executor(doc, schedule="1f1b")
    ex.step()
    ex.step()
    orig = native.gemm
    log = []

    def traced(a, b, out, **kw):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s = kw.get("stream")
        if s is not None:
            e0.record(s)
        else:
            e0.record()
        r = orig(a, b, out, **kw)
        if s is not None:
            e1.record(s)
        else:
            e1.record()
        M, K = a.shape[-2:]
        N = b.shape[-1]
        batch = out.numel() // (out.shape[-2] * out.shape[-1])
        lay = ("T" if a.stride(-1) != 1 else "N") + ("T" if b.stride(-1) != 1 else "N")
        log.append(((batch, M, N, K, lay, str(out.dtype)[6:], kw.get("epilogue", 0)),
                    2.0 * batch * M * N * K, e0, e1))
        return r
    native.gemm = traced
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    ex.runner.run_step(record=False, update=True)
    ev1.record()
    torch.cuda.synchronize()
    native.gemm = orig
    step = ev0.elapsed_time(ev1)
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for key, fl, a, b in log:
        agg[key][0] += 1
        agg[key][1] += a.elapsed_time(b)
        agg[key][2] += fl
    tot = sum(v[1] for v in agg.values())
    print(f"step {step:.2f} ms ({args.mb} microbatches); GEMM launch time sum {tot:.2f} ms "
          f"({100 * tot / step:.1f}%)")
    print(f"{'batch':>5} {'M':>6} {'N':>6} {'K':>6} lay out  epi {'n':>5} {'ms':>8} {'TF/s':>7}")
    for key, (n, ms, fl) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{key[0]:5d} {key[1]:6d} {key[2]:6d} {key[3]:6d} {key[4]:>3} {key[5]:>4} {key[6]:3d} "
              f"{n:5d} {ms:8.2f} {fl / ms / 1e9:7.0f}")


if __name__ == "__main__":
    main()
