"""Per-op and per-relayout device time of one executor step (MPEXEC_OP_TIMING=1:
CUDA events around every op and every relayout on the compute stream).
Under torchrun every rank prints its own table (rank, stage).

  python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \\
      scripts/op_breakdown.py plans/gpt13b_n4_tp/plan.json --mb 8
"""
import argparse
import json
import os
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ["MPEXEC_OP_TIMING"] = "1"

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("plan")
    ap.add_argument("--mb", type=int, default=8)
    ap.add_argument("--ranks", default="0", help="comma list of ranks that print")
    a = ap.parse_args()
    doc = json.loads(Path(a.plan).read_text())
    doc["num_microbatches"] = a.mb
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        local = int(os.environ["LOCAL_RANK"])
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2201_12023_b200.runtime import Executor
    ex = Executor(doc, schedule="1f1b")
    ex.step()
    r = ex.runner
    r.op_timer.clear()
    r.relayout_timer.clear()
    ex.barrier()
    dt = ex.step()
    rank = dist.get_rank() if world > 1 else 0
    ops = defaultdict(lambda: [0, 0.0, 0.0])
    rel = defaultdict(lambda: [0, 0.0, 0])
    for phase, name, e0, e1, rl in r.op_timer:
        t = e0.elapsed_time(e1)
        inner = sum(b.elapsed_time(c) for _, _, b, c in rl)
        k = ops[(phase, name)]
        k[0] += 1
        k[1] += t
        k[2] += inner
    for kind, nbytes, e0, e1 in r.relayout_timer:
        k = rel[kind]
        k[0] += 1
        k[1] += e0.elapsed_time(e1)
        k[2] += nbytes
    if str(rank) in a.ranks.split(","):
        tot = sum(v[1] for v in ops.values())
        lines = [f"rank {rank} stage {r.st.index} mesh {r.mesh}: step {dt * 1e3:.1f} ms, "
                 f"ops {tot:.1f} ms over {a.mb} microbatches"]
        for (ph, name), (n, t, inner) in sorted(ops.items(), key=lambda kv: -kv[1][1])[:16]:
            lines.append(f"  {ph} {name:14s} {n:5d} {t:9.2f} ms (relayout inside {inner:7.2f} ms)")
        for kind, (n, t, nb) in sorted(rel.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"  relayout {kind:13s} {n:5d} {t:9.2f} ms  {nb / 2**30:6.2f} GiB global "
                         f"({nb / max(t, 1e-9) / 1e6:6.1f} GB/s of global tensor)")
        print("\n".join(lines), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
