"""Per-kernel GPU time of one executor step (torch.profiler / CUPTI), grouped by
kernel name.  For orientation only; ncu launch lists are the committed evidence.

  python scripts/profile_step.py [plan] [--mb N]
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
    ap.add_argument("plan", nargs="?", default=str(ROOT / "plans/gpt13b_n1/plan.json"))
    ap.add_argument("--mb", type=int, default=2, help="microbatches to run (override plan B)")
    ap.add_argument("--rank", type=int, default=0, help="the rank that prints")
    args = ap.parse_args()
    doc = json.loads(Path(args.plan).read_text())
    doc["num_microbatches"] = args.mb
    import os
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        local = int(os.environ["LOCAL_RANK"])
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2201_12023_b200.runtime import Executor
    ex = Executor(doc, schedule="1f1b")
    ex.step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        dt = ex.step()
        torch.cuda.synchronize()
    agg = defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            name = ev.name
            if "gemm_bf16_kernel" in name:
                name = "gemm " + name[name.find("<"):name.find(">") + 1] if "<" in name else name
            agg[name][0] += 1
            agg[name][1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
    if world > 1 and dist.get_rank() != args.rank:
        dist.barrier()
        return
    total = sum(v[1] for v in agg.values())
    print(f"rank {args.rank}: step device time {dt*1e3:.1f} ms, kernel sum {total/1e3:.1f} ms")
    for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
        print(f"{us/1e3:10.2f} ms {100*us/total:6.2f}% {n:7d}  {name[:110]}")
    cpu = defaultdict(lambda: [0, 0.0])
    for ev in prof.key_averages():
        if ev.device_type == torch.autograd.DeviceType.CPU:
            cpu[ev.key] = [ev.count, ev.self_cpu_time_total]
    print("top CPU ops (self time):")
    for name, (n, us) in sorted(cpu.items(), key=lambda kv: -kv[1][1])[:12]:
        print(f"{us/1e3:10.2f} ms {n:7d}  {name[:100]}")
    if world > 1:
        dist.barrier()


if __name__ == "__main__":
    main()
