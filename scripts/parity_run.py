"""torchrun entry: execute a plan on N GPUs and compare with the CPU oracle.

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
      scripts/parity_run.py plans/tiny_gpt_n2/plan.json [--schedule 1f1b]
Rank 0 prints one JSON line with the errors and exits non-zero on a miss."""
import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("plan")
    ap.add_argument("--schedule", default="1f1b")
    ap.add_argument("--train-steps", type=int, default=0,
                    help="instead of the oracle check: run N steps with Adam updates and "
                         "print the per-step losses (used to compare optimizer paths)")
    ap.add_argument("--no-oracle", action="store_true",
                    help="with --train-steps: skip the oracle's training run")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.train_steps:
        from parity_harness import train_losses
        res = train_losses(args.plan, args.schedule, args.train_steps,
                           oracle=not args.no_oracle)
        if res is not None:
            res["plan"] = args.plan
            print(json.dumps(res), flush=True)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    from parity_harness import run_plan
    errs = run_plan(args.plan, args.schedule)
    rc = 0
    if errs is not None:
        errs["plan"] = args.plan
        errs["schedule"] = args.schedule
        errs["world"] = world
        print(json.dumps(errs), flush=True)
        rc = 0 if errs["ok"] else 1
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    sys.exit(rc)


if __name__ == "__main__":
    main()
