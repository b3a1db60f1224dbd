"""`execute` — the executor's twin of the reference's `meshplan simulate`
(cli.py:176-200, parser cli.py:296-303, exit codes cli.py:322-342).

    python -m paper_2201_12023_b200 execute --plan plans/gpt13b_n1/plan.json \\
        --schedule 1f1b --steps 3 --out run/
    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \\
        -m paper_2201_12023_b200 execute --plan plans/gpt13b_n4/plan.json --out run/

Runs the plan on this box's GPUs (one process per device, rank = device id),
writes the reference's `sim.json` (ExecResult.trace_json: measured makespan,
utilization, peak bytes, events) and `gantt.json` (gantt_rows) on rank 0, and
prints the planned T*, the measured makespan and the reference simulator's
modeled makespan for the same program.  Exit codes as the reference: 0 ok,
1 usage / plan errors, 2 execution failure (out of memory, deadlock: the
SimError cases; also NCCL / kernel failures).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

SCHEDULES = ("gpipe", "1f1b")


class UsageError(Exception):
    pass


def _load_doc(path: str) -> dict:
    p = Path(path)
    if p.suffix == ".toml":
        import tomllib
        return tomllib.loads(p.read_text())
    return json.loads(p.read_text())


def cmd_execute(args) -> int:
    import torch
    import torch.distributed as dist

    from . import runtime, schedule as sched
    from .plan import load_plan

    doc = json.loads(Path(args.plan).read_text())
    plan = load_plan(doc)
    if args.cluster:
        given = _load_doc(args.cluster)
        given = given.get("cluster", given)
        if json.dumps(given, sort_keys=True) != json.dumps(doc["cluster"], sort_keys=True):
            raise UsageError("--cluster does not match the cluster embedded in the plan")
    if args.steps < 1:
        raise UsageError("--steps must be >= 1")
    schedule = args.schedule or doc.get("config", {}).get("schedule", "gpipe")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != plan.num_devices:
        raise UsageError(f"plan needs {plan.num_devices} devices (one process each); "
                         f"running on {world}")
    if world > 1 and not dist.is_initialized():
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank = dist.get_rank() if dist.is_initialized() else 0
    program = sched.build_program(plan, schedule)
    res = runtime.execute(plan, program, steps=args.steps, seed=args.seed,
                          device_memory=args.device_memory, timeout=args.timeout)
    if rank == 0:
        out = Path(args.out)
        out.mkdir(parents=True, exist_ok=True)
        (out / "sim.json").write_text(res.trace_json() + "\n")
        (out / "gantt.json").write_text(
            json.dumps(res.gantt_rows(program), sort_keys=True, indent=2) + "\n")
        modeled = sched.modeled_makespan(program, plan, zero_transfer=args.transfer == "zero")
        sys.stdout.write(
            f"schedule={schedule} transfer={args.transfer} steps={args.steps} "
            f"devices={world}\n"
            f"T* (planned)       = {float(program.t_star):.6e} s\n"
            f"makespan (sim)     = {float(modeled):.6e} s\n"
            f"makespan (B200)    = {res.makespan:.6e} s\n"
            f"difference         = {res.makespan - float(program.t_star):.6e} s\n"
            f"loss               = {res.loss:.6e}\n")
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2201_12023_b200",
                                 description="B200 executor for reference (Alpa) plans")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("execute", help="execute a plan file on this box's GPUs")
    p.add_argument("--plan", required=True, help="plan.json path")
    p.add_argument("--cluster", help="must match the embedded cluster")
    p.add_argument("--schedule", choices=SCHEDULES)
    p.add_argument("--transfer", choices=("model", "zero"), default="model",
                   help="transfer mode of the modeled makespan printed beside the measured one")
    p.add_argument("--steps", type=int, default=1, help="training steps (the last is reported)")
    p.add_argument("--seed", type=int, default=0, help="synthetic weights / inputs seed")
    p.add_argument("--device-memory", type=int, default=None,
                   help="per-device byte cap (exceeding it is an out-of-memory failure)")
    p.add_argument("--timeout", type=float, default=None,
                   help="seconds before an unfinished step is reported as a deadlock")
    p.add_argument("--out", default=".", help="output directory")
    p.set_defaults(func=cmd_execute)
    return ap


def main(argv=None) -> int:
    from .plan import PlanError
    from .runtime import ExecError
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except ExecError as e:
        sys.stderr.write(f"execution failed: {e}\n")
        return 2
    except (UsageError, PlanError, OSError, json.JSONDecodeError) as e:
        sys.stderr.write(f"error: {e}\n")
        return 1


if __name__ == "__main__":
    sys.exit(main())
