"""The executor's drop-in contract on the GPU: a plan run through
the `execute` CLI writes the reference's sim.json / gantt.json documents, and
the simulator's failure modes map to ExecError naming device, stage and
instruction (sim.py:152-160 out of memory, sim.py:172-178 deadlock)."""
import json
import os
import subprocess
import sys
import textwrap
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
ENV = {**os.environ, "PYTHONPATH": str(ROOT)}


def test_cli_execute_writes_sim_documents(tmp_path):
    r = subprocess.run([sys.executable, "-m", "paper_2201_12023_b200", "execute", "--plan",
                        "plans/tiny_gpt_n1/plan.json", "--schedule", "1f1b", "--steps", "2",
                        "--out", str(tmp_path)], capture_output=True, text=True, cwd=ROOT,
                       env=ENV, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "makespan (B200)" in r.stdout and "T* (planned)" in r.stdout
    doc = json.loads((tmp_path / "sim.json").read_text())
    assert {"makespan", "makespan_seconds", "utilization", "peak_bytes", "events"} <= set(doc)
    assert doc["makespan_seconds"] > 0 and 0 < doc["utilization"]["0"] <= 1.0
    assert doc["peak_bytes"]["0"] > 0
    from paper_2201_12023_b200.plan import load_plan
    from paper_2201_12023_b200.runtime import _label
    from paper_2201_12023_b200.schedule import build_program
    prog = build_program(load_plan(ROOT / "plans/tiny_gpt_n1/plan.json"), "1f1b")
    mine = sorted((e["op"], e["label"]) for e in doc["events"])
    assert mine == sorted((i.op, _label(i)) for i in prog.stages[0].instructions)
    assert all(e["end"] >= e["start"] >= 0 for e in doc["events"])
    gantt = json.loads((tmp_path / "gantt.json").read_text())
    assert set(gantt) == {"0"} and gantt["0"]


def test_out_of_memory_names_the_instruction():
    """A byte cap between the resident state and the step's needs: the first
    allocation past it raises ExecError(kind="oom") naming device, stage and
    instruction, in the reference's message shape."""
    code = textwrap.dedent("""
        import json, torch
        from paper_2201_12023_b200.runtime import Executor, ExecError
        torch.cuda.set_device(0)
        ex = Executor("plans/gpt13b_block1_n1/plan.json", schedule="1f1b")
        torch.cuda.synchronize(); torch.cuda.empty_cache()
        cap = torch.cuda.memory_reserved() + (64 << 20)
        total = torch.cuda.get_device_properties(0).total_memory
        torch.cuda.set_per_process_memory_fraction(cap / total)
        try:
            ex.step()
            print(json.dumps({"ok": True}))
        except ExecError as e:
            print(json.dumps({"kind": e.kind, "rank": e.rank, "stage": e.stage,
                              "instruction": e.instruction, "msg": str(e)}))
    """)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT,
                       env=ENV, timeout=600)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert lines, r.stdout + r.stderr
    res = json.loads(lines[-1])
    assert res.get("kind") == "oom", res
    assert res["rank"] == 0 and res["stage"] == 0 and res["instruction"], res
    assert res["msg"].startswith("out of memory on device 0 (stage 0) at "), res


def test_cli_device_memory_cap_exit_code(tmp_path):
    r = subprocess.run([sys.executable, "-m", "paper_2201_12023_b200", "execute", "--plan",
                        "plans/gpt13b_block1_n1/plan.json", "--device-memory", str(1 << 20),
                        "--out", str(tmp_path)], capture_output=True, text=True, cwd=ROOT,
                       env=ENV, timeout=600)
    assert r.returncode == 2, r.stdout + r.stderr
    assert "execution failed: out of memory on device 0 (stage 0)" in r.stderr, r.stderr


def test_deadlock_names_the_blocked_instruction():
    """Two stages; stage 0 drops its forward sends.  Stage 1's watchdog fires on
    its first recv (tag f:0>1:0), aborts the communicators and raises
    ExecError(kind="deadlock") naming it (sim.py:172-178's message shape)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    code = textwrap.dedent("""
        import faulthandler, json, os, sys, torch, torch.distributed as dist
        faulthandler.dump_traceback_later(90, exit=True, file=sys.stderr)
        from paper_2201_12023_b200 import runtime
        from paper_2201_12023_b200.runtime import Executor, ExecError
        r = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(r)
        dist.init_process_group("nccl", device_id=torch.device("cuda", r))
        ex = Executor("plans/tiny_gpt_n2/plan.json", schedule="1f1b")
        if r == 0:
            ex.runner.send = lambda ins: None
        ex.barrier(); torch.cuda.synchronize()
        try:
            ex.step(timeout=20)
            out = {"rank": r, "ok": True}
        except ExecError as e:
            out = {"rank": r, "kind": e.kind, "instruction": e.instruction, "msg": str(e)}
        print(json.dumps(out), flush=True)
        os._exit(0)
    """)
    script = ROOT / "gpurun_out" / "_deadlock_probe.py"
    script.parent.mkdir(exist_ok=True)
    script.write_text(code)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr", "127.0.0.1", "--master-port",
                        "29517", str(script)], capture_output=True, text=True, cwd=ROOT,
                       env=ENV, timeout=300)
    outs = {d["rank"]: d for d in (json.loads(l) for l in r.stdout.splitlines()
                                   if l.startswith("{"))}
    assert 1 in outs, r.stdout + r.stderr
    assert outs[1].get("kind") == "deadlock", outs
    assert outs[1]["instruction"] == "f:0>1:0", outs
    assert outs[1]["msg"].startswith("deadlock: rank 1 stage 1 waiting on recv f:0>1:0"), outs


def test_cli_execute_two_stages(tmp_path):
    """The CLI twin under torchrun on a 2-stage plan: rank 0 writes one sim.json with
    both stages' utilization, both devices' peaks and every instruction of both
    stages, and gantt rows for both devices."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr", "127.0.0.1", "--master-port",
                        "29541", "-m", "paper_2201_12023_b200", "execute", "--plan",
                        "plans/tiny_gpt_n2/plan.json", "--schedule", "1f1b", "--steps", "2",
                        "--out", str(tmp_path)], capture_output=True, text=True, cwd=ROOT,
                       env=ENV, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    doc = json.loads((tmp_path / "sim.json").read_text())
    assert set(doc["utilization"]) == {"0", "1"} and set(doc["peak_bytes"]) == {"0", "1"}
    from paper_2201_12023_b200.plan import load_plan
    from paper_2201_12023_b200.runtime import _label
    from paper_2201_12023_b200.schedule import build_program
    prog = build_program(load_plan(ROOT / "plans/tiny_gpt_n2/plan.json"), "1f1b")
    want = sorted((sp.stage, i.op, _label(i)) for sp in prog.stages for i in sp.instructions)
    assert sorted((e["stage"], e["op"], e["label"]) for e in doc["events"]) == want
    gantt = json.loads((tmp_path / "gantt.json").read_text())
    assert set(gantt) == {"0", "1"} and gantt["0"] and gantt["1"]
