"""GPU executor vs CPU oracle on the same seeded inputs (used by the gpu tests,
by scripts/parity_run.py under torchrun, and by __graft_entry__.smoke()).

Tolerances (bf16 storage, fp32 accumulation on the GPU; float64 oracle):
  loss                    relative error  <= 2e-2
  forward output          relative Frobenius error <= 3e-2
  parameter gradients     relative Frobenius error <= 5e-2 (each parameter)
"""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
TOL = {"loss": 2e-2, "output": 3e-2, "grad": 5e-2}


def synth(doc: dict, seed: int = 0):
    nodes = doc["graph"]["nodes"]
    rng = np.random.default_rng(seed)
    params = {n["id"]: (rng.standard_normal(n["shape"]["dims"]) / np.sqrt(n["shape"]["dims"][0]))
              .astype(np.float32) for n in nodes if n["kind"] == "parameter"}
    cache = {}

    def inputs(mb, nid):
        if (mb, nid) not in cache:
            r = np.random.default_rng(1000 * (seed + 1) + 7 * mb + nid)
            cache[(mb, nid)] = r.standard_normal(nodes[nid]["shape"]["dims"]).astype(np.float32)
        return cache[(mb, nid)]
    return params, inputs


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def bf16_round(x):
    """Round fp32 values to bf16 (what the GPU sees of the same inputs)."""
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def compare(doc, result, params, inputs):
    """Oracle (dense float64 on bf16-rounded inputs) vs the executor result."""
    from oracle import dense
    p16 = {k: bf16_round(v) for k, v in params.items()}
    L, G, O = dense.run(doc, p16, lambda mb, nid: bf16_round(inputs(mb, nid)),
                        doc["num_microbatches"])
    errs = {"loss": abs(result.loss - L) / abs(L), "oracle_loss": L, "gpu_loss": result.loss}
    errs["grad"] = max(rel(result.grads[k], G[k]) for k in G) if G else 0.0
    outs = [rel(result.outputs[(mb, y)], O[mb]) for (mb, y) in result.outputs] if result.outputs else [0.0]
    errs["output"] = max(outs)
    errs["ok"] = errs["loss"] <= TOL["loss"] and errs["grad"] <= TOL["grad"] and \
        errs["output"] <= TOL["output"]
    return errs


def run_plan(plan_path, schedule="1f1b", seed=0):
    """Execute one step (collect grads, no update) on this process group and
    compare on rank 0.  Returns the error dict (rank 0) or None."""
    import torch.distributed as dist
    from paper_2201_12023_b200.runtime import execute
    doc = json.loads(Path(plan_path).read_text())
    params, inputs = synth(doc, seed)
    res = execute(doc, schedule=schedule, steps=1, params=params, inputs=inputs, collect=True,
                  update=False, seed=seed)
    rank = dist.get_rank() if dist.is_initialized() else 0
    if rank != 0:
        return None
    errs = compare(doc, res, params, inputs)
    errs["gpu_launches"] = res.gpu_launches
    errs["makespan_s"] = res.makespan
    return errs
