"""GPU executor vs CPU oracle on the same seeded inputs (used by the gpu tests,
by scripts/parity_run.py under torchrun, and by __graft_entry__.smoke()).

Tolerances (bf16 storage, fp32 accumulation on the GPU; float64 oracle):
  loss                    relative error  <= 2e-2
  forward output          relative Frobenius error <= 3e-2
  parameter gradients     relative Frobenius error <= 5e-2 (each parameter), and
                          <= 1e-2 over all parameters together
  never stricter than      2x the error of the oracle with every node value
                          rounded to bf16 (bf16_storage_errors): deep graphs
                          without normalisation (Wide-ResNet, 50 layers) lose
                          ~2.3% to storage rounding alone
  MoE routing             expert choices equal to the oracle's on every token
                          whose top-3 logit gaps are >= ROUTE_TIE; numerics are
                          compared with the executor's routing replayed
  deep stacks (> 2 blocks): each parameter <= 8e-2 — bf16 rounding compounds
                          through 24 blocks of backward; measured on the
                          24-block single-device plan: max 5.8e-2, global 4.7e-3,
                          and the (1,2) key-split plan of the same graph agrees
                          with it to 1e-4 (profiles/r1_summary.md)
"""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
TOL = {"loss": 2e-2, "output": 3e-2, "grad": 5e-2, "grad_deep": 8e-2, "grad_global": 1e-2}
ROUTE_TIE = 0.05   # logit gap below which bf16 rounding may flip a routing decision


def _blocks(nodes) -> int:
    return max(1, sum(1 for n in nodes if n["kind"] == "batched_matmul") // 6)


def synth(doc: dict, seed: int = 0):
    nodes = doc["graph"]["nodes"]
    rng = np.random.default_rng(seed)
    # deep stacks (no LayerNorm in the IR): damp every weight by 1/sqrt(blocks)
    # past 2 blocks so the float64 reference stays well conditioned
    blocks = _blocks(nodes)
    gain = 1.0 if blocks <= 2 else 1.0 / np.sqrt(blocks)
    # scale by the contraction length (dims[-2]: rows of a 2-D weight, the
    # per-expert fan-in of a 3-D MoE expert weight)
    params = {}
    for n in nodes:
        if n["kind"] == "parameter":
            w = rng.standard_normal(n["shape"]["dims"], dtype=np.float32)
            w *= np.float32(gain / np.sqrt(n["shape"]["dims"][-2]))
            params[n["id"]] = w
    cache = {}

    def inputs(mb, nid):
        if (mb, nid) not in cache:
            r = np.random.default_rng(1000 * (seed + 1) + 7 * mb + nid)
            cache[(mb, nid)] = r.standard_normal(nodes[nid]["shape"]["dims"], dtype=np.float32)
        return cache[(mb, nid)]
    return params, inputs


def gate_nodes(doc) -> list[int]:
    from oracle import ir
    b = ir.bind(doc["graph"]["nodes"])
    return sorted({info[1] for code, info in b.values() if code == "combine_grad"})


def routing_margin(doc, params, inputs) -> float:
    """Smallest logit gap (top-1 vs top-2, top-2 vs top-3) over every token of
    every MoE gate in the oracle run: routing is discrete, so a GPU/oracle
    comparison is meaningful only when bf16 rounding cannot flip a decision."""
    from oracle import dense
    gids = gate_nodes(doc)
    if not gids:
        return float("inf")
    trace = {g: [] for g in gids}
    p16 = {k: bf16_round(v) for k, v in params.items()}
    dense.run(doc, p16, lambda mb, nid: bf16_round(inputs(mb, nid)), doc["num_microbatches"],
              trace=trace)
    m = float("inf")
    for vals in trace.values():
        for g in vals:
            lg = np.sort(np.log(np.maximum(g, 1e-300)), axis=1)[:, ::-1]
            m = min(m, float((lg[:, 0] - lg[:, 1]).min()))
            if lg.shape[1] > 2:
                m = min(m, float((lg[:, 1] - lg[:, 2]).min()))
    return m


def bf16_storage_errors(doc, p16, x16, routes, L, G, O, dtype=np.float64) -> dict:
    """Errors of the float64 oracle with every node's value rounded to bf16 (what
    bf16 activation storage alone costs on this graph), against the plain oracle."""
    from oracle import dense
    orig = dense.eval_node

    def rounded(*a, **k):
        r = orig(*a, **k)
        return bf16_round(r).astype(dtype) if isinstance(r, np.ndarray) else r
    dense.eval_node = rounded
    try:
        L2, G2, O2 = dense.run(doc, p16, x16, doc["num_microbatches"], routes=routes, dtype=dtype)
    finally:
        dense.eval_node = orig
    out = {"loss": abs(L2 - L) / abs(L), "grad": max((rel(G2[k], G[k]) for k in G), default=0.0),
           "output": max((rel(O2[m], O[m]) for m in O), default=0.0)}
    num = sum(float(np.sum((G2[k] - G[k]) ** 2)) for k in G)
    den = sum(float(np.sum(G[k] ** 2)) for k in G)
    out["grad_global"] = float(np.sqrt(num / max(den, 1e-300))) if G else 0.0
    return out


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def bf16_round(x):
    """Round fp32 values to bf16 (what the GPU sees of the same inputs)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    r = (u >> 16) & np.uint32(1)
    r += np.uint32(0x7FFF)
    r += u                      # wraps only for NaN payloads
    r &= np.uint32(0xFFFF0000)
    return r.view(np.float32)


def compare(doc, result, params, inputs, dtype=np.float64):
    """Oracle (dense float64 on bf16-rounded inputs) vs the executor result.
    dtype=np.float32 for the full-size plans (fp32 accumulation error ~1e-6,
    three orders below the bf16 tolerances; half the oracle's time and memory)."""
    from oracle import dense
    p16 = {k: bf16_round(v) for k, v in params.items()}
    x16 = lambda mb, nid: bf16_round(inputs(mb, nid))  # noqa: E731
    routes = getattr(result, "routes", None) or None
    route_errs = {}
    if routes:
        # MoE: routing is discrete.  The GPU's expert choices must equal the
        # oracle's on every token whose top-3 logit gaps exceed ROUTE_TIE; the
        # numerics are then compared with the GPU's decisions replayed.
        trace = {g: [] for g in gate_nodes(doc)}
        dense.run(doc, p16, x16, doc["num_microbatches"], trace=trace, dtype=dtype)
        mism = ties = 0
        for (mb, gid), tab in routes.items():
            lg = np.log(np.maximum(trace[gid][mb], 1e-300))
            order = np.argsort(-lg, axis=1, kind="stable")
            top = np.take_along_axis(lg, order, axis=1)
            gap = np.minimum(top[:, 0] - top[:, 1], top[:, 1] - top[:, 2]) \
                if lg.shape[1] > 2 else top[:, 0] - top[:, 1]
            clear = gap >= ROUTE_TIE
            ties += int((~clear).sum())
            mism += int(((order[:, 0] != tab[:, 0]) | (order[:, 1] != tab[:, 2]))[clear].sum())
        route_errs = {"route_mismatch": mism, "route_near_ties": ties}
    L, G, O = dense.run(doc, p16, x16, doc["num_microbatches"], routes=routes, dtype=dtype)
    errs = {"loss": abs(result.loss - L) / abs(L), "oracle_loss": L, "gpu_loss": result.loss}
    errs.update(route_errs)
    emu = bf16_storage_errors(doc, p16, x16, routes, L, G, O, dtype)
    errs["bf16_storage"] = emu
    per = {k: rel(result.grads[k], G[k]) for k in G}
    errs["grad"] = max(per.values()) if per else 0.0
    errs["grad_worst"] = sorted(per.items(), key=lambda kv: -kv[1])[:4]
    if G:
        num = sum(float(np.sum((np.asarray(result.grads[k], np.float64) - G[k]) ** 2)) for k in G)
        den = sum(float(np.sum(np.asarray(G[k], np.float64) ** 2)) for k in G)
        errs["grad_global"] = float(np.sqrt(num / max(den, 1e-300)))
    outs = [rel(result.outputs[(mb, y)], O[mb]) for (mb, y) in result.outputs] if result.outputs else [0.0]
    errs["output"] = max(outs)
    tol_grad = TOL["grad"] if _blocks(doc["graph"]["nodes"]) <= 2 else TOL["grad_deep"]
    # never stricter than twice the error of merely storing every node in bf16
    tol_grad = max(tol_grad, 2 * emu["grad"])
    tol_glob = max(TOL["grad_global"], 2 * emu["grad_global"])
    tol_out = max(TOL["output"], 2 * emu["output"])
    tol_loss = max(TOL["loss"], 2 * emu["loss"])
    errs["tol"] = {"loss": tol_loss, "grad": tol_grad, "grad_global": tol_glob, "output": tol_out}
    errs["ok"] = errs["loss"] <= tol_loss and errs["grad"] <= tol_grad and \
        errs.get("grad_global", 0.0) <= tol_glob and errs["output"] <= tol_out \
        and errs.get("route_mismatch", 0) == 0
    return errs


def run_plan(plan_path, schedule="1f1b", seed=0, dtype=np.float64):
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
    errs = compare(doc, res, params, inputs, dtype=dtype)
    errs["gpu_launches"] = res.gpu_launches
    errs["makespan_s"] = res.makespan
    errs["fused"] = res.fused
    return errs


TRAIN_LR = 1e-3     # large enough that three Adam steps move the loss visibly


def train_losses(plan_path, schedule="1f1b", steps=3, seed=0, oracle=True, lr=TRAIN_LR):
    """`steps` training steps (Adam updates between them) on this process group.
    Rank 0 returns {"losses": executor losses, "oracle": the oracle's
    (oracle/adam.py: same update rule, fp32 master, bf16 working weights),
    "err": max relative loss error, "zero_params": parameters under the ZeRO
    rewrite on rank 0}; other ranks None."""
    import torch.distributed as dist
    from paper_2201_12023_b200.runtime import AdamConfig, Executor
    doc = json.loads(Path(plan_path).read_text())
    params, inputs = synth(doc, seed)
    ex = Executor(doc, schedule=schedule, params=params, inputs=inputs, seed=seed,
                  adam=AdamConfig(lr=lr))
    out = []
    for _ in range(steps):
        ex.barrier()
        ex.step()
        out.append(ex.loss())
    rank = dist.get_rank() if dist.is_initialized() else 0
    if rank != 0:
        return None
    res = {"losses": out, "zero_params": len(ex.runner.zero)}
    if oracle:
        from oracle import adam
        a = AdamConfig(lr=lr)
        ref, _ = adam.train(doc, params, inputs, steps, lr=a.lr, beta1=a.beta1, beta2=a.beta2,
                            eps=a.eps, weight_decay=a.weight_decay)
        res["oracle"] = ref
        res["err"] = max(abs(x - y) / abs(y) for x, y in zip(out, ref))
    return res
