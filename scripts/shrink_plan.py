"""Re-dimension a committed plan: keep its stages, meshes and per-node sharding
specs (the planner's decisions) but swap in the same-structure graph built at
small dims by the reference builder, so a plan the planner made for GPT-1.3B
(e.g. key-split attention on (1,2) stages) can be executed against the CPU
oracle in seconds.  Run HERE (needs /root/reference); the output is committed.

  python scripts/shrink_plan.py plans/gpt13b_n4_tp/plan.json plans/tiny_gpt_tp_n4/plan.json \\
      --blocks 24 --batch 2 --seq 256 --hidden 128 --heads 2 --microbatches 4
"""
import argparse
import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("dst")
    ap.add_argument("--reference-src", default="/root/reference/pkg/src")
    ap.add_argument("--blocks", type=int, default=0)
    ap.add_argument("--batch", type=int, required=True)
    ap.add_argument("--seq", type=int, default=0)
    ap.add_argument("--hidden", type=int, default=0)
    ap.add_argument("--heads", type=int, default=0)
    ap.add_argument("--microbatches", type=int, default=None)
    ap.add_argument("--builder", choices=("transformer", "moe", "wresnet"), default="transformer")
    ap.add_argument("--image", type=int, default=32, help="wresnet: image side")
    ap.add_argument("--base", type=int, default=8, help="wresnet: base channels")
    ap.add_argument("--width", type=int, default=1, help="wresnet: width factor")
    ap.add_argument("--classes", type=int, default=16, help="wresnet: classes")
    ap.add_argument("--experts", type=int, default=None, help="moe: experts")
    ap.add_argument("--ffn-mult", type=int, default=8, help="moe: FFN width / hidden")
    a = ap.parse_args()
    sys.path.insert(0, a.reference_src)
    from meshplan import graph as graph_mod
    from meshplan.graph import build_transformer_blocks
    doc = json.loads(Path(a.src).read_text())
    if a.builder == "wresnet":
        sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
        from paper_2201_12023_b200.builders import build_wide_resnet
        g = build_wide_resnet(a.batch, a.image, a.base, a.width, classes=a.classes,
                              elem_bytes=2, backward=True)
    elif a.builder == "moe":
        sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
        from paper_2201_12023_b200.builders import build_moe
        g = build_moe(a.blocks, a.batch, a.seq, a.hidden, a.heads, a.experts,
                      ffn_mult=a.ffn_mult, elem_bytes=2, backward=True)
    else:
        g = build_transformer_blocks(a.blocks, a.batch, a.seq, a.hidden, a.heads, elem_bytes=2,
                                     backward=True)
    new = json.loads(graph_mod.serialize(g))
    old = doc["graph"]
    if len(new["nodes"]) != len(old["nodes"]):
        raise SystemExit(f"structure differs: {len(new['nodes'])} vs {len(old['nodes'])} nodes")
    for n, o in zip(new["nodes"], old["nodes"]):
        keys = [k for k in o if k not in ("shape", "flop")]
        if any(n.get(k) != o.get(k) for k in keys):
            raise SystemExit(f"node {o['id']} differs in structure")
    doc["graph"] = new
    if a.microbatches:
        doc["num_microbatches"] = a.microbatches
    doc["config"] = dict(doc.get("config", {}), shrunk_from=str(a.src),
                         dims=dict(builder=a.builder, blocks=a.blocks, batch=a.batch, seq=a.seq,
                                   hidden=a.hidden, heads=a.heads, experts=a.experts))
    Path(a.dst).parent.mkdir(parents=True, exist_ok=True)
    Path(a.dst).write_text(json.dumps(doc, sort_keys=True))
    print("wrote", a.dst)


if __name__ == "__main__":
    main()
