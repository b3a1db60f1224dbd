"""Config 5 (BASELINE.json configs[4]): cross-mesh resharding sweep.

2-D bf16 tensors (rows, 8192), 1 MiB .. 1 GiB, between disjoint submeshes of the
(1,N) box: every (src, dst) pair in {(1,1),(1,2),(1,4)}^2 that fits on the GPUs
of this run, every spec pair of `enumerate_specs` style (all legal specs), with
the reference's optimize=True (send/recv of distinct tiles + local all-gather on
the destination replica group, reshard.py:133-156) vs optimize=False (every
destination device receives its whole tile over the inter-mesh link,
reshard.py:128-131).  Index plans come from xmesh.cross_mesh_plan (bit-exact with
the reference, tests/test_plan_parity.py); the data path is the executor's:
mp_pack_box -> NCCL P2P -> mp_unpack_box (+ NCCL all-gather).

Reported per case: time (max over ranks, CUDA events), algorithmic bytes =
inter_mesh_bytes + sum over gathers of (g-1)/g * nbytes per device,
and bus GB/s = max over devices of (egress or ingress bytes) / time, against
900 GB/s/dir nominal (770 measured peer copy).

  python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
      scripts/xmesh_sweep.py [--sizes-mib 1,2,4,...,1024] [--out gpurun_out/xmesh.jsonl]

bench.py runs the same sweep (every size, every pair that fits) after its 8-GPU
measurement and adds the per-pair best bus GB/s to its JSON line (`xmesh`).
"""
import argparse
import itertools
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2201_12023_b200 import native  # noqa: E402
from paper_2201_12023_b200.plan import Mesh, Spec, device_box, format_spec, local_dims  # noqa: E402
from paper_2201_12023_b200.xmesh import cross_mesh_plan  # noqa: E402


def specs_2d(mesh: Mesh, dims):
    out = []
    axes = [a for a in (0, 1) if mesh.extent(a) > 1]
    for assign in itertools.product([None, 0, 1], repeat=len(axes)):
        d = [[], []]
        for a, k in zip(axes, assign):
            if k is not None:
                d[k].append(a)
        sp = Spec(tuple(tuple(x) for x in d))
        if all(e % mesh.group_extent(ax) == 0 for e, ax in zip(dims, sp.dims)) and sp not in out:
            out.append(sp)
    return out


def run_case(rank, dims, sspec, smesh, dspec, dmesh, optimize, groups, iters=5):
    """-> (seconds per reshard, max over ranks; inter-mesh bytes; algorithmic bytes;
    busiest device's egress-or-ingress bytes)."""
    xp = cross_mesh_plan(dims, 2, sspec, smesh, dspec, dmesh, optimize)
    dev = torch.device("cuda", torch.cuda.current_device())
    src_local = dst_local = None
    if rank in smesh.device_ids:
        src_local = torch.randn(local_dims(dims, sspec, smesh), device=dev).to(torch.bfloat16)
    if rank in dmesh.device_ids:
        dst_local = torch.empty(local_dims(dims, dspec, dmesh), device=dev, dtype=torch.bfloat16)
    world_pg = groups["world"]

    def once():
        sends, recvs = [], []
        if src_local is not None:
            org = [lo for lo, _ in device_box(dims, sspec, smesh, rank)]
            for t in xp.transfers:
                if t.src_device == rank:
                    lo = [a - o for (a, _), o in zip(t.box, org)]
                    ext = [b - a for a, b in t.box]
                    view = native.box_view(src_local, lo, ext)
                    buf = view if view is not None else native.pack_box(src_local, lo, ext)
                    sends.append(dist.P2POp(dist.isend, buf, t.dst_device, group=groups["pair"]))
        if dst_local is not None:
            org = [lo for lo, _ in device_box(dims, dspec, dmesh, rank)]
            for t in xp.transfers:
                if t.dst_device == rank:
                    n = 1
                    for a, b in t.box:
                        n *= b - a
                    lo = [a - o for (a, _), o in zip(t.box, org)]
                    view = native.box_view(dst_local, lo, [b - a for a, b in t.box])
                    buf = view if view is not None else torch.empty(n, device=dev, dtype=torch.bfloat16)
                    recvs.append((buf, t, view is None))
                    sends.append(dist.P2POp(dist.irecv, buf, t.src_device, group=groups["pair"]))
        if sends:
            for w in dist.batch_isend_irecv(sends):
                w.wait()
        if dst_local is not None:
            org = [lo for lo, _ in device_box(dims, dspec, dmesh, rank)]
            for buf, t, packed in recvs:
                if packed:
                    native.unpack_box(buf, dst_local, [a - o for (a, _), o in zip(t.box, org)],
                                      [b - a for a, b in t.box])
            for g in xp.gathers:
                if rank not in g.devices:
                    continue
                rows = [p[0][1] - p[0][0] for p in g.pieces]
                r = g.devices.index(rank)
                flat = dst_local.view(-1)
                row_elems = dst_local.numel() // dst_local.shape[0]
                grp = groups[("gather", g.devices)]
                if all(x == rows[0] for x in rows):
                    n = rows[0] * row_elems
                    dist.all_gather_into_tensor(flat, flat[r * n:(r + 1) * n], group=grp)
                else:
                    starts = [p[0][0] - g.box[0][0] for p in g.pieces]
                    ops = []
                    mine = flat[starts[r] * row_elems:(starts[r] + rows[r]) * row_elems]
                    for q, d in enumerate(g.devices):
                        if q == r:
                            continue
                        if rows[r]:
                            ops.append(dist.P2POp(dist.isend, mine, d, group=grp))
                        if rows[q]:
                            ops.append(dist.P2POp(dist.irecv, flat[starts[q] * row_elems:(starts[q] + rows[q]) * row_elems], d, group=grp))
                    for w in dist.batch_isend_irecv(ops):
                        w.wait()

    for _ in range(2):
        once()
    torch.cuda.synchronize()
    dist.barrier(group=world_pg)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        once()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters * 1e-3], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=world_pg)
    # per-device egress / ingress bytes
    eg, ing = {}, {}
    for tr in xp.transfers:
        eg[tr.src_device] = eg.get(tr.src_device, 0) + tr.nbytes
        ing[tr.dst_device] = ing.get(tr.dst_device, 0) + tr.nbytes
    for g in xp.gathers:
        share = g.nbytes * (len(g.devices) - 1) // len(g.devices)
        for d in g.devices:
            ing[d] = ing.get(d, 0) + share
            eg[d] = eg.get(d, 0) + share // max(len(g.devices) - 1, 1) * (len(g.devices) - 1)
    algo = xp.inter_mesh_bytes + sum(g.nbytes * (len(g.devices) - 1) // len(g.devices) * len(g.devices)
                                     for g in xp.gathers)
    peak_dev = max(list(eg.values()) + list(ing.values()) + [1])
    return float(t.item()), xp.inter_mesh_bytes, algo, peak_dev


SIZES_MIB = [1 << i for i in range(11)]            # 1 MiB .. 1 GiB


def make_groups(world):
    shapes = [(1, 1), (1, 2), (1, 4)]
    pairs = [(s, d) for s in shapes for d in shapes if s[1] + d[1] <= world]
    groups = {"world": dist.new_group(list(range(world))), "pair": dist.new_group(list(range(world)))}
    for s, d in pairs:
        dm = Mesh(1, d[1], tuple(range(s[1], s[1] + d[1])))
        # every gather group a replica spec can form inside dst
        for k in (2, 4):
            if k <= d[1]:
                for start in range(0, d[1], k):
                    devs = tuple(range(s[1] + start, s[1] + start + k))
                    if ("gather", devs) not in groups:
                        groups[("gather", devs)] = dist.new_group(list(devs))
        devs = tuple(dm.device_ids)
        if len(devs) > 1 and ("gather", devs) not in groups:
            groups[("gather", devs)] = dist.new_group(list(devs))
    return pairs, groups


def sweep(rank, world, sizes_mib, out=None, log=print, iters=5):
    """Every (src, dst) pair of {(1,1),(1,2),(1,4)} that fits on `world` GPUs
    (src on the first devices, dst on the next), every spec pair, both optimize
    settings, every size.  Returns the rows (rank 0; None elsewhere)."""
    pairs, groups = make_groups(world)
    rows_out = [] if rank == 0 else None
    for mib in sizes_mib:
        rows = mib * 1024 * 1024 // (8192 * 2)
        dims = (rows, 8192)
        for s, d in pairs:
            sm = Mesh(1, s[1], tuple(range(0, s[1])))
            dm = Mesh(1, d[1], tuple(range(s[1], s[1] + d[1])))
            for ss in specs_2d(sm, dims):
                for ds in specs_2d(dm, dims):
                    res = {}
                    for opt in (True, False):
                        try:
                            res[opt] = run_case(rank, dims, ss, sm, ds, dm, opt, groups, iters)
                        except KeyError:
                            res[opt] = (float("nan"), 0, 0, 1)
                    if rank != 0:
                        continue
                    for opt in (True, False):
                        t, inter, algo, peak = res[opt]
                        row = {"mib": mib, "src": list(s), "dst": list(d),
                               "src_spec": format_spec(ss), "dst_spec": format_spec(ds),
                               "optimize": opt, "time_s": t, "inter_mesh_bytes": inter,
                               "algorithmic_bytes": algo,
                               "bus_gbs": peak / t / 1e9 if t == t and t > 0 else None,
                               "speedup_vs_naive": res[False][0] / t if opt else None}
                        rows_out.append(row)
                        if out is not None:
                            out.write(json.dumps(row) + "\n")
                            out.flush()
                        if opt and log is not None:
                            log(f"{mib:5d} MiB {s}->{d} {format_spec(ss):>6}->{format_spec(ds):<6} "
                                f"opt {t*1e3:8.3f} ms  naive {res[False][0]*1e3:8.3f} ms  "
                                f"x{res[False][0]/t:4.2f}  bus {row['bus_gbs']:.0f} GB/s")
    return rows_out


def summarize(rows):
    """Per (src, dst, optimize): best bus GB/s over spec pairs at each size."""
    best = {}
    for r in rows:
        if r["bus_gbs"] is None:
            continue
        k = (f"{r['src'][1]}->{r['dst'][1]}", "opt" if r["optimize"] else "naive")
        cur = best.setdefault(k, {})
        cur[r["mib"]] = max(cur.get(r["mib"], 0.0), round(r["bus_gbs"], 1))
    return {f"(1,{k[0].split('->')[0]})->(1,{k[0].split('->')[1]}) {k[1]}": v
            for k, v in sorted(best.items())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mib", default=",".join(str(x) for x in SIZES_MIB))
    ap.add_argument("--out", default=str(ROOT / "gpurun_out/xmesh_sweep.jsonl"))
    args = ap.parse_args()
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    native.load()
    out = open(args.out, "a") if rank == 0 else None
    rows = sweep(rank, world, [int(x) for x in args.sizes_mib.split(",")], out,
                 log=lambda m: print(m, flush=True))
    if rank == 0:
        print(json.dumps({"summary_best_bus_gbs": summarize(rows)}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
