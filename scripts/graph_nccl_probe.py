"""Probe: can torch.distributed NCCL ops be captured in a CUDA graph here?"""
import os, sys
import torch
import torch.distributed as dist

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
g = dist.new_group(list(range(world)))
x = torch.ones(1 << 20, device="cuda") * (rank + 1)
y = torch.empty(world << 20, device="cuda")
s = torch.cuda.Stream()
res = {}
for name, fn in [("all_reduce", lambda: dist.all_reduce(x, group=g)),
                 ("all_gather", lambda: dist.all_gather_into_tensor(y, x, group=g)),
                 ("p2p", lambda: [w.wait() for w in dist.batch_isend_irecv(
                     [dist.P2POp(dist.isend, x, (rank + 1) % world, group=g),
                      dist.P2POp(dist.irecv, y[: 1 << 20], (rank - 1) % world, group=g)])])]:
    try:
        fn()  # warm
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(graph, stream=s):
                fn()
        torch.cuda.synchronize()
        x.fill_(rank + 1)
        graph.replay()
        torch.cuda.synchronize()
        res[name] = ("ok", float(x[0]) if name == "all_reduce" else float(y[:1].item()))
    except Exception as e:
        res[name] = ("fail", repr(e)[:200])
print(rank, res, flush=True)
dist.barrier()
dist.destroy_process_group()
