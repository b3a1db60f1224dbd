"""cProfile of one executor step on every rank; rank 0 prints the top entries."""
import cProfile, io, json, os, pstats, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
import torch.distributed as dist


def main():
    plan = sys.argv[1]
    mb = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    doc = json.loads(Path(plan).read_text())
    doc["num_microbatches"] = mb
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        local = int(os.environ["LOCAL_RANK"])
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2201_12023_b200.runtime import Executor
    ex = Executor(doc, schedule="1f1b")
    ex.step()
    pr = cProfile.Profile()
    pr.enable()
    dt = ex.step()
    pr.disable()
    if world == 1 or dist.get_rank() == 0:
        s = io.StringIO()
        pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
        print(f"device step {dt*1e3:.1f} ms")
        print(s.getvalue()[:6000])
    if world > 1:
        dist.barrier()


if __name__ == "__main__":
    main()
