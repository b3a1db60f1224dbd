"""HBM bandwidth of mp_pack_box / mp_unpack_box on the relayout shapes of the
tensor-parallel plans (RS^1 <-> S^1R halves of (8192, 1024|2048) bf16)."""
import json

import torch

from paper_2201_12023_b200 import native


def main():
    for rows, cols in ((8192, 1024), (8192, 2048), (8192, 8192)):
        t = torch.randn(rows, cols // 2, device="cuda").to(torch.bfloat16)   # an RS^1 tile
        lo, ext = (rows // 2, 0), (rows // 2, cols // 2)
        out = torch.empty(ext[0] * ext[1], device="cuda", dtype=torch.bfloat16)
        # 50 launches captured in a CUDA graph: device time, not the host launch rate
        native.pack_box(t, lo, ext, out=out)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(50):
                native.pack_box(t, lo, ext, out=out)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 50 * 1e3
        nbytes = 2 * out.numel() * 2
        print(json.dumps({"box": ext, "us": us, "gbs": nbytes / us / 1e3}), flush=True)


if __name__ == "__main__":
    main()
