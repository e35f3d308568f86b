#!/usr/bin/env python
"""K2 fused router at the verify shape of the bench plan: T = bs·(n_cand+1) tokens of
Mixtral-8x22B (H 6144, 8 experts).  Graph-timed; algorithmic bytes = x read once (T·H·2)
+ x_perm written (2T·H·2) + gate weights (E·H·2)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_10259_b200 import native  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
DEV = "cuda:0"


def main(T=4608, H=6144, E=8, reps=20):
    g = torch.Generator(device=DEV).manual_seed(0)
    x = torch.randn(T, H, device=DEV, generator=g).to(torch.bfloat16)
    wg = (torch.randn(E, H, device=DEV, generator=g) * 0.02).to(torch.bfloat16)
    offs = torch.empty(E + 1, dtype=torch.int32, device=DEV)
    perm = torch.empty(2 * T, dtype=torch.int32, device=DEV)
    roww = torch.empty(2 * T, dtype=torch.float32, device=DEV)
    trows = torch.empty((T, 2), dtype=torch.int32, device=DEV)
    xperm = torch.empty((2 * T, H), dtype=torch.bfloat16, device=DEV)
    ws = torch.empty(native.router_workspace_bytes(T, E), dtype=torch.uint8, device=DEV)
    f = lambda: native.router_top2(x, wg, offs, perm, roww, trows, xperm, ws)  # noqa: E731
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(3):
            f()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(reps):
            f()
    gr.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    gr.replay()
    b.record()
    b.synchronize()
    t = a.elapsed_time(b) / reps * 1e-3
    nbytes = T * H * 2 + 2 * T * H * 2 + E * H * 2
    print(json.dumps({"T": T, "H": H, "E": E, "us": t * 1e6, "GBps": nbytes / t / 1e9,
                      "frac_of_hbm_peak": nbytes / t / 1e9 / PEAK}))


if __name__ == "__main__":
    main(reps=3 if len(sys.argv) > 1 else 20)
