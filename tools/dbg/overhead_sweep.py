"""Fixed-cost probe: decode-step GEMM (K5c, split-K, tiled) over K at N = 4096,
M = 64, and verify attention (K6 TMA vs K6c) over context length, CUDA-event
timed; the intercept of time vs bytes is the per-launch fixed cost."""
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from paper_2505_10259_b200 import native  # noqa: E402
from attn_bench import run as attn_run  # noqa: E402

DEV = "cuda:0"


def timed(fn, reps=30, graph=True):
    """µs per call; graph=True: the calls captured in one CUDA graph (device time)."""
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        a.record()
        g.replay()
    else:
        a.record()
        for _ in range(reps):
            fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    g = torch.Generator(device=DEV).manual_seed(0)
    x = torch.randn(64, 4096, device=DEV, generator=g).to(torch.bfloat16)
    n = torch.empty(64, 4096, dtype=torch.bfloat16, device=DEV)
    w1 = torch.ones(4096, dtype=torch.bfloat16, device=DEV)
    print(json.dumps({"rmsnorm_64x4096_us_eager": timed(lambda: native.rmsnorm(x, w1, n, 1e-5), graph=False),
                      "rmsnorm_64x4096_us_graph": timed(lambda: native.rmsnorm(x, w1, n, 1e-5))}), flush=True)
    for K in (256, 1024, 4096, 8192, 14336):
        a = torch.randn(64, K, device=DEV, generator=g).to(torch.bfloat16)
        copies = max(1, -(-256 * 2**20 // (4096 * K * 2)))
        ws = [(torch.randn(4096, K, device=DEV, generator=g) / math.sqrt(K)).to(torch.bfloat16) for _ in range(copies)]
        out = torch.empty(64, 4096, dtype=torch.bfloat16, device=DEV)
        cyc = [0]

        def nxt():
            cyc[0] = (cyc[0] + 1) % copies
            return ws[cyc[0]]
        row = {"K": K, "MB": 4096 * K * 2 / 1e6}
        for v, label in ((4, "k5c"), (1, "splitk"), (3, "tiled")):
            row[label] = timed(lambda: native.gemm(a, nxt(), out, variant=v))
        print(json.dumps(row), flush=True)
        del ws
        torch.cuda.empty_cache()
    for ctx in (64, 256, 520, 1024, 2000):
        for v, label in ((0, "tma"), (2, "tcgen05")):
            r = attn_run(bs=248, n=8, ctx=ctx, variant=v)
            print(json.dumps({"ctx": ctx, "kernel": label, "us": r["us"], "MB": r["kv_MB"]}), flush=True)


if __name__ == "__main__":
    main()
