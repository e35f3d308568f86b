#!/usr/bin/env python
"""Verify-attention (K6) bandwidth at the bench shape: 8x22B heads (48 q / 8 kv × 128),
bs sequences × (n_cand+1) queries over ctx keys, 16-token pages.

    python tools/attn_bench.py

KV bytes read per launch = bs · (ctx + n + 1) · n_kv · dh · 2 (K,V) · 2 B; GB/s against
the measured HBM copy peak (MEASURED_PEAKS.json).  Caches larger than L2 (126 MB), so
every launch streams from HBM.
"""
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_10259_b200 import native  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def run(bs=248, n=8, ctx=520, hq=48, hkv=8, dh=128, ps=16, reps=20, variant=0):
    dev = "cuda:0"
    q_len = n + 1
    max_len = ctx + q_len
    pps = (max_len + ps - 1) // ps
    npages = bs * pps
    g = torch.Generator(device=dev).manual_seed(0)
    kc = torch.randn(npages, hkv, ps, dh, device=dev, generator=g).to(torch.bfloat16)
    vc = torch.randn(npages, hkv, ps, dh, device=dev, generator=g).to(torch.bfloat16)
    bt = torch.arange(npages, dtype=torch.int32, device=dev).view(bs, pps)
    qs = torch.arange(bs + 1, dtype=torch.int32, device=dev) * q_len
    kvb = torch.full((bs,), ctx, dtype=torch.int32, device=dev)
    q = torch.randn(bs * q_len, hq * dh, device=dev, generator=g).to(torch.bfloat16)
    out = torch.empty_like(q)
    f = lambda: native.attn_paged(q, kc, vc, bt, qs, kvb, q_len, hq, hkv, dh, ps, 1 / math.sqrt(dh), out,
                                      variant=variant)  # noqa
    # reps launches in one CUDA graph: device time, without the per-call host enqueue
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
    kv_bytes = bs * (ctx + q_len) * hkv * dh * 2 * 2
    # causal FLOPs: QKᵀ and PV over the keys each query row sees (ctx + j + 1)
    flops = 4.0 * bs * hq * dh * sum(ctx + j + 1 for j in range(q_len))
    return {"bs": bs, "n_cand": n, "ctx": ctx, "hq": hq, "us": t * 1e6, "kv_MB": kv_bytes / 1e6,
            "GBps": kv_bytes / t / 1e9, "frac_of_hbm_peak": kv_bytes / t / 1e9 / PEAK, "tflops": flops / t / 1e12}


if __name__ == "__main__":
    if len(sys.argv) > 1:  # one variant at the verify shape of the bench plan (profiling)
        v = int(sys.argv[1])
        print(json.dumps(run(bs=488, n=8, ctx=520, variant=v, reps=5)))
        sys.exit(0)
    for variant, label in ((1, "cp_async"), (0, "auto (tma; K6d for decode)"), (2, "tcgen05"), (3, "k6d")):
        for r in [run(variant=variant), run(bs=128, n=4, variant=variant), run(bs=248, n=8, ctx=2000, variant=variant),
                  run(bs=488, n=8, ctx=520, variant=variant), run(bs=64, n=519, ctx=1, hq=32, hkv=8, variant=variant),
                  run(bs=64, n=0, ctx=520, hq=32, hkv=8, variant=variant)]:
            r["staging"] = label
            print(json.dumps(r))
