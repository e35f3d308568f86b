#!/usr/bin/env python
"""GEMM throughput on the path's real shapes, 1-CTA vs CTA-pair (cta_group::2) tiles.

    python tools/gemm_bench.py > gpurun_out/gemm_bench.json

CUDA-event timing of 20 launches captured in one CUDA graph (device time, no per-call host overhead), 3 warm-up launches, best of 3 interleaved trials per variant; TFLOP/s against
the measured cuBLAS bf16 burst peak (MEASURED_PEAKS.json).  Weights are
re-used across launches (L2-resident up to 126 MB; the MoE shapes exceed it).
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

DEV = "cuda:0"
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1590.0


def timed(fn, reps=10):
    """Seconds per call of ``fn``: ``reps`` calls captured in one CUDA graph and
    replayed, so the figure is device time — a per-call Python/ctypes enqueue
    (≈ 10 µs) would otherwise bound any kernel shorter than that."""
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


def main():
    only = sys.argv[1] if len(sys.argv) > 1 else None  # substring filter on the shape name (profiling)
    g = torch.Generator(device=DEV).manual_seed(0)
    rows = []
    shapes = [
        # name, M(rows), N, K, epilogue, grouped experts (0 = dense)
        ("8x22B MoE gate_up (bs 248, n 8)", 4464, 32768, 6144, native.EPI_SWIGLU, 8),
        ("8x22B MoE down (bs 248, n 8)", 4464, 6144, 16384, native.EPI_BF16_ROWSCALE, 8),
        ("8x22B MoE gate_up (bs 472, n 8)", 8496, 32768, 6144, native.EPI_SWIGLU, 8),
        ("8x22B MoE down (bs 472, n 8)", 8496, 6144, 16384, native.EPI_BF16_ROWSCALE, 8),
        ("8x22B MoE gate_up (refill prefill 16k tokens)", 32768, 32768, 6144, native.EPI_SWIGLU, 8),
        ("8x22B MoE down (refill prefill 16k tokens)", 32768, 6144, 16384, native.EPI_BF16_ROWSCALE, 8),
        ("8x22B QKV (T 2232)", 2232, 8192, 6144, native.EPI_BF16, 0),
        ("8x22B LM head (T 2232)", 2232, 32768, 6144, native.EPI_F32, 0),
        ("Mistral-7B re-prefill gate_up (64 seqs x 520)", 33280, 28672, 4096, native.EPI_SWIGLU, 0),
        ("Mistral-7B re-prefill down", 33280, 4096, 14336, native.EPI_BF16_RESID, 0),
        ("Mistral-7B re-prefill O", 33280, 4096, 4096, native.EPI_BF16_RESID, 0),
        ("Mistral-7B re-prefill QKV", 33280, 6144, 4096, native.EPI_BF16, 0),
        ("Mistral-7B re-prefill down (32 seqs x 520)", 16640, 4096, 14336, native.EPI_BF16_RESID, 0),
        ("Mistral-7B re-prefill gate_up (32 seqs x 520)", 16640, 28672, 4096, native.EPI_SWIGLU, 0),
        ("square 8192^3", 8192, 8192, 8192, native.EPI_BF16, 0),
        ("draft decode step QKV (64 seqs)", 64, 6144, 4096, native.EPI_BF16, 0),
        ("draft decode step O (64 seqs)", 64, 4096, 4096, native.EPI_BF16_RESID, 0),
        ("draft decode step gate_up (64 seqs)", 64, 28672, 4096, native.EPI_SWIGLU, 0),
        ("draft decode step down (64 seqs)", 64, 4096, 14336, native.EPI_BF16_RESID, 0),
        ("draft decode step down (112 seqs)", 112, 4096, 14336, native.EPI_BF16_RESID, 0),
        ("draft decode step QKV (128 seqs)", 128, 6144, 4096, native.EPI_BF16, 0),
        ("draft decode step O (128 seqs)", 128, 4096, 4096, native.EPI_BF16_RESID, 0),
        ("draft decode step LM head (64 seqs)", 64, 32768, 4096, native.EPI_F32, 0),
    ]
    for name, M, N, K, epi, E in shapes:
        if only and only not in name:
            continue
        a = torch.randn(M, K, device=DEV, generator=g).to(torch.bfloat16)
        wbytes = max(E, 1) * N * K * 2
        # decode-step shapes read each layer's weights once per step from HBM: cycle through enough
        # copies (> 2 × the 126 MB L2) that no launch finds its weights L2-resident
        copies = max(1, -(-256 * 2**20 // wbytes)) if M <= 128 else 1
        bs_ = [(torch.randn(max(E, 1) * N, K, device=DEV, generator=g) / math.sqrt(K)).to(torch.bfloat16)
               for _ in range(copies)]
        b = bs_[0]
        cyc = [0]

        def nxt():
            cyc[0] = (cyc[0] + 1) % copies
            return bs_[cyc[0]]
        out_cols = N // 2 if epi == native.EPI_SWIGLU else N
        out = torch.empty(M, out_cols, dtype=torch.float32 if epi == native.EPI_F32 else torch.bfloat16, device=DEV)
        aux = None
        if epi == native.EPI_BF16_RESID:
            aux = torch.randn(M, N, device=DEV, generator=g).to(torch.bfloat16)
        elif epi == native.EPI_BF16_ROWSCALE:
            aux = torch.rand(M, device=DEV, generator=g)
        if E:
            cnt = np.full(E, M // E)
            cnt[: M - cnt.sum()] += 1
            offs = torch.tensor(np.concatenate([[0], np.cumsum(cnt)]), dtype=torch.int32, device=DEV)
            fn = lambda v: native.gemm_grouped(a, b.data_ptr(), offs, E, N, out, epi, aux, variant=v)  # noqa: E731
        else:
            fn = lambda v: native.gemm(a, nxt(), out, epi, aux, variant=v)  # noqa: E731
        flops = 2.0 * M * N * K
        res = {"shape": name, "M": M, "N": N, "K": K, "weight_copies_cycled": copies}
        variants = ((3, "tile_per_cta_auto"), (0, "persistent_auto"), (1, "cta1"), (2, "cta_pair"))
        if M <= 128 and not E:
            variants = ((3, "tile_per_cta_auto"), (1, "splitk_cta1"), (4, "k5c_cluster_splitk"))
        best = {}
        for _ in range(3):  # interleaved trials, best of 3 (clocks drift under the power cap)
            for variant, label in variants:
                t = timed(lambda: fn(variant), reps=20)
                best[label] = min(best.get(label, t), t)
        for _, label in variants:
            t = best[label]
            res[label] = {"ms": t * 1e3, "tflops": flops / t / 1e12, "frac_of_peak": flops / t / 1e12 / PEAK,
                          "weight_GBps": wbytes / t / 1e9}
        rows.append(res)
        print(json.dumps(res), flush=True)
        del a, b, bs_, out, aux
        torch.cuda.empty_cache()
    print(json.dumps({"peak_tflops": PEAK, "rows": rows}))


if __name__ == "__main__":
    main()
