#!/usr/bin/env python
"""C5 planner sweep on hardware (BASELINE.json configs[4]): Mixtral-8x22B-shaped
target offloaded (XC4-coded streaming) + Mistral-7B draft, draft length ×
batch size × HBM budget — measured decode tokens/s beside the planner's
prediction and the host-link roofline.

    python tools/sweep.py --out gpurun_out/sweep.json

For each HBM budget one engine (weights, pinned/streamed split of that
budget's n_cand = 8 plan) serves every policy: per point the planner picks
the batch and the draft-KV split for that draft length on the engine's split
(plus a half-batch point), then synthetic context → first draft → 2 warm-up
rounds → 3 timed rounds (CUDA events on the verify stream).  The rates of the
cost model are then re-fit to the measured rounds (planner_b200.calibrate_rounds,
the reference's calibrate, planner.py:215-319).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/sweep.json")
    ap.add_argument("--p", type=float, default=0.8)
    ap.add_argument("--ctx", type=int, default=503)
    ap.add_argument("--timed", type=int, default=3)
    ap.add_argument("--budgets", default="0", help="HBM budgets in GB, comma-separated (0 = the whole device); "
                                                   "run one budget per process: the pinned host store is per process")
    args = ap.parse_args()

    import numpy as np
    import torch

    from bench import h2d_peak, mem_available
    from paper_2505_10259_b200 import MIXTRAL_8X22B, MISTRAL_7B_V3
    from paper_2505_10259_b200 import codec as C
    from paper_2505_10259_b200.acceptance import AcceptanceModel, expected_accepted
    from paper_2505_10259_b200.api import build_engine
    from paper_2505_10259_b200.planner_b200 import B200Rates, plan_offload
    from paper_2505_10259_b200.streamer import HostStore

    dev = torch.device("cuda", 0)
    link = h2d_peak(torch, dev)
    host = mem_available() - int(14e9)
    g = torch.Generator(device=dev).manual_seed(12345)
    probe = torch.empty(1 << 26, dtype=torch.bfloat16, device=dev).normal_(0.0, 0.02, generator=g)
    enc = C.Encoder(dev)
    ratio = enc.encode(probe)[0].numel() / (2 * probe.numel()) * 1.002
    enc.release()
    del probe
    torch.cuda.empty_cache()
    rates = B200Rates(h2d_bytes_per_s=link)
    max_new = 4 * 9 + 2
    ring = 4 * (192 << 20)
    rows = []
    for budget_gb in [float(b) for b in args.budgets.split(",")]:
        free, _ = torch.cuda.mem_get_info(dev)
        hbm = int(budget_gb * 1e9) if budget_gb else free
        big = plan_offload(MIXTRAL_8X22B, MISTRAL_7B_V3, hbm, host, 8, args.p, args.ctx, max_new, rates,
                           stream_ratio=ratio, ring_bytes=ring)
        eng = build_engine(MIXTRAL_8X22B, MISTRAL_7B_V3, device=dev, stream_layers=set(big.stream_layers), seed=1,
                           trace=False, host_store=HostStore(), stream_attn=big.stream_attn, codec="xc4")
        st = eng.target.streamer
        for n in (2, 4, 6, 8):
            best = plan_offload(MIXTRAL_8X22B, MISTRAL_7B_V3, hbm, host, n, args.p, args.ctx, max_new, rates,
                                stream_ratio=ratio, ring_bytes=ring, max_pinned=len(big.pinned_layers),
                                stream_attn_modes=(big.stream_attn,))
            for bs in (best.bs_decoding, best.bs_decoding // 2):
                pl = best if bs == best.bs_decoding else plan_offload(
                    MIXTRAL_8X22B, MISTRAL_7B_V3, hbm, host, n, args.p, args.ctx, max_new, rates,
                    stream_ratio=ratio, ring_bytes=ring, max_pinned=len(big.pinned_layers),
                    stream_attn_modes=(big.stream_attn,), bs_candidates=[bs])
                torch.cuda.empty_cache()
                s = eng.new_session(2 * pl.bs_decoding, pl.bs_decoding, args.ctx + max_new + n + 2, n,
                                    forced_p=args.p, seed=0, bs_draft=pl.bs_draft, draft_kv=pl.draft_kv,
                                    draft_cached=pl.draft_cached)
                eng.synthetic_context(s, args.ctx, max_new)
                eng.first_draft(s)
                for _ in range(2):
                    eng.round(s)
                c0, b0 = s.committed_decode, st.bytes_issued
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(eng.tgt_stream)
                eng.round_times.clear()
                for _ in range(args.timed):
                    eng.round(s)
                b.record(eng.tgt_stream)
                b.synchronize()
                dt = a.elapsed_time(b) * 1e-3
                tps = (s.committed_decode - c0) / dt
                link_s = (st.bytes_issued - b0) / args.timed / link
                e = expected_accepted(AcceptanceModel(args.p, n))
                rows.append({"hbm_budget_gb": budget_gb or round(free / 1e9, 1), "n_cand": n,
                             "policy": [2 * pl.bs_decoding, pl.bs_decoding, pl.bs_draft, n],
                             "draft_kv": pl.draft_kv, "draft_cached": pl.draft_cached,
                             "pinned": len(big.pinned_layers), "streamed": len(big.stream_layers),
                             "tokens_per_s": tps, "round_s": dt / args.timed, "link_s": link_s,
                             "draft_stream_s": float(np.mean([d for d, _ in eng.round_times])) * 1e-3,
                             "predicted_tokens_per_s": pl.tokens_per_s,
                             "roofline_tokens_per_s": pl.bs_decoding * e / max(link_s, 1e-9),
                             "streamed_bytes": st.bytes_issued - b0, "expected_tokens_per_round": pl.bs_decoding * e,
                             "hbm_allocated_gb": round(torch.cuda.max_memory_allocated(dev) / 1e9, 1)})
                print(json.dumps(rows[-1]), flush=True)
                del s
        del eng, st
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    json.dump({"link_peak_Bps": link, "host_budget": host, "stream_ratio": ratio, "points": rows},
              open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
