#!/usr/bin/env python
"""C5 planner sweep on hardware: measure decode tokens/s for several policies of
the 8x22B offloaded pair, then re-fit the B200 rates of the cost model to the
measurements (the reference's calibrate, planner.py:215-319, north-star item 4).

    python tools/sweep.py --out gpurun_out/sweep.json

One engine (weights, pinned/streamed split of the largest policy) serves every
policy; each point runs: synthetic context → first draft → 2 warm-up rounds →
3 timed rounds (CUDA events on the verify stream).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/sweep.json")
    ap.add_argument("--p", type=float, default=0.8)
    ap.add_argument("--ctx", type=int, default=503)
    ap.add_argument("--timed", type=int, default=3)
    args = ap.parse_args()

    import torch

    from bench import h2d_peak, mem_available
    from paper_2505_10259_b200 import MIXTRAL_8X22B, MISTRAL_7B_V3, Policy
    from paper_2505_10259_b200.acceptance import AcceptanceModel, expected_accepted
    from paper_2505_10259_b200.api import build_engine
    from paper_2505_10259_b200.planner_b200 import B200Rates, plan_offload
    from paper_2505_10259_b200.streamer import HostStore

    dev = torch.device("cuda", 0)
    link = h2d_peak(torch, dev)
    free, _ = torch.cuda.mem_get_info(dev)
    host = mem_available() - int(14e9)
    points = [(n, bs, kv) for n in (2, 4, 8) for bs, kv in ((64, "cached"), (128, "cached"), (224, "reprefill"))]
    max_new = 4 * 9 + 2
    big = plan_offload(MIXTRAL_8X22B, MISTRAL_7B_V3, free, host, 8, args.p, args.ctx, max_new, B200Rates(link),
                       bs_candidates=[224], draft_kv_modes=("reprefill",))
    eng = build_engine(MIXTRAL_8X22B, MISTRAL_7B_V3, device=dev, stream_layers=set(big.stream_layers), seed=1,
                       trace=False, host_store=HostStore(), stream_attn=big.stream_attn)
    S = len(big.stream_layers) * eng.target.streamer.layer_bytes
    rows = []
    for n, bs, kv in points:
        torch.cuda.empty_cache()
        s = eng.new_session(2 * bs, bs, args.ctx + max_new + n + 2, n, forced_p=args.p, seed=0,
                            bs_draft=min(bs, 64) if kv == "reprefill" else bs, draft_kv=kv)
        eng.synthetic_context(s, args.ctx, max_new)
        eng.first_draft(s)
        for _ in range(2):
            eng.round(s)
        c0 = s.committed_decode
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(eng.tgt_stream)
        for _ in range(args.timed):
            eng.round(s)
        b.record(eng.tgt_stream)
        b.synchronize()
        dt = a.elapsed_time(b) * 1e-3
        tps = (s.committed_decode - c0) / dt
        rows.append({"policy": [2 * bs, bs, s.bs_draft, n], "draft_kv": kv, "streamed_bytes": S,
                     "tokens_per_s": tps, "round_s": dt / args.timed,
                     "expected_tokens_per_round": bs * expected_accepted(AcceptanceModel(args.p, n))})
        print(json.dumps(rows[-1]), flush=True)
        del s
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    json.dump({"link_peak_Bps": link, "hbm_free": free, "host_budget": host, "points": rows}, open(args.out, "w"),
              indent=1)


if __name__ == "__main__":
    main()
