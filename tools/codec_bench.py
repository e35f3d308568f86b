#!/usr/bin/env python
"""K9 XC4 decoder bandwidth at the bench's unit size (one Mixtral-8x22B FFN
unit, 4.83 GB raw, 24 frames), HBM → HBM.

    python tools/codec_bench.py

Algorithmic bytes per launch = encoded frame bytes read + 2 B per decoded
weight written; GB/s against the measured HBM copy peak (MEASURED_PEAKS.json).
Also times the encoder (setup-time cost per layer).
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_10259_b200 import codec, native  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def main(n=4_831_838_208 // 2, reps=10):
    dev = "cuda:0"
    g = torch.Generator(device=dev).manual_seed(0)
    w = torch.empty(n, dtype=torch.bfloat16, device=dev).normal_(0.0, 0.02, generator=g)
    enc = codec.Encoder(dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    unit, h = enc.encode(w)
    t1.record()
    t1.synchronize()
    enc_ms = t0.elapsed_time(t1)
    host = unit.cpu()
    out = torch.empty_like(w)
    f = lambda: native.xc4_decode(host.data_ptr(), unit.data_ptr(), 0, h.n_frames, out.data_ptr())  # noqa: E731
    for _ in range(3):
        f()
    t0.record()
    for _ in range(reps):
        f()
    t1.record()
    t1.synchronize()
    t = t0.elapsed_time(t1) / reps * 1e-3
    assert torch.equal(out.view(torch.int16), w.view(torch.int16))
    algo = unit.numel() + 2 * n
    # context: the same unit as ONE frame (launch-granularity effects), and a plain
    # device copy moving the same bytes in as many launches
    big = {}
    scratch = torch.empty(native.xc4_scratch_bytes(n, 1 << 30), dtype=torch.uint8, device=dev)
    nb1, _ = native.xc4_encode(w, 1 << 30, None, scratch)
    u1 = torch.empty(nb1, dtype=torch.uint8, device=dev)
    _, h1 = native.xc4_encode(w, 1 << 30, u1, scratch)
    h1host = u1.cpu()
    f1 = lambda: native.xc4_decode(h1host.data_ptr(), u1.data_ptr(), 0, h1.n_frames, out.data_ptr())  # noqa: E731
    for _ in range(3):
        f1()
    t0.record()
    for _ in range(reps):
        f1()
    t1.record()
    t1.synchronize()
    tb = t0.elapsed_time(t1) / reps * 1e-3
    big = {"frames": h1.n_frames, "decode_ms": tb * 1e3, "GBps": (nb1 + 2 * n) / tb / 1e9}
    del u1, scratch
    src8 = unit[: unit.numel() // h.n_frames * h.n_frames].view(h.n_frames, -1)
    dst8 = out.view(torch.uint8)[: src8.numel()].view(h.n_frames, -1)
    t0.record()
    for _ in range(reps):
        for i in range(h.n_frames):
            dst8[i].copy_(src8[i])
    t1.record()
    t1.synchronize()
    tc = t0.elapsed_time(t1) / reps * 1e-3
    copy = {"bytes": 2 * src8.numel(), "ms": tc * 1e3, "GBps": 2 * src8.numel() / tc / 1e9}
    print(json.dumps({"one_frame": big, "device_copy_same_launches": copy}))
    print(json.dumps({"n_elems": n, "frames": h.n_frames, "ratio": unit.numel() / (2 * n), "escapes": h.n_escapes,
                      "decode_ms": t * 1e3, "decode_GBps": algo / t / 1e9, "frac_of_hbm_peak": algo / t / 1e9 / PEAK,
                      "encode_ms": enc_ms, "bit_exact": True}))


if __name__ == "__main__":
    main()
