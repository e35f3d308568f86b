"""Encode one synthetic Mixtral-8x22B FFN unit with the default encoder and with a
split-window (frame-aligned) encoder; print sizes and headers."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2505_10259_b200 import MIXTRAL_8X22B, codec as C  # noqa: E402
from paper_2505_10259_b200.weights import ffn_offsets  # noqa: E402

dev = "cuda:0"
gu, dn, nbytes = ffn_offsets(MIXTRAL_8X22B)
g = torch.Generator(device=dev).manual_seed(1)
unit = torch.empty(nbytes // 2, dtype=torch.bfloat16, device=dev).normal_(0.0, 0.02, generator=g)
for name, enc in (("default", C.Encoder(dev)), ("aligned", C.Encoder(dev, align_elems=gu)),
                  ("bits3", C.Encoder(dev, code_bits=3)), ("bits4", C.Encoder(dev, code_bits=4))):
    d, h = enc.encode(unit)
    print(json.dumps({"enc": name, "bytes": d.numel(), "ratio": d.numel() / nbytes, "frame_elems": h.frame_elems,
                      "n_frames": h.n_frames, "version": h.version, "escapes": h.n_escapes}), flush=True)
    enc.release()
    torch.cuda.empty_cache()
for n in (1 << 26, 1 << 27, 100663296):
    probe = unit[:n].contiguous()
    d, h = C.Encoder(dev).encode(probe)
    print(json.dumps({"probe_elems": n, "ratio": d.numel() / (2 * n), "version": h.version}), flush=True)
