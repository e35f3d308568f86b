"""Phase timeline of one K5c launch (debug build: make -C paper_2505_10259_b200/csrc EXTRA=-DSO_GEMV_TRACE).
Slots: 0 entry, 1 setup done, 2 first TMA issued, 3 last MMA committed, 4 accumulator ready (epilogue),
5 all partials ready (cluster), 6 reduction done, 7 exit.  Prints per-slot min / median / max over CTAs,
in µs after the earliest entry."""
import ctypes
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2505_10259_b200 import native  # noqa: E402

DEV = "cuda:0"
for (M, N, K) in [(64, 4096, 256), (64, 4096, 4096), (64, 4096, 14336)]:
    g = torch.Generator(device=DEV).manual_seed(0)
    a = torch.randn(M, K, device=DEV, generator=g).to(torch.bfloat16)
    b = (torch.randn(N, K, device=DEV, generator=g) / math.sqrt(K)).to(torch.bfloat16)
    out = torch.empty(M, N, dtype=torch.bfloat16, device=DEV)
    for _ in range(3):
        native.gemm(a, b, out, variant=4)
    torch.cuda.synchronize()
    buf = np.zeros((1024, 8), np.uint64)
    native.lib().so_gemv_trace_copy(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
    # ctas that ran this launch: entry stamp within 1 ms of the latest entry
    ent = buf[:, 0].astype(np.int64)
    live = ent > ent.max() - 1_000_000
    t = (buf[live].astype(np.int64) - ent[live].min()) / 1e3
    print(json.dumps({"M": M, "N": N, "K": K, "ctas": int(live.sum()),
                      "slots_us_min_med_max": [[round(float(t[:, i].min()), 2), round(float(np.median(t[:, i])), 2),
                                                round(float(t[:, i].max()), 2)] for i in range(8)]}))
