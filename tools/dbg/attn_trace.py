"""Where K6c's roles wait (debug build: make -C paper_2505_10259_b200/csrc EXTRA=-DSO_ATTN_TRACE).
Per wait site: mean cycles per CTA (producer = thread 0, MMA = thread 32, softmax = thread 64), as a
fraction of the softmax thread's total cycles; one launch at the bench's verify shape and one prefill."""
import ctypes
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from paper_2505_10259_b200 import native  # noqa: E402
from attn_bench import run  # noqa: E402

NAMES = ["prod:q_empty", "prod:k_empty", "prod:v_empty", "mma:k_full", "mma:s_empty", "mma:q_full", "mma:o_empty",
         "mma:v_full", "mma:p_full", "soft:s_full", "soft:p_empty_rescale", "soft:v_full", "soft:p_empty",
         "soft:o_full", "soft:total", "mma:total"]
for kw in [dict(bs=488, n=8, ctx=520), dict(bs=64, n=519, ctx=1, hq=32, hkv=8), dict(bs=64, n=0, ctx=520, hq=32, hkv=8)]:
    buf = np.zeros((1024, 16), np.uint64)
    native.lib().so_attn_trace_copy(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes), 1)
    r = run(variant=2, reps=1, **kw)
    torch.cuda.synchronize()
    native.lib().so_attn_trace_copy(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes), 1)
    live = buf[:, 14] > 0
    mean = buf[live].astype(np.float64).mean(0)
    # reps=1 but run() warms up 3× and the graph replays once more: 5 launches accumulated
    tot = mean[14]
    print(json.dumps({"shape": kw, "us": r["us"], "ctas": int(live.sum()),
                      "frac_of_softmax_total": {NAMES[i]: round(mean[i] / tot, 3) for i in range(16)}}))
