"""Attention time vs KV page size (verify, re-prefill and decode shapes; K6 TMA / cp.async and K6c)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "tools"))
sys.path.insert(0, ROOT)
from attn_bench import run  # noqa: E402

for ps in (16, 32, 64):
    for shape in (dict(bs=512, n=8, ctx=520), dict(bs=64, n=519, ctx=1, hq=32, hkv=8), dict(bs=64, n=0, ctx=520, hq=32, hkv=8)):
        for v, label in ((0, "auto"), (1, "cp_async"), (2, "tcgen05")):
            r = run(ps=ps, variant=v, **shape)
            print(json.dumps({"ps": ps, "kernel": label, **{k: shape[k] for k in ("bs", "n", "ctx")}, "us": round(r["us"], 1),
                              "frac_hbm": round(r["frac_of_hbm_peak"], 3), "tflops": round(r["tflops"], 1)}), flush=True)
