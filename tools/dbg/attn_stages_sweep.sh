#!/bin/bash
# K6 ring depth sweep (SO_ATTN_STAGES) at the bench's verify / re-prefill / decode shapes, 32-token pages.
mkdir -p gpurun_out
for st in 2 3 4 6 8; do
  touch paper_2505_10259_b200/csrc/attention.cu
  make -s -j8 -C paper_2505_10259_b200/csrc EXTRA=-DSO_ATTN_STAGES=$st > /dev/null 2>&1 || { echo "stages $st: build failed"; continue; }
  timeout 120 python - <<PY
import json, sys, os
sys.path.insert(0, "tools"); sys.path.insert(0, ".")
from attn_bench import run
for shape in (dict(bs=512, n=8, ctx=520), dict(bs=64, n=0, ctx=520, hq=32, hkv=8)):
    for v in (0, 1):
        r = run(ps=32, variant=v, **shape)
        print(json.dumps({"stages": $st, "variant": v, "n": shape["n"], "us": round(r["us"], 1), "frac_hbm": round(r["frac_of_hbm_peak"], 3)}))
PY
done
touch paper_2505_10259_b200/csrc/attention.cu; make -s -j8 -C paper_2505_10259_b200/csrc > /dev/null 2>&1
