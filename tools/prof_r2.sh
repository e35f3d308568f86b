#!/bin/bash
# Round-2 kernel measurements (run under gpurun from the repo root): verify/draft
# attention variants and decode-step GEMMs timed with CUDA events, then one
# ncu --set full capture per kernel of interest.
set -x
mkdir -p gpurun_out
timeout 300 python tools/attn_bench.py > gpurun_out/attn_bench_r2.jsonl 2>&1
timeout 300 python tools/gemm_bench.py "draft decode" > gpurun_out/gemm_decode_r2.jsonl 2>&1
for v in 0 2; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn -s 3 -c 1 \
    -o gpurun_out/ncu_attn_v${v}_r2 -f python tools/attn_bench.py $v > gpurun_out/ncu_attn_v${v}_r2.log 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemv_tc -s 6 -c 1 \
  -o gpurun_out/ncu_gemv_down_r2 -f python tools/gemm_bench.py "draft decode step down (64" > gpurun_out/ncu_gemv_r2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemv_tc -s 6 -c 1 \
  -o gpurun_out/ncu_gemv_o_r2 -f python tools/gemm_bench.py "draft decode step O" > gpurun_out/ncu_gemv_o_r2.log 2>&1
ls -la gpurun_out
