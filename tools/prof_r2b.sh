#!/bin/bash
# K6c / K5c check: kernel tests, CUDA-event benches, one ncu --set full capture each.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -rs -k "attn or gemv or splitk or gemm_dense" > gpurun_out/pytest_k_r2i.log 2>&1
echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_k_r2i.log
timeout 300 python tools/attn_bench.py > gpurun_out/attn_bench_r2i.jsonl 2>&1
timeout 300 python tools/gemm_bench.py "draft decode" > gpurun_out/gemm_decode_r2i.jsonl 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 3 -c 1 \
  -o gpurun_out/ncu_attn_tc_r2i -f python tools/attn_bench.py 2 > gpurun_out/ncu_attn_tc_r2i.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemv_tc -s 6 -c 1 \
  -o gpurun_out/ncu_gemv_o_r2i -f python tools/gemm_bench.py "draft decode step O (64" > gpurun_out/ncu_gemv_o_r2i.log 2>&1
echo done
