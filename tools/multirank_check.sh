#!/bin/bash
# N > 1 functional check on one GPU (gloo; both ranks share the device): the torchrun path of
# bench.py with host-streamed XC4 slices and HBM shards (profiles/multirank_gloo_r1.md).
mkdir -p gpurun_out
for extra in "" "--max-pinned 0 --no-shards" "--max-pinned 0"; do
  L=$([ -z "$extra" ] && echo 8 || echo 4)
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
    bench.py --gpus 2 --dist-backend gloo --layers $L --hbm-gb 80 --host-gb 60 --steps 2 --warmup 3 \
    --no-cpu-baseline --no-e2e-generate --no-parity $extra > gpurun_out/multirank_$L${extra// /_}.log 2>&1
  echo "layers $L extra '$extra' rc=$?"
  grep -h "plan:" gpurun_out/multirank_$L${extra// /_}.log | head -2
  tail -c 300 gpurun_out/multirank_$L${extra// /_}.log | tr '\n' ' '; echo
done
