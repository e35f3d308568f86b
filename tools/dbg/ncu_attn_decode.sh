mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_paged -s 3 -c 1 -o gpurun_out/ncu_attn_decode_r2ee -f python - <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
from attn_bench import run
print(run(bs=64, n=0, ctx=520, hq=32, hkv=8, ps=32, variant=0, reps=2))
PY
echo rc=$?
