cd paper_2505_10259_b200/csrc
for cfg in "3 4" "4 3" "4 2" "3 3"; do set -- $cfg
  touch attention.cu; make -s EXTRA="-DSO_ATTN_MINB=$1 -DSO_ATTN_STAGES=$2" > /dev/null 2>&1
  echo "MINB=$1 STAGES=$2"; (cd ../..; timeout 120 python tools/attn_bench.py | python -c "import sys,json; [print(' ', json.loads(l)['bs'], json.loads(l)['ctx'], round(json.loads(l)['GBps']), round(json.loads(l)['frac_of_hbm_peak'],3)) for l in sys.stdin]")
done
