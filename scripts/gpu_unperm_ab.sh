#!/bin/bash
# A/B of the k > 2 un-permute kernels on the N=1 DeepSeek bench (quick mode):
# MONTA_UNPERM_VAR (vectors per thread x 10 + slots in flight), MONTA_UNPERM_GRID (CTAs per SM).
mkdir -p gpurun_out/unperm
for cfg in "41 16" "41 64" "22 16" "22 64" "21 16" "21 64" "23 16" "23 64" "41 8" "22 8"; do
  set -- $cfg
  MONTA_UNPERM_VAR=$1 MONTA_UNPERM_GRID=$2 timeout 300 python bench.py --quick --steps 20 --warmup 5 > gpurun_out/unperm/v$1g$2.json 2> gpurun_out/unperm/v$1g$2.err
  python - "v$1 g$2" gpurun_out/unperm/v$1g$2.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"], 1), {k: round(v["avg_us"], 1) for k, v in d["stages"].items()}, round(d["roofline"]["frac"], 3))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
