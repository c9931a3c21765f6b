#!/bin/bash
# A/B of the N=1 permute kernels on the DeepSeek bench (quick mode):
# MONTA_AA_BULK=0 (warp-per-item register copy) vs the TMA bulk ring with
# MONTA_AA_STAGES / MONTA_AA_DEPTH / MONTA_AA_CPS.
mkdir -p gpurun_out/aa
IFS=, read -ra LIST <<< "${CFGS:-0 8 4 2,1 8 4 2}"
for cfg in "${LIST[@]}"; do
  set -- $cfg
  tag=b$1s$2d$3c$4
  MONTA_AA_BULK=$1 MONTA_AA_STAGES=$2 MONTA_AA_DEPTH=$3 MONTA_AA_CPS=$4 timeout 300 python bench.py --quick --steps 20 --warmup 5 ${BENCH_ARGS:-} > gpurun_out/aa/$tag.json 2> gpurun_out/aa/$tag.err
  python - "$tag" gpurun_out/aa/$tag.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"], 1), {k: round(v["avg_us"], 1) for k, v in d["stages"].items()}, d["roofline"]["kernel"], round(d["roofline"]["frac"], 3))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
