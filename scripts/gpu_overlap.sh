#!/bin/bash
# Experts overlapped with the reverse AllToAll: multi-GPU parity (incl. bit-equality
# with the sequential order) and the N=2 / N=4 bench lines' experts legs.
mkdir -p gpurun_out/overlap
timeout 300 python -m pytest tests/test_gpu_experts.py -x -q 2>&1 | tail -1; timeout 900 python -m pytest tests/test_multigpu.py -x -q -k "experts" > gpurun_out/overlap/t_mgpu.log 2>&1; echo "mgpu experts rc=$?"; tail -3 gpurun_out/overlap/t_mgpu.log
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2975$n bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/overlap/b_n$n.json 2> gpurun_out/overlap/b_n$n.err
  echo "bench n=$n rc=$?"
  python - gpurun_out/overlap/b_n$n.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
x = d.get("experts") or {}
print(d["n_gpus"], round(d["value"], 1), d["schedule"]["level"], {k: round(v["avg_us"], 1) for k, v in d["stages"].items()},
      "experts:", {k: (round(v, 1) if isinstance(v, float) else v) for k, v in x.items() if k.startswith("us_") or k == "experts_us"},
      round((x.get("roofline") or {}).get("frac", 0), 3))
PY
done
