#!/bin/bash
# Round-2 multi-GPU validation on 4 B200s: the multi-GPU suite and the N=2 / N=4 bench lines.
mkdir -p gpurun_out/mfinal
timeout 2400 python -m pytest tests -m multigpu -x -q > gpurun_out/mfinal/t_mgpu.log 2>&1; echo "mgpu rc=$?"; tail -3 gpurun_out/mfinal/t_mgpu.log
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2985$n bench.py --gpus $n > gpurun_out/mfinal/bench_n$n.json 2> gpurun_out/mfinal/bench_n$n.err
  echo "bench n=$n rc=$?"
  python - gpurun_out/mfinal/bench_n$n.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
x = d.get("experts") or {}
print(d["n_gpus"], round(d["value"], 1), d["schedule"]["level"], {k: round(v["avg_us"], 1) for k, v in d["stages"].items()},
      "e2e", round(d["e2e"]["value"], 1), "experts", round(x.get("us_per_layer_with_experts", 0), 1), round(x.get("us_per_layer_with_experts_no_overlap") or 0, 1))
PY
done
