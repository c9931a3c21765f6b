#!/bin/bash
# Round-2 validation on one B200: the whole GPU suite (1-GPU tests), smoke, the
# driver-like N=1 bench (default workload), its ncu launch list, the reference arm.
mkdir -p gpurun_out/final
timeout 1800 python -m pytest tests -m "gpu and not multigpu" -x -q > gpurun_out/final/t_gpu.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/final/t_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final/bench_n1.json 2> gpurun_out/final/bench_n1.err; echo "bench rc=$?"
python - gpurun_out/final/bench_n1.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(round(d["value"], 1), d["config"]["workload"], {k: round(v["avg_us"], 1) for k, v in d["stages"].items()},
      d["roofline"]["kernel"], round(d["roofline"]["frac"], 3), "e2e", round(d["e2e"]["value"], 1), "cpu", round(d["cpu_baseline"]["value"]),
      "launches", d["gpu_launches"], d["clocks"])
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_n1.csv python bench.py --steps 2 --warmup 3 > gpurun_out/final/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/ref_n1.json 2> gpurun_out/final/ref_n1.err; echo "ref rc=$?"; tail -c 400 gpurun_out/final/ref_n1.json
