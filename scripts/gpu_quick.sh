mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not multigpu" -x -q > gpurun_out/t_gpu.log 2>&1; echo "gpu rc=$?"; tail -5 gpurun_out/t_gpu.log
timeout 300 python scripts/front_debug.py > gpurun_out/front_debug.txt 2>&1; grep -E "E=160|E=8" gpurun_out/front_debug.txt | head -4 | cut -c1-60
timeout 300 python bench.py --steps 20 --warmup 5 --quick > gpurun_out/b_q.json 2>gpurun_out/b_q.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/b_q.json')); print(d['value'], {k: round(v['avg_us'],1) for k,v in d['stages'].items()})"
