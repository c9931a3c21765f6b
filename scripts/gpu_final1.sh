mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m "gpu and not multigpu" -x -q > gpurun_out/t_gpu.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/t_gpu.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ref1.json 2> gpurun_out/ref1.err; echo "ref rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/ref1.json')); print(d['value'], d['cpu_baseline'])"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
