mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m "gpu and not multigpu" -x -q > gpurun_out/t_gpu.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/t_gpu.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ref1.json 2> gpurun_out/ref1.err; echo "ref rc=$?"; head -c 400 gpurun_out/ref1.json; echo
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/b_n1.json 2> gpurun_out/b_n1.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/b_n1.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], {k: round(v['avg_us'],1) for k,v in d['stages'].items()}, (d['experts'] or {}).get('roofline',{}).get('frac'))"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
