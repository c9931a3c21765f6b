timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/b_e2e.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/b_e2e.json')); print(d['value'], d['e2e'])"
