# Every BASELINE workload at N=1 and N=4 (dev: fills DESIGN's per-config table).
mkdir -p gpurun_out
for c in toy mixtral 70b deepseek; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/cfg_${c}_n1.json 2> gpurun_out/cfg_${c}_n1.err; echo "$c n1 rc=$?"
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2956${#c} bench.py --gpus 4 --config $c --steps 10 --warmup 3 > gpurun_out/cfg_${c}_n4.json 2> gpurun_out/cfg_${c}_n4.err; echo "$c n4 rc=$?"
done
python - <<'PY'
import json
for c in ("toy", "mixtral", "70b", "deepseek"):
    for n in (1, 4):
        try:
            d = json.loads(open(f"gpurun_out/cfg_{c}_n{n}.json").read().strip().splitlines()[-1])
        except Exception as exc:
            print(c, n, "FAILED", exc); continue
        nv = (d.get("naive") or {})
        print(f"{c:9s} N={n} {d['config']['topology']} {d['schedule']['level']:8s} {d['value']:9.1f} us  naive {nv.get('us_per_layer')}  "
              f"exposedAA {d.get('exposed_alltoall_us')} / {nv.get('exposed_alltoall_us')}  roofline {d['roofline']['bound']} {d['roofline']['frac']:.2f}  "
              f"cpu {(d.get('cpu_baseline') or {}).get('value')}  e2e {(d.get('e2e') or {}).get('value')}")
PY
