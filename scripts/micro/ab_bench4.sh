# A/B on 4 GPUs (torchrun): in-tree library (A) vs ab_alt/<name>/libmonta.so, interleaved.
#   bash scripts/micro/ab_bench4.sh "head" [bench args...]
show='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(sys.argv[1], round(d["value"],2), {k: round(v,1) for k, v in (d.get("roles_busy_us") or {}).items()})'
run='python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1'
for r in 1 2; do
  timeout 300 $run --master-port 2958$r bench.py --gpus 4 --steps 20 --warmup 5 --quick "${@:2}" 2>/dev/null | python -c "$show" "A(tree)"
  for b in $1; do
    MONTA_LIB=ab_alt/$b/libmonta.so timeout 300 $run --master-port 2959$r bench.py --gpus 4 --steps 20 --warmup 5 --quick "${@:2}" 2>/dev/null | python -c "$show" "B($b)"
  done
done
