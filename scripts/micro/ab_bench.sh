# A/B: bench.py --quick with the in-tree library (A) and with each ab_alt/<name>/libmonta.so, interleaved.
#   bash scripts/micro/ab_bench.sh "old pf" [bench args...]
# ab_alt/ is git-ignored but travels with gpurun.  Prints us/layer and the per-stage span averages.
show='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(sys.argv[1], round(d["value"],2), {k: round(v["avg_us"],2) for k, v in (d.get("stages") or {}).items()})'
for r in 1 2 3; do
  timeout 200 python bench.py --steps 30 --warmup 5 --quick "${@:2}" 2>/dev/null | python -c "$show" "A(tree)"
  for b in $1; do
    MONTA_LIB=ab_alt/$b/libmonta.so timeout 200 python bench.py --steps 30 --warmup 5 --quick "${@:2}" 2>/dev/null | python -c "$show" "B($b)"
  done
done
