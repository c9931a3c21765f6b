# A/B: bench.py --quick with the in-tree library and with scripts/micro/alt_lib/$1, alternating
for r in 1 2 3; do
  timeout 200 python bench.py --steps 30 --warmup 5 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('A(tree)', round(d['value'],2))"
  MONTA_LIB=scripts/micro/alt_lib/$1 timeout 200 python bench.py --steps 30 --warmup 5 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B($1)', round(d['value'],2))"
done
