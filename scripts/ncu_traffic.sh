#!/bin/bash
# ncu --set full of the N=1 forward kernels (front, token-side permute, un-permute) for every
# BASELINE workload; scripts/ncu_traffic.py turns the reports into profiles/ncu_traffic.json.
mkdir -p gpurun_out
for c in toy mixtral 70b deepseek; do
  timeout 300 python bench.py --config $c --steps 2 --warmup 3 --quick > gpurun_out/ncu_plain_$c.log 2>&1 || { echo "$c plain failed"; continue; }
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_unpermute|k_aa_token|k_aa_bulk|k_front" -s 3 -c 3 \
    -o gpurun_out/fwd_$c python bench.py --config $c --steps 2 --warmup 3 --quick > gpurun_out/ncu_$c.log 2>&1
  echo "$c ncu rc=$?"
done
