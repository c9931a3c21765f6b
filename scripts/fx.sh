for c in 74 37; do
  echo "### MONTA_OVL_CTAS=$c"
  MONTA_OVL_CTAS=$c timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2976$((c % 10)) scripts/overlap_timeline.py 1 4 8 2>&1 | grep -v "^\*\|OMP\|Warn\|NCCL" | grep "==\|unpermute\|experts\|caa" | tail -40
done
