for f in 0.25 0.5 0.75; do
  for n in 2 4; do
    MONTA_AG_FRAC=$f timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29540 scripts/timeline.py --level O2 --chunks $n > gpurun_out/tlx_${f}_$n.txt 2>&1; echo $f $n rc=$?
  done
done
