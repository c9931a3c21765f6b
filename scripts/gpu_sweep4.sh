mkdir -p gpurun_out
for cfg in mixtral deepseek 70b toy; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2960$((RANDOM%10)) scripts/sweep_levels.py --config $cfg > gpurun_out/sweep_$cfg.jsonl 2> gpurun_out/sweep_$cfg.err; echo "sweep $cfg rc=$?"; tail -2 gpurun_out/sweep_$cfg.err | head -2
done
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/b_n$n.json 2> gpurun_out/b_n$n.err; echo "bench$n rc=$?"; tail -2 gpurun_out/b_n$n.err
done
