# 2/4-GPU checks: multi-GPU parity (incl. experts), EP>DP priority contention, N=2/N=4 bench lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_multigpu.py tests/test_multigpu_backward.py -x -q > gpurun_out/t_mgpu.log 2>&1; echo "mgpu rc=$?"; tail -3 gpurun_out/t_mgpu.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 scripts/micro/priority_bench.py --config mixtral > gpurun_out/prio2.json 2> gpurun_out/prio2.err; echo "prio2 rc=$?"; cat gpurun_out/prio2.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 scripts/micro/priority_bench.py --config mixtral > gpurun_out/prio4.json 2> gpurun_out/prio4.err; echo "prio4 rc=$?"; cat gpurun_out/prio4.json
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/b_n$n.json 2> gpurun_out/b_n$n.err; echo "bench$n rc=$?"; head -c 600 gpurun_out/b_n$n.json; echo; tail -2 gpurun_out/b_n$n.err
done
