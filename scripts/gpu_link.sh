mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layer.py -k "link_rate or autotune or routing_checks" tests/test_gpu_layer_backward.py -x -q > gpurun_out/t_link.log 2>&1; echo "t rc=$?"; tail -2 gpurun_out/t_link.log
for cfg in mixtral deepseek; do for rate in 100; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2964$((RANDOM%10)) bench.py --gpus 4 --steps 10 --warmup 3 --config $cfg --link-gbs $rate > gpurun_out/link_${cfg}_$rate.json 2> gpurun_out/link_${cfg}_$rate.err; echo "link $cfg $rate rc=$?"; tail -1 gpurun_out/link_${cfg}_$rate.err
done; done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 scripts/micro/backward_layer_bench.py > gpurun_out/bwd4g.json 2> gpurun_out/bwd4g.err; echo "bwd4 rc=$?"; grep metric -v gpurun_out/bwd4g.json | tail -1
