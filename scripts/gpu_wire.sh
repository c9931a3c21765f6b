mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py -k "fp8 or 2x2_all or two_gpus" tests/test_multigpu_backward.py -x -q > gpurun_out/t_mgpu2.log 2>&1; echo "mgpu rc=$?"; tail -3 gpurun_out/t_mgpu2.log
for cfg in deepseek mixtral; do
for mode in "--no-persistent" "--wire fp8"; do
tag=$(echo $mode | tr -d ' -')
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus 4 --steps 10 --warmup 3 --config $cfg --level o1 $mode > gpurun_out/w_${cfg}_$tag.json 2> gpurun_out/w_${cfg}_$tag.err; echo "$cfg $tag rc=$?"; tail -2 gpurun_out/w_${cfg}_$tag.err
done; done
