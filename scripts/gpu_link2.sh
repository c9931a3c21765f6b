mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_wire.py tests/test_gpu_layer.py -k "wire or link" -x -q > gpurun_out/t_link2.log 2>&1; echo "t rc=$?"; tail -1 gpurun_out/t_link2.log
for cfg in mixtral deepseek; do for mode in "--no-persistent" "--wire fp8"; do
tag=$(echo $mode | tr -d ' -')
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2966$((RANDOM%10)) bench.py --gpus 4 --steps 10 --warmup 3 --config $cfg --link-gbs 100 --level o1 $mode > gpurun_out/lw_${cfg}_$tag.json 2> gpurun_out/lw_${cfg}_$tag.err; echo "$cfg $tag rc=$?"; tail -1 gpurun_out/lw_${cfg}_$tag.err
done; done
