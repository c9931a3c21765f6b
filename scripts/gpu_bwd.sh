mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layer_backward.py tests/test_gpu_layer.py tests/test_gpu_experts.py -x -q > gpurun_out/t_bwd.log 2>&1; echo "t rc=$?"; tail -3 gpurun_out/t_bwd.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 scripts/micro/backward_layer_bench.py > gpurun_out/bwd4.json 2> gpurun_out/bwd4.err; echo "bwd4 rc=$?"; cat gpurun_out/bwd4.json; tail -3 gpurun_out/bwd4.err
timeout 1200 python -m pytest tests/test_multigpu.py tests/test_multigpu_backward.py -x -q > gpurun_out/t_mgpu.log 2>&1; echo "mgpu rc=$?"; tail -3 gpurun_out/t_mgpu.log
