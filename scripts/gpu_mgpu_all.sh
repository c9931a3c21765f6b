mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_wire.py -x -q > gpurun_out/t_wire.log 2>&1; echo "wire rc=$?"; tail -2 gpurun_out/t_wire.log
timeout 1500 python -m pytest tests/test_multigpu.py tests/test_multigpu_backward.py -x -q > gpurun_out/t_mgpu.log 2>&1; echo "mgpu rc=$?"; tail -3 gpurun_out/t_mgpu.log
