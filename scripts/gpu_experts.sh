mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_experts.py -x -q > gpurun_out/t_experts.log 2>&1; echo "experts rc=$?"; tail -30 gpurun_out/t_experts.log
if [ "$1" = "all" ]; then timeout 900 python -m pytest tests -m "gpu and not multigpu" -x -q > gpurun_out/t_gpu.log 2>&1; echo "gpu rc=$?"; tail -5 gpurun_out/t_gpu.log; fi
if [ "$1" = "bench" ]; then timeout 300 python scripts/micro/gemm_bench.py --iters 10 > gpurun_out/gemm_bench.jsonl 2>&1; echo "bench rc=$?"; cat gpurun_out/gemm_bench.jsonl | tail -8; fi
