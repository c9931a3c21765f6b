mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_experts.py -x -q > gpurun_out/t_experts.log 2>&1; echo "experts rc=$?"; tail -30 gpurun_out/t_experts.log
timeout 300 python scripts/micro/gemm_bench.py --iters 10 > gpurun_out/gemm_bench.jsonl 2>&1; echo "bench rc=$?"; cat gpurun_out/gemm_bench.jsonl | tail -8
