mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:"k_grouped_gemm" -c 2 -o gpurun_out/prof_gemm_ds1 python scripts/micro/gemm_bench.py --iters 1 --cases deepseek > gpurun_out/ncu_gemm_ds1.log 2>&1; echo "ncu rc=$?"
