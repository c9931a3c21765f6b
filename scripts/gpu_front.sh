# front-kernel phase stamps + one ncu --set full capture of the N=1 DeepSeek step's kernels
mkdir -p gpurun_out
timeout 300 python scripts/front_debug.py > gpurun_out/front_debug.txt 2>&1; echo "front_debug rc=$?"; cat gpurun_out/front_debug.txt
timeout 300 python bench.py --steps 2 --warmup 3 --quick > gpurun_out/ncu_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_front|k_aa_token|k_unpermute" -s 3 -c 3 -o gpurun_out/prof_ds_n1 python bench.py --steps 2 --warmup 3 --quick > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_grouped_gemm" -c 2 -o gpurun_out/prof_gemm python scripts/micro/gemm_bench.py --iters 1 --cases deepseek_ep4 > gpurun_out/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"; tail -3 gpurun_out/ncu_gemm.log
