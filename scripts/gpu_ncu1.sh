mkdir -p gpurun_out
timeout 300 python bench.py --steps 2 --warmup 3 --quick > gpurun_out/ncu_plain.log 2>&1; echo "plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1.csv python bench.py --steps 2 --warmup 3 --quick > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_front|k_aa_token|k_unpermute" -s 3 -c 3 -o gpurun_out/prof_ds_n1b python bench.py --steps 2 --warmup 3 --quick > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
