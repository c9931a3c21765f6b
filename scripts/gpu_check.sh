#!/bin/bash
# GPU checks used during development: parity tests, bench lines, optional ncu.
# usage: bash scripts/gpu_check.sh [tests] [mgpu] [bench1] [bench2] [bench4] [ncu1] [calib4]
mkdir -p gpurun_out
for what in "$@"; do
case $what in
  tests) timeout 900 python -m pytest tests -m "gpu and not multigpu" -x -q > gpurun_out/t_gpu.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_gpu.log;;
  mgpu) timeout 900 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/t_mgpu.log 2>&1; echo "mgpu rc=$?"; tail -3 gpurun_out/t_mgpu.log;;
  bench1) timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/b_n1.json 2> gpurun_out/b_n1.err; echo "bench1 rc=$?";;
  bench2) timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/b_n2.json 2> gpurun_out/b_n2.err; echo "bench2 rc=$?";;
  bench4) timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/b_n4.json 2> gpurun_out/b_n4.err; echo "bench4 rc=$?";;
  ncu1) timeout 300 python bench.py --steps 2 --warmup 3 --quick > gpurun_out/ncu_plain.log 2>&1 && \
        timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches.csv python bench.py --steps 2 --warmup 3 --quick > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
        timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_unpermute|k_aa_token|k_front" -s 3 -c 3 -o gpurun_out/prof_n1 python bench.py --steps 2 --warmup 3 --quick > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?";;
  ncul) timeout 300 python bench.py --steps 2 --warmup 3 --quick > gpurun_out/ncu_plain.log 2>&1 && \
        timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches.csv python bench.py --steps 2 --warmup 3 --quick > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?";;
  calib4) timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 -m paper_2411_00662_b200.calibrate --out gpurun_out/calib > gpurun_out/calib4.log 2>&1; echo "calib4 rc=$?";;
  calib8) timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29534 -m paper_2411_00662_b200.calibrate --out gpurun_out/calib > gpurun_out/calib8.log 2>&1; echo "calib8 rc=$?";;
esac
done
for what in "$@"; do
case $what in
  sweep4) timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29535 scripts/sweep_levels.py > gpurun_out/sweep4.jsonl 2> gpurun_out/sweep4.err; echo "sweep4 rc=$?";;
  sweep2) timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29536 scripts/sweep_levels.py > gpurun_out/sweep2.jsonl 2> gpurun_out/sweep2.err; echo "sweep2 rc=$?";;
esac
done
