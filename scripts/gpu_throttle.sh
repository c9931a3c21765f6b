# B1-throttled regime (cross-node AllToAll legs capped) at 2x2 + EP>DP gate contention
mkdir -p gpurun_out
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 scripts/micro/priority_bench.py --config mixtral > gpurun_out/prio4g.json 2> gpurun_out/prio4g.err; echo "prio4 rc=$?"; cat gpurun_out/prio4g.json
for cfg in deepseek mixtral; do for cap in 8 16; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2957$cap bench.py --gpus 4 --steps 10 --warmup 3 --config $cfg --level o1 --aa-ctas $cap > gpurun_out/thr_${cfg}_$cap.json 2> gpurun_out/thr_${cfg}_$cap.err; echo "thr $cfg $cap rc=$?"; tail -2 gpurun_out/thr_${cfg}_$cap.err
done; done
