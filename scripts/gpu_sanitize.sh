# compute-sanitizer over the product kernels: memcheck / racecheck / synccheck on small
# single-GPU layer runs (virtual 2x2 incl. experts and the device-side backward) and
# memcheck on a 2-process NVLink run (--target-processes all)
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="test_gpu_layer.py::test_dispatch_chunked test_gpu_layer.py::test_routing_checks_pass_and_catch_corruption test_gpu_layer_backward.py::test_ctx_backward_device_side test_gpu_experts.py::test_layer_with_experts test_gpu_kernels.py::test_route_topk_signed_zero_ties"
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 20 --target-processes all python -m pytest -x -q -p no:cacheprovider $(for s in $SEL; do echo tests/$s; done) -k "2-2-8 or signed or 1-1-160" > gpurun_out/sanitize/$tool.log 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize/$tool.log | tail -3
done
timeout 1200 $CS --tool memcheck --error-exitcode 9 --target-processes all python -m pytest -x -q tests/test_multigpu.py -k "two_gpus" > gpurun_out/sanitize/memcheck_2gpu.log 2>&1; echo "memcheck 2gpu rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize/memcheck_2gpu.log | tail -4
