mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
for tool in memcheck racecheck synccheck initcheck; do
timeout 1500 compute-sanitizer --tool $tool --print-limit 200 --error-exitcode 7 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adam.py -q -x \
   -k "test_grad_parity and 37 or test_render_parity and 37 or binning_large_bucket or dense_buckets or degenerate or step_matches or bucket_over or all_binners or overflow or skips_when or sharded_apply and 300" > gpurun_out/san_$tool.log 2>&1
echo $tool=$?; tail -4 gpurun_out/san_$tool.log
done
