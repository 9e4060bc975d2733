# GPU test suite (all failures, slowest durations) + the default bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=15 -p no:cacheprovider "$@" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -25
grep -A18 "slowest" gpurun_out/pytest_gpu.log | head -20
timeout 900 python bench.py --steps 200 --warmup 5 --no-cpu > gpurun_out/bench_default.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_default.log | cut -c1-3000
