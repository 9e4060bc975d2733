# the driver's round-end commands: default bench (N=1), the reference arm, smoke
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_default.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_reference.log 2>&1; echo ref=$?; tail -1 gpurun_out/bench_reference.log
