# GPU tests + short benches of both backward modes
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
for m in 0 1; do
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu --no-e2e --backward-mode $m > gpurun_out/bench_m$m.log 2>&1; echo bench$m=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_m$m.log').read().strip().splitlines()[-1])
print('mode $m', round(d['value'],1), 'it/s', {k: round(v*1e3,1) for k,v in d['kernel_ms_per_step'].items()}, 'frac', round(d['roofline']['frac'],3), d['render'])
"
done
