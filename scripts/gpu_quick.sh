# GPU tests + short benches of both backward modes
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log | grep -vE "^\s*$" | tail -4
for extra in "--backward-mode 0" "--backward-mode 1"; do
timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu --no-e2e $extra > gpurun_out/bq.log 2>&1 || tail -20 gpurun_out/bq.log
python -c "
import json; d=json.loads(open('gpurun_out/bq.log').read().strip().splitlines()[-1])
r=d['roofline'] or {}
print('$extra', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,1), 'us/step; raster', round(r.get('avg_ms',0)*1e3,1), 'us frac', round(r.get('frac',0),3), {k: round(v*1e3,1) for k,v in (d['kernel_ms_per_step'] or {}).items()}, d['render'].get('x1',{}).get('mpix_s'))
"
done
