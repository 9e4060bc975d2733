# iteration helper: GPU tests (optional), short benches, optional ncu raster capture
mkdir -p gpurun_out
if [ "${TESTS:-1}" = 1 ]; then
timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log | grep -vE "^\s*$" | tail -4
fi
for cfg in ${CFGS:-kodak}; do
timeout 300 python bench.py --config $cfg --steps ${STEPS:-500} --warmup 10 --no-cpu --no-e2e > gpurun_out/bq.log 2>&1 || tail -20 gpurun_out/bq.log
python -c "
import json; d=json.loads(open('gpurun_out/bq.log').read().strip().splitlines()[-1])
r=d['roofline'] or {}
print('$cfg', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,1), 'us/step; raster', round(r.get('avg_ms',0)*1e3,1), 'us frac', round(r.get('frac',0),3), {k: round(v*1e3,1) for k,v in (d['kernel_ms_per_step'] or {}).items()}, {k: round(v.get('mpix_s',0)) for k,v in d['render'].items()})
"
done
if [ -n "$NCU" ]; then
ncu --set full --clock-control none --import-source on -k regex:"$NCU" -s 8 -c 1 -f -o gpurun_out/prof_$NCU_TAG \
    python bench.py --config ${NCU_CFG:-kodak} --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu.log 2>&1
echo ncu=$?
fi
