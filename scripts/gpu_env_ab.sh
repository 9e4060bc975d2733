# A/B of environment switches on one build: ENVS="X=1 Y=1" (each run with one of them, plus a baseline)
mkdir -p gpurun_out
for cfg in ${CFGS:-kodak}; do
for e in base ${ENVS}; do
if [ "$e" = base ]; then envs=""; else envs="$e"; fi
env $envs timeout 600 python bench.py --config $cfg --steps ${STEPS:-500} --warmup 10 --no-cpu --no-e2e > gpurun_out/bq.log 2>&1 || tail -5 gpurun_out/bq.log
python -c "
import json; d=json.loads(open('gpurun_out/bq.log').read().strip().splitlines()[-1])
r=d['roofline'] or {}
print('$cfg $e', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,1), 'us/step; raster', round(r.get('avg_ms',0)*1e3,1), 'us frac', round(r.get('frac',0),3), {k: round(v*1e3,1) for k,v in (d['kernel_ms_per_step'] or {}).items()})
"
done; done
