# env A/B: ENVS="A=1 B=2" (space-separated NAME=VALUE settings, 'none' = baseline)
mkdir -p gpurun_out
for cfg in ${CFGS:-8k}; do
for ev in ${ENVS:-none}; do
if [ "$ev" = none ]; then envset=""; else envset="$ev"; fi
env $envset timeout 600 python bench.py --config $cfg --steps ${STEPS:-100} --warmup 5 --no-cpu --no-e2e > gpurun_out/bq.log 2>&1 || tail -5 gpurun_out/bq.log
python -c "
import json; d=json.loads(open('gpurun_out/bq.log').read().strip().splitlines()[-1])
r=d['roofline'] or {}
print('$cfg $ev', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,1), 'us/step; raster', round(r.get('avg_ms',0)*1e3,1), {k: round(v*1e3,1) for k,v in (d['kernel_ms_per_step'] or {}).items()}, {k: round(v.get('mpix_s',0)) for k,v in d['render'].items()})
"
done; done
