# A/B of environment settings on one library, interleaved twice:
# ENVS="SMOE_PERM=0 SMOE_PERM=1" CFGS="kodak"
mkdir -p gpurun_out
for rep in 1 2; do
for cfg in ${CFGS:-kodak}; do
for e in ${ENVS:-X=0}; do
env $e timeout 600 python bench.py --config $cfg --steps ${STEPS:-400} --warmup 10 --no-cpu --no-e2e $BENCH_ARGS > gpurun_out/bq.log 2>&1 || tail -5 gpurun_out/bq.log
python -c "
import json; d=json.loads(open('gpurun_out/bq.log').read().strip().splitlines()[-1])
r=d['roofline'] or {}
print('$cfg $e', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,1), 'us/step; raster', round(r.get('avg_ms',0)*1e3,1), 'us', {k: round(v*1e3,1) for k,v in (d['kernel_ms_per_step'] or {}).items()})
"
done; done; done
