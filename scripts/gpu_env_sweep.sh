# A/B an environment knob of the library on the bench: VAR=SMOE_PRE_TPK VALS="1 2 4 8" CFGS="kodak"
mkdir -p gpurun_out
for rep in 1 2; do
for cfg in ${CFGS:-kodak}; do
for v in ${VALS}; do
  env $VAR=$v timeout 300 python bench.py --config $cfg --steps ${STEPS:-300} --warmup 10 --no-cpu --no-e2e > gpurun_out/sw.log 2>&1 || tail -5 gpurun_out/sw.log
  python -c "
import json; d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1])
r=d['roofline'] or {}; k=d.get('kernel_ms_per_step') or {}
print('$rep $cfg $VAR=$v', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,1), 'us; raster', round(r.get('avg_ms',0)*1e3,1), {a: round(b*1e3,1) for a,b in k.items()})
"
done; done; done
