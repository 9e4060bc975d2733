# A/B of library builds (SMOE_LIB) on the bench: LIBS="old new m5" CFGS="kodak div2k"
mkdir -p gpurun_out
for rep in 1 2; do
for cfg in ${CFGS:-kodak div2k}; do
for lib in ${LIBS:-old new}; do
  so=paper_2510_05814_b200/libsmoe_$lib.so; [ $lib = new ] && so=paper_2510_05814_b200/libsmoe.so
  SMOE_LIB=$so timeout 300 python bench.py --config $cfg --steps ${STEPS:-300} --warmup 10 --no-cpu --no-e2e > gpurun_out/ab.log 2>&1 || tail -5 gpurun_out/ab.log
  python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
r=d['roofline'] or {}; k=d.get('kernel_ms_per_step') or {}
print('$rep $cfg $lib', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,1), 'us; raster', round(r.get('avg_ms',0)*1e3,1), 'us frac', round(r.get('frac',0),3), {a: round(b*1e3,1) for a,b in k.items()}, 'x4' , d['render'].get('x4',{}).get('mpix_s'))
"
done; done; done
