mkdir -p gpurun_out
run() {
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu --no-e2e > gpurun_out/bq.log 2>&1 || tail -20 gpurun_out/bq.log
python -c "
import json; d=json.loads(open('gpurun_out/bq.log').read().strip().splitlines()[-1])
r=d['roofline'] or {}
print('$1', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,1), 'us/step; raster', round(r.get('avg_ms',0)*1e3,1), 'us frac', round(r.get('frac',0),3), {k: round(v*1e3,1) for k,v in (d['kernel_ms_per_step'] or {}).items()})
"
}
SMOE_LIB=$PWD/paper_2510_05814_b200/libsmoe_ab.so run "A(head)"
run "B(snake occ12)"
SMOE_RASTER_CTAS_PER_SM=8 run "B(snake occ8)"
SMOE_RASTER_CTAS_PER_SM=6 run "B(snake occ6)"
SMOE_NO_LPT=1 run "B(nolpt)"
