# A/B of library variants, interleaved twice: VARIANTS="base old" CFGS="kodak div2k"
mkdir -p gpurun_out
for rep in 1 2; do
for cfg in ${CFGS:-kodak}; do
for v in ${VARIANTS:-base}; do
lib=$PWD/paper_2510_05814_b200/libsmoe_$v.so; [ "$v" = base ] && lib=$PWD/paper_2510_05814_b200/libsmoe.so
SMOE_LIB=$lib timeout 600 python bench.py --config $cfg --steps ${STEPS:-400} --warmup 10 --no-cpu --no-e2e $BENCH_ARGS > gpurun_out/bq.log 2>&1 || tail -5 gpurun_out/bq.log
python -c "
import json; d=json.loads(open('gpurun_out/bq.log').read().strip().splitlines()[-1])
r=d['roofline'] or {}
rr={k: round(v.get('mpix_s',0)) for k,v in (d.get('render') or {}).items()}
print('$cfg $v', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,1), 'us/step; raster', round(r.get('avg_ms',0)*1e3,1), 'us frac', round(r.get('frac',0),3), {k: round(v*1e3,1) for k,v in (d['kernel_ms_per_step'] or {}).items()}, rr)
"
done; done; done
