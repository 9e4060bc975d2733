mkdir -p gpurun_out
for cfg in tiny denoise div2k 8k; do for m in 0 1; do
timeout 900 python bench.py --config $cfg --steps ${STEPS:-100} --warmup 5 --no-cpu --no-e2e --backward-mode $m > gpurun_out/bc_$cfg.log 2>&1 || tail -20 gpurun_out/bc_$cfg.log
python -c "
import json; d=json.loads(open('gpurun_out/bc_$cfg.log').read().strip().splitlines()[-1])
r=d['roofline'] or {}
print('$cfg m$m', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,1), 'us/step; raster', round(r.get('avg_ms',0)*1e3,1), 'us frac', round(r.get('frac',0),3), {k: round(v*1e3,1) for k,v in (d['kernel_ms_per_step'] or {}).items()})
"
done; done
