mkdir -p gpurun_out
for extra in "" "--no-profile"; do
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu --no-e2e $extra > gpurun_out/bv.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bv.log').read().strip().splitlines()[-1])
print('$extra', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['kernel_ms_per_step'].items()})
"
done
