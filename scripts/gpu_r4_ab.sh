# four-pixels-per-lane rasters: parity under SMOE_RASTER4=1 / SMOE_RENDER4=1, then A/B on the bench
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_raster_forms.py -m gpu -q -p no:cacheprovider > gpurun_out/pt_forms.log 2>&1; echo forms=$?; tail -3 gpurun_out/pt_forms.log
SMOE_RASTER4=1 SMOE_RENDER4=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adam.py tests/test_gpu_multirank.py -m gpu -q -p no:cacheprovider -k "grad or fit or step or sampled or bucket or rbf or dense or degenerate or single_kernel or band or trajectory or two_ranks or checkpoint or multimodel or binners or box_mode_pixels or render or sharpen" > gpurun_out/pt_r4.log 2>&1; echo pytest_r4=$?; grep -E "passed|failed|FAILED" gpurun_out/pt_r4.log | tail -12
for rep in 1 2; do
for cfg in ${CFGS:-kodak div2k denoise 8k}; do
for v in "0 0" "1 0" "1 1"; do
  set -- $v
  SMOE_RASTER4=$1 SMOE_RENDER4=$2 timeout 600 python bench.py --config $cfg --steps ${STEPS:-200} --warmup 10 --no-cpu --no-e2e > gpurun_out/ab.log 2>&1 || tail -3 gpurun_out/ab.log
  python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
r=d['roofline'] or {}; k=d.get('kernel_ms_per_step') or {}
print('$rep $cfg r4=$1 render4=$2', round(d['value'],1), 'it/s', round(d['ms_per_step']*1e3,1), 'us; raster', round(r.get('avg_ms',0)*1e3,1), 'frac', round(r.get('frac',0),3), {a: round(b*1e3,1) for a,b in k.items()}, {s: round(x['mpix_s']) for s,x in d['render'].items()})
"
done; done; done
