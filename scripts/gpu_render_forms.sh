mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_raster_forms.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "render or forms or multimodel or sampled or sharpen or rbf" > gpurun_out/pt_rf.log 2>&1; echo pytest=$?; grep -E "passed|failed|FAILED" gpurun_out/pt_rf.log | tail -6
for cfg in kodak div2k denoise 8k; do for f in 0 1 auto; do
  if [ $f = auto ]; then unset SMOE_RENDER4; else export SMOE_RENDER4=$f; fi
  timeout 600 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu --no-e2e --no-profile > gpurun_out/rf.log 2>&1 || tail -3 gpurun_out/rf.log
  python -c "
import json; d=json.loads(open('gpurun_out/rf.log').read().strip().splitlines()[-1]); print('$cfg render4=$f', {s: round(x['mpix_s']) for s,x in d['render'].items()})"
done; done
