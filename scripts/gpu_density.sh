# backward-form crossover: kernel-parallel vs pixel-parallel at rising density (config 4 geometry)
mkdir -p gpurun_out
for K in ${KS:-20000 40000 80000}; do
for m in 0 1; do
timeout 300 python bench.py --config denoise --K $K --steps 200 --warmup 10 --no-cpu --no-e2e --no-profile --backward-mode $m > gpurun_out/bq.log 2>&1 || tail -5 gpurun_out/bq.log
python -c "
import json; d=json.loads(open('gpurun_out/bq.log').read().strip().splitlines()[-1])
r=d['roofline'] or {}
print('K=$K m$m', round(d['value'],1), 'it/s raster', round(r.get('avg_ms',0)*1e3,1), 'kbar', round(d['fit_stats']['avg_kernels_per_block'],1))
"
done; done
