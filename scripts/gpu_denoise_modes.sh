mkdir -p gpurun_out
for m in 0 1; do
timeout 300 python bench.py --config denoise --steps 300 --warmup 10 --no-cpu --no-e2e --backward-mode $m > gpurun_out/bq.log 2>&1 || tail -5 gpurun_out/bq.log
python -c "
import json; d=json.loads(open('gpurun_out/bq.log').read().strip().splitlines()[-1])
r=d['roofline'] or {}
print('denoise m$m', round(d['value'],1), 'it/s raster', round(r.get('avg_ms',0)*1e3,1))
"
done
ncu --set full --clock-control none --import-source on -k regex:k_raster -s 8 -c 1 -f -o gpurun_out/prof_raster_kodak_c python bench.py --config kodak --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu.log 2>&1; echo ncu=$?
