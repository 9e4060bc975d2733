# one ncu --set full capture of the train raster kernel (argument: backward mode)
mkdir -p gpurun_out
M=${1:-0}; CFG=${CFG:-kodak}; TAG=${TAG:-}
ncu --set full --clock-control none --import-source on -k regex:'k_raster' -s 8 -c 1 -f -o gpurun_out/raster_${CFG}_m$M$TAG \
    python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu --no-e2e --backward-mode $M > gpurun_out/ncu_raster_m$M.log 2>&1
echo ncu=$?
