# ncu --set full of one train-raster launch with source correlation, exported
# on the box to CSV (raw metrics + per-SASS-line source page); CFG=div2k
mkdir -p gpurun_out
CFG=${CFG:-div2k}; TAG=${TAG:-cur}; K=${KREGEX:-k_raster}
ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-8} -c 1 -f -o gpurun_out/src_${CFG}_$TAG \
    python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu --no-e2e --no-profile > gpurun_out/ncu_src.log 2>&1
echo ncu=$?
ncu -i gpurun_out/src_${CFG}_$TAG.ncu-rep --page raw --csv > gpurun_out/src_${CFG}_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/src_${CFG}_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${CFG}_${TAG}_sass.csv 2>/dev/null
ncu -i gpurun_out/src_${CFG}_$TAG.ncu-rep --page details --csv > gpurun_out/src_${CFG}_${TAG}_details.csv 2>/dev/null
ls -la gpurun_out/src_${CFG}_${TAG}*
