# ncu launch list + one full capture of each library kernel (one step's worth)
mkdir -p gpurun_out
CFG=${CFG:-kodak}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}.csv \
    python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch_bench.log 2>&1
echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:'^k_' -s 40 -c 6 -f -o gpurun_out/prof_${CFG} \
    python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_full.log 2>&1
echo full=$?
tail -3 gpurun_out/ncu_full.log
