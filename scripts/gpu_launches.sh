mkdir -p gpurun_out
CFG=${CFG:-kodak}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}.csv \
    python bench.py --config $CFG --steps 30 --warmup 3 --no-cpu --no-e2e --no-profile > gpurun_out/ncu_launch_bench.log 2>&1
echo launches=$?
