# launch list + one --set full capture of every library kernel of a step (config $CFG)
mkdir -p gpurun_out
CFG=${CFG:-kodak}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}.csv \
    python bench.py --config $CFG --steps 30 --warmup 3 --no-cpu --no-e2e --no-profile > /dev/null 2>&1
echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:'^k_' -s 20 -c 4 -f -o gpurun_out/prof_${CFG} \
    python bench.py --config $CFG --steps 10 --warmup 5 --no-cpu --no-e2e --no-profile > /dev/null 2>&1
echo full=$?
