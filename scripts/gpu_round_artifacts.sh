# Refresh every committed measurement record of the round (TAG=r02): smoke,
# GPU suite, default bench (config 3) + reference arm, the other configs, the
# box modes and the per-rank projection, f3/f4 MM runs, compute-sanitizer,
# ncu launch lists + full captures (configs 2-5).  PHASE=a|b|all splits it.
mkdir -p gpurun_out/art
TAG=${TAG:-r02}
O=gpurun_out/art
PHASE=${PHASE:-all}
if [ $PHASE = a ] || [ $PHASE = all ]; then
python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > $O/${TAG}_pytest_gpu.log 2>&1; echo pytest=$?; tail -1 $O/${TAG}_pytest_gpu.log
timeout 900 python bench.py > $O/${TAG}_bench_default.log 2>&1; echo bench=$?; tail -1 $O/${TAG}_bench_default.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $O/${TAG}_bench_reference.log 2>&1; echo ref=$?
for cfg in tiny kodak denoise 8k; do
  nocpu=""; [ $cfg = 8k ] && nocpu=--no-cpu   # the dense oracle sample is too slow at K = 10^6
  timeout 900 python bench.py --config $cfg --steps 500 --warmup 10 $nocpu > $O/bc_$cfg.log 2>&1; echo $cfg=$?
  tail -1 $O/bc_$cfg.log > $O/${TAG}_bench_$cfg.json
done
for cfg in kodak div2k denoise; do
  timeout 900 python bench.py --config $cfg --steps 200 --warmup 5 --no-cpu --no-e2e --box-modes > $O/bm_$cfg.log 2>&1; echo boxmodes_$cfg=$?
  tail -1 $O/bm_$cfg.log > $O/${TAG}_box_modes_$cfg.json
done
timeout 900 python bench.py --config 8k --project 1,2,4,8 --steps 20 --warmup 3 > $O/${TAG}_projection_8k.json 2>$O/proj.err; echo project=$?
rm -f $O/${TAG}_bench_mm_denoise.jsonl $O/${TAG}_bench_mm_seg_denoise.jsonl
for H in 1 8; do
  timeout 900 python bench.py --config denoise --mm $H --steps 2000 --warmup 5 2>/dev/null | tail -1 >> $O/${TAG}_bench_mm_denoise.jsonl
done
timeout 900 python bench.py --config denoise --mm 8 --seg 20 --steps 2000 --warmup 5 2>/dev/null | tail -1 >> $O/${TAG}_bench_mm_seg_denoise.jsonl
echo mm done
fi
if [ $PHASE = b ] || [ $PHASE = all ]; then
export PYTHONFAULTHANDLER=1
# device bounds checks of the -DSMOE_DEBUG build (in place of compute-sanitizer where the pool closed it)
make -s -C paper_2510_05814_b200/csrc variant NAME=dbg EXTRA=-DSMOE_DEBUG
SMOE_LIB=$PWD/paper_2510_05814_b200/libsmoe_dbg.so timeout 1800 python -m pytest tests -m gpu -q > $O/${TAG}_pytest_gpu_debug_checks.log 2>&1
echo debug_checks=$?; tail -1 $O/${TAG}_pytest_gpu_debug_checks.log
for tool in ${SANITIZER_TOOLS:-}; do
timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 7 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adam.py tests/test_gpu_fused_records.py -q -x \
   -k "test_grad_parity and 37 or test_render_parity and 37 or binning_large_bucket or dense_buckets or degenerate or step_matches or bucket_over or all_binners or overflow or skips_when or sharded_apply and 300 or fused_records_match and two_stage and 3-0" > $O/${TAG}_sanitizer_$tool.txt 2>&1
echo $tool=$?; tail -2 $O/${TAG}_sanitizer_$tool.txt
done
for CFG in ${NCU_CFGS:-kodak div2k denoise 8k}; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_${CFG}.csv \
    python bench.py --config $CFG --steps 30 --warmup 3 --no-cpu --no-e2e --no-profile > /dev/null 2>&1
echo launches_$CFG=$?
ncu --set full --clock-control none --import-source on -k regex:'^k_' -s 20 -c 5 -f -o $O/prof_${CFG} \
    python bench.py --config $CFG --steps 10 --warmup 5 --no-cpu --no-e2e --no-profile > /dev/null 2>&1
echo full_$CFG=$?
SMOE_PROFILES_DIR=$O/profiles python scripts/ncu_summary.py ${TAG}_ncu_${CFG} $CFG $O/${TAG}_launches_${CFG}.csv $O/prof_${CFG}.ncu-rep > /dev/null 2>&1; echo summary_$CFG=$?
[ $CFG = div2k ] || rm -f $O/prof_${CFG}.ncu-rep
done
fi
du -sh $O
