export SMOE_RASTER4=1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_adam.py tests/test_gpu_multirank.py -m gpu -q -p no:cacheprovider -k "grad or fit or step or sampled or bucket or rbf or dense or degenerate or single_kernel or band or trajectory or two_ranks or checkpoint or multimodel or binners or box_mode_pixels" > gpurun_out/pt_r4.log 2>&1; echo pytest_r4=$?; grep -E "passed|failed|FAILED" gpurun_out/pt_r4.log | tail -8
unset SMOE_RASTER4
cp paper_2510_05814_b200/libsmoe.so paper_2510_05814_b200/libsmoe_base.so
LIBS="base r4 r4m10 r4m14" CFGS="kodak div2k denoise 8k" STEPS=200 bash scripts/gpu_ab_libs.sh 2>&1 | grep -v "^ \|Trace\|json"
