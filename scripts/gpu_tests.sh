mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q "$@" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_gpu.log | grep -vE "^\s*$" | tail -25
