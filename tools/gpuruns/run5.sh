bash tools/ncu_run.sh r01a tsmm d 8x8 32x32 64x64
bash tools/ncu_run.sh r01a tsmttsm d 32x32 64x64 1x1
timeout 900 python -m pytest tests -m gpu -q -k "jit or explicit or bad_config or full_size_tsmm or determinism or walsh or nan or error" > gpurun_out/pytest_gpu4.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu4.log
