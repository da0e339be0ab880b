bash tools/ncu_run.sh r01b tsmttsm d 48x48 64x64
bash tools/ncu_run.sh r01b tsmttsm z 33x33 48x48
bash tools/ncu_run.sh r01b tsmm d 64x64 41x41
timeout 900 python bench.py --steps 3 --warmup 3 --report gpurun_out/bench_report12.json > gpurun_out/bench12.log 2>&1; echo bench rc=$?; head -c 800 gpurun_out/bench12.log
