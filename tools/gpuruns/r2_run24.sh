# r2 run 24: bench with the end-of-step L2 drain; sanitizers over every family on the final kernels / tables
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/r24_bench_report.json > gpurun_out/r24_bench.log 2>&1; echo bench rc=$?; tail -c 300 gpurun_out/r24_bench.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize.py > gpurun_out/r24_san_$tool.log 2>&1
  echo $tool rc=$?; grep -h "SANITIZE_OK\|ERROR SUMMARY\|RACECHECK SUMMARY" gpurun_out/r24_san_$tool.log
done
