# r2 run 2: validate the round-2 fixes (e505bab) -- smoke, full GPU tests, bench, sanitizer
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke rc=$?; tail -n 3 gpurun_out/r2_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -n 5 gpurun_out/r2_pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/r2_bench_report.json > gpurun_out/r2_bench.log 2>&1; echo bench rc=$?; tail -c 600 gpurun_out/r2_bench.log
timeout 900 python tools/sanitize.py > gpurun_out/r2_san_plain.log 2>&1; echo plain rc=$?; tail -3 gpurun_out/r2_san_plain.log
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 100 python tools/sanitize.py > gpurun_out/r2_san_$tool.log 2>&1
  echo $tool rc=$?; tail -4 gpurun_out/r2_san_$tool.log
done
