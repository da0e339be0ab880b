set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python tools/sanitize.py > gpurun_out/r2_san_plain.log 2>&1; echo plain rc=$?
tail -3 gpurun_out/r2_san_plain.log
for tool in memcheck synccheck racecheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 100 python tools/sanitize.py > gpurun_out/r2_san_$tool.log 2>&1
  echo $tool rc=$?
  tail -4 gpurun_out/r2_san_$tool.log
done
