# r2 run 4: remaining new parity tests (strided all widths, full-size, configs[4]),
# sanitizers on the fixed code, ncu of the top kernels (default and inline-edge),
# small-K flush modes
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests/test_next_gpu.py tests/test_fullsize_gpu.py tests/test_configs4_gpu.py tests/test_kernels_gpu.py::test_tsmm_cstb_edge_columns -q > gpurun_out/r4_pytest_new.log 2>&1; echo pytest_new rc=$?; tail -n 8 gpurun_out/r4_pytest_new.log
timeout 600 python tools/sanitize.py > gpurun_out/r4_san_plain.log 2>&1; echo plain rc=$?; tail -2 gpurun_out/r4_san_plain.log
for tool in synccheck memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize.py > gpurun_out/r4_san_$tool.log 2>&1
  echo $tool rc=$?; tail -3 gpurun_out/r4_san_$tool.log
done
NCU="ncu --set full --clock-control none --import-source on -s 2 -c 1"
timeout 400 $NCU -k regex:tsmm_cstb -o gpurun_out/r4_ncu_tsmm_d_63 python tools/one_config.py tsmm d 63 63 '{"NBW": 3, "NT": 416, "PLAIN": 1, "R": 64, "WR": 1, "ctas": 1, "impl": 4, "stages": 6}' --reps 3 > gpurun_out/r4_ncu1.log 2>&1; echo ncu1 rc=$?
timeout 400 $NCU -k regex:tsmttsm_mma -o gpurun_out/r4_ncu_tsmttsm_d_57_pad python tools/one_config.py tsmttsm d 57 57 '{"AP": 57, "BP": 57, "MT": 4, "NT": 544, "NTL": 4, "PLAIN": 1, "R": 64, "ctas": 1, "impl": 1, "stages": 3}' --reps 3 > gpurun_out/r4_ncu2.log 2>&1; echo ncu2 rc=$?
timeout 400 $NCU -k regex:tsmttsm_mma -o gpurun_out/r4_ncu_tsmttsm_d_57_ei python tools/one_config.py tsmttsm d 57 57 '{"AP": 57, "BP": 57, "EI": 1, "MT": 4, "NT": 544, "NTL": 4, "R": 64, "ctas": 1, "impl": 1, "stages": 3}' --reps 3 > gpurun_out/r4_ncu3.log 2>&1; echo ncu3 rc=$?
timeout 400 $NCU -k regex:tsmm_mma -o gpurun_out/r4_ncu_tsmm_d_57 python tools/one_config.py tsmm d 57 57 '{"AP": 57, "NOP": 57, "NT": 288, "R": 128, "WR": 2, "ctas": 1, "impl": 1, "stages": 2}' --reps 3 > gpurun_out/r4_ncu4.log 2>&1; echo ncu4 rc=$?
for fl in read none; do
  timeout 300 python tools/smallk.py --widths 8,32 --Ks 1e4,1e5,1e6,1e7 --flush $fl --json gpurun_out/r4_smallk_$fl.json > gpurun_out/r4_smallk_$fl.log 2>&1; echo smallk_$fl rc=$?; cat gpurun_out/r4_smallk_$fl.log
done
