# r2 run 3: new parity tests (every tuned plan at full size, configs[4] at K=2^28,
# cstb edge columns), the new bench line, small-K study, autotune of the cstb
# edge-column candidates (TSMM D), inline-edge TSMTTSM D 41-63 best configs
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; free -g | head -2
timeout 1500 python -m pytest tests/test_kernels_gpu.py::test_tsmm_cstb_edge_columns tests/test_next_gpu.py tests/test_fullsize_gpu.py tests/test_configs4_gpu.py -q -x > gpurun_out/r3_pytest_new.log 2>&1; echo pytest_new rc=$?; tail -n 5 gpurun_out/r3_pytest_new.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/r3_bench_report.json > gpurun_out/r3_bench.log 2>&1; echo bench rc=$?; tail -c 3000 gpurun_out/r3_bench.log
timeout 600 python tools/smallk.py --json gpurun_out/r3_smallk.json > gpurun_out/r3_smallk.log 2>&1; echo smallk rc=$?; tail -n 40 gpurun_out/r3_smallk.log
W=$(python -c "print(','.join(str(i) for i in range(9,64) if i % 8))")
timeout 1800 python tools/autotune.py --ops tsmm --dtypes d --widths $W --filter "c.get('impl')==4 and c.get('EDGE')" --out gpurun_out/r3_tune_cstb_ec.json > gpurun_out/r3_tune_cstb_ec.log 2>&1; echo tune_ec rc=$?; tail -n 60 gpurun_out/r3_tune_cstb_ec.log
W2=$(python -c "print(','.join(str(i) for i in range(41,64) if i % 8))")
timeout 1200 python tools/autotune.py --ops tsmttsm --dtypes d --widths $W2 --filter "c.get('EI')" --out gpurun_out/r3_tune_ei.json > gpurun_out/r3_tune_ei.log 2>&1; echo tune_ei rc=$?; tail -n 30 gpurun_out/r3_tune_ei.log
