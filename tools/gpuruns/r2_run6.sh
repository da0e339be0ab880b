# r2 run 6: validate the 16-row windows / NCP change, synccheck on the fixed
# barrier, retune TSMM D (windows apply to kernels 1 / 4 with odd widths, NCP to kernel 1),
# the bench (plain and through the NCCL communicator path at world 1)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "win16 or cstb_edge or every_family or tsmm_3m" > gpurun_out/r6_pytest.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/r6_pytest.log
timeout 700 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize.py > gpurun_out/r6_san_synccheck.log 2>&1; echo synccheck rc=$?; tail -3 gpurun_out/r6_san_synccheck.log
W=$(python -c "print(','.join(str(i) for i in list(range(9,33,2)) + list(range(33,65))))")
timeout 1500 python tools/autotune.py --ops tsmm --dtypes d --widths $W --time-budget 1400 --out gpurun_out/r6_tune_tsmm_d.json > gpurun_out/r6_tune_tsmm_d.log 2>&1; echo tune rc=$?
python tools/merge_tune.py gpurun_out/r6_tune_tsmm_d.json --dry | tail -60
timeout 600 python bench.py --force-comm --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/r6_bench_comm.log 2>&1; echo bench_comm rc=$?; tail -c 1500 gpurun_out/r6_bench_comm.log
