# r2 run 33: MPERM (permuted k-steps for one-row-block warps at odd D strides): GPU suite, A/B old/new on the tuned configurations it changes, bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
declare -a CFGS=(
 'tsmm d 19 19 {"AP": 19, "NOP": 19, "NT": 288, "PLAIN": 1, "R": 192, "WR": 1, "ctas": 1, "impl": 1, "stages": 4}'
 'tsmm d 29 29 {"AP": 29, "NOP": 29, "NT": 160, "PLAIN": 1, "R": 96, "WR": 1, "ctas": 2, "impl": 1, "stages": 3}'
 'tsmm d 35 35 {"AP": 35, "NOP": 35, "NT": 544, "R": 128, "WR": 1, "ctas": 1, "impl": 1, "stages": 4}'
 'tsmm d 37 37 {"AP": 37, "NOP": 37, "NT": 544, "R": 128, "WR": 1, "ctas": 1, "impl": 1, "stages": 4}'
 'tsmm d 39 39 {"AP": 39, "NOP": 39, "NT": 416, "R": 96, "WR": 1, "ctas": 1, "impl": 1, "stages": 4}'
 'tsmm d 41 41 {"AP": 41, "NOP": 41, "NT": 416, "R": 96, "WR": 1, "ctas": 1, "impl": 1, "stages": 4}'
 'tsmm d 43 43 {"AP": 43, "NOP": 43, "NT": 416, "R": 96, "WR": 1, "ctas": 1, "impl": 1, "stages": 4}'
 'tsmm d 45 45 {"AP": 45, "NOP": 45, "NT": 416, "R": 96, "WR": 1, "ctas": 1, "impl": 1, "stages": 4}'
 'tsmm d 51 51 {"AP": 51, "NOP": 51, "NT": 416, "R": 96, "WR": 1, "ctas": 1, "impl": 1, "stages": 4}'
 'tsmm d 53 53 {"AP": 53, "NOP": 53, "NT": 416, "R": 96, "WR": 1, "ctas": 1, "impl": 1, "stages": 4}'
 'tsmm d 55 55 {"AP": 55, "NOP": 55, "NT": 416, "R": 96, "WR": 1, "ctas": 1, "impl": 1, "stages": 3}'
 'tsmm d 59 59 {"AP": 59, "NOP": 59, "NT": 416, "R": 96, "WR": 1, "ctas": 1, "impl": 1, "stages": 3}'
 'tsmm d 61 61 {"AP": 61, "NOP": 61, "NT": 416, "R": 96, "WR": 1, "ctas": 1, "impl": 1, "stages": 3}'
 'tsmm d 63 63 {"AP": 63, "NOP": 63, "NT": 416, "R": 96, "WR": 1, "ctas": 1, "impl": 1, "stages": 3}'
)
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r33_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/r33_pytest_gpu.log
for round in 1 2; do
for c in "${CFGS[@]}"; do
  set -- $c; op=$1; dt=$2; M=$3; N=$4; shift 4; cfg="$*"
  o=$(cd oldtree && timeout 120 python tools/one_config.py $op $dt $M $N "$cfg" --reps 9 2>/dev/null | tail -1 | python -c "import json,sys; print(round(json.load(sys.stdin)['ms'],4))")
  n=$(timeout 120 python tools/one_config.py $op $dt $M $N "$cfg" --reps 9 2>/dev/null | tail -1 | python -c "import json,sys; print(round(json.load(sys.stdin)['ms'],4))")
  echo "AB $op $dt $M old $o new $n"
done
done 2>&1 | tee gpurun_out/r33_ab.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/r33_bench_report.json > gpurun_out/r33_bench.log 2>&1; echo bench rc=$?; tail -c 200 gpurun_out/r33_bench.log
