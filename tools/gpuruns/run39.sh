# r39: retune TSMM D 33..64 after the cstb row-permutation change (keep-better against the stored autotune times)
cp tune/b200.json gpurun_out/b200_r39.json
timeout 1500 python tools/autotune.py --ops tsmm --dtypes d --widths 33-64 --keep-better --time-budget 1300 --out gpurun_out/b200_r39.json > gpurun_out/autotune39.log 2>&1; echo autotune rc=$?
