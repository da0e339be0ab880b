# r42: inline-edge TSMTTSM over the wider candidate space (keep-better against the stored autotune times)
cp tune/b200.json gpurun_out/b200_r42.json
timeout 1500 python tools/autotune.py --ops tsmttsm --dtypes d --widths 33,34,35,36,41,42,43,44,49,50,51,52,57,58,59,60 --filter "c.get('EI')" --keep-better --time-budget 1300 --out gpurun_out/b200_r42.json > gpurun_out/autotune42d.log 2>&1; echo autotune-d rc=$?
timeout 1500 python tools/autotune.py --ops tsmttsm --dtypes z --widths 17,18,19,20,25,26,27,28,33,34,35,36,41,42,43,44 --filter "c.get('EI')" --keep-better --time-budget 1300 --out gpurun_out/b200_r42.json > gpurun_out/autotune42z.log 2>&1; echo autotune-z rc=$?
