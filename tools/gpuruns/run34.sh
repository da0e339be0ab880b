# r34: N3 small-K fixed costs at world 1 (local / NCCL allreduce / fused peer); ncu of the edge-warp kernels (Z 17 3M+edge, D 41 edge)
timeout 900 python tools/peer_time.py --json gpurun_out/peer_time34.json > gpurun_out/peer_time34.log 2>&1; echo peer-time rc=$?; tail -n 4 gpurun_out/peer_time34.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tsmttsm -s 2 -c 1 -o gpurun_out/r34_tsmttsm_z_17x17_g3edge python tools/one_config.py tsmttsm z 17 17 '{"MT": 1, "NTL": 2, "NT": 288, "R": 32, "impl": 1, "AP": 17, "BP": 17, "EDGE": 4, "G3": 1, "stages": 4, "ctas": 2}' --reps 3 > gpurun_out/r34_z17.log 2>&1; echo ncu-z17 rc=$?
bash tools/ncu_run.sh r34 tsmttsm d 41x41
