# r33: fused peer-memory reduction (N3) -- GPU tests, bench path check (world 1), small-K timing of the fused path
timeout 900 python -m pytest tests/test_peer_gpu.py -m gpu -q -x > gpurun_out/pytest_peer33.log 2>&1; echo pytest-peer rc=$?; tail -n 30 gpurun_out/pytest_peer33.log
timeout 600 python bench.py --steps 2 --warmup 3 --force-comm --peer --no-e2e --no-cpu > gpurun_out/bench33_peer.log 2>&1; echo bench-peer rc=$?; tail -c 300 gpurun_out/bench33_peer.log
