"""bench.py contract checks that need no GPU: the reference arm (the CPU
oracle, bench.py --impl reference) prints one JSON line with the fields the
driver reads, and under torchrun only rank 0 prints."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                         text=True, env=e, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return [l for l in out.stdout.splitlines() if l.strip()]


def test_reference_arm_json_line():
    lines = run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-k", "4096"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("configs[1] sweep")


def test_reference_arm_only_rank0_prints():
    lines = run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-k", "4096", "--gpus", "2"],
                env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert lines == []


def _bench_module():
    import importlib.util
    spec = importlib.util.spec_from_file_location("_bench", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_tile_work_counts_blocks_by_hand():
    """bench.tile_work: executed multiply-adds per useful one, counted by hand
    from the block structure (8 x 8 DMMA blocks of C; 4-deep k-steps x 8
    columns for TSMM; L-blocks; DFMA edges as useful work)."""
    tw = _bench_module().tile_work
    assert tw("tsmttsm", 8, 8, False, "dfma") == 1.0
    assert tw("tsmttsm", 64, 64, False, "dmma+tma+pair") == 1.0
    # D 42 padded: 6 x 6 blocks; L-blocks: 5 x 5 core blocks + max(ceil(40/6), ceil(40/6)) = 7
    assert abs(tw("tsmttsm", 42, 42, False, "dmma") - 36 * 64 / 42 ** 2) < 1e-12
    assert abs(tw("tsmttsm", 42, 42, False, "dmma+l-blocks") - 32 * 64 / 42 ** 2) < 1e-12
    # D 49 with DFMA edge warps: the 49^2 - 48^2 edge cells are executed unpadded
    assert tw("tsmttsm", 49, 49, False, "dmma+dfma-edgex4") == 1.0
    # TSMM D 63: 16 k-steps of 4 rows of C x 8 blocks of 8 columns
    assert abs(tw("tsmm", 63, 63, False, "dmma(p0=WR,p1=AP,p2=NOP)") - 64 * 64 / 63 ** 2) < 1e-12
    # TSMM D 41 with DFMA edge columns: 44 x 40 by DMMA + the 41 x 1 edge column
    assert abs(tw("tsmm", 41, 41, False, "dmma-cstationary+bulk+dfma-edge-columns") - (44 * 40 + 41) / 41 ** 2) < 1e-12
    # complex-as-real: the real kernel on 2M x 2N
    assert abs(tw("tsmttsm", 13, 13, True, "dmma+complex-as-real(2Mx2N)") - 32 * 32 / 26 ** 2) < 1e-12
