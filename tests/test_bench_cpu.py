"""bench.py host logic on the CPU: the reference arm runs the unmodified
reference (baseline/_ref) and prints the same config dict as our arm; a
--gpus / WORLD_SIZE mismatch fails instead of timing the wrong world size."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_config_dicts():
    for cfg in bench.CONFIGS:
        w = bench.config_dict(cfg, 4, "weak")
        s = bench.config_dict(cfg, 4, "strong")
        B = bench.CONFIGS[cfg]["B"]
        assert w["global_batch"] == 4 * B and w["batch_per_gpu"] == B
        assert s["global_batch"] == B and s["batch_per_gpu"] == -(-B // 4)
        assert w["parallelism"] == "batch-dp4"


def test_peaks_are_measured():
    pk = bench._peaks()
    for k in ("fp32", "fp64", "mufu"):
        assert "measured" in pk[k][2] and pk[k][0] > 0


@pytest.mark.skipif(not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "structdist")),
                    reason="unmodified reference not installed in baseline/_ref")
def test_reference_arm_runs_unmodified_reference():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"
    assert line["config"] == bench.config_dict("c1", 1, "weak")
    assert line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0


def test_world_size_mismatch_fails():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--no-cpu"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in (out.stderr + out.stdout)
