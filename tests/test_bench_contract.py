"""bench.py keeps the driver's contract: one JSON line with the required
keys, on the small parity configuration (the reference arm on the CPU here,
our arm on the GPU)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"]


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                       capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    j = _run("--impl", "reference", "--steps", "1", "--warmup", "0",
             "--config", "llama2-4k-1layer")
    for k in BASE + ["impl", "cpu_baseline"]:
        assert k in j, k
    assert j["impl"] == "reference" and j["value"] > 0
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["cpu_baseline"]["kind"] == "port"
    assert j["config"]["workload"] == "llama2-4k-1layer"


@pytest.mark.gpu
def test_our_arm_line():
    j = _run("--config", "llama2-4k-1layer", "--steps", "5", "--warmup", "3",
             "--no-cpu-baseline", "--no-encode")
    for k in BASE + ["roofline", "gpu_launches", "clocks", "f16_value_codebook_mode"]:
        assert k in j, k
    r = j["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] == pytest.approx(
        r["achieved"] / r["peak"])
    e = j["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert j["gpu_launches"] == 5 and j["n_gpus"] == 1 and j["higher_is_better"] is True
    assert "NOT flushed" in j["config"]["l2"]  # 16.8 MB of codes: an L2-resident figure
