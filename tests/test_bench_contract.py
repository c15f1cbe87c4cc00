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


def test_launcher_two_ranks_shard_plan():
    """`bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks
    (torch.distributed.run); --dry-run does the rendezvous on gloo and prints
    every rank's shard plan: batch sharding for config 2 (weak), KV heads
    [0, 4) / [4, 8) for config 3, token halves for config 4 with the recent
    window on the last rank."""
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--dry-run"], capture_output=True, text=True, cwd=ROOT, timeout=300,
                       env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    j = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert j["n_gpus"] == 2 and len(j["plans"]) == 2
    by = {(p["rank"], p["workload"]): p for plans in j["plans"] for p in plans}
    assert by[(0, "llama2-32k")]["mode"] == "batch" and by[(1, "llama2-32k")]["jobs"] == 2
    assert by[(0, "llama3-gqa-32k")]["kv_heads"] == [0, 4]
    assert by[(1, "llama3-gqa-32k")]["kv_heads"] == [4, 8]
    assert by[(1, "llama3-gqa-32k")]["Hq"] == 16
    a, b = by[(0, "llama3-gqa-128k")], by[(1, "llama3-gqa-128k")]
    assert a["tok"] == [0, 65536] and b["tok"] == [65536, 131072]
    assert (a["tail"], b["tail"]) == (False, True)
    assert j["configs"]["llama2-32k"]["global_batch"] == 2


def test_launcher_refuses_missing_gpus():
    """--gpus N with fewer than N visible GPUs exits non-zero (no silent 1-GPU run)."""
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "1"], capture_output=True, text=True, cwd=ROOT,
                       timeout=300, env=env)
    assert r.returncode != 0 and "GPU(s) visible" in r.stderr


@pytest.mark.gpu
def test_sequence_split_path_on_one_gpu():
    """Config 4 through the sequence-split path with a one-rank NCCL group: the
    per-layer (m, l, acc) records, the NCCL all-gather and the rank-ordered
    merge are captured in the step's CUDA graph (as at N > 1)."""
    j = _run("--config", "llama3-gqa-128k", "--seq-split-one", "--steps", "2", "--warmup", "3",
             "--no-cpu-baseline", "--no-encode", "--no-f16-mode")
    assert j["sequence_split"]["step_mode"] == "cuda graph"
    assert j["sequence_split"]["merge_ms_per_step"] > 0 and j["value"] > 0
