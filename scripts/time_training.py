"""Diagnostic: wall time of train_codebooks (m64b8, d=128) on the GPU."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2504_03661_b200 import PQConfig, train_codebooks
from paper_2504_03661_b200.harness import SynthSpec, synth_kv
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
K, _ = synth_kv(SynthSpec(n_tokens=n, d=128, seed=0, outlier_channels=[7, 63]))
cfg = PQConfig(128, 64, 8)
train_codebooks(K[:2048], PQConfig(128, 64, 8, kmeans_iters=2))  # warm-up
t0 = time.perf_counter()
cb = train_codebooks(K, cfg)
print(f"train_codebooks m64b8 on {n} x 128 samples: {time.perf_counter() - t0:.2f} s")
