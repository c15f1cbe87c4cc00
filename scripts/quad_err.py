"""Diagnostic: the fp16 four-head kernel's error vs the fp64 oracle on a
config-3-like layer, as a fraction of the stated tolerance (rtol 2e-3, atol 2e-4)."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from test_gpu_full_shapes import _layer, _decode, _oracle
for seed, n in ((31, 32768), (5, 4000), (7, 300)):
    x = _layer(4, 32, 8, n, 31, seed=seed)
    want = _oracle(x)
    got = _decode(x, 32, 8, half=True, f16_key_table=True)
    ratio = np.abs(got - want) / (2e-4 + 2e-3 * np.abs(want))
    print(f"n={n} seed={seed}: max err / tolerance = {ratio.max():.3f}, p99 {np.percentile(ratio, 99):.3f}")
