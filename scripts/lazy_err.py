"""Max error of the fp16 modes vs the oracle at a few query scales (the lazy
rescale A/B: run with PQKV_SM100_LIB pointing at a PQKV_LAZY_RESCALE=0 build)."""
import os, sys
_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [_ROOT, os.path.join(_ROOT, "tests")]
import numpy as np
from test_gpu_parity import _batched_case
for qs in (1.0, 2.0, 3.0):
    for keys in (False, True):
        got, want, want16 = _batched_case(2, 8, 2, 9000, [8999, 4321], [5, 32], half_cv=True,
                                          f16_keys=keys, q_scale=qs)
        err = np.abs(got - want16)
        tol = 2e-4 + 2e-3 * np.abs(want16)
        print(f"q x{qs} keys16={keys}: max abs {err.max():.2e}, max err/tol {(err / tol).max():.3f}")
