import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import torch
from test_gpu_parity import _batched_case
for keys in (False, True):
    got, want, want16 = _batched_case(4, 32, 8, 9000, [9000, 8000, 1, 4500], [31, 0, 3, 17], half_cv=True, f16_keys=keys)
    err = np.abs(got - want) - (2e-4 + 2e-3 * np.abs(want))
    bad = np.argwhere(err > 0)
    print("f16_keys", keys, "max abs err", np.abs(got - want).max(), "viol", len(bad), bad[:5].tolist())
    d = np.abs(got - want).max(axis=2)
    print("  per-seq max abs err", d.max(axis=1))
