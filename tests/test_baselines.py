"""The reference's integer-quantization and prefill-attention baselines
(baselines.py) against tests/golden/baselines.npz, made by running the
reference: integer codes, scale and zero point bit-identical, prefill
attention to float64 rounding.  CPU tests run the same torch code on the
host device; the GPU test on the B200."""

import os

import numpy as np
import pytest


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "baselines.npz"))


def _check(g, device):
    from paper_2504_03661_b200 import integer_dequantize, integer_quantize, prefill_attention
    for nb in (2, 4, 8):
        for mode in ("symmetric", "asymmetric"):
            Q, prm = integer_quantize(g["iq_X"], nb, mode, device=device)
            np.testing.assert_array_equal(Q, g[f"iq_{mode}_{nb}_Q"])
            assert (prm.s, prm.z) == tuple(g[f"iq_{mode}_{nb}_sz"]) and prm.mode == mode
            np.testing.assert_array_equal(integer_dequantize(Q, prm, device=device),
                                          g[f"iq_{mode}_{nb}_Xh"])
    for nb in (2, 3, 4):  # grid-valued inputs: exact .5 boundaries (true division)
        for mode in ("symmetric", "asymmetric"):
            Q, prm = integer_quantize(g["iqg_X"], nb, mode, device=device)
            np.testing.assert_array_equal(Q, g[f"iqg_{mode}_{nb}_Q"])
            assert (prm.s, prm.z) == tuple(g[f"iqg_{mode}_{nb}_sz"])
    np.testing.assert_allclose(prefill_attention(g["pf_Q"], g["pf_K"], g["pf_V"], device=device),
                               g["pf_causal"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(prefill_attention(g["pf_Q"], g["pf_K"], g["pf_V"], causal=False,
                                                 scale=0.3, device=device),
                               g["pf_full"], rtol=1e-12, atol=1e-13)


def test_baselines_host(g):
    _check(g, "cpu")


def test_baseline_edges():
    from paper_2504_03661_b200 import integer_quantize, prefill_attention
    with pytest.raises(ValueError, match="empty"):
        integer_quantize(np.zeros((0,)), 4, device="cpu")
    with pytest.raises(ValueError, match="non-finite"):
        integer_quantize(np.array([np.inf]), 4, device="cpu")
    with pytest.raises(ValueError, match="unknown mode"):
        integer_quantize(np.ones(3), 4, "odd", device="cpu")
    Q, p = integer_quantize(np.full((2, 2), 3.0), 4, device="cpu")
    assert (Q == 0).all() and p.s == 1.0 and p.z == 0
    Q, p = integer_quantize(np.zeros(4), 4, "symmetric", device="cpu")
    assert (Q == 0).all() and p.s == 1.0
    with pytest.raises(ValueError, match="inconsistent"):
        prefill_attention(np.ones((2, 3)), np.ones((4, 5)), np.ones((4, 5)), device="cpu")


@pytest.mark.gpu
def test_baselines_gpu(g):
    _check(g, None)
