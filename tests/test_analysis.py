"""The reference's outlier / sensitivity studies (analysis.py) on the GPU
against tests/golden/analysis.npz, made by running the reference."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "analysis.npz"))


def test_channel_stats_and_outliers(g):
    from paper_2504_03661_b200 import analysis as A
    st = A.channel_stats(g["X"])
    np.testing.assert_allclose(st.mean, g["cs_mean"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(st.std, g["cs_std"], rtol=1e-12)
    np.testing.assert_array_equal(st.absmax, g["cs_absmax"])
    np.testing.assert_allclose([st.global_absmax, st.outlier_threshold], g["cs_misc"],
                               rtol=1e-12)
    assert st.outlier_channels == list(g["cs_outliers"]) == [3, 20]
    entries, filt = A.isolate_outliers(g["X"], 0.01)
    np.testing.assert_array_equal(np.array(entries), g["io_entries"])
    np.testing.assert_allclose(filt, g["io_filtered"], rtol=1e-12, atol=1e-14)
    with pytest.raises(ValueError):
        A.isolate_outliers(g["X"], 1.0)
    with pytest.raises(ValueError):
        A.channel_stats(g["X"][:1])


def test_compare_quantizers_and_sensitivity(g):
    import paper_2504_03661_b200 as P
    from paper_2504_03661_b200 import analysis as A
    cfg = P.PQConfig(d=32, M=16, nbits=4, kmeans_iters=8, seed=2)
    cq = A.compare_quantizers(g["X"], cfg, 4)
    np.testing.assert_allclose([cq[k] for k in sorted(cq)], g["cq"], rtol=1e-12)
    # the integer study is exact; the PQ one retrains on the de-spiked tensor,
    # whose channel means are reduced in another order on the device
    np.testing.assert_allclose(A.sensitivity_study(g["X"], cfg, 0.01, "int").sensitivity,
                               g["ss_int"][2], rtol=1e-12)
    r = A.sensitivity_study(g["X"], cfg, 0.01, "pq")
    np.testing.assert_allclose([r.err_full, r.err_filtered, r.sensitivity], g["ss_pq"],
                               rtol=1e-6)
    with pytest.raises(ValueError, match="unknown quantizer"):
        A.sensitivity_study(g["X"], cfg, 0.01, "fp8")
