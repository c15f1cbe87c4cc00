"""Codebook training (training.py) against the reference's kmeans_train /
train_codebooks (pq_core.py:171-266), through tests/golden/kmeans.npz made by
running the reference: bit-identical centroids and distortion histories.
The CPU tests run the same torch code on the host device; the GPU test runs
the distance / argmin part on the B200."""

import numpy as np
import pytest
import torch

CASES = ["blobs", "gauss", "few", "dups", "oned"]


def _case(golden_kmeans, name, device):
    from paper_2504_03661_b200.training import kmeans_train
    g = golden_kmeans
    k, iters, tol, seed = g[f"{name}_args"]
    C, hist = kmeans_train(g[f"{name}_X"], int(k), iters=int(iters), tol=float(tol),
                           seed=int(seed), device=device)
    np.testing.assert_array_equal(C, g[f"{name}_C"])
    np.testing.assert_array_equal(np.array(hist), g[f"{name}_hist"])
    assert all(b <= a for a, b in zip(hist, hist[1:]))  # non-increasing


@pytest.fixture(scope="module")
def golden_kmeans():
    import os
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "kmeans.npz"))


@pytest.mark.parametrize("name", CASES)
def test_kmeans_bit_identical_host(golden_kmeans, name):
    _case(golden_kmeans, name, "cpu")


def test_train_codebooks_bit_identical_host(golden_kmeans):
    from paper_2504_03661_b200 import PQConfig, train_codebooks
    cfg = PQConfig(d=16, M=8, nbits=4, kmeans_iters=12, seed=7)
    cb = train_codebooks(golden_kmeans["train_X"], cfg, kind="key", device="cpu")
    np.testing.assert_array_equal(cb.centroids, golden_kmeans["train_C"])
    assert cb.kind == "key" and cb.centroids.shape == (8, 16, 2)


def test_training_errors():
    from paper_2504_03661_b200 import PQConfig, kmeans_train, train_codebooks
    with pytest.raises(ValueError, match="at least one sample"):
        kmeans_train(np.zeros((0, 2)), 4, device="cpu")
    with pytest.raises(ValueError, match="k must be"):
        kmeans_train(np.zeros((5, 2)), 0, device="cpu")
    with pytest.raises(ValueError, match="finite"):
        kmeans_train(np.array([[np.nan, 0.0]]), 1, device="cpu")
    with pytest.raises(ValueError, match="samples must be"):
        train_codebooks(np.zeros((10, 8)), PQConfig(16, 8, 4), device="cpu")
    with pytest.warns(UserWarning, match="samples <"):
        train_codebooks(np.random.default_rng(0).standard_normal((10, 16)),
                        PQConfig(16, 8, 4, kmeans_iters=2), device="cpu")


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_kmeans_bit_identical_gpu(golden_kmeans, name):
    _case(golden_kmeans, name, "cuda")


@pytest.mark.gpu
def test_train_codebooks_bit_identical_gpu(golden_kmeans):
    from paper_2504_03661_b200 import PQConfig, train_codebooks
    cfg = PQConfig(d=16, M=8, nbits=4, kmeans_iters=12, seed=7)
    cb = train_codebooks(golden_kmeans["train_X"], cfg, kind="key")
    np.testing.assert_array_equal(cb.centroids, golden_kmeans["train_C"])
