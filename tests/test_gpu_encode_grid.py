"""The candidate-grid encoder (pqkv_encode_grid, dsub = 2): per subspace a
64 x 64 grid of candidate lists; the fp32 filter scans a point's list instead
of every centroid, near ties still go to the exact fp64 scan over all of them,
so the codes must equal the reference's (assign_codes, pq_core.py:269-287)
bit for bit -- checked here against the fp64 oracle and the full-scan encoder
on the inputs that stress the lists: outliers outside the grid, points on
centroids and midpoints (ties), ulp nudges, duplicate and degenerate
codebooks, trained (clustered) codebooks, half-precision inputs and the
decode layout."""

import numpy as np
import pytest
import torch

from oracle import pqkv_oracle as O

pytestmark = pytest.mark.gpu


def _both(X, cents, nbits=8, **kw):
    from paper_2504_03661_b200 import kernels as K
    x = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    c = torch.from_numpy(np.ascontiguousarray(cents)).cuda()
    grid = K.encode_grid(c, nbits)
    assert grid is not None
    return (K.encode(x, c, nbits, grid=grid, **kw).cpu().numpy(),
            K.encode(x, c, nbits, **kw).cpu().numpy())


@pytest.mark.parametrize("scale", [1e-3, 1.0, 1e3])
def test_grid_random_and_outliers(scale):
    rng = np.random.default_rng(1)
    M, n = 64, 20000
    cents = (rng.standard_normal((M, 256, 2)) * scale).astype(np.float32)
    X = (rng.standard_normal((n, 2 * M)) * scale).astype(np.float32)
    X[::97] *= 40.0  # far outside the centroids' box: full scans
    got, full = _both(X, cents)
    np.testing.assert_array_equal(got, full)
    np.testing.assert_array_equal(got, O.c_assign_codes(X, cents, 8))


def test_grid_ties_nudges_duplicates():
    rng = np.random.default_rng(11)
    M, ksub, n = 64, 256, 12000
    cents = rng.standard_normal((M, ksub, 2)).astype(np.float32)
    cents[:, 200] = cents[:, 17]  # exact duplicates: the lower index
    X = np.empty((n, 2 * M), dtype=np.float32)
    for i in range(M):
        a, b = rng.integers(0, ksub, n), rng.integers(0, ksub, n)
        ca, cb = cents[i, a].astype(np.float64), cents[i, b].astype(np.float64)
        mid = ((ca + cb) / 2).astype(np.float32)
        kind = np.arange(n) % 4
        x = np.where(kind[:, None] == 0, cents[i, a], mid)
        nudge = np.nextafter(mid, np.float32(np.inf) * np.sign(rng.standard_normal((n, 2))))
        x = np.where(kind[:, None] == 2, nudge, x)
        x = np.where(kind[:, None] == 3, cents[i, 17], x)
        X[:, 2 * i: 2 * i + 2] = x
    got, full = _both(X, cents)
    np.testing.assert_array_equal(got, full)
    np.testing.assert_array_equal(got, O.assign_codes(X, cents, 8))
    assert (got[3::4] == 17).all()


def test_grid_degenerate_codebooks():
    """Centroids on a line, all equal, tiny spread, and a cluster plus a far
    outlier centroid: the grid box degenerates or most cells crowd."""
    rng = np.random.default_rng(3)
    M, n = 8, 6000
    cents = rng.standard_normal((M, 256, 2)).astype(np.float32)
    cents[0, :, 1] = 0.5                          # a line
    cents[1] = 0.25                               # all equal
    cents[2] *= 1e-6                              # tiny
    cents[3, :255] *= 0.01
    cents[3, 255] = (100.0, -100.0)               # far outlier centroid
    cents[4, :, 0] = np.round(cents[4, :, 0] * 4) / 4  # coarse lattice: many exact ties
    cents[4, :, 1] = np.round(cents[4, :, 1] * 4) / 4
    X = rng.standard_normal((n, 2 * M)).astype(np.float32)
    X[:, 4:6] = 1e-6 * rng.standard_normal((n, 2)).astype(np.float32)
    X[:, 8:10] = np.round(X[:, 8:10] * 8) / 8      # on the lattice / midpoints
    got, full = _both(X, cents)
    np.testing.assert_array_equal(got, full)
    np.testing.assert_array_equal(got, O.assign_codes(X, cents, 8))


def test_grid_trained_codebooks_and_smaller_ksub():
    """k-means centroids of clustered data (the codebooks the reference trains),
    and nbits 4 / 6 (ksub 16 / 64)."""
    from paper_2504_03661_b200 import kernels as K
    rng = np.random.default_rng(5)
    for nbits, M in ((8, 64), (6, 16), (4, 8)):
        ksub = 1 << nbits
        centers = rng.standard_normal((M, 12, 2)) * 2
        data = (centers[:, rng.integers(0, 12, 4000)] +
                0.3 * rng.standard_normal((M, 4000, 2))).astype(np.float32)
        cents = np.stack([data[i, rng.choice(4000, ksub, replace=False)] for i in range(M)])
        X = data.transpose(1, 0, 2).reshape(4000, 2 * M).copy()
        got, full = _both(X, cents, nbits)
        np.testing.assert_array_equal(got, full)
        np.testing.assert_array_equal(got, O.assign_codes(X, cents, nbits))
    assert K.encode_grid(torch.zeros((16, 256, 8), device="cuda"), 8) is None  # dsub 8: no grid


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_grid_half_inputs(dtype):
    from paper_2504_03661_b200 import kernels as K
    rng = np.random.default_rng(6)
    cents = rng.standard_normal((64, 256, 2)).astype(np.float32)
    X = torch.from_numpy(rng.standard_normal((4096, 128)).astype(np.float32)).to(dtype).cuda()
    c = torch.from_numpy(cents).cuda()
    got = K.encode(X, c, 8, grid=K.encode_grid(c, 8)).cpu().numpy()
    np.testing.assert_array_equal(got, O.assign_codes(X.float().cpu().numpy(), cents, 8))


def test_grid_decode_layout_and_batched():
    """The decode layout (row 0 at token t_first) and the batched form (one
    grid per problem) equal the full-scan encoder."""
    from paper_2504_03661_b200 import kernels as K
    rng = np.random.default_rng(8)
    Z, n = 3, 4100
    cents = torch.from_numpy(rng.standard_normal((Z, 64, 256, 2)).astype(np.float32)).cuda()
    X = torch.from_numpy(rng.standard_normal((Z, n, 128)).astype(np.float32)).cuda()
    grids = torch.stack([K.encode_grid(cents[z], 8) for z in range(Z)])
    for z in range(Z):
        a = K.encode(X[z], cents[z], 8, layout="decode", t_first=5, grid=grids[z])
        b = K.encode(X[z], cents[z], 8, layout="decode", t_first=5)
        assert torch.equal(a, b)
    a = K.encode_batched(X, cents, 8, layout="decode", t_first=3, grids=grids)
    b = K.encode_batched(X, cents, 8, layout="decode", t_first=3)
    assert torch.equal(a, b)


def test_grid_lists_are_short():
    """The point of the grid: on N(0,1) data most points scan a handful of
    candidates (the kernel's speed, not its result, depends on this)."""
    from paper_2504_03661_b200 import kernels as K
    rng = np.random.default_rng(9)
    c = torch.from_numpy(rng.standard_normal((64, 256, 2)).astype(np.float32)).cuda()
    g = K.encode_grid(c, 8).cpu().numpy()
    rec = g.size // 64
    counts = g.reshape(64, rec)[:, 32 + 2 * 4096: 32 + 3 * 4096]
    inner = counts.reshape(64, 64, 64)[:, 16:48, 16:48]  # the centroids' box
    assert (inner != 255).mean() > 0.99 and np.median(inner[inner != 255]) <= 8
