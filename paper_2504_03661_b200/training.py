"""Offline codebook training: ``kmeans_train`` and
``train_codebooks`` with the reference's names, arguments, errors and results
(``pq_core.py:171-266``).

The O(n·k) part -- the float64 distance matrix, its argmin and the assignment
errors -- runs on the GPU; the O(n) bookkeeping stays on the host in the
reference's own arithmetic.  Every float64 value is formed exactly as the
reference forms it, so the centroids and the distortion history are
bit-identical to ``pqkv.kmeans_train`` (pinned by ``tests/golden/kmeans.npz``):

* distances ``(Σx² − 2·x·c) + Σc²`` clamped at 0 (``pq_core.py:158-168``),
  with ``x·c`` accumulated as OpenBLAS dgemm does for the short inner
  dimension: a product, then one fused multiply-add per further term;
* k-means++ seeding with the same ``numpy.random.Generator`` call sequence
  (``:171-188``), its totals summed on the host;
* Lloyd steps (``:191-250``): first-index argmin, distortion summed on the
  host, the tolerance stop, cluster means as sequential row sums in sample
  order divided by the count, empty clusters re-seeded to the worst-covered
  sample.
"""

from __future__ import annotations

import warnings

import numpy as np
import torch

from .pq_core import Codebook, PQConfig, default_device


def _sqdist(X: torch.Tensor, C: torch.Tensor, xx: torch.Tensor) -> torch.Tensor:
    """(n, m) float64: (xx − 2·X@C.T) + Σc², clamped at 0."""
    xc = X[:, 0:1] * C[:, 0][None, :]
    for j in range(1, X.shape[1]):  # one fused multiply-add per further term
        xc = torch.addcmul(xc, X[:, j:j + 1], C[:, j][None, :])
    cc = (C * C).sum(dim=1)
    return ((xx[:, None] - 2.0 * xc) + cc[None, :]).clamp_min_(0.0)


def _kmeans_plusplus(X: torch.Tensor, xx: torch.Tensor, k: int,
                     rng: np.random.Generator) -> np.ndarray:
    n = X.shape[0]
    Xh = X.cpu().numpy()
    cents = np.empty((k, X.shape[1]), dtype=np.float64)
    cents[0] = Xh[rng.integers(n)]
    dist_sq = _sqdist(X, X.new_tensor(cents[:1]), xx)[:, 0]
    for i in range(1, k):
        d_h = dist_sq.cpu().numpy()
        total = d_h.sum()
        if total <= 0.0:
            for j in range(i, k):
                cents[j] = cents[j % i]
            break
        cents[i] = Xh[rng.choice(n, p=d_h / total)]
        dist_sq = torch.minimum(dist_sq, _sqdist(X, X.new_tensor(cents[i:i + 1]), xx)[:, 0])
    return cents


def kmeans_train(samples, k: int, iters: int = 25, tol: float = 1e-4, seed: int = 0,
                 device=None) -> tuple[np.ndarray, list[float]]:
    """Lloyd k-means with k-means++ seeding (``pq_core.kmeans_train``).
    Returns the (k, dsub) float32 centroids and the distortion history."""
    Xh = np.asarray(samples, dtype=np.float64)
    if Xh.ndim == 1:
        Xh = Xh[:, None]
    if Xh.shape[0] == 0:
        raise ValueError("k-means requires at least one sample")
    if k < 1:
        raise ValueError("k must be >= 1")
    if not np.all(np.isfinite(Xh)):
        raise ValueError("k-means samples must be finite")
    dev = torch.device(device) if device is not None else default_device()
    X = torch.from_numpy(np.ascontiguousarray(Xh)).to(dev)
    xx = (X * X).sum(dim=1)
    n = Xh.shape[0]

    rng = np.random.default_rng(seed)
    cents = _kmeans_plusplus(X, xx, k, rng)

    history: list[float] = []
    for _ in range(max(1, iters)):
        d2 = _sqdist(X, X.new_tensor(cents), xx)
        lab_d = d2.argmin(dim=1)
        errs = d2.gather(1, lab_d[:, None])[:, 0].cpu().numpy()
        labels = lab_d.cpu().numpy()
        distortion = float(errs.sum())
        history.append(distortion)
        if len(history) >= 2:
            prev = history[-2]
            if prev <= 0.0 or (prev - distortion) <= tol * prev:
                break
        # cluster means: rows summed in sample order, divided by the count
        counts = np.bincount(labels, minlength=k)
        order = np.argsort(labels, kind="stable")
        nz = np.flatnonzero(counts)
        starts = np.concatenate(([0], np.cumsum(counts)[:-1]))[nz]
        sums = np.add.reduceat(Xh[order], starts, axis=0)
        cents[nz] = sums / counts[nz][:, None]
        for j in np.flatnonzero(counts == 0):
            worst = int(errs.argmax())
            cents[j] = Xh[worst]
            errs[worst] = 0.0
    return cents.astype(np.float32), history


def train_codebooks(samples, config: PQConfig, kind: str = "key", scope: str = "layer",
                    device=None) -> Codebook:
    """One codebook per subspace on (n, d) samples (``pq_core.train_codebooks``)."""
    X = np.asarray(samples, dtype=np.float64)
    if X.ndim != 2 or X.shape[1] != config.d:
        raise ValueError(f"samples must be (n, {config.d}), got {X.shape}")
    if X.shape[0] < config.ksub:
        warnings.warn(f"training with {X.shape[0]} samples < {config.ksub} centroids; "
                      "surplus centroid rows will be duplicates", stacklevel=2)
    ds = config.dsub
    cents = np.empty((config.M, config.ksub, ds), dtype=np.float32)
    for i in range(config.M):
        cents[i], _ = kmeans_train(X[:, i * ds:(i + 1) * ds], config.ksub, config.kmeans_iters,
                                   config.kmeans_tol, seed=config.seed + i, device=device)
    return Codebook(config=config, centroids=cents, kind=kind, scope=scope)
