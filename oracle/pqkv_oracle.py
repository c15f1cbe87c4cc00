"""CPU oracle for the PQ KV-cache hot path -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the sm_100a product path in
``paper_2504_03661_b200``.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product path never calls it (the package fails loudly when its CUDA
library is missing).

It is a from-scratch numpy restatement of the reference algorithm
(arXiv 2504.03661 "MILLION", reference package ``pqkv``), float64 throughout
like the reference.  Every function cites the reference file:line it follows
(paths relative to the reference's ``pkg/src/pqkv/``).

Parity pinning: the restatement is checked against golden vectors produced by
running the reference itself in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``, see
``tests/test_oracle_golden.py``).  The hot inner loops optionally run through
the C restatement in ``oracle/pqkv_oracle.c`` (same arithmetic order), which
is what the CPU baseline times.
"""

from __future__ import annotations

import ctypes
import os
import struct
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))

# --------------------------------------------------------------------------
# geometry (pq_core.py:31-75)
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class Geometry:
    """d, M, nbits with the derived quantities of PQConfig (pq_core.py:31-75)."""

    d: int
    M: int
    nbits: int

    def __post_init__(self):
        if self.M <= 0 or self.d <= 0 or self.d % self.M:
            raise ValueError("bad geometry")
        if not 1 <= self.nbits <= 16:
            raise ValueError("nbits out of range")

    @property
    def dsub(self) -> int:
        return self.d // self.M

    @property
    def ksub(self) -> int:
        return 1 << self.nbits

    @property
    def code_dtype(self):
        return np.uint8 if self.nbits <= 8 else np.uint16


# --------------------------------------------------------------------------
# encoder (pq_core.py:158-168 _squared_distances, :269-287 assign_codes)
# --------------------------------------------------------------------------


def subspace_distances(x_sub: np.ndarray, cents: np.ndarray) -> np.ndarray:
    """fp64 expanded-form squared distances, (n, ksub).

    Follows pq_core.py:158-168: d2 = (||x||^2 - 2 x.c) + ||c||^2, clamped at 0.
    Inputs are float32 values promoted to float64, so every product is exact.
    x.c is a sequential k-loop (OpenBLAS dgemm order, checked bit-for-bit for
    k in 2..16); the norms use numpy's pairwise row sum.
    """
    X = np.asarray(x_sub, dtype=np.float64)
    C = np.asarray(cents, dtype=np.float64)
    n, dsub = X.shape
    # row norms: numpy's pairwise axis-1 sum (8 accumulators from 8 terms up),
    # exactly what pq_core.py:163,165 evaluates
    xx = np.sum(X * X, axis=1)
    cc = np.sum(C * C, axis=1)
    xc = np.zeros((n, C.shape[0]))
    for j in range(dsub):                 # dgemm k-loop: FMA chain == exact products + sequential adds
        xc = xc + X[:, j : j + 1] * C[None, :, j]
    d2 = (xx[:, None] - 2.0 * xc) + cc[None, :]
    return np.maximum(d2, 0.0)


def assign_codes(X: np.ndarray, centroids: np.ndarray, nbits: int) -> np.ndarray:
    """Nearest-centroid codes (n, M), ties -> lowest index (pq_core.py:269-287)."""
    X = np.asarray(X, dtype=np.float64)
    M, ksub, dsub = centroids.shape
    if X.ndim != 2 or X.shape[1] != M * dsub:
        raise ValueError("X must be (n, d)")
    if not np.all(np.isfinite(X)):
        raise ValueError("X must be finite")
    out = np.empty((X.shape[0], M), dtype=np.uint8 if nbits <= 8 else np.uint16)
    for i in range(M):
        d2 = subspace_distances(X[:, i * dsub : (i + 1) * dsub], centroids[i])
        out[:, i] = np.argmin(d2, axis=1)    # first occurrence of the minimum
    return out


def reconstruct(codes: np.ndarray, centroids: np.ndarray) -> np.ndarray:
    """Dequantize (n, M) codes to (n, d) float32 (pq_core.py:290-304)."""
    M, ksub, dsub = centroids.shape
    codes = np.asarray(codes)
    if codes.size and int(codes.max()) >= ksub:
        raise ValueError("corrupted cache: code value out of codebook range")
    out = np.empty((codes.shape[0], M * dsub), dtype=np.float32)
    for i in range(M):
        out[:, i * dsub : (i + 1) * dsub] = centroids[i][codes[:, i]]
    return out


# --------------------------------------------------------------------------
# attention (attention.py)
# --------------------------------------------------------------------------


@dataclass
class Partial:
    """Online-softmax state (m, l, acc) -- attention.py:46-53, 66-67."""

    m: float
    l: float
    acc: np.ndarray


def empty(d: int) -> Partial:
    return Partial(-np.inf, 0.0, np.zeros(d))


def default_scale(d: int) -> float:
    return 1.0 / np.sqrt(d)                # attention.py:77-78, 235-236


def key_lut(q: np.ndarray, cents_k: np.ndarray, scale: float | None = None) -> np.ndarray:
    """table[i, c] = scale * <q_i, C_K[i, c]> in float64 (attention.py:70-83)."""
    M, ksub, dsub = cents_k.shape
    q = np.asarray(q, dtype=np.float64).ravel()
    if q.shape[0] != M * dsub:
        raise ValueError("query width mismatch")
    if scale is None:
        scale = default_scale(M * dsub)
    qs = q.reshape(M, dsub)
    return (cents_k.astype(np.float64) * qs[:, None, :]).sum(axis=2) * scale


def score_codes(table: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """s_t = sum_i table[i, codes[t, i]] (_kernels.py:27-34, 46-53)."""
    n, M = codes.shape
    if n == 0:
        return np.zeros(0)
    g = table[np.arange(M)[None, :], codes.astype(np.int64)]
    s = np.zeros(n)
    for i in range(M):                     # sequential over subspaces, like the JIT loop
        s = s + g[:, i]
    return s


def accumulate_mass(codes: np.ndarray, p: np.ndarray, ksub: int) -> np.ndarray:
    """h[i, c] = sum of p_t over tokens with codes[t, i] == c (_kernels.py:37-43, 56-65)."""
    n, M = codes.shape
    h = np.zeros((M, ksub))
    for i in range(M):
        h[i] = np.bincount(codes[:, i].astype(np.int64), weights=p, minlength=ksub)
    return h


def mass_to_acc(h: np.ndarray, cents_v: np.ndarray) -> np.ndarray:
    """acc[i*dsub:(i+1)*dsub] = h[i] @ C_V[i] (attention.py:103-111)."""
    M, ksub, dsub = cents_v.shape
    return np.concatenate([h[i] @ cents_v[i].astype(np.float64) for i in range(M)])


def quantized_partial(table: np.ndarray, codes_k: np.ndarray, codes_v: np.ndarray,
                      cents_v: np.ndarray, strategy: str = "auto") -> Partial:
    """Softmax partial over a quantized span (attention.py:114-166)."""
    M, ksub, dsub = cents_v.shape
    if codes_k.shape[0] != codes_v.shape[0]:
        raise ValueError("key/value token counts differ")
    n = codes_k.shape[0]
    if n == 0:
        return empty(M * dsub)
    if strategy == "auto":
        strategy = "centroid_accumulate" if n > 4 * ksub else "gather"
    if strategy not in ("gather", "centroid_accumulate"):
        raise ValueError(f"unknown strategy {strategy!r}")
    s = score_codes(table, codes_k)
    m = float(s.max())
    p = np.exp(s - m)
    l = float(p.sum())
    if strategy == "gather":
        acc = p @ reconstruct(codes_v, cents_v).astype(np.float64)
    else:
        acc = mass_to_acc(accumulate_mass(codes_v, p, ksub), cents_v)
    return Partial(m, l, acc)


def dense_partial(q: np.ndarray, K: np.ndarray, V: np.ndarray,
                  scale: float | None = None) -> Partial:
    """Exact softmax partial over full-precision rows (attention.py:169-190)."""
    q = np.asarray(q, dtype=np.float64).ravel()
    K = np.asarray(K, dtype=np.float64).reshape(-1, q.shape[0])
    V = np.asarray(V, dtype=np.float64)
    V = V[None, :] if V.ndim == 1 else V
    if K.shape[0] != V.shape[0]:
        raise ValueError("K rows != V rows")
    if K.shape[0] == 0:
        raise ValueError("dense partial requires at least the current token")
    if scale is None:
        scale = default_scale(q.shape[0])
    s = scale * (K @ q)
    m = float(s.max())
    p = np.exp(s - m)
    return Partial(m, float(p.sum()), p @ V)


def merge(a: Partial, b: Partial) -> Partial:
    """Associative online-softmax merge with empty identity (attention.py:193-204)."""
    if a.acc.shape != b.acc.shape:
        raise ValueError("partial widths differ")
    if a.l == 0.0:
        return Partial(b.m, b.l, b.acc.copy())
    if b.l == 0.0:
        return Partial(a.m, a.l, a.acc.copy())
    m = max(a.m, b.m)
    wa, wb = np.exp(a.m - m), np.exp(b.m - m)
    return Partial(m, a.l * wa + b.l * wb, a.acc * wa + b.acc * wb)


def finalize(p: Partial) -> np.ndarray:
    """acc / l (attention.py:207-211)."""
    if p.l <= 0.0:
        raise ValueError("cannot finalize an empty softmax partial")
    return p.acc / p.l


def decode_from_snapshot(q, k_n, v_n, codes_k, codes_v, recent_k, recent_v,
                         cents_k, cents_v, scale=None, strategy="auto",
                         block_size: int = 1024) -> np.ndarray:
    """decode_step (attention.py:214-287) minus the trailing append: blockwise
    quantized partials over [0, n_q), dense partial over recent rows + the
    current token, merge, finalize."""
    M, ksub, dsub = cents_k.shape
    d = M * dsub
    if scale is None:
        scale = default_scale(d)
    table = key_lut(q, cents_k, scale)
    res = empty(d)
    n_q = codes_k.shape[0]
    for a in range(0, n_q, block_size):
        b = min(a + block_size, n_q)
        res = merge(res, quantized_partial(table, codes_k[a:b], codes_v[a:b],
                                           cents_v, strategy))
    Kd = np.vstack([np.asarray(recent_k, np.float64).reshape(-1, d),
                    np.asarray(k_n, np.float64)[None, :]])
    Vd = np.vstack([np.asarray(recent_v, np.float64).reshape(-1, d),
                    np.asarray(v_n, np.float64)[None, :]])
    res = merge(res, dense_partial(q, Kd, Vd, scale))
    return finalize(res)


def naive_attention(q, K, V, scale=None) -> np.ndarray:
    """softmax(scale q K^T) V, single max subtraction (oracle.py:17-31)."""
    q = np.asarray(q, np.float64)
    K = np.asarray(K, np.float64)
    V = np.asarray(V, np.float64)
    if K.shape[0] == 0:
        raise ValueError("attention over zero tokens is undefined")
    if scale is None:
        scale = default_scale(q.shape[-1])
    s = scale * (K @ q)
    w = np.exp(s - s.max())
    return (w[:, None] * V).sum(axis=0) / w.sum()


def naive_quantized_attention(q, codes_k, codes_v, cents_k, cents_v,
                              recent_k, recent_v, k_n, v_n, scale=None):
    """Dequantize-then-attend reference (oracle.py:44-64)."""
    d = cents_k.shape[0] * cents_k.shape[2]
    K = np.vstack([reconstruct(codes_k, cents_k).astype(np.float64),
                   np.asarray(recent_k, np.float64).reshape(-1, d),
                   np.asarray(k_n, np.float64)[None, :]])
    V = np.vstack([reconstruct(codes_v, cents_v).astype(np.float64),
                   np.asarray(recent_v, np.float64).reshape(-1, d),
                   np.asarray(v_n, np.float64)[None, :]])
    return naive_attention(q, K, V, scale)


# --------------------------------------------------------------------------
# cache state machine (kv_cache.py:42-302), synchronous semantics only
# --------------------------------------------------------------------------


class CacheModel:
    """Sync-mode model of LayerKVCache's visible state (kv_cache.py:55-302).

    Tracks the published quantized span and the full-precision recent rows;
    flushes encode whole batches of the oldest `flush_threshold` rows.
    """

    def __init__(self, cents_k, cents_v, nbits, recent_capacity=32, flush_threshold=32):
        if recent_capacity < 0 or flush_threshold < 1:
            raise ValueError("recent_capacity >= 0 and flush_threshold >= 1 required")
        self.ck, self.cv, self.nbits = cents_k, cents_v, nbits
        self.R, self.R_f = recent_capacity, flush_threshold
        M = cents_k.shape[0]
        dt = np.uint8 if nbits <= 8 else np.uint16
        self.codes_k = np.zeros((0, M), dt)
        self.codes_v = np.zeros((0, M), dt)
        self.recent: list[tuple[np.ndarray, np.ndarray]] = []

    @property
    def d(self):
        return self.ck.shape[0] * self.ck.shape[2]

    @property
    def n_q(self):
        return self.codes_k.shape[0]

    @property
    def n_total(self):
        return self.n_q + len(self.recent)

    def _encode_oldest(self, batch: int) -> None:
        rk = np.stack([r[0] for r in self.recent[:batch]])
        rv = np.stack([r[1] for r in self.recent[:batch]])
        self.codes_k = np.vstack([self.codes_k, assign_codes(rk, self.ck, self.nbits)])
        self.codes_v = np.vstack([self.codes_v, assign_codes(rv, self.cv, self.nbits)])
        del self.recent[:batch]

    def prefill(self, K, V) -> None:
        """prefill_ingest (kv_cache.py:120-141): keep min(R, n) trailing rows."""
        K = np.asarray(K, np.float32)
        V = np.asarray(V, np.float32)
        n = K.shape[0]
        keep = min(self.R, n)
        if n - keep > 0:
            self.codes_k = np.vstack([self.codes_k, assign_codes(K[: n - keep], self.ck, self.nbits)])
            self.codes_v = np.vstack([self.codes_v, assign_codes(V[: n - keep], self.cv, self.nbits)])
        for t in range(n - keep, n):
            self.recent.append((K[t].copy(), V[t].copy()))

    def append(self, k, v) -> None:
        """append_decode with an inline (sync) flush (kv_cache.py:143-162)."""
        self.recent.append((np.asarray(k, np.float32).ravel().copy(),
                            np.asarray(v, np.float32).ravel().copy()))
        while len(self.recent) >= self.R_f:
            self._encode_oldest(self.R_f)

    def snapshot(self):
        d = self.d
        rk = np.stack([r[0] for r in self.recent]) if self.recent else np.zeros((0, d), np.float32)
        rv = np.stack([r[1] for r in self.recent]) if self.recent else np.zeros((0, d), np.float32)
        return self.codes_k, self.codes_v, rk, rv


# --------------------------------------------------------------------------
# codebook file (fileio.py:71-96)
# --------------------------------------------------------------------------

CODEBOOK_MAGIC = b"PQKV"


def parse_codebook(raw: bytes):
    """Return (kind_id, d, M, nbits, centroids) from .pqkv bytes (fileio.py:80-96).

    Layout: magic 'PQKV', then little-endian u32 version, u8 kind, u32 d,
    u32 M, u32 nbits (21-byte header, unaligned float body, subspace-major).
    """
    if raw[:4] != CODEBOOK_MAGIC:
        raise ValueError("bad magic")
    version, kind, d, M, nbits = struct.unpack_from("<IBIII", raw, 4)
    if version != 1:
        raise ValueError("unsupported version")
    if kind not in (0, 1):
        raise ValueError("unknown kind tag")
    g = Geometry(d, M, nbits)
    body = np.frombuffer(raw, dtype="<f4", offset=21)
    if body.size != M * g.ksub * g.dsub:
        raise ValueError("size mismatch")
    return kind, d, M, nbits, body.reshape(M, g.ksub, g.dsub).copy()


# --------------------------------------------------------------------------
# optional C restatement of the hot loops (oracle/pqkv_oracle.c)
# --------------------------------------------------------------------------

_clib = None


def c_library():
    """Load oracle/_build/libpqkv_oracle.so (built by oracle/Makefile) or None."""
    global _clib
    if _clib is None:
        path = os.path.join(_HERE, "_build", "libpqkv_oracle.so")
        if not os.path.exists(path):
            return None
        lib = ctypes.CDLL(path)
        P = ctypes.c_void_p
        lib.oracle_decode_head.argtypes = [P, P, P, P, P, ctypes.c_int64, P, P,
                                           ctypes.c_int64, P, P, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_double, ctypes.c_int64, P]
        lib.oracle_decode_head.restype = ctypes.c_int
        lib.oracle_decode_heads_mt.argtypes = [P, P, P, P, P, ctypes.c_int64, ctypes.c_int64,
                                               P, P, ctypes.c_int64, P, P, ctypes.c_int,
                                               ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                               ctypes.c_int64, P, ctypes.c_int, ctypes.c_int]
        lib.oracle_decode_heads_mt.restype = ctypes.c_int
        I, I64 = ctypes.c_int, ctypes.c_int64
        lib.oracle_decode_gqa_mt.argtypes = [P, P, P, P, P, I, I, I, P, I64, P, P, P, I64, P, P,
                                             I, I, I, ctypes.c_double, I64, P, I]
        lib.oracle_decode_gqa_mt.restype = ctypes.c_int
        lib.oracle_assign_codes.argtypes = [P, ctypes.c_int64, P, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int, P, ctypes.c_int]
        lib.oracle_assign_codes.restype = ctypes.c_int
        _clib = lib
    return _clib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def c_assign_codes(X, centroids, nbits, threads=1):
    """C restatement of assign_codes (same fp64 arithmetic); uint8/uint16 out."""
    lib = c_library()
    X = np.ascontiguousarray(X, np.float32)
    C = np.ascontiguousarray(centroids, np.float32)
    M, ksub, dsub = C.shape
    out = np.empty((X.shape[0], M), np.uint8 if nbits <= 8 else np.uint16)
    rc = lib.oracle_assign_codes(_p(X), X.shape[0], _p(C), M, nbits, dsub, _p(out), threads)
    if rc:
        raise RuntimeError("oracle_assign_codes failed")
    return out


def c_decode_head(q, k_n, v_n, codes_k, codes_v, recent_k, recent_v, cents_k, cents_v,
                  nbits, scale=None, block_size=8192):
    """C restatement of decode_from_snapshot with strategy 'auto' (fp64)."""
    lib = c_library()
    M, ksub, dsub = cents_k.shape
    d = M * dsub
    if scale is None:
        scale = default_scale(d)
    q = np.ascontiguousarray(q, np.float64)
    k_n = np.ascontiguousarray(k_n, np.float32)
    v_n = np.ascontiguousarray(v_n, np.float32)
    cdt = np.uint8 if nbits <= 8 else np.uint16
    ck = np.ascontiguousarray(codes_k, cdt)
    cv = np.ascontiguousarray(codes_v, cdt)
    rk = np.ascontiguousarray(recent_k, np.float32).reshape(-1, d)
    rv = np.ascontiguousarray(recent_v, np.float32).reshape(-1, d)
    CK = np.ascontiguousarray(cents_k, np.float32)
    CV = np.ascontiguousarray(cents_v, np.float32)
    out = np.empty(d)
    rc = lib.oracle_decode_head(_p(q), _p(k_n), _p(v_n), _p(ck), _p(cv), ck.shape[0],
                                _p(rk), _p(rv), rk.shape[0], _p(CK), _p(CV), M, nbits,
                                dsub, float(scale), int(block_size), _p(out))
    if rc:
        raise RuntimeError("oracle_decode_head failed")
    return out


def c_decode_batched(q, k_n, v_n, codes_k, codes_v, n_q, recent_k, recent_v, n_recent,
                     cents_k, cents_v, nbits, scale=None, block_size=8192, threads=None):
    """C restatement of the per-query-head decode over a batched GQA cache:
    q (B, Hq, d); codes (B, Hkv, cap, M) in the reference row layout; n_q (B,);
    recent (B, Hkv, R, d) with n_recent (B,) live rows; k_n / v_n (B, Hkv, d).
    Returns (B, Hq, d) float64.  All host cores by default."""
    lib = c_library()
    if lib is None:
        raise RuntimeError("oracle C library not built (make -C oracle)")
    M, ksub, dsub = cents_k.shape
    d = M * dsub
    B, Hq, _ = q.shape
    Hkv = codes_k.shape[1]
    if scale is None:
        scale = default_scale(d)
    if threads is None:
        threads = len(os.sched_getaffinity(0))
    cdt = np.uint8 if nbits <= 8 else np.uint16
    qd = np.ascontiguousarray(q, np.float64)
    kn = np.ascontiguousarray(k_n, np.float32)
    vn = np.ascontiguousarray(v_n, np.float32)
    ck = np.ascontiguousarray(codes_k, cdt)
    cv = np.ascontiguousarray(codes_v, cdt)
    rk = np.ascontiguousarray(recent_k, np.float32)
    rv = np.ascontiguousarray(recent_v, np.float32)
    nq = np.ascontiguousarray(n_q, np.int32)
    nr = np.ascontiguousarray(n_recent, np.int32)
    CK = np.ascontiguousarray(cents_k, np.float32)
    CV = np.ascontiguousarray(cents_v, np.float32)
    out = np.empty((B, Hq, d))
    rc = lib.oracle_decode_gqa_mt(_p(qd), _p(kn), _p(vn), _p(ck), _p(cv), B, Hq, Hkv, _p(nq),
                                  ck.shape[2], _p(rk), _p(rv), _p(nr), rk.shape[2], _p(CK),
                                  _p(CV), M, nbits, dsub, float(scale), int(block_size),
                                  _p(out), int(threads))
    if rc:
        raise RuntimeError(f"oracle_decode_gqa_mt failed ({rc})")
    return out
