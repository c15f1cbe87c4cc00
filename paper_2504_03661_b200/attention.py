"""Decode-step attention over a PQ KV cache -- drop-in for the reference ``attention``.

Same names, arguments and errors as the reference's ``attention.py``
(Lut :37-43, SoftmaxPartial :46-53, Counters :56-63, empty_partial :66-67,
build_key_lut :70-83, score_tokens :86-100, quantized_partial :114-166,
dense_partial :169-190, merge_partials :193-204, finalize :207-211,
decode_step :214-287).  The arithmetic runs in libpqkv_sm100.so:

* build_key_lut      -> pqkv_build_lut (float32 table, centroid-major; the
                        decode kernel builds the same table in shared memory)
* score_tokens       -> pqkv_score_codes
* quantized_partial  -> pqkv_decode_partials + pqkv_decode_finish: one fused
                        kernel (LUT gather, online softmax, value accumulation
                        in registers from the shared-memory codebook), split
                        over every SM and merged in a fixed order;
* dense_partial      -> pqkv_decode_finish (recent rows, no quantized span)
* decode_step        -> one launch per token for a LayerKVCache with device
                        tensors (pqkv_step_run: LUT in shared memory, fused
                        partials, dense/current-token merge, finalize, and the
                        append of (k_n, v_n) to the recent ring by the
                        finishing CTA); other caches / host inputs take the
                        fused decode launch followed by the cache append.

The reference accumulates in float64 on the CPU; this path accumulates in
float32 on the GPU.  Outputs agree within the tolerance stated in DESIGN.md
(1e-5 relative on the oracle cases).  numpy inputs give numpy float64 results
like the reference; CUDA tensors give CUDA tensors and never synchronise.
``strategy`` is validated as in the reference; both values select the same
kernel (the value path never materialises V), and
``block_size`` only affects the reference's CPU blocking, so it is accepted
and ignored (the GPU split is chosen per SM count).
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import kernels as K
from .pq_core import Codebook, CodesMatrix, _is_tensor, default_device, to_device

__all__ = ["Lut", "SoftmaxPartial", "Counters", "empty_partial", "build_key_lut",
           "score_tokens", "quantized_partial", "dense_partial", "merge_partials", "finalize",
           "decode_step"]

_STRATEGIES = ("auto", "gather", "centroid_accumulate")


@dataclass
class Lut:
    """Scaled query-centroid dot products.  ``table`` is (M, 2^nbits) like the
    reference; ``device_table`` is the centroid-major (2^nbits, M) float32 copy
    the kernels read."""

    table: object
    nbits: int
    device_table: torch.Tensor | None = None


@dataclass
class SoftmaxPartial:
    """Online-softmax state (m, l, acc); empty = (-inf, 0, 0)."""

    m: float
    l: float
    acc: object


@dataclass
class Counters:
    lut_lookups: int = 0
    adds: int = 0
    code_bytes_read: int = 0
    dense_bytes_read: int = 0


def empty_partial(d: int) -> SoftmaxPartial:
    return SoftmaxPartial(m=-np.inf, l=0.0, acc=np.zeros(d, dtype=np.float64))


def _scale(d: int, scale):
    return 1.0 / np.sqrt(d) if scale is None else float(scale)


def build_key_lut(q_n, cb_K: Codebook, scale: float | None = None) -> Lut:
    """table[i][c] = scale * dot(q_n subvector i, key centroid c of subspace i).

    ``table`` is float64 like the reference (pqkv_build_lut_f64); the kernels'
    float32 centroid-major table (pqkv_build_lut) rides along as
    ``device_table``."""
    cfg = cb_K.config
    host = not _is_tensor(q_n)
    q64 = to_device(np.asarray(q_n, dtype=np.float64).ravel() if host else q_n.reshape(-1),
                    torch.float64)
    if q64.shape[0] != cfg.d:
        raise ValueError(f"query width {q64.shape[0]} != codebook d {cfg.d}")
    dev = q64.device
    sc = _scale(cfg.d, scale)
    cents = cb_K.device_centroids(dev)
    cm = K.build_lut(q64.float().view(1, -1), cents, cfg.nbits, sc)[0]
    t64 = K.build_lut_f64(q64.view(1, -1), cents, cfg.nbits, sc)[0]
    table = t64.cpu().numpy() if host else t64
    return Lut(table=table, nbits=cfg.nbits, device_table=cm)


def _device_table(lut: Lut) -> torch.Tensor:
    if lut.device_table is not None:
        return lut.device_table
    t = lut.table
    t = to_device(np.asarray(t, dtype=np.float32) if not _is_tensor(t) else t, torch.float32)
    lut.device_table = t.t().contiguous()
    return lut.device_table


def _check_codes_for_table(tab: torch.Tensor, codes_K: CodesMatrix) -> None:
    """The reference's range check (attention.py:88-91): only when the cell
    can hold a value >= ksub."""
    ksub = tab.shape[0]
    if codes_K.n_tokens and ksub <= (255 if codes_K.cell_width == 1 else 65535):
        from .pq_core import _max_code
        if _max_code(codes_K.codes) >= ksub:
            raise ValueError("code value out of range for lookup table")


def score_tokens(lut: Lut, codes_K: CodesMatrix, counters: Counters | None = None):
    """scores[t] = sum_i lut[i][codes[t][i]] (keys stay quantized)."""
    tab = _device_table(lut)
    c = codes_K.codes
    n = codes_K.n_tokens
    _check_codes_for_table(tab, codes_K)
    if counters is not None:
        counters.lut_lookups += n * codes_K.M
        counters.adds += n * codes_K.M
        counters.code_bytes_read += n * codes_K.M * codes_K.cell_width
    host = not _is_tensor(c)
    if n == 0:
        return np.empty(0, dtype=np.float64) if host else torch.empty(0, device=tab.device)
    # the float64 seam with the reference's summation order (_kernels.py:27-34)
    from . import _kernels
    t64 = lut.table if _is_tensor(lut.table) else to_device(
        np.asarray(lut.table, dtype=np.float64), torch.float64, tab.device)
    s = _kernels.score_codes(t64, codes_K.device_codes(tab.device))
    return s.cpu().numpy() if host else s


def _decode_codes(codes: torch.Tensor, cfg) -> torch.Tensor:
    """Reference row-layout codes -> the layout the decode kernel reads."""
    if K.is_fast_geometry(cfg.d, cfg.M, cfg.nbits):
        return K.relayout(codes, to_decode=True)
    return codes.contiguous()


_tls = threading.local()


def _step_workspace(cfg, dev) -> "K.DecodeWorkspace":
    """decode_step's single-head workspace, one per (thread, device, geometry)
    (its arrival counters make a workspace single-stream)."""
    cache = getattr(_tls, "ws", None)
    if cache is None:
        cache = _tls.ws = {}
    key = (str(dev), cfg.d, cfg.M, cfg.nbits)
    if key not in cache:
        cache[key] = K.DecodeWorkspace(1, 1, cfg.d, cfg.M, cfg.nbits, device=dev)
    return cache[key]


class _Staging:
    """decode_step's pinned host <-> device staging (q, k_n, v_n, lengths)."""

    def __init__(self, d, dev):
        self.host = torch.empty(3 * d + 2, dtype=torch.float32).pin_memory()
        self.host_i = self.host.view(torch.int32)
        self.dev = torch.empty(3 * d + 2, dtype=torch.float32, device=dev)
        self.dev_i = self.dev.view(torch.int32)
        self.out = torch.empty(d, dtype=torch.float32).pin_memory()


def _step_staging(d, dev) -> _Staging:
    cache = getattr(_tls, "staging", None)
    if cache is None:
        cache = _tls.staging = {}
    key = (str(dev), d)
    if key not in cache:
        cache[key] = _Staging(d, dev)
    return cache[key]


def _n_tensor(n: int, device) -> torch.Tensor:
    # a fill launch with the value as its argument: no host->device copy, no sync
    return torch.full((1,), n, dtype=torch.int32, device=device)


def _partial_from_record(rec: torch.Tensor, host: bool) -> SoftmaxPartial:
    vals = rec.double().cpu().numpy()
    m, l = float(vals[0]), float(vals[1])
    acc = vals[4:].copy() if host else rec[4:].double().clone()
    if l == 0.0:
        m = -np.inf
    return SoftmaxPartial(m=m, l=l, acc=acc)


def quantized_partial(lut: Lut, codes_K: CodesMatrix, codes_V: CodesMatrix, cb_V: Codebook,
                      strategy: str = "auto", counters: Counters | None = None,
                      timings: dict | None = None) -> SoftmaxPartial:
    """Softmax partial over the quantized token span (fused sm_100a kernel)."""
    if codes_K.n_tokens != codes_V.n_tokens:
        raise ValueError(f"key/value token counts differ: {codes_K.n_tokens} vs "
                         f"{codes_V.n_tokens}")
    cfg = cb_V.config
    n = codes_K.n_tokens
    host = not _is_tensor(codes_K.codes)
    if n == 0:
        return empty_partial(cfg.d)
    if strategy not in _STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}")
    tab = _device_table(lut)
    dev = tab.device
    t0 = time.perf_counter()
    _check_codes_for_table(tab, codes_K)  # score_tokens' range check (:88-91) ...
    if counters is not None:  # ... and its work accounting (:93-96), then :153-154
        counters.lut_lookups += n * codes_K.M
        counters.adds += n * codes_K.M
        counters.code_bytes_read += n * codes_K.M * codes_K.cell_width
        counters.code_bytes_read += n * cfg.M * codes_V.cell_width
    ws = _step_workspace(cfg, dev)
    ck = _decode_codes(codes_K.device_codes(dev), cfg).view(1, 1, n, cfg.M)
    cv = _decode_codes(codes_V.device_codes(dev), cfg).view(1, 1, n, cfg.M)
    nq = _n_tensor(n, dev)
    K.decode_partials_lut(ws, 1, tab.view(1, *tab.shape), ck, cv, nq,
                          cb_V.device_value_layout(dev))
    merged = torch.empty((1, cfg.d + 4), dtype=torch.float32, device=dev)
    K.decode_finish(ws, 1, nq, None, 1.0, merged=merged)
    part = _partial_from_record(merged[0], host)
    if timings is not None:
        timings["score"] = timings.get("score", 0.0) + (time.perf_counter() - t0)
    return part


def dense_partial(q_n, K_dense, V_dense, scale: float | None = None,
                  counters: Counters | None = None) -> SoftmaxPartial:
    """Standard softmax partial over full-precision rows, in float64 like the
    reference (pqkv_dense_partial_f64)."""
    host = not _is_tensor(q_n)
    q = to_device(np.asarray(q_n, dtype=np.float64).ravel() if host else q_n.reshape(-1),
                  torch.float64)
    d = q.shape[0]
    Kd = to_device(K_dense if _is_tensor(K_dense) else np.asarray(K_dense, dtype=np.float64),
                   torch.float64, q.device).reshape(-1, d)
    Vd = to_device(V_dense if _is_tensor(V_dense) else np.asarray(V_dense, dtype=np.float64),
                   torch.float64, q.device)
    if Vd.dim() == 1:
        Vd = Vd.view(1, -1)
    if Kd.shape[0] != Vd.shape[0]:
        raise ValueError(f"K rows {Kd.shape[0]} != V rows {Vd.shape[0]}")
    if Kd.shape[0] == 0:
        raise ValueError("dense partial requires at least the current token")
    r = Kd.shape[0]
    if counters is not None:
        counters.dense_bytes_read += 2 * r * d * 4
    rec = K.dense_partial_f64(q, Kd, Vd, _scale(d, scale))
    return _partial_from_record(rec, host)


def merge_partials(a: SoftmaxPartial, b: SoftmaxPartial) -> SoftmaxPartial:
    """Associative, commutative online-softmax merge (attention.py:193-204).

    Device partials merge with pqkv_merge_partials; host partials (the
    reference's own numpy types) use the same closed form."""
    if tuple(a.acc.shape) != tuple(b.acc.shape):
        raise ValueError("partial widths differ")
    if _is_tensor(a.acc) or _is_tensor(b.acc):
        dev = a.acc.device if _is_tensor(a.acc) else b.acc.device
        d = a.acc.shape[0]
        recs = torch.zeros((2, 1, d + 4), dtype=torch.float32, device=dev)
        for k, p in enumerate((a, b)):
            recs[k, 0, 0] = float(p.m) if p.l != 0.0 else 0.0
            recs[k, 0, 1] = float(p.l)
            recs[k, 0, 4:] = to_device(p.acc, torch.float32, dev)
        out = torch.empty((1, d + 4), dtype=torch.float32, device=dev)
        K.merge_partials(recs, merged=out)
        return _partial_from_record(out[0], host=False)
    if a.l == 0.0:
        return SoftmaxPartial(m=b.m, l=b.l, acc=b.acc.copy())
    if b.l == 0.0:
        return SoftmaxPartial(m=a.m, l=a.l, acc=a.acc.copy())
    m = max(a.m, b.m)
    wa = np.exp(a.m - m)
    wb = np.exp(b.m - m)
    return SoftmaxPartial(m=m, l=a.l * wa + b.l * wb, acc=a.acc * wa + b.acc * wb)


def finalize(p: SoftmaxPartial):
    """Normalized attention output acc / l."""
    if p.l <= 0.0:
        raise ValueError("cannot finalize an empty softmax partial")
    return p.acc / p.l


def _decode_step_plan(q_n, k_n, v_n, cache, cb_K, cb_V, sc, dev, counters):
    """decode_step for a LayerKVCache with device tensors: the cache's step
    plan runs the fused decode (lengths read on the device, in stream order)
    and the append of (k_n, v_n) in one library call."""
    cfg = cb_K.config
    d = cfg.d
    q = to_device(q_n, torch.float32, dev).reshape(-1)
    kc = to_device(k_n, torch.float32, dev).reshape(-1)
    vc = to_device(v_n, torch.float32, dev).reshape(-1)
    if q.shape[0] != d:
        raise ValueError(f"query width {q.shape[0]} != codebook d {d}")
    if kc.shape[0] != d or vc.shape[0] != d:
        raise ValueError(f"k_n/v_n width must be d={d}")
    if counters is not None:
        n_q, r = cache.n_q, cache.recent_len()
        counters.lut_lookups += n_q * cfg.M
        counters.adds += n_q * cfg.M
        counters.code_bytes_read += 2 * n_q * cfg.M * cfg.cell_width
        counters.dense_bytes_read += 2 * (r + 1) * d * 4
    out = torch.empty(d, dtype=torch.float32, device=dev)
    cache.decode_append(q.contiguous(), kc.contiguous(), vc.contiguous(), sc,
                        cb_K.device_key_layout(dev), cb_V.device_value_layout(dev),
                        _step_workspace(cfg, dev), out)
    return out


def decode_step(q_n, k_n, v_n, cache, cb_K: Codebook, cb_V: Codebook,
                scale: float | None = None, strategy: str = "auto", block_size: int = 1024,
                counters: Counters | None = None, timings: dict | None = None):
    """One attention decode step against a LayerKVCache, then append (k_n, v_n).

    The snapshot's quantized span is scored through the LUT by the fused
    kernel; recent rows plus the current token form the dense partial; the
    current token is never scored against a quantized copy of itself."""
    cfg = cb_K.config
    if strategy not in _STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}")
    if block_size <= 0:
        raise ValueError("block_size must be positive")
    sc = _scale(cfg.d, scale)
    host = not _is_tensor(q_n)
    dev = getattr(cache, "device", None) or default_device()
    fast = (timings is None and hasattr(cache, "raw_snapshot")
            and K.is_fast_geometry(cfg.d, cfg.M, cfg.nbits))
    if fast and not host and hasattr(cache, "decode_append"):
        return _decode_step_plan(q_n, k_n, v_n, cache, cb_K, cb_V, sc, dev, counters)
    if fast and hasattr(cache, "raw_view"):  # one fused launch: views, stream-ordered
        ck_raw, cv_raw, rk, rv, n_q, _ = cache.raw_view()
    elif hasattr(cache, "raw_snapshot"):     # this package's GPU cache: no layout copies
        ck_raw, cv_raw, rk, rv, n_q, _ = cache.raw_snapshot()
        ck_raw, cv_raw = ck_raw.contiguous(), cv_raw.contiguous()
    else:                                    # any object with the reference snapshot()
        snap = cache.snapshot()
        n_q = snap.codes_K.n_tokens
        ck_raw = _decode_codes(snap.codes_K.device_codes(dev), cfg) if n_q else None
        cv_raw = _decode_codes(snap.codes_V.device_codes(dev), cfg) if n_q else None
        rk, rv = snap.recent_K, snap.recent_V
    if host and fast:
        # one pinned staging transfer for q, k_n, v_n and both lengths
        qh = np.asarray(q_n, dtype=np.float32).ravel()
        kh = np.asarray(k_n, dtype=np.float32).ravel()
        vh = np.asarray(v_n, dtype=np.float32).ravel()
        if qh.shape[0] != cfg.d:
            raise ValueError(f"query width {qh.shape[0]} != codebook d {cfg.d}")
        if kh.shape[0] != cfg.d or vh.shape[0] != cfg.d:
            raise ValueError(f"k_n/v_n width must be d={cfg.d}")
        st = _step_staging(cfg.d, dev)
        d = cfg.d
        st.host[:d] = torch.from_numpy(qh)
        st.host[d:2 * d] = torch.from_numpy(kh)
        st.host[2 * d:3 * d] = torch.from_numpy(vh)
        st.host_i[3 * d] = n_q
        st.host_i[3 * d + 1] = int(rk.shape[0])
        st.dev.copy_(st.host, non_blocking=True)
        q, kc, vc = st.dev[:d], st.dev[d:2 * d], st.dev[2 * d:3 * d]
        nq_dev, nr_dev = st.dev_i[3 * d:3 * d + 1], st.dev_i[3 * d + 1:3 * d + 2]
    else:
        q = to_device(np.asarray(q_n, dtype=np.float64).ravel() if host else q_n.reshape(-1),
                      torch.float32, dev)
        if q.shape[0] != cfg.d:
            raise ValueError(f"query width {q.shape[0]} != codebook d {cfg.d}")
        kc = to_device(k_n if _is_tensor(k_n) else np.asarray(k_n, dtype=np.float32),
                       torch.float32, dev).reshape(-1)
        vc = to_device(v_n if _is_tensor(v_n) else np.asarray(v_n, dtype=np.float32),
                       torch.float32, dev).reshape(-1)
        nq_dev = nr_dev = None
    if kc.shape[0] != cfg.d or vc.shape[0] != cfg.d:
        raise ValueError(f"k_n/v_n width must be d={cfg.d}")

    if fast:
        # one fused launch (quantized span + recent rows + current token, merge,
        # finalize) with a per-thread cached workspace
        ws = _step_workspace(cfg, dev)
        r = int(rk.shape[0])
        out = torch.empty((1, cfg.d), dtype=torch.float32, device=dev)
        if n_q:
            ck = ck_raw.view(1, 1, n_q, cfg.M)
            cv = cv_raw.view(1, 1, n_q, cfg.M)
        else:  # nothing quantized yet: any valid buffer (no code is read)
            ck = cv = torch.zeros((1, 1, 1, cfg.M), dtype=torch.uint8, device=dev)
        K.decode_attention(ws, 1, q.view(1, -1), sc, cb_K.device_key_layout(dev), ck, cv,
                           nq_dev if nq_dev is not None else _n_tensor(n_q, dev),
                           cb_V.device_value_layout(dev),
                           recent_k=rk.view(1, 1, r, cfg.d) if r else None,
                           recent_v=rv.view(1, 1, r, cfg.d) if r else None,
                           n_recent=(nr_dev if nr_dev is not None else _n_tensor(r, dev))
                           if r else None,
                           k_cur=kc.view(1, 1, -1), v_cur=vc.view(1, 1, -1), out=out)
        if counters is not None:
            counters.lut_lookups += n_q * cfg.M
            counters.adds += n_q * cfg.M
            counters.code_bytes_read += 2 * n_q * cfg.M * cfg.cell_width
            counters.dense_bytes_read += 2 * (r + 1) * cfg.d * 4
        if host:
            st.out.copy_(out[0], non_blocking=True)
            cache.append_decode(kc, vc)  # the device rows already uploaded
            torch.cuda.current_stream(dev).synchronize()
            return st.out.numpy().astype(np.float64)
        cache.append_decode(k_n, v_n)
        return out[0]

    t0 = time.perf_counter()
    ws = K.DecodeWorkspace(1, 1, cfg.d, cfg.M, cfg.nbits, device=dev)
    nq_t = _n_tensor(n_q, dev)
    if n_q:  # the LUT is built inside the fused kernel (lut_build time is part of "score")
        ck = ck_raw.view(1, 1, n_q, cfg.M)
        cv = cv_raw.view(1, 1, n_q, cfg.M)
        K.decode_partials(ws, 1, q.view(1, -1), sc, cb_K.device_key_layout(dev), ck, cv, nq_t,
                          cb_V.device_value_layout(dev))
    if counters is not None:
        counters.lut_lookups += n_q * cfg.M
        counters.adds += n_q * cfg.M
        counters.code_bytes_read += 2 * n_q * cfg.M * cfg.cell_width
    if timings is not None:
        t1 = time.perf_counter()
        timings["score"] = timings.get("score", 0.0) + (t1 - t0)
        t0 = t1
    r = int(rk.shape[0])
    rkd = to_device(rk if _is_tensor(rk) else np.asarray(rk, dtype=np.float32), torch.float32,
                    dev).contiguous().view(1, 1, r, cfg.d) if r else None
    rvd = to_device(rv if _is_tensor(rv) else np.asarray(rv, dtype=np.float32), torch.float32,
                    dev).contiguous().view(1, 1, r, cfg.d) if r else None
    if counters is not None:
        counters.dense_bytes_read += 2 * (r + 1) * cfg.d * 4
    # quantized span: the split records merged (fixed order) into one record;
    # dense rows (recent + current token) in float64 as the reference
    # (dense_partial :169-190), merged and finalized in float64 (:193-211)
    dense = K.dense_partial_f64(
        q.double(), torch.cat([rkd.view(r, cfg.d).double() if r else kc.new_empty((0, cfg.d),
                                                                                   dtype=torch.float64),
                               _row64(k_n, dev)]),
        torch.cat([rvd.view(r, cfg.d).double() if r else vc.new_empty((0, cfg.d),
                                                                       dtype=torch.float64),
                   _row64(v_n, dev)]), sc)
    if n_q:
        qrec = torch.empty((1, cfg.d + 4), dtype=torch.float32, device=dev)
        K.decode_finish(ws, 1, nq_t, q.view(1, -1), sc, merged=qrec)
        out = _merge_finalize64(qrec[0].double(), dense)
    else:
        out = dense[4:] / dense[1]
    out = out.view(1, -1)
    if timings is not None:
        t1 = time.perf_counter()
        timings["dense"] = timings.get("dense", 0.0) + (t1 - t0)
        t0 = t1
    flush_before = getattr(cache, "inline_flush_seconds", 0.0)
    cache.append_decode(k_n, v_n)
    if timings is not None:
        t1 = time.perf_counter()
        flush = getattr(cache, "inline_flush_seconds", 0.0) - flush_before
        timings["flush_wait"] = timings.get("flush_wait", 0.0) + flush
        timings["append"] = timings.get("append", 0.0) + (t1 - t0 - flush)
    return out[0].double().cpu().numpy() if host else out[0]


def _row64(x, dev) -> torch.Tensor:
    """The current token's row in float64, as the reference stacks it (:266-267)."""
    return to_device(x if _is_tensor(x) else np.asarray(x, dtype=np.float64), torch.float64,
                     dev).reshape(1, -1)


def _merge_finalize64(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """merge_partials + finalize (:193-211) of two (m, l, 0, 0, acc) float64
    records on the device."""
    if float(a[1]) == 0.0:
        return b[4:] / b[1]
    m = torch.maximum(a[0], b[0])
    wa, wb = torch.exp(a[0] - m), torch.exp(b[0] - m)
    return (a[4:] * wa + b[4:] * wb) / (a[1] * wa + b[1] * wb)


def __getattr__(name):
    # the reference's attention.py also defines prefill_attention (:290-311);
    # here it is in baselines.py (it imports this package's modules)
    if name == "prefill_attention":
        from .baselines import prefill_attention
        return prefill_attention
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
