"""Typed torch wrappers over the C ABI (include/pqkv_sm100.h).

This is the B200 counterpart of the reference's lower seam
(``_kernels.py:46-65``) plus the fused decode entry points.  Every function
takes CUDA tensors, enqueues on the current (or given) stream and never
synchronises.  Shapes are validated here, before the call, as the reference
validates in Python (attention.py:75-76, 129-132; pq_core.py:275-278).
"""

from __future__ import annotations

import ctypes
import math

import torch

from . import _native as N


def _call(dev, name, *args):
    """One C-ABI call with `dev` as the current device, so the library's
    launches (and its per-device SM count / attributes) target the tensors'
    GPU even when it is not the caller's current device."""
    with torch.cuda.device(dev):
        return N.call(name, *args)


def _first_dev(*ts):
    for t in ts:
        if t is not None:
            return t.device
    return torch.device("cuda", torch.cuda.current_device())


def _dev_check(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("expected CUDA tensors on the PQ KV-cache path")


def _contig(t):
    return t if t is None or t.is_contiguous() else t.contiguous()


def code_dtype(nbits: int) -> torch.dtype:
    return torch.uint8 if nbits <= 8 else torch.uint16


def encode_grid(centroids: torch.Tensor, nbits: int, stream=None) -> torch.Tensor | None:
    """The candidate grid of a (M, ksub, 2) codebook for encode(..., grid=)
    (pqkv_build_encode_grid; None for geometries without one)."""
    M, ksub, dsub = centroids.shape
    nb = int(N.load(require_cuda=False).pqkv_encode_grid_bytes(M * dsub, M, nbits))
    if nb <= 0:
        return None
    cents = _contig(centroids.float())
    grid = torch.empty(nb, dtype=torch.uint8, device=cents.device)
    _call(cents.device, "pqkv_build_encode_grid", N.ptr(cents), M * dsub, M, nbits, N.ptr(grid),
          N.stream_ptr(stream, cents.device))
    return grid


def encode(x: torch.Tensor, centroids: torch.Tensor, nbits: int, out: torch.Tensor | None = None,
           stream=None, layout: str = "rows", t_first: int = 0, grid=None) -> torch.Tensor:
    """Nearest-centroid codes of x (n, d) -> (n, M); bit-exact with assign_codes.

    layout="rows" is the reference CodesMatrix order; layout="decode" (m64b8)
    writes the decode kernel's layout with row 0 at token index t_first.
    grid: the codebook's encode_grid() (dsub = 2): the filter scans each
    point's candidate list instead of every centroid -- the same codes."""
    _dev_check(x, centroids)
    M, ksub, dsub = centroids.shape
    d = M * dsub
    if x.dim() != 2 or x.shape[1] != d:
        raise ValueError(f"X must be (n, {d}), got {tuple(x.shape)}")
    if x.dtype not in N.DTYPE_CODE:
        x = x.float()
    if x.stride(1) != 1:
        x = x.contiguous()
    n = x.shape[0]
    if out is None:
        out = torch.empty((n, M), dtype=code_dtype(nbits), device=x.device)
    if out.shape[0] != n or out.shape[1] != M or out.stride(1) != 1:
        raise ValueError("codes output must be (n, M) with unit column stride")
    cents = _contig(centroids.float())
    rot = _rot_base(layout, t_first)
    if grid is not None:
        _call(x.device, "pqkv_encode_grid", N.ptr(x), N.DTYPE_CODE[x.dtype], n, d, x.stride(0),
              N.ptr(cents), N.ptr(grid), M, nbits, N.ptr(out), out.stride(0), rot,
              N.stream_ptr(stream, x.device))
        return out
    _call(x.device, "pqkv_encode", N.ptr(x), N.DTYPE_CODE[x.dtype], n, d, x.stride(0), N.ptr(cents), M,
           nbits, N.ptr(out), out.stride(0), rot, N.stream_ptr(stream, x.device))
    return out


def encode_batched(x: torch.Tensor, centroids: torch.Tensor, nbits: int,
                   out: torch.Tensor | None = None, stream=None, layout: str = "rows",
                   t_first: int = 0, grids=None) -> torch.Tensor:
    """encode() over a batch of independent problems in one launch: x (Z, n, d),
    centroids (Z, M, ksub, dsub) -> (Z, n, M) -- e.g. every layer of a cache
    flush, each with its own codebook."""
    _dev_check(x, centroids)
    Z, M, ksub, dsub = centroids.shape
    d = M * dsub
    if x.dim() != 3 or x.shape[0] != Z or x.shape[2] != d:
        raise ValueError(f"X must be ({Z}, n, {d}), got {tuple(x.shape)}")
    x = _contig(x.float())
    n = x.shape[1]
    cents = _contig(centroids.float())
    if out is None:
        out = torch.empty((Z, n, M), dtype=code_dtype(nbits), device=x.device)
    if tuple(out.shape) != (Z, n, M) or not out.is_contiguous():
        raise ValueError("codes output must be a contiguous (Z, n, M) tensor")
    if grids is not None:  # (Z, grid bytes): each problem's encode_grid()
        grids = _contig(grids)
        _call(x.device, "pqkv_encode_batched_grid", N.ptr(x), Z, n, d, d, n * d, N.ptr(cents),
              M * ksub * dsub, N.ptr(grids), grids.shape[1], M, nbits, N.ptr(out), M, n * M,
              _rot_base(layout, t_first), N.stream_ptr(stream, x.device))
        return out
    _call(x.device, "pqkv_encode_batched", N.ptr(x), N.DTYPE_CODE[torch.float32], Z, n, d, d, n * d,
           N.ptr(cents), M * ksub * dsub, M, nbits, N.ptr(out), M, n * M,
           _rot_base(layout, t_first), N.stream_ptr(stream, x.device))
    return out


def _rot_base(layout: str, t_first: int) -> int:
    if layout == "rows":
        return -1
    if layout == "decode":
        if t_first < 0:
            raise ValueError("t_first must be >= 0")
        return int(t_first)
    raise ValueError(f"unknown code layout {layout!r}")


def relayout(codes: torch.Tensor, to_decode: bool, t_first: int = 0, out=None, stream=None):
    """Rows <-> decode layout of an (..., n, 64) uint8 m64b8 code buffer; row
    index counts from t_first along the token axis (dim -2)."""
    _dev_check(codes)
    if codes.shape[-1] != 64 or codes.dtype != torch.uint8:
        raise ValueError("the decode layout exists only for m64b8 uint8 codes")
    src = codes.contiguous()
    out = torch.empty_like(src) if out is None else out
    lead = src.numel() // (src.shape[-2] * 64) if src.numel() else 0
    n = src.shape[-2]
    s2 = src.view(lead, n, 64) if lead else src
    o2 = out.view(lead, n, 64) if lead else out
    if lead > 1 and n % 8 == 0:
        # the layout depends on the token index mod 8 only: all heads at once
        s2, o2, n, lead = s2.view(1, lead * n, 64), o2.view(1, lead * n, 64), lead * n, 1
    for h in range(lead):
        _call(src.device, "pqkv_relayout_codes", N.ptr(s2[h]), 64, N.ptr(o2[h]), 64, n, t_first,
               1 if to_decode else 0, 128, 64, 8, N.stream_ptr(stream, src.device))
    return out


def reconstruct(codes: torch.Tensor, centroids: torch.Tensor, nbits: int, stream=None):
    _dev_check(codes, centroids)
    M, ksub, dsub = centroids.shape
    n = codes.shape[0]
    out = torch.empty((n, M * dsub), dtype=torch.float32, device=codes.device)
    if n == 0:
        return out
    if codes.stride(1) != 1:
        codes = codes.contiguous()
    _call(codes.device, "pqkv_reconstruct", N.ptr(codes), n, codes.stride(0), N.ptr(_contig(centroids)),
           M * dsub, M, nbits, N.ptr(out), N.stream_ptr(stream, codes.device))
    return out


def build_lut(q: torch.Tensor, cb_k: torch.Tensor, nbits: int, scale: float,
              out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """(H, d) queries -> (H, ksub, M) float32 centroid-major key tables."""
    _dev_check(q, cb_k)
    M, ksub, dsub = cb_k.shape
    q = _contig(q.float().reshape(-1, M * dsub))
    H = q.shape[0]
    if out is None:
        out = torch.empty((H, ksub, M), dtype=torch.float32, device=q.device)
    _call(q.device, "pqkv_build_lut", N.ptr(q), H, M * dsub, N.ptr(_contig(cb_k)), M, nbits, float(scale),
           N.ptr(out), N.stream_ptr(stream, q.device))
    return out


def build_lut_f64(q: torch.Tensor, cb_k: torch.Tensor, nbits: int, scale: float,
                  out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """(H, d) float64 queries -> (H, M, ksub) float64 tables (the reference's
    Lut.table layout, build_key_lut attention.py:70-83)."""
    _dev_check(q, cb_k)
    M, ksub, dsub = cb_k.shape
    q = _contig(q.double().reshape(-1, M * dsub))
    H = q.shape[0]
    if out is None:
        out = torch.empty((H, M, ksub), dtype=torch.float64, device=q.device)
    _call(q.device, "pqkv_build_lut_f64", N.ptr(q), H, M * dsub, N.ptr(_contig(cb_k.float())), M,
          nbits, float(scale), N.ptr(out), N.stream_ptr(stream, q.device))
    return out


def dense_partial_f64(q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, scale: float,
                      stream=None) -> torch.Tensor:
    """float64 (m, l, 0, 0, acc[d]) record of softmax(scale q K^T) over the
    rows of K, V (dense_partial, attention.py:169-190)."""
    _dev_check(q, K, V)
    d = q.shape[-1]
    q, K, V = _contig(q.double().reshape(d)), _contig(K.double()), _contig(V.double())
    rec = torch.empty(d + 4, dtype=torch.float64, device=q.device)
    _call(q.device, "pqkv_dense_partial_f64", N.ptr(q), N.ptr(K), N.ptr(V), K.shape[0], d,
          float(scale), N.ptr(rec), N.stream_ptr(stream, q.device))
    return rec


def is_fast_geometry(d: int, M: int, nbits: int) -> bool:
    return d == 128 and M == 64 and nbits == 8


def _layout_out(out, n: int, dtype, device):
    if out is None:
        return torch.empty(n, dtype=dtype, device=device)
    if out.numel() != n or out.dtype != dtype or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous {dtype} buffer of {n} elements")
    return out


def key_codebook_layout(cb_k: torch.Tensor, nbits: int, stream=None, out=None) -> torch.Tensor:
    """The key codebook as the decode kernel reads it (centroid-major for m64b8).
    `out` may place it in a caller buffer (e.g. one allocation for all layers,
    kept L2-resident with pqkv_l2_persist)."""
    M, ksub, dsub = cb_k.shape
    cb_k = _contig(cb_k.float())
    if not is_fast_geometry(M * dsub, M, nbits):
        return cb_k
    out = _layout_out(out, M * ksub * dsub, torch.float32, cb_k.device)
    _call(cb_k.device, "pqkv_prepare_key_codebook", N.ptr(cb_k), M * dsub, M, nbits, N.ptr(out),
           N.stream_ptr(stream, cb_k.device))
    return out


def value_codebook_layout(cb_v: torch.Tensor, nbits: int, stream=None,
                          half: bool = False, out=None) -> torch.Tensor:
    """The value codebook as the decode kernel reads it (re-laid out for m64b8).
    half=True: the fp16 layout for decode_attention(..., f16_value_codebook=True)
    (4-byte gathers; a stated-tolerance mode)."""
    M, ksub, dsub = cb_v.shape
    cb_v = _contig(cb_v.float())
    if half:
        if not is_fast_geometry(M * dsub, M, nbits):
            raise ValueError("the fp16 value-codebook mode exists only for m64b8")
        out = _layout_out(out, M * ksub * dsub, torch.float16, cb_v.device)
        _call(cb_v.device, "pqkv_prepare_value_codebook_f16", N.ptr(cb_v), M * dsub, M, nbits, N.ptr(out),
               N.stream_ptr(stream, cb_v.device))
        return out
    if not is_fast_geometry(M * dsub, M, nbits):
        return cb_v
    out = _layout_out(out, M * ksub * dsub, torch.float32, cb_v.device)
    _call(cb_v.device, "pqkv_prepare_value_codebook", N.ptr(cb_v), M * dsub, M, nbits, N.ptr(out),
           N.stream_ptr(stream, cb_v.device))
    return out


class DecodeWorkspace:
    """Device scratch for one decode launch shape: LUTs and split partials."""

    def __init__(self, B: int, Hq: int, d: int, M: int, nbits: int, device=None,
                 num_ctas: int | None = None):
        self.B, self.Hq, self.d, self.M, self.nbits = B, Hq, d, M, nbits
        self.ksub = 1 << nbits
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        with torch.cuda.device(self.device):
            self.num_ctas = num_ctas or N.decode_grid(d, M, nbits)
        nf = N.partials_floats(self.num_ctas, B, Hq, d)
        self.partials = torch.empty(nf, dtype=torch.float32, device=self.device)
        # arrival counters of the fused launch (self-resetting)
        self.counters = torch.zeros(B * Hq, dtype=torch.int32, device=self.device)
        # the fast path builds its tables in shared memory; other geometries
        # need a global LUT scratch
        self.lut = None if is_fast_geometry(d, M, nbits) else torch.empty(
            (B * Hq, self.ksub, M), dtype=torch.float32, device=self.device)


def _check_codes(ws: DecodeWorkspace, Hkv: int, codes_k, codes_v):
    B, Hq = ws.B, ws.Hq
    if codes_k.shape != codes_v.shape or codes_k.dim() != 4 or tuple(codes_k.shape[:2]) != (B, Hkv):
        raise ValueError("codes must be (B, Hkv, cap, M) and K/V shapes must agree")
    if codes_k.shape[3] != ws.M or not codes_k.is_contiguous() or not codes_v.is_contiguous():
        raise ValueError("codes must be contiguous (B, Hkv, cap, M)")
    if Hq % Hkv:
        raise ValueError(f"Hq={Hq} is not a multiple of Hkv={Hkv}")


def decode_partials(ws: DecodeWorkspace, Hkv: int, q, scale: float, cb_k_layout, codes_k,
                    codes_v, n_q, cb_v_layout, stream=None) -> None:
    """Fused LUT build / score / online softmax / value accumulation over the
    quantized span of every (b, hq).  q: (B*Hq, d) float32; codes (B, Hkv, cap,
    M); n_q (B,) int32 device; codebooks from key/value_codebook_layout."""
    _check_codes(ws, Hkv, codes_k, codes_v)
    _call(codes_k.device, "pqkv_decode_partials", N.ptr(q), float(scale), N.ptr(cb_k_layout), N.ptr(ws.lut),
           ws.B, ws.Hq, Hkv, N.ptr(codes_k), N.ptr(codes_v), codes_k.shape[2], N.ptr(n_q),
           N.ptr(cb_v_layout), ws.d, ws.M, ws.nbits, ws.num_ctas, N.ptr(ws.partials),
           N.stream_ptr(stream, codes_k.device))


def decode_partials_lut(ws: DecodeWorkspace, Hkv: int, lut, codes_k, codes_v, n_q, cb_v_layout,
                        stream=None) -> None:
    """Same from precomputed tables lut (B*Hq, ksub, M) (the Lut-taking API)."""
    _check_codes(ws, Hkv, codes_k, codes_v)
    lut = _contig(lut)
    if tuple(lut.shape) != (ws.B * ws.Hq, ws.ksub, ws.M):
        raise ValueError("lut must be (B*Hq, ksub, M)")
    _call(codes_k.device, "pqkv_decode_partials_lut", N.ptr(lut), ws.B, ws.Hq, Hkv, N.ptr(codes_k),
           N.ptr(codes_v), codes_k.shape[2], N.ptr(n_q), N.ptr(cb_v_layout), ws.d, ws.M,
           ws.nbits, ws.num_ctas, N.ptr(ws.partials), N.stream_ptr(stream, codes_k.device))


def decode_finish(ws: DecodeWorkspace | None, Hkv: int, n_q, q, scale: float, recent_k=None,
                  recent_v=None, n_recent=None, k_cur=None, v_cur=None, out=None, lse=None,
                  merged=None, B: int | None = None, Hq: int | None = None, d: int | None = None,
                  stream=None) -> None:
    """Merge split partials + dense window + current token, finalize.

    recent_k/v: (B, Hkv, R, d) float32; n_recent: (B,) int32; k_cur/v_cur:
    (B, Hkv, d) float32; out: (B*Hq, d); lse: (B*Hq,); merged: (B*Hq, d+4).
    """
    if ws is not None:
        B, Hq, d = ws.B, ws.Hq, ws.d
    ld_recent = 0
    if recent_k is not None:
        if recent_k.shape != recent_v.shape or recent_k.dim() != 4:
            raise ValueError("recent_k/recent_v must both be (B, Hkv, R, d)")
        ld_recent = recent_k.shape[2]
    _call((ws.device if ws is not None else _first_dev(out, merged, lse, q)), "pqkv_decode_finish", N.ptr(ws.partials) if ws is not None else None,
           ws.num_ctas if ws is not None else 0, B, Hq, Hkv, d, N.ptr(n_q), N.ptr(q),
           float(scale), N.ptr(recent_k), N.ptr(recent_v), ld_recent, N.ptr(n_recent),
           N.ptr(k_cur), N.ptr(v_cur), N.ptr(out), N.ptr(lse), N.ptr(merged),
           N.stream_ptr(stream, (ws.device if ws is not None else _first_dev(out, merged, lse, q))))


def decode_attention(ws: DecodeWorkspace, Hkv: int, q, scale: float, cb_k_layout, codes_k,
                     codes_v, n_q, cb_v_layout, recent_k=None, recent_v=None, n_recent=None,
                     k_cur=None, v_cur=None, out=None, lse=None, merged=None, pdl: bool = False,
                     static_codebooks: bool = False, early_codes: bool = False,
                     one_head_per_cta: bool = False, f16_key_table: bool = False,
                     key_table_pairs: bool = False, stream=None) -> None:
    """One fused launch per layer (m64b8): quantized span + dense window +
    fixed-order merge + finalize for every (b, hq); other geometries fall back
    to decode_partials + decode_finish inside the library.

    q: (B*Hq, d) float32; codes (B, Hkv, cap, M); recent (B, Hkv, R, d);
    out (B*Hq, d); lse (B*Hq,); merged (B*Hq, d+4).  pdl lets the launch
    overlap the previous kernel's tail; static_codebooks additionally loads
    the value codebook before waiting for it (the codebooks must then have
    been written before the previous kernel started, e.g. at load time);
    early_codes likewise for n_q and the codes below it (appended by earlier
    steps): the work split and the first code loads then precede the wait.
    f16_key_table (with the fp16 value codebook and an even GQA group): the
    query heads of a CTA share one packed fp16 key table (stated tolerance,
    tests/test_gpu_gqa_tables.py): four per CTA when the group is a multiple
    of 4 (key_table_pairs=True keeps two), else two."""
    _check_codes(ws, Hkv, codes_k, codes_v)
    ld_recent = 0
    if recent_k is not None:
        if recent_k.shape != recent_v.shape or recent_k.dim() != 4:
            raise ValueError("recent_k/recent_v must both be (B, Hkv, R, d)")
        ld_recent = recent_k.shape[2]
    flags = (N.DECODE_PDL if pdl else 0) | (N.DECODE_STATIC_CODEBOOKS if static_codebooks else 0)
    if early_codes:
        flags |= N.DECODE_EARLY_CODES
    if one_head_per_cta:
        flags |= N.DECODE_ONE_HEAD_PER_CTA
    if f16_key_table:
        flags |= N.DECODE_F16_KEY_TABLE
    if key_table_pairs:
        flags |= N.DECODE_KEY_TABLE_PAIRS
    if cb_v_layout.dtype == torch.float16:  # value_codebook_layout(..., half=True)
        flags |= N.DECODE_F16_VALUE_CODEBOOK
    _call(codes_k.device, "pqkv_decode_attention", N.ptr(q), float(scale), N.ptr(cb_k_layout), N.ptr(ws.lut),
           ws.B, ws.Hq, Hkv, N.ptr(codes_k), N.ptr(codes_v), codes_k.shape[2], N.ptr(n_q),
           N.ptr(cb_v_layout), ws.d, ws.M, ws.nbits, N.ptr(recent_k), N.ptr(recent_v), ld_recent,
           N.ptr(n_recent), N.ptr(k_cur), N.ptr(v_cur), ws.num_ctas, N.ptr(ws.partials),
           N.ptr(ws.counters), N.ptr(out), N.ptr(lse), N.ptr(merged), flags,
           N.stream_ptr(stream, codes_k.device))


class StepPlan:
    """pqkv_step_plan for one LayerKVCache head (decode_step's per-token
    path): the per-cache constants are bound once; run() is one C call that
    launches the fused decode and the append of (k, v) to the ring."""

    def __init__(self, cache, cb_k_layout, cb_v_layout, scale: float, ws: DecodeWorkspace):
        cfg = cache.config
        if not is_fast_geometry(cfg.d, cfg.M, cfg.nbits) or ws.B * ws.Hq != 1:
            raise ValueError("StepPlan: m64b8 single-head workspace only")
        self.device = cache.device
        self._keep = (cache._store_k, cache._store_v, cb_k_layout, cb_v_layout, ws)
        h = ctypes.c_void_p()
        _call(self.device, "pqkv_step_plan_create", N.ptr(cb_k_layout), N.ptr(cb_v_layout),
              N.ptr(cache._store_k), N.ptr(cache._store_v), cache._store_k.shape[0],
              N.ptr(cache._lens), float(scale), cfg.d, cfg.M, cfg.nbits, ws.num_ctas,
              N.ptr(ws.partials), N.ptr(ws.counters), ctypes.byref(h))
        self._h = h.value
        self._run = N.load().pqkv_step_run
        self._dev_index = self.device.index if self.device.index is not None else \
            torch.cuda.current_device()

    def run(self, q, k, v, rk_ptr: int, rv_ptr: int, ld_recent: int, out,
            num_ctas: int = 0) -> None:
        if torch.cuda.current_device() != self._dev_index:
            with torch.cuda.device(self._dev_index):
                return self.run(q, k, v, rk_ptr, rv_ptr, ld_recent, out, num_ctas)
        rc = self._run(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), rk_ptr, rv_ptr,
                       ld_recent, num_ctas, out.data_ptr(),
                       torch.cuda.current_stream().cuda_stream)
        if rc:
            N.check(rc, "pqkv_step_run")

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            try:
                N.load().pqkv_step_plan_destroy(h)
            except Exception:  # interpreter teardown
                pass


def merge_partials(parts: torch.Tensor, out=None, lse=None, merged=None, stream=None) -> None:
    """parts (n_parts, n_heads, d+4) -> merged in index order / finalized."""
    n_parts, n_heads, w = parts.shape
    _call(parts.device, "pqkv_merge_partials", N.ptr(_contig(parts)), n_parts, n_heads, w - N.PARTIAL_HEADER,
           N.ptr(out), N.ptr(lse), N.ptr(merged), N.stream_ptr(stream, parts.device))


def score_codes(lut_cm: torch.Tensor, codes: torch.Tensor, nbits: int, stream=None):
    """scores[t] = sum_i lut[code[t,i], i] (lut centroid-major (ksub, M))."""
    n, M = codes.shape
    out = torch.empty(n, dtype=torch.float32, device=codes.device)
    _call(codes.device, "pqkv_score_codes", N.ptr(_contig(lut_cm)), N.ptr(_contig(codes)), n, M, nbits,
           N.ptr(out), N.stream_ptr(stream, codes.device))
    return out


def accumulate_mass(codes: torch.Tensor, p: torch.Tensor, nbits: int, stream=None):
    n, M = codes.shape
    h = torch.empty((M, 1 << nbits), dtype=torch.float32, device=codes.device)
    _call(codes.device, "pqkv_accumulate_mass", N.ptr(_contig(codes)), N.ptr(_contig(p.float())), n, M, nbits,
           N.ptr(h), N.stream_ptr(stream, codes.device))
    return h


def default_scale(d: int) -> float:
    return 1.0 / math.sqrt(d)
