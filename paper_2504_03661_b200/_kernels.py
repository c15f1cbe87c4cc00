"""The reference's lower seam (``pqkv._kernels``, _kernels.py:46-65) on the GPU.

``score_codes(lut, codes)`` and ``accumulate_mass(codes, p, ksub)`` keep the
reference's signatures, layouts and float64 results.  They run in
libpqkv_sm100.so (``pqkv_score_codes_f64`` / ``pqkv_accumulate_mass_f64``)
with the numba loops' summation orders -- per token over subspaces from 0.0;
per bin over tokens in order -- so given the same inputs they are
bit-identical to ``_score_codes_jit`` / ``_accumulate_mass_jit``
(_kernels.py:27-43).  numpy in -> numpy float64 out; CUDA tensors in -> CUDA
float64 tensors out (no host sync).

The fused decode kernel does not call this seam: it folds the score into
shared-memory table gathers and the mass / _mass_to_acc GEMV into per-token
FMAs ("Why a register gather").  This module is for reference
callers that use the seam directly.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .pq_core import _is_tensor, to_device

__all__ = ["score_codes", "accumulate_mass", "HAVE_NUMBA"]

HAVE_NUMBA = False  # the reference's flag; the loops here are CUDA kernels


def _codes_dev(codes, dev=None):
    c = codes if _is_tensor(codes) else np.ascontiguousarray(codes)
    if not _is_tensor(c) and c.dtype not in (np.uint8, np.uint16):
        raise ValueError(f"codes must be uint8 or uint16, got {c.dtype}")
    t = to_device(c, device=dev)
    if t.dtype not in (torch.uint8, torch.uint16):
        raise ValueError(f"codes must be uint8 or uint16, got {t.dtype}")
    if t.dim() != 2:
        raise ValueError("codes must be 2-D (n_tokens, M)")
    return t.contiguous()


def _nbits_for(ksub: int) -> int:
    nb = int(ksub).bit_length() - 1
    if ksub < 2 or (1 << nb) != ksub or nb > 16:
        raise ValueError(f"ksub must be a power of two in [2, 65536], got {ksub}")
    return nb


def score_codes(lut, codes):
    """scores[t] = sum_i lut[i, codes[t, i]], float64 (lut is (M, ksub))."""
    host = not _is_tensor(codes)
    c = _codes_dev(codes)
    tab = to_device(lut if _is_tensor(lut) else np.asarray(lut, np.float64), torch.float64,
                    c.device).contiguous()
    n, M = c.shape
    if tab.dim() != 2 or tab.shape[0] != M:
        raise ValueError(f"lut must be (M={M}, ksub), got {tuple(tab.shape)}")
    out = torch.empty(n, dtype=torch.float64, device=c.device)
    if n:
        with torch.cuda.device(c.device):
            N.call("pqkv_score_codes_f64", N.ptr(tab), N.ptr(c), n, M,
                   _nbits_for(tab.shape[1]), N.ptr(out), N.stream_ptr())
    return out.cpu().numpy() if host else out


def accumulate_mass(codes, p, ksub: int):
    """h[i, c] = sum of p[t] over tokens with codes[t, i] == c, float64 (M, ksub)."""
    host = not _is_tensor(codes)
    c = _codes_dev(codes)
    n, M = c.shape
    pd = to_device(p if _is_tensor(p) else np.asarray(p, np.float64), torch.float64,
                   c.device).reshape(-1).contiguous()
    if pd.shape[0] != n:
        raise ValueError(f"p has {pd.shape[0]} weights for {n} tokens")
    h = torch.empty((M, int(ksub)), dtype=torch.float64, device=c.device)
    with torch.cuda.device(c.device):
        N.call("pqkv_accumulate_mass_f64", N.ptr(c), N.ptr(pd), n, M, _nbits_for(ksub),
               N.ptr(h), N.stream_ptr())
    return h.cpu().numpy() if host else h
