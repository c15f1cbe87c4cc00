"""The reference's full-precision and integer baselines, on the GPU, for
drop-in users: ``IntQuantParams`` / ``integer_quantize`` /
``integer_dequantize`` (``pq_core.py:149-156, 312-354``) and
``prefill_attention`` (``attention.py:290-311``).  Off the PQ decode path
(they feed the accuracy comparisons and the prompt phase); float64 torch
arithmetic on the device, numpy in → numpy out, tensors in → tensors out.

``integer_quantize`` is bit-identical to the reference (the scale and zero
point are formed on the host exactly as there; X / s + z, round-half-to-even
and the clip are elementwise IEEE float64).  ``prefill_attention`` matches
to float64 rounding (its matrix products accumulate in a different order).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .pq_core import _is_tensor, default_device


@dataclass(frozen=True)
class IntQuantParams:
    """Scale / zero-point pair for uniform integer quantization."""

    nbits: int
    s: float
    z: int
    mode: str  # "symmetric" or "asymmetric"


def _f64(x, device):
    if _is_tensor(x):
        return x.to(dtype=torch.float64), True
    dev = torch.device(device) if device is not None else default_device()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).to(dev), False


def integer_quantize(X, nbits: int, mode: str = "asymmetric", device=None):
    """Uniform integer quantization with round-half-to-even (pq_core.py:312-349)."""
    t, was_tensor = _f64(X, device)
    if t.numel() == 0:
        raise ValueError("cannot quantize an empty tensor")
    if not bool(torch.isfinite(t).all()):
        raise ValueError("cannot quantize non-finite values")
    if mode not in ("symmetric", "asymmetric"):
        raise ValueError(f"unknown mode {mode!r}")
    out = (lambda q: q) if was_tensor else (lambda q: q.cpu().numpy())
    if mode == "symmetric":
        half = 1 << (nbits - 1)
        q_min, q_max = -(half - 1), half - 1
        amax = float(t.abs().max())
        if amax == 0.0:
            return (out(torch.zeros(t.shape, dtype=torch.int32, device=t.device)),
                    IntQuantParams(nbits=nbits, s=1.0, z=0, mode=mode))
        s = 2.0 * amax / (q_max - q_min)
        z = 0
    else:
        q_min, q_max = 0, (1 << nbits) - 1
        x_min, x_max = float(t.min()), float(t.max())
        if x_max == x_min:
            z = int(np.round(q_min))
            return (out(torch.full(t.shape, z, dtype=torch.int32, device=t.device)),
                    IntQuantParams(nbits=nbits, s=1.0, z=z, mode=mode))
        s = (x_max - x_min) / (q_max - q_min)
        z = int(np.round(q_min - x_min / s))
    # true division by a device tensor: a Python-float divisor would become a
    # multiply by its rounded reciprocal (1 ulp off at .5 boundaries)
    s_t = torch.tensor(s, dtype=torch.float64, device=t.device)
    Q = torch.clamp(torch.round(t / s_t + z), q_min, q_max).to(torch.int32)
    return out(Q), IntQuantParams(nbits=nbits, s=s, z=z, mode=mode)


def integer_dequantize(Q_X, params: IntQuantParams, device=None):
    """X_hat = (Q_X - z) * s (pq_core.py:352-354)."""
    t, was_tensor = _f64(Q_X, device)
    r = (t - params.z) * params.s
    return r if was_tensor else r.cpu().numpy()


def prefill_attention(Q, K, V, causal: bool = True, scale: float | None = None, device=None):
    """Full-precision prefill attention with causal masking (attention.py:290-311)."""
    q, was_tensor = _f64(Q, device)
    k, _ = _f64(K, q.device if device is None else device)
    v, _ = _f64(V, q.device if device is None else device)
    k, v = k.to(q.device), v.to(q.device)
    if q.shape[1] != k.shape[1] or k.shape[0] != v.shape[0]:
        raise ValueError(f"inconsistent shapes Q{tuple(q.shape)} K{tuple(k.shape)} "
                         f"V{tuple(v.shape)}")
    if scale is None:
        scale = 1.0 / np.sqrt(q.shape[1])
    scores = scale * (q @ k.T)
    if causal:
        n_q, n_k = scores.shape
        ar_k = torch.arange(n_k, device=q.device)[None, :]
        ar_q = torch.arange(n_q, device=q.device)[:, None]
        scores = scores.masked_fill(ar_k > ar_q + (n_k - n_q), float("-inf"))
    scores = scores - scores.max(dim=1, keepdim=True).values
    w = torch.exp(scores)
    r = (w @ v) / w.sum(dim=1, keepdim=True)
    return r if was_tensor else r.cpu().numpy()
