"""PQ codec types and the GPU encoder -- drop-in for the reference ``pq_core``.

Mirrors ``pq_core.py`` of the reference package (PQConfig :31-75, PRESETS
:80-83, Codebook :86-111, CodesMatrix :114-145, assign_codes :269-287,
reconstruct :290-304, bits_per_value :307-309) with the same names, argument
meaning and errors.  Arrays may be numpy arrays (results come back as numpy,
like the reference) or CUDA tensors (results stay on the device, nothing
synchronises).  The arithmetic always runs in libpqkv_sm100.so; there is no
CPU path.  The reference's training names (``kmeans_train``,
``train_codebooks``) are re-exported from ``training.py`` (k-means++ / Lloyd,
offline) and its integer-quantization baseline from
``baselines.py``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import kernels as K

__all__ = ["PQConfig", "PRESETS", "Codebook", "CodesMatrix", "assign_codes", "reconstruct",
           "bits_per_value", "default_device"]


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the PQ KV-cache path needs a CUDA device (sm_100a); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def _is_tensor(x) -> bool:
    return isinstance(x, torch.Tensor)


def to_device(x, dtype=None, device=None) -> torch.Tensor:
    """numpy / torch -> CUDA tensor (no copy if already there with that dtype)."""
    dev = device if device is not None else (x.device if _is_tensor(x) and x.is_cuda
                                             else default_device())
    if _is_tensor(x):
        t = x.to(device=dev, dtype=dtype) if dtype is not None else x.to(device=dev)
    else:
        a = np.asarray(x)
        if dtype is None and a.dtype == np.float64:
            dtype = torch.float32
        t = torch.from_numpy(np.ascontiguousarray(a)).to(device=dev)
        if dtype is not None:
            t = t.to(dtype)
    return t


@dataclass(frozen=True)
class PQConfig:
    """Subspace geometry (pq_core.py:31-75).  kmeans_* / seed drive the
    offline codebook training (training.py)."""

    d: int
    M: int
    nbits: int
    kmeans_iters: int = 25
    kmeans_tol: float = 1e-4
    seed: int = 0

    def __post_init__(self):
        if self.M <= 0 or self.d <= 0:
            raise ValueError(f"d={self.d} and M={self.M} must be positive")
        if self.d % self.M != 0:
            raise ValueError(f"M={self.M} must divide d={self.d}")
        if not 1 <= self.nbits <= 16:
            raise ValueError(f"nbits={self.nbits} out of range [1, 16]")

    @property
    def dsub(self) -> int:
        return self.d // self.M

    @property
    def ksub(self) -> int:
        return 1 << self.nbits

    @property
    def cell_width(self) -> int:
        return 1 if self.nbits <= 8 else 2

    @property
    def code_dtype(self) -> np.dtype:
        return np.dtype(np.uint8 if self.nbits <= 8 else np.uint16)

    @property
    def torch_code_dtype(self) -> torch.dtype:
        return K.code_dtype(self.nbits)


PRESETS: dict[str, tuple[int, int]] = {"m64b8": (64, 8), "m32b12": (32, 12)}


@dataclass
class Codebook:
    """Centroids (M, 2^nbits, dsub) float32 for keys or values of one layer
    (pq_core.py:86-111).  Immutable; the device copies are made once per
    device and cached (codebook load is the only host->device transfer)."""

    config: PQConfig
    centroids: np.ndarray
    kind: str = "key"
    scope: str = "layer"
    _dev: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        expect = (self.config.M, self.config.ksub, self.config.dsub)
        if tuple(self.centroids.shape) != expect:
            raise ValueError(f"centroids shape {tuple(self.centroids.shape)} != expected {expect}")
        c = self.centroids
        finite = bool(torch.isfinite(c).all()) if _is_tensor(c) else bool(np.all(np.isfinite(c)))
        if not finite:
            raise ValueError("codebook contains non-finite centroids")
        if self.kind not in ("key", "value"):
            raise ValueError(f"kind must be 'key' or 'value', got {self.kind!r}")
        if not _is_tensor(c):
            self.centroids = np.ascontiguousarray(np.asarray(c, dtype=np.float32))

    def nbytes(self) -> int:
        return int(np.prod(self.centroids.shape)) * 4

    def device_centroids(self, device=None) -> torch.Tensor:
        dev = torch.device(device) if device is not None else default_device()
        key = ("c", str(dev))
        if key not in self._dev:
            self._dev[key] = to_device(self.centroids, torch.float32, dev).contiguous()
        return self._dev[key]

    def device_encode_grid(self, device=None):
        """The encoder's candidate grid (kernels.encode_grid; None when the
        geometry has none), built once per device."""
        dev = torch.device(device) if device is not None else default_device()
        key = ("g", str(dev))
        if key not in self._dev:
            self._dev[key] = K.encode_grid(self.device_centroids(dev), self.config.nbits)
        return self._dev[key]

    def device_key_layout(self, device=None) -> torch.Tensor:
        """Key codebook as the decode kernel reads it (pqkv_prepare_key_codebook)."""
        dev = torch.device(device) if device is not None else default_device()
        key = ("k", str(dev))
        if key not in self._dev:
            self._dev[key] = K.key_codebook_layout(self.device_centroids(dev), self.config.nbits)
        return self._dev[key]

    def device_value_layout(self, device=None) -> torch.Tensor:
        """Value codebook as the decode kernel reads it (pqkv_prepare_value_codebook)."""
        dev = torch.device(device) if device is not None else default_device()
        key = ("v", str(dev))
        if key not in self._dev:
            self._dev[key] = K.value_codebook_layout(self.device_centroids(dev), self.config.nbits)
        return self._dev[key]


@dataclass
class CodesMatrix:
    """Packed centroid indices, one row of M cells per token (pq_core.py:114-145).

    ``codes`` is a numpy array or a CUDA tensor of uint8 (nbits <= 8) / uint16."""

    codes: object
    nbits: int

    def __post_init__(self):
        c = self.codes
        if c.ndim != 2:
            raise ValueError("codes must be 2-D (n_tokens, M)")
        itemsize = c.element_size() if _is_tensor(c) else c.dtype.itemsize
        size = c.numel() if _is_tensor(c) else c.size
        # cells as wide as nbits can't hold an out-of-range value (pq_core.py:127-130)
        if size and self.nbits < 8 * itemsize and _max_code(c) >= (1 << self.nbits):
            raise ValueError("code value out of range for nbits")

    @property
    def n_tokens(self) -> int:
        return int(self.codes.shape[0])

    @property
    def M(self) -> int:
        return int(self.codes.shape[1])

    @property
    def cell_width(self) -> int:
        c = self.codes
        return c.element_size() if _is_tensor(c) else c.dtype.itemsize

    def nbytes(self) -> int:
        return self.n_tokens * self.M * self.cell_width

    def device_codes(self, device=None) -> torch.Tensor:
        c = self.codes
        if _is_tensor(c) and c.is_cuda:
            return c
        a = np.asarray(c)
        t = torch.from_numpy(np.ascontiguousarray(a.astype(np.uint8 if self.nbits <= 8
                                                           else np.uint16, copy=False)))
        return t.to(device if device is not None else default_device())


def _max_code(c) -> int:
    if _is_tensor(c):
        return int(c.to(torch.int32).max().item())
    return int(np.asarray(c).max())


def _finite_or_raise(x: torch.Tensor) -> None:
    if not bool(torch.isfinite(x).all()):
        raise ValueError("X must be finite")


def assign_codes(X, cb: Codebook) -> CodesMatrix:
    """Encode (n, d) vectors to nearest-centroid indices (pq_core.py:269-287).

    Bit-exact with the reference for float32 / bfloat16 / float16 inputs; ties
    break to the lowest centroid index.  float64 numpy input is rounded to
    float32 first (the reference's cache stores float32, kv_cache.py:115, 123).
    """
    host = not _is_tensor(X)
    if host:
        a = np.asarray(X)
        if a.ndim != 2 or a.shape[1] != cb.config.d:
            raise ValueError(f"X must be (n, {cb.config.d}), got {a.shape}")
        if not np.all(np.isfinite(a)):
            raise ValueError("X must be finite")
        x = to_device(a.astype(np.float32, copy=False), torch.float32)
    else:
        if X.dim() != 2 or X.shape[1] != cb.config.d:
            raise ValueError(f"X must be (n, {cb.config.d}), got {tuple(X.shape)}")
        x = to_device(X)
        if x.dtype not in (torch.float32, torch.bfloat16, torch.float16):
            x = x.float()
        _finite_or_raise(x)
    codes = K.encode(x, cb.device_centroids(x.device), cb.config.nbits,
                     grid=cb.device_encode_grid(x.device))
    if host:
        return CodesMatrix(codes=codes.cpu().numpy(), nbits=cb.config.nbits)
    return CodesMatrix(codes=codes, nbits=cb.config.nbits)


def reconstruct(codes: CodesMatrix, cb: Codebook):
    """Decode codes back to (n, d) float32 (pq_core.py:290-304).  Diagnostic
    only: the attention path never dequantizes."""
    cfg = cb.config
    if codes.M != cfg.M:
        raise ValueError(f"codes have M={codes.M}, codebook expects {cfg.M}")
    c = codes.codes
    host = not _is_tensor(c)
    n = codes.n_tokens
    if n:
        if _max_code(c) >= cfg.ksub:
            raise ValueError("corrupted cache: code value out of codebook range")
    dc = codes.device_codes()
    out = K.reconstruct(dc, cb.device_centroids(dc.device), cfg.nbits)
    return out.cpu().numpy() if host else out


def bits_per_value(config: PQConfig) -> float:
    return config.M * config.nbits / config.d


# The reference's pq_core also defines k-means training (:171-266) and the
# integer-quantization baseline (:149-156, :312-354); here they live in
# training.py / baselines.py and are re-exported lazily (they import this module).
_LAZY = {"kmeans_train": "training", "train_codebooks": "training",
         "IntQuantParams": "baselines", "integer_quantize": "baselines",
         "integer_dequantize": "baselines"}


def __getattr__(name):
    if name in _LAZY:
        import importlib
        return getattr(importlib.import_module(f".{_LAZY[name]}", __package__), name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
