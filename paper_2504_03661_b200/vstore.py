"""Paged code store: growth without copies (include/pqkv_sm100.h, csrc/vstore.cu).

The reference's code store doubles and copies when it fills
(kv_cache.py:74-76, 217-228).  ``PagedCodeStore`` reserves virtual address
space for ``n_regions`` independent streams of code rows (one per head and
kind) and maps physical pages (CUDA VMM, 2 MiB granules) at the end of every
region as the rows grow; rows never move, so a head's codes stay one
contiguous run for the decode kernel (``ld_tok`` = the region's row
capacity) and the caches grow without copying or re-pointing anything a
captured CUDA graph holds.

``tensor`` views the whole reservation, shape ``(n_regions, max_rows,
*row_shape)``; only rows below ``mapped_rows`` are backed by memory, and every
user reads or writes below the cache's row count, which ``ensure`` maps first.
"""

from __future__ import annotations

import ctypes

import torch

from . import _native as N

__all__ = ["PagedCodeStore"]

_TYPESTR = {torch.uint8: "|u1", torch.uint16: "<u2", torch.int16: "<i2", torch.int32: "<i4"}


class _View:
    """__cuda_array_interface__ exporter over the reservation (keeps the store
    alive as long as any tensor made from it)."""

    def __init__(self, store, shape, dtype):
        self._store = store
        self.__cuda_array_interface__ = {
            "shape": tuple(shape), "typestr": _TYPESTR[dtype], "strides": None,
            "data": (store.base, False), "version": 3}


class PagedCodeStore:
    def __init__(self, n_regions: int, max_rows: int, row_shape: tuple, dtype=torch.uint8,
                 device=None, initial_rows: int = 1):
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        if self.device.type != "cuda":
            raise ValueError("PagedCodeStore lives in device memory")
        dev_index = self.device.index if self.device.index is not None else \
            torch.cuda.current_device()
        self.device = torch.device("cuda", dev_index)
        self.row_shape, self.dtype = tuple(row_shape), dtype
        elt = torch.empty((), dtype=dtype).element_size()
        self.row_bytes = elt
        for s in self.row_shape:
            self.row_bytes *= int(s)
        lib = N.load()
        h, base = ctypes.c_void_p(), ctypes.c_void_p()
        with torch.cuda.device(self.device):
            N.check(lib.pqkv_vstore_create(dev_index, int(n_regions),
                                           int(max_rows) * self.row_bytes, ctypes.byref(h),
                                           ctypes.byref(base)), "pqkv_vstore_create")
        self._h, self.base = h, int(base.value)
        self.n_regions = int(n_regions)
        # the reservation is rounded up to whole pages: a region's row capacity
        self.max_rows = int(lib.pqkv_vstore_region_bytes(h)) // self.row_bytes
        if self.max_rows * self.row_bytes != int(lib.pqkv_vstore_region_bytes(h)):
            raise ValueError("the row size must divide the allocation granularity")
        self.ensure(max(1, initial_rows))
        self.tensor = torch.as_tensor(
            _View(self, (self.n_regions, self.max_rows, *self.row_shape), dtype),
            device=self.device)

    @property
    def mapped_rows(self) -> int:
        return int(N.load().pqkv_vstore_mapped(self._h)) // self.row_bytes

    def ensure(self, rows: int) -> None:
        """Back at least `rows` rows of every region with memory (no copy)."""
        if rows > self.max_rows:
            raise ValueError(f"{rows} rows exceed the store's reservation of {self.max_rows}")
        with torch.cuda.device(self.device):
            N.check(N.load().pqkv_vstore_ensure(self._h, int(rows) * self.row_bytes),
                    "pqkv_vstore_ensure")

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            try:
                N.load().pqkv_vstore_destroy(self._h)
            finally:
                self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass
