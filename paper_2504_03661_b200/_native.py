"""ctypes binding of libpqkv_sm100.so (the C ABI declared in include/pqkv_sm100.h).

There is no fallback: if the library is missing or no CUDA device is present,
every entry point raises.  Errors map to the reference's exception classes:
PQKV_EINVAL -> ValueError, PQKV_ECUDA -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from .build import LIB

PQKV_OK, PQKV_EINVAL, PQKV_ECUDA, PQKV_EFORMAT, PQKV_EIO = 0, 1, 2, 3, 4
FILE_HOST, CODES_ROWS, CODES_DECODE = 1, 0, 1
DTYPE_CODE = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2}
PARTIAL_HEADER = 4
DECODE_PDL, DECODE_STATIC_CODEBOOKS, DECODE_F16_VALUE_CODEBOOK, DECODE_EARLY_CODES = 1, 2, 4, 8
DECODE_ONE_HEAD_PER_CTA, DECODE_F16_KEY_TABLE, DECODE_KEY_TABLE_PAIRS = 16, 32, 64
DECODE_APPEND_RECENT = 128  # one head: the finishing CTA appends (k_cur, v_cur) to the ring

_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_F = ctypes.c_float
_PI = ctypes.POINTER(ctypes.c_int)
_PI64 = ctypes.POINTER(ctypes.c_int64)

# name -> (restype, argtypes); mirrors include/pqkv_sm100.h
SIGNATURES = {
    "pqkv_version": (_I, []),
    "pqkv_last_error": (ctypes.c_char_p, []),
    "pqkv_encode": (_I, [_P, _I, _I64, _I, _I64, _P, _I, _I, _P, _I64, _I64, _P]),
    "pqkv_encode_batched": (_I, [_P, _I, _I, _I64, _I, _I64, _I64, _P, _I64, _I, _I, _P, _I64,
                                 _I64, _I64, _P]),
    "pqkv_encode_grid_bytes": (_I64, [_I, _I, _I]),
    "pqkv_build_encode_grid": (_I, [_P, _I, _I, _I, _P, _P]),
    "pqkv_encode_grid": (_I, [_P, _I, _I64, _I, _I64, _P, _P, _I, _I, _P, _I64, _I64, _P]),
    "pqkv_encode_batched_grid": (_I, [_P, _I, _I64, _I, _I64, _I64, _P, _I64, _P, _I64, _I, _I,
                                      _P, _I64, _I64, _I64, _P]),
    "pqkv_relayout_codes": (_I, [_P, _I64, _P, _I64, _I64, _I64, _I, _I, _I, _I, _P]),
    "pqkv_reconstruct": (_I, [_P, _I64, _I64, _P, _I, _I, _I, _P, _P]),
    "pqkv_build_lut": (_I, [_P, _I64, _I, _P, _I, _I, _F, _P, _P]),
    "pqkv_prepare_value_codebook": (_I, [_P, _I, _I, _I, _P, _P]),
    "pqkv_prepare_value_codebook_f16": (_I, [_P, _I, _I, _I, _P, _P]),
    "pqkv_decode_grid": (_I, [_I, _I, _I, ctypes.POINTER(_I)]),
    "pqkv_l2_persist": (_I, [_P, ctypes.c_size_t, _F, _P]),
    "pqkv_partials_floats": (_I64, [_I, _I, _I, _I]),
    "pqkv_prepare_key_codebook": (_I, [_P, _I, _I, _I, _P, _P]),
    "pqkv_decode_partials": (_I, [_P, _F, _P, _P, _I, _I, _I, _P, _P, _I64, _P, _P, _I, _I, _I,
                                  _I, _P, _P]),
    "pqkv_decode_partials_lut": (_I, [_P, _I, _I, _I, _P, _P, _I64, _P, _P, _I, _I, _I, _I, _P,
                                      _P]),
    "pqkv_decode_finish": (_I, [_P, _I, _I, _I, _I, _I, _P, _P, _F, _P, _P, _I64, _P, _P, _P,
                                _P, _P, _P, _P]),
    "pqkv_merge_partials": (_I, [_P, _I, _I64, _I, _P, _P, _P, _P]),
    "pqkv_decode_attention": (_I, [_P, _F, _P, _P, _I, _I, _I, _P, _P, _I64, _P, _P, _I, _I, _I,
                                   _P, _P, _I64, _P, _P, _P, _I, _P, _P, _P, _P, _P, _I, _P]),
    "pqkv_score_codes": (_I, [_P, _P, _I64, _I, _I, _P, _P]),
    "pqkv_accumulate_mass": (_I, [_P, _P, _I64, _I, _I, _P, _P]),
    "pqkv_score_codes_f64": (_I, [_P, _P, _I64, _I, _I, _P, _P]),
    "pqkv_accumulate_mass_f64": (_I, [_P, _P, _I64, _I, _I, _P, _P]),
    "pqkv_build_lut_f64": (_I, [_P, _I64, _I, _P, _I, _I, ctypes.c_double, _P, _P]),
    "pqkv_dense_partial_f64": (_I, [_P, _P, _P, _I64, _I, ctypes.c_double, _P, _P]),
    "pqkv_codebook_file_info": (_I, [ctypes.c_char_p, _PI, _PI, _PI, _PI]),
    "pqkv_read_codebook": (_I, [ctypes.c_char_p, _I, _P, _P, _P]),
    "pqkv_write_codebook": (_I, [ctypes.c_char_p, _I, _I, _I, _I, _P, _I, _P]),
    "pqkv_cache_dump_info": (_I, [ctypes.c_char_p, _I64, _PI, _PI, _PI, _PI64, _PI, _PI64]),
    "pqkv_write_cache_dumps": (_I, [ctypes.c_char_p, _I, _I, _I, _I, _I64, _I, _P, _P, _I64, _I,
                                    _P, _P, _I64, _P]),
    "pqkv_read_cache_dumps": (_I, [ctypes.c_char_p, _I, _I, _I, _I, _I64, _I, _P, _P, _I64, _I,
                                   _P, _P, _I64, _P]),
    "pqkv_debug_delayed_fill": (_I, [_P, _I, _I, ctypes.c_longlong, _P]),
    "pqkv_append_recent": (_I, [_P, _P, _P, _P, _P, _I, _P]),
    "pqkv_publish_lengths": (_I, [_P, _I, _P]),
    "pqkv_step_plan_create": (_I, [_P, _P, _P, _P, _I64, _P, _F, _I, _I, _I, _I, _P, _P,
                                   ctypes.POINTER(_P)]),
    "pqkv_step_run": (_I, [_P, _P, _P, _P, _P, _P, _I64, _I, _P, _P]),
    "pqkv_step_plan_destroy": (_I, [_P]),
    "pqkv_vstore_granularity": (_I64, [_I]),
    "pqkv_vstore_create": (_I, [_I, _I64, _I64, _P, _P]),
    "pqkv_vstore_ensure": (_I, [_P, _I64]),
    "pqkv_vstore_mapped": (_I64, [_P]),
    "pqkv_vstore_region_bytes": (_I64, [_P]),
    "pqkv_vstore_destroy": (_I, [_P]),
}

_lib = None
_lock = threading.Lock()


def library_path() -> str:
    return os.environ.get("PQKV_SM100_LIB", LIB)


def load(require_cuda: bool = True):
    """Load the sm_100a library (idempotent).  Raises if it is missing."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                path = library_path()
                if not os.path.exists(path):
                    raise RuntimeError(
                        f"libpqkv_sm100.so not found at {path}; build it with "
                        "`python -m paper_2504_03661_b200.build` (there is no CPU fallback)")
                lib = ctypes.CDLL(path)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(lib, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = lib
    if require_cuda and not torch.cuda.is_available():
        raise RuntimeError("the PQ KV-cache path needs a CUDA device (sm_100a); none is visible")
    return _lib


def check(rc: int, what: str) -> None:
    if rc == PQKV_OK:
        return
    msg = load(require_cuda=False).pqkv_last_error().decode(errors="replace")
    if rc == PQKV_EINVAL:
        raise ValueError(msg or what)
    if rc == PQKV_EFORMAT:
        from .fileio import FormatError
        raise FormatError(msg or what)
    if rc == PQKV_EIO:
        raise OSError(msg or what)
    raise RuntimeError(msg or what)


def call(name: str, *args) -> int:
    rc = getattr(load(), name)(*args)
    if SIGNATURES[name][0] is _I and name not in ("pqkv_version",):
        check(rc, name)
    return rc


def ptr(t) -> int | None:
    """Device pointer of a tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None, device=None) -> int:
    """The given stream, else the current stream of `device` (default: the
    current device)."""
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream


def decode_grid(d: int, M: int, nbits: int) -> int:
    n = _I(0)
    call("pqkv_decode_grid", d, M, nbits, ctypes.byref(n))
    return n.value


def partials_floats(num_ctas: int, B: int, Hq: int, d: int) -> int:
    return int(load(require_cuda=False).pqkv_partials_floats(num_ctas, B, Hq, d))
