"""CPU-side checks of the drop-in boundary: the C-ABI library loads without a
GPU, exports every entry point include/pqkv_sm100.h declares, validates
arguments before touching CUDA, and the Python mirror keeps the reference's
signatures and errors."""

import inspect
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "pqkv_sm100.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*(pqkv_\w+)\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2504_03661_b200 import _native as N
    from paper_2504_03661_b200 import build as B
    if not os.path.exists(N.library_path()):
        B.build()
    return N.load(require_cuda=False)


def test_header_symbols_exported(lib):
    names = _declared()
    assert len(names) >= 12
    from paper_2504_03661_b200 import _native as N
    for name in names:
        assert hasattr(lib, name), name
        assert name in N.SIGNATURES, f"{name} has no ctypes signature"


def test_no_torch_types_in_header():
    src = open(os.path.join(ROOT, "include", "pqkv_sm100.h")).read()
    assert "torch" not in src.replace("no torch", "") and "at::" not in src
    assert 'extern "C"' in src


def test_bad_arguments_fail_before_cuda(lib):
    from paper_2504_03661_b200 import _native as N
    assert lib.pqkv_version() == 1
    # d not divisible by M -> EINVAL with a message, no CUDA call needed
    rc = lib.pqkv_encode(None, 0, 10, 130, 130, None, 64, 8, None, 64, -1, None)
    assert rc == N.PQKV_EINVAL
    assert b"geometry" in lib.pqkv_last_error()
    rc = lib.pqkv_decode_partials(None, 0.1, None, None, 1, 6, 4, None, None, 0, None, None,
                                  128, 64, 8, 1, None, None)
    assert rc == N.PQKV_EINVAL and b"multiple" in lib.pqkv_last_error()
    rc = lib.pqkv_prepare_value_codebook(None, 128, 32, 8, None, None)
    assert rc == N.PQKV_EINVAL
    with pytest.raises(ValueError):
        N.check(N.PQKV_EINVAL, "x")
    # n == 0 is a no-op success
    assert lib.pqkv_encode(None, 0, 0, 128, 128, None, 64, 8, None, 64, -1, None) == 0
    # the decode layout exists only for m64b8
    assert lib.pqkv_encode(None, 0, 5, 64, 64, None, 32, 8, None, 32, 0, None) == N.PQKV_EINVAL
    # the fused ring append is a one-head flag; the step plan checks its pointers
    rc = lib.pqkv_decode_attention(None, 0.1, None, None, 2, 2, 2, None, None, 0, None, None,
                                   128, 64, 8, None, None, 0, None, None, None, 4, None, None,
                                   None, None, None, N.DECODE_APPEND_RECENT, None)
    assert rc == N.PQKV_EINVAL and b"APPEND_RECENT" in lib.pqkv_last_error()
    assert lib.pqkv_step_run(None, None, None, None, None, None, 0, 0, None,
                             None) == N.PQKV_EINVAL


def test_partials_size(lib):
    from paper_2504_03661_b200 import _native as N
    # split records + one dense-window record per head
    assert N.partials_floats(148, 16, 32, 128) == (4 * 148 + 2 * 16 * 32) * 132


def test_reference_signatures_kept():
    """Same parameter names/defaults as the reference public API (pqkv/__init__.py)."""
    import paper_2504_03661_b200 as P
    exp = {
        "assign_codes": ["X", "cb"],
        "reconstruct": ["codes", "cb"],
        "build_key_lut": ["q_n", "cb_K", "scale"],
        "score_tokens": ["lut", "codes_K", "counters"],
        "quantized_partial": ["lut", "codes_K", "codes_V", "cb_V", "strategy", "counters",
                              "timings"],
        "dense_partial": ["q_n", "K_dense", "V_dense", "scale", "counters"],
        "merge_partials": ["a", "b"],
        "finalize": ["p"],
        "decode_step": ["q_n", "k_n", "v_n", "cache", "cb_K", "cb_V", "scale", "strategy",
                        "block_size", "counters", "timings"],
        "read_codebook": ["path", "config_overrides"],
    }
    for name, params in exp.items():
        got = list(inspect.signature(getattr(P, name)).parameters)
        assert got == params, (name, got)
    cache_params = list(inspect.signature(P.LayerKVCache).parameters)
    assert cache_params[:5] == ["cb_K", "cb_V", "recent_capacity", "flush_threshold", "worker"]
    for m in ("prefill_ingest", "append_decode", "flush_recent", "flush_step", "drain",
              "snapshot", "load_snapshot", "memory_usage", "close"):
        assert hasattr(P.LayerKVCache, m), m


def test_pqconfig_validation_matches_reference():
    import paper_2504_03661_b200 as P
    with pytest.raises(ValueError):
        P.PQConfig(d=130, M=64, nbits=8)
    with pytest.raises(ValueError):
        P.PQConfig(d=128, M=64, nbits=17)
    with pytest.raises(ValueError):
        P.PQConfig(d=0, M=1, nbits=8)
    c = P.PQConfig(128, 64, 8)
    assert (c.dsub, c.ksub, c.cell_width) == (2, 256, 1)
    assert P.PQConfig(128, 32, 12).cell_width == 2
    assert P.bits_per_value(c) == 4.0
    assert P.PRESETS == {"m64b8": (64, 8), "m32b12": (32, 12)}


def test_codebook_and_codes_validation():
    import paper_2504_03661_b200 as P
    cfg = P.PQConfig(8, 4, 2)
    with pytest.raises(ValueError):
        P.Codebook(cfg, np.zeros((4, 4, 3), np.float32))
    bad = np.zeros((4, 4, 2), np.float32)
    bad[0, 0, 0] = np.nan
    with pytest.raises(ValueError):
        P.Codebook(cfg, bad)
    with pytest.raises(ValueError):
        P.Codebook(cfg, np.zeros((4, 4, 2), np.float32), kind="query")
    with pytest.raises(ValueError):
        P.CodesMatrix(np.array([[0, 4, 1, 1]], np.uint8), nbits=2)
    with pytest.raises(ValueError):
        P.CodesMatrix(np.zeros(4, np.uint8), nbits=2)
    cm = P.CodesMatrix(np.array([[255, 0]], np.uint8), nbits=8)
    assert (cm.n_tokens, cm.M, cm.cell_width, cm.nbytes()) == (1, 2, 1, 2)


def test_fileio_host_roundtrip(golden, tmp_path):
    import paper_2504_03661_b200 as P
    g = golden("fileio")
    for gi in range(3):
        p = tmp_path / f"cb{gi}.pqkv"
        p.write_bytes(g[f"f{gi}_raw"].tobytes())
        cb = P.read_codebook(p)
        d, M, nbits, kind = (int(v) for v in g[f"f{gi}_geom"])
        assert (cb.config.d, cb.config.M, cb.config.nbits) == (d, M, nbits)
        assert cb.kind == ("key" if kind == 0 else "value")
        np.testing.assert_array_equal(cb.centroids, g[f"f{gi}_cents"])
        P.write_codebook(tmp_path / "w.pqkv", cb)
        assert (tmp_path / "w.pqkv").read_bytes() == p.read_bytes()
    raw = g["f0_raw"].tobytes()
    for bad in (b"XXXX" + raw[4:], raw[:-4], raw[:4] + b"\x02" + raw[5:]):
        (tmp_path / "bad.pqkv").write_bytes(bad)
        with pytest.raises(P.FormatError):
            P.read_codebook(tmp_path / "bad.pqkv")
    assert issubclass(P.FormatError, ValueError)


def test_cache_dump_roundtrip_host(tmp_path):
    import paper_2504_03661_b200 as P
    rng = np.random.default_rng(0)
    cfg = P.PQConfig(8, 4, 2)
    snap = P.CacheSnapshot(P.CodesMatrix(rng.integers(0, 4, (5, 4)).astype(np.uint8), 2),
                           P.CodesMatrix(rng.integers(0, 4, (5, 4)).astype(np.uint8), 2),
                           rng.standard_normal((3, 8)).astype(np.float32),
                           rng.standard_normal((3, 8)).astype(np.float32), 5, 8)
    P.write_cache_dump(tmp_path / "c.pqkc", snap, cfg)
    back, cfg2 = P.read_cache_dump(tmp_path / "c.pqkc")
    assert cfg2 == cfg and back.n_q == 5 and back.n_total == 8
    np.testing.assert_array_equal(back.codes_K.codes, snap.codes_K.codes)
    np.testing.assert_array_equal(back.recent_V, snap.recent_V)
    raw = (tmp_path / "c.pqkc").read_bytes()
    (tmp_path / "t.pqkc").write_bytes(raw[:-1])
    with pytest.raises(P.FormatError):
        P.read_cache_dump(tmp_path / "t.pqkc")


def test_shard_tokens_cover_exactly_once():
    from paper_2504_03661_b200.engine import shard_tokens
    for n in (0, 1, 7, 131072, 131071):
        for w in (1, 2, 3, 8):
            spans = [shard_tokens(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))


def test_plain_c_consumer_links_and_runs(lib, tmp_path):
    """A C99 host includes the header and links libpqkv_sm100.so directly (the
    serving-engine integration of INTEGRATION.md): version, argument errors
    with messages, no GPU needed for either."""
    import shutil
    import subprocess
    from paper_2504_03661_b200 import _native as N
    if shutil.which("gcc") is None:
        pytest.skip("no C compiler")
    src = tmp_path / "host.c"
    src.write_text(r'''
#include <stdio.h>
#include <string.h>
#include "pqkv_sm100.h"
int main(void) {
    if (pqkv_version() != 1) return 10;
    int rc = pqkv_decode_attention(NULL, 0.1f, NULL, NULL, 1, 6, 4, NULL, NULL, 0, NULL, NULL,
                                   128, 64, 8, NULL, NULL, 0, NULL, NULL, NULL, 1, NULL, NULL,
                                   NULL, NULL, NULL, PQKV_DECODE_PDL, NULL);
    if (rc != PQKV_EINVAL) return 11;
    if (strstr(pqkv_last_error(), "multiple") == NULL) return 12;
    printf("ok %s\n", pqkv_last_error());
    return 0;
}
''')
    libdir = os.path.dirname(N.library_path())
    exe = tmp_path / "host"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    str(src), "-o", str(exe), "-L", libdir, "-l:" + os.path.basename(
                        N.library_path()), "-Wl,-rpath," + libdir], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert r.stdout.startswith("ok")


@pytest.mark.gpu
def test_integration_ctypes_binding_snippet():
    """The ctypes binding INTEGRATION.md shows a pqkv maintainer (a drop-in for
    _kernels.score_codes) runs against the built library and agrees with the
    reference formula on random tables and codes."""
    import re
    import torch
    from paper_2504_03661_b200 import _native as N
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"```python\n(# pqkv/_kernels_sm100\.py.*?)```", doc, re.S).group(1)
    code = code.replace('ctypes.CDLL("libpqkv_sm100.so")', f'ctypes.CDLL({N.library_path()!r})')
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    rng = np.random.default_rng(3)
    lut = rng.standard_normal((16, 256))           # reference Lut.table: (M, ksub)
    codes = rng.integers(0, 256, (500, 16), dtype=np.uint8)
    got = ns["score_codes"](lut, codes)
    want = lut[np.arange(16)[None, :], codes].sum(axis=1)
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5)
    assert torch.cuda.is_available()


def test_product_path_has_no_cpu_fallback():
    """No GPU (this container) -> the reference-API calls raise instead of
    computing on the host; a missing library raises naming the build step
    (a subprocess: the library handle is process-global)."""
    import subprocess
    import sys
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paper_2504_03661_b200 as P
    rng = np.random.default_rng(0)
    cfg = P.PQConfig(128, 64, 8)
    cb = P.Codebook(cfg, rng.standard_normal((64, 256, 2)).astype(np.float32), "key")
    with pytest.raises(RuntimeError, match="CUDA device"):
        P.assign_codes(rng.standard_normal((4, 128)), cb)
    with pytest.raises(RuntimeError, match="CUDA device"):
        P.build_key_lut(rng.standard_normal(128), cb)
    code = ("import os, numpy as np\n"
            "os.environ['PQKV_SM100_LIB'] = '/nonexistent/libpqkv_sm100.so'\n"
            "from paper_2504_03661_b200 import _native as N\n"
            "try:\n    N.load(require_cuda=False)\nexcept RuntimeError as e:\n"
            "    print('raised:', e)\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT,
                       timeout=120)
    assert "raised:" in r.stdout and "no CPU fallback" in r.stdout, r.stdout + r.stderr
