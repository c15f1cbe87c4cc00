"""Binary formats through the C library (reference fileio.py:71-160; its tests
pkg/tests/test_fileio.py:55-157 ported).  Codebook parsing / writing from host
buffers runs on the CPU; the device paths (file <-> HBM, decode layout
converted on the GPU, serving-cache dumps) are ``-m gpu``."""

import numpy as np
import pytest


def _pair(cfg, rng):
    import paper_2504_03661_b200 as P
    shape = (cfg.M, cfg.ksub, cfg.dsub)
    return (P.Codebook(cfg, rng.standard_normal(shape).astype(np.float32), "key"),
            P.Codebook(cfg, rng.standard_normal(shape).astype(np.float32), "value"))


# ------------------------------------------------------------ CPU (host) --

def test_codebook_roundtrip_and_kind(tmp_path):
    import paper_2504_03661_b200 as P
    ck, cv = _pair(P.PQConfig(8, 4, 2), np.random.default_rng(0))
    P.write_codebook(tmp_path / "k.pqkv", ck)
    P.write_codebook(tmp_path / "v.pqkv", cv)
    back = P.read_codebook(tmp_path / "k.pqkv")
    assert back.kind == "key" and back.config.d == 8 and back.config.M == 4
    np.testing.assert_array_equal(back.centroids, ck.centroids)
    assert P.read_codebook(tmp_path / "v.pqkv").kind == "value"
    assert P.fileio.codebook_file_info(tmp_path / "v.pqkv") == ("value", 8, 4, 2)


def test_codebook_c_writer_matches_reference_bytes(golden, tmp_path):
    """The C writer's bytes == files written by the reference (fileio.npz)."""
    import paper_2504_03661_b200 as P
    g = golden("fileio")
    for gi in range(3):
        d, M, nbits, kind = (int(v) for v in g[f"f{gi}_geom"])
        cb = P.Codebook(P.PQConfig(d, M, nbits), g[f"f{gi}_cents"],
                        "key" if kind == 0 else "value")
        P.write_codebook(tmp_path / "w.pqkv", cb)
        assert (tmp_path / "w.pqkv").read_bytes() == g[f"f{gi}_raw"].tobytes()


@pytest.mark.parametrize("mutate,match", [
    (lambda r: b"NOPE" + r[4:], "magic"),
    (lambda r: r[:-4], "floats"),
    (lambda r: r[:-3], "float32"),
    (lambda r: r[:4] + (2).to_bytes(4, "little") + r[8:], "version"),
    (lambda r: r[:8] + b"\x07" + r[9:], "kind"),
    (lambda r: r[:10], "truncated"),
])
def test_codebook_format_errors(tmp_path, mutate, match):
    import paper_2504_03661_b200 as P
    ck, _ = _pair(P.PQConfig(8, 4, 2), np.random.default_rng(1))
    P.write_codebook(tmp_path / "k.pqkv", ck)
    (tmp_path / "bad.pqkv").write_bytes(mutate((tmp_path / "k.pqkv").read_bytes()))
    with pytest.raises(P.FormatError, match=match):
        P.read_codebook(tmp_path / "bad.pqkv")


def test_codebook_wide_cells_roundtrip(tmp_path):
    import paper_2504_03661_b200 as P
    cb, _ = _pair(P.PQConfig(4, 2, 9), np.random.default_rng(2))  # 16-bit cells
    P.write_codebook(tmp_path / "w.pqkv", cb)
    np.testing.assert_array_equal(P.read_codebook(tmp_path / "w.pqkv").centroids, cb.centroids)


def test_missing_file_is_oserror(tmp_path):
    import paper_2504_03661_b200 as P
    with pytest.raises(OSError):
        P.read_codebook(tmp_path / "nope.pqkv")


def test_cache_dump_header_info(tmp_path):
    """The C header parser on a dump written by the reference-format writer."""
    import ctypes
    import paper_2504_03661_b200 as P
    from paper_2504_03661_b200 import fileio
    rng = np.random.default_rng(3)
    snap = P.CacheSnapshot(P.CodesMatrix(rng.integers(0, 4, (5, 4)).astype(np.uint8), 2),
                           P.CodesMatrix(rng.integers(0, 4, (5, 4)).astype(np.uint8), 2),
                           rng.standard_normal((3, 8)).astype(np.float32),
                           rng.standard_normal((3, 8)).astype(np.float32), 5, 8)
    P.write_cache_dump(tmp_path / "c.pqkc", snap, P.PQConfig(8, 4, 2))
    v = [ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int64(), ctypes.c_int(),
         ctypes.c_int64()]
    fileio._host_call("pqkv_cache_dump_info", fileio._cpath(tmp_path / "c.pqkc"), 0,
                      *[ctypes.byref(x) for x in v])
    assert [x.value for x in v] == [8, 4, 2, 5, 3, 32 + 2 * 20 + 2 * 3 * 8 * 4]
    raw = (tmp_path / "c.pqkc").read_bytes()
    (tmp_path / "t.pqkc").write_bytes(raw[:-1])
    with pytest.raises(P.FormatError, match="bytes"):
        fileio._host_call("pqkv_cache_dump_info", fileio._cpath(tmp_path / "t.pqkc"), 0,
                          *[ctypes.byref(x) for x in v])


# -------------------------------------------------------------------- GPU --

@pytest.mark.gpu
def test_codebook_file_straight_to_device(golden, tmp_path):
    """read_codebook(device=): centroids land in HBM from the file, and for
    m64b8 the decode kernel's layout of the file's kind is written on the
    device (== kernels.key/value_codebook_layout)."""
    import torch
    import paper_2504_03661_b200 as P
    from paper_2504_03661_b200 import kernels as K
    g = golden("fileio")
    for gi in range(3):
        p = tmp_path / f"cb{gi}.pqkv"
        p.write_bytes(g[f"f{gi}_raw"].tobytes())
        cb = P.read_codebook(p, device="cuda")
        assert cb.centroids.is_cuda
        np.testing.assert_array_equal(cb.centroids.cpu().numpy(), g[f"f{gi}_cents"])
        d, M, nbits, kind = (int(v) for v in g[f"f{gi}_geom"])
        if K.is_fast_geometry(d, M, nbits):
            ref = torch.from_numpy(g[f"f{gi}_cents"]).cuda()
            want = (K.key_codebook_layout(ref, nbits) if kind == 0
                    else K.value_codebook_layout(ref, nbits))
            got = cb.device_key_layout() if kind == 0 else cb.device_value_layout()
            assert torch.equal(got, want)
        P.write_codebook(tmp_path / "w.pqkv", cb)  # device centroids -> same bytes
        assert (tmp_path / "w.pqkv").read_bytes() == p.read_bytes()


def _gpu_cache(P, cfg, rng, n=300, R=16, R_f=8, worker="sync"):
    ck, cv = _pair(cfg, rng)
    cache = P.LayerKVCache(ck, cv, recent_capacity=R, flush_threshold=R_f, worker=worker)
    import torch
    X = torch.from_numpy(rng.standard_normal((n, cfg.d)).astype(np.float32)).cuda()
    cache.prefill_ingest(X, X.flip(0).contiguous())
    for t in range(5):
        cache.append_decode(X[t], X[-t - 1])
    return cache, ck, cv


@pytest.mark.gpu
@pytest.mark.parametrize("geom", [(128, 64, 8), (8, 4, 2), (16, 4, 10)])
def test_layer_cache_dump_and_restore(tmp_path, geom):
    """dump_cache (C writer, device store -> reference rows) reads back with the
    reference-format parser equal to the snapshot; restore_cache (C reader,
    file -> device store) gives the same state and the same decode output."""
    import torch
    import paper_2504_03661_b200 as P
    rng = np.random.default_rng(4)
    cfg = P.PQConfig(*geom)
    cache, ck, cv = _gpu_cache(P, cfg, rng)
    path = tmp_path / "c.pqkc"
    P.dump_cache(path, cache)
    snap, cfg2 = P.read_cache_dump(path)
    want = cache.snapshot()
    assert cfg2 == cfg and (snap.n_q, snap.n_total) == (want.n_q, want.n_total)
    np.testing.assert_array_equal(snap.codes_K.codes, want.codes_K.codes.cpu().numpy())
    np.testing.assert_array_equal(snap.codes_V.codes, want.codes_V.codes.cpu().numpy())
    np.testing.assert_array_equal(snap.recent_K, want.recent_K.cpu().numpy())
    np.testing.assert_array_equal(snap.recent_V, want.recent_V.cpu().numpy())
    fresh = P.fileio.restore_cache(path, ck, cv, recent_capacity=16, flush_threshold=8)
    assert (fresh.n_q, fresh.n_total) == (cache.n_q, cache.n_total)
    a, b = cache.snapshot(), fresh.snapshot()
    assert torch.equal(a.codes_K.codes, b.codes_K.codes)
    assert torch.equal(a.recent_V, b.recent_V)
    q = torch.randn(cfg.d, device="cuda")
    k, v = torch.randn(cfg.d, device="cuda"), torch.randn(cfg.d, device="cuda")
    o1 = P.decode_step(q, k, v, cache, ck, cv)
    o2 = P.decode_step(q, k, v, fresh, ck, cv)
    assert torch.equal(o1, o2)


@pytest.mark.gpu
def test_dump_errors_on_device_paths(tmp_path):
    import paper_2504_03661_b200 as P
    rng = np.random.default_rng(5)
    cfg = P.PQConfig(8, 4, 2)
    cache, ck, cv = _gpu_cache(P, cfg, rng, n=40, R=4)
    path = tmp_path / "c.pqkc"
    P.dump_cache(path, cache)
    raw = bytearray(path.read_bytes())
    bad = bytearray(raw)
    bad[0] ^= 0xFF
    (tmp_path / "m.pqkc").write_bytes(bytes(bad))
    with pytest.raises(P.FormatError, match="magic"):
        P.fileio.restore_cache(tmp_path / "m.pqkc", ck, cv)
    (tmp_path / "t.pqkc").write_bytes(bytes(raw[:-1]))
    with pytest.raises(P.FormatError, match="bytes"):
        P.fileio.restore_cache(tmp_path / "t.pqkc", ck, cv)
    bad = bytearray(raw)
    bad[32] = 0xFF  # first K cell: out of range for nbits 2
    (tmp_path / "o.pqkc").write_bytes(bytes(bad))
    with pytest.raises(P.FormatError, match="corrupted"):
        P.fileio.restore_cache(tmp_path / "o.pqkc", ck, cv)
    empty = P.LayerKVCache(ck, cv)
    P.dump_cache(tmp_path / "e.pqkc", empty)
    snap, _ = P.read_cache_dump(tmp_path / "e.pqkc")
    assert snap.n_total == 0


@pytest.mark.gpu
@pytest.mark.parametrize("async_flush", [False, True])
def test_serving_cache_dump_load_roundtrip(tmp_path, async_flush):
    """A whole ServingCache (layers x sequences x KV heads) to one file of
    .pqkc records and back: every record equals snapshot(l, b, h) through the
    reference-format parser, and a fresh cache loaded from the file decodes
    bit-identically."""
    import torch
    from paper_2504_03661_b200 import fileio
    from paper_2504_03661_b200.engine import PQDecoder
    from paper_2504_03661_b200.pq_core import PQConfig
    from paper_2504_03661_b200.serving_cache import ServingCache
    rng = np.random.default_rng(6)
    L, B, H, Hq, d = 2, 2, 2, 4, 128
    cfg = PQConfig(d, 64, 8)
    cks = [torch.from_numpy(rng.standard_normal((64, 256, 2)).astype(np.float32)).cuda()
           for _ in range(L)]
    cvs = [torch.from_numpy(rng.standard_normal((64, 256, 2)).astype(np.float32)).cuda()
           for _ in range(L)]
    cache = ServingCache(L, B, H, cfg, cks, cvs, capacity=256, async_flush=async_flush)
    cache.prefill(torch.randn((L, B, H, 120, d), device="cuda"),
                  torch.randn((L, B, H, 120, d), device="cuda"))
    for _ in range(13):
        cache.append(torch.randn((L, B, H, d), device="cuda"),
                     torch.randn((L, B, H, d), device="cuda"))
    path = tmp_path / "serving.pqkc"
    fileio.dump_serving_cache(path, cache)
    raw = path.read_bytes()
    nq, nr = cache.n_quantized, cache.n_recent_rows
    rec = 32 + 2 * nq * 64 + 2 * nr * d * 4
    assert len(raw) == rec * L * B * H
    k = 0
    for l in range(L):
        for b in range(B):
            for h in range(H):
                (tmp_path / "one.pqkc").write_bytes(raw[k * rec:(k + 1) * rec])
                snap, _ = fileio.read_cache_dump(tmp_path / "one.pqkc")
                ck, cv, rk, rv = cache.snapshot(l, b, h)
                np.testing.assert_array_equal(snap.codes_K.codes, ck)
                np.testing.assert_array_equal(snap.codes_V.codes, cv)
                np.testing.assert_array_equal(snap.recent_K, rk)
                np.testing.assert_array_equal(snap.recent_V, rv)
                k += 1
    fresh = ServingCache(L, B, H, cfg, cks, cvs, capacity=256, async_flush=async_flush)
    fileio.load_serving_cache(path, fresh)
    assert (fresh.n_quantized, fresh.n_recent_rows) == (nq, nr)
    dec = PQDecoder(B, Hq, H, cfg)
    q = torch.randn((B, Hq, d), device="cuda")
    kc, vc = torch.randn((B, H, d), device="cuda"), torch.randn((B, H, d), device="cuda")
    for l in range(L):
        o1 = dec(q, k_cur=kc, v_cur=vc, **cache.layer(l)).clone()
        o2 = dec(q, k_cur=kc, v_cur=vc, **fresh.layer(l))
        assert torch.equal(o1, o2)
