"""Pin the CPU oracle (oracle/) against golden vectors produced by the
reference itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import pqkv_oracle as O


def test_encode_random_geometries_bit_exact(golden):
    g = golden("encode")
    gi = 0
    while f"g{gi}_geom" in g:
        d, M, nbits = g[f"g{gi}_geom"]
        got = O.assign_codes(g[f"g{gi}_X"], g[f"g{gi}_cents"], int(nbits))
        np.testing.assert_array_equal(got, g[f"g{gi}_codes"], err_msg=f"geom {gi}")
        gi += 1
    assert gi >= 8


def test_encode_exact_ties_lowest_index(golden):
    g = golden("encode")
    got = O.assign_codes(g["tie_X"], g["tie_cents"], 3)
    np.testing.assert_array_equal(got, g["tie_codes"])


def test_encode_trained_codebooks_bit_exact(golden):
    g = golden("encode")
    for kind in ("k", "v"):
        got = O.assign_codes(g[f"trained_X_{kind}"], g[f"trained_cents_{kind}"], 8)
        np.testing.assert_array_equal(got, g[f"trained_codes_{kind}"])


def test_c_oracle_encoder_matches(golden):
    if O.c_library() is None:
        pytest.skip("oracle C library not built (make -C oracle)")
    g = golden("encode")
    for gi in range(8):
        d, M, nbits = g[f"g{gi}_geom"]
        got = O.c_assign_codes(g[f"g{gi}_X"], g[f"g{gi}_cents"], int(nbits))
        np.testing.assert_array_equal(got, g[f"g{gi}_codes"])
    got = O.c_assign_codes(g["trained_X_k"], g["trained_cents_k"], 8)
    np.testing.assert_array_equal(got, g["trained_codes_k"])


def _replay(g, ci, use_c=False):
    d, M, nbits, R, R_f, npre, steps, bs = (int(x) for x in g[f"c{ci}_params"])
    ck, cv = g[f"c{ci}_cents_k"], g[f"c{ci}_cents_v"]
    cache = O.CacheModel(ck, cv, nbits, R, R_f)
    cache.codes_k = g[f"c{ci}_snap0_codes_k"].copy()
    cache.codes_v = g[f"c{ci}_snap0_codes_v"].copy()
    rk, rv = g[f"c{ci}_snap0_recent_k"], g[f"c{ci}_snap0_recent_v"]
    cache.recent = [(rk[i].copy(), rv[i].copy()) for i in range(rk.shape[0])]
    outs = []
    for s in range(steps):
        assert cache.n_q == g[f"c{ci}_nq"][s]
        k_n, v_n = g[f"c{ci}_steps_k"][s], g[f"c{ci}_steps_v"][s]
        codes_k, codes_v, rk, rv = cache.snapshot()
        q = g[f"c{ci}_q"][s]
        if use_c:
            o = O.c_decode_head(q, k_n, v_n, codes_k, codes_v, rk, rv, ck, cv, nbits,
                                block_size=bs)
        else:
            o = O.decode_from_snapshot(q, k_n, v_n, codes_k, codes_v, rk, rv, ck, cv,
                                       block_size=bs)
        outs.append(o)
        cache.append(k_n, v_n)
    return np.stack(outs), cache


@pytest.mark.parametrize("ci", range(10))
def test_decode_replay_matches_reference(golden, ci):
    g = golden("attention")
    outs, cache = _replay(g, ci)
    np.testing.assert_allclose(outs, g[f"c{ci}_out"], rtol=1e-10, atol=1e-12)
    np.testing.assert_array_equal(cache.codes_k, g[f"c{ci}_final_codes_k"])
    np.testing.assert_array_equal(cache.codes_v, g[f"c{ci}_final_codes_v"])


@pytest.mark.parametrize("ci", range(10))
def test_c_decode_replay_matches_reference(golden, ci):
    if O.c_library() is None:
        pytest.skip("oracle C library not built (make -C oracle)")
    g = golden("attention")
    outs, _ = _replay(g, ci, use_c=True)
    np.testing.assert_allclose(outs, g[f"c{ci}_out"], rtol=1e-10, atol=1e-12)


def test_lut_and_quantized_partial(golden):
    g = golden("attention")
    for ci in range(int(g["ncases"])):
        ck, cv = g[f"c{ci}_cents_k"], g[f"c{ci}_cents_v"]
        q = g[f"c{ci}_q"][0]
        table = O.key_lut(q, ck)
        np.testing.assert_allclose(table, g[f"c{ci}_lut0"], rtol=1e-12, atol=1e-14)
        if f"c{ci}_qp" in g:
            p = O.quantized_partial(table, g[f"c{ci}_snap0_codes_k"], g[f"c{ci}_snap0_codes_v"], cv)
            want = g[f"c{ci}_qp"]
            assert p.m == pytest.approx(want[0], rel=1e-12)
            assert p.l == pytest.approx(want[1], rel=1e-10)
            np.testing.assert_allclose(p.acc, want[2:], rtol=1e-9, atol=1e-12)


def test_merge_dense_finalize(golden):
    g = golden("attention")
    q, K, V = g["merge_q"], g["merge_K"], g["merge_V"]
    a = O.dense_partial(q, K[:13], V[:13])
    b = O.dense_partial(q, K[13:], V[13:])
    ab = O.merge(a, b)
    np.testing.assert_allclose([ab.m, ab.l, *ab.acc], g["merge_ab"], rtol=1e-12)
    np.testing.assert_allclose(O.finalize(ab), g["merge_final"], rtol=1e-12)
    np.testing.assert_allclose(O.finalize(ab), O.naive_attention(q, K, V), rtol=1e-9)


def test_cache_sequences(golden):
    g = golden("cache")
    for tr in range(int(g["ntrials"])):
        R, R_f, npre, n = (int(x) for x in g[f"t{tr}_params"])
        c = O.CacheModel(g["cents_k"], g["cents_v"], 2, R, R_f)
        K, V = g[f"t{tr}_K"], g[f"t{tr}_V"]
        if npre:
            c.prefill(K[:npre], V[:npre])
        for t in range(npre, npre + n):
            c.append(K[t], V[t])
        ck, cv, rk, rv = c.snapshot()
        np.testing.assert_array_equal(ck, g[f"t{tr}_codes_k"])
        np.testing.assert_array_equal(cv, g[f"t{tr}_codes_v"])
        np.testing.assert_array_equal(rk, g[f"t{tr}_recent_k"])
        assert c.n_q == g[f"t{tr}_nq"][0] and c.n_total == g[f"t{tr}_nq"][1]


def test_codebook_file_parse(golden):
    g = golden("fileio")
    for gi in range(3):
        raw = g[f"f{gi}_raw"].tobytes()
        kind, d, M, nbits, cents = O.parse_codebook(raw)
        assert [d, M, nbits, kind] == list(g[f"f{gi}_geom"])
        np.testing.assert_array_equal(cents, g[f"f{gi}_cents"])
    with pytest.raises(ValueError):
        O.parse_codebook(b"XXXX" + raw[4:])
    with pytest.raises(ValueError):
        O.parse_codebook(raw[:-4])


def test_naive_quantized_matches_decode(golden):
    """The dequantize-then-attend oracle agrees with the blockwise restatement."""
    g = golden("attention")
    ci = 2
    d, M, nbits, R, R_f, npre, steps, bs = (int(x) for x in g[f"c{ci}_params"])
    ck, cv = g[f"c{ci}_cents_k"], g[f"c{ci}_cents_v"]
    args = (g[f"c{ci}_snap0_codes_k"], g[f"c{ci}_snap0_codes_v"], ck, cv,
            g[f"c{ci}_snap0_recent_k"], g[f"c{ci}_snap0_recent_v"],
            g[f"c{ci}_steps_k"][0], g[f"c{ci}_steps_v"][0])
    a = O.naive_quantized_attention(g[f"c{ci}_q"][0], *args)
    np.testing.assert_allclose(a, g[f"c{ci}_out"][0], rtol=1e-9)


# ------------------------------------------------ wide codes, seam, batched --

@pytest.mark.parametrize("ci", range(2))
def test_oracle_replays_wide_code_streams(golden, ci):
    """uint16 cells (nbits 12 / 10): the oracle replays the reference's
    decode_step streams (attention_wide.npz)."""
    g = golden("attention_wide")
    outs, cache = _replay(g, ci)
    np.testing.assert_allclose(outs, g[f"c{ci}_out"], rtol=1e-10, atol=1e-12)
    np.testing.assert_array_equal(cache.codes_k, g[f"c{ci}_final_codes_k"])
    np.testing.assert_array_equal(cache.codes_v, g[f"c{ci}_final_codes_v"])


def test_oracle_seam_bit_exact(golden):
    """The oracle's score / mass loops equal the reference's numba seam bit for bit."""
    g = golden("seam")
    for ci in range(3):
        codes, lut, p = g[f"s{ci}_codes"], g[f"s{ci}_lut"], g[f"s{ci}_p"]
        np.testing.assert_array_equal(O.score_codes(lut, codes), g[f"s{ci}_scores"])
        np.testing.assert_array_equal(O.accumulate_mass(codes, p, lut.shape[1]),
                                      g[f"s{ci}_mass"])


def test_c_batched_gqa_oracle_matches_numpy_oracle():
    """oracle_decode_gqa_mt (the full-shape GPU tests' checker) == the numpy
    oracle per query head, ragged lengths and recent windows."""
    if O.c_library() is None:
        pytest.skip("oracle C library not built (make -C oracle)")
    rng = np.random.default_rng(0)
    B, Hq, Hkv, n, R = 3, 6, 2, 400, 5
    ck = rng.standard_normal((64, 256, 2)).astype(np.float32)
    cv = rng.standard_normal((64, 256, 2)).astype(np.float32)
    q = rng.standard_normal((B, Hq, 128))
    kc = rng.integers(0, 256, (B, Hkv, n, 64), dtype=np.uint8)
    vc = rng.integers(0, 256, (B, Hkv, n, 64), dtype=np.uint8)
    rk = rng.standard_normal((B, Hkv, R, 128)).astype(np.float32)
    rv = rng.standard_normal((B, Hkv, R, 128)).astype(np.float32)
    kn = rng.standard_normal((B, Hkv, 128)).astype(np.float32)
    vn = rng.standard_normal((B, Hkv, 128)).astype(np.float32)
    nq = np.array([400, 0, 17], np.int32)
    nr = np.array([5, 2, 0], np.int32)
    got = O.c_decode_batched(q, kn, vn, kc, vc, nq, rk, rv, nr, ck, cv, 8, threads=2)
    G = Hq // Hkv
    for b in range(B):
        for h in range(Hq):
            kv = h // G
            want = O.decode_from_snapshot(q[b, h], kn[b, kv], vn[b, kv], kc[b, kv, :nq[b]],
                                          vc[b, kv, :nq[b]], rk[b, kv, :nr[b]],
                                          rv[b, kv, :nr[b]], ck, cv, block_size=8192)
            np.testing.assert_allclose(got[b, h], want, rtol=1e-12, atol=1e-13)
