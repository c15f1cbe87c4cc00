"""Parity of the sm_100a path (through the C ABI) against the reference's golden
vectors and the CPU oracle.  Needs a B200: run with ``-m gpu``.

Tolerances: codes are bit-exact; attention outputs are float32 on the GPU vs
float64 in the reference, compared at rtol 1e-5 (atol 1e-6) on unit-scale
data -- the reference's own acceptance bar (test_acceptance.py:41-72).
"""

import numpy as np
import pytest
import torch

from oracle import pqkv_oracle as O

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-5, 1e-6


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2504_03661_b200._native as N
    N.load()  # fails loudly if the library is missing


def _np(x):
    """snapshot fields: numpy when the cache was fed numpy (as the reference),
    CUDA tensors when it was fed tensors"""
    return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


def _cb(cents, kind, nbits):
    import paper_2504_03661_b200 as P
    M, ksub, dsub = cents.shape
    return P.Codebook(P.PQConfig(M * dsub, M, nbits), np.asarray(cents, np.float32), kind)


# ------------------------------------------------------------------ encode --

def test_encode_golden_geometries(golden):
    import paper_2504_03661_b200 as P
    g = golden("encode")
    gi = 0
    while f"g{gi}_geom" in g:
        d, M, nbits = (int(v) for v in g[f"g{gi}_geom"])
        cb = _cb(g[f"g{gi}_cents"], "key", nbits)
        got = P.assign_codes(g[f"g{gi}_X"], cb).codes
        np.testing.assert_array_equal(got, g[f"g{gi}_codes"], err_msg=f"geometry {d, M, nbits}")
        gi += 1


def test_encode_exact_ties_lowest_index(golden):
    import paper_2504_03661_b200 as P
    g = golden("encode")
    cb = _cb(g["tie_cents"], "key", 3)
    np.testing.assert_array_equal(P.assign_codes(g["tie_X"], cb).codes, g["tie_codes"])


def test_encode_trained_codebooks(golden):
    import paper_2504_03661_b200 as P
    g = golden("encode")
    for kind in ("k", "v"):
        cb = _cb(g[f"trained_cents_{kind}"], "key", 8)
        np.testing.assert_array_equal(P.assign_codes(g[f"trained_X_{kind}"], cb).codes,
                                      g[f"trained_codes_{kind}"])


def test_encode_large_m64b8_vs_c_oracle():
    """32K vectors of the BASELINE geometry, bit-exact against the C oracle."""
    from paper_2504_03661_b200 import kernels as K
    if O.c_library() is None:
        pytest.skip("oracle C library not built")
    rng = np.random.default_rng(5)
    cents = rng.standard_normal((64, 256, 2)).astype(np.float32)
    X = (rng.standard_normal((32768, 128)) * 1.3).astype(np.float32)
    got = K.encode(torch.from_numpy(X).cuda(), torch.from_numpy(cents).cuda(), 8).cpu().numpy()
    want = O.c_assign_codes(X, cents, 8)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("scale,n", [(1.0, 3072), (1e-3, 3072), (1e3, 3072), (1.0, 12289)])
def test_encode_near_ties_vs_oracle(scale, n):
    """The fp32 filter of the dsub=2 encoder hands near ties to the exact fp64
    scan: vectors on centroids, on midpoints between centroid pairs (exact and
    rounded ties), and nudged by a few ulps off midpoints -- bit-exact against
    the fp64 restatement of assign_codes at three magnitudes, on both the
    4- and the 8-vectors-per-thread scan (n >= 8192) with a ragged tail."""
    from paper_2504_03661_b200 import kernels as K
    rng = np.random.default_rng(11)
    M, ksub = 64, 256
    cents = (rng.standard_normal((M, ksub, 2)) * scale).astype(np.float32)
    # exact duplicate centroids: ties in fp64 -> lowest index
    cents[:, 200] = cents[:, 17]
    X = np.empty((n, 2 * M), dtype=np.float32)
    for i in range(M):
        a = rng.integers(0, ksub, n)
        b = rng.integers(0, ksub, n)
        ca, cb = cents[i, a].astype(np.float64), cents[i, b].astype(np.float64)
        mid = ((ca + cb) / 2).astype(np.float32)
        kind = np.arange(n) % 4
        x = np.where(kind[:, None] == 0, cents[i, a], mid)
        nudge = np.nextafter(mid, np.float32(np.inf) * np.sign(rng.standard_normal((n, 2))))
        x = np.where(kind[:, None] == 2, nudge, x)
        x = np.where(kind[:, None] == 3, cents[i, 17], x)
        X[:, 2 * i: 2 * i + 2] = x
    got = K.encode(torch.from_numpy(X).cuda(), torch.from_numpy(cents).cuda(), 8).cpu().numpy()
    want = O.assign_codes(X, cents, 8)
    np.testing.assert_array_equal(got, want)
    assert (got[3::4] == 17).all()  # duplicates of centroid 17 resolve to the lower index


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_encode_half_inputs(dtype):
    """bf16/f16 rows are upcast exactly; codes equal the oracle on the upcast values."""
    from paper_2504_03661_b200 import kernels as K
    rng = np.random.default_rng(6)
    cents = rng.standard_normal((64, 256, 2)).astype(np.float32)
    X = torch.from_numpy(rng.standard_normal((2048, 128)).astype(np.float32)).to(dtype)
    got = K.encode(X.cuda(), torch.from_numpy(cents).cuda(), 8).cpu().numpy()
    want = O.assign_codes(X.float().numpy(), cents, 8)
    np.testing.assert_array_equal(got, want)


def test_encode_strided_output_rows():
    """Encoding straight into a slice of a larger code store (the cache flush path)."""
    from paper_2504_03661_b200 import kernels as K
    rng = np.random.default_rng(7)
    cents = rng.standard_normal((64, 256, 2)).astype(np.float32)
    X = rng.standard_normal((100, 128)).astype(np.float32)
    store = torch.full((300, 64), 7, dtype=torch.uint8, device="cuda")
    K.encode(torch.from_numpy(X).cuda(), torch.from_numpy(cents).cuda(), 8, out=store[50:150])
    s = store.cpu().numpy()
    np.testing.assert_array_equal(s[50:150], O.assign_codes(X, cents, 8))
    assert (s[:50] == 7).all() and (s[150:] == 7).all()


@pytest.mark.parametrize("t_first", [0, 3, 1000])
def test_encode_decode_layout_is_relayout_of_rows(t_first):
    """The decode layout written by the encoder == relayout(row layout), and
    relayout round-trips."""
    from paper_2504_03661_b200 import kernels as K
    rng = np.random.default_rng(9)
    cents = torch.from_numpy(rng.standard_normal((64, 256, 2)).astype(np.float32)).cuda()
    X = torch.from_numpy(rng.standard_normal((333, 128)).astype(np.float32)).cuda()
    rows = K.encode(X, cents, 8)
    dec = K.encode(X, cents, 8, layout="decode", t_first=t_first)
    assert torch.equal(dec, K.relayout(rows, True, t_first=t_first))
    assert torch.equal(K.relayout(dec, False, t_first=t_first), rows)
    if t_first % 8:
        assert not torch.equal(dec, K.relayout(rows, True, t_first=0))


def test_reconstruct_matches_oracle():
    import paper_2504_03661_b200 as P
    rng = np.random.default_rng(8)
    for (d, M, nbits) in [(128, 64, 8), (8, 4, 2), (128, 32, 12)]:
        cfg = P.PQConfig(d, M, nbits)
        cents = rng.standard_normal((M, cfg.ksub, cfg.dsub)).astype(np.float32)
        codes = rng.integers(0, cfg.ksub, (77, M)).astype(cfg.code_dtype)
        cb = P.Codebook(cfg, cents, "value")
        got = P.reconstruct(P.CodesMatrix(codes, nbits), cb)
        np.testing.assert_array_equal(got, O.reconstruct(codes, cents))


# -------------------------------------------------------------- attention --

def test_lut_matches_golden(golden):
    import paper_2504_03661_b200 as P
    g = golden("attention")
    for ci in range(int(g["ncases"])):
        d, M, nbits = (int(v) for v in g[f"c{ci}_params"][:3])
        lut = P.build_key_lut(g[f"c{ci}_q"][0], _cb(g[f"c{ci}_cents_k"], "key", nbits))
        np.testing.assert_allclose(lut.table, g[f"c{ci}_lut0"], rtol=2e-6, atol=2e-6)


def test_quantized_partial_matches_golden(golden):
    import paper_2504_03661_b200 as P
    g = golden("attention")
    seen = 0
    for ci in range(int(g["ncases"])):
        if f"c{ci}_qp" not in g:
            continue
        d, M, nbits = (int(v) for v in g[f"c{ci}_params"][:3])
        ck, cv = _cb(g[f"c{ci}_cents_k"], "key", nbits), _cb(g[f"c{ci}_cents_v"], "value", nbits)
        lut = P.build_key_lut(g[f"c{ci}_q"][0], ck)
        p = P.quantized_partial(lut, P.CodesMatrix(g[f"c{ci}_snap0_codes_k"], nbits),
                                P.CodesMatrix(g[f"c{ci}_snap0_codes_v"], nbits), cv)
        want = g[f"c{ci}_qp"]
        assert p.m == pytest.approx(want[0], rel=RTOL, abs=ATOL)
        np.testing.assert_allclose(P.finalize(p), want[2:] / want[1], rtol=RTOL, atol=ATOL)
        seen += 1
    assert seen >= 5


@pytest.mark.parametrize("ci", range(10))
def test_decode_step_replay_matches_reference(golden, ci):
    """Replay the reference's decode_step streams through the GPU cache."""
    import paper_2504_03661_b200 as P
    g = golden("attention")
    d, M, nbits, R, R_f, npre, steps, bs = (int(x) for x in g[f"c{ci}_params"])
    ck, cv = _cb(g[f"c{ci}_cents_k"], "key", nbits), _cb(g[f"c{ci}_cents_v"], "value", nbits)
    cache = P.LayerKVCache(ck, cv, recent_capacity=R, flush_threshold=R_f, worker="sync")
    snap0 = P.CacheSnapshot(P.CodesMatrix(g[f"c{ci}_snap0_codes_k"], nbits),
                            P.CodesMatrix(g[f"c{ci}_snap0_codes_v"], nbits),
                            g[f"c{ci}_snap0_recent_k"], g[f"c{ci}_snap0_recent_v"],
                            int(g[f"c{ci}_nq"][0]),
                            int(g[f"c{ci}_nq"][0]) + g[f"c{ci}_snap0_recent_k"].shape[0])
    cache.load_snapshot(snap0)
    outs = []
    for s in range(steps):
        assert cache.n_q == g[f"c{ci}_nq"][s]
        outs.append(P.decode_step(g[f"c{ci}_q"][s], g[f"c{ci}_steps_k"][s],
                                  g[f"c{ci}_steps_v"][s], cache, ck, cv, block_size=bs))
    np.testing.assert_allclose(np.stack(outs), g[f"c{ci}_out"], rtol=RTOL, atol=ATOL)
    fin = cache.snapshot()
    np.testing.assert_array_equal(_np(fin.codes_K.codes), g[f"c{ci}_final_codes_k"])
    np.testing.assert_array_equal(_np(fin.codes_V.codes), g[f"c{ci}_final_codes_v"])


def test_dense_merge_finalize_golden(golden):
    import paper_2504_03661_b200 as P
    g = golden("attention")
    q, Kd, Vd = g["merge_q"], g["merge_K"], g["merge_V"]
    a = P.dense_partial(q, Kd[:13], Vd[:13])
    b = P.dense_partial(q, Kd[13:], Vd[13:])
    np.testing.assert_allclose([a.m, a.l, *a.acc], g["merge_a"], rtol=RTOL, atol=ATOL)
    ab = P.merge_partials(a, b)
    np.testing.assert_allclose(P.finalize(ab), g["merge_final"], rtol=RTOL, atol=ATOL)
    # device partials merge on the GPU
    da = P.SoftmaxPartial(a.m, a.l, torch.from_numpy(a.acc).float().cuda())
    db = P.SoftmaxPartial(b.m, b.l, torch.from_numpy(b.acc).float().cuda())
    dab = P.merge_partials(da, db)
    np.testing.assert_allclose(P.finalize(dab).cpu().numpy(), g["merge_final"], rtol=RTOL,
                               atol=ATOL)
    with pytest.raises(ValueError):
        P.dense_partial(q, Kd[:0], Vd[:0])
    with pytest.raises(ValueError):
        P.finalize(P.empty_partial(8))


def test_empty_cache_first_step_returns_v1():
    """test_attention.py:207-215: with nothing cached the output is v_n."""
    import paper_2504_03661_b200 as P
    rng = np.random.default_rng(3)
    cfg = P.PQConfig(128, 64, 8)
    ck = P.Codebook(cfg, rng.standard_normal((64, 256, 2)).astype(np.float32), "key")
    cv = P.Codebook(cfg, rng.standard_normal((64, 256, 2)).astype(np.float32), "value")
    cache = P.LayerKVCache(ck, cv)
    v = rng.standard_normal(128).astype(np.float32)
    out = P.decode_step(rng.standard_normal(128), rng.standard_normal(128), v, cache, ck, cv)
    np.testing.assert_allclose(out, v, rtol=1e-6, atol=1e-6)


# ------------------------------------------------------------- batched path --

def _oracle_heads(q, ck_codes, cv_codes, n_q, rk, rv, n_r, kcur, vcur, cents_k, cents_v, G):
    """Per (b, hq) oracle: snapshot -> LUT -> quantized + dense partials -> finalize."""
    B, Hq, d = q.shape
    out = np.zeros((B, Hq, d))
    for b in range(B):
        for h in range(Hq):
            kv = h // G
            n = n_q[b]
            out[b, h] = O.decode_from_snapshot(
                q[b, h], kcur[b, kv], vcur[b, kv], ck_codes[b, kv, :n], cv_codes[b, kv, :n],
                rk[b, kv, :n_r[b]], rv[b, kv, :n_r[b]], cents_k, cents_v, block_size=1 << 30)
    return out


def _batched_case(B, Hq, Hkv, cap, n_q, n_r, R=32, seed=0, num_ctas=None, half_cv=False,
                  f16_keys=False, pairs=False, q_scale=1.0):
    from paper_2504_03661_b200 import kernels as K
    from paper_2504_03661_b200.engine import PQDecoder
    import paper_2504_03661_b200 as P
    rng = np.random.default_rng(seed)
    cfg = P.PQConfig(128, 64, 8)
    cents_k = rng.standard_normal((64, 256, 2)).astype(np.float32)
    cents_v = rng.standard_normal((64, 256, 2)).astype(np.float32)
    q = (rng.standard_normal((B, Hq, 128)) * q_scale).astype(np.float32)
    codes_k = rng.integers(0, 256, (B, Hkv, cap, 64), dtype=np.uint8)
    codes_v = rng.integers(0, 256, (B, Hkv, cap, 64), dtype=np.uint8)
    rk = rng.standard_normal((B, Hkv, R, 128)).astype(np.float32)
    rv = rng.standard_normal((B, Hkv, R, 128)).astype(np.float32)
    kc = rng.standard_normal((B, Hkv, 128)).astype(np.float32)
    vc = rng.standard_normal((B, Hkv, 128)).astype(np.float32)
    dev = torch.device("cuda")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    dec = PQDecoder(B, Hq, Hkv, cfg, num_ctas=num_ctas, f16_key_table=f16_keys,
                    key_table_pairs=pairs)
    cbk = K.key_codebook_layout(t(cents_k), 8)
    cbv = K.value_codebook_layout(t(cents_v), 8, half=half_cv)
    dk, dv = K.relayout(t(codes_k), True), K.relayout(t(codes_v), True)  # decode layout
    out = dec(t(q), dk, dv, t(np.array(n_q, np.int32)), cbk, cbv, t(rk), t(rv),
              t(np.array(n_r, np.int32)), t(kc), t(vc))
    want = _oracle_heads(q, codes_k, codes_v, n_q, rk, rv, n_r, kc, vc, cents_k, cents_v,
                         Hq // Hkv)
    if half_cv:  # the oracle on the fp16-rounded value codebook too
        want16 = _oracle_heads(q, codes_k, codes_v, n_q, rk, rv, n_r, kc, vc, cents_k,
                               cents_v.astype(np.float16).astype(np.float32), Hq // Hkv)
        return out.cpu().numpy(), want, want16
    return out.cpu().numpy(), want


@pytest.mark.parametrize("B,Hq,Hkv,cap,n_q,n_r", [
    (1, 4, 4, 3000, [3000], [31]),                    # MHA, multi-CTA per head
    (2, 8, 2, 5000, [4999, 1234], [5, 32]),           # GQA 4:1, ragged lengths
    (3, 2, 1, 700, [0, 1, 7], [0, 3, 0]),             # empty / tiny quantized spans
    (1, 1, 1, 100000, [100000], [0]),                 # long single head
])
def test_batched_decoder_vs_oracle(B, Hq, Hkv, cap, n_q, n_r):
    got, want = _batched_case(B, Hq, Hkv, cap, n_q, n_r)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("q_scale", [0.05, 8.0])
@pytest.mark.parametrize("B,Hq,Hkv,cap,n_q,n_r", [
    (1, 4, 4, 6000, [6000], [31]),                    # MHA
    (2, 8, 2, 9000, [8999, 4321], [5, 32]),           # GQA 4:1 (exact: CTA pairs)
])
def test_lazy_rescale_dynamic_range(B, Hq, Hkv, cap, n_q, n_r, q_scale):
    """The online softmax moves its running max only past a 2^8 margin
    (decode.cu kLazyRescale): flat (q x 0.05) and very peaked (q x 8, scores
    spanning hundreds of log2 units, many max jumps) distributions stay
    within the exact tolerance -- its atol scaled by max(1, q_scale): the fp32
    table's absolute score error grows with |q| (the same bits with the lazy
    margin off, PQKV_LAZY_RESCALE=0); the fp16 modes at q x 2, the largest
    scale their stated tolerance covers (test_gpu_gqa_tables.py; at q x 3 the
    packed fp16 key table exceeds it with or without the lazy margin,
    scripts/lazy_err.py)."""
    got, want = _batched_case(B, Hq, Hkv, cap, n_q, n_r, q_scale=q_scale)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL * max(1.0, q_scale))
    s16 = min(q_scale, 2.0)
    for keys in ([False, True] if Hq != Hkv else [False]):
        got, want, want16 = _batched_case(B, Hq, Hkv, cap, n_q, n_r, half_cv=True,
                                          f16_keys=keys, q_scale=s16)
        np.testing.assert_allclose(got, want16, rtol=2e-3, atol=2e-4)


@pytest.mark.parametrize("B,Hq,Hkv,cap,n_q,n_r,num_ctas", [
    (2, 8, 2, 5000, [4999, 1234], [5, 32], None),           # G = 4
    (1, 8, 1, 20000, [20000], [7], None),                   # G = 8: two virtual heads
    (4, 32, 8, 3000, [3000, 17, 0, 2222], [31, 0, 3, 17], None),  # Llama-3 grouping, ragged
    (3, 4, 1, 700, [0, 1, 9], [0, 3, 31], 2),               # one pair, tiny / empty spans
    (2, 16, 4, 4000, [4000, 2500], [8, 8], 9),              # odd grid: 4 pairs
])
def test_gqa_exact_cta_pairs(B, Hq, Hkv, cap, n_q, n_r, num_ctas):
    """Exact GQA with a group that is a multiple of 4: clusters of two CTAs
    (decode_gqa_pair), each CTA one half of the subspaces for four query heads,
    partial scores exchanged through distributed shared memory -- the exact
    path's tolerance, and the one-head-per-CTA launch agrees."""
    got, want = _batched_case(B, Hq, Hkv, cap, n_q, n_r, num_ctas=num_ctas)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


def test_gqa_exact_pairs_match_one_head_per_cta():
    from paper_2504_03661_b200 import kernels as K
    B, Hq, Hkv, n, R = 2, 8, 2, 6000, 16
    x = _fused_inputs(B, Hq, Hkv, n, R, 19)
    cv = K.value_codebook_layout(
        torch.from_numpy(np.random.default_rng(19).standard_normal((64, 256, 2)).astype(
            np.float32)).cuda(), 8)
    nq = torch.tensor([6000, 2500], dtype=torch.int32, device="cuda")
    nr = torch.tensor([16, 3], dtype=torch.int32, device="cuda")
    outs = []
    for one in (False, True):
        ws = K.DecodeWorkspace(B, Hq, 128, 64, 8)
        out = torch.empty((B * Hq, 128), device="cuda")
        for _ in range(2):  # the self-resetting counters serve a second launch
            K.decode_attention(ws, Hkv, x["q"], 0.09, x["cbk"], x["ck"], x["cv"], nq, cv,
                               recent_k=x["rk"], recent_v=x["rv"], n_recent=nr, k_cur=x["kc"],
                               v_cur=x["vc"], out=out, one_head_per_cta=one)
        assert int(ws.counters.abs().sum()) == 0
        outs.append(out.cpu().numpy())
    np.testing.assert_allclose(outs[0], outs[1], rtol=2e-6, atol=1e-6)


@pytest.mark.parametrize("num_ctas", [7, 148, 150, 1000])
def test_gqa_shared_stream_grids(num_ctas):
    """GQA 8:1 exact: the 8 CTAs of a group split the same token ranges of one
    KV head's 8 query heads (shared code stream); grids not divisible by 8
    fall back to groups of 4, 2 or 1 -- all match the oracle."""
    got, want = _batched_case(2, 16, 2, 6000, [6000, 2500], [9, 31], num_ctas=num_ctas)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("B,Hq,Hkv,cap,n_q,n_r", [
    (1, 4, 4, 3000, [3000], [31]),                   # MHA: one query head per CTA
    (2, 8, 2, 5000, [4999, 1234], [5, 32]),          # G = 4: two query heads per CTA
    (3, 2, 1, 700, [0, 1, 7], [0, 3, 0]),            # G = 2, empty / tiny spans
    (2, 6, 2, 4100, [4100, 333], [31, 0]),           # G = 3 (odd): one head per CTA
    (1, 8, 1, 20000, [20000], [7]),                  # G = 8, many CTAs per virtual head
])
def test_f16_value_codebook_mode(B, Hq, Hkv, cap, n_q, n_r):
    """PQKV_DECODE_F16_VALUE_CODEBOOK: the value codebook is stored as fp16
    and the softmax weights enter the value sums as fp16 (round to nearest,
    2^-12 relative each); the sums and the normaliser stay fp32.  Stated
    tolerance: vs the fp64 oracle run on the fp16-rounded codebook, rtol 1e-3
    / atol 1e-4 (the weight rounding alone); vs the fp64 oracle on the
    original codebook, rtol 2e-3 / atol 2e-4."""
    got, want, want16 = _batched_case(B, Hq, Hkv, cap, n_q, n_r, half_cv=True)
    np.testing.assert_allclose(got, want16, rtol=1e-3, atol=1e-4)
    np.testing.assert_allclose(got, want, rtol=2e-3, atol=2e-4)


def test_f16_two_heads_per_cta_matches_one():
    """The fp16 GQA pairing (a CTA serves two query heads, one value gather per
    code for both) agrees with the one-head-per-CTA launch within the mode's
    weight rounding: the split points differ, so the running maxima the fp16
    weights are rounded against differ (2^-12 relative per weight)."""
    from paper_2504_03661_b200 import kernels as K
    B, Hq, Hkv, n, R = 2, 8, 2, 6000, 16
    x = _fused_inputs(B, Hq, Hkv, n, R, 9)
    cv16 = K.value_codebook_layout(
        torch.from_numpy(np.random.default_rng(9).standard_normal((64, 256, 2)).astype(
            np.float32)).cuda(), 8, half=True)
    nq = torch.tensor([6000, 2500], dtype=torch.int32, device="cuda")
    nr = torch.tensor([16, 3], dtype=torch.int32, device="cuda")
    outs = []
    for one in (False, True):
        ws = K.DecodeWorkspace(B, Hq, 128, 64, 8)
        out = torch.empty((B * Hq, 128), device="cuda")
        K.decode_attention(ws, Hkv, x["q"], 0.09, x["cbk"], x["ck"], x["cv"], nq, cv16,
                           recent_k=x["rk"], recent_v=x["rv"], n_recent=nr, k_cur=x["kc"],
                           v_cur=x["vc"], out=out, one_head_per_cta=one)
        assert int(ws.counters.abs().sum()) == 0
        outs.append(out.cpu().numpy())
    np.testing.assert_allclose(outs[0], outs[1], rtol=1e-3, atol=1e-4)


@pytest.mark.parametrize("half", [False, True])
def test_static_codebook_staging_bit_identical(half):
    """With static codebooks and early codes (PQKV_DECODE_STATIC_CODEBOOKS |
    EARLY_CODES, PDL) the value codebook and the first code ring are loaded
    before the grid-dependency wait; the result is bit-identical to the plain
    launch."""
    from paper_2504_03661_b200 import kernels as K
    B, Hq, Hkv, n, R = 2, 8, 8, 7000, 20
    x = _fused_inputs(B, Hq, Hkv, n, R, 21)
    cbv = x["cbv"]
    if half:
        cbv = K.value_codebook_layout(
            torch.from_numpy(np.random.default_rng(21).standard_normal((64, 256, 2)).astype(
                np.float32)).cuda(), 8, half=True)
    nq = torch.tensor([7000, 1234], dtype=torch.int32, device="cuda")
    nr = torch.tensor([20, 0], dtype=torch.int32, device="cuda")
    outs = []
    for static in (False, True, True):
        ws = K.DecodeWorkspace(B, Hq, 128, 64, 8)
        out = torch.empty((B * Hq, 128), device="cuda")
        K.decode_attention(ws, Hkv, x["q"], 0.09, x["cbk"], x["ck"], x["cv"], nq, cbv,
                           recent_k=x["rk"], recent_v=x["rv"], n_recent=nr, k_cur=x["kc"],
                           v_cur=x["vc"], out=out, pdl=static, static_codebooks=static,
                           early_codes=static)
        torch.cuda.synchronize()
        outs.append(out)
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])


def _fused_inputs(B, Hq, Hkv, n, R, seed):
    from paper_2504_03661_b200 import kernels as K
    rng = np.random.default_rng(seed)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    return dict(
        q=t(rng.standard_normal((B * Hq, 128)).astype(np.float32)),
        cbk=K.key_codebook_layout(t(rng.standard_normal((64, 256, 2)).astype(np.float32)), 8),
        cbv=K.value_codebook_layout(t(rng.standard_normal((64, 256, 2)).astype(np.float32)), 8),
        ck=t(rng.integers(0, 256, (B, Hkv, n, 64), dtype=np.uint8)),
        cv=t(rng.integers(0, 256, (B, Hkv, n, 64), dtype=np.uint8)),
        rk=t(rng.standard_normal((B, Hkv, R, 128)).astype(np.float32)),
        rv=t(rng.standard_normal((B, Hkv, R, 128)).astype(np.float32)),
        kc=t(rng.standard_normal((B, Hkv, 128)).astype(np.float32)),
        vc=t(rng.standard_normal((B, Hkv, 128)).astype(np.float32)))


@pytest.mark.parametrize("pdl", [False, True])
def test_fused_launch_matches_two_launch_path(pdl):
    """pqkv_decode_attention (one launch: dense window by the CTA holding a
    head's last tokens, last-arriver merge) == pqkv_decode_partials +
    pqkv_decode_finish, for out, lse and the merged record; counters return to
    zero.  The fused launch splits GQA heads differently (the CTAs of one KV
    head's query heads share token ranges), so the partial sums associate
    differently: fp32 reassociation tolerance."""
    from paper_2504_03661_b200 import kernels as K
    B, Hq, Hkv, n, R = 3, 8, 4, 9000, 32
    x = _fused_inputs(B, Hq, Hkv, n, R, 5)
    nq = torch.tensor([9000, 17, 0], dtype=torch.int32, device="cuda")
    nr = torch.tensor([31, 0, 5], dtype=torch.int32, device="cuda")
    ws = K.DecodeWorkspace(B, Hq, 128, 64, 8)
    sc = K.default_scale(128)
    o1 = torch.empty((B * Hq, 128), device="cuda")
    l1 = torch.empty(B * Hq, device="cuda")
    m1 = torch.empty((B * Hq, 132), device="cuda")
    K.decode_partials(ws, Hkv, x["q"], sc, x["cbk"], x["ck"], x["cv"], nq, x["cbv"])
    K.decode_finish(ws, Hkv, nq, x["q"], sc, x["rk"], x["rv"], nr, x["kc"], x["vc"], out=o1,
                    lse=l1, merged=m1)
    o2, l2, m2 = torch.empty_like(o1), torch.empty_like(l1), torch.empty_like(m1)
    for _ in range(3):  # repeated launches reuse the self-resetting counters
        K.decode_attention(ws, Hkv, x["q"], sc, x["cbk"], x["ck"], x["cv"], nq, x["cbv"],
                           x["rk"], x["rv"], nr, x["kc"], x["vc"], out=o2, lse=l2, merged=m2,
                           pdl=pdl, static_codebooks=pdl)
    torch.cuda.synchronize()
    assert int(ws.counters.abs().sum()) == 0
    np.testing.assert_allclose(o2.cpu().numpy(), o1.cpu().numpy(), rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(l2.cpu().numpy(), l1.cpu().numpy(), rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(m2.cpu().numpy(), m1.cpu().numpy(), rtol=1e-5, atol=1e-5)


def test_fused_graph_replay_deterministic():
    """A CUDA-graph-captured multi-layer step with PDL launches replays to the
    same bits every time (fixed merge order, static work split)."""
    from paper_2504_03661_b200 import kernels as K
    B, Hq, Hkv, n, R, L = 1, 32, 32, 6000, 31, 3
    xs = [_fused_inputs(B, Hq, Hkv, n, R, 40 + l) for l in range(L)]
    nq = torch.tensor([n], dtype=torch.int32, device="cuda")
    nr = torch.tensor([R], dtype=torch.int32, device="cuda")
    ws = K.DecodeWorkspace(B, Hq, 128, 64, 8)
    outs = torch.zeros((L, B * Hq, 128), device="cuda")
    torch.cuda.synchronize()
    st = torch.cuda.Stream()

    def step():
        for l, x in enumerate(xs):
            K.decode_attention(ws, Hkv, x["q"], K.default_scale(128), x["cbk"], x["ck"], x["cv"],
                               nq, x["cbv"], x["rk"], x["rv"], nr, x["kc"], x["vc"],
                               out=outs[l], pdl=True, static_codebooks=True, stream=st)

    with torch.cuda.stream(st):
        step()
    st.synchronize()
    ref = outs.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        step()
    for _ in range(4):
        outs.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(outs, ref)
    # and against the oracle for one head of each layer
    for l, x in enumerate(xs):
        h = 7
        ckr = K.relayout(x["ck"], False).cpu().numpy()
        cvr = K.relayout(x["cv"], False).cpu().numpy()
        want = O.decode_from_snapshot(
            x["q"][h].cpu().numpy(), x["kc"][0, h].cpu().numpy(), x["vc"][0, h].cpu().numpy(),
            ckr[0, h], cvr[0, h], x["rk"][0, h].cpu().numpy(), x["rv"][0, h].cpu().numpy(),
            *_plain_codebooks(x), block_size=1 << 30)
        np.testing.assert_allclose(ref[l, h].cpu().numpy(), want, rtol=RTOL, atol=ATOL)


def _plain_codebooks(x):
    """Invert the fast-path codebook layouts back to (M, ksub, dsub)."""
    ck = x["cbk"].view(256, 64, 2).permute(1, 0, 2).contiguous().cpu().numpy()
    cv = x["cbv"].view(2, 256, 32, 2).permute(0, 2, 1, 3).reshape(64, 256, 2).cpu().numpy()
    return ck, cv


def test_batched_decoder_more_ctas_than_tokens():
    got, want = _batched_case(2, 2, 2, 64, [40, 9], [1, 2], num_ctas=300)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


def test_batched_decoder_config2_layer_vs_c_oracle():
    """One Llama-2-7B layer at 32K context (BASELINE config 2 shape), all 32
    heads, against the float64 C oracle."""
    from paper_2504_03661_b200 import kernels as K
    from paper_2504_03661_b200.engine import PQDecoder
    import paper_2504_03661_b200 as P
    if O.c_library() is None:
        pytest.skip("oracle C library not built")
    rng = np.random.default_rng(11)
    H, n, R = 32, 32768, 31
    cents_k = rng.standard_normal((64, 256, 2)).astype(np.float32)
    cents_v = rng.standard_normal((64, 256, 2)).astype(np.float32)
    q = rng.standard_normal((1, H, 128)).astype(np.float32)
    ck = rng.integers(0, 256, (1, H, n, 64), dtype=np.uint8)
    cv = rng.integers(0, 256, (1, H, n, 64), dtype=np.uint8)
    rk = rng.standard_normal((1, H, R, 128)).astype(np.float32)
    rv = rng.standard_normal((1, H, R, 128)).astype(np.float32)
    kc = rng.standard_normal((1, H, 128)).astype(np.float32)
    vc = rng.standard_normal((1, H, 128)).astype(np.float32)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    dec = PQDecoder(1, H, H, P.PQConfig(128, 64, 8))
    out = dec(t(q), K.relayout(t(ck), True), K.relayout(t(cv), True), t(np.array([n], np.int32)),
              K.key_codebook_layout(t(cents_k), 8),
              K.value_codebook_layout(t(cents_v), 8), t(rk), t(rv),
              t(np.array([R], np.int32)), t(kc), t(vc)).cpu().numpy()[0]
    lib = O.c_library()
    want = np.empty((H, 128))
    import ctypes
    P_ = ctypes.c_void_p
    qd = np.ascontiguousarray(q[0], np.float64)
    rc = lib.oracle_decode_heads_mt(
        qd.ctypes.data_as(P_), kc[0].ctypes.data_as(P_), vc[0].ctypes.data_as(P_),
        ck[0].ctypes.data_as(P_), cv[0].ctypes.data_as(P_), n, n,
        rk[0].ctypes.data_as(P_), rv[0].ctypes.data_as(P_), R,
        cents_k.ctypes.data_as(P_), cents_v.ctypes.data_as(P_), 64, 8, 2,
        1.0 / np.sqrt(128.0), 8192, want.ctypes.data_as(P_), H, 8)
    assert rc == 0
    np.testing.assert_allclose(out, want, rtol=RTOL, atol=ATOL)


# ---------------------------------------------- full-size properties (config 2) --

def _full_layer(seed=13, H=32, n=32768, R=31):
    """One config-2 layer as device tensors (decode layout) + a decoder."""
    from paper_2504_03661_b200 import kernels as K
    from paper_2504_03661_b200.engine import PQDecoder
    import paper_2504_03661_b200 as P
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    x = dict(q=torch.randn((1, H, 128), generator=g, device="cuda"),
             ck=torch.randint(0, 256, (1, H, n, 64), generator=g, device="cuda",
                              dtype=torch.uint8),
             cv=torch.randint(0, 256, (1, H, n, 64), generator=g, device="cuda",
                              dtype=torch.uint8),
             cents_k=torch.randn((64, 256, 2), generator=g, device="cuda"),
             cents_v=torch.randn((64, 256, 2), generator=g, device="cuda"),
             rk=torch.randn((1, H, R, 128), generator=g, device="cuda"),
             rv=torch.randn((1, H, R, 128), generator=g, device="cuda"),
             kc=torch.randn((1, H, 128), generator=g, device="cuda"),
             vc=torch.randn((1, H, 128), generator=g, device="cuda"),
             nq=torch.tensor([n], dtype=torch.int32, device="cuda"),
             nr=torch.tensor([R], dtype=torch.int32, device="cuda"))
    dec = PQDecoder(1, H, H, P.PQConfig(128, 64, 8))

    def run(ck=None, cv=None, cents_v=None, rv=None, vc=None):
        ck = x["ck"] if ck is None else ck
        cv = x["cv"] if cv is None else cv
        return dec(x["q"], K.relayout(ck, True), K.relayout(cv, True), x["nq"],
                   K.key_codebook_layout(x["cents_k"], 8),
                   K.value_codebook_layout(x["cents_v"] if cents_v is None else cents_v, 8),
                   x["rk"], x["rv"] if rv is None else rv, x["nr"], x["kc"],
                   x["vc"] if vc is None else vc)
    return x, run


def test_full_layer_constant_values_pass_through():
    """All 32K value codes of every subspace on one centroid, and the recent /
    current value rows equal to that centroid's reconstruction: the output is
    that vector whatever the scores (a convex combination of one point)."""
    x, run = _full_layer()
    cv = torch.full_like(x["cv"], 7)
    v7 = x["cents_v"][:, 7, :].reshape(-1)  # (128,)
    H = x["q"].shape[1]
    out = run(cv=cv, rv=v7.expand_as(x["rv"]).contiguous(), vc=v7.expand_as(x["vc"]).contiguous())
    np.testing.assert_allclose(out.cpu().numpy(), v7.expand(1, H, 128).cpu().numpy(),
                               rtol=1e-5, atol=1e-5)


def test_full_layer_token_permutation_invariance():
    """Permuting the quantized tokens (K and V codes together) leaves the
    output unchanged: the kernel's split points see different tokens, the
    softmax does not care (fp32 reassociation only)."""
    x, run = _full_layer(seed=17)
    perm = torch.randperm(x["ck"].shape[2], device="cuda")
    a = run().cpu().numpy()
    b = run(ck=x["ck"][:, :, perm].contiguous(), cv=x["cv"][:, :, perm].contiguous()).cpu().numpy()
    np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6)


def test_full_layer_affine_in_values():
    """out(a C_V + b, a V_recent + b, a v_n + b) = a out(...) + b: the output
    is a softmax-weighted average of value rows, the weights depend on keys
    only."""
    x, run = _full_layer(seed=19)
    a_, b_ = 1.75, -0.5
    base = run().cpu().numpy()
    out = run(cents_v=a_ * x["cents_v"] + b_, rv=a_ * x["rv"] + b_,
              vc=a_ * x["vc"] + b_).cpu().numpy()
    np.testing.assert_allclose(out, a_ * base + b_, rtol=1e-5, atol=1e-5)


def test_sequence_split_merge_equals_full():
    """Sequence split (config 4 pattern) on one GPU: W token ranges decoded to
    partial records, merged in rank order == the unsplit decode."""
    from paper_2504_03661_b200 import kernels as K
    from paper_2504_03661_b200.engine import PQDecoder, shard_tokens
    import paper_2504_03661_b200 as P
    rng = np.random.default_rng(12)
    B, Hq, Hkv, n, W = 2, 8, 2, 20000, 4
    cfg = P.PQConfig(128, 64, 8)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    cbk = K.key_codebook_layout(t(rng.standard_normal((64, 256, 2)).astype(np.float32)), 8)
    cbv = K.value_codebook_layout(t(rng.standard_normal((64, 256, 2)).astype(np.float32)), 8)
    q = t(rng.standard_normal((B, Hq, 128)).astype(np.float32))
    ckr = t(rng.integers(0, 256, (B, Hkv, n, 64), dtype=np.uint8))   # row layout
    cvr = t(rng.integers(0, 256, (B, Hkv, n, 64), dtype=np.uint8))
    ck, cv = K.relayout(ckr, True), K.relayout(cvr, True)
    rk = t(rng.standard_normal((B, Hkv, 16, 128)).astype(np.float32))
    rv = t(rng.standard_normal((B, Hkv, 16, 128)).astype(np.float32))
    nr = t(np.array([16, 3], np.int32))
    kc = t(rng.standard_normal((B, Hkv, 128)).astype(np.float32))
    vc = t(rng.standard_normal((B, Hkv, 128)).astype(np.float32))
    dec = PQDecoder(B, Hq, Hkv, cfg)
    full = dec(q, ck, cv, t(np.array([n, n], np.int32)), cbk, cbv, rk, rv, nr, kc, vc)
    recs = []
    for r in range(W):
        a, b = shard_tokens(n, r, W)
        tail = r == W - 1
        rec = torch.empty((B * Hq, 132), device="cuda")
        # each rank stores its own shard; the decode layout counts from its row 0
        dec(q, K.relayout(ckr[:, :, a:b], True), K.relayout(cvr[:, :, a:b], True),
            t(np.array([b - a] * B, np.int32)), cbk, cbv, rk if tail else None,
            rv if tail else None, nr if tail else None, kc if tail else None,
            vc if tail else None, merged=rec, finalize=False)
        recs.append(rec)
    out = torch.empty_like(full)
    K.merge_partials(torch.stack(recs), out=out)
    np.testing.assert_allclose(out.cpu().numpy(), full.cpu().numpy(), rtol=2e-6, atol=1e-6)


# ------------------------------------------------------------------- cache --

def test_cache_sequences_match_reference(golden):
    import paper_2504_03661_b200 as P
    g = golden("cache")
    for tr in range(int(g["ntrials"])):
        R, R_f, npre, n = (int(x) for x in g[f"t{tr}_params"])
        ck, cv = _cb(g["cents_k"], "key", 2), _cb(g["cents_v"], "value", 2)
        c = P.LayerKVCache(ck, cv, recent_capacity=R, flush_threshold=R_f)
        K_, V_ = g[f"t{tr}_K"], g[f"t{tr}_V"]
        if npre:
            c.prefill_ingest(K_[:npre], V_[:npre])
        for t_ in range(npre, npre + n):
            c.append_decode(K_[t_], V_[t_])
        s = c.snapshot()
        np.testing.assert_array_equal(_np(s.codes_K.codes), g[f"t{tr}_codes_k"])
        np.testing.assert_array_equal(_np(s.codes_V.codes), g[f"t{tr}_codes_v"])
        np.testing.assert_array_equal(_np(s.recent_K), g[f"t{tr}_recent_k"])
        assert (s.n_q, s.n_total) == tuple(int(v) for v in g[f"t{tr}_nq"])


@pytest.mark.parametrize("worker", ["thread", "manual"])
def test_async_worker_bit_identical_to_sync(worker):
    """C4 (test_acceptance.py:134-199): any flush schedule drains to the sync state,
    and every snapshot covers each token exactly once."""
    import paper_2504_03661_b200 as P
    rng = np.random.default_rng(21)
    cfg = P.PQConfig(128, 64, 8)
    ck = P.Codebook(cfg, rng.standard_normal((64, 256, 2)).astype(np.float32), "key")
    cv = P.Codebook(cfg, rng.standard_normal((64, 256, 2)).astype(np.float32), "value")
    Kr = rng.standard_normal((700, 128)).astype(np.float32)
    Vr = rng.standard_normal((700, 128)).astype(np.float32)
    sync = P.LayerKVCache(ck, cv, 16, 8, "sync")
    other = P.LayerKVCache(ck, cv, 16, 8, worker)
    for c in (sync, other):
        c.prefill_ingest(Kr[:300], Vr[:300])
    for t_ in range(300, 700):
        sync.append_decode(Kr[t_], Vr[t_])
        other.append_decode(Kr[t_], Vr[t_])
        if worker == "manual" and rng.random() < 0.3:
            other.flush_step()
        s = other.snapshot()
        assert s.n_q + s.recent_K.shape[0] == s.n_total == t_ + 1
    other.drain()
    a, b = sync.snapshot(), other.snapshot()
    assert (a.n_q, a.n_total) == (b.n_q, b.n_total)
    np.testing.assert_array_equal(_np(a.codes_K.codes), _np(b.codes_K.codes))
    np.testing.assert_array_equal(_np(a.codes_V.codes), _np(b.codes_V.codes))
    np.testing.assert_array_equal(_np(a.recent_K), _np(b.recent_K))


def test_codebook_file_to_device(golden, tmp_path):
    import paper_2504_03661_b200 as P
    g = golden("fileio")
    raw = g["f0_raw"].tobytes()
    p = tmp_path / "cb.pqkv"
    p.write_bytes(raw)
    cb = P.read_codebook(p)
    np.testing.assert_array_equal(cb.device_centroids().cpu().numpy(), g["f0_cents"])
    P.write_codebook(tmp_path / "back.pqkv", cb)
    assert (tmp_path / "back.pqkv").read_bytes() == raw


@pytest.mark.parametrize("seed", range(6))
def test_randomized_batched_configs(seed):
    """Seeded random shapes through the fused path (PQDecoder): batch 1-3,
    GQA groups 1/2/3/4/8, ragged and empty lengths, recent windows 0-32,
    grids from 5 CTAs to 2 waves, exact and fp16 value-codebook modes."""
    rng = np.random.default_rng(1000 + seed)
    G = int(rng.choice([1, 2, 3, 4, 8]))
    Hkv = int(rng.integers(1, 3))
    B = int(rng.integers(1, 4))
    cap = int(rng.integers(300, 3000))
    n_q = [int(rng.integers(0, cap + 1)) for _ in range(B)]
    n_r = [int(rng.integers(0, 33)) for _ in range(B)]
    num_ctas = int(rng.choice([5, 37, 148, 296]))
    half = bool(seed % 2)
    res = _batched_case(B, G * Hkv, Hkv, cap, n_q, n_r, seed=seed, num_ctas=num_ctas,
                        half_cv=half)
    if half:
        got, want, want16 = res
        np.testing.assert_allclose(got, want16, rtol=1e-3, atol=1e-4)
    else:
        got, want = res
        np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("worker", ["sync", "thread"])
def test_decode_step_plan_device_stream(worker, monkeypatch):
    """decode_step with device tensors goes through the cache's step plan
    (pqkv_step_run: fused decode + append in one call).  Every step equals
    the oracle on the snapshot taken before it, across ring regrowth and
    compaction, background flushes, a scale change and a reloaded cache
    (the plan is rebuilt when a bound pointer or constant moves)."""
    import paper_2504_03661_b200 as P
    # a ring of 8 rows: compactions (without a host wait) every few steps
    monkeypatch.setattr(P.LayerKVCache, "RING_MIN", 8)
    monkeypatch.setattr(P.LayerKVCache, "RING_CYCLES", 1)
    rng = np.random.default_rng(11)
    cfg = P.PQConfig(128, 64, 8)
    ck = rng.standard_normal((64, 256, 2)).astype(np.float32)
    cv = rng.standard_normal((64, 256, 2)).astype(np.float32)
    cbk, cbv = P.Codebook(cfg, ck, "key"), P.Codebook(cfg, cv, "value")
    cache = P.LayerKVCache(cbk, cbv, recent_capacity=4, flush_threshold=4, worker=worker)
    X = rng.standard_normal((300, 128)).astype(np.float32)
    cache.prefill_ingest(torch.from_numpy(X[:200]).cuda(), torch.from_numpy(X[100:300]).cuda())
    cache.drain()
    plans = set()
    for s in range(40):
        q, k, v = (rng.standard_normal(128).astype(np.float32) for _ in range(3))
        scale = None if s < 30 else 0.05
        if s == 20:  # reload into a new cache: new stores, same codebooks
            fresh = P.LayerKVCache(cbk, cbv, recent_capacity=4, flush_threshold=4,
                                   worker=worker)
            fresh.load_snapshot(cache.snapshot())
            cache.close()
            cache = fresh
        snap = cache.snapshot()
        ck_h, cv_h = _np(snap.codes_K.codes), _np(snap.codes_V.codes)
        rk, rv = _np(snap.recent_K), _np(snap.recent_V)
        got = P.decode_step(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(),
                            torch.from_numpy(v).cuda(), cache, cbk, cbv, scale=scale)
        plans.add(cache._plan[0])
        want = O.decode_from_snapshot(q, k, v, ck_h, cv_h, rk, rv, ck, cv, scale=scale,
                                      block_size=1 << 30)
        np.testing.assert_allclose(got.cpu().numpy(), want, rtol=RTOL, atol=ATOL)
    cache.drain()
    assert cache.n_total == 240 and len(plans) >= 2
    cache.close()
