"""The reference's lower seam and drop-in details on the GPU (``-m gpu``).

* ``_kernels.score_codes`` / ``accumulate_mass`` (reference _kernels.py:46-65)
  bit-identical to the reference's numba loops (seam.npz, made by running the
  reference), uint8 and uint16 cells;
* ``Counters`` accounting as the reference's test_attention.py:99-107;
* decode_step streams with uint16 cells (nbits 12 / 10) replayed against the
  reference (attention_wide.npz) -- the generic decode path;
* snapshots of a cache fed numpy are numpy (kv_cache.py:269-290);
* the float32 seam entry points (pqkv_score_codes / pqkv_accumulate_mass).
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
    N.load()


@pytest.mark.parametrize("ci", range(3))
def test_seam_bit_identical_to_reference(golden, ci):
    from paper_2504_03661_b200 import _kernels
    g = golden("seam")
    codes, lut, p = g[f"s{ci}_codes"], g[f"s{ci}_lut"], g[f"s{ci}_p"]
    s = _kernels.score_codes(lut, codes)
    assert isinstance(s, np.ndarray) and s.dtype == np.float64
    np.testing.assert_array_equal(s, g[f"s{ci}_scores"])
    h = _kernels.accumulate_mass(codes, p, lut.shape[1])
    assert h.shape == (codes.shape[1], lut.shape[1]) and h.dtype == np.float64
    np.testing.assert_array_equal(h, g[f"s{ci}_mass"])
    # CUDA tensors in -> CUDA tensors out, same bits
    ct = torch.from_numpy(codes.astype(np.int32)).cuda().to(
        torch.uint8 if codes.dtype == np.uint8 else torch.uint16)
    st = _kernels.score_codes(torch.from_numpy(lut).cuda(), ct)
    assert st.is_cuda
    np.testing.assert_array_equal(st.cpu().numpy(), g[f"s{ci}_scores"])
    ht = _kernels.accumulate_mass(ct, torch.from_numpy(p).cuda(), lut.shape[1])
    np.testing.assert_array_equal(ht.cpu().numpy(), g[f"s{ci}_mass"])


def test_seam_errors():
    from paper_2504_03661_b200 import _kernels
    with pytest.raises(ValueError):
        _kernels.score_codes(np.zeros((3, 256)), np.zeros((5, 4), np.uint8))  # M mismatch
    with pytest.raises(ValueError):
        _kernels.accumulate_mass(np.zeros((5, 4), np.uint8), np.ones(4), 256)  # n mismatch
    with pytest.raises(ValueError):
        _kernels.accumulate_mass(np.zeros((5, 4), np.uint8), np.ones(5), 100)  # ksub


def test_float32_seam_entry_points():
    """pqkv_score_codes / pqkv_accumulate_mass (float32 variants of the seam)
    against the oracle at float32 tolerance."""
    from paper_2504_03661_b200 import kernels as K
    rng = np.random.default_rng(3)
    n, M = 4000, 64
    codes = rng.integers(0, 256, (n, M), dtype=np.uint8)
    lut = rng.standard_normal((M, 256)).astype(np.float32)
    p = rng.random(n).astype(np.float32)
    ct = torch.from_numpy(codes).cuda()
    s = K.score_codes(torch.from_numpy(lut.T.copy()).cuda(), ct, 8).cpu().numpy()
    np.testing.assert_allclose(s, O.score_codes(lut.astype(np.float64), codes), rtol=1e-5,
                               atol=1e-4)
    h = K.accumulate_mass(ct, torch.from_numpy(p).cuda(), 8).cpu().numpy()
    np.testing.assert_allclose(h, O.accumulate_mass(codes, p.astype(np.float64), 256),
                               rtol=1e-5, atol=1e-5)


def test_counters_match_reference(golden):
    """Counters through score_tokens / quantized_partial / dense_partial, as
    the reference's test_work_accounting (test_attention.py:99-107)."""
    import paper_2504_03661_b200 as P
    g = golden("seam")
    cfg = P.PQConfig(8, 4, 2)
    ck = P.Codebook(cfg, g["ctr_cents_k"], "key")
    cv = P.Codebook(cfg, g["ctr_cents_v"], "value")
    X = g["ctr_X"]
    codes_k, codes_v = P.assign_codes(X, ck), P.assign_codes(X, cv)
    lut = P.build_key_lut(g["ctr_q"], ck)
    got = []
    c1 = P.Counters()
    P.score_tokens(lut, codes_k, c1)
    c2 = P.Counters()
    P.quantized_partial(lut, codes_k, codes_v, cv, counters=c2)
    c3 = P.Counters()
    P.dense_partial(g["ctr_q"], X[:5], X[5:10], counters=c3)
    for c in (c1, c2, c3):
        got.append([c.lut_lookups, c.adds, c.code_bytes_read, c.dense_bytes_read])
    np.testing.assert_array_equal(np.array(got), g["ctr"])
    n = X.shape[0]
    assert c1.lut_lookups == n * 4 and c1.adds == n * 4 and c1.code_bytes_read == n * 4
    assert c2.code_bytes_read == 2 * n * 4


@pytest.mark.parametrize("ci", range(2))
def test_wide_code_decode_replay_matches_reference(golden, ci):
    """nbits 12 / 10 (uint16 cells): the reference's decode_step streams
    through LayerKVCache + decode_step on the GPU (generic decode path)."""
    import paper_2504_03661_b200 as P
    g = golden("attention_wide")
    d, M, nbits, R, R_f, npre, steps, bs = (int(x) for x in g[f"c{ci}_params"])
    cfg = P.PQConfig(d, M, nbits)
    ck = P.Codebook(cfg, g[f"c{ci}_cents_k"], "key")
    cv = P.Codebook(cfg, g[f"c{ci}_cents_v"], "value")
    cache = P.LayerKVCache(ck, cv, recent_capacity=R, flush_threshold=R_f, worker="sync")
    nq0 = int(g[f"c{ci}_nq"][0])
    snap0 = P.CacheSnapshot(P.CodesMatrix(g[f"c{ci}_snap0_codes_k"], nbits),
                            P.CodesMatrix(g[f"c{ci}_snap0_codes_v"], nbits),
                            g[f"c{ci}_snap0_recent_k"], g[f"c{ci}_snap0_recent_v"], nq0,
                            nq0 + g[f"c{ci}_snap0_recent_k"].shape[0])
    cache.load_snapshot(snap0)
    outs = []
    for s in range(steps):
        assert cache.n_q == g[f"c{ci}_nq"][s]
        outs.append(P.decode_step(g[f"c{ci}_q"][s], g[f"c{ci}_steps_k"][s],
                                  g[f"c{ci}_steps_v"][s], cache, ck, cv, block_size=bs))
    np.testing.assert_allclose(np.stack(outs), g[f"c{ci}_out"], rtol=RTOL, atol=ATOL)
    fin = cache.snapshot()
    assert isinstance(fin.codes_K.codes, np.ndarray) and fin.codes_K.codes.dtype == np.uint16
    np.testing.assert_array_equal(fin.codes_K.codes, g[f"c{ci}_final_codes_k"])
    np.testing.assert_array_equal(fin.codes_V.codes, g[f"c{ci}_final_codes_v"])


def test_snapshot_types_follow_inputs():
    """numpy in -> numpy snapshot (the reference's types); tensors in -> tensors."""
    import paper_2504_03661_b200 as P
    rng = np.random.default_rng(9)
    cfg = P.PQConfig(128, 64, 8)
    ck = P.Codebook(cfg, rng.standard_normal((64, 256, 2)).astype(np.float32), "key")
    cv = P.Codebook(cfg, rng.standard_normal((64, 256, 2)).astype(np.float32), "value")
    X = rng.standard_normal((100, 128)).astype(np.float32)
    a = P.LayerKVCache(ck, cv)
    a.prefill_ingest(X, X)
    sa = a.snapshot()
    assert isinstance(sa.codes_K.codes, np.ndarray) and sa.codes_K.codes.dtype == np.uint8
    assert isinstance(sa.recent_K, np.ndarray) and sa.recent_K.dtype == np.float32
    b = P.LayerKVCache(ck, cv)
    b.prefill_ingest(torch.from_numpy(X).cuda(), torch.from_numpy(X).cuda())
    sb = b.snapshot()
    assert isinstance(sb.codes_K.codes, torch.Tensor) and sb.codes_K.codes.is_cuda
    np.testing.assert_array_equal(sa.codes_K.codes, sb.codes_K.codes.cpu().numpy())
    np.testing.assert_array_equal(sa.recent_V, sb.recent_V.cpu().numpy())
    # the snapshot restores into a fresh cache (load_snapshot, kv_cache.py:292-302)
    c = P.LayerKVCache(ck, cv)
    c.load_snapshot(sa)
    np.testing.assert_array_equal(c.snapshot().codes_V.codes, sa.codes_V.codes)
