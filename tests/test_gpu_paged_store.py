"""Paged code store (vstore.py / csrc/vstore.cu): the caches grow by mapping
pages at the end of each head's virtual region instead of doubling and
copying (the reference's kv_cache.py:74-76, 217-228).

* the store itself: rows written before a growth keep their address and
  value across it; every region grows together; page granularity;
* LayerKVCache across a page boundary (32 Ki rows of 64 B = one 2 MiB page):
  its store never moves, and decode_step stays within the exact tolerance of
  the oracle (reference attention.py:214-287);
* ServingCache across a page boundary: flushes map pages on the side stream's
  behalf, the fused decode reads each head as one contiguous run, and the
  code store equals encoding the whole stream at once (C4 bit-identity,
  reference test_kv_cache.py:176-212).
"""

import numpy as np
import pytest
import torch

from oracle import pqkv_oracle as O

pytestmark = pytest.mark.gpu


def test_store_grows_in_place():
    from paper_2504_03661_b200.vstore import PagedCodeStore
    st = PagedCodeStore(3, 1 << 20, (64,), torch.uint8, "cuda")
    rows0 = st.mapped_rows
    assert rows0 >= 1 and st.max_rows >= 1 << 20
    t = st.tensor
    assert t.shape == (3, st.max_rows, 64) and t.is_contiguous()
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    a = torch.randint(0, 256, (3, rows0, 64), generator=g, device="cuda", dtype=torch.uint8)
    t[:, :rows0] = a
    ptr = t.data_ptr()
    st.ensure(3 * rows0 + 5)  # two or more growth steps' worth
    assert st.mapped_rows >= 3 * rows0 + 5
    assert st.tensor.data_ptr() == ptr
    b = torch.randint(0, 256, (3, st.mapped_rows - rows0, 64), generator=g, device="cuda",
                      dtype=torch.uint8)
    t[:, rows0:st.mapped_rows] = b
    torch.cuda.synchronize()
    assert torch.equal(t[:, :rows0], a)  # the first pages are untouched
    assert torch.equal(t[:, rows0:st.mapped_rows], b)
    with pytest.raises(ValueError):
        st.ensure(st.max_rows + 1)
    st.close()


def test_layer_cache_crosses_a_page_without_moving():
    import paper_2504_03661_b200 as P
    rng = np.random.default_rng(7)
    cfg = P.PQConfig(128, 64, 8)
    ck = rng.standard_normal((64, 256, 2)).astype(np.float32)
    cv = rng.standard_normal((64, 256, 2)).astype(np.float32)
    cbk, cbv = P.Codebook(cfg, ck, "key"), P.Codebook(cfg, cv, "value")
    cache = P.LayerKVCache(cbk, cbv, recent_capacity=16, flush_threshold=16, worker="sync")
    first_page = cache._store.mapped_rows
    ptr = cache._store_k.data_ptr()
    n0 = first_page - 40  # the appends below cross into the second page
    X = rng.standard_normal((n0, 128)).astype(np.float32)
    Y = rng.standard_normal((n0, 128)).astype(np.float32)
    cache.prefill_ingest(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda())
    for s in range(64):
        q = rng.standard_normal(128).astype(np.float32)
        k = rng.standard_normal(128).astype(np.float32)
        v = rng.standard_normal(128).astype(np.float32)
        snap = cache.snapshot()
        ck_h = snap.codes_K.codes.cpu().numpy()
        cv_h = snap.codes_V.codes.cpu().numpy()
        rk, rv = snap.recent_K.cpu().numpy(), snap.recent_V.cpu().numpy()
        got = P.decode_step(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(),
                            torch.from_numpy(v).cuda(), cache, cbk, cbv)
        if s % 16 == 15:
            want = O.decode_from_snapshot(q, k, v, ck_h, cv_h, rk, rv, ck, cv,
                                          block_size=1 << 30)
            np.testing.assert_allclose(got.cpu().numpy(), want, rtol=1e-5, atol=1e-6)
    assert cache.n_q > first_page and cache._store.mapped_rows > first_page
    assert cache._store_k.data_ptr() == ptr  # grown in place, never copied
    # the whole store equals one-shot encoding of every flushed row (C4)
    snap = cache.snapshot()
    n = snap.n_q
    assert np.array_equal(snap.codes_K.codes.cpu().numpy()[:n0 - 16],
                          O.assign_codes(X[:n0 - 16], ck, 8))


@pytest.mark.parametrize("async_flush", [False, True])
def test_serving_cache_crosses_a_page(async_flush):
    from paper_2504_03661_b200.engine import PQDecoder
    from paper_2504_03661_b200.pq_core import PQConfig
    from paper_2504_03661_b200.serving_cache import ServingCache
    rng = np.random.default_rng(3)
    L, B, Hkv, Hq, d = 1, 2, 1, 2, 128
    cfg = PQConfig(d, 64, 8)
    ck = [rng.standard_normal((64, 256, 2)).astype(np.float32)]
    cv = [rng.standard_normal((64, 256, 2)).astype(np.float32)]
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    cache = ServingCache(L, B, Hkv, cfg, [t(c) for c in ck], [t(c) for c in cv],
                         capacity=1 << 20, async_flush=async_flush)
    page = cache.mapped_rows
    ptr = cache.codes_k.data_ptr()
    n0 = page + 32 - 70  # quantized rows end 70 - 32 = 38 rows below the page end
    Kp = rng.standard_normal((L, B, Hkv, n0, d)).astype(np.float32)
    Vp = rng.standard_normal((L, B, Hkv, n0, d)).astype(np.float32)
    cache.prefill(t(Kp), t(Vp))
    dec = PQDecoder(B, Hq, Hkv, cfg, pdl=True, static_codebooks=True, early_codes=True)
    ks, vs = [], []
    for s in range(100):
        q = rng.standard_normal((L, B, Hq, d)).astype(np.float32)
        kc = rng.standard_normal((L, B, Hkv, d)).astype(np.float32)
        vc = rng.standard_normal((L, B, Hkv, d)).astype(np.float32)
        out = dec(t(q[0]), k_cur=t(kc[0]), v_cur=t(vc[0]), **cache.layer(0))
        if s % 25 == 24:
            torch.cuda.synchronize()
            got = out.cpu().numpy()
            for b in range(B):
                for h in range(Hq):
                    codes_k, codes_v, rk, rv = cache.snapshot(0, b, 0)
                    want = O.decode_from_snapshot(q[0, b, h], kc[0, b, 0], vc[0, b, 0], codes_k,
                                                  codes_v, rk, rv, ck[0], cv[0],
                                                  block_size=1 << 30)
                    np.testing.assert_allclose(got[b, h], want, rtol=1e-5, atol=1e-6)
        cache.append(t(kc), t(vc))
        ks.append(kc)
        vs.append(vc)
    cache.drain()
    assert cache.n_quantized > page and cache.mapped_rows > page
    assert cache.codes_k.data_ptr() == ptr
    # every flushed row, prefill + appends, equals one-shot encoding (C4)
    allk = np.concatenate([Kp[0, 1, 0], np.stack([k[0, 1, 0] for k in ks])])
    codes_k, _, _, _ = cache.snapshot(0, 1, 0)
    n = codes_k.shape[0]
    assert np.array_equal(codes_k, O.assign_codes(allk[:n], ck[0], 8))
