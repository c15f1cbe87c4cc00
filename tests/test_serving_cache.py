"""ServingCache (batched multi-layer GPU cache) + PQDecoder against the
oracle, per (layer, sequence, query head), through prefill, appends, flush
batches (sync and on the side stream) and publication -- the reference's
LayerKVCache semantics (kv_cache.py:42-302) for every head at once."""

import numpy as np
import pytest
import torch

from oracle import pqkv_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("async_flush", [False, True])
def test_serving_cache_decode_matches_oracle(async_flush):
    from paper_2504_03661_b200.engine import PQDecoder
    from paper_2504_03661_b200.pq_core import PQConfig
    from paper_2504_03661_b200.serving_cache import ServingCache
    rng = np.random.default_rng(21)
    L, B, Hkv, Hq, n0, steps, d = 2, 2, 2, 4, 100, 70, 128
    cfg = PQConfig(d, 64, 8)
    ck = [rng.standard_normal((64, 256, 2)).astype(np.float32) for _ in range(L)]
    cv = [rng.standard_normal((64, 256, 2)).astype(np.float32) for _ in range(L)]
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    cache = ServingCache(L, B, Hkv, cfg, [t(c) for c in ck], [t(c) for c in cv], capacity=256,
                         async_flush=async_flush)
    Kp = rng.standard_normal((L, B, Hkv, n0, d)).astype(np.float32)
    Vp = rng.standard_normal((L, B, Hkv, n0, d)).astype(np.float32)
    cache.prefill(t(Kp), t(Vp))
    assert cache.n_quantized == n0 - 32 and cache.n_recent_rows == 32
    dec = PQDecoder(B, Hq, Hkv, cfg)
    G = Hq // Hkv
    seen_nq = set()
    for s in range(steps):
        q = rng.standard_normal((L, B, Hq, d)).astype(np.float32)
        kc = rng.standard_normal((L, B, Hkv, d)).astype(np.float32)
        vc = rng.standard_normal((L, B, Hkv, d)).astype(np.float32)
        outs = [dec(t(q[l]), k_cur=t(kc[l]), v_cur=t(vc[l]), **cache.layer(l)) for l in range(L)]
        torch.cuda.synchronize()
        seen_nq.add(cache.n_quantized)
        if s % 7 == 0 or s == steps - 1:
            for l in range(L):
                got = outs[l].cpu().numpy()
                for b in range(B):
                    for h in range(Hq):
                        codes_k, codes_v, rk, rv = cache.snapshot(l, b, h // G)
                        want = O.decode_from_snapshot(q[l, b, h], kc[l, b, h // G],
                                                      vc[l, b, h // G], codes_k, codes_v, rk, rv,
                                                      ck[l], cv[l], block_size=1 << 30)
                        np.testing.assert_allclose(got[b, h], want, rtol=1e-5, atol=1e-6)
        cache.append(t(kc), t(vc))
    cache.drain()
    assert cache.n_quantized + cache.n_recent_rows == n0 + steps
    assert len(seen_nq) >= 3  # flushes were published along the way


def test_serving_cache_codes_equal_direct_encode():
    """After drain, the code store equals encoding the whole stream at once
    (the C4 bit-identity of the reference, test_kv_cache.py:176-212)."""
    from paper_2504_03661_b200 import kernels as K
    from paper_2504_03661_b200.pq_core import PQConfig
    from paper_2504_03661_b200.serving_cache import ServingCache
    rng = np.random.default_rng(5)
    L, B, Hkv, n0, steps, d = 1, 2, 3, 40, 90, 128
    cfg = PQConfig(d, 64, 8)
    ck = torch.from_numpy(rng.standard_normal((64, 256, 2)).astype(np.float32)).cuda()
    cv = torch.from_numpy(rng.standard_normal((64, 256, 2)).astype(np.float32)).cuda()
    cache = ServingCache(L, B, Hkv, cfg, [ck], [cv], capacity=512, async_flush=True)
    Ks = torch.randn((L, B, Hkv, n0 + steps, d), device="cuda")
    Vs = torch.randn_like(Ks)
    cache.prefill(Ks[:, :, :, :n0], Vs[:, :, :, :n0])
    for s in range(steps):
        cache.append(Ks[:, :, :, n0 + s], Vs[:, :, :, n0 + s])
    cache.drain()
    n = cache.n_quantized
    for b in range(B):
        for h in range(Hkv):
            want_k = K.encode(Ks[0, b, h, :n].contiguous(), ck, 8, layout="decode")
            want_v = K.encode(Vs[0, b, h, :n].contiguous(), cv, 8, layout="decode")
            assert torch.equal(cache.codes_k[0, b, h, :n], want_k)
            assert torch.equal(cache.codes_v[0, b, h, :n], want_v)


def test_encode_batched_equals_per_problem():
    """pqkv_encode_batched == one pqkv_encode per batch (row and decode layouts)."""
    from paper_2504_03661_b200 import kernels as K
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    x = torch.randn((5, 200, 128), generator=g, device="cuda")
    c = torch.randn((5, 64, 256, 2), generator=g, device="cuda")
    for layout, t0 in (("rows", 0), ("decode", 24)):
        got = K.encode_batched(x, c, 8, layout=layout, t_first=t0)
        for z in range(5):
            assert torch.equal(got[z], K.encode(x[z], c[z], 8, layout=layout, t_first=t0))


def test_serving_cache_edges():
    """Short prefill (n < R keeps every row full precision), capacity checks,
    prefill-once, shape checks."""
    from paper_2504_03661_b200.pq_core import PQConfig
    from paper_2504_03661_b200.serving_cache import ServingCache
    cfg = PQConfig(128, 64, 8)
    c = torch.randn((64, 256, 2), device="cuda")
    cache = ServingCache(1, 1, 1, cfg, [c], [c], capacity=40, async_flush=False)
    x = torch.randn((1, 1, 1, 10, 128), device="cuda")
    cache.prefill(x, x)
    assert cache.n_quantized == 0 and cache.n_recent_rows == 10
    with pytest.raises(RuntimeError):
        cache.prefill(x, x)
    for _ in range(22):  # 32 rows -> one flush of 32
        cache.append(torch.randn((1, 1, 1, 128), device="cuda"),
                     torch.randn((1, 1, 1, 128), device="cuda"))
    assert cache.n_quantized == 32 and cache.n_recent_rows == 0
    with pytest.raises(RuntimeError):  # the next flush would exceed capacity 40
        for _ in range(32):
            cache.append(torch.randn((1, 1, 1, 128), device="cuda"),
                         torch.randn((1, 1, 1, 128), device="cuda"))
    with pytest.raises(ValueError):
        ServingCache(2, 1, 1, cfg, [c], [c], capacity=8)
    bad = ServingCache(1, 1, 1, cfg, [c], [c], capacity=8)
    with pytest.raises(ValueError):
        bad.prefill(torch.randn((1, 1, 2, 4, 128), device="cuda"),
                    torch.randn((1, 1, 2, 4, 128), device="cuda"))
