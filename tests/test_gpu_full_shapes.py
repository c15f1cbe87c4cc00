"""Parity at BASELINE's full GQA shapes and on the serving loop's launch flags.

* config 3 (Llama-3-8B GQA 32:8, B=16, 32K) and config 4 (B=4, 128K): one
  whole layer through the fused launch, exact and fp16 value-codebook modes
  (the latter also with the packed fp16 key tables),
  against the fp64 C restatement of the reference run per query head
  (snapshot -> build_key_lut -> quantized / dense partials -> merge ->
  finalize; reference attention.py:114-166, :214-287);
* config 4 split over 8 simulated ranks (each rank's token range decoded to
  (m, l, acc) records, merged in rank order) == the unsplit launch;
* the INTEGRATION.md serving loop: ServingCache + PQDecoder(pdl=True,
  static_codebooks=True, early_codes=True) across several flush publications,
  sync and async, against the oracle;
* early_codes re-validation: a length update that lands after the decode's
  pre-wait reads (pqkv_debug_delayed_fill) gives the same bits as a plain
  launch on the new lengths.

Tolerances as tests/test_gpu_parity.py: exact mode rtol 1e-5 / atol 1e-6;
fp16 value-codebook mode rtol 2e-3 / atol 2e-4 (its stated tolerance).
"""

import numpy as np
import pytest
import torch

from oracle import pqkv_oracle as O

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-5, 1e-6
RTOL16, ATOL16 = 2e-3, 2e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2504_03661_b200._native as N
    N.load()
    if O.c_library() is None:
        import subprocess
        import os
        subprocess.run(["make", "-s", "-C", os.path.join(os.path.dirname(O.__file__))],
                       check=True)
        O._clib = None
        assert O.c_library() is not None


def _layer(B, Hq, Hkv, n, R, seed):
    """A full layer's inputs: device tensors (codes in the row layout) + host copies."""
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    dev = "cuda"
    x = dict(
        q=torch.randn((B, Hq, 128), generator=g, device=dev),
        ck=torch.randint(0, 256, (B, Hkv, n, 64), generator=g, device=dev, dtype=torch.uint8),
        cv=torch.randint(0, 256, (B, Hkv, n, 64), generator=g, device=dev, dtype=torch.uint8),
        cents_k=torch.randn((64, 256, 2), generator=g, device=dev),
        cents_v=torch.randn((64, 256, 2), generator=g, device=dev),
        rk=torch.randn((B, Hkv, R, 128), generator=g, device=dev),
        rv=torch.randn((B, Hkv, R, 128), generator=g, device=dev),
        kc=torch.randn((B, Hkv, 128), generator=g, device=dev),
        vc=torch.randn((B, Hkv, 128), generator=g, device=dev),
    )
    # ragged lengths: every sequence but the first is a little shorter
    nq = [n] + [n - 977 * b for b in range(1, B)]
    nr = [R] + [(7 * b) % (R + 1) for b in range(1, B)]
    x["nq"] = torch.tensor(nq, dtype=torch.int32, device=dev)
    x["nr"] = torch.tensor(nr, dtype=torch.int32, device=dev)
    return x


def _oracle(x):
    h = {k: v.cpu().numpy() for k, v in x.items()}
    return O.c_decode_batched(h["q"], h["kc"], h["vc"], h["ck"], h["cv"], h["nq"], h["rk"],
                              h["rv"], h["nr"], h["cents_k"], h["cents_v"], 8)


def _decode(x, Hq, Hkv, half=False, **flags):
    from paper_2504_03661_b200 import kernels as K
    from paper_2504_03661_b200.engine import PQDecoder
    from paper_2504_03661_b200.pq_core import PQConfig
    B = x["q"].shape[0]
    dec = PQDecoder(B, Hq, Hkv, PQConfig(128, 64, 8), **flags)
    ck, cv = K.relayout(x["ck"], True), K.relayout(x["cv"], True)
    out = dec(x["q"], ck, cv, x["nq"], K.key_codebook_layout(x["cents_k"], 8),
              K.value_codebook_layout(x["cents_v"], 8, half=half), x["rk"], x["rv"], x["nr"],
              x["kc"], x["vc"])
    return out.cpu().numpy()


@pytest.mark.parametrize("cfg", ["config3", "config4"])
def test_full_gqa_layer_vs_c_oracle(cfg):
    """A whole BASELINE config-3 / config-4 layer, every (b, query head)."""
    B, n = (16, 32768) if cfg == "config3" else (4, 131072)
    x = _layer(B, 32, 8, n, 31, seed=31 if cfg == "config3" else 41)
    want = _oracle(x)
    got = _decode(x, 32, 8)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)
    got16 = _decode(x, 32, 8, half=True)
    np.testing.assert_allclose(got16, want, rtol=RTOL16, atol=ATOL16)
    # + the four query heads' key tables of a CTA as one packed fp16 table
    got16k = _decode(x, 32, 8, half=True, f16_key_table=True)
    np.testing.assert_allclose(got16k, want, rtol=RTOL16, atol=ATOL16)
    # ... and two query heads per CTA (one half2 table)
    got16p = _decode(x, 32, 8, half=True, f16_key_table=True, key_table_pairs=True)
    np.testing.assert_allclose(got16p, want, rtol=RTOL16, atol=ATOL16)


def test_config4_eight_way_split_equals_unsplit():
    """Config 4 sequence split over 8 simulated ranks on one GPU: each rank's
    contiguous token range [r n / 8, (r+1) n / 8) to (m, l, acc) records, the
    tail rank adding the recent rows + current token, merged in rank order
    (pqkv_merge_partials) == the unsplit decode, and both == the oracle."""
    from paper_2504_03661_b200 import kernels as K
    from paper_2504_03661_b200.engine import PQDecoder, shard_tokens
    from paper_2504_03661_b200.pq_core import PQConfig
    B, Hq, Hkv, n, W = 4, 32, 8, 131072, 8
    x = _layer(B, Hq, Hkv, n, 31, seed=43)
    x["nq"].fill_(n)  # a sequence split cuts equal-length sequences
    full = _decode(x, Hq, Hkv)
    cbk = K.key_codebook_layout(x["cents_k"], 8)
    cbv = K.value_codebook_layout(x["cents_v"], 8)
    dec = PQDecoder(B, Hq, Hkv, PQConfig(128, 64, 8))
    recs = torch.empty((W, B * Hq, 132), device="cuda")
    for r in range(W):
        a, b = shard_tokens(n, r, W)
        tail = r == W - 1
        ck = K.relayout(x["ck"][:, :, a:b].contiguous(), True)
        cv = K.relayout(x["cv"][:, :, a:b].contiguous(), True)
        dec(x["q"], ck, cv, torch.full((B,), b - a, dtype=torch.int32, device="cuda"), cbk, cbv,
            x["rk"] if tail else None, x["rv"] if tail else None, x["nr"] if tail else None,
            x["kc"] if tail else None, x["vc"] if tail else None, merged=recs[r],
            finalize=False)
        del ck, cv
    out = torch.empty((B, Hq, 128), device="cuda")
    K.merge_partials(recs, out=out)
    got = out.cpu().numpy()
    np.testing.assert_allclose(got, full, rtol=2e-6, atol=1e-6)
    np.testing.assert_allclose(got, _oracle(x), rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("mode", ["exact", "f16_quad", "f16_pair"])
@pytest.mark.parametrize("grow", [True, False])
def test_early_codes_revalidates_lengths(grow, mode):
    """PQKV_DECODE_EARLY_CODES reads n_q before its grid-dependency wait.  A
    kernel that releases the decode at once and rewrites n_q 200 us later
    (pqkv_debug_delayed_fill) makes that pre-wait copy stale; the decode must
    notice after the wait and redo its split: same bits as a plain launch on
    the new lengths -- for the exact GQA CTA pairs (group 4) and the fp16
    four- and two-heads-per-CTA kernels."""
    from paper_2504_03661_b200 import _native as N
    from paper_2504_03661_b200 import kernels as K
    from paper_2504_03661_b200.engine import PQDecoder
    from paper_2504_03661_b200.pq_core import PQConfig
    B, Hq, Hkv, n = 3, 8, 2, 20000
    x = _layer(B, Hq, Hkv, n, 16, seed=5)
    ck, cv = K.relayout(x["ck"], True), K.relayout(x["cv"], True)
    cbk = K.key_codebook_layout(x["cents_k"], 8)
    cbv = K.value_codebook_layout(x["cents_v"], 8, half=mode != "exact")
    old_n, new_n = (6000, 19000) if grow else (19000, 6000)
    cfg = PQConfig(128, 64, 8)
    kw = {} if mode == "exact" else dict(f16_key_table=True,
                                         key_table_pairs=mode == "f16_pair")
    plain = PQDecoder(B, Hq, Hkv, cfg, **kw)
    early = PQDecoder(B, Hq, Hkv, cfg, pdl=True, static_codebooks=True, early_codes=True, **kw)
    args = (ck, cv, x["nq"], cbk, cbv, x["rk"], x["rv"], x["nr"], x["kc"], x["vc"])
    x["nq"].fill_(new_n)
    want = plain(x["q"], *args).clone()
    for _ in range(3):
        x["nq"].fill_(old_n)
        torch.cuda.synchronize()
        N.call("pqkv_debug_delayed_fill", N.ptr(x["nq"]), B, new_n, 200_000, N.stream_ptr())
        got = early(x["q"], *args)
        torch.cuda.synchronize()
        assert int(x["nq"][0]) == new_n
        assert torch.equal(got, want)
    # and the oracle agrees with the new lengths
    x["nq"].fill_(new_n)
    tol = (RTOL, ATOL) if mode == "exact" else (RTOL16, ATOL16)
    np.testing.assert_allclose(want.cpu().numpy(), _oracle(x), rtol=tol[0], atol=tol[1])


@pytest.mark.parametrize("async_flush", [False, True])
@pytest.mark.parametrize("R,R_f", [(32, 32), (32, 8)])
def test_serving_loop_pdl_early_codes_matches_oracle(async_flush, R, R_f):
    """INTEGRATION.md's serving loop: PQDecoder(pdl=True, static_codebooks=True,
    early_codes=True) over a ServingCache through prefill, appends and at least
    three flush publications, every layer decoded back to back (PDL-chained),
    against the oracle per (layer, sequence, query head)."""
    from paper_2504_03661_b200.engine import PQDecoder
    from paper_2504_03661_b200.pq_core import PQConfig
    from paper_2504_03661_b200.serving_cache import ServingCache
    rng = np.random.default_rng(77)
    L, B, Hkv, Hq, n0, steps, d = 3, 2, 2, 8, 150, 75, 128
    cfg = PQConfig(d, 64, 8)
    ck = [rng.standard_normal((64, 256, 2)).astype(np.float32) for _ in range(L)]
    cv = [rng.standard_normal((64, 256, 2)).astype(np.float32) for _ in range(L)]
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    cache = ServingCache(L, B, Hkv, cfg, [t(c) for c in ck], [t(c) for c in cv], capacity=512,
                         recent_capacity=R, flush_threshold=R_f, async_flush=async_flush)
    Kp = rng.standard_normal((L, B, Hkv, n0, d)).astype(np.float32)
    Vp = rng.standard_normal((L, B, Hkv, n0, d)).astype(np.float32)
    cache.prefill(t(Kp), t(Vp))
    dec = PQDecoder(B, Hq, Hkv, cfg, pdl=True, static_codebooks=True, early_codes=True)
    G = Hq // Hkv
    seen_nq = set()
    for s in range(steps):
        q = rng.standard_normal((L, B, Hq, d)).astype(np.float32)
        kc = rng.standard_normal((L, B, Hkv, d)).astype(np.float32)
        vc = rng.standard_normal((L, B, Hkv, d)).astype(np.float32)
        qd, kd, vd = t(q), t(kc), t(vc)
        outs = [dec(qd[l], k_cur=kd[l], v_cur=vd[l], **cache.layer(l)) for l in range(L)]
        nq_now = cache.n_quantized
        new_pub = nq_now not in seen_nq
        seen_nq.add(nq_now)
        if new_pub or s % 9 == 0 or s == steps - 1:
            for l in range(L):
                got = outs[l].cpu().numpy()
                for b in range(B):
                    for h in range(Hq):
                        codes_k, codes_v, rk, rv = cache.snapshot(l, b, h // G)
                        want = O.decode_from_snapshot(q[l, b, h], kc[l, b, h // G],
                                                      vc[l, b, h // G], codes_k, codes_v, rk,
                                                      rv, ck[l], cv[l], block_size=1 << 30)
                        np.testing.assert_allclose(got[b, h], want, rtol=RTOL, atol=ATOL)
        cache.append(kd, vd)
    cache.drain()
    assert cache.n_quantized + cache.n_recent_rows == n0 + steps
    assert len(seen_nq) >= 4  # >= 3 publications after the prefill
    if not async_flush:
        assert cache.n_recent_rows < R_f  # whole batches until below the threshold
