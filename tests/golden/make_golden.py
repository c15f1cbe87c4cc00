"""Generate golden fixtures by running the REFERENCE package (read-only at
/root/reference/pkg/src) in the build container.

The GPU box has no /root/reference, so the outputs are committed as small
``.npz`` files next to this script; tests and smoke() read only the .npz.

    python tests/golden/make_golden.py            # rewrites tests/golden/*.npz

Cases mirror the reference's own tests (pkg/tests/conftest.py make_codebook_pair,
test_pq_core.py:129-197, test_attention.py:42-253, test_acceptance.py:41-72,
test_kv_cache.py:51-212, test_fileio.py) at sizes that keep each file small.
"""

from __future__ import annotations

import io
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import pqkv  # noqa: F401
    from pqkv import attention, fileio, harness, kv_cache, pq_core
    return pq_core, attention, kv_cache, fileio, harness


def codebook_pair(pq_core, cfg, rng, spread=1.0):
    """Same draw order as the reference fixture make_codebook_pair (conftest.py:12-22)."""
    shape = (cfg.M, cfg.ksub, cfg.dsub)
    ck = (spread * rng.standard_normal(shape)).astype(np.float32)
    cv = (spread * rng.standard_normal(shape)).astype(np.float32)
    return (pq_core.Codebook(config=cfg, centroids=ck, kind="key"),
            pq_core.Codebook(config=cfg, centroids=cv, kind="value"))


def make_encode(pq_core, harness):
    out = {}
    rng = np.random.default_rng(1234)
    geoms = [(8, 4, 2), (32, 8, 4), (128, 64, 8), (128, 8, 4), (16, 2, 3),
             (64, 4, 5), (128, 32, 12), (128, 64, 4)]
    for gi, (d, M, nbits) in enumerate(geoms):
        cfg = pq_core.PQConfig(d=d, M=M, nbits=nbits)
        ck, _ = codebook_pair(pq_core, cfg, rng)
        n = 256 if nbits < 12 else 64
        X = rng.standard_normal((n, d)).astype(np.float32) * np.float32(1.5)
        codes = pq_core.assign_codes(X, ck).codes
        out[f"g{gi}_geom"] = np.array([d, M, nbits])
        out[f"g{gi}_cents"] = ck.centroids
        out[f"g{gi}_X"] = X
        out[f"g{gi}_codes"] = codes

    # exact ties: integer centroids, vectors on midpoints -> lowest index wins
    cfg = pq_core.PQConfig(d=8, M=4, nbits=3)
    cents = rng.integers(-4, 5, size=(4, 8, 2)).astype(np.float32) * 2
    cb = pq_core.Codebook(config=cfg, centroids=cents, kind="key")
    rows = []
    for _ in range(200):
        x = np.empty(8, np.float32)
        for i in range(4):
            a, b = rng.choice(8, 2, replace=False)
            x[2 * i:2 * i + 2] = (cents[i, a] + cents[i, b]) / 2
        rows.append(x)
    X = np.stack(rows)
    out["tie_cents"] = cents
    out["tie_X"] = X
    out["tie_codes"] = pq_core.assign_codes(X, cb).codes

    # trained m64b8 codebook on outlier-channel synthetic keys (harness.py:209-212)
    cfg = pq_core.PQConfig(d=128, M=64, nbits=8, kmeans_iters=6)
    spec = harness.SynthSpec(n_tokens=2048, d=128, seed=0, outlier_channels=[7, 63])
    K, V = harness.synth_kv(spec)
    cbk = pq_core.train_codebooks(K, cfg, kind="key")
    cbv = pq_core.train_codebooks(V, cfg, kind="value")
    spec2 = harness.SynthSpec(n_tokens=1024, d=128, seed=5, outlier_channels=[7, 63],
                              outlier_rate=0.001)
    K2, V2 = harness.synth_kv(spec2)
    out["trained_cents_k"] = cbk.centroids
    out["trained_cents_v"] = cbv.centroids
    out["trained_X_k"] = K2
    out["trained_X_v"] = V2
    out["trained_codes_k"] = pq_core.assign_codes(K2, cbk).codes
    out["trained_codes_v"] = pq_core.assign_codes(V2, cbv).codes
    np.savez_compressed(os.path.join(OUT, "encode.npz"), **out)


def make_attention(pq_core, attention, kv_cache):
    out = {}
    rng = np.random.default_rng(42)
    cases = [
        # d, M, nbits, R, R_f, n_prefill, steps, block_size
        (128, 64, 8, 0, 1, 300, 3, 1024),
        (128, 64, 8, 16, 16, 300, 3, 1024),
        (128, 64, 8, 32, 32, 257, 3, 1024),
        (128, 64, 8, 32, 32, 2100, 2, 8192),   # n > 4*ksub -> centroid_accumulate
        (128, 64, 8, 0, 1, 1300, 2, 1024),     # two blocks, gather
        (8, 4, 2, 0, 1, 64, 4, 1024),
        (8, 4, 2, 16, 16, 40, 4, 1024),
        (128, 8, 4, 16, 16, 200, 3, 1024),
        (32, 8, 8, 4, 4, 100, 3, 16),          # many tiny blocks
        (128, 64, 8, 32, 32, 0, 3, 1024),      # empty cache start
    ]
    for ci, (d, M, nbits, R, R_f, npre, steps, bs) in enumerate(cases):
        cfg = pq_core.PQConfig(d=d, M=M, nbits=nbits)
        ck, cv = codebook_pair(pq_core, cfg, np.random.default_rng(100 + ci))
        n = npre + steps
        K = rng.standard_normal((n, d)).astype(np.float32)
        V = rng.standard_normal((n, d)).astype(np.float32)
        cache = kv_cache.LayerKVCache(ck, cv, recent_capacity=R, flush_threshold=R_f,
                                      worker="sync")
        if npre:
            cache.prefill_ingest(K[:npre], V[:npre])
        qs, outs, nqs, lut0 = [], [], [], None
        snaps = []
        for s in range(steps):
            q = rng.standard_normal(d)
            snap = cache.snapshot()
            nqs.append(snap.n_q)
            if s == 0:
                snaps = [snap.codes_K.codes.copy(), snap.codes_V.codes.copy(),
                         snap.recent_K.copy(), snap.recent_V.copy()]
                lut0 = attention.build_key_lut(q, ck).table
                if snap.n_q:
                    qp = attention.quantized_partial(
                        attention.build_key_lut(q, ck), snap.codes_K, snap.codes_V, cv)
                    out[f"c{ci}_qp"] = np.concatenate([[qp.m, qp.l], qp.acc])
            o = attention.decode_step(q, K[npre + s], V[npre + s], cache, ck, cv,
                                      block_size=bs)
            qs.append(q)
            outs.append(o)
        fin = cache.snapshot()
        out[f"c{ci}_params"] = np.array([d, M, nbits, R, R_f, npre, steps, bs])
        out[f"c{ci}_cents_k"] = ck.centroids
        out[f"c{ci}_cents_v"] = cv.centroids
        out[f"c{ci}_steps_k"] = K[npre:]
        out[f"c{ci}_steps_v"] = V[npre:]
        out[f"c{ci}_q"] = np.stack(qs)
        out[f"c{ci}_out"] = np.stack(outs)
        out[f"c{ci}_nq"] = np.array(nqs)
        out[f"c{ci}_lut0"] = lut0
        out[f"c{ci}_snap0_codes_k"], out[f"c{ci}_snap0_codes_v"] = snaps[0], snaps[1]
        out[f"c{ci}_snap0_recent_k"], out[f"c{ci}_snap0_recent_v"] = snaps[2], snaps[3]
        out[f"c{ci}_final_codes_k"] = fin.codes_K.codes
        out[f"c{ci}_final_codes_v"] = fin.codes_V.codes
        out[f"c{ci}_final_recent_k"] = fin.recent_K
    out["ncases"] = np.array(len(cases))

    # merge / dense / finalize pins (test_attention.py:172-236 style)
    q = rng.standard_normal(8)
    Kd = rng.standard_normal((30, 8))
    Vd = rng.standard_normal((30, 8))
    a = attention.dense_partial(q, Kd[:13], Vd[:13])
    b = attention.dense_partial(q, Kd[13:], Vd[13:])
    mg = attention.merge_partials(a, b)
    out["merge_q"], out["merge_K"], out["merge_V"] = q, Kd, Vd
    out["merge_a"] = np.concatenate([[a.m, a.l], a.acc])
    out["merge_b"] = np.concatenate([[b.m, b.l], b.acc])
    out["merge_ab"] = np.concatenate([[mg.m, mg.l], mg.acc])
    out["merge_final"] = attention.finalize(mg)
    np.savez_compressed(os.path.join(OUT, "attention.npz"), **out)


def make_fileio(pq_core, fileio):
    import tempfile
    out = {}
    rng = np.random.default_rng(7)
    for gi, (d, M, nbits, kind) in enumerate([(128, 64, 8, "key"), (8, 4, 2, "value"),
                                              (32, 8, 10, "key")]):
        cfg = pq_core.PQConfig(d=d, M=M, nbits=nbits)
        cents = rng.standard_normal((M, cfg.ksub, cfg.dsub)).astype(np.float32)
        cb = pq_core.Codebook(config=cfg, centroids=cents, kind=kind)
        with tempfile.TemporaryDirectory() as td:
            p = os.path.join(td, "cb.pqkv")
            fileio.write_codebook(p, cb)
            raw = open(p, "rb").read()
            back = fileio.read_codebook(p)
        out[f"f{gi}_raw"] = np.frombuffer(raw, np.uint8)
        out[f"f{gi}_geom"] = np.array([d, M, nbits, 0 if kind == "key" else 1])
        out[f"f{gi}_cents"] = back.centroids
    np.savez_compressed(os.path.join(OUT, "fileio.npz"), **out)


def make_cache(pq_core, kv_cache):
    """Random append/flush_recent sequences on the sync cache (test_kv_cache.py:102-212)."""
    out = {}
    rng = np.random.default_rng(99)
    cfg = pq_core.PQConfig(d=8, M=4, nbits=2)
    ck, cv = codebook_pair(pq_core, cfg, np.random.default_rng(0))
    out["cents_k"], out["cents_v"] = ck.centroids, cv.centroids
    for tr in range(12):
        R = int(rng.choice([0, 4, 16]))
        R_f = int(rng.choice([1, 4, 16]))
        n = int(rng.integers(10, 50))
        npre = int(rng.integers(0, 20))
        K = rng.standard_normal((npre + n, 8)).astype(np.float32)
        V = rng.standard_normal((npre + n, 8)).astype(np.float32)
        cache = kv_cache.LayerKVCache(ck, cv, recent_capacity=R, flush_threshold=R_f)
        if npre:
            cache.prefill_ingest(K[:npre], V[:npre])
        for t in range(npre, npre + n):
            cache.append_decode(K[t], V[t])
        s = cache.snapshot()
        out[f"t{tr}_params"] = np.array([R, R_f, npre, n])
        out[f"t{tr}_K"], out[f"t{tr}_V"] = K, V
        out[f"t{tr}_codes_k"], out[f"t{tr}_codes_v"] = s.codes_K.codes, s.codes_V.codes
        out[f"t{tr}_recent_k"], out[f"t{tr}_recent_v"] = s.recent_K, s.recent_V
        out[f"t{tr}_nq"] = np.array([s.n_q, s.n_total])
    out["ntrials"] = np.array(12)
    np.savez_compressed(os.path.join(OUT, "cache.npz"), **out)


def make_synth(harness):
    """The reference's synthetic KV streams (harness.py:37-93) for three specs."""
    out = {}
    specs = [dict(n_tokens=64, d=128, seed=0),
             dict(n_tokens=50, d=128, seed=3, outlier_channels=[7, 63]),
             dict(n_tokens=40, d=64, seed=9, sigma=0.5, outlier_channels=[1],
                  outlier_rate=0.01, outlier_magnitude=30.0)]
    for si, sp in enumerate(specs):
        K, V = harness.synth_kv(harness.SynthSpec(**sp))
        out[f"s{si}_K"], out[f"s{si}_V"] = K, V
    np.savez_compressed(os.path.join(OUT, "synth.npz"), **out)


def make_kmeans(pq_core, harness):
    """kmeans_train / train_codebooks (pq_core.py:171-266): separated blobs,
    a Gaussian cloud, fewer distinct points than k, duplicated rows, and a
    train_codebooks run on synth_kv keys (m8b4, d=16)."""
    out = {}
    rng = np.random.default_rng(21)
    centers = np.array([[0, 0], [8, 0], [0, 8], [8, 8]], np.float64)
    blobs = (centers[rng.integers(0, 4, 400)] + 0.3 * rng.standard_normal((400, 2)))
    cases = {
        "blobs": (blobs.astype(np.float32), 4, 25, 1e-4, 0),
        "gauss": (rng.standard_normal((2000, 2)).astype(np.float32), 16, 25, 1e-4, 3),
        "few": (np.repeat(np.array([[1, 2], [3, 4], [5, 6]], np.float32), 4, axis=0), 5, 10,
                1e-4, 1),
        "dups": (np.round(rng.standard_normal((300, 2)) * 2).astype(np.float32), 8, 30, 0.0, 2),
        "oned": (rng.standard_normal(500).astype(np.float32), 6, 25, 1e-4, 4),
    }
    for name, (X, k, iters, tol, seed) in cases.items():
        C, hist = pq_core.kmeans_train(X, k, iters=iters, tol=tol, seed=seed)
        out[f"{name}_X"], out[f"{name}_C"], out[f"{name}_hist"] = X, C, np.array(hist)
        out[f"{name}_args"] = np.array([k, iters, tol, seed], np.float64)
    K, _ = harness.synth_kv(harness.SynthSpec(n_tokens=600, d=16, seed=5))
    cfg = pq_core.PQConfig(d=16, M=8, nbits=4, kmeans_iters=12, seed=7)
    cb = pq_core.train_codebooks(K, cfg, kind="key")
    out["train_X"], out["train_C"] = K.astype(np.float32), cb.centroids
    np.savez_compressed(os.path.join(OUT, "kmeans.npz"), **out)


def make_baselines(pq_core, attention):
    """integer_quantize / integer_dequantize (pq_core.py:312-354) and
    prefill_attention (attention.py:290-311)."""
    out = {}
    rng = np.random.default_rng(31)
    X = (rng.standard_normal((64, 48)) * 3).astype(np.float32)
    X[0, :4] = [0.5, 1.5, 2.5, -0.5]  # ties for round-half-to-even
    for nb in (2, 4, 8):
        for mode in ("symmetric", "asymmetric"):
            Q, prm = pq_core.integer_quantize(X, nb, mode)
            out[f"iq_{mode}_{nb}_Q"] = Q
            out[f"iq_{mode}_{nb}_sz"] = np.array([prm.s, prm.z], np.float64)
            out[f"iq_{mode}_{nb}_Xh"] = pq_core.integer_dequantize(Q, prm)
    out["iq_X"] = X
    # grid-valued data: many exact .5 boundaries after X / s + z
    Xg = (np.arange(-15, 16) / 10).reshape(1, -1)
    out["iqg_X"] = Xg
    for nb in (2, 3, 4):
        for mode in ("symmetric", "asymmetric"):
            Q, prm = pq_core.integer_quantize(Xg, nb, mode)
            out[f"iqg_{mode}_{nb}_Q"] = Q
            out[f"iqg_{mode}_{nb}_sz"] = np.array([prm.s, prm.z], np.float64)
    Qp, Kp, Vp = (rng.standard_normal((n, 64)) for n in (7, 19, 19))
    out["pf_Q"], out["pf_K"], out["pf_V"] = Qp, Kp, Vp
    out["pf_causal"] = attention.prefill_attention(Qp, Kp, Vp)
    out["pf_full"] = attention.prefill_attention(Qp, Kp, Vp, causal=False, scale=0.3)
    np.savez_compressed(os.path.join(OUT, "baselines.npz"), **out)


def make_analysis(pq_core, harness):
    """channel_stats / isolate_outliers / sensitivity_study / compare_quantizers
    (analysis.py:59-192) on synth_kv keys with outlier channels."""
    from pqkv import analysis
    out = {}
    K, _ = harness.synth_kv(harness.SynthSpec(n_tokens=700, d=32, seed=9,
                                              outlier_channels=[3, 20]))
    out["X"] = K
    st = analysis.channel_stats(K)
    out["cs_mean"], out["cs_std"], out["cs_absmax"] = st.mean, st.std, st.absmax
    out["cs_misc"] = np.array([st.global_absmax, st.outlier_threshold])
    out["cs_outliers"] = np.array(st.outlier_channels)
    entries, filt = analysis.isolate_outliers(K, 0.01)
    out["io_entries"] = np.array(entries)
    out["io_filtered"] = filt
    cfg = pq_core.PQConfig(d=32, M=16, nbits=4, kmeans_iters=8, seed=2)
    cq = analysis.compare_quantizers(K, cfg, 4)
    out["cq"] = np.array([cq[k] for k in sorted(cq)])
    for q in ("pq", "int"):
        r = analysis.sensitivity_study(K, cfg, fraction=0.01, quantizer=q)
        out[f"ss_{q}"] = np.array([r.err_full, r.err_filtered, r.sensitivity])
    np.savez_compressed(os.path.join(OUT, "analysis.npz"), **out)


def make_attention_wide(pq_core, attention, kv_cache):
    """decode_step streams with codes wider than a byte (uint16 cells: nbits
    12 and 10, the m32b12-style presets pq_core.py:80-83) at sizes that keep
    the codebooks small; same record layout as make_attention."""
    out = {}
    rng = np.random.default_rng(57)
    cases = [
        # d, M, nbits, R, R_f, n_prefill, steps, block_size
        (8, 2, 12, 16, 16, 500, 3, 1024),
        (16, 4, 10, 8, 8, 300, 4, 128),
    ]
    for ci, (d, M, nbits, R, R_f, npre, steps, bs) in enumerate(cases):
        cfg = pq_core.PQConfig(d=d, M=M, nbits=nbits)
        ck, cv = codebook_pair(pq_core, cfg, np.random.default_rng(200 + ci))
        n = npre + steps
        K = rng.standard_normal((n, d)).astype(np.float32)
        V = rng.standard_normal((n, d)).astype(np.float32)
        cache = kv_cache.LayerKVCache(ck, cv, recent_capacity=R, flush_threshold=R_f,
                                      worker="sync")
        cache.prefill_ingest(K[:npre], V[:npre])
        snap = cache.snapshot()
        out[f"c{ci}_snap0_codes_k"], out[f"c{ci}_snap0_codes_v"] = (snap.codes_K.codes.copy(),
                                                                    snap.codes_V.codes.copy())
        out[f"c{ci}_snap0_recent_k"] = snap.recent_K.copy()
        out[f"c{ci}_snap0_recent_v"] = snap.recent_V.copy()
        qs, outs, nqs = [], [], []
        for s in range(steps):
            q = rng.standard_normal(d)
            nqs.append(cache.snapshot().n_q)
            outs.append(attention.decode_step(q, K[npre + s], V[npre + s], cache, ck, cv,
                                              block_size=bs))
            qs.append(q)
        fin = cache.snapshot()
        out[f"c{ci}_params"] = np.array([d, M, nbits, R, R_f, npre, steps, bs])
        out[f"c{ci}_cents_k"], out[f"c{ci}_cents_v"] = ck.centroids, cv.centroids
        out[f"c{ci}_steps_k"], out[f"c{ci}_steps_v"] = K[npre:], V[npre:]
        out[f"c{ci}_q"], out[f"c{ci}_out"] = np.stack(qs), np.stack(outs)
        out[f"c{ci}_nq"] = np.array(nqs)
        out[f"c{ci}_final_codes_k"] = fin.codes_K.codes
        out[f"c{ci}_final_codes_v"] = fin.codes_V.codes
    out["ncases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(OUT, "attention_wide.npz"), **out)


def make_seam(pq_core, attention):
    """The lower seam (_kernels.score_codes / accumulate_mass, _kernels.py:46-65,
    numba loops :27-43) and the Counters accounting (attention.py:56-63,
    test_attention.py:99-107)."""
    from pqkv import _kernels
    out = {}
    rng = np.random.default_rng(61)
    for ci, (M, nbits, n) in enumerate([(64, 8, 3000), (4, 12, 5000), (8, 3, 777)]):
        ksub = 1 << nbits
        dt = np.uint8 if nbits <= 8 else np.uint16
        codes = rng.integers(0, ksub, (n, M)).astype(dt)
        codes[:7] = codes[7:14]  # repeated rows: same-bin collisions
        lut = rng.standard_normal((M, ksub))
        p = np.exp(rng.standard_normal(n) * 3)
        out[f"s{ci}_codes"], out[f"s{ci}_lut"], out[f"s{ci}_p"] = codes, lut, p
        out[f"s{ci}_scores"] = _kernels.score_codes(lut, codes)
        out[f"s{ci}_mass"] = _kernels.accumulate_mass(codes, p, ksub)
    # Counters through the public API (d=8, M=4, nbits=2 as test_attention.py)
    cfg = pq_core.PQConfig(d=8, M=4, nbits=2)
    ck, cv = codebook_pair(pq_core, cfg, np.random.default_rng(62))
    X = rng.standard_normal((37, 8))
    codes_k, codes_v = pq_core.assign_codes(X, ck), pq_core.assign_codes(X, cv)
    q = rng.standard_normal(8)
    lut = attention.build_key_lut(q, ck)
    c1 = attention.Counters()
    attention.score_tokens(lut, codes_k, c1)
    c2 = attention.Counters()
    attention.quantized_partial(lut, codes_k, codes_v, cv, counters=c2)
    c3 = attention.Counters()
    attention.dense_partial(q, X[:5], X[5:10], counters=c3)
    out["ctr_X"], out["ctr_q"] = X, q
    out["ctr_cents_k"], out["ctr_cents_v"] = ck.centroids, cv.centroids
    out["ctr"] = np.array([[c.lut_lookups, c.adds, c.code_bytes_read, c.dense_bytes_read]
                           for c in (c1, c2, c3)])
    np.savez_compressed(os.path.join(OUT, "seam.npz"), **out)


def main():
    pq_core, attention, kv_cache, fileio, harness = _ref()
    if "--wide-only" in sys.argv:
        make_attention_wide(pq_core, attention, kv_cache)
        make_seam(pq_core, attention)
        return
    if "--synth-only" in sys.argv:
        make_synth(harness)
        return
    if "--kmeans-only" in sys.argv:
        make_kmeans(pq_core, harness)
        return
    if "--baselines-only" in sys.argv:
        make_baselines(pq_core, attention)
        return
    if "--baselines-only" in sys.argv:
        make_baselines(pq_core, attention)
        return
    if "--analysis-only" in sys.argv:
        make_analysis(pq_core, harness)
        return
    make_synth(harness)
    make_encode(pq_core, harness)
    make_attention(pq_core, attention, kv_cache)
    make_fileio(pq_core, fileio)
    make_cache(pq_core, kv_cache)
    make_kmeans(pq_core, harness)
    make_baselines(pq_core, attention)
    make_analysis(pq_core, harness)
    make_attention_wide(pq_core, attention, kv_cache)
    make_seam(pq_core, attention)
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
