"""PQKV_DECODE_F16_KEY_TABLE (GQA, stated tolerance): with the fp16 value
codebook and an even group, the CTA serving the query heads of a KV head keeps
their key tables as ONE packed fp16 table -- entry (c, i) holds the heads'
build_key_lut values (attention.py:70-83) rounded to fp16 -- so one gather per
key code feeds every head's score, summed in fp32 (mixed f32 + f16 adds).
Groups that are a multiple of 4 run four query heads per CTA (8-byte entries,
decode_gqa4_f16, fp32 softmax weights); key_table_pairs=True (and groups of 2)
run two (4-byte entries, fp16 weights).  Each table entry carries a relative rounding error
of at most 2^-11, so a score's absolute error is at most
2^-11 * sum_i |lut[i][code_i]|; the softmax weights and the value path are
those of the fp16 value-codebook mode.

Stated tolerance, as the fp16 value-codebook mode: rtol 2e-3 / atol 2e-4 vs
the fp64 oracle per query head (spans of a few tokens sit at the edge of it in
both fp16 modes: the value codebook's rounding does not average out there) (quantized_partial attention.py:114-166,
dense_partial :169-190, merge :193-211).  Odd groups and MHA ignore the flag
(one fp32 table per head), so there the result is bit-identical to the fp16
value-codebook mode."""

import numpy as np
import pytest
import torch

from test_gpu_parity import _batched_case, _fused_inputs  # noqa: F401

pytestmark = pytest.mark.gpu

RTOL16, ATOL16 = 2e-3, 2e-4


@pytest.mark.parametrize("pairs", [False, True])
@pytest.mark.parametrize("B,Hq,Hkv,cap,n_q,n_r", [
    (2, 8, 2, 5000, [4999, 1234], [5, 32]),          # G = 4: four (or two) heads per CTA
    (3, 2, 1, 700, [0, 1, 7], [0, 3, 0]),            # G = 2, empty / tiny spans
    (1, 8, 1, 20000, [20000], [7]),                  # G = 8, many CTAs per virtual head
    (4, 32, 8, 9000, [9000, 8000, 2500, 4500], [31, 0, 3, 17]),  # Llama-3 grouping, ragged
    (5, 16, 4, 300, [0, 64, 170, 299, 96], [1, 0, 32, 5, 9]),     # empty / short spans, G = 4
])
def test_f16_key_table_vs_oracle(B, Hq, Hkv, cap, n_q, n_r, pairs):
    got, want, want16 = _batched_case(B, Hq, Hkv, cap, n_q, n_r, half_cv=True, f16_keys=True,
                                      pairs=pairs)
    # vs the oracle on the fp16-rounded value codebook: the key-table and
    # weight roundings only
    np.testing.assert_allclose(got, want16, rtol=RTOL16, atol=ATOL16)
    np.testing.assert_allclose(got, want, rtol=RTOL16, atol=ATOL16)


@pytest.mark.parametrize("B,Hq,Hkv,cap,n_q,n_r", [
    (1, 4, 4, 3000, [3000], [31]),                   # MHA
    (2, 6, 2, 4100, [4100, 333], [31, 0]),           # G = 3 (odd)
])
def test_f16_key_table_ignored_without_pairs(B, Hq, Hkv, cap, n_q, n_r):
    a = _batched_case(B, Hq, Hkv, cap, n_q, n_r, half_cv=True, f16_keys=True)[0]
    b = _batched_case(B, Hq, Hkv, cap, n_q, n_r, half_cv=True, f16_keys=False)[0]
    assert np.array_equal(a, b)


def test_f16_key_table_scaled_scores():
    """Larger scores (queries 2x N(0,1)): the fp16 table's absolute score
    error grows with the entries; still within the stated tolerance at the
    BASELINE magnitudes (N(0,1) queries and codebooks, scale up to 4/sqrt(d))."""
    from paper_2504_03661_b200 import kernels as K
    import paper_2504_03661_b200 as P
    from test_gpu_parity import _oracle_heads
    rng = np.random.default_rng(5)
    B, Hq, Hkv, n, R = 1, 8, 2, 4000, 8
    ck = rng.standard_normal((64, 256, 2)).astype(np.float32)
    cv = rng.standard_normal((64, 256, 2)).astype(np.float32)
    q = rng.standard_normal((B, Hq, 128)).astype(np.float32) * 2.0
    codes_k = rng.integers(0, 256, (B, Hkv, n, 64), dtype=np.uint8)
    codes_v = rng.integers(0, 256, (B, Hkv, n, 64), dtype=np.uint8)
    rk = rng.standard_normal((B, Hkv, R, 128)).astype(np.float32)
    rv = rng.standard_normal((B, Hkv, R, 128)).astype(np.float32)
    kc = rng.standard_normal((B, Hkv, 128)).astype(np.float32)
    vc = rng.standard_normal((B, Hkv, 128)).astype(np.float32)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    from paper_2504_03661_b200.engine import PQDecoder
    dec = PQDecoder(B, Hq, Hkv, P.PQConfig(128, 64, 8), f16_key_table=True)
    out = dec(t(q), K.relayout(t(codes_k), True), K.relayout(t(codes_v), True),
              t(np.array([n], np.int32)), K.key_codebook_layout(t(ck), 8),
              K.value_codebook_layout(t(cv), 8, half=True), t(rk), t(rv),
              t(np.array([R], np.int32)), t(kc), t(vc))
    want = _oracle_heads(q, codes_k, codes_v, [n], rk, rv, [R], kc, vc, ck, cv, Hq // Hkv)
    np.testing.assert_allclose(out.cpu().numpy(), want, rtol=RTOL16, atol=ATOL16)
