"""Checks the lane mapping of decode_gqa_pair (csrc/decode.cu, exact GQA, a
cluster of two CTAs each owning one half of the 64 subspaces) on the stored
m64b8 decode layout (common.cuh): lane (s, w) of CTA c reads the 8 bytes
[32c + 8w, 32c + 8w + 8) of token s (instruction A) and s + 8 (instruction B)
of every 16-token unit, rotated left by rho = 2 bytes when s & 2 (one PRMT pair
per 8 bytes).  Asserts that A and B touch the same subspace at every step, that
the 4 lanes of a token cover the CTA's 32 subspaces, and that every warp
instruction is bank-conflict free for 8-byte gathers: 16 distinct subspaces
mod 16 per half-warp (the fp32 float2 key tables and value codebook, address
code << 8 | (i & 31) << 3)."""


def rot(l):
    return ((l & 15) + (l >> 4)) & 15


def sub_at(t, b):  # subspace stored at byte b of token t's row
    q = b >> 4
    return 16 * q + (((b & 15) + rot(4 * (t & 7) + q)) & 15)


for c in (0, 1):
    for j in range(8):
        for which in ("A", "B"):
            subs = []
            for lane in range(32):
                s, w = lane >> 2, lane & 3
                rho = 2 if s & 2 else 0
                t = s if which == "A" else s + 8
                subs.append(sub_at(t, 32 * c + 8 * w + ((j + rho) & 7)))
            for hw in (0, 1):
                assert len({x % 16 for x in subs[16 * hw:16 * hw + 16]}) == 16, (c, which, j, hw)
            assert all(x >> 5 == c for x in subs)
    for s in range(8):
        cov = sorted(sub_at(s, 32 * c + 8 * w + j) for w in range(4) for j in range(8))
        assert cov == list(range(32 * c, 32 * c + 32))
# PQKV_PAIR_PERMW: the subspaces of lane w have local bit 4 == w >> 1, so the
# key tables swap their head-pair regions for local subspaces 16..31
for c in (0, 1):
    for lane in range(32):
        s, w = lane >> 2, lane & 3
        rho = 2 if s & 2 else 0
        for t in (s, s + 8):
            for j in range(8):
                assert (sub_at(t, 32 * c + 8 * w + ((j + rho) & 7)) - 32 * c) >> 4 == w >> 1
print("gqa pair lane mapping: conflict free, A/B subspaces equal, halves covered")
