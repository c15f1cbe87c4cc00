"""Checks the lane mapping of decode_gqa4_f16 (csrc/decode.cu) on the stored
m64b8 decode layout (common.cuh decode_layout_pos): lane (s, w) reads bytes
[8w, 8w+8) of token A = {0,1,4,5}[s] and bytes [8(w^1), ...) of token B = A+2
of every 8-token unit.  Asserts that A and B touch the same subspace at every
step, that the 8 lanes of a token cover all 64 subspaces, and that every warp
instruction is bank-conflict free: 16 distinct subspaces mod 16 per half-warp
(8-byte key-table gathers) and 32 distinct mod 32 per warp (4-byte value
gathers)."""


def rot(l):
    return ((l & 15) + (l >> 4)) & 15


def sub_at(t, b):  # subspace stored at byte b of token t's row
    q = b >> 4
    return 16 * q + (((b & 15) + rot(4 * (t & 7) + q)) & 15)


TAU_A = [0, 1, 4, 5]
for j in range(8):
    for which in ("A", "B"):
        subs = []
        for lane in range(32):
            s, w = lane >> 3, lane & 7
            t, b = (TAU_A[s], 8 * w + j) if which == "A" else (TAU_A[s] + 2, 8 * (w ^ 1) + j)
            subs.append(sub_at(t, b))
        for hw in (0, 1):
            assert len({x % 16 for x in subs[16 * hw:16 * hw + 16]}) == 16, (which, j, hw)
        assert len({x % 32 for x in subs}) == 32, (which, j)
for lane in range(32):
    s, w = lane >> 3, lane & 7
    for j in range(8):
        assert sub_at(TAU_A[s], 8 * w + j) == sub_at(TAU_A[s] + 2, 8 * (w ^ 1) + j)
for s in range(4):
    assert sorted(sub_at(TAU_A[s], 8 * w + j) for w in range(8) for j in range(8)) == list(range(64))
# PQKV_GQA4_PERM: every subspace a lane reads has i >> 4 == w >> 1, so the
# table's head order k ^ (i >> 4) is the lane's; simulate token_reduce_own
for lane in range(32):
    s, w = lane >> 3, lane & 7
    for j in range(8):
        assert sub_at(TAU_A[s], 8 * w + j) >> 4 == w >> 1
vals = {(w, h): 10.0 ** w * (h + 1) for w in range(8) for h in range(4)}  # lane w's head-h partial
def v(w, k):  # slot k of lane w holds head k ^ (w >> 1)
    return vals[(w, k ^ (w >> 1))]
for w in range(8):
    k0 = v(w, 0) + v(w ^ 4, 2)
    k1 = lambda x: v(x, 1) + v(x ^ 4, 3)
    k = k0 + k1(w ^ 2)
    kk = lambda x: (v(x, 0) + v(x ^ 4, 2)) + k1(x ^ 2)
    got = k + kk(w ^ 1)
    h = (w >> 1) & 3
    assert abs(got - sum(vals[(x, h)] for x in range(8))) < 1e-6 * got, (w, got)
print("gqa4 lane mapping: conflict free, A/B subspaces equal, rows covered")
