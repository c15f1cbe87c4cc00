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
print("gqa4 lane mapping: conflict free, A/B subspaces equal, rows covered")
