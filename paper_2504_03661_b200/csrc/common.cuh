// Shared helpers for the sm_100a PQ KV-cache library (libpqkv_sm100.so).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <string>

#include "../../include/pqkv_sm100.h"

namespace pqkv {

// ---------------------------------------------------------------- errors --
void set_error(const std::string &msg);
int fail(int code, const char *fmt, ...);

#define PQKV_CHECK_ARG(cond, ...)                                    \
    do {                                                             \
        if (!(cond)) return ::pqkv::fail(PQKV_EINVAL, __VA_ARGS__);  \
    } while (0)

inline int launch_status(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return fail(PQKV_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return PQKV_OK;
}

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// --------------------------------------------------------------- geometry --
inline bool geometry_ok(int d, int M, int nbits) {
    return M > 0 && d > 0 && d % M == 0 && nbits >= 1 && nbits <= 16;
}
inline int cell_bytes(int nbits) { return nbits <= 8 ? 1 : 2; }

// The m64b8 fast path: d=128, M=64 (dsub=2), nbits=8.
inline bool is_fast_geometry(int d, int M, int nbits) {
    return d == 128 && M == 64 && nbits == 8;
}

// ---------------------------------------------------------- decode layout ---
// m64b8 decode layout of a 64-byte code row.  The decode kernel's lane owns
// SPL consecutive subspaces ("part" p) of one token slot s and reads its SPL
// bytes in register order; byte j is subspace decode_lane_subspace(lane, j).
// The per-lane byte rotation makes the 32 lanes of a warp touch 32 distinct
// subspaces mod 32 at every step (the key table's banks) and 16 distinct
// subspaces mod 16 per half-warp (the 8-byte value-codebook slots) -- bank
// conflict free for ANY code values, with no in-register shuffling.  A
// bijection per row, so uniform random codes stay uniform.
//   PQKV_LANE8 = 0: SPL = 16, lane = 4 s + p (s = t & 7),
//                   byte j <-> 16 p + ((j + r) & 15), r = ((lane & 15) + (lane >> 4)) & 15
//   PQKV_LANE8 = 1: SPL = 8, lane = 8 s + p (s = t & 3),
//                   byte j <-> 8 p + ((j + 2 s + g(p)) & 7), g = 0 2 4 6 1 3 5 7
#ifndef PQKV_LANE8
#define PQKV_LANE8 0
#endif
__host__ __device__ __forceinline__ int decode_lane_rot(int lane) {
    return ((lane & 15) + (lane >> 4)) & 15;
}
__host__ __device__ __forceinline__ int lane8_rot(int s, int p) {
    return (2 * s + (((p & 3) << 1) | (p >> 2))) & 7;
}
__host__ __device__ __forceinline__ int decode_lane_subspace(int lane, int j) {
#if PQKV_LANE8
    const int p = lane & 7, s = lane >> 3;
    return 8 * p + ((j + lane8_rot(s, p)) & 7);
#else
    return 16 * (lane & 3) + ((j + decode_lane_rot(lane)) & 15);
#endif
}
// byte position of subspace i in the decode-layout row of token t
__host__ __device__ __forceinline__ int decode_layout_pos(int i, int64_t t) {
#if PQKV_LANE8
    const int p = i >> 3, s = (int)(t & 3);
    return 8 * p + (((i & 7) - lane8_rot(s, p)) & 7);
#else
    const int q = i >> 4;
    const int r = decode_lane_rot(4 * (int)(t & 7) + q);
    return 16 * q + (((i & 15) - r) & 15);
#endif
}

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ------------------------------------------------------- work partition ---
// Every (b, hq) head is laid out on a flattened *cost* axis, head-major:
// kSwitchCost setup units (the head's key-LUT build, paid by every CTA that
// switches onto the head) followed by max(n_q[b], 1) token units (an empty
// head still owns one unit, so exactly one CTA emits its empty record and
// finalizes it).  The axis is cut into equal chunks, one per persistent CTA,
// so a CTA that crosses a head boundary is charged for its extra LUT build
// and the grid stays balanced.  A (CTA c, head bh) overlap of the *token*
// units is a segment; its partial lives in slot c + bh, which is unique
// because both c and bh are non-decreasing along the axis.  The decode and
// finish kernels both evaluate this map from the device-resident n_q, so the
// host never needs the lengths.
constexpr int kChunkAlign = 16;
#ifndef PQKV_SWITCH_COST
#define PQKV_SWITCH_COST 1536
#endif
constexpr int kSwitchCost = PQKV_SWITCH_COST;  // tokens-equivalent of a head switch (measured)
// kDenseCost trailing units: the dense partial (recent rows + current token)
// paid by the CTA holding the head's end, so that CTA gets fewer tokens
#ifndef PQKV_DENSE_COST
#define PQKV_DENSE_COST 0
#endif
constexpr int kDenseCost = PQKV_DENSE_COST;

// Launch-order ramp: in a PDL-chained sequence of launches the highest CTA
// indices are dispatched last, onto the SMs the previous launch frees last
// (its last arrivers), and reach their main loop up to ~3 us late
// (profiles/r02_step_timeline.txt).  The last kRampCtas CTAs therefore get
// kRampSlope, 2 kRampSlope, ... fewer cost units (CTA n-1 the fewest).  The
// split stays a pure function of (n_q, grid): results are deterministic.
#ifndef PQKV_RAMP_CTAS
#define PQKV_RAMP_CTAS 0  // measured: every ramp tried lost 3-5%
#endif
#ifndef PQKV_RAMP_SLOPE
#define PQKV_RAMP_SLOPE 16
#endif
constexpr int kRampCtas = PQKV_RAMP_CTAS, kRampSlope = PQKV_RAMP_SLOPE;
static_assert(kRampSlope % kChunkAlign == 0, "ramp steps keep chunks aligned");

struct CostMap {
    int64_t total;
    int64_t chunk;  // cost units of an unramped CTA
    int n;          // CTAs (or CTA groups)
    int ramp;       // the last `ramp` CTAs are ramped ...
    int64_t slope;  // ... by `slope`, 2 `slope`, ... units
};

// first cost position of CTA c (c == n: past the end)
__device__ __forceinline__ int64_t cta_begin(const CostMap &cm, int c) {
    const int64_t j = max(0, c - (cm.n - cm.ramp));
    return (int64_t)c * cm.chunk - cm.slope * (j * (j + 1) / 2);
}
// CTA holding cost position pos
__device__ __forceinline__ int cta_of(const CostMap &cm, int64_t pos) {
    const int first = cm.n - cm.ramp;
    if (pos < (int64_t)first * cm.chunk) return (int)(pos / cm.chunk);
    int c = first;
    while (c + 1 < cm.n && cta_begin(cm, c + 1) <= pos) ++c;
    return c;
}

__device__ __forceinline__ int64_t head_span(int n) {
    return kSwitchCost + (int64_t)max(n, 1) + kDenseCost;
}

__device__ __forceinline__ CostMap cost_map(const int32_t *__restrict__ n_q, int B, int Hq,
                                            int num_ctas, int P = 1) {
    int64_t tot = 0;
    for (int b = 0; b < B; ++b) tot += (int64_t)Hq * head_span(n_q[b]);
    // groups of P CTAs: P times fewer groups, each P times steeper
    int ramp = kRampCtas / P;
    int64_t slope = (int64_t)kRampSlope * P;
    if (num_ctas < 4 * ramp) ramp = 0;
    auto chunk_for = [&](int r) {
        int64_t c = (tot + slope * ((int64_t)r * (r + 1) / 2) + num_ctas - 1) / num_ctas;
        c = (c + kChunkAlign - 1) / kChunkAlign * kChunkAlign;
        return c < kChunkAlign ? (int64_t)kChunkAlign : c;
    };
    int64_t chunk = chunk_for(ramp);
    if (ramp && chunk - slope * ramp < 4 * slope) {  // small problems: no ramp
        ramp = 0;
        chunk = chunk_for(0);
    }
    return {tot, chunk, num_ctas, ramp, ramp ? slope : 0};
}

// Cost-axis position of token 0 of head bh; *len = n_q[b] (>= 0).
__device__ __forceinline__ int64_t head_token0(const int32_t *__restrict__ n_q, int Hq, int bh,
                                               int *len) {
    const int b = bh / Hq, hq = bh - b * Hq;
    int64_t base = 0;
    for (int bb = 0; bb < b; ++bb) base += (int64_t)Hq * head_span(n_q[bb]);
    const int n = max(n_q[b], 0);
    *len = n;
    return base + (int64_t)hq * head_span(n) + kSwitchCost;
}

// CTAs [*c_first, *c_last] hold the segments of head bh.
__device__ __forceinline__ void head_ctas(const int32_t *__restrict__ n_q, int Hq, int bh,
                                          const CostMap &cm, int *c_first, int *c_last, int *len) {
    const int64_t t0 = head_token0(n_q, Hq, bh, len);
    *c_first = cta_of(cm, t0);
    *c_last = cta_of(cm, t0 + max(*len, 1) + kDenseCost - 1);
}

struct Segment {
    int bh;     // head b * Hq + hq
    int lo, hi; // token range [lo, hi) (empty for an empty head)
    int len;    // n_q[b]
    bool first; // this CTA holds the head's first token unit (c == c_first)
    bool last;  // this CTA holds the head's last token unit (c == c_last)
};

// Next segment of the chunk [*pos, end); advances *pos.  False when done.
__device__ __forceinline__ bool next_segment(const int32_t *__restrict__ n_q, int B, int Hq,
                                             int64_t *pos, int64_t end, Segment *s) {
    while (*pos < end) {
        int64_t base = 0;
        int b = 0;
        for (; b < B; ++b) {
            const int64_t span = (int64_t)Hq * head_span(n_q[b]);
            if (*pos < base + span) break;
            base += span;
        }
        if (b == B) {  // past the axis (cannot happen for pos < total)
            *pos = end;
            return false;
        }
        const int n = max(n_q[b], 0);
        const int64_t hs = head_span(n);
        const int hq = (int)((*pos - base) / hs);
        const int64_t h0 = base + (int64_t)hq * hs;   // head start (setup units)
        const int64_t t0 = h0 + kSwitchCost;           // token 0
        const int64_t seg_end = min(end, h0 + hs);
        const int64_t a = max(*pos, t0);
        *pos = seg_end;
        if (a < seg_end) {
            s->bh = b * Hq + hq;
            s->lo = (int)min(a - t0, (int64_t)n);  // == n inside the dense units
            s->hi = (int)min(seg_end - t0, (int64_t)n);
            s->len = n;
            s->first = (a == t0);
            s->last = (seg_end == h0 + hs);
            return true;
        }
    }
    return false;
}

}  // namespace pqkv
