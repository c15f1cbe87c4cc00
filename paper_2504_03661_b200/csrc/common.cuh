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
// m64b8 decode layout of a 64-byte code row: the decode kernel's lane
// (slot s = t & 7, quarter q) reads bytes [16q, 16q+16) and processes them in
// the order j = 0..15 against subspace 16q + ((j + r) & 15), where
// r = ((lane & 15) + (lane >> 4)) & 15 for lane = 4s + q.  Storing subspace i
// of token t at byte 16q + ((i - r) & 15) lets every lane take its bytes in
// register order while the 32 lanes of a warp still hit 32 distinct
// subspaces (= shared-memory banks) at every step -- no in-register
// rotation.  A bijection per row, so uniform random codes stay uniform.
__host__ __device__ __forceinline__ int decode_lane_rot(int lane) {
    return ((lane & 15) + (lane >> 4)) & 15;
}
__host__ __device__ __forceinline__ int decode_layout_pos(int i, int slot) {
    const int q = i >> 4;
    const int r = decode_lane_rot(4 * slot + q);
    return 16 * q + (((i & 15) - r) & 15);
}

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ------------------------------------------------------- work partition ---
// The token space of all (b, hq) heads is flattened head-major
// (pos = Hq * sum_{b'<b} n_q[b'] + hq * n_q[b] + t) and cut into equal
// chunks, one per persistent CTA.  A (CTA c, head bh) overlap is a segment;
// its partial lives in slot c + bh, which is unique because both c and bh are
// non-decreasing along the flattened order.  decode and finish kernels both
// evaluate this map, so the host never needs the device-resident n_q.
constexpr int kChunkAlign = 16;

struct FlatMap {
    int64_t total;
    int64_t chunk;
};

__device__ __forceinline__ FlatMap flat_map(const int32_t *__restrict__ n_q, int B, int Hq,
                                            int num_ctas) {
    int64_t tot = 0;
    for (int b = 0; b < B; ++b) tot += (int64_t)Hq * (int64_t)max(n_q[b], 0);
    int64_t chunk = (tot + num_ctas - 1) / num_ctas;
    chunk = (chunk + kChunkAlign - 1) / kChunkAlign * kChunkAlign;
    if (chunk < kChunkAlign) chunk = kChunkAlign;
    return {tot, chunk};
}

// Flattened start of head bh and its length.
__device__ __forceinline__ int64_t head_start(const int32_t *__restrict__ n_q, int Hq, int bh,
                                              int *len) {
    const int b = bh / Hq, hq = bh - b * Hq;
    int64_t base = 0;
    for (int bb = 0; bb < b; ++bb) base += (int64_t)Hq * (int64_t)max(n_q[bb], 0);
    const int n = max(n_q[b], 0);
    *len = n;
    return base + (int64_t)hq * n;
}

// Locate the head containing flattened position pos (pos < total).
__device__ __forceinline__ void locate(const int32_t *__restrict__ n_q, int B, int Hq, int64_t pos,
                                       int *bh, int *t, int *len) {
    int64_t base = 0;
    for (int b = 0; b < B; ++b) {
        const int n = max(n_q[b], 0);
        const int64_t span = (int64_t)Hq * n;
        if (pos < base + span) {
            const int64_t off = pos - base;
            const int hq = (int)(off / n);
            *bh = b * Hq + hq;
            *t = (int)(off - (int64_t)hq * n);
            *len = n;
            return;
        }
        base += span;
    }
    *bh = -1;
    *t = 0;
    *len = 0;
}

}  // namespace pqkv
