// K1 -- nearest-centroid PQ encoder, bit-exact with the reference.
//
// Reference: pq_core.py:269-287 (assign_codes) over _squared_distances
// (:158-168).  For each subspace the reference evaluates, in float64,
//     d2 = (np.sum(X*X, axis=1) - 2 * (X @ C.T)) + np.sum(C*C, axis=1)
// clamps at 0 and takes the first argmin.  Inputs are float32 (or narrower)
// values, so every product is exact in float64; the only roundings are the
// additions, whose order we reproduce: numpy's pairwise row sum for the
// norms and a sequential k-loop for x.c (OpenBLAS dgemm order; both verified
// bit-for-bit against numpy).  Ties keep the lowest index
// (strict < scan from c = 0).
//
// Layout: one thread per (vector, subspace); a CTA owns one subspace and 256
// vectors, with that subspace's centroids and norms staged in shared memory
// as float64 (warp-uniform broadcast reads).  FP64 bound: 256 * ~7 DFMA-class
// ops per (vector, subspace) for m64b8.
#include <algorithm>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace pqkv {
namespace {

// Destination cell of code (row v, subspace i): the reference row layout, or
// (rot_base >= 0, m64b8 only) the decode layout in which each 16-byte quarter
// of a row is stored rotated by its decode lane's constant (see common.cuh).
__device__ __forceinline__ int64_t code_cell(int64_t v, int i, int64_t ld_codes, int64_t rot_base) {
    if (rot_base < 0) return v * ld_codes + i;
    return v * ld_codes + decode_layout_pos(i, rot_base + v);
}

template <typename TX>
__device__ __forceinline__ double load_x(const TX *p);
template <>
__device__ __forceinline__ double load_x<float>(const float *p) { return (double)__ldg(p); }
template <>
__device__ __forceinline__ double load_x<__nv_bfloat16>(const __nv_bfloat16 *p) {
    return (double)__bfloat162float(*p);
}
template <>
__device__ __forceinline__ double load_x<__half>(const __half *p) {
    return (double)__half2float(*p);
}

// the subspace's two input values (one 8- or 4-byte load when aligned)
template <typename TX>
__device__ __forceinline__ void load_pair(const TX *p, float &a, float &b) {
    if ((reinterpret_cast<uintptr_t>(p) & (2 * sizeof(TX) - 1)) == 0) {
        if constexpr (sizeof(TX) == 4) {
            const float2 v = __ldg(reinterpret_cast<const float2 *>(p));
            a = v.x;
            b = v.y;
        } else {
            const uint32_t v = __ldg(reinterpret_cast<const unsigned int *>(p));
            TX lo, hi;
            memcpy(&lo, &v, 2);
            const uint16_t h = (uint16_t)(v >> 16);
            memcpy(&hi, &h, 2);
            a = (float)load_x<TX>(&lo);
            b = (float)load_x<TX>(&hi);
        }
    } else {
        a = (float)load_x<TX>(p);
        b = (float)load_x<TX>(p + 1);
    }
}

// numpy pairwise_sum for float64 (n < 8: sequential from 0.0; n <= 128: eight
// strided accumulators; else recursive halves rounded down to a multiple of 8).
template <typename Get>
__device__ double np_pairwise(Get get, int lo, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r += get(lo + i);
        return r;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = get(lo + j);
        int i = 8;
        for (; i < n - (n % 8); i += 8)
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] += get(lo + i + j);
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += get(lo + i);
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise(get, lo, n2) + np_pairwise(get, lo + n2, n - n2);
}

// Compile-time dsub (<= 16): x lives in registers, centroids + norms in smem.
template <typename TX, typename CT, int DSUB>
__global__ void __launch_bounds__(256) encode_staged(const TX *__restrict__ x, int64_t n,
                                                     int64_t ld_x, const float *__restrict__ cents,
                                                     int ksub, CT *__restrict__ codes,
                                                     int64_t ld_codes, int64_t rot_base) {
    extern __shared__ double sm[];
    double *c_s = sm;                      // [ksub][DSUB]
    double *cc_s = sm + (size_t)ksub * DSUB;  // [ksub]
    const int i = blockIdx.y;
    const float *ci = cents + (size_t)i * ksub * DSUB;
    for (int idx = threadIdx.x; idx < ksub * DSUB; idx += blockDim.x) c_s[idx] = (double)ci[idx];
    __syncthreads();
    for (int c = threadIdx.x; c < ksub; c += blockDim.x) {
        const double *cr = c_s + (size_t)c * DSUB;
        cc_s[c] = np_pairwise([&](int j) { return cr[j] * cr[j]; }, 0, DSUB);
    }
    __syncthreads();

    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    double xr[DSUB];
#pragma unroll
    for (int j = 0; j < DSUB; ++j) xr[j] = load_x<TX>(x + v * ld_x + (int64_t)i * DSUB + j);
    const double xx = np_pairwise([&](int j) { return xr[j] * xr[j]; }, 0, DSUB);

    double best = INFINITY;
    int arg = 0;
#pragma unroll 4
    for (int c = 0; c < ksub; ++c) {
        const double *cr = c_s + (size_t)c * DSUB;
        double xc = xr[0] * cr[0];
#pragma unroll
        for (int j = 1; j < DSUB; ++j) xc = fma(xr[j], cr[j], xc);  // products exact: == mul+add
        double d2 = (xx - 2.0 * xc) + cc_s[c];
        d2 = fmax(d2, 0.0);
        if (d2 < best) {
            best = d2;
            arg = c;
        }
    }
    codes[code_cell(v, i, ld_codes, rot_base)] = (CT)arg;
}

// dsub == 2 (the m64b8 geometry): VPT vectors per thread share every
// centroid read (one 16-byte + one 8-byte broadcast LDS per centroid per VPT
// vectors), leaving four FP64 ops per (vector, centroid) for the distance:
//   xc = x0 c0 (exact) ; xc = fma(x1, c1, xc) = round(x0 c0 + x1 c1)
//   t  = fma(-2, xc, xx) = round(xx - 2 xc)   (2 xc is exact)
//   d2 = t + cc
// -- the reference's roundings in the reference's order -- then the clamp at
// 0 and the strict first-minimum scan.
#ifndef PQKV_ENC_VPT
#define PQKV_ENC_VPT 4
#endif
#ifndef PQKV_ENC_FILTER
#define PQKV_ENC_FILTER 1
#endif
template <typename TX, typename CT, int VPT>
__global__ void __launch_bounds__(256) encode_dsub2(const TX *__restrict__ x, int64_t n,
                                                    int64_t ld_x, const float *__restrict__ cents,
                                                    int ksub, CT *__restrict__ codes,
                                                    int64_t ld_codes, int64_t rot_base) {
    extern __shared__ double sm[];
    double2 *c_s = reinterpret_cast<double2 *>(sm);  // [ksub] (c0, c1)
    double *cc_s = sm + 2 * (size_t)ksub;             // [ksub] c0^2 + c1^2 (numpy order)
    const int i = blockIdx.y;
    const float2 *ci = reinterpret_cast<const float2 *>(cents + (size_t)i * ksub * 2);
    for (int c = threadIdx.x; c < ksub; c += blockDim.x) {
        const float2 f = __ldg(ci + c);
        const double a = f.x, b = f.y;
        c_s[c] = make_double2(a, b);
        cc_s[c] = __dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b));  // squares exact
    }
    __syncthreads();

    const int64_t v0 = (int64_t)blockIdx.x * blockDim.x * VPT + threadIdx.x;
    double x0[VPT], x1[VPT], xx[VPT], best[VPT];
    int arg[VPT];
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const int64_t v = v0 + (int64_t)k * blockDim.x;
        const int64_t vv = v < n ? v : n - 1;
        x0[k] = load_x<TX>(x + vv * ld_x + (int64_t)i * 2);
        x1[k] = load_x<TX>(x + vv * ld_x + (int64_t)i * 2 + 1);
        xx[k] = __dadd_rn(__dmul_rn(x0[k], x0[k]), __dmul_rn(x1[k], x1[k]));
        best[k] = INFINITY;
        arg[k] = 0;
    }
#pragma unroll 2
    for (int c = 0; c < ksub; ++c) {
        const double2 cv = c_s[c];
        const double cc = cc_s[c];
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            const double xc = __fma_rn(x1[k], cv.y, __dmul_rn(x0[k], cv.x));
            const double d2 = fmax(__dadd_rn(__fma_rn(-2.0, xc, xx[k]), cc), 0.0);
            if (d2 < best[k]) {
                best[k] = d2;
                arg[k] = c;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const int64_t v = v0 + (int64_t)k * blockDim.x;
        if (v < n) codes[code_cell(v, i, ld_codes, rot_base)] = (CT)arg[k];
    }
}

// dsub == 2 with an fp32 filter: the FP64 pipe of this part is narrow, so the
// scan over the centroids runs in fp32 on the direct form (x - c)^2 (no
// cancellation) while tracking the best and second-best distance.  When the
// two are further apart than the combined error bound of the fp32 distances
// and of the reference's fp64 expanded form, the fp32 argmin IS the
// reference's argmin (no other centroid can reach it, and no exact fp64 tie
// is possible); otherwise -- near ties, exact ties, x on a centroid -- the
// (vector, subspace) is re-scanned with the exact FP64 formula above.
#ifndef PQKV_ENC_FILTER_VPT
#define PQKV_ENC_FILTER_VPT 8  // vectors per thread of the filter scan (4: -3%)
#endif
#ifndef PQKV_ENC_PAIR
#define PQKV_ENC_PAIR 2  // 0: one centroid per step in scalar fp32 (measured 20% slower)
#endif
template <typename TX, typename CT, int VPT>
__global__ void __launch_bounds__(256) encode_dsub2_filter(const TX *__restrict__ x, int64_t n,
                                                           int64_t ld_x,
                                                           const float *__restrict__ cents,
                                                           int ksub, CT *__restrict__ codes,
                                                           int64_t ld_codes, int64_t rot_base,
                                                           int64_t x_bs, int64_t c_bs,
                                                           int64_t codes_bs) {
    // batch blockIdx.z (e.g. one layer each): its own rows, codebook and codes
    x += blockIdx.z * x_bs;
    cents += blockIdx.z * c_bs;
    codes += blockIdx.z * codes_bs;
    extern __shared__ double sm[];
    double2 *c_s = reinterpret_cast<double2 *>(sm);                   // [ksub]
    double *cc_s = sm + 2 * (size_t)ksub;                              // [ksub]
    float2 *cf_s = reinterpret_cast<float2 *>(sm + 3 * (size_t)ksub);  // [ksub]
    __shared__ float ccmax_s;
    const int i = blockIdx.x;  // subspace fastest: the M blocks of a row block share its x sectors and code lines in L2
    const float2 *ci = reinterpret_cast<const float2 *>(cents + (size_t)i * ksub * 2);
    if (threadIdx.x == 0) ccmax_s = 0.f;
    __syncthreads();
    float ccmax = 0.f;
    for (int c = threadIdx.x; c < ksub; c += blockDim.x) {
        const float2 f = __ldg(ci + c);
        const double a = f.x, b = f.y;
        c_s[c] = make_double2(a, b);
        cc_s[c] = __dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b));
#if PQKV_ENC_PAIR == 2
        // centroid pairs as (-x_2p, -x_2p+1, -y_2p, -y_2p+1): packed f32x2 operands
        float *cp = reinterpret_cast<float *>(cf_s) + 4 * (c >> 1) + (c & 1);
        cp[0] = -f.x;
        cp[2] = -f.y;
#else
        cf_s[c] = f;
#endif
        ccmax = fmaxf(ccmax, (float)cc_s[c]);
    }
    atomicMax(reinterpret_cast<int *>(&ccmax_s), __float_as_int(ccmax));  // non-negative floats
    __syncthreads();
    ccmax = ccmax_s;

    const int64_t v0 = (int64_t)blockIdx.y * blockDim.x * VPT + threadIdx.x;
    // best / second-best as sortable keys: the distance's bits (d >= 0, so its
    // bit pattern orders like the value) with the low mantissa bits replaced
    // by the centroid index -- one LOP3 + three integer min/max per centroid
    const uint32_t cmask = (uint32_t)ksub - 1u;  // ksub is a power of two
    float xf0[VPT], xf1[VPT];
    uint32_t b1[VPT], b2[VPT];
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const int64_t v = v0 + (int64_t)k * blockDim.x;
        const int64_t vv = v < n ? v : n - 1;
        xf0[k] = (float)load_x<TX>(x + vv * ld_x + (int64_t)i * 2);
        xf1[k] = (float)load_x<TX>(x + vv * ld_x + (int64_t)i * 2 + 1);
        b1[k] = 0xffffffffu;
        b2[k] = 0xffffffffu;
    }
#if PQKV_ENC_PAIR == 2
    // two centroids per step, their distances in packed f32x2 arithmetic (the
    // same roundings as the scalar form, so the same keys), and the three-input
    // min update below
    const float4 *cf4 = reinterpret_cast<const float4 *>(cf_s);
    unsigned long long xp0[VPT], xp1[VPT];
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        asm("mov.b64 %0, {%1,%1};" : "=l"(xp0[k]) : "f"(xf0[k]));
        asm("mov.b64 %0, {%1,%1};" : "=l"(xp1[k]) : "f"(xf1[k]));
    }
    for (int c = 0; c < ksub; c += 2) {
        const float4 cv = cf4[c >> 1];
        unsigned long long ncx, ncy;
        asm("mov.b64 %0, {%1,%2};" : "=l"(ncx) : "f"(cv.x), "f"(cv.y));
        asm("mov.b64 %0, {%1,%2};" : "=l"(ncy) : "f"(cv.z), "f"(cv.w));
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            unsigned long long dx, dy, dd;
            asm("add.rn.f32x2 %0, %1, %2;" : "=l"(dx) : "l"(xp0[k]), "l"(ncx));
            asm("add.rn.f32x2 %0, %1, %2;" : "=l"(dy) : "l"(xp1[k]), "l"(ncy));
            asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(dd) : "l"(dx));
            asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(dd) : "l"(dy));
            uint32_t da, db;
            asm("mov.b64 {%0,%1}, %2;" : "=r"(da), "=r"(db) : "l"(dd));
            const uint32_t ka = (da & ~cmask) | (uint32_t)c;
            const uint32_t kb = (db & ~cmask) | (uint32_t)(c + 1);
            const uint32_t lo = min(ka, kb), hi = max(ka, kb);
            b2[k] = min(min(b2[k], hi), max(b1[k], lo));
            b1[k] = min(b1[k], lo);
        }
    }
#else
#pragma unroll 2
    for (int c = 0; c < ksub; ++c) {
        const float2 cv = cf_s[c];
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            const float dx = xf0[k] - cv.x, dy = xf1[k] - cv.y;
            const uint32_t key = (__float_as_uint(fmaf(dy, dy, dx * dx)) & ~cmask) | (uint32_t)c;
            b2[k] = min(b2[k], max(b1[k], key));
            b1[k] = min(b1[k], key);
        }
    }
#endif
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const int64_t v = v0 + (int64_t)k * blockDim.x;
        if (v >= n) continue;
        // |d32 - d_true| <= ~4 u d_true (u = 2^-24); the reference's fp64
        // expanded form is within ~4 * 2^-53 (|x|^2 + 2|x.c| + |c|^2) of d_true;
        // the keys drop log2(ksub) mantissa bits (relative 2^(nbits - 23))
        const float xx = fmaf(xf1[k], xf1[k], xf0[k] * xf0[k]);
        const float d1 = __uint_as_float(b1[k] & ~cmask), d2k = __uint_as_float(b2[k] & ~cmask);
        const float trunc = __uint_as_float(0x3f800000u | cmask) - 1.f;  // ksub * 2^-23
        const float tol = (2e-6f + 2.f * trunc) * d1 + 1e-13f * (xx + ccmax) + 1e-30f;
        int a = (int)(b1[k] & cmask);
        if (!(d2k > d1 + tol)) {  // near tie: the exact scan
            const double x0 = (double)xf0[k], x1 = (double)xf1[k];
            const double xxd = __dadd_rn(__dmul_rn(x0, x0), __dmul_rn(x1, x1));
            double best = INFINITY;
            for (int c = 0; c < ksub; ++c) {
                const double2 cv = c_s[c];
                const double xc = __fma_rn(x1, cv.y, __dmul_rn(x0, cv.x));
                const double d2 = fmax(__dadd_rn(__fma_rn(-2.0, xc, xxd), cc_s[c]), 0.0);
                if (d2 < best) {
                    best = d2;
                    a = c;
                }
            }
        }
        codes[code_cell(v, i, ld_codes, rot_base)] = (CT)a;
    }
}

// ---- dsub == 2 with a candidate grid (nbits <= 8) ------------------------
// A 2-D subspace is a plane: per subspace a 64 x 64 grid over the centroids'
// bounding box (+25% each side) lists, per cell, every centroid that can be
// the nearest -- or within 1/128 relative (+ an absolute margin) of it -- for
// a point of the cell (cells widened by 2% for the index rounding).  The
// bound: for x in cell B, d(x, nearest)^2 <= U = min_c max_{y in B} |y - c|^2,
// so a centroid with min_{y in B} |y - c|^2 > U (1 + 1/128) + abs is never
// within the filter's tolerance of the best.  The encoder then runs the same
// fp32 filter (the same keys, the same near-tie test, the same exact fp64
// re-scan over ALL centroids on a near tie) over the cell's list instead of
// all ksub centroids; points outside the grid and cells whose list did not
// fit scan all of them.  Results are therefore the fp32 filter's, i.e. the
// reference's, bit for bit.
// Record per subspace: header (lo_x, lo_y, 1/h_x, 1/h_y, pool bytes used) |
// offs[cells] uint16 | cnt[cells] uint8 (255: full scan) | pool of uint8
// centroid indices (at most EG_POOL bytes, so a CTA stages ~45 KB).
constexpr int EG = 64;                              // cells per axis
constexpr int EG_CELLS = EG * EG;
#ifndef PQKV_ENC_GRID_POOL
#define PQKV_ENC_GRID_POOL 28
#endif
constexpr int EG_POOL = PQKV_ENC_GRID_POOL * 1024;  // candidate-index bytes per subspace
constexpr int EG_LMAX = 24;                         // a longer list -> full scan
constexpr int EG_HDR = 32;
constexpr int EG_OFFS = EG_HDR, EG_CNT = EG_OFFS + 2 * EG_CELLS, EG_PL = EG_CNT + EG_CELLS;
constexpr int EG_REC = EG_PL + EG_POOL;             // bytes per subspace
static_assert(EG_REC % 16 == 0 && EG_PL % 16 == 0, "grid records stay 16-byte aligned");

__global__ void __launch_bounds__(256) build_encode_grid_kernel(const float *__restrict__ cents,
                                                                int ksub,
                                                                unsigned char *__restrict__ grid) {
    const int i = blockIdx.x;
    __shared__ double2 c_s[256];
    __shared__ float hdr_s[4];
    __shared__ double absm_s;
    __shared__ unsigned char n_s[EG_CELLS];
    __shared__ uint16_t off_s[EG_CELLS];
    __shared__ int used_s;
    const float2 *ci = reinterpret_cast<const float2 *>(cents + (size_t)i * ksub * 2);
    unsigned char *rec = grid + (size_t)i * EG_REC;
    for (int c = threadIdx.x; c < ksub; c += blockDim.x) {
        const float2 f = __ldg(ci + c);
        c_s[c] = make_double2(f.x, f.y);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY, amax = 0.0;
        for (int c = 0; c < ksub; ++c) {
            x0 = fmin(x0, c_s[c].x);
            x1 = fmax(x1, c_s[c].x);
            y0 = fmin(y0, c_s[c].y);
            y1 = fmax(y1, c_s[c].y);
            amax = fmax(amax, fmax(fabs(c_s[c].x), fabs(c_s[c].y)));
        }
        const double floor_span = fmax(amax * 0x1p-10, 1e-20);
        const double sx = fmax(x1 - x0, floor_span), sy = fmax(y1 - y0, floor_span);
        const float lx = (float)(x0 - 0.25 * sx), ly = (float)(y0 - 0.25 * sy);
        hdr_s[0] = lx;
        hdr_s[1] = ly;
        hdr_s[2] = (float)(EG / (1.5 * sx));
        hdr_s[3] = (float)(EG / (1.5 * sy));
        const double ext = fmax(amax, fmax(fabs((double)lx), fabs((double)ly))) + 2.0 * fmax(sx, sy);
        absm_s = 1e-9 * ext * ext;  // absolute margin (>> the filter's 1e-13 (|x|^2 + max|c|^2))
    }
    __syncthreads();
    const double lx = hdr_s[0], ly = hdr_s[1];
    const double hx = 1.0 / (double)hdr_s[2], hy = 1.0 / (double)hdr_s[3];
    const double absm = absm_s;
    // pass 1: list lengths; pass 2 (after the offsets): the lists
    for (int pass = 0; pass < 2; ++pass) {
        for (int cell = threadIdx.x; cell < EG_CELLS; cell += blockDim.x) {
            const int ix = cell % EG, iy = cell / EG;
            const double bx0 = lx + (ix - 0.02) * hx, bx1 = lx + (ix + 1.02) * hx;
            const double by0 = ly + (iy - 0.02) * hy, by1 = ly + (iy + 1.02) * hy;
            if (pass == 1 && n_s[cell] == 255) continue;
            double U = INFINITY;
            for (int c = 0; c < ksub; ++c) {
                const double dx = fmax(fabs(c_s[c].x - bx0), fabs(c_s[c].x - bx1));
                const double dy = fmax(fabs(c_s[c].y - by0), fabs(c_s[c].y - by1));
                U = fmin(U, dx * dx + dy * dy);
            }
            const double thr = U * (1.0 + 1.0 / 128) + absm;
            int n = 0;
            unsigned char *dst = rec + EG_PL + (pass ? off_s[cell] : 0);
            for (int c = 0; c < ksub; ++c) {
                const double dx = fmax(0.0, fmax(bx0 - c_s[c].x, c_s[c].x - bx1));
                const double dy = fmax(0.0, fmax(by0 - c_s[c].y, c_s[c].y - by1));
                if (dx * dx + dy * dy <= thr) {
                    if (pass == 1) dst[n] = (unsigned char)c;
                    ++n;
                }
            }
            if (pass == 0) n_s[cell] = n <= EG_LMAX ? (unsigned char)n : (unsigned char)255;
        }
        __syncthreads();
        if (pass == 0 && threadIdx.x == 0) {  // offsets; lists past the pool -> full scan
            int off = 0;
            for (int cell = 0; cell < EG_CELLS; ++cell) {
                const int n = n_s[cell];
                // lists start on 4-byte boundaries: the encoder reads 4 candidates per load
                const int n4 = (n + 3) & ~3;
                if (n == 255 || off + n4 > EG_POOL) {
                    n_s[cell] = 255;
                    off_s[cell] = 0;
                } else {
                    off_s[cell] = (uint16_t)off;
                    off += n4;
                }
            }
            used_s = off;
        }
        __syncthreads();
    }
    if (threadIdx.x < 4) reinterpret_cast<float *>(rec)[threadIdx.x] = hdr_s[threadIdx.x];
    if (threadIdx.x == 4) reinterpret_cast<int *>(rec)[4] = used_s;
    for (int cell = threadIdx.x; cell < EG_CELLS; cell += blockDim.x) {
        reinterpret_cast<uint16_t *>(rec + EG_OFFS)[cell] = off_s[cell];
        rec[EG_CNT + cell] = n_s[cell];
    }
}

#ifndef PQKV_ENC_GRID_VPT
#define PQKV_ENC_GRID_VPT 2  // vectors per thread per pass (their loads in flight together)
#endif
#ifndef PQKV_ENC_GRID_CTAS
#define PQKV_ENC_GRID_CTAS 4  // persistent CTAs per SM over (subspace, row block) pairs
#endif
template <typename TX, typename CT, int VPT>
__global__ void __launch_bounds__(256) encode_dsub2_grid(const TX *__restrict__ x, int64_t n,
                                                         int64_t ld_x,
                                                         const float *__restrict__ cents,
                                                         const unsigned char *__restrict__ grid,
                                                         int ksub, CT *__restrict__ codes,
                                                         int64_t ld_codes, int64_t rot_base,
                                                         int64_t x_bs, int64_t c_bs, int64_t g_bs,
                                                         int64_t codes_bs) {
    x += blockIdx.z * x_bs;
    cents += blockIdx.z * c_bs;
    grid += blockIdx.z * g_bs;
    codes += blockIdx.z * codes_bs;
    extern __shared__ double sm[];
    double2 *c_s = reinterpret_cast<double2 *>(sm);                   // [ksub]
    double *cc_s = sm + 2 * (size_t)ksub;                              // [ksub]
    float2 *cf_s = reinterpret_cast<float2 *>(sm + 3 * (size_t)ksub);  // [ksub]
    unsigned char *g_s = reinterpret_cast<unsigned char *>(sm + 4 * (size_t)ksub);  // record
    __shared__ float ccmax_s;
    const int i = blockIdx.x;
    const float2 *ci = reinterpret_cast<const float2 *>(cents + (size_t)i * ksub * 2);
    const unsigned char *rec = grid + (size_t)i * EG_REC;
    if (threadIdx.x == 0) ccmax_s = 0.f;
    {
        // header, offsets, counts and the used part of the pool
        const int used = __ldg(reinterpret_cast<const int *>(rec) + 4);
        const int bytes = EG_PL + ((used + 15) & ~15);
        const uint4 *src = reinterpret_cast<const uint4 *>(rec);
        uint4 *dst = reinterpret_cast<uint4 *>(g_s);
        for (int k = threadIdx.x; k < bytes / 16; k += blockDim.x) dst[k] = __ldg(src + k);
    }
    __syncthreads();
    float ccmax = 0.f;
    for (int c = threadIdx.x; c < ksub; c += blockDim.x) {
        const float2 f = __ldg(ci + c);
        const double a = f.x, b = f.y;
        c_s[c] = make_double2(a, b);
        cc_s[c] = __dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b));
        cf_s[c] = f;
        ccmax = fmaxf(ccmax, (float)cc_s[c]);
    }
    atomicMax(reinterpret_cast<int *>(&ccmax_s), __float_as_int(ccmax));
    __syncthreads();
    ccmax = ccmax_s;
    const float *hdr = reinterpret_cast<const float *>(g_s);
    const float lx = hdr[0], ly = hdr[1], ihx = hdr[2], ihy = hdr[3];
    const uint16_t *off_s = reinterpret_cast<const uint16_t *>(g_s + EG_OFFS);
    const unsigned char *cnt_s = g_s + EG_CNT;
    const unsigned char *pool_s = g_s + EG_PL;
    const uint32_t cmask = (uint32_t)ksub - 1u;
    const float trunc = __uint_as_float(0x3f800000u | cmask) - 1.f;  // ksub * 2^-23

    for (int64_t v0 = ((int64_t)blockIdx.y * VPT) * blockDim.x + threadIdx.x; v0 < n;
         v0 += (int64_t)gridDim.y * VPT * blockDim.x) {
        float xa[VPT], xb[VPT];
#pragma unroll
        for (int k = 0; k < VPT; ++k) {  // every load of the pass in flight at once
            const int64_t v = v0 + (int64_t)k * blockDim.x;
            const int64_t vv = v < n ? v : n - 1;
            load_pair<TX>(x + vv * ld_x + (int64_t)i * 2, xa[k], xb[k]);
        }
#pragma unroll
        for (int k = 0; k < VPT; ++k) {  // unrolled: xa / xb stay in registers
            const int64_t v = v0 + (int64_t)k * blockDim.x;
            if (v >= n) break;
            const float xf0 = xa[k], xf1 = xb[k];
            const float fx = (xf0 - lx) * ihx, fy = (xf1 - ly) * ihy;
            int nc = 255, off = 0;
            if (fx >= 0.f && fx < (float)EG && fy >= 0.f && fy < (float)EG) {
                const int cell = (int)fy * EG + (int)fx;
                nc = cnt_s[cell];
                off = off_s[cell];
            }
            // best / second-best keys (encode_dsub2_filter): the same distance
            // formula, so the same keys for the same centroids
            auto key_of = [&](int c) {
                const float2 cv = cf_s[c];
                const float dx = xf0 + (-cv.x), dy = xf1 + (-cv.y);
                return (__float_as_uint(fmaf(dy, dy, dx * dx)) & ~cmask) | (uint32_t)c;
            };
            uint32_t b1 = 0xffffffffu, b2;
            if (nc != 255) {
                b2 = 0x7f7fffffu;  // a one-entry list has no competitor: FLT_MAX
                const uint32_t *pw = reinterpret_cast<const uint32_t *>(pool_s + off);
                uint32_t word = 0;
                for (int k2 = 0; k2 < nc; ++k2) {
                    if ((k2 & 3) == 0) word = pw[k2 >> 2];  // 4 candidates per load
                    const uint32_t key = key_of((int)((word >> (8 * (k2 & 3))) & 0xffu));
                    b2 = min(b2, max(b1, key));
                    b1 = min(b1, key);
                }
            } else {
                b2 = 0xffffffffu;
                for (int c = 0; c < ksub; ++c) {
                    const uint32_t key = key_of(c);
                    b2 = min(b2, max(b1, key));
                    b1 = min(b1, key);
                }
            }
            const float xx = fmaf(xf1, xf1, xf0 * xf0);
            const float d1 = __uint_as_float(b1 & ~cmask), d2k = __uint_as_float(b2 & ~cmask);
            const float tol = (2e-6f + 2.f * trunc) * d1 + 1e-13f * (xx + ccmax) + 1e-30f;
            int a = (int)(b1 & cmask);
            if (!(d2k > d1 + tol)) {  // near tie: the exact scan over every centroid
                const double x0 = (double)xf0, x1 = (double)xf1;
                const double xxd = __dadd_rn(__dmul_rn(x0, x0), __dmul_rn(x1, x1));
                double best = INFINITY;
                for (int c = 0; c < ksub; ++c) {
                    const double2 cv = c_s[c];
                    const double xc = __fma_rn(x1, cv.y, __dmul_rn(x0, cv.x));
                    const double d2 = fmax(__dadd_rn(__fma_rn(-2.0, xc, xxd), cc_s[c]), 0.0);
                    if (d2 < best) {
                        best = d2;
                        a = c;
                    }
                }
            }
            codes[code_cell(v, i, ld_codes, rot_base)] = (CT)a;
        }
    }
}

template <typename TX, typename CT>
int launch_dsub2_grid(const void *x, int64_t n, int64_t ld_x, const float *cents,
                      const unsigned char *grid, int M, int ksub, void *codes, int64_t ld_codes,
                      int64_t rot_base, cudaStream_t st, int batches = 1, int64_t x_bs = 0,
                      int64_t c_bs = 0, int64_t g_bs = 0, int64_t codes_bs = 0) {
    constexpr int VPT = PQKV_ENC_GRID_VPT;
    const size_t smem = (size_t)256 * 4 * sizeof(double) + EG_REC;  // the pool's worst case
    auto k = encode_dsub2_grid<TX, CT, VPT>;
    static int attr_set[64] = {0};  // the attribute is per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 64 || !attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return fail(PQKV_ECUDA, "encode: %s", cudaGetErrorString(e));
        if (dev < 64) attr_set[dev] = 1;
    }
    // persistent row blocks: ~4 CTAs (of ~54 KB shared memory) per SM over
    // (subspace, row block) pairs
    int64_t blocks = (n + 256 * VPT - 1) / (256 * VPT);
    const int64_t target =
        std::max<int64_t>(1, (int64_t)PQKV_ENC_GRID_CTAS * 148 / std::max(1, M * batches));
    blocks = std::min<int64_t>(blocks, target);
    dim3 g((unsigned)M, (unsigned)std::min<int64_t>(blocks, 65535), (unsigned)batches);
    k<<<g, 256, smem, st>>>((const TX *)x, n, ld_x, cents, grid, ksub, (CT *)codes, ld_codes,
                            rot_base, x_bs, c_bs, g_bs, codes_bs);
    return launch_status("pqkv_encode_grid");
}

template <typename TX, typename CT, int VPT>
int launch_dsub2_filter_vpt(const void *x, int64_t n, int64_t ld_x, const float *cents, int M,
                            int ksub, void *codes, int64_t ld_codes, int64_t rot_base,
                            cudaStream_t st, int batches, int64_t x_bs, int64_t c_bs,
                            int64_t codes_bs) {
    const size_t smem = (size_t)ksub * (3 * sizeof(double) + sizeof(float2));
    auto k = encode_dsub2_filter<TX, CT, VPT>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return fail(PQKV_ECUDA, "encode: %s", cudaGetErrorString(e));
    }
    dim3 grid((unsigned)M, (unsigned)((n + 256 * VPT - 1) / (256 * VPT)), (unsigned)batches);
    k<<<grid, 256, smem, st>>>((const TX *)x, n, ld_x, cents, ksub, (CT *)codes, ld_codes,
                               rot_base, x_bs, c_bs, codes_bs);
    return launch_status("pqkv_encode");
}

// 8 vectors per thread for large inputs (prefill); 4 for small batches (the
// append path's 32-row flushes), where 8 would leave half the lanes idle
template <typename TX, typename CT>
int launch_dsub2_filter(const void *x, int64_t n, int64_t ld_x, const float *cents, int M,
                        int ksub, void *codes, int64_t ld_codes, int64_t rot_base,
                        cudaStream_t st, int batches = 1, int64_t x_bs = 0, int64_t c_bs = 0,
                        int64_t codes_bs = 0) {
    if (n >= 256 * PQKV_ENC_FILTER_VPT * 4)
        return launch_dsub2_filter_vpt<TX, CT, PQKV_ENC_FILTER_VPT>(
            x, n, ld_x, cents, M, ksub, codes, ld_codes, rot_base, st, batches, x_bs, c_bs,
            codes_bs);
    return launch_dsub2_filter_vpt<TX, CT, 4>(x, n, ld_x, cents, M, ksub, codes, ld_codes,
                                             rot_base, st, batches, x_bs, c_bs, codes_bs);
}

template <typename TX, typename CT>
int launch_dsub2(const void *x, int64_t n, int64_t ld_x, const float *cents, int M, int ksub,
                 void *codes, int64_t ld_codes, int64_t rot_base, cudaStream_t st) {
    constexpr int VPT = PQKV_ENC_VPT;
    const size_t smem = (size_t)ksub * 3 * sizeof(double);
    auto k = encode_dsub2<TX, CT, VPT>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return fail(PQKV_ECUDA, "encode: %s", cudaGetErrorString(e));
    }
    dim3 grid((unsigned)((n + 256 * VPT - 1) / (256 * VPT)), (unsigned)M);
    k<<<grid, 256, smem, st>>>((const TX *)x, n, ld_x, cents, ksub, (CT *)codes, ld_codes,
                               rot_base);
    return launch_status("pqkv_encode");
}

// Any dsub: operands read from global memory (L1-resident per subspace).
template <typename TX, typename CT>
__global__ void __launch_bounds__(256) encode_generic(const TX *__restrict__ x, int64_t n,
                                                      int64_t ld_x, const float *__restrict__ cents,
                                                      int ksub, int dsub, CT *__restrict__ codes,
                                                      int64_t ld_codes, int64_t rot_base) {
    const int i = blockIdx.y;
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const TX *xr = x + v * ld_x + (int64_t)i * dsub;
    const float *ci = cents + (size_t)i * ksub * dsub;
    const double xx = np_pairwise(
        [&](int j) {
            const double a = load_x<TX>(xr + j);
            return a * a;
        },
        0, dsub);
    double best = INFINITY;
    int arg = 0;
    for (int c = 0; c < ksub; ++c) {
        const float *cr = ci + (size_t)c * dsub;
        double xc = load_x<TX>(xr) * (double)__ldg(cr);
        for (int j = 1; j < dsub; ++j) xc = fma(load_x<TX>(xr + j), (double)__ldg(cr + j), xc);
        const double cc = np_pairwise(
            [&](int j) {
                const double a = (double)__ldg(cr + j);
                return a * a;
            },
            0, dsub);
        double d2 = fmax((xx - 2.0 * xc) + cc, 0.0);
        if (d2 < best) {
            best = d2;
            arg = c;
        }
    }
    codes[code_cell(v, i, ld_codes, rot_base)] = (CT)arg;
}

template <typename TX, typename CT, int DSUB>
int launch_staged(const void *x, int64_t n, int64_t ld_x, const float *cents, int M, int ksub,
                  void *codes, int64_t ld_codes, int64_t rot_base, cudaStream_t st) {
    const size_t smem = (size_t)ksub * (DSUB + 1) * sizeof(double);
    auto k = encode_staged<TX, CT, DSUB>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return fail(PQKV_ECUDA, "encode: %s", cudaGetErrorString(e));
    }
    dim3 grid((unsigned)((n + 255) / 256), (unsigned)M);
    k<<<grid, 256, smem, st>>>((const TX *)x, n, ld_x, cents, ksub, (CT *)codes, ld_codes,
                               rot_base);
    return launch_status("pqkv_encode");
}

template <typename TX, typename CT>
int dispatch_encode(const void *x, int64_t n, int d, int64_t ld_x, const float *cents, int M,
                    int nbits, void *codes, int64_t ld_codes, int64_t rot_base, cudaStream_t st) {
    const int ksub = 1 << nbits, dsub = d / M;
    const size_t staged_smem = (size_t)ksub * (dsub + 1) * sizeof(double);
    if (staged_smem <= 160 * 1024) {
        switch (dsub) {
            case 1: return launch_staged<TX, CT, 1>(x, n, ld_x, cents, M, ksub, codes, ld_codes, rot_base, st);
            case 2:
#if PQKV_ENC_VPT > 0
#if PQKV_ENC_FILTER
                if (ksub * 32 <= 160 * 1024 && n <= (int64_t)65535 * 256 * PQKV_ENC_FILTER_VPT)
                    return launch_dsub2_filter<TX, CT>(x, n, ld_x, cents, M, ksub, codes,
                                                       ld_codes, rot_base, st);
#endif
                if (ksub * 3 * sizeof(double) <= 160 * 1024)
                    return launch_dsub2<TX, CT>(x, n, ld_x, cents, M, ksub, codes, ld_codes,
                                                rot_base, st);
#endif
                return launch_staged<TX, CT, 2>(x, n, ld_x, cents, M, ksub, codes, ld_codes, rot_base, st);
            case 4: return launch_staged<TX, CT, 4>(x, n, ld_x, cents, M, ksub, codes, ld_codes, rot_base, st);
            case 8: return launch_staged<TX, CT, 8>(x, n, ld_x, cents, M, ksub, codes, ld_codes, rot_base, st);
            case 16: return launch_staged<TX, CT, 16>(x, n, ld_x, cents, M, ksub, codes, ld_codes, rot_base, st);
            default: break;
        }
    }
    dim3 grid((unsigned)((n + 255) / 256), (unsigned)M);
    encode_generic<TX, CT><<<grid, 256, 0, st>>>((const TX *)x, n, ld_x, cents, ksub, dsub,
                                                  (CT *)codes, ld_codes, rot_base);
    return launch_status("pqkv_encode");
}

template <typename TX>
int dispatch_cell(const void *x, int64_t n, int d, int64_t ld_x, const float *cents, int M,
                  int nbits, void *codes, int64_t ld_codes, int64_t rot_base, cudaStream_t st) {
    if (nbits <= 8)
        return dispatch_encode<TX, uint8_t>(x, n, d, ld_x, cents, M, nbits, codes, ld_codes,
                                            rot_base, st);
    return dispatch_encode<TX, uint16_t>(x, n, d, ld_x, cents, M, nbits, codes, ld_codes,
                                         rot_base, st);
}

}  // namespace
}  // namespace pqkv

using namespace pqkv;

extern "C" int pqkv_encode_batched(const void *x, int x_dtype, int batches, int64_t n, int d,
                                   int64_t ld_x, int64_t x_bstride, const float *centroids,
                                   int64_t c_bstride, int M, int nbits, void *codes,
                                   int64_t ld_codes, int64_t codes_bstride, int64_t rot_base,
                                   void *stream) {
    PQKV_CHECK_ARG(batches >= 0 && batches <= 65535, "pqkv_encode_batched: bad batch count");
    PQKV_CHECK_ARG(geometry_ok(d, M, nbits), "pqkv_encode_batched: bad geometry");
    PQKV_CHECK_ARG(x_bstride >= 0 && c_bstride >= 0 && codes_bstride >= 0,
                   "pqkv_encode_batched: negative batch stride");
    if (batches == 0 || n == 0) return PQKV_OK;
    const int ksub = 1 << nbits, esz = x_dtype == PQKV_DTYPE_F32 ? 4 : 2, csz = nbits <= 8 ? 1 : 2;
    // one launch for the batch on the dsub = 2 fast path (f32 rows); else per batch
    if (d == 2 * M && x_dtype == PQKV_DTYPE_F32 && PQKV_ENC_VPT > 0 && PQKV_ENC_FILTER &&
        ksub * 32 <= 160 * 1024 && x && centroids && codes && ld_x >= d && ld_codes >= M &&
        n <= (int64_t)65535 * 256 * PQKV_ENC_VPT &&
        (rot_base < 0 || is_fast_geometry(d, M, nbits))) {
        cudaStream_t st = as_stream(stream);
        return nbits <= 8
                   ? launch_dsub2_filter<float, uint8_t>(x, n, ld_x, centroids, M, ksub, codes,
                                                         ld_codes, rot_base, st, batches,
                                                         x_bstride, c_bstride, codes_bstride)
                   : launch_dsub2_filter<float, uint16_t>(x, n, ld_x, centroids, M, ksub, codes,
                                                          ld_codes, rot_base, st, batches,
                                                          x_bstride, c_bstride, codes_bstride);
    }
    for (int b = 0; b < batches; ++b) {
        int rc = pqkv_encode((const char *)x + b * x_bstride * esz, x_dtype, n, d, ld_x,
                             centroids + b * c_bstride, M, nbits,
                             (char *)codes + b * codes_bstride * csz, ld_codes, rot_base, stream);
        if (rc) return rc;
    }
    return PQKV_OK;
}

static bool grid_geometry(int d, int M, int nbits) { return d == 2 * M && nbits <= 8; }

extern "C" int64_t pqkv_encode_grid_bytes(int d, int M, int nbits) {
    return (geometry_ok(d, M, nbits) && grid_geometry(d, M, nbits)) ? (int64_t)M * EG_REC : 0;
}

extern "C" int pqkv_build_encode_grid(const float *centroids, int d, int M, int nbits, void *grid,
                                      void *stream) {
    PQKV_CHECK_ARG(geometry_ok(d, M, nbits) && grid_geometry(d, M, nbits),
                   "pqkv_build_encode_grid: the candidate grid exists for dsub = 2, nbits <= 8");
    PQKV_CHECK_ARG(centroids && grid, "pqkv_build_encode_grid: null pointer");
    build_encode_grid_kernel<<<M, 256, 0, as_stream(stream)>>>(centroids, 1 << nbits,
                                                               (unsigned char *)grid);
    return launch_status("pqkv_build_encode_grid");
}

extern "C" int pqkv_encode_grid(const void *x, int x_dtype, int64_t n, int d, int64_t ld_x,
                                const float *centroids, const void *grid, int M, int nbits,
                                void *codes, int64_t ld_codes, int64_t rot_base, void *stream) {
    if (grid == nullptr)
        return pqkv_encode(x, x_dtype, n, d, ld_x, centroids, M, nbits, codes, ld_codes, rot_base,
                           stream);
    PQKV_CHECK_ARG(geometry_ok(d, M, nbits) && grid_geometry(d, M, nbits),
                   "pqkv_encode_grid: the candidate grid exists for dsub = 2, nbits <= 8");
    PQKV_CHECK_ARG(n >= 0, "pqkv_encode_grid: n must be >= 0");
    PQKV_CHECK_ARG(ld_x >= d && ld_codes >= M, "pqkv_encode_grid: row strides too small");
    if (n == 0) return PQKV_OK;
    PQKV_CHECK_ARG(x && centroids && codes, "pqkv_encode_grid: null pointer");
    PQKV_CHECK_ARG(rot_base < 0 || is_fast_geometry(d, M, nbits),
                   "pqkv_encode_grid: the decode layout exists only for m64b8");
    cudaStream_t st = as_stream(stream);
    const int ksub = 1 << nbits;
    const unsigned char *g = (const unsigned char *)grid;
    switch (x_dtype) {
        case PQKV_DTYPE_F32:
            return launch_dsub2_grid<float, uint8_t>(x, n, ld_x, centroids, g, M, ksub, codes,
                                                     ld_codes, rot_base, st);
        case PQKV_DTYPE_BF16:
            return launch_dsub2_grid<__nv_bfloat16, uint8_t>(x, n, ld_x, centroids, g, M, ksub,
                                                             codes, ld_codes, rot_base, st);
        case PQKV_DTYPE_F16:
            return launch_dsub2_grid<__half, uint8_t>(x, n, ld_x, centroids, g, M, ksub, codes,
                                                      ld_codes, rot_base, st);
        default:
            return fail(PQKV_EINVAL, "pqkv_encode_grid: unknown dtype %d", x_dtype);
    }
}

extern "C" int pqkv_encode_batched_grid(const void *x, int batches, int64_t n, int d,
                                        int64_t ld_x, int64_t x_bstride, const float *centroids,
                                        int64_t c_bstride, const void *grid, int64_t g_bstride,
                                        int M, int nbits, void *codes, int64_t ld_codes,
                                        int64_t codes_bstride, int64_t rot_base, void *stream) {
    PQKV_CHECK_ARG(batches >= 0 && batches <= 65535, "pqkv_encode_batched_grid: bad batch count");
    PQKV_CHECK_ARG(geometry_ok(d, M, nbits) && grid_geometry(d, M, nbits),
                   "pqkv_encode_batched_grid: the candidate grid exists for dsub = 2, nbits <= 8");
    PQKV_CHECK_ARG(x_bstride >= 0 && c_bstride >= 0 && g_bstride >= 0 && codes_bstride >= 0,
                   "pqkv_encode_batched_grid: negative batch stride");
    if (batches == 0 || n == 0) return PQKV_OK;
    PQKV_CHECK_ARG(x && centroids && grid && codes && ld_x >= d && ld_codes >= M,
                   "pqkv_encode_batched_grid: bad arguments");
    PQKV_CHECK_ARG(rot_base < 0 || is_fast_geometry(d, M, nbits),
                   "pqkv_encode_batched_grid: the decode layout exists only for m64b8");
    return launch_dsub2_grid<float, uint8_t>(x, n, ld_x, centroids, (const unsigned char *)grid,
                                             M, 1 << nbits, codes, ld_codes, rot_base,
                                             as_stream(stream), batches, x_bstride, c_bstride,
                                             g_bstride, codes_bstride);
}

extern "C" int pqkv_encode(const void *x, int x_dtype, int64_t n, int d, int64_t ld_x,
                           const float *centroids, int M, int nbits, void *codes,
                           int64_t ld_codes, int64_t rot_base, void *stream) {
    PQKV_CHECK_ARG(geometry_ok(d, M, nbits), "pqkv_encode: bad geometry d=%d M=%d nbits=%d", d,
                   M, nbits);
    PQKV_CHECK_ARG(n >= 0, "pqkv_encode: n must be >= 0");
    PQKV_CHECK_ARG(ld_x >= d && ld_codes >= M, "pqkv_encode: row strides too small");
    if (n == 0) return PQKV_OK;
    PQKV_CHECK_ARG(x && centroids && codes, "pqkv_encode: null pointer");
    PQKV_CHECK_ARG(n <= (int64_t)65535 * 256 * 1024, "pqkv_encode: n too large");
    PQKV_CHECK_ARG(rot_base < 0 || is_fast_geometry(d, M, nbits),
                   "pqkv_encode: the decode layout exists only for m64b8 (d=128, M=64, nbits=8)");
    cudaStream_t st = as_stream(stream);
    switch (x_dtype) {
        case PQKV_DTYPE_F32:
            return dispatch_cell<float>(x, n, d, ld_x, centroids, M, nbits, codes, ld_codes,
                                        rot_base, st);
        case PQKV_DTYPE_BF16:
            return dispatch_cell<__nv_bfloat16>(x, n, d, ld_x, centroids, M, nbits, codes,
                                                ld_codes, rot_base, st);
        case PQKV_DTYPE_F16:
            return dispatch_cell<__half>(x, n, d, ld_x, centroids, M, nbits, codes, ld_codes,
                                         rot_base, st);
        default:
            return fail(PQKV_EINVAL, "pqkv_encode: unknown dtype %d", x_dtype);
    }
}
