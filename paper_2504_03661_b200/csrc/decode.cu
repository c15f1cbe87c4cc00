// K2/K3 -- decode attention over a product-quantized KV cache.
//
// Reference semantics (paths relative to pkg/src/pqkv/):
//   quantized_partial  attention.py:114-166  scores via the key LUT
//                      (score_codes, _kernels.py:27-34), m = max, p = e^(s-m),
//                      l = sum p, acc = sum_t p_t * V_hat_t computed without
//                      materialising V_hat (attention.py:103-111 / :155-157)
//   merge_partials     attention.py:193-204
//   dense_partial      attention.py:169-190 (recent rows + current token)
//   finalize           attention.py:207-211
//   decode_step        attention.py:214-287 (block split -> our CTA split)
//
// decode_partials_m64b8 (the fast path, d=128 M=64 nbits=8), one fused
// launch per layer (pqkv_decode_attention), PDL-chained:
//   * persistent grid, one CTA per SM (16 warps on the exact path); the
//     flattened token space of all heads is cut into equal chunks
//     (common.cuh CostMap); a (CTA, head) overlap is a segment;
//   * shared memory: the head's key LUT, centroid-major [256][64] fp32
//     (64 KiB), and the value codebook as two [256][32] float2 halves
//     (128 KiB, loaded once per CTA);
//   * a warp handles 16 tokens per unit (two independent 8-token halves, one
//     merged softmax update): lane = (token slot, 16-subspace quarter) loads
//     the 16 K-code and 16 V-code bytes of its quarter with one 128-bit load
//     each (coalesced: the warp reads 4 x 512 contiguous B) into a static
//     RING-unit register ring driven by running pointers; the loop body is
//     straight-line (masked tail units) so no branch drains the ring;
//   * codes are stored in the decode layout (common.cuh): each quarter is
//     pre-rotated by its lane constant r, so at every unrolled step the 32
//     lanes touch 32 distinct subspaces mod 32 without any in-register
//     shuffling: the LUT gather (bank = subspace mod 32) and the 64-bit
//     codebook gather (8-byte slot = subspace mod 16 per half-warp) are
//     bank-conflict free for ANY code values;
//   * one PRMT per code byte forms the shared-memory byte address
//     (code << 8 | lane offset | half << 16);
//   * the 4 lanes of a token combine their partial scores with 2 shuffles;
//     each token slot keeps its own online-softmax state (m, l) and 32 fp32
//     value accumulators (its quarter's 16 subspaces x dsub 2);
//   * epilogue: slot partials are rescaled to the CTA max and summed through
//     shared memory into one (m, l, acc[128]) record per segment; the CTA
//     holding a head's last tokens adds the dense record (recent rows +
//     current token); the last CTA to arrive (acq_rel counter) merges the
//     head's records in CTA order and finalizes;
//   * fp16 value-codebook mode: 4-byte value gathers + mixed f16 x f16 + f32
//     FMAs; with an even GQA group a CTA serves HG = 2 query heads (two key
//     tables, one value gather per code shared by both);
//   * GQA shared code stream (Args::share = P): the P CTAs serving the P
//     virtual heads of one KV head split the same token ranges at the same
//     time, so each code line is fetched from DRAM once.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace pqkv {
namespace {

constexpr int kPS = PQKV_PARTIAL_HEADER;  // record = [m, l, 0, 0, acc[d]]

// ============================================================ fast path ====
// PDL (programmatic dependent launch): a grid launched with the
// programmatic-serialization attribute may start while the previous kernel on
// the stream drains; griddepcontrol.wait blocks until that kernel finished
// and its memory is visible.  Both are no-ops without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

namespace fast {
constexpr int M = 64, KSUB = 256, D = 128;
// Lazy rescaling of the online softmax: the running max moves only when a
// score exceeds it by more than kLazyRescale (log2 units), so weights are at
// most 2^kLazyRescale and the accumulators are rescaled a few times per
// segment instead of on most units.  Any reference point gives the same
// (m, l, acc) record up to rounding (the merge rescales records by their m).
#ifndef PQKV_LAZY_RESCALE
#define PQKV_LAZY_RESCALE 8
#endif
constexpr float kLazyRescale = PQKV_LAZY_RESCALE;
#ifndef PQKV_WARPS
#define PQKV_WARPS 16
#endif
constexpr int WARPS = PQKV_WARPS, NT = WARPS * 32;  // one persistent CTA per SM
static_assert(NT % 128 == 0, "WARPS must be a multiple of 4");
#ifndef PQKV_RING
#define PQKV_RING 2
#endif
constexpr int RING = PQKV_RING;  // register ring depth (units of 16 tokens per warp)
#ifndef PQKV_EARLY_KEYS
#define PQKV_EARLY_KEYS 1
#endif
#ifndef PQKV_GROUP
#define PQKV_GROUP 1
#endif
constexpr int GROUP = PQKV_GROUP;  // units processed together (key phase, one max update, value phase)
// Lane geometry (common.cuh decode layout): a lane owns SPL consecutive
// subspaces (code bytes) of a token; TL lanes per token, TS token slots per
// warp instruction, a unit = UT = 2 TS tokens per warp (halves A and B).
constexpr int SPL = PQKV_LANE8 ? 8 : 16;
constexpr int TL = M / SPL;
constexpr int TS = 32 / TL;
constexpr int UT = 2 * TS;
constexpr int NPK = SPL / 2;  // lane-constant pack words per kind
constexpr int LUT_BYTES = KSUB * M * 4;     // 65536
constexpr int CV_BYTES = KSUB * M * 2 * 4;  // 131072
// shared-memory map (bytes from the dynamic base)
// sized for up to PQKV_WARPS_MAX warps and two heads per CTA
#define PQKV_WARPS_MAX 24
constexpr int WMAX = PQKV_WARPS_MAX;
constexpr int OFF_RED = LUT_BYTES + CV_BYTES;                 // red_m[2][W], red_l[2][W]
constexpr int OFF_COL = OFF_RED + 4 * WMAX * 4;               // colsum[2 * NG][128]
constexpr int OFF_DNS = OFF_COL + 2 * (WMAX / 4) * D * 4;     // dense m[W], l[W], acc[W][128]
constexpr int OFF_BAR = OFF_DNS + (2 * WMAX + WMAX * D) * 4;  // 2 mbarriers
constexpr int OFF_FLAG = OFF_BAR + 16;  // finisher flags [W / 4], then the stale-n_q flag
constexpr int OFF_NQ = OFF_FLAG + 4 * (WMAX / 4 + 4);           // n_q copy [kNqCache]
constexpr int kNqCache = 256;  // batches whose lengths are kept in shared memory
constexpr int SMEM_BYTES = OFF_NQ + 4 * kNqCache;

#ifdef PQKV_TRACE
// debug-only timeline: per (launch mod 64, CTA) [smid, t_entry, t_ready,
// t_loop0_end, t_exit, nseg, t_segs_done, t_post_wait, t_lut_pre, t_cv_ready]
constexpr int kTraceLaunches = 64, kTraceCtas = 256;
constexpr int kTraceSlots = 32;
__device__ unsigned long long g_trace[kTraceLaunches * kTraceCtas * kTraceSlots];
__device__ unsigned long long g_wtrace[kTraceLaunches * kTraceCtas * 32];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define PQKV_TR(slot, val)                                                          \
    if (threadIdx.x == 0 && blockIdx.x < kTraceCtas)                                \
    g_trace[((A.trace_id % kTraceLaunches) * kTraceCtas + blockIdx.x) * kTraceSlots + (slot)] = (val)
// intra-CTA phase: SM cycles since the grid-dependency wait returned
#define PQKV_TRC(slot) PQKV_TR(slot, clock64() - clk_pw_)
#else
#define PQKV_TR(slot, val)
#endif

struct Args {
    const float *q;
    float scale;
    const float *ck;   // key codebook layout (kLutFromQ) ...
    const float *lut;  // ... or precomputed tables [B*Hq][256][64]
    int B, Hq, Hkv;
    const uint8_t *codes_k, *codes_v;
    int64_t ld_tok;
    const int32_t *n_q;
    const float *cv;
    int num_ctas;
    float *parts;
    // fused finish (counters == nullptr: partial records only)
    int32_t *counters;
    const float *recent_k, *recent_v;
    int64_t ld_recent;
    const int32_t *n_recent;
    const float *k_cur, *v_cur;
    float *out, *lse, *merged;
    int early_cv;     // codebooks may be read before the grid-dependency wait
    int early_codes;  // n_q and the codes below it may be read before it, too
    int share;        // P > 1: CTAs c = P j + k (k < P) split the same token ranges of the
                      // P virtual heads of one KV head (P j .. P j + P - 1), concurrently,
                      // so each code line is fetched from DRAM once and hit in L2 P - 1 times
    int trace_id;  // PQKV_TRACE builds: launch sequence number
    int append;    // PQKV_DECODE_APPEND_RECENT (one head): the finisher appends (k_cur, v_cur)
};

#if PQKV_LANE8
__device__ __forceinline__ uint2 ld_stream8(const uint8_t *p) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "=r"(r.x), "=r"(r.y)
                 : "l"(p));
    return r;
}
#endif
__device__ __forceinline__ uint4 ld_stream(const uint8_t *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// Shared-memory addresses on sm_100 are (CgaCtaId << 24) + window offset,
// and with no static __shared__ the dynamic buffer starts at window offset
// 0x400 (after the 1 KiB system reservation).  The PRMT-built address holds
// the code byte, the lane offset and the CTA-id byte; the region offset rides
// in the LDS immediate, so each lookup is exactly PRMT + LDS.
constexpr uint32_t kDynBase = 0x400;

// key table of head k (of HG) at dynamic offset k * 64 KiB
template <int IMM>
__device__ __forceinline__ float lds_f32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(a), "n"(IMM));
    return v;
}

// value codebook after the HG key tables: fp32 [2][256][32] float2, or fp16
// [256][2][32] half2 (256-byte rows, subspace half in byte 7 of the address)
template <int HG>
__device__ __forceinline__ unsigned long long lds_cv(uint32_t a) {
    unsigned long long v;
    asm volatile("ld.shared.b64 %0, [%1+%2];" : "=l"(v) : "r"(a), "n"(0x400 + HG * 0x10000));
    return v;
}
template <int HG>
__device__ __forceinline__ uint32_t lds_cv32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(0x400 + HG * 0x10000));
    return v;
}

// acc.xy += p16 * (half2) c: two mixed-precision FMAs (f16 x f16 products
// are exact in fp32; the sums are fp32)
__device__ __forceinline__ void fhfma2(unsigned long long &acc, uint16_t p16, uint32_t h) {
    float a, b;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(acc));
    asm("{\n.reg .f16 lo, hi, pp;\nmov.b32 {lo, hi}, %2;\nmov.b16 pp, %3;\n"
        "fma.rn.f32.f16 %0, lo, pp, %0;\nfma.rn.f32.f16 %1, hi, pp, %1;\n}"
        : "+f"(a), "+f"(b)
        : "r"(h), "h"(p16));
    asm("mov.b64 %0, {%1,%2};" : "=l"(acc) : "f"(a), "f"(b));
}
__device__ __forceinline__ uint16_t f2h(float x) {
    uint16_t h;
    asm("cvt.rn.f16.f32 %0, %1;" : "=h"(h) : "f"(x));
    return h;
}
__device__ __forceinline__ float h2f(uint16_t h) {
    float x;
    asm("cvt.f32.f16 %0, %1;" : "=f"(x) : "h"(h));
    return x;
}

// acc.xy += p * c.xy  (one FFMA2 with a broadcast scalar)
__device__ __forceinline__ void ffma2(unsigned long long &acc, float p, unsigned long long c) {
    unsigned long long pp;
    asm("mov.b64 %0, {%1,%1};" : "=l"(pp) : "f"(p));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(pp), "l"(c));
}

__device__ __forceinline__ void fmul2(unsigned long long &acc, float f) {
    unsigned long long ff;
    asm("mov.b64 %0, {%1,%1};" : "=l"(ff) : "f"(f));
    asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(ff));
}

__device__ __forceinline__ float2 unpack2(unsigned long long v) {
    float2 r;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}

// PRMT selector for rotated byte j: [offset byte (j&1) of b, code byte (j&3)
// of a, byte 2 of b, byte 3 of b]
__device__ __forceinline__ constexpr uint32_t sel_for(int j) {
    return (uint32_t)(4 + (j & 1)) | ((uint32_t)(j & 3) << 4) | (6u << 8) | (7u << 12);
}

// ---- TMA bulk copy (global -> shared) completing on an mbarrier ------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes,
                                         uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(dst), "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar), "r"(phase)
        : "memory");
}

// One unit = 16 tokens [16u, 16u + 16) of a head: lane slot s takes tokens
// 16u + s (A) and 16u + 8 + s (B), one 128-bit K load and one V load each.
// The codes are in the decode layout (common.cuh), so the lane uses its bytes
// in register order.
#if PQKV_LANE8
using CodeVec = uint2;  // a lane's 8 code bytes of one token
__device__ __forceinline__ CodeVec ld_codes(const uint8_t *p) { return ld_stream8(p); }
__device__ __forceinline__ uint32_t cword(const uint2 v, int k) { return k == 0 ? v.x : v.y; }
#else
using CodeVec = uint4;  // a lane's 16 code bytes of one token
__device__ __forceinline__ CodeVec ld_codes(const uint8_t *p) { return ld_stream(p); }
__device__ __forceinline__ uint32_t cword(const uint4 v, int k) {
    return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
}
#endif
struct Unit {
    CodeVec ka, va, kb, vb;
};

// the same from a running pointer p = (K code row of token t) and the
// constant V - K base distance: no address arithmetic beyond an immediate
__device__ __forceinline__ void load_keys_at(Unit &U, const uint8_t *p, int t, int lo, int hi) {
    if (t >= lo && t < hi) U.ka = ld_codes(p);
    if (t + TS >= lo && t + TS < hi) U.kb = ld_codes(p + TS * M);
}
__device__ __forceinline__ void load_values_at(Unit &U, const uint8_t *p, int t, int lo, int hi) {
    if (t >= lo && t < hi) U.va = ld_codes(p);
    if (t + TS >= lo && t + TS < hi) U.vb = ld_codes(p + TS * M);
}
__device__ __forceinline__ void load_unit(Unit &U, const uint8_t *kbase, const uint8_t *vbase,
                                          int u, int slot, int lo, int hi) {
    const int ta = u * UT + slot, tb = ta + TS;
    if (ta >= lo && ta < hi) {
        U.ka = ld_codes(kbase + (int64_t)ta * M);
        U.va = ld_codes(vbase + (int64_t)ta * M);
    }
    if (tb >= lo && tb < hi) {
        U.kb = ld_codes(kbase + (int64_t)tb * M);
        U.vb = ld_codes(vbase + (int64_t)tb * M);
    }
}

// Online-softmax state of one token slot for the HG query heads a CTA serves
// (HG = 2: two query heads of one KV head share every value gather).
template <int HG>
struct SlotState {
    float m[HG], l[HG];
    unsigned long long acc[HG][SPL];  // float2 per (rotated) subspace of this lane's share
};

// sp0 += lo half of h2, sp1 += hi half (mixed f32 + f16 adds: FHADD)
__device__ __forceinline__ void fhadd2(float &sp0, float &sp1, uint32_t h2) {
    asm("{\n.reg .f16 lo, hi;\nmov.b32 {lo, hi}, %2;\n"
        "add.rn.f32.f16 %0, lo, %0;\nadd.rn.f32.f16 %1, hi, %1;\n}"
        : "+f"(sp0), "+f"(sp1)
        : "r"(h2));
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(0x400));
    return v;
}

// kHalfLut (HG = 2): the two heads' tables are one half2 table, entry (c, i) =
// (head 0, head 1) in fp16 -- one 4-byte gather per code byte for both heads
template <int HG, bool kHalfLut = false>
__device__ __forceinline__ void lut_score(const CodeVec k, const uint32_t (&packK)[NPK],
                                          float (&out)[HG]) {
    float sp[HG][4];
#pragma unroll
    for (int j = 0; j < SPL; ++j) {
        const uint32_t a = __byte_perm(cword(k, j >> 2), packK[j >> 1], sel_for(j));
        if constexpr (kHalfLut) {
            static_assert(HG == 2, "the packed table holds two heads");
            const uint32_t x = lds_u32(a);
            if (j < 4) sp[0][j] = sp[1][j] = 0.f;
            fhadd2(sp[0][j & 3], sp[1][j & 3], x);
        } else {
#pragma unroll
            for (int h = 0; h < HG; ++h) {
                const float x = h == 0 ? lds_f32<0x400>(a) : lds_f32<0x10400>(a);
                if (j < 4)
                    sp[h][j] = x;
                else
                    sp[h][j & 3] += x;
            }
        }
    }
#pragma unroll
    for (int h = 0; h < HG; ++h) out[h] = (sp[h][0] + sp[h][1]) + (sp[h][2] + sp[h][3]);
}

// NU units (2 NU tokens per lane) in one pass: all key gathers first, one
// running-max update per head, then all value gathers -- more independent
// work per phase for the latency-bound warp.  Masked tokens (outside the
// segment) take p = 0 without a branch (a branch in the loop body makes the
// compiler drain the ring's pending loads); only the rare running-max
// increase branches.
// after_keys() runs once the key codes are consumed (the ring refills the key
// registers there, half a unit earlier than the value registers).
template <bool kHalfCV, int NU, int HG, bool kHalfLut, typename AfterKeys>
__device__ __forceinline__ void process_units(const Unit *U, SlotState<HG> &S,
                                              const uint32_t (&packK)[NPK],
                                              const uint32_t (&packV)[NPK], const bool *okA,
                                              const bool *okB, AfterKeys after_keys) {
    float sa[NU][HG], sb[NU][HG];
#pragma unroll
    for (int n = 0; n < NU; ++n) {
        lut_score<HG, kHalfLut>(U[n].ka, packK, sa[n]);
        lut_score<HG, kHalfLut>(U[n].kb, packK, sb[n]);
    }
#pragma unroll
    for (int off = 1; off < TL; off <<= 1)  // the TL lanes of a token
#pragma unroll
        for (int n = 0; n < NU; ++n)
#pragma unroll
            for (int h = 0; h < HG; ++h) {
                sa[n][h] += __shfl_xor_sync(0xffffffffu, sa[n][h], off);
                sb[n][h] += __shfl_xor_sync(0xffffffffu, sb[n][h], off);
            }
    after_keys();
    float pa[NU][HG], pb[NU][HG];
    uint16_t pa16[NU][HG], pb16[NU][HG];
#pragma unroll
    for (int h = 0; h < HG; ++h) {
        float mx = -INFINITY;
#pragma unroll
        for (int n = 0; n < NU; ++n)
            mx = fmaxf(mx, fmaxf(okA[n] ? sa[n][h] : -INFINITY, okB[n] ? sb[n][h] : -INFINITY));
        if (mx > S.m[h] + kLazyRescale * kLn2) {
            const float f = fast_exp2((S.m[h] - mx) * kLog2e);
            S.l[h] *= f;
#pragma unroll
            for (int k = 0; k < SPL; ++k) fmul2(S.acc[h][k], f);
            S.m[h] = mx;
        }
#pragma unroll
        for (int n = 0; n < NU; ++n) {
            pa[n][h] = okA[n] ? fast_exp2((sa[n][h] - S.m[h]) * kLog2e) : 0.f;
            pb[n][h] = okB[n] ? fast_exp2((sb[n][h] - S.m[h]) * kLog2e) : 0.f;
            if (kHalfCV) {  // fp16 weights for the mixed-precision FMAs; l sums the same
                pa16[n][h] = f2h(pa[n][h]);
                pb16[n][h] = f2h(pb[n][h]);
                pa[n][h] = h2f(pa16[n][h]);
                pb[n][h] = h2f(pb16[n][h]);
            }
            S.l[h] += pa[n][h] + pb[n][h];
        }
    }
#pragma unroll
    for (int n = 0; n < NU; ++n) {
#pragma unroll
        for (int j = 0; j < SPL; ++j) {
            const uint32_t wa = cword(U[n].va, j >> 2), wb = cword(U[n].vb, j >> 2);
            if (kHalfCV) {  // 4-byte gathers, shared by the HG heads
                const uint32_t ca = lds_cv32<HG>(__byte_perm(wa, packV[j >> 1], sel_for(j)));
                const uint32_t cb = lds_cv32<HG>(__byte_perm(wb, packV[j >> 1], sel_for(j)));
#pragma unroll
                for (int h = 0; h < HG; ++h) {
                    fhfma2(S.acc[h][j], pa16[n][h], ca);
                    fhfma2(S.acc[h][j], pb16[n][h], cb);
                }
            } else {
                const unsigned long long ca =
                    lds_cv<HG>(__byte_perm(wa, packV[j >> 1], sel_for(j)));
                const unsigned long long cb =
                    lds_cv<HG>(__byte_perm(wb, packV[j >> 1], sel_for(j)));
#pragma unroll
                for (int h = 0; h < HG; ++h) {
                    ffma2(S.acc[h][j], pa[n][h], ca);
                    ffma2(S.acc[h][j], pb[n][h], cb);
                }
            }
        }
    }
}

// Dense partial of the recent rows + current token (dense_partial,
// attention.py:169-190), per warp: warp w takes rows w, w + 16, ... with its
// own online softmax; the 16 states are merged after the next barrier.  Out
// of line, so the hot loop's register allocation is not shaped by it.
__device__ __noinline__ void dense_warp_state(const float *q, float scale, const float *recent_k,
                                              const float *recent_v, int64_t ld_recent,
                                              const int32_t *n_recent, const float *k_cur,
                                              const float *v_cur, int Hkv, int bh, int b, int hkv,
                                              int warp, int nwarps, int lane, float *dn_m,
                                              float *dn_l, float (*dn_acc)[D]) {
    const int nr = (n_recent != nullptr && recent_k != nullptr) ? max(n_recent[b], 0) : 0;
    const int rows = nr + (k_cur != nullptr ? 1 : 0);
    const float4 qv = __ldg(reinterpret_cast<const float4 *>(q + (int64_t)bh * D) + lane);
    const int64_t rbase = ((int64_t)b * Hkv + hkv) * ld_recent * D;
    const int64_t cbase = ((int64_t)b * Hkv + hkv) * D;
    float dm = -INFINITY, dl = 0.f;
    float4 da = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int rr = warp; rr < rows; rr += nwarps) {
        const float *kr = rr < nr ? recent_k + rbase + (int64_t)rr * D : k_cur + cbase;
        const float *vr = rr < nr ? recent_v + rbase + (int64_t)rr * D : v_cur + cbase;
        const float4 kk = __ldg(reinterpret_cast<const float4 *>(kr) + lane);
        const float4 vv = __ldg(reinterpret_cast<const float4 *>(vr) + lane);
        float sdot = qv.x * kk.x + qv.y * kk.y + qv.z * kk.z + qv.w * kk.w;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, off);
        const float sc = scale * sdot;
        const float mn = fmaxf(dm, sc);
        const float f = expf(dm - mn), p = expf(sc - mn);
        dl = dl * f + p;
        da.x = da.x * f + p * vv.x;
        da.y = da.y * f + p * vv.y;
        da.z = da.z * f + p * vv.z;
        da.w = da.w * f + p * vv.w;
        dm = mn;
    }
    if (lane == 0) {
        dn_m[warp] = dm;
        dn_l[warp] = dl;
    }
    reinterpret_cast<float4 *>(dn_acc[warp])[lane] = da;
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// merge_partials (attention.py:193-204) of record (mb, lb, ab) into (m, l, acc);
// identity on lb == 0
__device__ __forceinline__ void merge1(float &m, float &l, float &acc, float mb, float lb,
                                       float ab) {
    if (lb == 0.f) return;
    if (l == 0.f) {
        m = mb;
        l = lb;
        acc = ab;
        return;
    }
    const float mm = fmaxf(m, mb);
    const float wa = expf(m - mm), wb = expf(mb - mm);
    l = l * wa + lb * wb;
    acc = acc * wa + ab * wb;
    m = mm;
}

// The last CTA to finish head bh (arrival counter) merges the head's split
// records in CTA order (deterministic), then its dense record, and finalizes
// (merge_partials :193-204, finalize :207-211).  Threads tid < D, one output
// dimension each.  Out of line: runs once per head.
// Records of (split c, virtual head vh, head h of HG) live at HG (c + vh) + h;
// bh is the query head (dense record dense_base + bh, outputs row bh).  With
// a shared code stream (Args::share = P) c and vh count CTA groups and
// virtual-head groups, and member `half` of the group is at
// HG ((c + vh) P + half) + h.
// PQKV_DECODE_APPEND_RECENT: after the merge, the finishing CTA's D threads
// write (k_cur, v_cur) at row n_recent of the ring and bump n_recent (every
// CTA of the head has arrived, so every read of the old length is done)
__device__ __noinline__ void ring_append(const float *k_cur, const float *v_cur, float *rk,
                                         float *rv, int32_t *n_recent, int64_t ld_recent,
                                         int gt, int bar) {
    const int r = __ldcg(n_recent);
    const bool fits = r < ld_recent;
    if (fits) {
        rk[(int64_t)r * D + gt] = __ldg(k_cur + gt);
        rv[(int64_t)r * D + gt] = __ldg(v_cur + gt);
    }
    named_bar_sync(bar, D);  // all D threads have read the old length
    if (gt == 0 && fits) n_recent[0] = r + 1;
}

#ifndef PQKV_FINISH_BATCH
#define PQKV_FINISH_BATCH 8
#endif
__device__ __noinline__ void finish_head(const float *parts, int64_t dense_base, int hg, int vh,
                                         int h, int bh, int c_first, int c_last, int tid,
                                         float *out, float *lse, float *merged, int P, int half) {
    const float *drec = parts + (dense_base + bh) * (D + kPS);
    // the dense record and the first batch are in flight before any is consumed
    const float dm = __ldcg(drec), dl = __ldcg(drec + 1), da = __ldcg(drec + kPS + tid);
    float m = -INFINITY, l = 0.f, acc = 0.f;
    constexpr int FB = PQKV_FINISH_BATCH;  // records in flight per round trip
    for (int c0 = c_first; c0 <= c_last; c0 += FB) {
        const int cnt = min(FB, c_last - c0 + 1);
        float rm[FB], rl[FB], ra[FB];
#pragma unroll
        for (int k = 0; k < FB; ++k) {
            if (k < cnt) {
                const float *rec =
                    parts + ((int64_t)hg * ((int64_t)(c0 + k + vh) * P + half) + h) * (D + kPS);
                rm[k] = __ldcg(rec);
                rl[k] = __ldcg(rec + 1);
                ra[k] = __ldcg(rec + kPS + tid);
            }
        }
#pragma unroll
        for (int k = 0; k < FB; ++k)
            if (k < cnt) merge1(m, l, acc, rm[k], rl[k], ra[k]);
    }
    merge1(m, l, acc, dm, dl, da);
    const float inv = (l > 0.f) ? 1.f / l : NAN;
    if (out) out[(int64_t)bh * D + tid] = acc * inv;
    if (merged) merged[(int64_t)bh * (D + kPS) + kPS + tid] = acc;
    if (tid == 0) {
        if (lse) lse[bh] = (l > 0.f) ? m + logf(l) : -INFINITY;
        if (merged) {
            float *rec = merged + (int64_t)bh * (D + kPS);
            rec[0] = m;
            rec[1] = l;
            rec[2] = 0.f;
            rec[3] = 0.f;
        }
    }
}

// build_key_lut (attention.py:70-83) into shared memory, centroid-major:
// lut[c][i] = scale * (q[2i] C[c][i].x + q[2i+1] C[c][i].y); thread tid owns
// subspaces 2(tid & 31), +1 of centroids tid / 32 + 16k (cc = its codebook slice)
// The key codebook layout is [256][32] float4 (two subspaces per float4);
// thread tid owns float4 slots f = tid + k * NT, i.e. subspaces 2(tid & 31),
// +1 (NT is a multiple of 32) of centroid f / 32.
constexpr int kLutSlots = KSUB * M / 2;  // 8192 float4 of the [256][64] float2 codebook
template <int NT>
constexpr int lut_iters() { return (kLutSlots + NT - 1) / NT; }
template <int NT>
__device__ __forceinline__ void lut_load(float4 (&cc)[lut_iters<NT>()], const float *ck, int tid) {
    constexpr int kLutIters = lut_iters<NT>();
    const float4 *src = reinterpret_cast<const float4 *>(ck);
#pragma unroll
    for (int k = 0; k < kLutIters; ++k)
        if (kLutSlots % NT == 0 || tid + k * NT < kLutSlots) cc[k] = __ldg(src + tid + k * NT);
}
template <int NT>
__device__ __forceinline__ void lut_build(float *lut_s, const float4 (&cc)[lut_iters<NT>()],
                                          const float *qh, float scale, int tid) {
    constexpr int kLutIters = lut_iters<NT>();
    const float4 qq = __ldg(reinterpret_cast<const float4 *>(qh) + (tid & 31));
#pragma unroll
    for (int k = 0; k < kLutIters; ++k) {
        if (kLutSlots % NT != 0 && tid + k * NT >= kLutSlots) break;
        float2 o;
        o.x = scale * fmaf(qq.y, cc[k].y, qq.x * cc[k].x);
        o.y = scale * fmaf(qq.w, cc[k].w, qq.z * cc[k].z);
        reinterpret_cast<float2 *>(lut_s)[tid + k * NT] = o;
    }
}

// the two heads' tables as one half2 table (kHalfLut): entry (c, i) = (head 0,
// head 1) rounded to fp16, the same 4-byte slots as one fp32 table
template <int NT>
__device__ __forceinline__ void lut_build_packed(uint32_t *lut_s, const float4 (&cc)[lut_iters<NT>()],
                                                 const float *q0, const float *q1, float scale,
                                                 int tid) {
    constexpr int kLutIters = lut_iters<NT>();
    const float4 qa = __ldg(reinterpret_cast<const float4 *>(q0) + (tid & 31));
    const float4 qb = __ldg(reinterpret_cast<const float4 *>(q1) + (tid & 31));
#pragma unroll
    for (int k = 0; k < kLutIters; ++k) {
        if (kLutSlots % NT != 0 && tid + k * NT >= kLutSlots) break;
        const float a0 = scale * fmaf(qa.y, cc[k].y, qa.x * cc[k].x);
        const float a1 = scale * fmaf(qa.w, cc[k].w, qa.z * cc[k].z);
        const float b0 = scale * fmaf(qb.y, cc[k].y, qb.x * cc[k].x);
        const float b1 = scale * fmaf(qb.w, cc[k].w, qb.z * cc[k].z);
        uint2 o;
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(o.x) : "f"(b0), "f"(a0));  // lo = head 0
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(o.y) : "f"(b1), "f"(a1));
        reinterpret_cast<uint2 *>(lut_s)[tid + k * NT] = o;
    }
}

// kLutFromQ: build each head's LUT in shared memory from q and the
// centroid-major key codebook ([256][64] float2, pqkv_prepare_key_codebook);
// otherwise copy a precomputed [B*Hq][256][64] LUT (the Lut-taking API).
// HG = 2 (fp16 value codebook, even GQA group): a CTA serves two query heads
// of one KV head -- a "virtual head" -- with two key tables (one PRMT per
// code byte feeds both) and one value gather per code shared by both heads.
// W warps per CTA.
template <bool kLutFromQ, bool kHalfCV, int HG, int W, int GROUP, bool kHalfLut = false>
__global__ void __launch_bounds__(W * 32, 1) decode_partials_m64b8(const Args A) {
    static_assert(RING % GROUP == 0, "the ring holds whole groups");
    static_assert(!kHalfLut || (HG == 2 && kHalfCV && kLutFromQ),
                  "packed fp16 key tables: two heads per CTA in the fp16 mode");
    static_assert(HG == 1 || (HG == 2 && kHalfCV && kLutFromQ), "two heads need the fp16 codebook");
    static_assert(W <= PQKV_WARPS_MAX, "the shared-memory map is sized for PQKV_WARPS_MAX warps");
    constexpr int WARPS = W, NT = W * 32, NG = NT / 128;
    constexpr int kCvBytes = kHalfCV ? CV_BYTES / 2 : CV_BYTES;
    constexpr int kCvOff = HG * LUT_BYTES;  // value codebook after the key tables
    const int Hqv = A.Hq / HG;              // virtual heads per sequence

    extern __shared__ __align__(128) unsigned char smem[];
#ifdef PQKV_TRACE
    unsigned smid_;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid_));
    PQKV_TR(0, smid_);
    PQKV_TR(1, gtime());
    int nseg_ = 0;
#endif
    float *lut_s = reinterpret_cast<float *>(smem);
    float *red_m = reinterpret_cast<float *>(smem + OFF_RED);
    float *red_l = red_m + 2 * WARPS;  // [HG][WARPS] each
    float(*colsum)[D] = reinterpret_cast<float(*)[D]>(smem + OFF_COL);
    float *dn_m = reinterpret_cast<float *>(smem + OFF_DNS);
    float *dn_l = dn_m + WARPS;
    float(*dn_acc)[D] = reinterpret_cast<float(*)[D]>(dn_l + WARPS);
    int *flag_s = reinterpret_cast<int *>(smem + OFF_FLAG);
    int *nq_s = reinterpret_cast<int *>(smem + OFF_NQ);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
    if ((sbase & 0xFFFFFFu) != kDynBase) __trap();  // layout assumption (see lds_f32)
    const uint32_t cta_byte = sbase & 0xFF000000u;
    const uint32_t bar_cv = sbase + OFF_BAR;
    const uint32_t bar_lut = sbase + OFF_BAR + 8;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int part = lane % TL, slot = lane / TL;  // SPL-subspace share, token slot
    // unit order of the warps, reversed: a segment's partial last round of
    // units goes to the high warps, which the issue arbiter favours (they end
    // their units ~0.5 us before warps 0-3, profiles/r02_step_timeline.txt)
    const int wu = WARPS - 1 - warp;

    // value codebook: one TMA bulk copy per CTA, overlapped with the first
    // segment's code prefetch and LUT build -- and, when the codebook is static
    // (early_cv), with the previous kernel's tail (PDL)
    if (tid == 0) {
        mbar_init(bar_cv, 1);
        mbar_init(bar_lut, 1);
        if (A.early_cv) {
            mbar_expect_tx(bar_cv, kCvBytes);
#pragma unroll
            for (int c = 0; c < kCvBytes / 16384; ++c)
                bulk_g2s(sbase + kCvOff + c * 16384,
                         reinterpret_cast<const char *>(A.cv) + c * 16384,
                         16384, bar_cv);
        }
    }
    // (the key codebook slice is NOT preloaded into registers before the wait:
    // 64 live registers across it spill the main loop -- measured)
    const int cta = blockIdx.x;
    const int group = A.Hq / A.Hkv;
    // shared code stream: the cost map runs over CTA groups and virtual-head
    // groups of P; member `half` of a CTA group serves member `half` of each
    // virtual-head group it holds
    const int P = A.share > 1 ? A.share : 1;
    const int pc = cta / P, half = cta - pc * P, Hqp = Hqv / P;
    auto vhead = [&](int ph) {
        const int bb = ph / Hqp;
        return bb * Hqv + (ph - bb * Hqp) * P + half;
    };
    // The first segment's code ring.  With early_codes (n_q and the codes
    // below it were written before the previous kernel on the stream started)
    // the cost map and these loads are issued before the grid-dependency wait;
    // otherwise right after it, ahead of the table build, so the ring's DRAM
    // latency overlaps the build.
    Unit Ur[RING];
#pragma unroll
    for (int rr = 0; rr < RING; ++rr) Ur[rr].ka = Ur[rr].va = Ur[rr].kb = Ur[rr].vb = CodeVec{};
    CostMap cm;
    Segment s0;
    bool have_s0 = false;
    int64_t pos = 0, end = 0;
    // the lengths are read from global memory once, here; the segment walks
    // below (after a barrier) use the shared-memory copy
    const bool nq_cached = A.B <= kNqCache;
    // early_codes needs the shared-memory copy of n_q to re-validate it
    const bool early = A.early_codes && nq_cached;
    auto first_ring = [&]() {
        // one snapshot of the lengths: every later walk reads nq_s
        const int32_t *src = A.n_q;
        if (nq_cached) {
            for (int bb = tid; bb < A.B; bb += NT) nq_s[bb] = __ldcg(A.n_q + bb);
            __syncthreads();
            src = nq_s;
        }
        cm = cost_map(src, A.B, Hqp, A.num_ctas / P, P);
        pos = cta_begin(cm, pc);
        end = min(cta_begin(cm, pc + 1), cm.total);
        int64_t p0 = pos;
        have_s0 = next_segment(src, A.B, Hqp, &p0, end, &s0);
        if (have_s0) {
            const int vh0 = vhead(s0.bh);
            const int b = vh0 / Hqv, hkv = (vh0 - b * Hqv) * HG / group;
            const int64_t head_off = ((int64_t)b * A.Hkv + hkv) * A.ld_tok * M;
            const int u0 = s0.lo / UT;
#pragma unroll
            for (int rr = 0; rr < RING; ++rr)
                load_unit(Ur[rr], A.codes_k + head_off + part * SPL,
                          A.codes_v + head_off + part * SPL, u0 + wu + rr * WARPS, slot, s0.lo,
                          s0.hi);
        }
    };
    int *stale_s = flag_s + (WMAX / 4);  // 1: the pre-wait n_q was stale
    if (early) {
        if (tid == 0) *stale_s = 0;
        first_ring();
    }
    pdl_launch_dependents();
    pdl_wait();  // q, n_q, recent rows, counters and partials belong to the stream order
#ifdef PQKV_TRACE
    PQKV_TR(7, gtime());
    const long long clk_pw_ = clock64();
#endif
    // early: the lengths read before the wait may predate the previous kernel
    // (e.g. a publication's n_q.fill_ right before this launch).  Re-read them
    // now -- the load overlaps the first table build -- and, if any changed,
    // redo the work split and the first ring from the fresh values (below).
    int nq_fresh = 0;
    if (early && tid < A.B) nq_fresh = __ldcg(A.n_q + tid);
    if (!early) first_ring();
#ifdef PQKV_TRACE
    PQKV_TRC(10);  // cost map read, first ring issued
#endif
    if (tid == 0 && !A.early_cv) {
        mbar_expect_tx(bar_cv, kCvBytes);
#pragma unroll
        for (int c = 0; c < kCvBytes / 16384; ++c)
            bulk_g2s(sbase + kCvOff + c * 16384,
                     reinterpret_cast<const char *>(A.cv) + c * 16384,
                     16384, bar_cv);
    }

    // lane-constant address bytes (see header comment)
    uint32_t packK[NPK], packV[NPK];
    const int vhalf = decode_lane_subspace(lane, 0) >> 5;  // this lane's subspace half
#pragma unroll
    for (int jp = 0; jp < NPK; ++jp) {
        uint32_t pk = 0, pv = 0;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int j = 2 * jp + e;
            const int i = decode_lane_subspace(lane, j);
            pk |= (uint32_t)(i * 4) << (8 * e);
            // fp32: [half][c][32] float2 -> half << 16 | code << 8 | slot * 8;
            // fp16: [c][half][32] half2 -> code << 8 | half << 7 | slot * 4
            pv |= (uint32_t)(kHalfCV ? vhalf * 128 + (i & 31) * 4 : (i & 31) * 8) << (8 * e);
        }
        packK[jp] = pk | cta_byte;
        packV[jp] = pv | (kHalfCV ? 0u : (uint32_t)vhalf << 16) | cta_byte;
    }

    bool cv_ready = false;
    uint32_t lut_phase = 0;

    const int32_t *nq = nq_cached ? nq_s : A.n_q;
    bool ring_loaded = have_s0;  // the first segment's ring is in flight
    Segment sg;
    // early launches: the first segment's barrier (or, for a CTA without
    // segments, the check after the loop) compares the pre-wait lengths with
    // nq_fresh; on a mismatch the CTA restarts from the fresh lengths
    bool validate = early;
    auto restart = [&]() {
        __syncthreads();  // every thread has read the flag
        if (tid < A.B) nq_s[tid] = nq_fresh;
        if (tid == 0) *stale_s = 0;
        __syncthreads();
        cm = cost_map(nq_s, A.B, Hqp, A.num_ctas / P, P);
        pos = cta_begin(cm, pc);
        end = min(cta_begin(cm, pc + 1), cm.total);
        ring_loaded = false;
    };
    bool stale_now = false;
  segments:
    while (next_segment(nq, A.B, Hqp, &pos, end, &sg)) {
        const int vh = vhead(sg.bh);  // virtual head: query heads hq0 .. hq0 + HG - 1
        const int b = vh / Hqv, hq0 = (vh - b * Hqv) * HG, hkv = hq0 / group;
        const int bh0 = b * A.Hq + hq0;
        const int64_t head_off = ((int64_t)b * A.Hkv + hkv) * A.ld_tok * M;
        const uint8_t *kbase = A.codes_k + head_off + part * SPL;
        const uint8_t *vbase = A.codes_v + head_off + part * SPL;
        const int lo = sg.lo, hi = sg.hi;             // token range of this segment
        const int u0 = lo / UT, u1 = (hi + UT - 1) / UT;  // UT-token units (absolute)

        // code prefetch: these loads fly while the LUT is built
        if (!ring_loaded) {
#pragma unroll
            for (int rr = 0; rr < RING; ++rr)
                load_unit(Ur[rr], kbase, vbase, u0 + wu + rr * WARPS, slot, lo, hi);
        }
        ring_loaded = false;
#ifdef PQKV_TRACE
        if (nseg_ == 0) PQKV_TRC(11);  // ring loads issued
#endif

        __syncthreads();  // previous segment's epilogue is done with lut_s
#ifdef PQKV_TRACE
        if (nseg_ == 0) PQKV_TRC(12);
#endif
        if (kLutFromQ) {
            float4 cc[lut_iters<NT>()];
            lut_load<NT>(cc, A.ck, tid);
            if constexpr (kHalfLut) {
                lut_build_packed<NT>(reinterpret_cast<uint32_t *>(lut_s), cc,
                                     A.q + (int64_t)bh0 * D, A.q + (int64_t)(bh0 + 1) * D,
                                     A.scale, tid);
            } else {
#pragma unroll
                for (int h = 0; h < HG; ++h)
                    lut_build<NT>(lut_s + h * (LUT_BYTES / 4), cc, A.q + (int64_t)(bh0 + h) * D,
                                  A.scale, tid);
            }
#ifdef PQKV_TRACE
            if (nseg_ == 0) PQKV_TRC(8);  // first table built
#endif
        } else if (tid == 0) {
            mbar_expect_tx(bar_lut, LUT_BYTES);
#pragma unroll
            for (int c = 0; c < LUT_BYTES / 16384; ++c)
                bulk_g2s(sbase + c * 16384,
                         reinterpret_cast<const char *>(A.lut + (int64_t)bh0 * KSUB * M) + c * 16384,
                         16384, bar_lut);
        }
        if (validate && tid < A.B && nq_fresh != nq_s[tid]) *stale_s = 1;  // read after the
                                                                            // barrier below
        // dense partial by the CTA holding the head's last tokens (for most CTAs
        // their first segment, so it overlaps the prologue)
#ifndef PQKV_NO_DENSE
        const bool do_dense = A.counters != nullptr && sg.last;
#else
        const bool do_dense = false;
#endif
        const int64_t dense_base = (int64_t)HG * A.num_ctas + (int64_t)A.B * A.Hq;
#pragma unroll
        for (int h = 0; h < HG; ++h) {
            if (h > 0) __syncthreads();  // the previous head's merge has read dn_*
            if (do_dense)
                dense_warp_state(A.q, A.scale, A.recent_k, A.recent_v, A.ld_recent, A.n_recent,
                                 A.k_cur, A.v_cur, A.Hkv, bh0 + h, b, hkv, warp, WARPS, lane, dn_m,
                                 dn_l, dn_acc);
#ifdef PQKV_TRACE
            if (nseg_ == 0) PQKV_TRC(13);
#endif
            if (h == 0) {
                if (!kLutFromQ) {
                    mbar_wait(bar_lut, lut_phase);
                    lut_phase ^= 1u;
                }
                if (!cv_ready) {
                    mbar_wait(bar_cv, 0);
                    cv_ready = true;
#ifdef PQKV_TRACE
                    PQKV_TRC(9);  // value codebook arrived
#endif
                }
            }
            __syncthreads();
#ifdef PQKV_TRACE
            if (nseg_ == 0) {
                PQKV_TR(2, gtime());
                PQKV_TRC(16);  // main loop starts
            }
#endif
            if (h == 0 && validate) {
                validate = false;
                stale_now = *stale_s != 0;
                if (stale_now) break;  // rare: restart from the fresh lengths (below)
            }
            if (do_dense && tid < D) {
                // merge the warps' dense states into record dense_base + bh0 + h
                float Mx = -INFINITY;
#pragma unroll
                for (int w = 0; w < WARPS; ++w)
                    if (dn_l[w] > 0.f) Mx = fmaxf(Mx, dn_m[w]);
                float L = 0.f, acc = 0.f;
                if (Mx != -INFINITY) {
#pragma unroll
                    for (int w = 0; w < WARPS; ++w) {
                        if (dn_l[w] > 0.f) {
                            const float f = expf(dn_m[w] - Mx);
                            L += dn_l[w] * f;
                            acc += dn_acc[w][tid] * f;
                        }
                    }
                }
                float *rec = A.parts + (dense_base + bh0 + h) * (D + kPS);
                rec[kPS + tid] = acc;
                if (tid == 0) {
                    rec[0] = Mx;
                    rec[1] = L;
                    rec[2] = 0.f;
                    rec[3] = 0.f;
                }
            }
        }

        if (stale_now) {
            stale_now = false;
            restart();
            continue;
        }
        SlotState<HG> S;
#pragma unroll
        for (int h = 0; h < HG; ++h) {
            S.m[h] = -INFINITY;
            S.l[h] = 0.f;
#pragma unroll
            for (int k = 0; k < 16; ++k) S.acc[h][k] = 0ull;
        }

        // static RING-unit register ring per warp: no register moves, a pending
        // load is only waited for when its unit is processed.  Straight-line
        // steady state: the warp's unit count rounded up to the ring depth,
        // every unit processed masked (units past the segment load nothing and
        // contribute p = 0) -- a branch in the body would make the compiler
        // drain the ring's pending loads.
        int u = u0 + wu;
        const int nunits = max(0, (u1 - u0 - wu + WARPS - 1) / WARPS);
        // running load position: the next unit to load is u + RING * WARPS
        constexpr int64_t kStep = (int64_t)WARPS * UT * M;  // bytes per unit step of a warp
        const int64_t dv = vbase - kbase;
        int tn = (u + RING * WARPS) * UT + slot;
        const uint8_t *kp = kbase + (int64_t)tn * M;
        static_assert(RING == 2, "the remainder below handles one leftover unit");
        for (int trip = 0; trip < nunits / RING; ++trip) {
            // pin the lane-constant address words in registers (no remat)
#pragma unroll
            for (int k = 0; k < NPK; ++k) asm volatile("" : "+r"(packK[k]), "+r"(packV[k]));
#pragma unroll
            for (int g = 0; g < RING / GROUP; ++g) {
                bool okA[GROUP], okB[GROUP];
#pragma unroll
                for (int n = 0; n < GROUP; ++n) {
                    const int ta = (u + n * WARPS) * UT + slot;
                    okA[n] = ta >= lo && ta < hi;
                    okB[n] = ta + TS >= lo && ta + TS < hi;
                }
                if constexpr (!kHalfCV && PQKV_EARLY_KEYS) {
                    // exact path: refill the key registers as soon as the key
                    // phase consumed them (measured +1%; the fp16 variants spill)
                    process_units<kHalfCV, GROUP, HG, kHalfLut>(
                        Ur + g * GROUP, S, packK, packV, okA, okB, [&]() {
#pragma unroll
                            for (int n = 0; n < GROUP; ++n)
                                load_keys_at(Ur[g * GROUP + n], kp + n * kStep,
                                             tn + n * WARPS * UT, lo, hi);
                        });
#pragma unroll
                    for (int n = 0; n < GROUP; ++n)
                        load_values_at(Ur[g * GROUP + n], kp + n * kStep + dv,
                                       tn + n * WARPS * UT, lo, hi);
                } else {
                    process_units<kHalfCV, GROUP, HG, kHalfLut>(Ur + g * GROUP, S, packK, packV, okA, okB,
                                                      []() {});
#pragma unroll
                    for (int n = 0; n < GROUP; ++n) {
                        load_keys_at(Ur[g * GROUP + n], kp + n * kStep, tn + n * WARPS * UT, lo,
                                     hi);
                        load_values_at(Ur[g * GROUP + n], kp + n * kStep + dv,
                                       tn + n * WARPS * UT, lo, hi);
                    }
                }
                u += GROUP * WARPS;
                kp += GROUP * kStep;
                tn += GROUP * WARPS * UT;
            }
        }

        if (nunits % RING) {
            // an odd unit count: the last unit alone (ring slot 0), outside the
            // straight-line body, instead of a masked full group
            bool okA[1], okB[1];
            const int ta = u * UT + slot;
            okA[0] = ta >= lo && ta < hi;
            okB[0] = ta + TS >= lo && ta + TS < hi;
            process_units<kHalfCV, 1, HG, kHalfLut>(Ur, S, packK, packV, okA, okB, []() {});
        }

        // ---- epilogue: one (m, l, acc) record for this (CTA, head) segment
#ifdef PQKV_TRACE
        if (nseg_ == 0 && lane == 0 && blockIdx.x < kTraceCtas)  // per-warp loop end
            g_wtrace[((A.trace_id % kTraceLaunches) * kTraceCtas + blockIdx.x) * 32 + warp] =
                gtime();
        if (nseg_++ == 0) PQKV_TR(3, gtime());
#endif
#pragma unroll
        for (int h = 0; h < HG; ++h) {
            float mw = S.m[h];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
                mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, off));
            if (lane == 0) red_m[h * WARPS + warp] = mw;
        }
        __syncthreads();  // all warps are past the main loop: lut_s is free
        float Mx[HG];
#pragma unroll
        for (int h = 0; h < HG; ++h) {
            Mx[h] = red_m[h * WARPS];
#pragma unroll
            for (int w = 1; w < WARPS; ++w) Mx[h] = fmaxf(Mx[h], red_m[h * WARPS + w]);
            const float f = (S.m[h] == -INFINITY) ? 0.f : fast_exp2((S.m[h] - Mx[h]) * kLog2e);
            float lw = (part == 0) ? S.l[h] * f : 0.f;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) lw += __shfl_xor_sync(0xffffffffu, lw, off);
            if (lane == 0) red_l[h * WARPS + warp] = lw;
            // head h's slot rows: [WARPS * TS][128] fp32 in the (now free) key tables
            float *rows = lut_s + (h * WARPS * TS + warp * TS + slot) * D;
#pragma unroll
            for (int j = 0; j < SPL; ++j) {
                const int i = decode_lane_subspace(lane, j);  // byte j <-> this subspace
                const float2 a = unpack2(S.acc[h][j]);
                rows[2 * i] = a.x * f;
                rows[2 * i + 1] = a.y * f;
            }
        }
        __syncthreads();
        {
            constexpr int RPP = WARPS * TS / NG;  // slot rows per 128-thread part
            const int col = tid & (D - 1), prt = tid >> 7;
#pragma unroll
            for (int h = 0; h < HG; ++h) {
                float cs = 0.f;
                const float *rows = lut_s + h * WARPS * TS * D;
#pragma unroll 8
                for (int rr = prt * RPP; rr < prt * RPP + RPP; ++rr) cs += rows[rr * D + col];
                colsum[h * NG + prt][col] = cs;
            }
        }
        __syncthreads();
        if (tid < D) {
#pragma unroll
            for (int h = 0; h < HG; ++h) {
                float *rec =
                    A.parts + ((int64_t)HG * ((int64_t)(pc + sg.bh) * P + half) + h) * (D + kPS);
                float a = colsum[h * NG][tid];
#pragma unroll
                for (int pp = 1; pp < NG; ++pp) a += colsum[h * NG + pp][tid];
                rec[kPS + tid] = a;
                if (tid == 0) {
                    float L = 0.f;
#pragma unroll
                    for (int w = 0; w < WARPS; ++w) L += red_l[h * WARPS + w];
                    rec[0] = Mx[h];
                    rec[1] = L;
                    rec[2] = 0.f;
                    rec[3] = 0.f;
                }
            }
        }
    }
#ifdef PQKV_TRACE
    PQKV_TR(6, gtime());
    const long long clk_segs = clock64();
#endif
    if (validate) {  // a CTA without segments in the pre-wait split checks here
        validate = false;
        if (tid < A.B && nq_fresh != nq_s[tid]) *stale_s = 1;
        __syncthreads();
        if (*stale_s) {
            restart();
            goto segments;
        }
    }
    // ---- arrivals, after all of this CTA's segments (kept out of the segment
    // loop, whose code generation it would otherwise disturb).  Thread group
    // g = tid / 128 handles segments g, g + 4, ... in parallel: its leader
    // bumps the head's arrival counter, and the last CTA to arrive merges the
    // head's records in CTA order (deterministic), then the dense record, and
    // finalizes.
    if (A.counters != nullptr) {
        __syncthreads();  // every record (and dense record) write of this CTA is done
        const int grp = tid >> 7, gt = tid & (D - 1);
        int64_t p2 = cta_begin(cm, pc);
        Segment s2;
        for (int k = 0; next_segment(nq, A.B, Hqp, &p2, end, &s2); ++k) {
            if (k % NG != grp) continue;
            int c_first, c_last, len;
            head_ctas(nq, Hqp, s2.bh, cm, &c_first, &c_last, &len);
            const int vh2 = vhead(s2.bh);
            if (gt == 0) {
                // acq_rel at gpu scope: releases this CTA's records (ordered
                // before by the barrier, fences are cumulative) and, for the
                // last arriver, acquires every other CTA's
                int old;
                asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;"
                             : "=r"(old)
                             : "l"(A.counters + vh2)
                             : "memory");
                const bool last = (old == c_last - c_first);
                if (last) A.counters[vh2] = 0;  // ready for the next launch
                flag_s[grp] = last ? 1 : 0;
#ifdef PQKV_TRACE
                if (k == 0) PQKV_TR(14, clock64() - clk_segs);  // cycles to the arrival
#endif
            }
            named_bar_sync(1 + grp, D);  // this group's 128 threads
            const bool last = flag_s[grp] != 0;
            named_bar_sync(1 + grp, D);  // flag_s[grp] is read before its reuse
            if (last) {
                const int b2 = vh2 / Hqv, bq0 = b2 * A.Hq + (vh2 - b2 * Hqv) * HG;
#pragma unroll
                for (int h = 0; h < HG; ++h)
                    finish_head(A.parts, (int64_t)HG * A.num_ctas + (int64_t)A.B * A.Hq, HG,
                                s2.bh, h, bq0 + h, c_first, c_last, gt, A.out, A.lse, A.merged,
                                P, half);
                if (A.append)
                    ring_append(A.k_cur, A.v_cur, const_cast<float *>(A.recent_k),
                                const_cast<float *>(A.recent_v), const_cast<int32_t *>(A.n_recent),
                                A.ld_recent, gt, 1 + grp);
#ifdef PQKV_TRACE
                if (k == 0) PQKV_TR(15, clock64() - clk_segs);  // cycles to the merge's end
#endif
            }
        }
    }
    if (!cv_ready) mbar_wait(bar_cv, 0);  // never exit with a bulk copy in flight
#ifdef PQKV_TRACE
    __syncthreads();
    PQKV_TR(4, gtime());
    PQKV_TR(5, nseg_);
#endif
}

// ================================================ GQA: four heads per CTA ==
// decode_gqa4_f16 -- PQKV_DECODE_F16_KEY_TABLE with a GQA group that is a
// multiple of 4 (stated tolerance, as the fp16 value-codebook mode).  One CTA
// serves four query heads of a KV head (a "virtual head"), so every key-code
// gather feeds all four heads' scores and every value-code gather all four
// heads' accumulators -- the per-query-head shared-memory work of the pair
// kernel above (HG = 2, two CTAs per group of four) is shared once more.
//   * shared memory: the four heads' key tables (build_key_lut,
//     attention.py:70-83) as ONE fp16 table of 8-byte entries (h0, h1, h2,
//     h3), laid out [half][256][32] (address half << 16 | code << 8 |
//     (i & 31) << 3, 128 KiB), and the fp16 value codebook [256][2][32] half2
//     (64 KiB, pqkv_prepare_value_codebook_f16);
//   * lane = (slot s, eighth w), 8 lanes per token: the lane's 8 code bytes
//     are bytes [8w, 8w + 8) of token A = 8u + {0,1,4,5}[s] and bytes
//     [8(w^1), 8(w^1) + 8) of token B = A + 2.  On the stored decode layout
//     (common.cuh) B's rotation is A's + 8 and its bytes sit 8 further into the
//     quarter, so both tokens touch the same 8 subspaces at every step (one set
//     of accumulators per lane), and a warp instruction touches 16 distinct
//     subspaces mod 16 per half-warp (8-byte table gathers) and 32 distinct
//     mod 32 (4-byte value gathers): bank-conflict free for ANY code values,
//     with the MHA kernel's stored layout unchanged (scripts/check_gqa4_lanes.py);
//   * the 8 lanes of a token reduce their four partial scores with a
//     transposing butterfly (4 shuffles: lanes 2h, 2h + 1 end with head h's
//     sum), keep head h's online-softmax state there (one max update, 2 NU
//     EX2 per unit group) and shuffle the weights to the token's 8 lanes;
//   * scores in log2 units (the table entries carry log2(e)), so a weight is
//     one FADD + EX2; the records' maxima are converted back to natural units;
//   * value path: the half2 codebook entry is widened to float2 and feeds one
//     FFMA2 per head with the fp32 weight (the pair kernel rounds the weights
//     to fp16; here only the codebook and the table entries are rounded).
#ifndef PQKV_GQA4_PERM
#define PQKV_GQA4_PERM 1
#endif
namespace g4 {
constexpr int HG = 4;
constexpr int UT = 8;                          // tokens per warp per unit
constexpr int TAB_BYTES = 2 * KSUB * 32 * 8;   // 131072: [half][256][32] x 8 B
constexpr int CV16_BYTES = KSUB * 2 * 32 * 4;  // 65536: [256][2][32] half2
constexpr int CV_IMM = 0x400 + TAB_BYTES;      // LDS immediate of the value codebook

__device__ __forceinline__ int tau_a(int s) { return (s & 1) | ((s & 2) << 1); }  // 0 1 4 5

// subspace of byte j of lane (s, w) -- for token A and, identically, token B
__device__ __forceinline__ int lane_subspace(int s, int w, int j) {
    const int q = w >> 1;
    const int r = decode_lane_rot(4 * tau_a(s) + q);
    return 16 * q + ((8 * (w & 1) + j + r) & 15);
}

struct Unit4 {
    uint2 ka, kb, va, vb;
};
struct State4 {
    float m, l;                     // head (w >> 1) & 3 of this lane's token slot (owner lanes)
    unsigned long long acc[HG][8];  // float2 per subspace of this lane, per head
};

__device__ __forceinline__ uint2 ld8(const uint8_t *p) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "=r"(r.x), "=r"(r.y)
                 : "l"(p));
    return r;
}
// refill in place: the destination is tied to the ring register's current
// value ("+r"), so the compiler has no reason to load into a fresh register and
// move it back (a move would wait for the load)
__device__ __forceinline__ void ld8_into(uint2 &r, const uint8_t *p) {
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "+r"(r.x), "+r"(r.y)
                 : "l"(p));
}
__device__ __forceinline__ uint2 lds_tab(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2+%3];" : "=r"(v.x), "=r"(v.y) : "r"(a), "n"(0x400));
    return v;
}
__device__ __forceinline__ uint32_t lds_cv16(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(CV_IMM));
    return v;
}
// half2 -> float2 (packed in a 64-bit register pair for FFMA2)
__device__ __forceinline__ unsigned long long widen(uint32_t h) {
    unsigned long long r;
    asm("{\n.reg .f16 lo, hi;\n.reg .f32 a, b;\nmov.b32 {lo, hi}, %1;\n"
        "cvt.f32.f16 a, lo;\ncvt.f32.f16 b, hi;\nmov.b64 %0, {a, b};\n}"
        : "=l"(r)
        : "r"(h));
    return r;
}

// unit u: tokens [8u, 8u + 8); lane takes A = 8u + tA (bytes 8w..) and B = A + 2
// (bytes 8(w^1)..): B's code row pointer is A's + dB
__device__ __forceinline__ void load_unit4(Unit4 &U, const uint8_t *kbase, const uint8_t *vbase,
                                           int u, int tA, int dB, int lo, int hi) {
    const int ta = u * UT + tA, tb = ta + 2;
    const int64_t o = (int64_t)ta * M;
    if (ta >= lo && ta < hi) {
        U.ka = ld8(kbase + o);
        U.va = ld8(vbase + o);
    }
    if (tb >= lo && tb < hi) {
        U.kb = ld8(kbase + o + dB);
        U.vb = ld8(vbase + o + dB);
    }
}

// four heads' partial scores of one token from this lane's 8 key codes
__device__ __forceinline__ void key_scores(const uint2 k, const uint32_t (&pk)[4],
                                           float (&out)[HG]) {
    float sp[HG][2] = {};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint2 e = lds_tab(__byte_perm(j < 4 ? k.x : k.y, pk[j >> 1], sel_for(j)));
        fhadd2(sp[0][j & 1], sp[1][j & 1], e.x);
        fhadd2(sp[2][j & 1], sp[3][j & 1], e.y);
    }
#pragma unroll
    for (int h = 0; h < HG; ++h) out[h] = sp[h][0] + sp[h][1];
}

// sum v[0..3] over the 8 lanes of a token: the transposing butterfly only --
// lane w returns head (w >> 1) & 3 (lanes w, w ^ 1 hold the same bits).
// PQKV_GQA4_PERM: the table stores subspace i's heads in the order k ^ (i >> 4)
// (tab_build4), and every subspace of lane w has i >> 4 = w >> 1, so v[k] is
// head k ^ (w >> 1): each level keeps v[0..] and sends v[2..] -- no selects.
__device__ __forceinline__ float token_reduce_own(const float (&v)[HG], int w) {
#if PQKV_GQA4_PERM
    (void)w;
    const float k0 = v[0] + __shfl_xor_sync(0xffffffffu, v[2], 4);
    const float k1 = v[1] + __shfl_xor_sync(0xffffffffu, v[3], 4);
    const float k = k0 + __shfl_xor_sync(0xffffffffu, k1, 2);
    return k + __shfl_xor_sync(0xffffffffu, k, 1);
#else
    const bool b4 = (w & 4) != 0, b2 = (w & 2) != 0;
    const float s0 = b4 ? v[0] : v[2], s1 = b4 ? v[1] : v[3];
    float k0 = b4 ? v[2] : v[0], k1 = b4 ? v[3] : v[1];
    k0 += __shfl_xor_sync(0xffffffffu, s0, 4);
    k1 += __shfl_xor_sync(0xffffffffu, s1, 4);
    const float s = b2 ? k0 : k1;
    float k = b2 ? k1 : k0;
    k += __shfl_xor_sync(0xffffffffu, s, 2);
    return k + __shfl_xor_sync(0xffffffffu, k, 1);
#endif
}

// NU units: key phase, then the softmax at the owner lanes (lane w of a token
// holds head (w >> 1) & 3: one running-max update, 2 NU EX2), the weights
// shuffled to the token's 8 lanes, value phase.  Masked tokens take p = 0
// without a branch; only a running-max increase (rare) branches.
template <int NU, typename AfterKeys>
__device__ __forceinline__ void process4(const Unit4 *U, State4 &S, const uint32_t (&pk)[4],
                                         const uint32_t (&pv)[4], const bool *okA,
                                         const bool *okB, int w, AfterKeys after_keys) {
    float sa[NU][HG], sb[NU][HG];
#pragma unroll
    for (int n = 0; n < NU; ++n) {
        key_scores(U[n].ka, pk, sa[n]);
        key_scores(U[n].kb, pk, sb[n]);
    }
    after_keys();
    float oa[NU], ob[NU];
#pragma unroll
    for (int n = 0; n < NU; ++n) {
        oa[n] = token_reduce_own(sa[n], w);
        ob[n] = token_reduce_own(sb[n], w);
    }
    const int base = (threadIdx.x & 31) & ~7;  // lane 0 of this token slot
    {
        float mx = -INFINITY;
#pragma unroll
        for (int n = 0; n < NU; ++n)
            mx = fmaxf(mx, fmaxf(okA[n] ? oa[n] : -INFINITY, okB[n] ? ob[n] : -INFINITY));
        const bool up = mx > S.m + kLazyRescale;
        if (__any_sync(0xffffffffu, up)) {  // rare: rescale the slot's accumulators
            const float f = up ? fast_exp2(S.m - mx) : 1.f;
            if (up) {
                S.l *= f;
                S.m = mx;
            }
#pragma unroll
            for (int h = 0; h < HG; ++h) {
                const float fh = __shfl_sync(0xffffffffu, f, base | (2 * h));
#pragma unroll
                for (int k = 0; k < 8; ++k) fmul2(S.acc[h][k], fh);
            }
        }
    }
    float pa[NU][HG], pb[NU][HG];
#pragma unroll
    for (int n = 0; n < NU; ++n) {
        const float qa = okA[n] ? fast_exp2(oa[n] - S.m) : 0.f;
        const float qb = okB[n] ? fast_exp2(ob[n] - S.m) : 0.f;
        S.l += qa + qb;
#pragma unroll
        for (int h = 0; h < HG; ++h) {
            pa[n][h] = __shfl_sync(0xffffffffu, qa, base | (2 * h));
            pb[n][h] = __shfl_sync(0xffffffffu, qb, base | (2 * h));
        }
    }
#pragma unroll
    for (int n = 0; n < NU; ++n) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t wa = j < 4 ? U[n].va.x : U[n].va.y;
            const uint32_t wb = j < 4 ? U[n].vb.x : U[n].vb.y;
            const unsigned long long ca = widen(lds_cv16(__byte_perm(wa, pv[j >> 1], sel_for(j))));
            const unsigned long long cb = widen(lds_cv16(__byte_perm(wb, pv[j >> 1], sel_for(j))));
#pragma unroll
            for (int h = 0; h < HG; ++h) {
                ffma2(S.acc[h][j], pa[n][h], ca);
                ffma2(S.acc[h][j], pb[n][h], cb);
            }
        }
    }
}

// e[k] <- e[k ^ pq] (pq < 4), with selects (no indexed registers)
__device__ __forceinline__ void perm_heads(float (&e)[HG], int pq) {
    float a0 = e[0], a1 = e[1], a2 = e[2], a3 = e[3];
    if (pq & 1) {
        const float t0 = a0, t2 = a2;
        a0 = a1, a1 = t0, a2 = a3, a3 = t2;
    }
    if (pq & 2) {
        const float t0 = a0, t1 = a1;
        a0 = a2, a1 = a3, a2 = t0, a3 = t1;
    }
    e[0] = a0, e[1] = a1, e[2] = a2, e[3] = a3;
}

// the four heads' tables as one fp16 table: entry (c, i) = (h0, h1, h2, h3);
// slot f = tid + k NT of the [256][32] float4 key codebook layout holds
// subspaces 2(f & 31), +1 of centroid f / 32 -> one 16-byte store
template <int NT>
__device__ __forceinline__ void tab_build4(unsigned char *tab, const float4 (&cc)[lut_iters<NT>()],
                                           const float *q0, float scale, int tid) {
    constexpr int kLutIters = lut_iters<NT>();
    float4 qh[HG];
#pragma unroll
    for (int h = 0; h < HG; ++h) qh[h] = __ldg(reinterpret_cast<const float4 *>(q0 + h * D) + (tid & 31));
#pragma unroll
    for (int k = 0; k < kLutIters; ++k) {
        const int f = tid + k * NT;
        if (kLutSlots % NT != 0 && f >= kLutSlots) break;
        float e0[HG], e1[HG];
#pragma unroll
        for (int h = 0; h < HG; ++h) {
            e0[h] = scale * fmaf(qh[h].y, cc[k].y, qh[h].x * cc[k].x);
            e1[h] = scale * fmaf(qh[h].w, cc[k].w, qh[h].z * cc[k].z);
        }
        const int c = f >> 5, i0 = 2 * (f & 31);
#if PQKV_GQA4_PERM
        const int pq = i0 >> 4;  // entry slot k holds head k ^ (i >> 4) (token_reduce_own)
#else
        const int pq = 0;
#endif
        perm_heads(e0, pq);
        perm_heads(e1, pq);
        uint4 o;
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(o.x) : "f"(e0[1]), "f"(e0[0]));  // lo = slot 0
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(o.y) : "f"(e0[3]), "f"(e0[2]));
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(o.z) : "f"(e1[1]), "f"(e1[0]));
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(o.w) : "f"(e1[3]), "f"(e1[2]));
        *reinterpret_cast<uint4 *>(tab + ((i0 >> 5) << 16) + (c << 8) + ((i0 & 31) << 3)) = o;
    }
}
}  // namespace g4

template <int W>
__global__ void __launch_bounds__(W * 32, 1) decode_gqa4_f16(const Args A) {
    constexpr int HG = g4::HG, UT = g4::UT, TAB_BYTES = g4::TAB_BYTES,
                  CV16_BYTES = g4::CV16_BYTES;
    using g4::tau_a, g4::lane_subspace, g4::Unit4, g4::State4, g4::load_unit4, g4::ld8,
        g4::process4, g4::tab_build4;
    constexpr int NT = W * 32, NG = NT / 128;
    static_assert(NT % 128 == 0, "W must be a multiple of 4");
    static_assert(HG * NG <= 2 * (WMAX / 4), "column sums fit the colsum region");
    static_assert(HG * W * 4 * D * 4 <= TAB_BYTES, "slot rows fit the key table");
    static_assert(2 * HG * W <= 4 * WMAX, "max / sum reductions fit the red region");
    static_assert(TAB_BYTES + CV16_BYTES <= OFF_RED, "tables before the reduction area");
    const int Hqv = A.Hq / HG;  // virtual heads per sequence

    extern __shared__ __align__(128) unsigned char smem[];
    float *rows_s = reinterpret_cast<float *>(smem);  // epilogue: slot rows in the key table
    float *red_m = reinterpret_cast<float *>(smem + OFF_RED);
    float *red_l = red_m + HG * W;
    float(*colsum)[D] = reinterpret_cast<float(*)[D]>(smem + OFF_COL);
    float *dn_m = reinterpret_cast<float *>(smem + OFF_DNS);
    float *dn_l = dn_m + W;
    float(*dn_acc)[D] = reinterpret_cast<float(*)[D]>(dn_l + W);
    int *flag_s = reinterpret_cast<int *>(smem + OFF_FLAG);
    int *nq_s = reinterpret_cast<int *>(smem + OFF_NQ);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
    if ((sbase & 0xFFFFFFu) != kDynBase) __trap();
    const uint32_t cta_byte = sbase & 0xFF000000u;
    const uint32_t bar_cv = sbase + OFF_BAR;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int w = lane & 7, slot = lane >> 3;
    const int tA = tau_a(slot);
    const int dB = 2 * M + 8 * ((w ^ 1) - w);  // token B's code bytes relative to A's
    const int wu = W - 1 - warp;               // unit order (see decode_partials_m64b8)

    if (tid == 0) {
        mbar_init(bar_cv, 1);
        if (A.early_cv) {
            mbar_expect_tx(bar_cv, CV16_BYTES);
#pragma unroll
            for (int c = 0; c < CV16_BYTES / 16384; ++c)
                bulk_g2s(sbase + TAB_BYTES + c * 16384,
                         reinterpret_cast<const char *>(A.cv) + c * 16384, 16384, bar_cv);
        }
    }
    const int cta = blockIdx.x;
    const int group = A.Hq / A.Hkv;
    const int P = A.share > 1 ? A.share : 1;
    const int pc = cta / P, half = cta - pc * P, Hqp = Hqv / P;
    auto vhead = [&](int ph) {
        const int bb = ph / Hqp;
        return bb * Hqv + (ph - bb * Hqp) * P + half;
    };
    Unit4 Ur[2];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) Ur[rr].ka = Ur[rr].kb = Ur[rr].va = Ur[rr].vb = uint2{0u, 0u};
    CostMap cm;
    Segment s0;
    bool have_s0 = false;
    int64_t pos = 0, end = 0;
    const bool nq_cached = A.B <= kNqCache;
    const bool early = A.early_codes && nq_cached;
    auto first_ring = [&]() {
        const int32_t *src = A.n_q;
        if (nq_cached) {
            for (int bb = tid; bb < A.B; bb += NT) nq_s[bb] = __ldcg(A.n_q + bb);
            __syncthreads();
            src = nq_s;
        }
        cm = cost_map(src, A.B, Hqp, A.num_ctas / P, P);
        pos = cta_begin(cm, pc);
        end = min(cta_begin(cm, pc + 1), cm.total);
        int64_t p0 = pos;
        have_s0 = next_segment(src, A.B, Hqp, &p0, end, &s0);
        if (have_s0) {
            const int vh0 = vhead(s0.bh);
            const int b = vh0 / Hqv, hkv = (vh0 - b * Hqv) * HG / group;
            const int64_t head_off = ((int64_t)b * A.Hkv + hkv) * A.ld_tok * M;
            const int u0 = s0.lo / UT;
#pragma unroll
            for (int rr = 0; rr < 2; ++rr)
                load_unit4(Ur[rr], A.codes_k + head_off + 8 * w, A.codes_v + head_off + 8 * w,
                           u0 + wu + rr * W, tA, dB, s0.lo, s0.hi);
        }
    };
    int *stale_s = flag_s + (WMAX / 4);
    if (early) {
        if (tid == 0) *stale_s = 0;
        first_ring();
    }
    pdl_launch_dependents();
    pdl_wait();
    int nq_fresh = 0;
    if (early && tid < A.B) nq_fresh = __ldcg(A.n_q + tid);
    if (!early) first_ring();
    if (tid == 0 && !A.early_cv) {
        mbar_expect_tx(bar_cv, CV16_BYTES);
#pragma unroll
        for (int c = 0; c < CV16_BYTES / 16384; ++c)
            bulk_g2s(sbase + TAB_BYTES + c * 16384, reinterpret_cast<const char *>(A.cv) + c * 16384,
                     16384, bar_cv);
    }

    // lane-constant address bytes: table [half][code][32] x 8 B, value
    // codebook [code][half][32] x 4 B (subspace half = w >> 2 for this lane)
    uint32_t pk[4], pv[4];
    const uint32_t khalf = (uint32_t)(w >> 2);
#pragma unroll
    for (int jp = 0; jp < 4; ++jp) {
        uint32_t a = 0, b = 0;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int i = lane_subspace(slot, w, 2 * jp + e);
            a |= (uint32_t)((i & 31) << 3) << (8 * e);
            b |= (uint32_t)(((i >> 5) << 7) | ((i & 31) << 2)) << (8 * e);
        }
        pk[jp] = a | (khalf << 16) | cta_byte;
        pv[jp] = b | cta_byte;
    }

    bool cv_ready = false;
    const int32_t *nq = nq_cached ? nq_s : A.n_q;
    bool ring_loaded = have_s0;
    Segment sg;
    bool validate = early;
    auto restart = [&]() {
        __syncthreads();
        if (tid < A.B) nq_s[tid] = nq_fresh;
        if (tid == 0) *stale_s = 0;
        __syncthreads();
        cm = cost_map(nq_s, A.B, Hqp, A.num_ctas / P, P);
        pos = cta_begin(cm, pc);
        end = min(cta_begin(cm, pc + 1), cm.total);
        ring_loaded = false;
    };
    bool stale_now = false;
  segments:
    while (next_segment(nq, A.B, Hqp, &pos, end, &sg)) {
        const int vh = vhead(sg.bh);
        const int b = vh / Hqv, hq0 = (vh - b * Hqv) * HG, hkv = hq0 / group;
        const int bh0 = b * A.Hq + hq0;
        const int64_t head_off = ((int64_t)b * A.Hkv + hkv) * A.ld_tok * M;
        const uint8_t *kbase = A.codes_k + head_off + 8 * w;
        const uint8_t *vbase = A.codes_v + head_off + 8 * w;
        const int lo = sg.lo, hi = sg.hi;
        const int u0 = lo / UT, u1 = (hi + UT - 1) / UT;
        if (!ring_loaded) {
#pragma unroll
            for (int rr = 0; rr < 2; ++rr)
                load_unit4(Ur[rr], kbase, vbase, u0 + wu + rr * W, tA, dB, lo, hi);
        }
        ring_loaded = false;

        __syncthreads();  // the previous segment's epilogue is done with the table
        {
            float4 cc[lut_iters<NT>()];
            lut_load<NT>(cc, A.ck, tid);
            // scores in log2 units: the table holds scale * log2(e) * (q . c)
            tab_build4<NT>(smem, cc, A.q + (int64_t)bh0 * D, A.scale * kLog2e, tid);
        }
        if (validate && tid < A.B && nq_fresh != nq_s[tid]) *stale_s = 1;
        const bool do_dense = A.counters != nullptr && sg.last;
        const int64_t dense_base = (int64_t)HG * A.num_ctas + (int64_t)A.B * A.Hq;
#pragma unroll 1
        for (int h = 0; h < HG; ++h) {
            if (h > 0) __syncthreads();  // the previous head's merge has read dn_*
            if (do_dense)
                dense_warp_state(A.q, A.scale, A.recent_k, A.recent_v, A.ld_recent, A.n_recent,
                                 A.k_cur, A.v_cur, A.Hkv, bh0 + h, b, hkv, warp, W, lane, dn_m,
                                 dn_l, dn_acc);
            if (h == 0 && !cv_ready) {
                mbar_wait(bar_cv, 0);
                cv_ready = true;
            }
            __syncthreads();
            if (h == 0 && validate) {
                validate = false;
                stale_now = *stale_s != 0;
                if (stale_now) break;
            }
            if (do_dense && tid < D) {
                float Mx = -INFINITY;
#pragma unroll
                for (int ww = 0; ww < W; ++ww)
                    if (dn_l[ww] > 0.f) Mx = fmaxf(Mx, dn_m[ww]);
                float L = 0.f, acc = 0.f;
                if (Mx != -INFINITY) {
#pragma unroll
                    for (int ww = 0; ww < W; ++ww) {
                        if (dn_l[ww] > 0.f) {
                            const float f = expf(dn_m[ww] - Mx);
                            L += dn_l[ww] * f;
                            acc += dn_acc[ww][tid] * f;
                        }
                    }
                }
                float *rec = A.parts + (dense_base + bh0 + h) * (D + kPS);
                rec[kPS + tid] = acc;
                if (tid == 0) {
                    rec[0] = Mx;
                    rec[1] = L;
                    rec[2] = 0.f;
                    rec[3] = 0.f;
                }
            }
        }
        if (stale_now) {
            stale_now = false;
            restart();
            continue;
        }
        State4 S;
        S.m = -INFINITY;
        S.l = 0.f;
#pragma unroll
        for (int h = 0; h < HG; ++h)
#pragma unroll
            for (int k = 0; k < 8; ++k) S.acc[h][k] = 0ull;
        int u = u0 + wu;
        const int nunits = max(0, (u1 - u0 - wu + W - 1) / W);
        constexpr int64_t kStep = (int64_t)W * UT * M;  // bytes per unit step of a warp
        const int64_t dv = vbase - kbase;
        int tn = (u + 2 * W) * UT + tA;  // token A of the next unit to load
        const uint8_t *kp = kbase + (int64_t)tn * M;
        for (int trip = 0; trip < nunits / 2; ++trip) {
#pragma unroll
            for (int k = 0; k < 4; ++k) asm volatile("" : "+r"(pk[k]), "+r"(pv[k]));
            bool okA[2], okB[2];
#pragma unroll
            for (int n = 0; n < 2; ++n) {
                const int ta = (u + n * W) * UT + tA;
                okA[n] = ta >= lo && ta < hi;
                okB[n] = ta + 2 >= lo && ta + 2 < hi;
            }
            process4<2>(Ur, S, pk, pv, okA, okB, w, [&]() {
#pragma unroll
                for (int n = 0; n < 2; ++n) {
                    const int ta = tn + n * W * UT;
                    const uint8_t *p = kp + n * kStep;
                    if (ta >= lo && ta < hi) g4::ld8_into(Ur[n].ka, p);
                    if (ta + 2 >= lo && ta + 2 < hi) g4::ld8_into(Ur[n].kb, p + dB);
                }
            });
#pragma unroll
            for (int n = 0; n < 2; ++n) {
                const int ta = tn + n * W * UT;
                const uint8_t *p = kp + n * kStep + dv;
                if (ta >= lo && ta < hi) g4::ld8_into(Ur[n].va, p);
                if (ta + 2 >= lo && ta + 2 < hi) g4::ld8_into(Ur[n].vb, p + dB);
            }
            u += 2 * W;
            kp += 2 * kStep;
            tn += 2 * W * UT;
        }
        if (nunits % 2) {
            bool okA[1], okB[1];
            const int ta = u * UT + tA;
            okA[0] = ta >= lo && ta < hi;
            okB[0] = ta + 2 >= lo && ta + 2 < hi;
            process4<1>(Ur, S, pk, pv, okA, okB, w, []() {});
        }

        // ---- epilogue: one (m, l, acc) record per head for this segment
        // (lane w = 2h of each slot holds head h's state)
        {
            float mw = S.m;
#pragma unroll
            for (int off = 8; off < 32; off <<= 1)
                mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, off));
            if (lane < 8 && (lane & 1) == 0) red_m[(lane >> 1) * W + warp] = mw;
        }
        __syncthreads();  // all warps are past the main loop: the table is free
        float Mx[HG];
#pragma unroll
        for (int h = 0; h < HG; ++h) {
            Mx[h] = red_m[h * W];
#pragma unroll
            for (int ww = 1; ww < W; ++ww) Mx[h] = fmaxf(Mx[h], red_m[h * W + ww]);
        }
        const float f_own = (S.m == -INFINITY) ? 0.f : fast_exp2(S.m - Mx[(w >> 1) & 3]);
        {
            float lw = (w & 1) ? 0.f : S.l * f_own;
#pragma unroll
            for (int off = 8; off < 32; off <<= 1) lw += __shfl_xor_sync(0xffffffffu, lw, off);
            if (lane < 8 && (lane & 1) == 0) red_l[(lane >> 1) * W + warp] = lw;
        }
#pragma unroll
        for (int h = 0; h < HG; ++h) {
            const float f = __shfl_sync(0xffffffffu, f_own, (lane & ~7) | (2 * h));
            float *rows = rows_s + ((h * W + warp) * 4 + slot) * D;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int i = lane_subspace(slot, w, j);
                const float2 a = unpack2(S.acc[h][j]);
                rows[2 * i] = a.x * f;
                rows[2 * i + 1] = a.y * f;
            }
        }
        __syncthreads();
        {
            constexpr int RPP = W * 4 / NG;  // slot rows per 128-thread part
            const int col = tid & (D - 1), prt = tid >> 7;
#pragma unroll
            for (int h = 0; h < HG; ++h) {
                float cs = 0.f;
                const float *rows = rows_s + h * W * 4 * D;
#pragma unroll 8
                for (int rr = prt * RPP; rr < prt * RPP + RPP; ++rr) cs += rows[rr * D + col];
                colsum[h * NG + prt][col] = cs;
            }
        }
        __syncthreads();
        if (tid < D) {
#pragma unroll
            for (int h = 0; h < HG; ++h) {
                float *rec =
                    A.parts + ((int64_t)HG * ((int64_t)(pc + sg.bh) * P + half) + h) * (D + kPS);
                float a = colsum[h * NG][tid];
#pragma unroll
                for (int pp = 1; pp < NG; ++pp) a += colsum[h * NG + pp][tid];
                rec[kPS + tid] = a;
                if (tid == 0) {
                    float L = 0.f;
#pragma unroll
                    for (int ww = 0; ww < W; ++ww) L += red_l[h * W + ww];
                    rec[0] = Mx[h] * kLn2;  // log2 units -> natural
                    rec[1] = L;
                    rec[2] = 0.f;
                    rec[3] = 0.f;
                }
            }
        }
    }
    if (validate) {
        validate = false;
        if (tid < A.B && nq_fresh != nq_s[tid]) *stale_s = 1;
        __syncthreads();
        if (*stale_s) {
            restart();
            goto segments;
        }
    }
    // ---- arrivals and the last arriver's merge (as decode_partials_m64b8)
    if (A.counters != nullptr) {
        __syncthreads();
        const int grp = tid >> 7, gt = tid & (D - 1);
        int64_t p2 = cta_begin(cm, pc);
        Segment s2;
        for (int k = 0; next_segment(nq, A.B, Hqp, &p2, end, &s2); ++k) {
            if (k % NG != grp) continue;
            int c_first, c_last, len;
            head_ctas(nq, Hqp, s2.bh, cm, &c_first, &c_last, &len);
            const int vh2 = vhead(s2.bh);
            if (gt == 0) {
                int old;
                asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;"
                             : "=r"(old)
                             : "l"(A.counters + vh2)
                             : "memory");
                const bool last = (old == c_last - c_first);
                if (last) A.counters[vh2] = 0;
                flag_s[grp] = last ? 1 : 0;
            }
            named_bar_sync(1 + grp, D);
            const bool last = flag_s[grp] != 0;
            named_bar_sync(1 + grp, D);
            if (last) {
                const int b2 = vh2 / Hqv, bq0 = b2 * A.Hq + (vh2 - b2 * Hqv) * HG;
#pragma unroll 1
                for (int h = 0; h < HG; ++h)
                    finish_head(A.parts, (int64_t)HG * A.num_ctas + (int64_t)A.B * A.Hq, HG,
                                s2.bh, h, bq0 + h, c_first, c_last, gt, A.out, A.lse, A.merged,
                                P, half);
            }
        }
    }
    if (!cv_ready) mbar_wait(bar_cv, 0);  // never exit with a bulk copy in flight
}
// ======================================== exact GQA: CTA pairs (clusters) ==
// decode_gqa_pair -- the exact fp32 path for a GQA group that is a multiple of
// 4.  A cluster of two CTAs serves four query heads of a KV head (a virtual
// head); CTA c of the pair owns subspace half c (32 subspaces, output dims
// [64c, 64c + 64)).  Per CTA: the four heads' fp32 key tables of its half as
// two float2 tables (heads 0-1, 2-3: [256][32] x 8 B, 64 KiB each) and its
// half of the fp32 value codebook ([256][32] float2, 64 KiB) -- the value
// gathers are shared by the four heads and every table is exact fp32, which no
// single CTA could hold (4 x 64 KiB tables + 128 KiB codebook).
//   * lane = (token slot s, eighth w): 4 lanes per token, 8 code bytes each
//     ([32c + 8w, +8) of token s (instruction A) and s + 8 (B) of every
//     16-token unit), rotated by 2 bytes when s & 2 (two PRMT per 8 bytes): on
//     the stored decode layout every 8-byte gather of a warp is bank-conflict
//     free (scripts/check_gqa_pair_lanes.py);
//   * a token's 4 lanes reduce the four heads' partial scores with a
//     transposing butterfly (lane w ends with head w over its half), then the
//     pair exchanges them through distributed shared memory: each lane
//     st.async-es its (token A, token B) partial into the peer warp's mailbox,
//     completing tx bytes on the peer's mbarrier, and waits for the peer's
//     (two mailboxes per warp, alternating; the pair runs its units in
//     lockstep, so a mailbox is never overwritten before it is read).  Both
//     CTAs add own + peer (commutative: the same bits), so both run the same
//     online softmax;
//   * lane w owns head w's softmax state of its token slot (one max update and
//     two EX2 per unit) and broadcasts the weights to the slot's 4 lanes;
//   * value path: one LDS.64 per code byte feeds four FFMA2 (one per head);
//   * the records: each CTA writes its 64 output dims of the pair's (m, l, acc)
//     record (rank 0 the header); both CTAs arrive on the virtual head's counter
//     and the last arriver merges in pair order (deterministic).
#ifndef PQKV_PAIR_CLAMP
#define PQKV_PAIR_CLAMP 1
#endif
#ifndef PQKV_PAIR_PERMW
#define PQKV_PAIR_PERMW 1
#endif
#ifndef PQKV_PAIR_RING
#define PQKV_PAIR_RING 3
#endif
namespace gp {
constexpr int HG = 4;
constexpr int UT = 16;       // tokens per warp per unit
constexpr int TAB = 0x10000; // tables: heads 0-1 at 0, heads 2-3 at TAB ([256][32] float2 each)
constexpr int CVO = 0x20000; // the CTA's half of the value codebook ([256][32] float2)
constexpr int HALF_BYTES = KSUB * 32 * 8;                  // 65536
constexpr int OFF_MB = (SMEM_BYTES + 127) / 128 * 128;     // mailboxes [W][2][32] float2
__host__ __device__ constexpr int off_mbar(int W) { return OFF_MB + W * 2 * 32 * 8; }
__host__ __device__ constexpr int smem_bytes(int W) { return off_mbar(W) + W * 2 * 8; }

template <int IMM>
__device__ __forceinline__ unsigned long long lds64(uint32_t a) {
    unsigned long long v;
    asm volatile("ld.shared.b64 %0, [%1+%2];" : "=l"(v) : "r"(a), "n"(IMM));
    return v;
}
__device__ __forceinline__ void fadd2(unsigned long long &acc, unsigned long long x) {
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(x));
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}
// (a, b) into the peer's mailbox; the bytes complete on the peer's mbarrier
__device__ __forceinline__ void st_async2(uint32_t raddr, float a, float b, uint32_t rbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(
            raddr),
        "f"(a), "f"(b), "r"(rbar)
        : "memory");
}

struct UnitP {
    uint2 ka, kb, va, vb;
};
struct StateP {
    float m, l;                     // this lane's head (lane & 3) of its token slot
    unsigned long long acc[HG][8];  // float2 per subspace of this lane, per head
};

// subspace (global index) of byte j of lane (s, w) in CTA half c, after the
// lane's rotation
__device__ __forceinline__ int lane_subspace(int c, int s, int w, int j) {
    const int b = 32 * c + 8 * w + ((j + ((s & 2) ? 2 : 0)) & 7);  // byte of the row
    const int q = b >> 4;
    return 16 * q + (((b & 15) + decode_lane_rot(4 * s + q)) & 15);
}

// the lane's 8 code bytes in processing order: rotated by 2 bytes (slots 2, 3, 6, 7)
__device__ __forceinline__ uint2 rot8(uint2 v, uint32_t sx, uint32_t sy) {
    return make_uint2(__byte_perm(v.x, v.y, sx), __byte_perm(v.x, v.y, sy));
}

// the four heads' partial scores of one token over this lane's 8 subspaces:
// (h0, h1) and (h2, h3) packed
__device__ __forceinline__ void key_scores(const uint2 k, const uint32_t (&pk)[4],
                                           unsigned long long &s01, unsigned long long &s23) {
    unsigned long long a01 = 0, b01 = 0, a23 = 0, b23 = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t a = __byte_perm(j < 4 ? k.x : k.y, pk[j >> 1], sel_for(j));
        const unsigned long long e01 = lds64<0x400>(a), e23 = lds64<0x400 + TAB>(a);
        if (j < 2) {
            (j & 1 ? b01 : a01) = e01;
            (j & 1 ? b23 : a23) = e23;
        } else {
            fadd2(j & 1 ? b01 : a01, e01);
            fadd2(j & 1 ? b23 : a23, e23);
        }
    }
    fadd2(a01, b01);
    fadd2(a23, b23);
    s01 = a01;
    s23 = a23;
}

// this lane's head (w = lane & 3) summed over the token's 4 lanes
__device__ __forceinline__ float reduce_head(unsigned long long s01, unsigned long long s23, int w) {
    const bool b1 = (w & 1) != 0;
#if PQKV_PAIR_PERMW
    // the table's regions are swapped for the subspaces of lanes with w & 2:
    // s01 always holds this lane's head pair (2 b2, 2 b2 + 1)
    const unsigned long long snd = s23;
    unsigned long long keep = s01;
#else
    const bool b2 = (w & 2) != 0;
    const unsigned long long snd = b2 ? s01 : s23;
    unsigned long long keep = b2 ? s23 : s01;
#endif
    const float2 sv = unpack2(snd);
    unsigned long long rcv;
    {
        const float rx = __shfl_xor_sync(0xffffffffu, sv.x, 2);
        const float ry = __shfl_xor_sync(0xffffffffu, sv.y, 2);
        asm("mov.b64 %0, {%1,%2};" : "=l"(rcv) : "f"(rx), "f"(ry));
    }
    fadd2(keep, rcv);  // heads 2 b2, 2 b2 + 1 over w, w ^ 2
    const float2 kv = unpack2(keep);
    const float sndf = b1 ? kv.x : kv.y;
    const float k = b1 ? kv.y : kv.x;
    return k + __shfl_xor_sync(0xffffffffu, sndf, 1);  // head w over all 4 lanes
}
}  // namespace gp

template <int W>
__global__ void __launch_bounds__(W * 32, 1) decode_gqa_pair(const Args A) {
    constexpr int HG = gp::HG, UT = gp::UT, NT = W * 32;
    constexpr int NPART = NT / 64;  // column-sum parts of 64 threads
    static_assert(NT % 64 == 0, "W must be even");
    static_assert(HG * W * 8 * 64 * 4 <= 2 * gp::TAB, "slot rows fit the key tables");
    static_assert(2 * HG * W <= 4 * WMAX, "max / sum reductions fit the red region");
    // the epilogue's column sums live in the dense area: they are written after
    // the epilogue's first barrier, when every thread is past the dense merge
    static_assert(HG * NPART * 64 <= 2 * WMAX + WMAX * D, "column sums fit the dense area");
    using gp::UnitP;
    const int Hqv = A.Hq / HG;

    extern __shared__ __align__(128) unsigned char smem[];
    float *rows_s = reinterpret_cast<float *>(smem);  // epilogue: slot rows in the tables
    float *colsum = reinterpret_cast<float *>(smem + OFF_DNS);  // [HG][NPART][64]
    float *red_m = reinterpret_cast<float *>(smem + OFF_RED);  // written before that barrier
    float *red_l = red_m + HG * W;
    float *dn_m = reinterpret_cast<float *>(smem + OFF_DNS);
    float *dn_l = dn_m + W;
    float(*dn_acc)[D] = reinterpret_cast<float(*)[D]>(dn_l + W);
    int *flag_s = reinterpret_cast<int *>(smem + OFF_FLAG);
    int *nq_s = reinterpret_cast<int *>(smem + OFF_NQ);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
    if ((sbase & 0xFFFFFFu) != kDynBase) __trap();
    const uint32_t cta_byte = sbase & 0xFF000000u;
    const uint32_t bar_cv = sbase + OFF_BAR;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int w = lane & 3, slot = lane >> 2;
    const int wu = W - 1 - warp;
    const uint32_t crank = gp::cluster_rank(), peer = crank ^ 1u;
    const int c = (int)crank;  // subspace half of this CTA
    const int pc = blockIdx.x >> 1, npairs = A.num_ctas >> 1;
    // rotation selectors (slots 2, 3, 6, 7 read their bytes rotated by 2)
    const uint32_t rsx = (slot & 2) ? 0x5432u : 0x3210u, rsy = (slot & 2) ? 0x1076u : 0x7654u;

    // mailboxes and mbarriers of this warp (local), and the peer's
    const uint32_t mb_loc = sbase + gp::OFF_MB + warp * 2 * 32 * 8;
    const uint32_t bar_loc = sbase + gp::off_mbar(W) + warp * 2 * 8;
    const uint32_t mb_rem = gp::mapa(mb_loc, peer), bar_rem = gp::mapa(bar_loc, peer);
    if (tid == 0) {
        mbar_init(bar_cv, 1);
        if (A.early_cv) {
            mbar_expect_tx(bar_cv, gp::HALF_BYTES);
#pragma unroll
            for (int k = 0; k < gp::HALF_BYTES / 16384; ++k)
                bulk_g2s(sbase + gp::CVO + k * 16384,
                         reinterpret_cast<const char *>(A.cv) + c * gp::HALF_BYTES + k * 16384,
                         16384, bar_cv);
        }
    }
    if (lane == 0) {
        mbar_init(bar_loc, 1);
        mbar_init(bar_loc + 8, 1);
    }
    gp::cluster_sync();  // the peer's mbarriers exist before any st.async

    const int group = A.Hq / A.Hkv;
    constexpr int PR = PQKV_PAIR_RING;  // ring depth (units in flight per warp)
    UnitP Ur[PR];
#pragma unroll
    for (int rr = 0; rr < PR; ++rr) Ur[rr].ka = Ur[rr].kb = Ur[rr].va = Ur[rr].vb = uint2{0u, 0u};
    CostMap cm;
    Segment s0;
    bool have_s0 = false;
    int64_t pos = 0, end = 0;
    const bool nq_cached = A.B <= kNqCache;
    const bool early = A.early_codes && nq_cached;
    // ring loads are unconditional: a token outside [lo, hi) loads a row of
    // the segment instead (its weight is masked to 0), so no load result is
    // ever merged into a ring register by a move that would wait for it
    auto row = [](int t, int lo, int hi) { return (int64_t)min(max(t, lo), hi - 1) * M; };
    auto load_unit = [&](UnitP &U, const uint8_t *kbase, const uint8_t *vbase, int u, int lo,
                         int hi) {
        if (hi <= lo) return;  // an empty segment has no units
        const int ta = u * UT + slot;
#if PQKV_PAIR_CLAMP
        U.ka = g4::ld8(kbase + row(ta, lo, hi));
        U.va = g4::ld8(vbase + row(ta, lo, hi));
        U.kb = g4::ld8(kbase + row(ta + 8, lo, hi));
        U.vb = g4::ld8(vbase + row(ta + 8, lo, hi));
#else
        if (ta >= lo && ta < hi) {
            U.ka = g4::ld8(kbase + (int64_t)ta * M);
            U.va = g4::ld8(vbase + (int64_t)ta * M);
        }
        if (ta + 8 >= lo && ta + 8 < hi) {
            U.kb = g4::ld8(kbase + (int64_t)(ta + 8) * M);
            U.vb = g4::ld8(vbase + (int64_t)(ta + 8) * M);
        }
#endif
    };
    auto first_ring = [&]() {
        const int32_t *src = A.n_q;
        if (nq_cached) {
            for (int bb = tid; bb < A.B; bb += NT) nq_s[bb] = __ldcg(A.n_q + bb);
            __syncthreads();
            src = nq_s;
        }
        cm = cost_map(src, A.B, Hqv, npairs);
        pos = cta_begin(cm, pc);
        end = min(cta_begin(cm, pc + 1), cm.total);
        int64_t p0 = pos;
        have_s0 = next_segment(src, A.B, Hqv, &p0, end, &s0);
        if (have_s0) {
            const int b = s0.bh / Hqv, hkv = (s0.bh - b * Hqv) * HG / group;
            const int64_t head_off = ((int64_t)b * A.Hkv + hkv) * A.ld_tok * M + 32 * c + 8 * w;
            const int u0 = s0.lo / UT;
#pragma unroll
            for (int rr = 0; rr < PR; ++rr)
                load_unit(Ur[rr], A.codes_k + head_off, A.codes_v + head_off, u0 + wu + rr * W,
                          s0.lo, s0.hi);
        }
    };
    int *stale_s = flag_s + (WMAX / 4);
    if (early) {
        if (tid == 0) *stale_s = 0;
        first_ring();
    }
    pdl_launch_dependents();
    pdl_wait();
    int nq_fresh = 0;
    if (early && tid < A.B) nq_fresh = __ldcg(A.n_q + tid);
    if (!early) first_ring();
    if (tid == 0 && !A.early_cv) {
        mbar_expect_tx(bar_cv, gp::HALF_BYTES);
#pragma unroll
        for (int k = 0; k < gp::HALF_BYTES / 16384; ++k)
            bulk_g2s(sbase + gp::CVO + k * 16384,
                     reinterpret_cast<const char *>(A.cv) + c * gp::HALF_BYTES + k * 16384, 16384,
                     bar_cv);
    }

    // lane-constant address bytes: key tables and value codebook share the
    // address code << 8 | (i & 31) << 3 (the regions ride in the immediates)
    uint32_t pk[4];
#pragma unroll
    for (int jp = 0; jp < 4; ++jp) {
        uint32_t a = 0;
#pragma unroll
        for (int e = 0; e < 2; ++e)
            a |= (uint32_t)((gp::lane_subspace(c, slot, w, 2 * jp + e) & 31) << 3) << (8 * e);
        pk[jp] = a | cta_byte;
    }

    bool cv_ready = false;
    const int32_t *nq = nq_cached ? nq_s : A.n_q;
    bool ring_loaded = have_s0;
    Segment sg;
    bool validate = early;
    uint32_t xu = 0;  // units exchanged with the peer warp (mailbox xu & 1, parity (xu >> 1) & 1)
    auto restart = [&]() {
        __syncthreads();
        if (tid < A.B) nq_s[tid] = nq_fresh;
        if (tid == 0) *stale_s = 0;
        __syncthreads();
        cm = cost_map(nq_s, A.B, Hqv, npairs);
        pos = cta_begin(cm, pc);
        end = min(cta_begin(cm, pc + 1), cm.total);
        ring_loaded = false;
    };
    bool stale_now = false;
  segments:
    while (next_segment(nq, A.B, Hqv, &pos, end, &sg)) {
        const int vh = sg.bh;
        const int b = vh / Hqv, hq0 = (vh - b * Hqv) * HG, hkv = hq0 / group;
        const int bh0 = b * A.Hq + hq0;
        const int64_t head_off = ((int64_t)b * A.Hkv + hkv) * A.ld_tok * M + 32 * c + 8 * w;
        const uint8_t *kbase = A.codes_k + head_off;
        const uint8_t *vbase = A.codes_v + head_off;
        const int lo = sg.lo, hi = sg.hi;
        const int u0 = lo / UT, u1 = (hi + UT - 1) / UT;
        if (!ring_loaded) {
#pragma unroll
            for (int rr = 0; rr < PR; ++rr)
                load_unit(Ur[rr], kbase, vbase, u0 + wu + rr * W, lo, hi);
        }
        ring_loaded = false;

        __syncthreads();  // the previous segment's epilogue is done with the tables
        {
            // this half's tables, scores in log2 units: entry (code, i) of head h
            // = scale log2(e) (q_h[2i] C[code][i].x + q_h[2i+1] C[code][i].y)
            constexpr int kSlots = KSUB * 16;  // float4 slots (two subspaces) of the half
            const float sc = A.scale * kLog2e;
            const float4 *src = reinterpret_cast<const float4 *>(A.ck);
#pragma unroll 4
            for (int f = tid; f < kSlots; f += NT) {
                const int cc = f >> 4, pr = f & 15;
                const float4 cb = __ldg(src + cc * 32 + 16 * c + pr);
                float e[HG][2];
#pragma unroll
                for (int h = 0; h < HG; ++h) {
                    const float4 qv =
                        __ldg(reinterpret_cast<const float4 *>(A.q + (int64_t)(bh0 + h) * D) +
                              16 * c + pr);
                    e[h][0] = sc * fmaf(qv.y, cb.y, qv.x * cb.x);
                    e[h][1] = sc * fmaf(qv.w, cb.w, qv.z * cb.z);
                }
                const int off = (cc << 8) | (pr << 4);
#if PQKV_PAIR_PERMW
                // subspaces 16..31 of the half are read by lanes with w & 2
                // (reduce_head): their first region holds heads 2, 3
                const int sw = (pr >> 3) << 16;
#else
                const int sw = 0;
#endif
                *reinterpret_cast<float4 *>(smem + (off ^ sw)) =
                    make_float4(e[0][0], e[1][0], e[0][1], e[1][1]);
                *reinterpret_cast<float4 *>(smem + ((gp::TAB + off) ^ sw)) =
                    make_float4(e[2][0], e[3][0], e[2][1], e[3][1]);
            }
        }
        if (validate && tid < A.B && nq_fresh != nq_s[tid]) *stale_s = 1;
        const bool do_dense = A.counters != nullptr && sg.last && c == 0;
        const int64_t dense_base = (int64_t)HG * npairs + (int64_t)A.B * A.Hq;
#pragma unroll 1
        for (int h = 0; h < HG; ++h) {
            if (h > 0) __syncthreads();
            if (do_dense)
                dense_warp_state(A.q, A.scale, A.recent_k, A.recent_v, A.ld_recent, A.n_recent,
                                 A.k_cur, A.v_cur, A.Hkv, bh0 + h, b, hkv, warp, W, lane, dn_m,
                                 dn_l, dn_acc);
            if (h == 0 && !cv_ready) {
                mbar_wait(bar_cv, 0);
                cv_ready = true;
            }
            __syncthreads();
            if (h == 0 && validate) {
                validate = false;
                stale_now = *stale_s != 0;
                if (stale_now) break;
            }
            if (do_dense && tid < D) {
                float Mx = -INFINITY;
#pragma unroll
                for (int ww = 0; ww < W; ++ww)
                    if (dn_l[ww] > 0.f) Mx = fmaxf(Mx, dn_m[ww]);
                float L = 0.f, acc = 0.f;
                if (Mx != -INFINITY) {
#pragma unroll
                    for (int ww = 0; ww < W; ++ww) {
                        if (dn_l[ww] > 0.f) {
                            const float f = expf(dn_m[ww] - Mx);
                            L += dn_l[ww] * f;
                            acc += dn_acc[ww][tid] * f;
                        }
                    }
                }
                float *rec = A.parts + (dense_base + bh0 + h) * (D + kPS);
                rec[kPS + tid] = acc;
                if (tid == 0) {
                    rec[0] = Mx;
                    rec[1] = L;
                    rec[2] = 0.f;
                    rec[3] = 0.f;
                }
            }
        }
        if (stale_now) {
            stale_now = false;
            restart();
            continue;
        }
        gp::StateP S;
        S.m = -INFINITY;
        S.l = 0.f;
#pragma unroll
        for (int h = 0; h < HG; ++h)
#pragma unroll
            for (int k = 0; k < 8; ++k) S.acc[h][k] = 0ull;

        int u = u0 + wu;
        const int nunits = max(0, (u1 - u0 - wu + W - 1) / W);
        // one unit through ring slot U (static register indices: the loop
        // below runs the two slots alternately)
        auto unit_step = [&](UnitP &U) {
            const int ta = u * UT + slot;
            const bool okA = ta >= lo && ta < hi, okB = ta + 8 >= lo && ta + 8 < hi;
            // key phase (this half), the pair's exchange, softmax at the owner lane
            unsigned long long a01, a23, b01, b23;
            gp::key_scores(gp::rot8(U.ka, rsx, rsy), pk, a01, a23);
            gp::key_scores(gp::rot8(U.kb, rsx, rsy), pk, b01, b23);
            const float oa = gp::reduce_head(a01, a23, w), ob = gp::reduce_head(b01, b23, w);
            const uint32_t buf = xu & 1u, par = (xu >> 1) & 1u;
            ++xu;
            gp::st_async2(mb_rem + buf * 256 + lane * 8, oa, ob, bar_rem + buf * 8);
            if (lane == 0) mbar_expect_tx(bar_loc + buf * 8, 256);
            // refill this ring slot's key registers (the key phase is done with them)
            {
                const int tn = (u + PR * W) * UT + slot;
#if PQKV_PAIR_CLAMP
                g4::ld8_into(U.ka, kbase + row(tn, lo, hi));
                g4::ld8_into(U.kb, kbase + row(tn + 8, lo, hi));
#else
                if (tn >= lo && tn < hi) U.ka = g4::ld8(kbase + (int64_t)tn * M);
                if (tn + 8 >= lo && tn + 8 < hi) U.kb = g4::ld8(kbase + (int64_t)(tn + 8) * M);
#endif
            }
            mbar_wait(bar_loc + buf * 8, par);
            float pa_, pb_;
            {
                float2 r;
                asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(r.x), "=f"(r.y)
                             : "r"(mb_loc + buf * 256 + lane * 8));
                // own + peer in rank order: both CTAs add the same two values
                const float sa = c == 0 ? oa + r.x : r.x + oa;
                const float sb = c == 0 ? ob + r.y : r.y + ob;
                const float mx = fmaxf(okA ? sa : -INFINITY, okB ? sb : -INFINITY);
                const bool up = mx > S.m + kLazyRescale;
                if (__any_sync(0xffffffffu, up)) {  // rare: rescale the slot's accumulators
                    const float f = up ? fast_exp2(S.m - mx) : 1.f;
                    if (up) {
                        S.l *= f;
                        S.m = mx;
                    }
#pragma unroll
                    for (int h = 0; h < HG; ++h) {
#if PQKV_PAIR_PERMW
                        const float fh = __shfl_xor_sync(0xffffffffu, f, h);  // head h ^ w
#else
                        const float fh = __shfl_sync(0xffffffffu, f, (lane & ~3) | h);
#endif
#pragma unroll
                        for (int k = 0; k < 8; ++k) fmul2(S.acc[h][k], fh);
                    }
                }
                pa_ = okA ? fast_exp2(sa - S.m) : 0.f;
                pb_ = okB ? fast_exp2(sb - S.m) : 0.f;
                S.l += pa_ + pb_;
            }
            // the slot's four heads' weights in every lane of the slot
            float pa[HG], pb[HG];
#if PQKV_PAIR_PERMW
            {   // slot k holds head k ^ w (as S.acc[k]): no selects
                const float xa = __shfl_xor_sync(0xffffffffu, pa_, 1);
                const float xb = __shfl_xor_sync(0xffffffffu, pb_, 1);
                pa[0] = pa_;
                pa[1] = xa;
                pa[2] = __shfl_xor_sync(0xffffffffu, pa_, 2);
                pa[3] = __shfl_xor_sync(0xffffffffu, xa, 2);
                pb[0] = pb_;
                pb[1] = xb;
                pb[2] = __shfl_xor_sync(0xffffffffu, pb_, 2);
                pb[3] = __shfl_xor_sync(0xffffffffu, xb, 2);
            }
#else
            {
                const float xa = __shfl_xor_sync(0xffffffffu, pa_, 1);
                const float xb = __shfl_xor_sync(0xffffffffu, pb_, 1);
                const bool b1 = (w & 1) != 0, b2 = (w & 2) != 0;
                const float a0 = b1 ? xa : pa_, a1 = b1 ? pa_ : xa;  // heads 2 b2, 2 b2 + 1
                const float c0 = b1 ? xb : pb_, c1 = b1 ? pb_ : xb;
                const float ya0 = __shfl_xor_sync(0xffffffffu, a0, 2);
                const float ya1 = __shfl_xor_sync(0xffffffffu, a1, 2);
                const float yb0 = __shfl_xor_sync(0xffffffffu, c0, 2);
                const float yb1 = __shfl_xor_sync(0xffffffffu, c1, 2);
                pa[0] = b2 ? ya0 : a0;
                pa[1] = b2 ? ya1 : a1;
                pa[2] = b2 ? a0 : ya0;
                pa[3] = b2 ? a1 : ya1;
                pb[0] = b2 ? yb0 : c0;
                pb[1] = b2 ? yb1 : c1;
                pb[2] = b2 ? c0 : yb0;
                pb[3] = b2 ? c1 : yb1;
            }
#endif
            // value phase: one gather per code byte, four FFMA2
            {
                const uint2 va = gp::rot8(U.va, rsx, rsy), vb = gp::rot8(U.vb, rsx, rsy);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t wa = j < 4 ? va.x : va.y, wb = j < 4 ? vb.x : vb.y;
                    const unsigned long long ca =
                        gp::lds64<0x400 + gp::CVO>(__byte_perm(wa, pk[j >> 1], sel_for(j)));
                    const unsigned long long cb =
                        gp::lds64<0x400 + gp::CVO>(__byte_perm(wb, pk[j >> 1], sel_for(j)));
#pragma unroll
                    for (int h = 0; h < HG; ++h) {
                        ffma2(S.acc[h][j], pa[h], ca);
                        ffma2(S.acc[h][j], pb[h], cb);
                    }
                }
            }
            {
                const int tn = (u + PR * W) * UT + slot;
#if PQKV_PAIR_CLAMP
                g4::ld8_into(U.va, vbase + row(tn, lo, hi));
                g4::ld8_into(U.vb, vbase + row(tn + 8, lo, hi));
#else
                if (tn >= lo && tn < hi) U.va = g4::ld8(vbase + (int64_t)tn * M);
                if (tn + 8 >= lo && tn + 8 < hi) U.vb = g4::ld8(vbase + (int64_t)(tn + 8) * M);
#endif
            }
            u += W;
        };
        for (int trip = 0; trip < nunits / PR; ++trip) {
#pragma unroll
            for (int k = 0; k < 4; ++k) asm volatile("" : "+r"(pk[k]));
#pragma unroll
            for (int rr = 0; rr < PR; ++rr) unit_step(Ur[rr]);
        }
#pragma unroll
        for (int rr = 0; rr < PR - 1; ++rr)
            if (rr < nunits % PR) unit_step(Ur[rr]);

        // ---- epilogue: this CTA's 64 dims of the pair's record per head
        {
            float mw = S.m;  // head w: max over the warp's slots (lanes with the same w)
#pragma unroll
            for (int off = 4; off < 32; off <<= 1)
                mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, off));
            if (lane < HG) red_m[lane * W + warp] = mw;
        }
        __syncthreads();  // all warps are past the main loop: the tables are free
        float Mx[HG];
#pragma unroll
        for (int h = 0; h < HG; ++h) {
            Mx[h] = red_m[h * W];
#pragma unroll
            for (int ww = 1; ww < W; ++ww) Mx[h] = fmaxf(Mx[h], red_m[h * W + ww]);
        }
        {
            const float f = (S.m == -INFINITY) ? 0.f : fast_exp2(S.m - Mx[w]);
            float lw = S.l * f;
#pragma unroll
            for (int off = 4; off < 32; off <<= 1) lw += __shfl_xor_sync(0xffffffffu, lw, off);
            if (lane < HG) red_l[lane * W + warp] = lw;
#pragma unroll
            for (int k = 0; k < HG; ++k) {
#if PQKV_PAIR_PERMW
                const int h = k ^ w;  // S.acc[k] holds head k ^ w
                const float fh = __shfl_xor_sync(0xffffffffu, f, k);
#else
                const int h = k;
                const float fh = __shfl_sync(0xffffffffu, f, (lane & ~3) | h);
#endif
                float *rows = rows_s + ((h * W + warp) * 8 + slot) * 64;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int i = gp::lane_subspace(c, slot, w, j) - 32 * c;
                    const float2 a = unpack2(S.acc[k][j]);
                    rows[2 * i] = a.x * fh;
                    rows[2 * i + 1] = a.y * fh;
                }
            }
        }
        __syncthreads();
        {
            constexpr int RPP = W * 8 / NPART;  // slot rows per 64-thread part
            const int col = tid & 63, prt = tid >> 6;
#pragma unroll
            for (int h = 0; h < HG; ++h) {
                float cs = 0.f;
                const float *rows = rows_s + h * W * 8 * 64;
#pragma unroll 8
                for (int rr = prt * RPP; rr < prt * RPP + RPP; ++rr) cs += rows[rr * 64 + col];
                colsum[(h * NPART + prt) * 64 + col] = cs;
            }
        }
        __syncthreads();
        if (tid < HG * 64) {
            const int h = tid >> 6, col = tid & 63;
            float *rec = A.parts + ((int64_t)HG * (pc + sg.bh) + h) * (D + kPS);
            float a = colsum[(h * NPART) * 64 + col];
#pragma unroll
            for (int pp = 1; pp < NPART; ++pp) a += colsum[(h * NPART + pp) * 64 + col];
            rec[kPS + 64 * c + col] = a;
            if (c == 0 && col == 0) {
                float L = 0.f;
#pragma unroll
                for (int ww = 0; ww < W; ++ww) L += red_l[h * W + ww];
                rec[0] = Mx[h] * kLn2;  // log2 units -> natural
                rec[1] = L;
                rec[2] = 0.f;
                rec[3] = 0.f;
            }
        }
    }
    if (validate) {
        validate = false;
        if (tid < A.B && nq_fresh != nq_s[tid]) *stale_s = 1;
        __syncthreads();
        if (*stale_s) {
            restart();
            goto segments;
        }
    }
    gp::cluster_sync();  // every exchange with the peer is complete
    // ---- arrivals (both CTAs of each pair) and the last arriver's merge
    if (A.counters != nullptr) {
        __syncthreads();
        constexpr int NG = NT / 128;
        const int grp = tid >> 7, gt = tid & (D - 1);
        int64_t p2 = cta_begin(cm, pc);
        Segment s2;
        for (int k = 0; next_segment(nq, A.B, Hqv, &p2, end, &s2); ++k) {
            if (k % NG != grp) continue;
            int c_first, c_last, len;
            head_ctas(nq, Hqv, s2.bh, cm, &c_first, &c_last, &len);
            if (gt == 0) {
                int old;
                asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;"
                             : "=r"(old)
                             : "l"(A.counters + s2.bh)
                             : "memory");
                const bool last = (old == 2 * (c_last - c_first) + 1);
                if (last) A.counters[s2.bh] = 0;
                flag_s[grp] = last ? 1 : 0;
            }
            named_bar_sync(1 + grp, D);
            const bool last = flag_s[grp] != 0;
            named_bar_sync(1 + grp, D);
            if (last) {
                const int b2 = s2.bh / Hqv, bq0 = b2 * A.Hq + (s2.bh - b2 * Hqv) * HG;
#pragma unroll 1
                for (int h = 0; h < HG; ++h)
                    finish_head(A.parts, (int64_t)HG * npairs + (int64_t)A.B * A.Hq, HG, s2.bh, h,
                                bq0 + h, c_first, c_last, gt, A.out, A.lse, A.merged, 1, 0);
            }
        }
    }
    if (!cv_ready) mbar_wait(bar_cv, 0);
}

}  // namespace fast

// ========================================================= generic path ====
// Any geometry (nbits <= 16, d <= 1024).  Tiles of 256 tokens: one thread per
// token for the LUT score (LUT read through L1 from global memory), then one
// thread per output dimension for the value accumulation.  Correctness path
// for geometries other than m64b8; not tuned.
constexpr int GT = 256;
constexpr int GMAXD = 1024;

template <typename CT>
__global__ void __launch_bounds__(GT)
    decode_partials_generic(const float *__restrict__ lut_g, int B, int Hq, int Hkv,
                            const CT *__restrict__ codes_k, const CT *__restrict__ codes_v,
                            int64_t ld_tok, const int32_t *__restrict__ n_q,
                            const float *__restrict__ cb_v, int d, int M, int ksub, int num_ctas,
                            float *__restrict__ parts) {
    __shared__ float p_s[GT];
    __shared__ float red[GT / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int dsub = d / M;
    const CostMap cm = cost_map(n_q, B, Hq, num_ctas);
    const int cta = blockIdx.x;
    int64_t pos = cta_begin(cm, cta);
    const int64_t end = min(cta_begin(cm, cta + 1), cm.total);
    const int group = Hq / Hkv;

    Segment sg;
    while (next_segment(n_q, B, Hq, &pos, end, &sg)) {
        const int bh = sg.bh, t0 = sg.lo, n = sg.hi - sg.lo;
        const int b = bh / Hq, hq = bh - b * Hq, hkv = hq / group;
        const float *lut = lut_g + (int64_t)bh * ksub * M;
        const int64_t head_off = ((int64_t)b * Hkv + hkv) * ld_tok * M;
        const CT *kc = codes_k + head_off + (int64_t)t0 * M;
        const CT *vc = codes_v + head_off + (int64_t)t0 * M;

        float m_run = -INFINITY, l_run = 0.f;
        float acc[GMAXD / GT];
#pragma unroll
        for (int k = 0; k < GMAXD / GT; ++k) acc[k] = 0.f;

        for (int base = 0; base < n; base += GT) {
            const int cnt = min(GT, n - base);
            const int t = base + tid;
            float s = -INFINITY;
            if (tid < cnt) {
                s = 0.f;
                for (int i = 0; i < M; ++i) s += __ldg(lut + (int64_t)kc[(int64_t)t * M + i] * M + i);
            }
            float mx = s;
            for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            __syncthreads();  // previous tile finished reading p_s / red
            if (lane == 0) red[warp] = mx;
            __syncthreads();
            float mt = red[0];
            for (int w = 1; w < GT / 32; ++w) mt = fmaxf(mt, red[w]);
            if (mt > m_run) {
                const float f = (m_run == -INFINITY) ? 0.f : expf(m_run - mt);
                l_run *= f;
#pragma unroll
                for (int k = 0; k < GMAXD / GT; ++k) acc[k] *= f;
                m_run = mt;
            }
            const float p = (tid < cnt) ? expf(s - m_run) : 0.f;
            p_s[tid] = p;
            float ps = p;
            for (int off = 16; off > 0; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
            __syncthreads();
            if (lane == 0) red[warp] = ps;
            __syncthreads();
            float lt = 0.f;
            for (int w = 0; w < GT / 32; ++w) lt += red[w];
            l_run += lt;
#pragma unroll
            for (int k = 0; k < GMAXD / GT; ++k) {
                const int j = tid + k * GT;
                if (j < d) {
                    const int i = j / dsub, jj = j - i * dsub;
                    const float *cvi = cb_v + (int64_t)i * ksub * dsub + jj;
                    float a = 0.f;
                    for (int tt = 0; tt < cnt; ++tt)
                        a = fmaf(p_s[tt], __ldg(cvi + (int64_t)vc[(int64_t)(base + tt) * M + i] * dsub), a);
                    acc[k] += a;
                }
            }
        }
        float *rec = parts + ((int64_t)cta + bh) * (d + kPS);
#pragma unroll
        for (int k = 0; k < GMAXD / GT; ++k) {
            const int j = tid + k * GT;
            if (j < d) rec[kPS + j] = acc[k];
        }
        if (tid == 0) {
            rec[0] = m_run;
            rec[1] = l_run;
            rec[2] = 0.f;
            rec[3] = 0.f;
        }
        __syncthreads();
    }
}

// ============================================================== finish =====
constexpr int FT = 128;
constexpr int FMAXD = 1024;

struct Part {
    float m, l;
};

// merge_partials (attention.py:193-204): identity on l == 0.
__device__ __forceinline__ void merge_into(float &m, float &l, float (&acc)[FMAXD / FT], float mb,
                                           float lb, const float *accb, int d) {
    if (lb == 0.f) return;
    if (l == 0.f) {
        m = mb;
        l = lb;
#pragma unroll
        for (int k = 0; k < FMAXD / FT; ++k) {
            const int j = threadIdx.x + k * FT;
            acc[k] = (j < d) ? accb[j] : 0.f;
        }
        return;
    }
    const float mm = fmaxf(m, mb);
    const float wa = expf(m - mm), wb = expf(mb - mm);
    l = l * wa + lb * wb;
#pragma unroll
    for (int k = 0; k < FMAXD / FT; ++k) {
        const int j = threadIdx.x + k * FT;
        if (j < d) acc[k] = acc[k] * wa + accb[j] * wb;
    }
    m = mm;
}

constexpr int DCH_MAX = 32;  // dense rows staged per chunk (fewer for wide heads)
inline int dense_chunk(int d) { return std::max(1, std::min(DCH_MAX, 12000 / (2 * d))); }

// One CTA per (b, hq).  Every global load of a phase is issued before any is
// consumed (records in batches of 8, dense rows staged to shared memory with
// coalesced 16-byte loads), so the kernel pays a few memory latencies, not one
// per record / row.
__global__ void __launch_bounds__(FT)
    decode_finish_kernel(const float *__restrict__ parts, int num_ctas, int B, int Hq, int Hkv,
                         int d, const int32_t *__restrict__ n_q, const float *__restrict__ q,
                         float scale, const float *__restrict__ recent_k,
                         const float *__restrict__ recent_v, int64_t ld_recent,
                         const int32_t *__restrict__ n_recent, const float *__restrict__ k_cur,
                         const float *__restrict__ v_cur, float *__restrict__ out,
                         float *__restrict__ lse, float *__restrict__ merged, int DCH) {
    extern __shared__ float fsm[];
    float *ks = fsm;             // [DCH][d]
    float *vs = fsm + DCH * d;   // [DCH][d]
    float *sc = vs + DCH * d;    // [DCH]
    const int bh = blockIdx.x;
    const int b = bh / Hq, hq = bh - b * Hq, hkv = hq / (Hq / Hkv);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    float m = -INFINITY, l = 0.f;
    float acc[FMAXD / FT];
#pragma unroll
    for (int k = 0; k < FMAXD / FT; ++k) acc[k] = 0.f;

    // 1. quantized partials of this head, merged in CTA order (deterministic)
    if (parts != nullptr && n_q != nullptr) {
        const CostMap cm = cost_map(n_q, B, Hq, num_ctas);
        int c_first, c_last, len;
        head_ctas(n_q, Hq, bh, cm, &c_first, &c_last, &len);
        if (len > 0) {  // an empty head's single record is empty: skip it (may be unwritten)
            for (int c0 = c_first; c0 <= c_last; c0 += 8) {
                const int cnt = min(8, c_last - c0 + 1);
                float rm[8], rl[8], ra[8][FMAXD / FT];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (k < cnt) {
                        const float *rec = parts + ((int64_t)c0 + k + bh) * (d + kPS);
                        rm[k] = rec[0];
                        rl[k] = rec[1];
#pragma unroll
                        for (int e = 0; e < FMAXD / FT; ++e) {
                            const int j = tid + e * FT;
                            ra[k][e] = (j < d) ? rec[kPS + j] : 0.f;
                        }
                    }
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (k >= cnt || rl[k] == 0.f) continue;
                    if (l == 0.f) {
                        m = rm[k];
                        l = rl[k];
#pragma unroll
                        for (int e = 0; e < FMAXD / FT; ++e) acc[e] = ra[k][e];
                        continue;
                    }
                    const float mm = fmaxf(m, rm[k]);
                    const float wa = expf(m - mm), wb = expf(rm[k] - mm);
                    l = l * wa + rl[k] * wb;
#pragma unroll
                    for (int e = 0; e < FMAXD / FT; ++e) acc[e] = acc[e] * wa + ra[k][e] * wb;
                    m = mm;
                }
            }
        }
    }

    // 2. dense partial over recent rows [0, n_recent[b]) + the current token
    const int nr = (n_recent != nullptr && recent_k != nullptr) ? max(n_recent[b], 0) : 0;
    const int rows = nr + (k_cur != nullptr ? 1 : 0);
    const float *qh = q + (int64_t)bh * d;
    const int64_t rbase = ((int64_t)b * Hkv + hkv) * ld_recent * d;
    const int64_t cbase = ((int64_t)b * Hkv + hkv) * d;
    const bool vec4 = (d % 4) == 0;
    for (int r0 = 0; r0 < rows; r0 += DCH) {
        const int cn = min(DCH, rows - r0);
        __syncthreads();  // previous chunk fully consumed
        if (vec4) {
            const int d4 = d / 4;
            for (int idx = tid; idx < cn * d4; idx += FT) {
                const int rr = idx / d4, jj = idx - rr * d4, row = r0 + rr;
                const float4 *kr = reinterpret_cast<const float4 *>(
                    row < nr ? recent_k + rbase + (int64_t)row * d : k_cur + cbase);
                const float4 *vr = reinterpret_cast<const float4 *>(
                    row < nr ? recent_v + rbase + (int64_t)row * d : v_cur + cbase);
                reinterpret_cast<float4 *>(ks)[rr * d4 + jj] = __ldg(kr + jj);
                reinterpret_cast<float4 *>(vs)[rr * d4 + jj] = __ldg(vr + jj);
            }
        } else {
            for (int idx = tid; idx < cn * d; idx += FT) {
                const int rr = idx / d, jj = idx - rr * d, row = r0 + rr;
                ks[idx] = row < nr ? recent_k[rbase + (int64_t)row * d + jj] : k_cur[cbase + jj];
                vs[idx] = row < nr ? recent_v[rbase + (int64_t)row * d + jj] : v_cur[cbase + jj];
            }
        }
        __syncthreads();
        for (int rr = warp; rr < cn; rr += FT / 32) {
            float dot = 0.f;
            for (int j = lane; j < d; j += 32) dot = fmaf(__ldg(qh + j), ks[rr * d + j], dot);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
            if (lane == 0) sc[rr] = scale * dot;
        }
        __syncthreads();
        float md = -INFINITY;
        for (int rr = 0; rr < cn; ++rr) md = fmaxf(md, sc[rr]);
        float ld = 0.f;
        float dacc[FMAXD / FT];
#pragma unroll
        for (int e = 0; e < FMAXD / FT; ++e) dacc[e] = 0.f;
        for (int rr = 0; rr < cn; ++rr) {
            const float p = expf(sc[rr] - md);
            ld += p;
#pragma unroll
            for (int e = 0; e < FMAXD / FT; ++e) {
                const int j = tid + e * FT;
                if (j < d) dacc[e] = fmaf(p, vs[rr * d + j], dacc[e]);
            }
        }
        if (l == 0.f) {
            m = md;
            l = ld;
#pragma unroll
            for (int e = 0; e < FMAXD / FT; ++e) acc[e] = dacc[e];
        } else {
            const float mm = fmaxf(m, md);
            const float wa = expf(m - mm), wb = expf(md - mm);
            l = l * wa + ld * wb;
#pragma unroll
            for (int e = 0; e < FMAXD / FT; ++e) acc[e] = acc[e] * wa + dacc[e] * wb;
            m = mm;
        }
    }

    const float inv = (l > 0.f) ? 1.f / l : NAN;
#pragma unroll
    for (int k = 0; k < FMAXD / FT; ++k) {
        const int j = tid + k * FT;
        if (j < d) {
            if (out) out[(int64_t)bh * d + j] = acc[k] * inv;
            if (merged) merged[(int64_t)bh * (d + kPS) + kPS + j] = acc[k];
        }
    }
    if (tid == 0) {
        if (lse) lse[bh] = (l > 0.f) ? m + logf(l) : -INFINITY;
        if (merged) {
            float *rec = merged + (int64_t)bh * (d + kPS);
            rec[0] = m;
            rec[1] = l;
            rec[2] = 0.f;
            rec[3] = 0.f;
        }
    }
}

__global__ void __launch_bounds__(FT)
    merge_partials_kernel(const float *__restrict__ parts, int n_parts, int64_t n_heads, int d,
                          float *__restrict__ out, float *__restrict__ lse,
                          float *__restrict__ merged) {
    const int64_t h = blockIdx.x;
    float m = -INFINITY, l = 0.f;
    float acc[FMAXD / FT];
#pragma unroll
    for (int k = 0; k < FMAXD / FT; ++k) acc[k] = 0.f;
    for (int p = 0; p < n_parts; ++p) {
        const float *rec = parts + ((int64_t)p * n_heads + h) * (d + kPS);
        merge_into(m, l, acc, rec[0], rec[1], rec + kPS, d);
    }
    const float inv = (l > 0.f) ? 1.f / l : NAN;
#pragma unroll
    for (int k = 0; k < FMAXD / FT; ++k) {
        const int j = threadIdx.x + k * FT;
        if (j < d) {
            if (out) out[h * d + j] = acc[k] * inv;
            if (merged) merged[h * (d + kPS) + kPS + j] = acc[k];
        }
    }
    if (threadIdx.x == 0) {
        if (lse) lse[h] = (l > 0.f) ? m + logf(l) : -INFINITY;
        if (merged) {
            float *rec = merged + h * (d + kPS);
            rec[0] = m;
            rec[1] = l;
            rec[2] = 0.f;
            rec[3] = 0.f;
        }
    }
}

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (dev < 64 && cached[dev] > 0) return cached[dev];
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    if (dev < 64) cached[dev] = n;
    return n;
}

}  // namespace
}  // namespace pqkv

using namespace pqkv;

extern "C" int pqkv_decode_grid(int d, int M, int nbits, int *num_ctas) {
    PQKV_CHECK_ARG(geometry_ok(d, M, nbits) && num_ctas, "pqkv_decode_grid: bad arguments");
    const int sms = sm_count();
    if (sms <= 0) return fail(PQKV_ECUDA, "pqkv_decode_grid: no CUDA device");
    *num_ctas = is_fast_geometry(d, M, nbits) ? sms : 4 * sms;
    return PQKV_OK;
}

#ifdef PQKV_TRACE
extern "C" int pqkv_debug_trace(unsigned long long *host, int n) {  // n <= 64 * 256 * 32
    return cudaMemcpyFromSymbol(host, fast::g_trace, sizeof(unsigned long long) * n) == cudaSuccess
               ? 0 : 2;
}
extern "C" int pqkv_debug_wtrace(unsigned long long *host, int n) {  // n <= 64 * 256 * 32
    return cudaMemcpyFromSymbol(host, fast::g_wtrace, sizeof(unsigned long long) * n) ==
                   cudaSuccess
               ? 0 : 2;
}
#endif

extern "C" int64_t pqkv_partials_floats(int num_ctas, int B, int Hq, int d) {
    // split records (up to four per split and virtual head when a CTA serves
    // several query heads) + one dense record per query head
    return (4 * (int64_t)num_ctas + 2 * (int64_t)B * Hq) * (int64_t)(d + kPS);
}

static int check_decode_args(const char *fn, int B, int Hq, int Hkv, int d, int M, int nbits,
                             int num_ctas, int64_t ld_tok) {
    PQKV_CHECK_ARG(geometry_ok(d, M, nbits), "%s: bad geometry", fn);
    PQKV_CHECK_ARG(B >= 0 && Hq > 0 && Hkv > 0 && Hq % Hkv == 0,
                   "%s: Hq must be a positive multiple of Hkv", fn);
    PQKV_CHECK_ARG(num_ctas > 0 && num_ctas <= (1 << 20), "%s: bad num_ctas", fn);
    PQKV_CHECK_ARG(ld_tok >= 0, "%s: bad ld_tok", fn);
    PQKV_CHECK_ARG(d <= GMAXD, "%s: d > %d unsupported", fn, GMAXD);
    return PQKV_OK;
}

#ifndef PQKV_SHARE
#define PQKV_SHARE 1
#endif
#ifndef PQKV_GQA2_WARPS
#define PQKV_GQA2_WARPS 12
#endif
#ifndef PQKV_F16_WARPS
#define PQKV_F16_WARPS 12
#endif
#ifndef PQKV_F16_GROUP
#define PQKV_F16_GROUP 2
#endif
#ifndef PQKV_GQA2_GROUP
#define PQKV_GQA2_GROUP 2
#endif
template <bool kLutFromQ, bool kHalfCV = false, int HG = 1, int W = fast::WARPS,
          int GROUP = fast::GROUP, bool kHalfLut = false>
static int launch_fast(const fast::Args &args, bool pdl, cudaStream_t st, const char *fn) {
    static int attr_set[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    auto kern = fast::decode_partials_m64b8<kLutFromQ, kHalfCV, HG, W, GROUP, kHalfLut>;
    if (dev >= 64 || !attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             fast::SMEM_BYTES);
        if (e != cudaSuccess) return fail(PQKV_ECUDA, "%s: %s", fn, cudaGetErrorString(e));
        if (dev < 64) attr_set[dev] = 1;
    }
#ifdef PQKV_TRACE
    static int trace_seq = 0;
    const_cast<fast::Args &>(args).trace_id = trace_seq++;
#endif
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(args.num_ctas);
    cfg.blockDim = dim3(W * 32);
    cfg.dynamicSmemBytes = fast::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args);
    if (e != cudaSuccess) return fail(PQKV_ECUDA, "%s: %s", fn, cudaGetErrorString(e));
    return launch_status(fn);
}

#ifndef PQKV_GQA4_WARPS
#define PQKV_GQA4_WARPS 12
#endif
template <int W>
static int launch_gqa4(const fast::Args &args, bool pdl, cudaStream_t st, const char *fn) {
    static int attr_set[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    auto kern = fast::decode_gqa4_f16<W>;
    if (dev >= 64 || !attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             fast::SMEM_BYTES);
        if (e != cudaSuccess) return fail(PQKV_ECUDA, "%s: %s", fn, cudaGetErrorString(e));
        if (dev < 64) attr_set[dev] = 1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(args.num_ctas);
    cfg.blockDim = dim3(W * 32);
    cfg.dynamicSmemBytes = fast::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args);
    if (e != cudaSuccess) return fail(PQKV_ECUDA, "%s: %s", fn, cudaGetErrorString(e));
    return launch_status(fn);
}

#ifndef PQKV_GQA_PAIR_WARPS
#define PQKV_GQA_PAIR_WARPS 12
#endif
// exact GQA (group a multiple of 4): clusters of two CTAs; the grid is the
// even number of CTAs that can be co-resident as pairs
template <int W>
static int launch_gqa_pair(fast::Args args, bool pdl, cudaStream_t st, const char *fn) {
    static int attr_set[64] = {0}, max_pairs[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    auto kern = fast::decode_gqa_pair<W>;
    const int smem = fast::gp::smem_bytes(W);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(W * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    if (dev >= 64 || !attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return fail(PQKV_ECUDA, "%s: %s", fn, cudaGetErrorString(e));
        int n = 0;
        cfg.gridDim = dim3(2 * 512);
        cfg.numAttrs = 1;
        e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
        if (e != cudaSuccess || n <= 0)
            return fail(PQKV_ECUDA, "%s: no co-resident CTA pairs (%s)", fn, cudaGetErrorString(e));
        if (dev < 64) {
            attr_set[dev] = 1;
            max_pairs[dev] = n;
        }
    }
    const int pairs = std::min(args.num_ctas / 2, dev < 64 ? max_pairs[dev] : args.num_ctas / 2);
    if (pairs < 1) return fail(PQKV_EINVAL, "%s: the exact GQA path needs num_ctas >= 2", fn);
    args.num_ctas = 2 * pairs;
    cfg.gridDim = dim3(args.num_ctas);
    cfg.numAttrs = pdl ? 2 : 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args);
    if (e != cudaSuccess) return fail(PQKV_ECUDA, "%s: %s", fn, cudaGetErrorString(e));
    return launch_status(fn);
}

static fast::Args fast_args(const float *q, float scale, const float *ck, const float *lut, int B,
                            int Hq, int Hkv, const void *codes_k, const void *codes_v,
                            int64_t ld_tok, const int32_t *n_q, const float *cb_v, int num_ctas,
                            float *partials) {
    fast::Args a = {};
    a.q = q;
    a.scale = scale;
    a.ck = ck;
    a.lut = lut;
    a.B = B;
    a.Hq = Hq;
    a.Hkv = Hkv;
    a.codes_k = (const uint8_t *)codes_k;
    a.codes_v = (const uint8_t *)codes_v;
    a.ld_tok = ld_tok;
    a.n_q = n_q;
    a.cv = cb_v;
    a.num_ctas = num_ctas;
    a.parts = partials;
    return a;
}

static int launch_generic(const float *lut, int B, int Hq, int Hkv, const void *codes_k,
                          const void *codes_v, int64_t ld_tok, const int32_t *n_q,
                          const float *cb_v, int d, int M, int nbits, int num_ctas,
                          float *partials, cudaStream_t st) {
    if (nbits <= 8)
        decode_partials_generic<uint8_t><<<num_ctas, GT, 0, st>>>(
            lut, B, Hq, Hkv, (const uint8_t *)codes_k, (const uint8_t *)codes_v, ld_tok, n_q, cb_v,
            d, M, 1 << nbits, num_ctas, partials);
    else
        decode_partials_generic<uint16_t><<<num_ctas, GT, 0, st>>>(
            lut, B, Hq, Hkv, (const uint16_t *)codes_k, (const uint16_t *)codes_v, ld_tok, n_q,
            cb_v, d, M, 1 << nbits, num_ctas, partials);
    return launch_status("pqkv_decode_partials");
}

extern "C" int pqkv_decode_partials(const float *q, float scale, const float *cb_k, float *lut_ws,
                                    int B, int Hq, int Hkv, const void *codes_k,
                                    const void *codes_v, int64_t ld_tok, const int32_t *n_q,
                                    const float *cb_v, int d, int M, int nbits, int num_ctas,
                                    float *partials, void *stream) {
    int rc = check_decode_args("pqkv_decode_partials", B, Hq, Hkv, d, M, nbits, num_ctas, ld_tok);
    if (rc) return rc;
    if (B == 0) return PQKV_OK;
    PQKV_CHECK_ARG(q && cb_k && codes_k && codes_v && n_q && cb_v && partials,
                   "pqkv_decode_partials: null pointer");
    cudaStream_t st = as_stream(stream);
    if (is_fast_geometry(d, M, nbits))
        return launch_fast<true>(fast_args(q, scale, cb_k, nullptr, B, Hq, Hkv, codes_k, codes_v,
                                           ld_tok, n_q, cb_v, num_ctas, partials),
                                 false, st, "pqkv_decode_partials");
    PQKV_CHECK_ARG(lut_ws != nullptr, "pqkv_decode_partials: this geometry needs lut_ws");
    rc = pqkv_build_lut(q, (int64_t)B * Hq, d, cb_k, M, nbits, scale, lut_ws, stream);
    if (rc) return rc;
    return launch_generic(lut_ws, B, Hq, Hkv, codes_k, codes_v, ld_tok, n_q, cb_v, d, M, nbits,
                          num_ctas, partials, st);
}

extern "C" int pqkv_decode_partials_lut(const float *lut, int B, int Hq, int Hkv,
                                        const void *codes_k, const void *codes_v, int64_t ld_tok,
                                        const int32_t *n_q, const float *cb_v, int d, int M,
                                        int nbits, int num_ctas, float *partials, void *stream) {
    int rc = check_decode_args("pqkv_decode_partials_lut", B, Hq, Hkv, d, M, nbits, num_ctas,
                               ld_tok);
    if (rc) return rc;
    if (B == 0) return PQKV_OK;
    PQKV_CHECK_ARG(lut && codes_k && codes_v && n_q && cb_v && partials,
                   "pqkv_decode_partials_lut: null pointer");
    cudaStream_t st = as_stream(stream);
    if (is_fast_geometry(d, M, nbits))
        return launch_fast<false>(fast_args(nullptr, 0.f, nullptr, lut, B, Hq, Hkv, codes_k,
                                            codes_v, ld_tok, n_q, cb_v, num_ctas, partials),
                                  false, st, "pqkv_decode_partials_lut");
    return launch_generic(lut, B, Hq, Hkv, codes_k, codes_v, ld_tok, n_q, cb_v, d, M, nbits,
                          num_ctas, partials, st);
}

extern "C" int pqkv_decode_finish(const float *partials, int num_ctas, int B, int Hq, int Hkv,
                                  int d, const int32_t *n_q, const float *q, float scale,
                                  const float *recent_k, const float *recent_v, int64_t ld_recent,
                                  const int32_t *n_recent, const float *k_cur, const float *v_cur,
                                  float *out, float *lse, float *merged, void *stream) {
    PQKV_CHECK_ARG(d > 0 && d <= FMAXD, "pqkv_decode_finish: d out of range");
    PQKV_CHECK_ARG(B >= 0 && Hq > 0 && Hkv > 0 && Hq % Hkv == 0,
                   "pqkv_decode_finish: Hq must be a positive multiple of Hkv");
    PQKV_CHECK_ARG(ld_recent >= 0 && ld_recent < (1 << 16), "pqkv_decode_finish: bad ld_recent");
    PQKV_CHECK_ARG((k_cur == nullptr) == (v_cur == nullptr),
                   "pqkv_decode_finish: k_cur and v_cur go together");
    PQKV_CHECK_ARG((recent_k == nullptr) == (recent_v == nullptr),
                   "pqkv_decode_finish: recent_k and recent_v go together");
    if (B == 0) return PQKV_OK;
    PQKV_CHECK_ARG(partials == nullptr || (n_q != nullptr && num_ctas > 0),
                   "pqkv_decode_finish: partials need n_q and num_ctas");
    PQKV_CHECK_ARG(q != nullptr || (k_cur == nullptr && recent_k == nullptr),
                   "pqkv_decode_finish: dense rows need q");
    const int dch = dense_chunk(d);
    const size_t smem = sizeof(float) * (size_t)(2 * dch * d + dch);
    decode_finish_kernel<<<B * Hq, FT, smem, as_stream(stream)>>>(
        partials, num_ctas, B, Hq, Hkv, d, n_q, q, scale, recent_k, recent_v, ld_recent, n_recent,
        k_cur, v_cur, out, lse, merged, dch);
    return launch_status("pqkv_decode_finish");
}

extern "C" int pqkv_decode_attention(
    const float *q, float scale, const float *cb_k, float *lut_ws, int B, int Hq, int Hkv,
    const void *codes_k, const void *codes_v, int64_t ld_tok, const int32_t *n_q,
    const float *cb_v, int d, int M, int nbits, const float *recent_k, const float *recent_v,
    int64_t ld_recent, const int32_t *n_recent, const float *k_cur, const float *v_cur,
    int num_ctas, float *partials, int32_t *counters, float *out, float *lse, float *merged,
    int flags, void *stream) {
    int rc = check_decode_args("pqkv_decode_attention", B, Hq, Hkv, d, M, nbits, num_ctas, ld_tok);
    if (rc) return rc;
    PQKV_CHECK_ARG(ld_recent >= 0 && ld_recent < (1 << 16),
                   "pqkv_decode_attention: bad ld_recent");
    PQKV_CHECK_ARG((k_cur == nullptr) == (v_cur == nullptr),
                   "pqkv_decode_attention: k_cur and v_cur go together");
    PQKV_CHECK_ARG((recent_k == nullptr) == (recent_v == nullptr),
                   "pqkv_decode_attention: recent_k and recent_v go together");
    PQKV_CHECK_ARG((flags & ~(PQKV_DECODE_PDL | PQKV_DECODE_STATIC_CODEBOOKS |
                              PQKV_DECODE_F16_VALUE_CODEBOOK | PQKV_DECODE_EARLY_CODES |
                              PQKV_DECODE_ONE_HEAD_PER_CTA | PQKV_DECODE_F16_KEY_TABLE |
                              PQKV_DECODE_KEY_TABLE_PAIRS | PQKV_DECODE_APPEND_RECENT)) == 0,
                   "pqkv_decode_attention: unknown flags");
    PQKV_CHECK_ARG(!(flags & PQKV_DECODE_APPEND_RECENT) ||
                       (B == 1 && Hq == 1 && Hkv == 1 && is_fast_geometry(d, M, nbits) &&
                        recent_k && n_recent && k_cur &&
                        !(flags & PQKV_DECODE_F16_VALUE_CODEBOOK)),
                   "pqkv_decode_attention: PQKV_DECODE_APPEND_RECENT needs one head (m64b8, "
                   "fp32 values) with a recent ring, its length and the current token");
    if (B == 0) return PQKV_OK;
    PQKV_CHECK_ARG(q && cb_k && codes_k && codes_v && n_q && cb_v && partials,
                   "pqkv_decode_attention: null pointer");
    cudaStream_t st = as_stream(stream);
    if (!is_fast_geometry(d, M, nbits)) {
        // generic geometries: tables, split partials, then the finish kernel
        rc = pqkv_decode_partials(q, scale, cb_k, lut_ws, B, Hq, Hkv, codes_k, codes_v, ld_tok,
                                  n_q, cb_v, d, M, nbits, num_ctas, partials, stream);
        if (rc) return rc;
        return pqkv_decode_finish(partials, num_ctas, B, Hq, Hkv, d, n_q, q, scale, recent_k,
                                  recent_v, ld_recent, n_recent, k_cur, v_cur, out, lse, merged,
                                  stream);
    }
    PQKV_CHECK_ARG(counters != nullptr, "pqkv_decode_attention: null counters");
    fast::Args a = fast_args(q, scale, cb_k, nullptr, B, Hq, Hkv, codes_k, codes_v, ld_tok, n_q,
                             cb_v, num_ctas, partials);
    a.counters = counters;
    a.recent_k = recent_k;
    a.recent_v = recent_v;
    a.ld_recent = ld_recent;
    a.n_recent = n_recent;
    a.k_cur = k_cur;
    a.v_cur = v_cur;
    a.out = out;
    a.lse = lse;
    a.merged = merged;
    a.early_cv = (flags & PQKV_DECODE_STATIC_CODEBOOKS) ? 1 : 0;
    a.early_codes = (flags & PQKV_DECODE_EARLY_CODES) ? 1 : 0;
    a.append = (flags & PQKV_DECODE_APPEND_RECENT) ? 1 : 0;
    const bool pdl = (flags & PQKV_DECODE_PDL) != 0;
    // GQA: the CTAs serving the virtual heads of one KV head stream its codes
    // concurrently (one DRAM fetch, L2 hits for the others) -- P = virtual
    // heads per KV head, reduced until it divides the grid
    const int group = Hq / Hkv;
    // four query heads per CTA: the packed fp16 key table with a group that
    // is a multiple of 4 (unless pairs are asked for)
    const bool four = (flags & PQKV_DECODE_F16_VALUE_CODEBOOK) &&
                      (flags & PQKV_DECODE_F16_KEY_TABLE) && group % 4 == 0 &&
                      !(flags & (PQKV_DECODE_ONE_HEAD_PER_CTA | PQKV_DECODE_KEY_TABLE_PAIRS));
    {
        const bool two = (flags & PQKV_DECODE_F16_VALUE_CODEBOOK) && group % 2 == 0 &&
                         !(flags & PQKV_DECODE_ONE_HEAD_PER_CTA);
        int P = PQKV_SHARE ? group / (four ? 4 : two ? 2 : 1) : 1;
        while (P > 1 && (num_ctas % P != 0 || P > 16)) P = (P % 2 == 0) ? P / 2 : 1;
        a.share = P;
    }
    if (four)
        return launch_gqa4<PQKV_GQA4_WARPS>(a, pdl, st, "pqkv_decode_attention");
    // exact path, a group that is a multiple of 4: CTA pairs serve four query
    // heads each (the subspace halves split across the pair)
    if (!(flags & (PQKV_DECODE_F16_VALUE_CODEBOOK | PQKV_DECODE_ONE_HEAD_PER_CTA)) &&
        group % 4 == 0 && num_ctas >= 2) {
        a.share = 1;
        return launch_gqa_pair<PQKV_GQA_PAIR_WARPS>(a, pdl, st, "pqkv_decode_attention");
    }
    if (flags & PQKV_DECODE_F16_VALUE_CODEBOOK) {
        // even GQA groups: one CTA serves two query heads of a KV head
        if ((Hq / Hkv) % 2 == 0 && !(flags & PQKV_DECODE_ONE_HEAD_PER_CTA)) {
            if (flags & PQKV_DECODE_F16_KEY_TABLE)
                return launch_fast<true, true, 2, PQKV_GQA2_WARPS, PQKV_GQA2_GROUP, true>(
                    a, pdl, st, "pqkv_decode_attention");
            return launch_fast<true, true, 2, PQKV_GQA2_WARPS, PQKV_GQA2_GROUP>(
                a, pdl, st, "pqkv_decode_attention");
        }
        return launch_fast<true, true, 1, PQKV_F16_WARPS, PQKV_F16_GROUP>(a, pdl, st,
                                                                          "pqkv_decode_attention");
    }
    return launch_fast<true, false>(a, pdl, st, "pqkv_decode_attention");
}

extern "C" int pqkv_merge_partials(const float *parts, int n_parts, int64_t n_heads, int d,
                                   float *out, float *lse, float *merged, void *stream) {
    PQKV_CHECK_ARG(d > 0 && d <= FMAXD && n_parts >= 0 && n_heads >= 0,
                   "pqkv_merge_partials: bad sizes");
    if (n_heads == 0) return PQKV_OK;
    PQKV_CHECK_ARG(parts || n_parts == 0, "pqkv_merge_partials: null parts");
    merge_partials_kernel<<<(unsigned)n_heads, FT, 0, as_stream(stream)>>>(parts, n_parts, n_heads,
                                                                           d, out, lse, merged);
    return launch_status("pqkv_merge_partials");
}

// ---- decode_step's per-token path for one cached head -----------------------
#ifndef PQKV_STEP_FUSED_APPEND
#define PQKV_STEP_FUSED_APPEND 1  // the append rides in the decode launch's finisher
#endif
struct pqkv_step_plan {
    const float *cb_k, *cb_v;
    const void *codes_k, *codes_v;
    int64_t ld_tok;
    int32_t *lens;
    float scale;
    int d, M, nbits, num_ctas;
    float *partials;
    int32_t *counters;
};

extern "C" int pqkv_step_plan_create(const float *cb_k, const float *cb_v, const void *codes_k,
                                     const void *codes_v, int64_t ld_tok, int32_t *lens,
                                     float scale, int d, int M, int nbits, int num_ctas,
                                     float *partials, int32_t *counters, void **plan) {
    PQKV_CHECK_ARG(plan && cb_k && cb_v && codes_k && codes_v && lens && partials && counters,
                   "pqkv_step_plan_create: null pointer");
    PQKV_CHECK_ARG(is_fast_geometry(d, M, nbits), "pqkv_step_plan_create: m64b8 only");
    PQKV_CHECK_ARG(num_ctas > 0 && ld_tok >= 0, "pqkv_step_plan_create: bad sizes");
    auto *p = new pqkv_step_plan{cb_k, cb_v, codes_k, codes_v, ld_tok, lens, scale, d, M,
                                 nbits, num_ctas, partials, counters};
    *plan = p;
    return PQKV_OK;
}

extern "C" int pqkv_step_plan_destroy(void *plan) {
    delete static_cast<pqkv_step_plan *>(plan);
    return PQKV_OK;
}

extern "C" int pqkv_step_run(void *plan, const float *q, const float *k_cur, const float *v_cur,
                             float *recent_k, float *recent_v, int64_t ld_recent, int num_ctas,
                             float *out, void *stream) {
    PQKV_CHECK_ARG(plan && q && k_cur && v_cur && recent_k && recent_v && out,
                   "pqkv_step_run: null pointer");
    const auto *p = static_cast<const pqkv_step_plan *>(plan);
    // a short context needs few CTAs: each pays the table build, and the
    // last arriver merges one record per CTA
    const int nc = num_ctas > 0 ? std::min(num_ctas, p->num_ctas) : p->num_ctas;
    int rc = pqkv_decode_attention(q, p->scale, p->cb_k, nullptr, 1, 1, 1, p->codes_k, p->codes_v,
                                   p->ld_tok, p->lens, p->cb_v, p->d, p->M, p->nbits, recent_k,
                                   recent_v, ld_recent, p->lens + 1, k_cur, v_cur, nc,
                                   p->partials, p->counters, out, nullptr, nullptr,
                                   PQKV_STEP_FUSED_APPEND ? PQKV_DECODE_APPEND_RECENT : 0, stream);
    if (rc || PQKV_STEP_FUSED_APPEND) return rc;
    return pqkv_append_recent(k_cur, v_cur, recent_k, recent_v, p->lens, p->d, stream);
}
