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
// decode_partials_m64b8 (the fast path, d=128 M=64 nbits=8):
//   * persistent grid, one 512-thread CTA per SM; the flattened token space
//     of all heads is cut into equal chunks (common.cuh FlatMap);
//   * shared memory: the head's key LUT, centroid-major [256][64] fp32
//     (64 KiB), and the value codebook as two [256][32] float2 halves
//     (128 KiB, loaded once per CTA);
//   * a warp handles 8 tokens per step: lane = (token slot, 16-subspace
//     quarter) and loads the 16 K-code and 16 V-code bytes of its quarter with
//     one 128-bit load each (coalesced: the warp reads 2 x 512 contiguous B);
//   * each lane rotates its 16 code bytes by a lane constant r so that at
//     every unrolled step the 32 lanes touch 32 distinct subspaces mod 32:
//     the LUT gather (bank = subspace mod 32) and the 64-bit codebook gather
//     (8-byte slot = subspace mod 16 per half-warp) are bank-conflict free
//     for ANY code values;
//   * one PRMT per code byte forms the shared-memory byte address
//     (code << 8 | lane offset | half << 16);
//   * the 4 lanes of a token combine their partial scores with 2 shuffles;
//     each token slot keeps its own online-softmax state (m, l) and 32 fp32
//     value accumulators (its quarter's 16 subspaces x dsub 2);
//   * epilogue: slot partials are rescaled to the CTA max and summed through
//     shared memory into one (m, l, acc[128]) record per segment.
#include "common.cuh"

namespace pqkv {
namespace {

constexpr int kPS = PQKV_PARTIAL_HEADER;  // record = [m, l, 0, 0, acc[d]]

// ============================================================ fast path ====
namespace fast {
constexpr int M = 64, KSUB = 256, D = 128;
constexpr int WARPS = 16, NT = WARPS * 32;
constexpr int LUT_BYTES = KSUB * M * 4;     // 65536
constexpr int CV_BYTES = KSUB * M * 2 * 4;  // 131072
constexpr int SMEM_BYTES = LUT_BYTES + CV_BYTES + (2 * WARPS + 4 * D) * 4;
constexpr int PREFETCH = 2;  // groups in flight per warp beyond the current one

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

__device__ __forceinline__ float lds_lut(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1+0x400];" : "=f"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ unsigned long long lds_cv(uint32_t a) {
    unsigned long long v;
    asm volatile("ld.shared.b64 %0, [%1+0x10400];" : "=l"(v) : "r"(a));
    return v;
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

// rotate the 16 bytes (w0..w3) so that out.byte[j] = in.byte[(j + r) & 15]
__device__ __forceinline__ void rotate16(const uint4 in, int r, uint32_t (&o)[4]) {
    uint32_t w0 = in.x, w1 = in.y, w2 = in.z, w3 = in.w;
    if (r & 4) {
        const uint32_t t = w0;
        w0 = w1; w1 = w2; w2 = w3; w3 = t;
    }
    if (r & 8) {
        uint32_t t = w0; w0 = w2; w2 = t;
        t = w1; w1 = w3; w3 = t;
    }
    const uint32_t sh = (uint32_t)(r & 3) * 8u;
    o[0] = __funnelshift_r(w0, w1, sh);
    o[1] = __funnelshift_r(w1, w2, sh);
    o[2] = __funnelshift_r(w2, w3, sh);
    o[3] = __funnelshift_r(w3, w0, sh);
}

// PRMT selector for rotated byte j: [offset byte (j&1) of b, code byte (j&3)
// of a, byte 2 of b, byte 3 of b]
__device__ __forceinline__ constexpr uint32_t sel_for(int j) {
    return (uint32_t)(4 + (j & 1)) | ((uint32_t)(j & 3) << 4) | (6u << 8) | (7u << 12);
}

__global__ void __launch_bounds__(NT, 1)
    decode_partials_m64b8(const float *__restrict__ lut_g, int B, int Hq, int Hkv,
                          const uint8_t *__restrict__ codes_k, const uint8_t *__restrict__ codes_v,
                          int64_t ld_tok, const int32_t *__restrict__ n_q,
                          const float *__restrict__ cv_g, int num_ctas,
                          float *__restrict__ parts) {
    extern __shared__ __align__(128) unsigned char smem[];
    float *lut_s = reinterpret_cast<float *>(smem);
    float *red_m = reinterpret_cast<float *>(smem + LUT_BYTES + CV_BYTES);
    float *red_l = red_m + WARPS;
    float(*colsum)[D] = reinterpret_cast<float(*)[D]>(red_l + WARPS);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
    if ((sbase & 0xFFFFFFu) != kDynBase) __trap();  // layout assumption (see lds_lut)
    const uint32_t cta_byte = sbase & 0xFF000000u;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q4 = lane & 3, slot = lane >> 2;
    const int r = ((lane & 15) + (lane >> 4)) & 15;

    // lane-constant address bytes (see header comment)
    uint32_t packK[8], packV[8];
#pragma unroll
    for (int jp = 0; jp < 8; ++jp) {
        uint32_t pk = 0, pv = 0;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int j = 2 * jp + e;
            const int i = 16 * q4 + ((j + r) & 15);
            pk |= (uint32_t)(i * 4) << (8 * e);
            pv |= (uint32_t)((i & 31) * 8) << (8 * e);
        }
        packK[jp] = pk | cta_byte;
        packV[jp] = pv | ((uint32_t)(q4 >> 1) << 16) | cta_byte;
    }

    // value codebook: once per CTA (already in the [half][c][32] layout)
    {
        const float4 *src = reinterpret_cast<const float4 *>(cv_g);
        float4 *dst = reinterpret_cast<float4 *>(smem + LUT_BYTES);
#pragma unroll 4
        for (int k = tid; k < CV_BYTES / 16; k += NT) dst[k] = __ldg(src + k);
    }

    const FlatMap fm = flat_map(n_q, B, Hq, num_ctas);
    const int cta = blockIdx.x;
    int64_t pos = (int64_t)cta * fm.chunk;
    const int64_t end = min(pos + fm.chunk, fm.total);
    const int group = Hq / Hkv;

    while (pos < end) {
        int bh, t0, len;
        locate(n_q, B, Hq, pos, &bh, &t0, &len);
        const int n = (int)min((int64_t)(len - t0), end - pos);
        const int b = bh / Hq, hq = bh - b * Hq, hkv = hq / group;

        __syncthreads();  // previous segment's epilogue is done with lut_s
        {
            const float4 *src = reinterpret_cast<const float4 *>(lut_g + (int64_t)bh * KSUB * M);
            float4 *dst = reinterpret_cast<float4 *>(smem);
#pragma unroll 4
            for (int k = tid; k < LUT_BYTES / 16; k += NT) dst[k] = __ldg(src + k);
        }
        __syncthreads();

        const int64_t head_off = ((int64_t)b * Hkv + hkv) * ld_tok * M;
        const uint8_t *kb = codes_k + head_off + (int64_t)t0 * M + q4 * 16;
        const uint8_t *vb = codes_v + head_off + (int64_t)t0 * M + q4 * 16;
        const int ngroups = (n + 7) >> 3;

        float m = -INFINITY, l = 0.f;
        unsigned long long acc[16];  // float2 per rotated subspace
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[k] = 0ull;

        uint4 kr[PREFETCH + 1], vr[PREFETCH + 1];
        bool ok[PREFETCH + 1];
#pragma unroll
        for (int s = 0; s <= PREFETCH; ++s) {
            const int t = (warp + s * WARPS) * 8 + slot;
            ok[s] = t < n;
            kr[s] = ok[s] ? ld_stream(kb + (int64_t)t * M) : make_uint4(0, 0, 0, 0);
            vr[s] = ok[s] ? ld_stream(vb + (int64_t)t * M) : make_uint4(0, 0, 0, 0);
        }

        for (int g = warp; g < ngroups; g += WARPS) {
            const uint4 kc = kr[0], vc = vr[0];
            const bool valid = ok[0];
#pragma unroll
            for (int s = 0; s < PREFETCH; ++s) {
                kr[s] = kr[s + 1];
                vr[s] = vr[s + 1];
                ok[s] = ok[s + 1];
            }
            {
                const int t = (g + (PREFETCH + 1) * WARPS) * 8 + slot;
                ok[PREFETCH] = t < n;
                kr[PREFETCH] = ok[PREFETCH] ? ld_stream(kb + (int64_t)t * M) : make_uint4(0, 0, 0, 0);
                vr[PREFETCH] = ok[PREFETCH] ? ld_stream(vb + (int64_t)t * M) : make_uint4(0, 0, 0, 0);
            }

            uint32_t RK[4], RV[4];
            rotate16(kc, r, RK);
            rotate16(vc, r, RV);

            float sp[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint32_t a = __byte_perm(RK[j >> 2], packK[j >> 1], sel_for(j));
                sp[j & 3] += lds_lut(a);
            }
            float s = (sp[0] + sp[1]) + (sp[2] + sp[3]);
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            s += __shfl_xor_sync(0xffffffffu, s, 2);

            if (valid) {
                if (s > m) {
                    const float f = fast_exp2((m - s) * kLog2e);
                    l *= f;
#pragma unroll
                    for (int k = 0; k < 16; ++k) fmul2(acc[k], f);
                    m = s;
                }
                const float p = fast_exp2((s - m) * kLog2e);
                l += p;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const uint32_t a = __byte_perm(RV[j >> 2], packV[j >> 1], sel_for(j));
                    ffma2(acc[j], p, lds_cv(a));
                }
            }
        }

        // ---- epilogue: one (m, l, acc) record for this (CTA, head) segment
        float mw = m;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, off));
        if (lane == 0) red_m[warp] = mw;
        __syncthreads();  // all warps are past the main loop: lut_s is free
        float Mx = red_m[0];
#pragma unroll
        for (int w = 1; w < WARPS; ++w) Mx = fmaxf(Mx, red_m[w]);
        const float f = (m == -INFINITY) ? 0.f : fast_exp2((m - Mx) * kLog2e);
        float lw = (q4 == 0) ? l * f : 0.f;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) lw += __shfl_xor_sync(0xffffffffu, lw, off);
        if (lane == 0) red_l[warp] = lw;
        float *rows = lut_s + (warp * 8 + slot) * D;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int i = 16 * q4 + ((j + r) & 15);
            const float2 a = unpack2(acc[j]);
            rows[2 * i] = a.x * f;
            rows[2 * i + 1] = a.y * f;
        }
        __syncthreads();
        {
            const int col = tid & (D - 1), part = tid >> 7;
            float cs = 0.f;
#pragma unroll 8
            for (int rr = part * 32; rr < part * 32 + 32; ++rr) cs += lut_s[rr * D + col];
            colsum[part][col] = cs;
        }
        __syncthreads();
        if (tid < D) {
            float *rec = parts + ((int64_t)cta + bh) * (D + kPS);
            rec[kPS + tid] = (colsum[0][tid] + colsum[1][tid]) + (colsum[2][tid] + colsum[3][tid]);
            if (tid == 0) {
                float L = 0.f;
#pragma unroll
                for (int w = 0; w < WARPS; ++w) L += red_l[w];
                rec[0] = Mx;
                rec[1] = L;
                rec[2] = 0.f;
                rec[3] = 0.f;
            }
        }
        pos += n;
    }
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
    const FlatMap fm = flat_map(n_q, B, Hq, num_ctas);
    const int cta = blockIdx.x;
    int64_t pos = (int64_t)cta * fm.chunk;
    const int64_t end = min(pos + fm.chunk, fm.total);
    const int group = Hq / Hkv;

    while (pos < end) {
        int bh, t0, len;
        locate(n_q, B, Hq, pos, &bh, &t0, &len);
        const int n = (int)min((int64_t)(len - t0), end - pos);
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
        pos += n;
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

__global__ void __launch_bounds__(FT)
    decode_finish_kernel(const float *__restrict__ parts, int num_ctas, int B, int Hq, int Hkv,
                         int d, const int32_t *__restrict__ n_q, const float *__restrict__ q,
                         float scale, const float *__restrict__ recent_k,
                         const float *__restrict__ recent_v, int64_t ld_recent,
                         const int32_t *__restrict__ n_recent, const float *__restrict__ k_cur,
                         const float *__restrict__ v_cur, float *__restrict__ out,
                         float *__restrict__ lse, float *__restrict__ merged) {
    extern __shared__ float sc[];  // dense scores, ld_recent + 1
    __shared__ float dense_acc_dummy;
    (void)dense_acc_dummy;
    const int bh = blockIdx.x;
    const int b = bh / Hq, hq = bh - b * Hq, hkv = hq / (Hq / Hkv);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    float m = -INFINITY, l = 0.f;
    float acc[FMAXD / FT];
#pragma unroll
    for (int k = 0; k < FMAXD / FT; ++k) acc[k] = 0.f;

    // 1. quantized partials of this head, in CTA order (deterministic)
    if (parts != nullptr && n_q != nullptr) {
        const FlatMap fm = flat_map(n_q, B, Hq, num_ctas);
        int len;
        const int64_t s0 = head_start(n_q, Hq, bh, &len);
        if (len > 0) {
            const int64_t c_first = s0 / fm.chunk, c_last = (s0 + len - 1) / fm.chunk;
            for (int64_t c = c_first; c <= c_last; ++c) {
                const float *rec = parts + (c + bh) * (int64_t)(d + kPS);
                merge_into(m, l, acc, rec[0], rec[1], rec + kPS, d);
            }
        }
    }

    // 2. dense partial over recent rows [0, n_recent[b]) + current token
    const int nr = (n_recent != nullptr && recent_k != nullptr) ? max(n_recent[b], 0) : 0;
    const int rows = nr + (k_cur != nullptr ? 1 : 0);
    if (rows > 0) {
        const float *qh = q + (int64_t)bh * d;
        const int64_t rbase = ((int64_t)b * Hkv + hkv) * ld_recent * d;
        for (int row = warp; row < rows; row += FT / 32) {
            const float *kr = row < nr ? recent_k + rbase + (int64_t)row * d
                                       : k_cur + ((int64_t)b * Hkv + hkv) * d;
            float dot = 0.f;
            for (int j = lane; j < d; j += 32) dot = fmaf(qh[j], kr[j], dot);
            for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
            if (lane == 0) sc[row] = scale * dot;
        }
        __syncthreads();
        float md = -INFINITY;
        for (int row = 0; row < rows; ++row) md = fmaxf(md, sc[row]);
        float ld = 0.f;
        float dacc[FMAXD / FT];
#pragma unroll
        for (int k = 0; k < FMAXD / FT; ++k) dacc[k] = 0.f;
        for (int row = 0; row < rows; ++row) {
            const float p = expf(sc[row] - md);
            ld += p;
            const float *vr = row < nr ? recent_v + rbase + (int64_t)row * d
                                       : v_cur + ((int64_t)b * Hkv + hkv) * d;
#pragma unroll
            for (int k = 0; k < FMAXD / FT; ++k) {
                const int j = tid + k * FT;
                if (j < d) dacc[k] = fmaf(p, vr[j], dacc[k]);
            }
        }
        // merge the dense partial (register-resident) into (m, l, acc)
        if (l == 0.f) {
            m = md;
            l = ld;
#pragma unroll
            for (int k = 0; k < FMAXD / FT; ++k) acc[k] = dacc[k];
        } else {
            const float mm = fmaxf(m, md);
            const float wa = expf(m - mm), wb = expf(md - mm);
            l = l * wa + ld * wb;
#pragma unroll
            for (int k = 0; k < FMAXD / FT; ++k) acc[k] = acc[k] * wa + dacc[k] * wb;
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

extern "C" int64_t pqkv_partials_floats(int num_ctas, int B, int Hq, int d) {
    return ((int64_t)num_ctas + (int64_t)B * Hq) * (int64_t)(d + kPS);
}

extern "C" int pqkv_decode_partials(const float *lut, int B, int Hq, int Hkv, const void *codes_k,
                                    const void *codes_v, int64_t ld_tok, const int32_t *n_q,
                                    const float *cb_v, int d, int M, int nbits, int num_ctas,
                                    float *partials, void *stream) {
    PQKV_CHECK_ARG(geometry_ok(d, M, nbits), "pqkv_decode_partials: bad geometry");
    PQKV_CHECK_ARG(B >= 0 && Hq > 0 && Hkv > 0 && Hq % Hkv == 0,
                   "pqkv_decode_partials: Hq must be a positive multiple of Hkv");
    PQKV_CHECK_ARG(num_ctas > 0 && num_ctas <= (1 << 20), "pqkv_decode_partials: bad num_ctas");
    PQKV_CHECK_ARG(ld_tok >= 0, "pqkv_decode_partials: bad ld_tok");
    PQKV_CHECK_ARG(d <= GMAXD, "pqkv_decode_partials: d > %d unsupported", GMAXD);
    if (B == 0) return PQKV_OK;
    PQKV_CHECK_ARG(lut && codes_k && codes_v && n_q && cb_v && partials,
                   "pqkv_decode_partials: null pointer");
    cudaStream_t st = as_stream(stream);
    if (is_fast_geometry(d, M, nbits)) {
        static bool attr_set = false;
        if (!attr_set) {
            cudaError_t e = cudaFuncSetAttribute(fast::decode_partials_m64b8,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 fast::SMEM_BYTES);
            if (e != cudaSuccess)
                return fail(PQKV_ECUDA, "pqkv_decode_partials: %s", cudaGetErrorString(e));
            attr_set = true;
        }
        fast::decode_partials_m64b8<<<num_ctas, fast::NT, fast::SMEM_BYTES, st>>>(
            lut, B, Hq, Hkv, (const uint8_t *)codes_k, (const uint8_t *)codes_v, ld_tok, n_q, cb_v,
            num_ctas, partials);
    } else if (nbits <= 8) {
        decode_partials_generic<uint8_t><<<num_ctas, GT, 0, st>>>(
            lut, B, Hq, Hkv, (const uint8_t *)codes_k, (const uint8_t *)codes_v, ld_tok, n_q, cb_v,
            d, M, 1 << nbits, num_ctas, partials);
    } else {
        decode_partials_generic<uint16_t><<<num_ctas, GT, 0, st>>>(
            lut, B, Hq, Hkv, (const uint16_t *)codes_k, (const uint16_t *)codes_v, ld_tok, n_q,
            cb_v, d, M, 1 << nbits, num_ctas, partials);
    }
    return launch_status("pqkv_decode_partials");
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
    const size_t smem = sizeof(float) * (size_t)(ld_recent + 1);
    decode_finish_kernel<<<B * Hq, FT, smem, as_stream(stream)>>>(
        partials, num_ctas, B, Hq, Hkv, d, n_q, q, scale, recent_k, recent_v, ld_recent, n_recent,
        k_cur, v_cur, out, lse, merged);
    return launch_status("pqkv_decode_finish");
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
