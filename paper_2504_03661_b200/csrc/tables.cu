// Small per-step / per-load kernels: key lookup tables, the value-codebook
// re-layout for the fast path, reconstruct (test helper), the reference's
// lower-seam kernels (_kernels.py), and the library's error/version plumbing.
#include <cuda_fp16.h>

#include <cstdarg>

#include "common.cuh"

namespace pqkv {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    set_error(buf);
    return code;
}

namespace {

// build_key_lut (attention.py:70-83): lut[h][c][i] = scale * <q_i, C_K[i, c]>.
// Block = 32 centroids x all M subspaces of one head, written contiguously
// (centroid-major, the decode kernel's shared-memory image).
__global__ void __launch_bounds__(256) build_lut_kernel(const float *__restrict__ q, int d,
                                                        const float *__restrict__ cb_k, int M,
                                                        int ksub, float scale,
                                                        float *__restrict__ lut) {
    extern __shared__ float q_s[];
    const int h = blockIdx.y;
    const int dsub = d / M;
    for (int j = threadIdx.x; j < d; j += blockDim.x) q_s[j] = q[(int64_t)h * d + j];
    __syncthreads();
    const int c0 = blockIdx.x * 32;
    const int cn = min(32, ksub - c0);
    float *out = lut + ((int64_t)h * ksub + c0) * M;
    for (int idx = threadIdx.x; idx < cn * M; idx += blockDim.x) {
        const int c = c0 + idx / M, i = idx % M;
        const float *cr = cb_k + ((int64_t)i * ksub + c) * dsub;
        const float *qi = q_s + i * dsub;
        float acc = qi[0] * __ldg(cr);
        for (int j = 1; j < dsub; ++j) acc = fmaf(qi[j], __ldg(cr + j), acc);
        out[idx] = acc * scale;
    }
}

// Value codebook -> [half][c][32] float2 for the m64b8 decode kernel.
__global__ void prepare_cv_kernel(const float2 *__restrict__ cb_v, float2 *__restrict__ out) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // over (i, c)
    if (idx >= 64 * 256) return;
    const int i = idx >> 8, c = idx & 255;
    out[((i >> 5) * 256 + c) * 32 + (i & 31)] = cb_v[idx];
}

// Value codebook -> [c][half][32] half2 (round to nearest) for the fp16 mode:
// 256-byte rows, so the decode kernel forms the address with one PRMT.
__global__ void prepare_cv_f16_kernel(const float2 *__restrict__ cb_v, __half2 *__restrict__ out) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // over (i, c)
    if (idx >= 64 * 256) return;
    const int i = idx >> 8, c = idx & 255;
    out[(c * 2 + (i >> 5)) * 32 + (i & 31)] = __float22half2_rn(cb_v[idx]);
}

// Key codebook -> centroid-major [c][i] float2 for the in-kernel LUT build.
__global__ void prepare_ck_kernel(const float2 *__restrict__ cb_k, float2 *__restrict__ out) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // over (i, c)
    if (idx >= 64 * 256) return;
    const int i = idx >> 8, c = idx & 255;
    out[c * 64 + i] = cb_k[idx];
}

// Reference row layout <-> m64b8 decode layout (common.cuh), one byte per thread.
__global__ void relayout_kernel(const uint8_t *__restrict__ src, int64_t ld_src,
                                uint8_t *__restrict__ dst, int64_t ld_dst, int64_t n,
                                int64_t t_first, int to_decode) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * 64) return;
    const int64_t v = idx >> 6;
    const int i = (int)(idx & 63);
    const int pos = decode_layout_pos(i, t_first + v);
    if (to_decode)
        dst[v * ld_dst + pos] = src[v * ld_src + i];
    else
        dst[v * ld_dst + i] = src[v * ld_src + pos];
}

template <typename CT>
__global__ void reconstruct_kernel(const CT *__restrict__ codes, int64_t n, int64_t ld_codes,
                                   const float *__restrict__ cents, int d, int M, int ksub,
                                   float *__restrict__ out) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * d) return;
    const int64_t t = idx / d;
    const int j = (int)(idx - t * d);
    const int dsub = d / M, i = j / dsub, jj = j - i * dsub;
    const int c = codes[t * ld_codes + i];
    out[idx] = cents[((int64_t)i * ksub + c) * dsub + jj];
}

template <typename CT>
__global__ void score_codes_kernel(const float *__restrict__ lut, const CT *__restrict__ codes,
                                   int64_t n, int M, float *__restrict__ scores) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    float s = 0.f;
    for (int i = 0; i < M; ++i) s += __ldg(lut + (int64_t)codes[t * M + i] * M + i);
    scores[t] = s;
}

template <typename CT>
__global__ void accumulate_mass_kernel(const CT *__restrict__ codes, const float *__restrict__ p,
                                       int64_t n, int M, int ksub, float *__restrict__ h) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * M) return;
    const int64_t t = idx / M;
    const int i = (int)(idx - t * M);
    atomicAdd(h + (int64_t)i * ksub + codes[idx], p[t]);
}

// The reference's lower seam in float64, with its loop orders
// (_kernels.py:27-43): score s_t = sum_i lut[i][code[t,i]] summed over i in
// order from 0.0; mass h[i][c] = sum of p_t over t in token order.  One thread
// per token (score) / per bin (mass: the block stages a tile of column i's
// codes and weights, every bin thread scans it in order), so both are
// bit-identical to the numba loops given the same inputs.
template <typename CT>
__global__ void score_codes_f64_kernel(const double *__restrict__ lut, int ksub,
                                       const CT *__restrict__ codes, int64_t n, int M,
                                       double *__restrict__ scores) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    double s = 0.0;
    for (int i = 0; i < M; ++i) s += lut[(int64_t)i * ksub + codes[t * M + i]];
    scores[t] = s;
}

constexpr int kMassTile = 1024;
template <typename CT>
__global__ void accumulate_mass_f64_kernel(const CT *__restrict__ codes,
                                           const double *__restrict__ p, int64_t n, int M,
                                           int ksub, double *__restrict__ h) {
    __shared__ int cs[kMassTile];
    __shared__ double ps[kMassTile];
    const int i = blockIdx.y;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    double acc = 0.0;
    for (int64_t t0 = 0; t0 < n; t0 += kMassTile) {
        const int cnt = (int)min((int64_t)kMassTile, n - t0);
        __syncthreads();
        for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
            cs[k] = codes[(t0 + k) * M + i];
            ps[k] = p[t0 + k];
        }
        __syncthreads();
        if (c < ksub)
            for (int k = 0; k < cnt; ++k)
                if (cs[k] == c) acc += ps[k];
    }
    if (c < ksub) h[(int64_t)i * ksub + c] = acc;
}

// The reference API's float64 small ops (build_key_lut attention.py:70-83,
// dense_partial :169-190), for callers of the reference API on the GPU: the
// table / partial in float64 like the reference (the decode kernels use their
// own float32 tables in shared memory).
__global__ void build_lut_f64_kernel(const double *__restrict__ q, int d,
                                     const float *__restrict__ cb, int M, int ksub, double scale,
                                     double *__restrict__ out) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)M * ksub) return;
    const int h = blockIdx.y, dsub = d / M;
    const int i = (int)(idx / ksub), c = (int)(idx - (int64_t)i * ksub);
    const double *qh = q + (int64_t)h * d + i * dsub;
    const float *cc = cb + ((int64_t)i * ksub + c) * dsub;
    double s = 0.0;
    for (int j = 0; j < dsub; ++j) s += (double)cc[j] * qh[j];
    out[(int64_t)h * M * ksub + idx] = s * scale;
}

// One CTA: online softmax over r rows in chunks of kDenseChunk (scores in
// shared memory), record (m, l, 0, 0, acc[d]) in float64.
constexpr int kDenseChunk = 1024, kDenseThreads = 256;
__global__ void __launch_bounds__(kDenseThreads)
    dense_partial_f64_kernel(const double *__restrict__ q, const double *__restrict__ K,
                             const double *__restrict__ V, int64_t r, int d, double scale,
                             double *__restrict__ rec) {
    __shared__ double sc[kDenseChunk];
    __shared__ double red[kDenseThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double m = -INFINITY, l = 0.0;
    constexpr int kAcc = 1024 / kDenseThreads;  // d <= 1024
    double acc[kAcc];
#pragma unroll
    for (int k = 0; k < kAcc; ++k) acc[k] = 0.0;
    for (int64_t t0 = 0; t0 < r; t0 += kDenseChunk) {
        const int cnt = (int)min((int64_t)kDenseChunk, r - t0);
        __syncthreads();
        for (int t = warp; t < cnt; t += kDenseThreads / 32) {  // warp per row
            double dot = 0.0;
            for (int j = lane; j < d; j += 32) dot += K[(t0 + t) * d + j] * q[j];
            for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
            if (lane == 0) sc[t] = scale * dot;
        }
        __syncthreads();
        double mc = -INFINITY;
        for (int t = tid; t < cnt; t += kDenseThreads) mc = fmax(mc, sc[t]);
        for (int off = 16; off > 0; off >>= 1) mc = fmax(mc, __shfl_xor_sync(0xffffffffu, mc, off));
        if (lane == 0) red[warp] = mc;
        __syncthreads();
        mc = red[0];
        for (int w = 1; w < kDenseThreads / 32; ++w) mc = fmax(mc, red[w]);
        const double mn = fmax(m, mc);
        const double f = (m == -INFINITY) ? 0.0 : exp(m - mn);
        l *= f;
#pragma unroll
        for (int k = 0; k < kAcc; ++k) acc[k] *= f;
        m = mn;
        double ls = 0.0;
        for (int t = 0; t < cnt; ++t) {
            const double p = exp(sc[t] - m);
            ls += p;
#pragma unroll
            for (int k = 0; k < kAcc; ++k) {
                const int j = tid + k * kDenseThreads;
                if (j < d) acc[k] += p * V[(t0 + t) * d + j];
            }
        }
        l += ls;
    }
#pragma unroll
    for (int k = 0; k < kAcc; ++k) {
        const int j = tid + k * kDenseThreads;
        if (j < d) rec[4 + j] = acc[k];
    }
    if (tid == 0) {
        rec[0] = m;
        rec[1] = l;
        rec[2] = 0.0;
        rec[3] = 0.0;
    }
}

// Test-only: lets the next PDL launch start at once, waits ns, then writes v
// to p[0..n) -- a length update the dependent kernel can only see after its
// griddepcontrol.wait (exercises the early_codes re-validation).
__global__ void delayed_fill_kernel(int32_t *p, int n, int32_t v, long long ns) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    do {
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    } while ((long long)(t - t0) < ns);
    for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = v;
}

// append_decode's row write (kv_cache.py:188-200) with the recent length on
// the device: rows n of rk / rv (n = *lens[1]) take k / v, then *lens[1] = n + 1
__global__ void append_recent_kernel(const float *__restrict__ k, const float *__restrict__ v,
                                     float *rk, float *rv, int32_t *lens, int d) {
    const int n = lens[1];
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        rk[(int64_t)n * d + i] = k[i];
        rv[(int64_t)n * d + i] = v[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) lens[1] = n + 1;
}

// a flush's publication on the device: n_q += batch, n_recent -= batch
__global__ void publish_lengths_kernel(int32_t *lens, int batch) {
    lens[0] += batch;
    lens[1] -= batch;
}

}  // namespace
}  // namespace pqkv

using namespace pqkv;

extern "C" int pqkv_append_recent(const float *k, const float *v, float *rk, float *rv,
                                  int32_t *lens, int d, void *stream) {
    PQKV_CHECK_ARG(k && v && rk && rv && lens && d > 0 && d <= 4096,
                   "pqkv_append_recent: bad arguments");
    append_recent_kernel<<<1, 128, 0, as_stream(stream)>>>(k, v, rk, rv, lens, d);
    return launch_status("pqkv_append_recent");
}

extern "C" int pqkv_publish_lengths(int32_t *lens, int batch, void *stream) {
    PQKV_CHECK_ARG(lens && batch >= 0, "pqkv_publish_lengths: bad arguments");
    publish_lengths_kernel<<<1, 1, 0, as_stream(stream)>>>(lens, batch);
    return launch_status("pqkv_publish_lengths");
}

extern "C" int pqkv_debug_delayed_fill(int32_t *p, int n, int32_t v, long long ns, void *stream) {
    PQKV_CHECK_ARG(p && n >= 0 && ns >= 0 && ns < 10000000000LL,
                   "pqkv_debug_delayed_fill: bad arguments");
    delayed_fill_kernel<<<1, 128, 0, as_stream(stream)>>>(p, n, v, ns);
    return launch_status("pqkv_debug_delayed_fill");
}

extern "C" int pqkv_version(void) { return 1; }

extern "C" const char *pqkv_last_error(void) { return g_last_error.c_str(); }

extern "C" int pqkv_build_lut(const float *q, int64_t n_heads, int d, const float *cb_k, int M,
                              int nbits, float scale, float *lut, void *stream) {
    PQKV_CHECK_ARG(geometry_ok(d, M, nbits), "pqkv_build_lut: bad geometry");
    PQKV_CHECK_ARG(n_heads >= 0 && n_heads <= 65535, "pqkv_build_lut: n_heads out of range");
    if (n_heads == 0) return PQKV_OK;
    PQKV_CHECK_ARG(q && cb_k && lut, "pqkv_build_lut: null pointer");
    const int ksub = 1 << nbits;
    dim3 grid((unsigned)((ksub + 31) / 32), (unsigned)n_heads);
    build_lut_kernel<<<grid, 256, d * sizeof(float), as_stream(stream)>>>(q, d, cb_k, M, ksub,
                                                                         scale, lut);
    return launch_status("pqkv_build_lut");
}

extern "C" int pqkv_prepare_value_codebook(const float *cb_v, int d, int M, int nbits, float *out,
                                           void *stream) {
    PQKV_CHECK_ARG(is_fast_geometry(d, M, nbits),
                   "pqkv_prepare_value_codebook: only the m64b8 (d=128) geometry is re-laid out");
    PQKV_CHECK_ARG(cb_v && out, "pqkv_prepare_value_codebook: null pointer");
    prepare_cv_kernel<<<64, 256, 0, as_stream(stream)>>>((const float2 *)cb_v, (float2 *)out);
    return launch_status("pqkv_prepare_value_codebook");
}

extern "C" int pqkv_prepare_value_codebook_f16(const float *cb_v, int d, int M, int nbits,
                                               void *out, void *stream) {
    PQKV_CHECK_ARG(is_fast_geometry(d, M, nbits),
                   "pqkv_prepare_value_codebook_f16: only the m64b8 (d=128) geometry");
    PQKV_CHECK_ARG(cb_v && out, "pqkv_prepare_value_codebook_f16: null pointer");
    prepare_cv_f16_kernel<<<64, 256, 0, as_stream(stream)>>>((const float2 *)cb_v,
                                                              (__half2 *)out);
    return launch_status("pqkv_prepare_value_codebook_f16");
}

extern "C" int pqkv_l2_persist(const void *base, size_t bytes, float hit_ratio, void *stream) {
    PQKV_CHECK_ARG(hit_ratio >= 0.f && hit_ratio <= 1.f, "pqkv_l2_persist: hit_ratio out of [0, 1]");
    int dev = 0, max_persist = 0, max_window = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev) != cudaSuccess)
        return fail(PQKV_ECUDA, "pqkv_l2_persist: device query failed");
    const size_t window = bytes < (size_t)max_window ? bytes : (size_t)max_window;
    const size_t carve = window < (size_t)max_persist ? window : (size_t)max_persist;
    cudaError_t e = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, base ? carve : 0);
    if (e != cudaSuccess) return fail(PQKV_ECUDA, "pqkv_l2_persist: %s", cudaGetErrorString(e));
    cudaStreamAttrValue v = {};
    v.accessPolicyWindow.base_ptr = const_cast<void *>(base);
    v.accessPolicyWindow.num_bytes = base ? window : 0;
    v.accessPolicyWindow.hitRatio = hit_ratio;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    e = cudaStreamSetAttribute(as_stream(stream), cudaStreamAttributeAccessPolicyWindow, &v);
    if (e != cudaSuccess) return fail(PQKV_ECUDA, "pqkv_l2_persist: %s", cudaGetErrorString(e));
    return PQKV_OK;
}

extern "C" int pqkv_prepare_key_codebook(const float *cb_k, int d, int M, int nbits, float *out,
                                         void *stream) {
    PQKV_CHECK_ARG(is_fast_geometry(d, M, nbits),
                   "pqkv_prepare_key_codebook: only the m64b8 (d=128) geometry is re-laid out");
    PQKV_CHECK_ARG(cb_k && out, "pqkv_prepare_key_codebook: null pointer");
    prepare_ck_kernel<<<64, 256, 0, as_stream(stream)>>>((const float2 *)cb_k, (float2 *)out);
    return launch_status("pqkv_prepare_key_codebook");
}

extern "C" int pqkv_relayout_codes(const void *src, int64_t ld_src, void *dst, int64_t ld_dst,
                                   int64_t n, int64_t t_first, int to_decode, int d, int M,
                                   int nbits, void *stream) {
    PQKV_CHECK_ARG(is_fast_geometry(d, M, nbits),
                   "pqkv_relayout_codes: the decode layout exists only for m64b8");
    PQKV_CHECK_ARG(n >= 0 && t_first >= 0 && ld_src >= M && ld_dst >= M,
                   "pqkv_relayout_codes: bad sizes");
    if (n == 0) return PQKV_OK;
    PQKV_CHECK_ARG(src && dst && src != dst, "pqkv_relayout_codes: null or aliased pointers");
    relayout_kernel<<<(unsigned)((n * 64 + 255) / 256), 256, 0, as_stream(stream)>>>(
        (const uint8_t *)src, ld_src, (uint8_t *)dst, ld_dst, n, t_first, to_decode);
    return launch_status("pqkv_relayout_codes");
}

extern "C" int pqkv_reconstruct(const void *codes, int64_t n, int64_t ld_codes,
                                const float *centroids, int d, int M, int nbits, float *out,
                                void *stream) {
    PQKV_CHECK_ARG(geometry_ok(d, M, nbits), "pqkv_reconstruct: bad geometry");
    PQKV_CHECK_ARG(n >= 0 && ld_codes >= M, "pqkv_reconstruct: bad sizes");
    if (n == 0) return PQKV_OK;
    PQKV_CHECK_ARG(codes && centroids && out, "pqkv_reconstruct: null pointer");
    const int64_t total = n * d;
    const unsigned blocks = (unsigned)((total + 255) / 256);
    if (nbits <= 8)
        reconstruct_kernel<uint8_t><<<blocks, 256, 0, as_stream(stream)>>>(
            (const uint8_t *)codes, n, ld_codes, centroids, d, M, 1 << nbits, out);
    else
        reconstruct_kernel<uint16_t><<<blocks, 256, 0, as_stream(stream)>>>(
            (const uint16_t *)codes, n, ld_codes, centroids, d, M, 1 << nbits, out);
    return launch_status("pqkv_reconstruct");
}

extern "C" int pqkv_score_codes(const float *lut, const void *codes, int64_t n, int M, int nbits,
                                float *scores, void *stream) {
    PQKV_CHECK_ARG(M > 0 && nbits >= 1 && nbits <= 16 && n >= 0, "pqkv_score_codes: bad args");
    if (n == 0) return PQKV_OK;
    PQKV_CHECK_ARG(lut && codes && scores, "pqkv_score_codes: null pointer");
    const unsigned blocks = (unsigned)((n + 255) / 256);
    if (nbits <= 8)
        score_codes_kernel<uint8_t><<<blocks, 256, 0, as_stream(stream)>>>(
            lut, (const uint8_t *)codes, n, M, scores);
    else
        score_codes_kernel<uint16_t><<<blocks, 256, 0, as_stream(stream)>>>(
            lut, (const uint16_t *)codes, n, M, scores);
    return launch_status("pqkv_score_codes");
}

extern "C" int pqkv_accumulate_mass(const void *codes, const float *p, int64_t n, int M,
                                    int nbits, float *h, void *stream) {
    PQKV_CHECK_ARG(M > 0 && nbits >= 1 && nbits <= 16 && n >= 0, "pqkv_accumulate_mass: bad args");
    PQKV_CHECK_ARG(h, "pqkv_accumulate_mass: null output");
    const int ksub = 1 << nbits;
    cudaStream_t st = as_stream(stream);
    cudaError_t e = cudaMemsetAsync(h, 0, sizeof(float) * (size_t)M * ksub, st);
    if (e != cudaSuccess) return fail(PQKV_ECUDA, "pqkv_accumulate_mass: %s", cudaGetErrorString(e));
    if (n == 0) return PQKV_OK;
    PQKV_CHECK_ARG(codes && p, "pqkv_accumulate_mass: null pointer");
    const unsigned blocks = (unsigned)((n * M + 255) / 256);
    if (nbits <= 8)
        accumulate_mass_kernel<uint8_t><<<blocks, 256, 0, st>>>((const uint8_t *)codes, p, n, M,
                                                                 ksub, h);
    else
        accumulate_mass_kernel<uint16_t><<<blocks, 256, 0, st>>>((const uint16_t *)codes, p, n, M,
                                                                  ksub, h);
    return launch_status("pqkv_accumulate_mass");
}

extern "C" int pqkv_score_codes_f64(const double *lut, const void *codes, int64_t n, int M,
                                    int nbits, double *scores, void *stream) {
    PQKV_CHECK_ARG(M > 0 && nbits >= 1 && nbits <= 16 && n >= 0,
                   "pqkv_score_codes_f64: bad args");
    if (n == 0) return PQKV_OK;
    PQKV_CHECK_ARG(lut && codes && scores, "pqkv_score_codes_f64: null pointer");
    const unsigned blocks = (unsigned)((n + 255) / 256);
    if (nbits <= 8)
        score_codes_f64_kernel<uint8_t><<<blocks, 256, 0, as_stream(stream)>>>(
            lut, 1 << nbits, (const uint8_t *)codes, n, M, scores);
    else
        score_codes_f64_kernel<uint16_t><<<blocks, 256, 0, as_stream(stream)>>>(
            lut, 1 << nbits, (const uint16_t *)codes, n, M, scores);
    return launch_status("pqkv_score_codes_f64");
}

extern "C" int pqkv_accumulate_mass_f64(const void *codes, const double *p, int64_t n, int M,
                                        int nbits, double *h, void *stream) {
    PQKV_CHECK_ARG(M > 0 && M <= 65535 && nbits >= 1 && nbits <= 16 && n >= 0,
                   "pqkv_accumulate_mass_f64: bad args");
    PQKV_CHECK_ARG(h && (n == 0 || (codes && p)), "pqkv_accumulate_mass_f64: null pointer");
    const int ksub = 1 << nbits;
    dim3 grid((unsigned)((ksub + 255) / 256), (unsigned)M);
    if (nbits <= 8)
        accumulate_mass_f64_kernel<uint8_t><<<grid, 256, 0, as_stream(stream)>>>(
            (const uint8_t *)codes, p, n, M, ksub, h);
    else
        accumulate_mass_f64_kernel<uint16_t><<<grid, 256, 0, as_stream(stream)>>>(
            (const uint16_t *)codes, p, n, M, ksub, h);
    return launch_status("pqkv_accumulate_mass_f64");
}

extern "C" int pqkv_build_lut_f64(const double *q, int64_t n_heads, int d, const float *cb_k,
                                  int M, int nbits, double scale, double *out, void *stream) {
    PQKV_CHECK_ARG(geometry_ok(d, M, nbits) && n_heads >= 0 && n_heads < 65536,
                   "pqkv_build_lut_f64: bad arguments");
    if (n_heads == 0) return PQKV_OK;
    PQKV_CHECK_ARG(q && cb_k && out, "pqkv_build_lut_f64: null pointer");
    const int64_t cells = (int64_t)M << nbits;
    dim3 grid((unsigned)((cells + 255) / 256), (unsigned)n_heads);
    build_lut_f64_kernel<<<grid, 256, 0, as_stream(stream)>>>(q, d, cb_k, M, 1 << nbits, scale,
                                                              out);
    return launch_status("pqkv_build_lut_f64");
}

extern "C" int pqkv_dense_partial_f64(const double *q, const double *K, const double *V,
                                      int64_t r, int d, double scale, double *rec, void *stream) {
    PQKV_CHECK_ARG(r >= 1 && d >= 1 && d <= 1024, "pqkv_dense_partial_f64: bad sizes");
    PQKV_CHECK_ARG(q && K && V && rec, "pqkv_dense_partial_f64: null pointer");
    dense_partial_f64_kernel<<<1, kDenseThreads, 0, as_stream(stream)>>>(q, K, V, r, d, scale,
                                                                         rec);
    return launch_status("pqkv_dense_partial_f64");
}
