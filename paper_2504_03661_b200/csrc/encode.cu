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
    return v * ld_codes + decode_layout_pos(i, (int)((rot_base + v) & 7));
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
            case 2: return launch_staged<TX, CT, 2>(x, n, ld_x, cents, M, ksub, codes, ld_codes, rot_base, st);
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
