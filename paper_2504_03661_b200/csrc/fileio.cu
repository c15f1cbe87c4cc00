// Binary formats at the boundary, read and written straight between files and
// device memory (reference fileio.py:71-160):
//   .pqkv codebook: "PQKV", <IBIII (version u32, kind u8, d, M, nbits) -- a
//                   21-byte header, so the float32 body is unaligned -- then
//                   M * 2^nbits * dsub float32, subspace-major;
//   .pqkc dump:     "PQKC", <IIIIQI (version, d, M, nbits, n_q u64,
//                   recent_len), then K codes, V codes (reference row layout),
//                   recent K rows, recent V rows (float32).
// Files of many caches (one per layer x sequence x KV head of a serving cache)
// are those records back to back, each readable by the reference's reader.
//
// The body moves with one pinned staging buffer and one (2-D, strided)
// copy per field for all heads; codes are converted between the decode
// layout and the reference row layout on the device (batched relayout).
// Error messages follow the reference's FormatError texts ("bad magic",
// "unsupported version", "expected N floats", "expected N bytes",
// "corrupted dump").
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"

namespace pqkv {
namespace {

constexpr int kCbHeader = 4 + 17;     // magic + <IBIII
constexpr int kCacheHeader = 4 + 28;  // magic + <IIIIQI
constexpr uint32_t kVersion = 1;

// ----------------------------------------------------------- host buffers ---
struct HostBuf {  // pinned when a device copy is involved (async copies need it)
    uint8_t *p = nullptr;
    size_t n = 0;
    bool pinned = false;
    ~HostBuf() {
        if (!p) return;
        if (pinned)
            cudaFreeHost(p);
        else
            free(p);
    }
    int alloc(size_t bytes, bool pin) {
        n = bytes;
        pinned = pin;
        if (bytes == 0) return PQKV_OK;
        if (pin) {
            if (cudaMallocHost(&p, bytes) != cudaSuccess) {
                p = nullptr;
                cudaGetLastError();
                return fail(PQKV_ECUDA, "pinned staging buffer of %zu bytes", bytes);
            }
        } else if (!(p = (uint8_t *)malloc(bytes))) {
            return fail(PQKV_EIO, "out of host memory (%zu bytes)", bytes);
        }
        return PQKV_OK;
    }
};

struct DevBuf {
    void *p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    int alloc(size_t bytes) {
        if (bytes == 0) return PQKV_OK;
        if (cudaMalloc(&p, bytes) != cudaSuccess) {
            p = nullptr;
            cudaGetLastError();
            return fail(PQKV_ECUDA, "device staging buffer of %zu bytes", bytes);
        }
        return PQKV_OK;
    }
};

int read_file(const char *path, HostBuf &buf, bool pin, size_t max_bytes = SIZE_MAX) {
    FILE *f = fopen(path, "rb");
    if (!f) return fail(PQKV_EIO, "%s: cannot open for reading", path);
    fseek(f, 0, SEEK_END);
    const long len = ftell(f);
    fseek(f, 0, SEEK_SET);
    const size_t want = (size_t)len < max_bytes ? (size_t)len : max_bytes;
    int rc = buf.alloc(want, pin);
    if (rc == PQKV_OK && want && fread(buf.p, 1, want, f) != want)
        rc = fail(PQKV_EIO, "%s: short read", path);
    fclose(f);
    return rc;
}

int write_file(const char *path, const uint8_t *p, size_t n) {
    FILE *f = fopen(path, "wb");
    if (!f) return fail(PQKV_EIO, "%s: cannot open for writing", path);
    const bool ok = fwrite(p, 1, n, f) == n;
    const bool closed = fclose(f) == 0;
    if (!ok || !closed) return fail(PQKV_EIO, "%s: write failed", path);
    return PQKV_OK;
}

template <typename T>
T get(const uint8_t *p) {  // unaligned little-endian field
    T v;
    memcpy(&v, p, sizeof(T));
    return v;
}
template <typename T>
void put(uint8_t *p, T v) {
    memcpy(p, &v, sizeof(T));
}

int cuda_status(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return PQKV_OK;
    cudaGetLastError();
    return fail(PQKV_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

// ------------------------------------------------------------- codebooks ---
struct CbInfo {
    int kind, d, M, nbits;
    int64_t floats;
};

int parse_cb_header(const char *path, const uint8_t *raw, size_t len, CbInfo *ci) {
    if (len < 4 || memcmp(raw, "PQKV", 4) != 0)
        return fail(PQKV_EFORMAT, "%s: bad magic", path);
    if (len < (size_t)kCbHeader) return fail(PQKV_EFORMAT, "%s: truncated header", path);
    const uint32_t version = get<uint32_t>(raw + 4);
    const uint8_t kind = raw[8];
    const uint32_t d = get<uint32_t>(raw + 9), M = get<uint32_t>(raw + 13),
                   nbits = get<uint32_t>(raw + 17);
    if (version != kVersion) return fail(PQKV_EFORMAT, "%s: unsupported version %u", path, version);
    if (kind > 1) return fail(PQKV_EFORMAT, "%s: unknown kind tag %u", path, kind);
    if (!(d <= (1u << 20) && M <= (1u << 20) && geometry_ok((int)d, (int)M, (int)nbits)))
        return fail(PQKV_EINVAL, "%s: bad geometry d=%u M=%u nbits=%u", path, d, M, nbits);
    ci->kind = kind;
    ci->d = (int)d;
    ci->M = (int)M;
    ci->nbits = (int)nbits;
    ci->floats = (int64_t)M * ((int64_t)1 << nbits) * (d / M);
    return PQKV_OK;
}

int check_cb_body(const char *path, size_t len, const CbInfo &ci) {
    const size_t body = len - kCbHeader;
    if (body % 4) return fail(PQKV_EFORMAT, "%s: body is not a whole number of float32", path);
    if ((int64_t)(body / 4) != ci.floats)
        return fail(PQKV_EFORMAT, "%s: expected %lld floats, found %lld", path,
                    (long long)ci.floats, (long long)(body / 4));
    return PQKV_OK;
}

// ------------------------------------------------------------ cache dumps ---
struct DumpInfo {
    int d, M, nbits, recent_len;
    int64_t n_q;
    size_t code_bytes, recent_bytes, record_bytes;
};

int parse_dump_header(const char *path, const uint8_t *raw, size_t len, DumpInfo *di) {
    if (len < 4 || memcmp(raw, "PQKC", 4) != 0)
        return fail(PQKV_EFORMAT, "%s: bad magic", path);
    if (len < (size_t)kCacheHeader) return fail(PQKV_EFORMAT, "%s: truncated header", path);
    const uint32_t version = get<uint32_t>(raw + 4);
    const uint32_t d = get<uint32_t>(raw + 8), M = get<uint32_t>(raw + 12),
                   nbits = get<uint32_t>(raw + 16);
    const uint64_t n_q = get<uint64_t>(raw + 20);
    const uint32_t recent = get<uint32_t>(raw + 28);
    if (version != kVersion) return fail(PQKV_EFORMAT, "%s: unsupported version %u", path, version);
    if (!(d <= (1u << 20) && M <= (1u << 20) && geometry_ok((int)d, (int)M, (int)nbits)) ||
        n_q > (1ull << 40) || recent > (1u << 24))
        return fail(PQKV_EINVAL, "%s: bad dump header", path);
    di->d = (int)d;
    di->M = (int)M;
    di->nbits = (int)nbits;
    di->n_q = (int64_t)n_q;
    di->recent_len = (int)recent;
    di->code_bytes = (size_t)n_q * M * cell_bytes((int)nbits);
    di->recent_bytes = (size_t)recent * d * 4;
    di->record_bytes = kCacheHeader + 2 * di->code_bytes + 2 * di->recent_bytes;
    return PQKV_OK;
}

// codes of `heads` caches between the decode layout and the row layout (m64b8)
__global__ void relayout_batched_kernel(const uint8_t *__restrict__ src, int64_t src_head,
                                        uint8_t *__restrict__ dst, int64_t dst_head, int64_t n,
                                        int to_decode) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * 64) return;
    const int64_t v = idx >> 6, h = blockIdx.y;
    const int i = (int)(idx & 63);
    const int pos = decode_layout_pos(i, v);
    const uint8_t *s = src + h * src_head + v * 64;
    uint8_t *o = dst + h * dst_head + v * 64;
    if (to_decode)
        o[pos] = s[i];
    else
        o[i] = s[pos];
}

// the largest code in `heads` x n x M cells (reference's corrupted-dump check)
template <typename CT>
__global__ void max_code_kernel(const CT *__restrict__ c, int64_t total, int *out) {
    int m = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, (int)c[i]);
    for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

}  // namespace
}  // namespace pqkv

using namespace pqkv;

extern "C" int pqkv_codebook_file_info(const char *path, int *kind, int *d, int *M, int *nbits) {
    PQKV_CHECK_ARG(path, "pqkv_codebook_file_info: null path");
    HostBuf head;
    int rc = read_file(path, head, false, kCbHeader);
    if (rc) return rc;
    CbInfo ci;
    if ((rc = parse_cb_header(path, head.p, head.n, &ci))) return rc;
    FILE *f = fopen(path, "rb");
    if (!f) return fail(PQKV_EIO, "%s: cannot open for reading", path);
    fseek(f, 0, SEEK_END);
    const long len = ftell(f);
    fclose(f);
    if ((rc = check_cb_body(path, (size_t)len, ci))) return rc;
    if (kind) *kind = ci.kind;
    if (d) *d = ci.d;
    if (M) *M = ci.M;
    if (nbits) *nbits = ci.nbits;
    return PQKV_OK;
}

extern "C" int pqkv_read_codebook(const char *path, int flags, float *centroids, float *layout,
                                  void *stream) {
    PQKV_CHECK_ARG(path, "pqkv_read_codebook: null path");
    PQKV_CHECK_ARG((flags & ~PQKV_FILE_HOST) == 0, "pqkv_read_codebook: unknown flags");
    const bool host = flags & PQKV_FILE_HOST;
    PQKV_CHECK_ARG(!(host && layout), "pqkv_read_codebook: the kernel layout is device memory");
    HostBuf raw;
    int rc = read_file(path, raw, !host);
    if (rc) return rc;
    CbInfo ci;
    if ((rc = parse_cb_header(path, raw.p, raw.n, &ci))) return rc;
    if ((rc = check_cb_body(path, raw.n, ci))) return rc;
    const size_t bytes = (size_t)ci.floats * 4;
    const uint8_t *body = raw.p + kCbHeader;  // unaligned for float32: byte copies only
    if (host) {
        if (centroids) memcpy(centroids, body, bytes);
        return PQKV_OK;
    }
    cudaStream_t st = as_stream(stream);
    DevBuf tmp;
    float *dcent = centroids;
    if (!dcent && layout) {
        if ((rc = tmp.alloc(bytes))) return rc;
        dcent = (float *)tmp.p;
    }
    if (dcent && (rc = cuda_status(cudaMemcpyAsync(dcent, body, bytes, cudaMemcpyHostToDevice, st),
                                   "pqkv_read_codebook")))
        return rc;
    if (layout) {
        PQKV_CHECK_ARG(is_fast_geometry(ci.d, ci.M, ci.nbits),
                       "pqkv_read_codebook: the decode-kernel layout exists only for m64b8");
        rc = ci.kind == 0 ? pqkv_prepare_key_codebook(dcent, ci.d, ci.M, ci.nbits, layout, stream)
                          : pqkv_prepare_value_codebook(dcent, ci.d, ci.M, ci.nbits, layout,
                                                        stream);
        if (rc) return rc;
    }
    // the pinned body (and the temporary) must outlive the copies
    return cuda_status(cudaStreamSynchronize(st), "pqkv_read_codebook");
}

extern "C" int pqkv_write_codebook(const char *path, int kind, int d, int M, int nbits,
                                   const float *centroids, int flags, void *stream) {
    PQKV_CHECK_ARG(path && centroids, "pqkv_write_codebook: null pointer");
    PQKV_CHECK_ARG(kind == 0 || kind == 1, "pqkv_write_codebook: kind must be 0 (key) or 1 (value)");
    PQKV_CHECK_ARG(geometry_ok(d, M, nbits), "pqkv_write_codebook: bad geometry");
    PQKV_CHECK_ARG((flags & ~PQKV_FILE_HOST) == 0, "pqkv_write_codebook: unknown flags");
    const bool host = flags & PQKV_FILE_HOST;
    const size_t bytes = (size_t)M * ((size_t)1 << nbits) * (d / M) * 4;
    HostBuf out;
    int rc = out.alloc(kCbHeader + bytes, !host);
    if (rc) return rc;
    memcpy(out.p, "PQKV", 4);
    put<uint32_t>(out.p + 4, kVersion);
    out.p[8] = (uint8_t)kind;
    put<uint32_t>(out.p + 9, (uint32_t)d);
    put<uint32_t>(out.p + 13, (uint32_t)M);
    put<uint32_t>(out.p + 17, (uint32_t)nbits);
    if (host) {
        memcpy(out.p + kCbHeader, centroids, bytes);
    } else {
        cudaStream_t st = as_stream(stream);
        if ((rc = cuda_status(cudaMemcpyAsync(out.p + kCbHeader, centroids, bytes,
                                              cudaMemcpyDeviceToHost, st),
                              "pqkv_write_codebook")))
            return rc;
        if ((rc = cuda_status(cudaStreamSynchronize(st), "pqkv_write_codebook"))) return rc;
    }
    return write_file(path, out.p, out.n);
}

extern "C" int pqkv_cache_dump_info(const char *path, int64_t offset, int *d, int *M, int *nbits,
                                    int64_t *n_q, int *recent_len, int64_t *record_bytes) {
    PQKV_CHECK_ARG(path && offset >= 0, "pqkv_cache_dump_info: bad arguments");
    FILE *f = fopen(path, "rb");
    if (!f) return fail(PQKV_EIO, "%s: cannot open for reading", path);
    fseek(f, 0, SEEK_END);
    const long len = ftell(f);
    uint8_t head[kCacheHeader];
    size_t got = 0;
    if (offset <= len) {
        fseek(f, (long)offset, SEEK_SET);
        got = fread(head, 1, kCacheHeader, f);
    }
    fclose(f);
    DumpInfo di;
    int rc = parse_dump_header(path, head, got, &di);
    if (rc) return rc;
    if ((size_t)(len - offset) < di.record_bytes)
        return fail(PQKV_EFORMAT, "%s: expected %zu bytes, found %lld", path,
                    di.record_bytes + (size_t)offset, (long long)len);
    if (d) *d = di.d;
    if (M) *M = di.M;
    if (nbits) *nbits = di.nbits;
    if (n_q) *n_q = di.n_q;
    if (recent_len) *recent_len = di.recent_len;
    if (record_bytes) *record_bytes = (int64_t)di.record_bytes;
    return PQKV_OK;
}

static int check_dump_args(const char *fn, int heads, int d, int M, int nbits, int64_t n_q,
                           int recent_len, int64_t code_stride, int layout,
                           int64_t recent_stride) {
    PQKV_CHECK_ARG(heads >= 1 && geometry_ok(d, M, nbits) && n_q >= 0 && recent_len >= 0,
                   "%s: bad sizes", fn);
    PQKV_CHECK_ARG(code_stride >= n_q * M && recent_stride >= (int64_t)recent_len * d,
                   "%s: head strides smaller than one head", fn);
    PQKV_CHECK_ARG(layout == PQKV_CODES_ROWS || layout == PQKV_CODES_DECODE, "%s: bad layout", fn);
    PQKV_CHECK_ARG(layout == PQKV_CODES_ROWS || is_fast_geometry(d, M, nbits),
                   "%s: the decode layout exists only for m64b8", fn);
    return PQKV_OK;
}

extern "C" int pqkv_write_cache_dumps(const char *path, int heads, int d, int M, int nbits,
                                      int64_t n_q, int recent_len, const void *codes_k,
                                      const void *codes_v, int64_t code_stride, int layout,
                                      const float *recent_k, const float *recent_v,
                                      int64_t recent_stride, void *stream) {
    PQKV_CHECK_ARG(path, "pqkv_write_cache_dumps: null path");
    int rc = check_dump_args("pqkv_write_cache_dumps", heads, d, M, nbits, n_q, recent_len,
                             code_stride, layout, recent_stride);
    if (rc) return rc;
    PQKV_CHECK_ARG((n_q == 0 || (codes_k && codes_v)) &&
                       (recent_len == 0 || (recent_k && recent_v)),
                   "pqkv_write_cache_dumps: null pointer");
    const size_t cell = cell_bytes(nbits);
    const size_t cb = (size_t)n_q * M * cell, rb = (size_t)recent_len * d * 4;
    const size_t rec = kCacheHeader + 2 * cb + 2 * rb;
    HostBuf out;
    if ((rc = out.alloc(rec * heads, true))) return rc;
    for (int h = 0; h < heads; ++h) {
        uint8_t *p = out.p + rec * h;
        memcpy(p, "PQKC", 4);
        put<uint32_t>(p + 4, kVersion);
        put<uint32_t>(p + 8, (uint32_t)d);
        put<uint32_t>(p + 12, (uint32_t)M);
        put<uint32_t>(p + 16, (uint32_t)nbits);
        put<uint64_t>(p + 20, (uint64_t)n_q);
        put<uint32_t>(p + 28, (uint32_t)recent_len);
    }
    cudaStream_t st = as_stream(stream);
    DevBuf rows;
    const uint8_t *ck = (const uint8_t *)codes_k, *cv = (const uint8_t *)codes_v;
    size_t cpitch = (size_t)code_stride * cell;
    if (n_q && layout == PQKV_CODES_DECODE) {  // decode layout -> reference rows, on the device
        if ((rc = rows.alloc(2 * cb * heads))) return rc;
        uint8_t *rk = (uint8_t *)rows.p, *rv = rk + cb * heads;
        dim3 grid((unsigned)((n_q * 64 + 255) / 256), (unsigned)heads);
        relayout_batched_kernel<<<grid, 256, 0, st>>>(ck, (int64_t)cpitch, rk, (int64_t)cb, n_q, 0);
        relayout_batched_kernel<<<grid, 256, 0, st>>>(cv, (int64_t)cpitch, rv, (int64_t)cb, n_q, 0);
        if ((rc = launch_status("pqkv_write_cache_dumps"))) return rc;
        ck = rk;
        cv = rv;
        cpitch = cb;
    }
    if (cb) {
        rc = cuda_status(cudaMemcpy2DAsync(out.p + kCacheHeader, rec, ck, cpitch, cb, heads,
                                           cudaMemcpyDeviceToHost, st),
                         "pqkv_write_cache_dumps");
        if (!rc)
            rc = cuda_status(cudaMemcpy2DAsync(out.p + kCacheHeader + cb, rec, cv, cpitch, cb,
                                               heads, cudaMemcpyDeviceToHost, st),
                             "pqkv_write_cache_dumps");
        if (rc) return rc;
    }
    if (rb) {
        const size_t rpitch = (size_t)recent_stride * 4;
        rc = cuda_status(cudaMemcpy2DAsync(out.p + kCacheHeader + 2 * cb, rec, recent_k, rpitch,
                                           rb, heads, cudaMemcpyDeviceToHost, st),
                         "pqkv_write_cache_dumps");
        if (!rc)
            rc = cuda_status(cudaMemcpy2DAsync(out.p + kCacheHeader + 2 * cb + rb, rec, recent_v,
                                               rpitch, rb, heads, cudaMemcpyDeviceToHost, st),
                             "pqkv_write_cache_dumps");
        if (rc) return rc;
    }
    if ((rc = cuda_status(cudaStreamSynchronize(st), "pqkv_write_cache_dumps"))) return rc;
    return write_file(path, out.p, out.n);
}

extern "C" int pqkv_read_cache_dumps(const char *path, int heads, int d, int M, int nbits,
                                     int64_t n_q, int recent_len, void *codes_k, void *codes_v,
                                     int64_t code_stride, int layout, float *recent_k,
                                     float *recent_v, int64_t recent_stride, void *stream) {
    PQKV_CHECK_ARG(path, "pqkv_read_cache_dumps: null path");
    int rc = check_dump_args("pqkv_read_cache_dumps", heads, d, M, nbits, n_q, recent_len,
                             code_stride, layout, recent_stride);
    if (rc) return rc;
    PQKV_CHECK_ARG((n_q == 0 || (codes_k && codes_v)) &&
                       (recent_len == 0 || (recent_k && recent_v)),
                   "pqkv_read_cache_dumps: null pointer");
    HostBuf raw;
    if ((rc = read_file(path, raw, true))) return rc;
    const size_t cell = cell_bytes(nbits);
    const size_t cb = (size_t)n_q * M * cell, rb = (size_t)recent_len * d * 4;
    const size_t rec = kCacheHeader + 2 * cb + 2 * rb;
    for (int h = 0; h < heads; ++h) {
        DumpInfo di;
        const size_t off = rec * h;
        if ((rc = parse_dump_header(path, off <= raw.n ? raw.p + off : raw.p,
                                    off <= raw.n ? raw.n - off : 0, &di)))
            return rc;
        if (di.d != d || di.M != M || di.nbits != nbits || di.n_q != n_q ||
            di.recent_len != recent_len)
            return fail(PQKV_EFORMAT, "%s: record %d does not match the destination geometry",
                        path, h);
    }
    if (raw.n != rec * heads)
        return fail(PQKV_EFORMAT, "%s: expected %zu bytes, found %zu", path, rec * heads, raw.n);
    cudaStream_t st = as_stream(stream);
    if (cb) {
        DevBuf tmp;
        uint8_t *dk = (uint8_t *)codes_k, *dv = (uint8_t *)codes_v;
        size_t dpitch = (size_t)code_stride * cell;
        if (layout == PQKV_CODES_DECODE) {
            if ((rc = tmp.alloc(2 * cb * heads))) return rc;
            dk = (uint8_t *)tmp.p;
            dv = dk + cb * heads;
            dpitch = cb;
        }
        rc = cuda_status(cudaMemcpy2DAsync(dk, dpitch, raw.p + kCacheHeader, rec, cb, heads,
                                           cudaMemcpyHostToDevice, st),
                         "pqkv_read_cache_dumps");
        if (!rc)
            rc = cuda_status(cudaMemcpy2DAsync(dv, dpitch, raw.p + kCacheHeader + cb, rec, cb,
                                               heads, cudaMemcpyHostToDevice, st),
                             "pqkv_read_cache_dumps");
        if (rc) return rc;
        if (nbits < 8 * (int)cell) {  // a cell can hold an out-of-range code
            DevBuf mx;
            if ((rc = mx.alloc(sizeof(int)))) return rc;
            cudaMemsetAsync(mx.p, 0, sizeof(int), st);
            for (uint8_t *c : {dk, dv})
                for (int h = 0; h < heads; ++h) {
                    const int64_t total = n_q * M;
                    if (cell == 1)
                        max_code_kernel<uint8_t><<<64, 256, 0, st>>>(c + dpitch * h, total,
                                                                     (int *)mx.p);
                    else
                        max_code_kernel<uint16_t><<<64, 256, 0, st>>>(
                            (const uint16_t *)(c + dpitch * h), total, (int *)mx.p);
                }
            int host_max = 0;
            if ((rc = cuda_status(cudaMemcpyAsync(&host_max, mx.p, sizeof(int),
                                                  cudaMemcpyDeviceToHost, st),
                                  "pqkv_read_cache_dumps")))
                return rc;
            if ((rc = cuda_status(cudaStreamSynchronize(st), "pqkv_read_cache_dumps"))) return rc;
            if (host_max >= (1 << nbits))
                return fail(PQKV_EFORMAT, "%s: corrupted dump, code value >= 2^nbits", path);
        }
        if (layout == PQKV_CODES_DECODE) {
            dim3 grid((unsigned)((n_q * 64 + 255) / 256), (unsigned)heads);
            const int64_t opitch = code_stride * (int64_t)cell;
            relayout_batched_kernel<<<grid, 256, 0, st>>>(dk, (int64_t)cb, (uint8_t *)codes_k,
                                                          opitch, n_q, 1);
            relayout_batched_kernel<<<grid, 256, 0, st>>>(dv, (int64_t)cb, (uint8_t *)codes_v,
                                                          opitch, n_q, 1);
            if ((rc = launch_status("pqkv_read_cache_dumps"))) return rc;
            // tmp is freed on return: finish the relayout first
            if ((rc = cuda_status(cudaStreamSynchronize(st), "pqkv_read_cache_dumps"))) return rc;
        }
    }
    if (rb) {
        const size_t rpitch = (size_t)recent_stride * 4;
        rc = cuda_status(cudaMemcpy2DAsync(recent_k, rpitch, raw.p + kCacheHeader + 2 * cb, rec,
                                           rb, heads, cudaMemcpyHostToDevice, st),
                         "pqkv_read_cache_dumps");
        if (!rc)
            rc = cuda_status(cudaMemcpy2DAsync(recent_v, rpitch,
                                               raw.p + kCacheHeader + 2 * cb + rb, rec, rb, heads,
                                               cudaMemcpyHostToDevice, st),
                             "pqkv_read_cache_dumps");
        if (rc) return rc;
    }
    return cuda_status(cudaStreamSynchronize(st), "pqkv_read_cache_dumps");
}
