/*
 * C restatement of the reference PQ KV-cache hot loops -- TEST / BASELINE
 * INFRASTRUCTURE ONLY (never linked into the product library).
 *
 * Restates, in fp64 like the reference (paths relative to the reference's
 * pkg/src/pqkv/):
 *   - pq_core.py:158-168 (_squared_distances) + :269-287 (assign_codes):
 *       d2 = (||x||^2 - 2 x.c) + ||c||^2, clamp >= 0, first-index argmin.
 *   - attention.py:70-83  build_key_lut      table[i][c] = scale * <q_i, C_K[i][c]>
 *   - _kernels.py:27-34   _score_codes_jit   s_t = sum_i table[i][code]
 *   - _kernels.py:37-43   _accumulate_mass_jit h[i][code] += p_t
 *   - attention.py:103-111 _mass_to_acc, :114-166 quantized_partial ("auto"),
 *     :169-190 dense_partial, :193-211 merge/finalize, :214-287 decode_step
 *     (blockwise, block_size chosen by the caller; no append).
 *
 * Used by bench.py's cpu_baseline / --impl reference legs (kind "port") and
 * cross-checked against the numpy oracle in tests.  Build: oracle/Makefile.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

typedef struct {
    double m, l;
    double *acc;
} partial_t;

static void merge_into(partial_t *a, double m, double l, const double *acc, int d) {
    /* attention.py:193-204: identity on l == 0, else rescale to the larger max */
    if (l == 0.0) return;
    if (a->l == 0.0) {
        a->m = m;
        a->l = l;
        memcpy(a->acc, acc, sizeof(double) * (size_t)d);
        return;
    }
    double mm = a->m > m ? a->m : m;
    double wa = exp(a->m - mm), wb = exp(m - mm);
    a->l = a->l * wa + l * wb;
    for (int j = 0; j < d; ++j) a->acc[j] = a->acc[j] * wa + acc[j] * wb;
    a->m = mm;
}

static inline int code_at(const void *codes, int nbits, int64_t idx) {
    return nbits <= 8 ? ((const uint8_t *)codes)[idx] : ((const uint16_t *)codes)[idx];
}

/* One head: LUT -> blockwise quantized partials -> dense partial -> finalize. */
int oracle_decode_head(const double *q, const float *k_n, const float *v_n,
                       const void *codes_k, const void *codes_v, int64_t n_q,
                       const float *recent_k, const float *recent_v, int64_t n_recent,
                       const float *cents_k, const float *cents_v, int M, int nbits,
                       int dsub, double scale, int64_t block_size, double *out) {
    const int ksub = 1 << nbits, d = M * dsub;
    if (block_size <= 0) return 1;
    double *lut = (double *)malloc(sizeof(double) * (size_t)M * ksub);
    double *h = (double *)malloc(sizeof(double) * (size_t)M * ksub);
    double *s = (double *)malloc(sizeof(double) * (size_t)(block_size + 1 + n_recent));
    double *acc = (double *)calloc((size_t)d, sizeof(double));
    double *racc = (double *)calloc((size_t)d, sizeof(double));
    if (!lut || !h || !s || !acc || !racc) return 2;
    partial_t res = {-INFINITY, 0.0, racc};

    for (int i = 0; i < M; ++i)
        for (int c = 0; c < ksub; ++c) {
            double t = 0.0;
            for (int j = 0; j < dsub; ++j)
                t += (double)cents_k[((size_t)i * ksub + c) * dsub + j] * q[i * dsub + j];
            lut[(size_t)i * ksub + c] = t * scale;
        }

    for (int64_t a = 0; a < n_q; a += block_size) {
        int64_t b = a + block_size < n_q ? a + block_size : n_q, n = b - a;
        double m = -INFINITY, l = 0.0;
        for (int64_t t = 0; t < n; ++t) {
            double st = 0.0;
            for (int i = 0; i < M; ++i) st += lut[(size_t)i * ksub + code_at(codes_k, nbits, (a + t) * M + i)];
            s[t] = st;
            if (st > m) m = st;
        }
        for (int64_t t = 0; t < n; ++t) {
            s[t] = exp(s[t] - m);
            l += s[t];
        }
        memset(acc, 0, sizeof(double) * (size_t)d);
        if (n > 4 * (int64_t)ksub) { /* centroid_accumulate */
            memset(h, 0, sizeof(double) * (size_t)M * ksub);
            for (int64_t t = 0; t < n; ++t)
                for (int i = 0; i < M; ++i) h[(size_t)i * ksub + code_at(codes_v, nbits, (a + t) * M + i)] += s[t];
            for (int i = 0; i < M; ++i)
                for (int j = 0; j < dsub; ++j) {
                    double v = 0.0;
                    for (int c = 0; c < ksub; ++c)
                        v += h[(size_t)i * ksub + c] * (double)cents_v[((size_t)i * ksub + c) * dsub + j];
                    acc[i * dsub + j] = v;
                }
        } else { /* gather */
            for (int64_t t = 0; t < n; ++t)
                for (int i = 0; i < M; ++i) {
                    int c = code_at(codes_v, nbits, (a + t) * M + i);
                    for (int j = 0; j < dsub; ++j)
                        acc[i * dsub + j] += s[t] * (double)(float)cents_v[((size_t)i * ksub + c) * dsub + j];
                }
        }
        merge_into(&res, m, l, acc, d);
    }

    /* dense partial over recent rows + current token */
    {
        int64_t n = n_recent + 1;
        double m = -INFINITY, l = 0.0;
        for (int64_t t = 0; t < n; ++t) {
            const float *k = t < n_recent ? recent_k + t * d : k_n;
            double dot = 0.0;
            for (int j = 0; j < d; ++j) dot += (double)k[j] * q[j];
            s[t] = scale * dot;
            if (s[t] > m) m = s[t];
        }
        memset(acc, 0, sizeof(double) * (size_t)d);
        for (int64_t t = 0; t < n; ++t) {
            const float *v = t < n_recent ? recent_v + t * d : v_n;
            double p = exp(s[t] - m);
            l += p;
            for (int j = 0; j < d; ++j) acc[j] += p * (double)v[j];
        }
        merge_into(&res, m, l, acc, d);
    }
    int rc = 0;
    if (res.l <= 0.0) rc = 3;
    else
        for (int j = 0; j < d; ++j) out[j] = res.acc[j] / res.l;
    free(lut); free(h); free(s); free(acc); free(racc);
    return rc;
}

/* Many independent heads (same codebooks), spread over `threads` POSIX
 * threads with a shared atomic head counter: the all-cores CPU baseline.
 * Head h uses q + h*d, codes + h*ld_codes tokens, recent + h*n_recent*d. */
typedef struct {
    const double *q; const float *k_n, *v_n; const void *codes_k, *codes_v;
    int64_t n_q, ld_codes; const float *recent_k, *recent_v; int64_t n_recent;
    const float *cents_k, *cents_v; int M, nbits, dsub; double scale; int64_t block_size;
    double *out; int heads; int next; int rc; pthread_mutex_t mu;
} mt_job_t;

static void *mt_worker(void *arg) {
    mt_job_t *j = (mt_job_t *)arg;
    const int d = j->M * j->dsub;
    const size_t cell = j->nbits <= 8 ? 1 : 2;
    for (;;) {
        pthread_mutex_lock(&j->mu);
        int hh = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (hh >= j->heads) break;
        int rc = oracle_decode_head(j->q + (size_t)hh * d, j->k_n + (size_t)hh * d, j->v_n + (size_t)hh * d,
                                    (const char *)j->codes_k + (size_t)hh * j->ld_codes * j->M * cell,
                                    (const char *)j->codes_v + (size_t)hh * j->ld_codes * j->M * cell, j->n_q,
                                    j->recent_k + (size_t)hh * j->n_recent * d,
                                    j->recent_v + (size_t)hh * j->n_recent * d, j->n_recent, j->cents_k,
                                    j->cents_v, j->M, j->nbits, j->dsub, j->scale, j->block_size,
                                    j->out + (size_t)hh * d);
        if (rc) {
            pthread_mutex_lock(&j->mu);
            j->rc = rc;
            pthread_mutex_unlock(&j->mu);
        }
    }
    return NULL;
}

int oracle_decode_heads_mt(const double *q, const float *k_n, const float *v_n,
                           const void *codes_k, const void *codes_v, int64_t n_q,
                           int64_t ld_codes, const float *recent_k, const float *recent_v,
                           int64_t n_recent, const float *cents_k, const float *cents_v,
                           int M, int nbits, int dsub, double scale, int64_t block_size,
                           double *out, int heads, int threads) {
    mt_job_t j = {q, k_n, v_n, codes_k, codes_v, n_q, ld_codes, recent_k, recent_v, n_recent,
                  cents_k, cents_v, M, nbits, dsub, scale, block_size, out, heads, 0, 0,
                  PTHREAD_MUTEX_INITIALIZER};
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    for (int t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, mt_worker, &j);
    mt_worker(&j);
    for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
    return j.rc;
}

/* The batched GQA layout of the GPU path: query head (b, h) reads KV head
 * (b, h / (Hq / Hkv)); codes [B][Hkv][ld_codes][M], n_q[b] tokens; recent rows
 * [B][Hkv][ld_recent][d] with n_recent[b] live; k_n / v_n [B][Hkv][d];
 * q [B][Hq][d] fp64 -> out [B][Hq][d].  Per query head this is the
 * reference's snapshot -> build_key_lut -> quantized / dense partials ->
 * merge -> finalize (no append per query head). */
typedef struct {
    const double *q; const float *k_n, *v_n; const void *codes_k, *codes_v;
    int B, Hq, Hkv; const int32_t *n_q; int64_t ld_codes;
    const float *recent_k, *recent_v; const int32_t *n_recent; int64_t ld_recent;
    const float *cents_k, *cents_v; int M, nbits, dsub; double scale; int64_t block_size;
    double *out; int next; int rc; pthread_mutex_t mu;
} gqa_job_t;

static void *gqa_worker(void *arg) {
    gqa_job_t *j = (gqa_job_t *)arg;
    const int d = j->M * j->dsub, G = j->Hq / j->Hkv;
    const size_t cell = j->nbits <= 8 ? 1 : 2;
    for (;;) {
        pthread_mutex_lock(&j->mu);
        int hh = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (hh >= j->B * j->Hq) break;
        const int b = hh / j->Hq, h = hh % j->Hq;
        const size_t kv = (size_t)b * j->Hkv + h / G;
        int rc = oracle_decode_head(
            j->q + (size_t)hh * d, j->k_n + kv * d, j->v_n + kv * d,
            (const char *)j->codes_k + kv * j->ld_codes * j->M * cell,
            (const char *)j->codes_v + kv * j->ld_codes * j->M * cell, j->n_q[b],
            j->recent_k + kv * j->ld_recent * d, j->recent_v + kv * j->ld_recent * d,
            j->n_recent[b], j->cents_k, j->cents_v, j->M, j->nbits, j->dsub, j->scale,
            j->block_size, j->out + (size_t)hh * d);
        if (rc) {
            pthread_mutex_lock(&j->mu);
            j->rc = rc;
            pthread_mutex_unlock(&j->mu);
        }
    }
    return NULL;
}

int oracle_decode_gqa_mt(const double *q, const float *k_n, const float *v_n,
                         const void *codes_k, const void *codes_v, int B, int Hq, int Hkv,
                         const int32_t *n_q, int64_t ld_codes, const float *recent_k,
                         const float *recent_v, const int32_t *n_recent, int64_t ld_recent,
                         const float *cents_k, const float *cents_v, int M, int nbits, int dsub,
                         double scale, int64_t block_size, double *out, int threads) {
    if (Hkv <= 0 || Hq % Hkv) return 1;
    gqa_job_t j = {q, k_n, v_n, codes_k, codes_v, B, Hq, Hkv, n_q, ld_codes, recent_k,
                   recent_v, n_recent, ld_recent, cents_k, cents_v, M, nbits, dsub, scale,
                   block_size, out, 0, 0, PTHREAD_MUTEX_INITIALIZER};
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    for (int t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, gqa_worker, &j);
    gqa_worker(&j);
    for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
    return j.rc;
}

/* numpy's pairwise float64 row sum (np.sum(..., axis=1), the order used by
 * pq_core.py:163,165): < 8 terms sequential from 0.0; <= 128 terms with 8
 * strided accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a
 * sequential tail; longer rows split in halves rounded down to a multiple of 8.
 * Verified bit-for-bit against numpy in this container for n in 3..17. */
static double np_pairwise_sum(const double *a, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r += a[i];
        return r;
    }
    if (n <= 128) {
        double r[8];
        int i;
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

/* assign_codes in fp64 with the reference's rounding sequence. */
int oracle_assign_codes(const float *X, int64_t n, const float *cents, int M, int nbits,
                        int dsub, void *codes, int threads) {
    const int ksub = 1 << nbits, d = M * dsub;
    double *cc = (double *)malloc(sizeof(double) * (size_t)M * ksub);
    double *sq = (double *)malloc(sizeof(double) * (size_t)dsub);
    if (!cc || !sq) return 2;
    for (int i = 0; i < M; ++i)
        for (int c = 0; c < ksub; ++c) {
            for (int j = 0; j < dsub; ++j) {
                double v = cents[((size_t)i * ksub + c) * dsub + j];
                sq[j] = v * v;
            }
            cc[(size_t)i * ksub + c] = np_pairwise_sum(sq, dsub);
        }
    for (int64_t t = 0; t < n; ++t) {
        for (int i = 0; i < M; ++i) {
            const float *x = X + t * d + i * dsub;
            for (int j = 0; j < dsub; ++j) sq[j] = (double)x[j] * (double)x[j];
            double xx = np_pairwise_sum(sq, dsub);
            int best = 0;
            double bd = INFINITY;
            for (int c = 0; c < ksub; ++c) {
                const float *cv = cents + ((size_t)i * ksub + c) * dsub;
                double xc = 0.0;
                for (int j = 0; j < dsub; ++j) xc += (double)x[j] * (double)cv[j];
                double d2 = (xx - 2.0 * xc) + cc[(size_t)i * ksub + c];
                if (d2 < 0.0) d2 = 0.0;
                if (d2 < bd) { bd = d2; best = c; }
            }
            if (nbits <= 8) ((uint8_t *)codes)[t * M + i] = (uint8_t)best;
            else ((uint16_t *)codes)[t * M + i] = (uint16_t)best;
        }
    }
    (void)threads; /* single-threaded: the reference encoder's hot loop is serial */
    free(cc);
    free(sq);
    return 0;
}
