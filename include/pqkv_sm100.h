/*
 * pqkv_sm100.h -- C ABI of the B200 (sm_100a) product-quantized KV-cache hot
 * path: KV encode, key lookup tables, quantized-span decode attention and the
 * log-sum-exp merge of softmax partials.
 *
 * Every entry point replaces a function of the reference package `pqkv`
 * (paths relative to the reference's pkg/src/pqkv/); the citation is on each
 * declaration.  Conventions:
 *   - all pointers are DEVICE pointers unless stated otherwise; sizes are in
 *     elements; no entry point allocates, synchronises or keeps global
 *     mutable state beyond a per-thread error string;
 *   - work is enqueued on `stream` (a cudaStream_t passed as void*; NULL means
 *     the legacy default stream) and is asynchronous;
 *   - the return value is 0 on success, PQKV_EINVAL for a bad argument
 *     (the reference raises ValueError) and PQKV_ECUDA for a CUDA launch
 *     error; pqkv_last_error() returns the calling thread's last message.
 *
 * Geometry: d = M * dsub, ksub = 2^nbits.  Codes are token-major rows of M
 * cells (uint8 when nbits <= 8 else uint16), exactly the reference's
 * CodesMatrix layout (pq_core.py:114-145).  Codebooks are (M, ksub, dsub)
 * float32, subspace-major (pq_core.py:86-111).
 */
#ifndef PQKV_SM100_H
#define PQKV_SM100_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PQKV_OK 0
#define PQKV_EINVAL 1
#define PQKV_ECUDA 2
#define PQKV_EFORMAT 3 /* malformed file: the reference's FormatError */
#define PQKV_EIO 4     /* file cannot be opened / read / written: OSError */

#define PQKV_DTYPE_F32 0
#define PQKV_DTYPE_BF16 1
#define PQKV_DTYPE_F16 2

/* Floats per softmax-partial record: (m, l, 2 pad, acc[d]) -> d + 4.
 * Mirrors SoftmaxPartial (attention.py:46-53); empty = (-inf, 0, 0). */
#define PQKV_PARTIAL_HEADER 4

int pqkv_version(void);
const char *pqkv_last_error(void);

/* Code layouts.  PQKV rows: token-major rows of M cells in subspace order,
 * the reference's CodesMatrix.  Decode layout (m64b8 only): the same rows
 * with each 16-byte quarter q of token t stored rotated, subspace i at byte
 * 16q + ((i - r) & 15), r = ((l & 15) + (l >> 4)) & 15, l = 4 (t & 7) + q;
 * the decode kernel's lanes then read their bytes in register order and still
 * hit 32 distinct shared-memory banks per step.  t counts rows from the start
 * of the buffer handed to the decode kernel.  A per-row bijection. */

/* Nearest-centroid encoder, bit-exact with assign_codes (pq_core.py:269-287
 * on top of _squared_distances :158-168): fp64 d2 = (|x|^2 - 2 x.c) + |c|^2
 * with numpy's pairwise norms and a sequential x.c, clamped at 0, lowest
 * index on ties.  x: n rows of d values (row stride ld_x elements, dtype
 * PQKV_DTYPE_*); codes: n rows of M cells, row stride ld_codes cells.
 * rot_base < 0 writes the row layout; rot_base >= 0 writes the decode layout
 * with row 0 being token index rot_base of the destination buffer. */
int pqkv_encode(const void *x, int x_dtype, int64_t n, int d, int64_t ld_x,
                const float *centroids, int M, int nbits, void *codes,
                int64_t ld_codes, int64_t rot_base, void *stream);

/* pqkv_encode over `batches` independent problems in one launch (e.g. the
 * layers of a cache flush, each with its own codebook): batch z reads rows at
 * x + z * x_bstride (elements), centroids at centroids + z * c_bstride and
 * writes codes at codes + z * codes_bstride (cells).  Same results as
 * `batches` pqkv_encode calls (which it falls back to off the fp32 dsub = 2
 * fast path). */
int pqkv_encode_batched(const void *x, int x_dtype, int batches, int64_t n, int d,
                        int64_t ld_x, int64_t x_bstride, const float *centroids,
                        int64_t c_bstride, int M, int nbits, void *codes, int64_t ld_codes,
                        int64_t codes_bstride, int64_t rot_base, void *stream);

/* ---- candidate grid of the dsub = 2 encoder (nbits <= 8) ----------------
 * Per subspace a 64 x 64 grid over the centroids' bounding box (+25% each
 * side); each cell lists the <= 24 centroids that can be the nearest -- or
 * within 1/128 relative of it -- for a point of the cell.  pqkv_encode_grid
 * runs pqkv_encode's fp32 filter over the cell's list instead of all ksub
 * centroids (same keys, same near-tie test, same exact fp64 re-scan over all
 * centroids on a near tie; points outside the grid and crowded cells scan all
 * of them), so its codes are pqkv_encode's -- the reference's -- bit for bit.
 * pqkv_encode_grid_bytes: bytes of a codebook's grid (0: no grid for this
 * geometry); pqkv_build_encode_grid fills it from the centroids (once per
 * codebook); grid == NULL makes pqkv_encode_grid a plain pqkv_encode.
 * pqkv_encode_batched_grid: the fp32 batched form (grid at grid + z *
 * g_bstride bytes). */
int64_t pqkv_encode_grid_bytes(int d, int M, int nbits);
int pqkv_build_encode_grid(const float *centroids, int d, int M, int nbits,
                           void *grid, void *stream);
int pqkv_encode_grid(const void *x, int x_dtype, int64_t n, int d, int64_t ld_x,
                     const float *centroids, const void *grid, int M, int nbits,
                     void *codes, int64_t ld_codes, int64_t rot_base, void *stream);
int pqkv_encode_batched_grid(const void *x, int batches, int64_t n, int d,
                             int64_t ld_x, int64_t x_bstride,
                             const float *centroids, int64_t c_bstride,
                             const void *grid, int64_t g_bstride, int M, int nbits,
                             void *codes, int64_t ld_codes,
                             int64_t codes_bstride, int64_t rot_base,
                             void *stream);

/* Convert n rows between the row layout and the decode layout (to_decode = 1:
 * rows -> decode, 0: decode -> rows); row 0 is token index t_first. */
int pqkv_relayout_codes(const void *src, int64_t ld_src, void *dst,
                        int64_t ld_dst, int64_t n, int64_t t_first,
                        int to_decode, int d, int M, int nbits, void *stream);

/* reconstruct (pq_core.py:290-304): out[t, i*dsub + j] = C[i, codes[t, i], j].
 * Test/diagnostic helper: the attention path never dequantizes. */
int pqkv_reconstruct(const void *codes, int64_t n, int64_t ld_codes,
                     const float *centroids, int d, int M, int nbits,
                     float *out, void *stream);

/* build_key_lut (attention.py:70-83) for n_heads queries at once:
 * lut[h, c, i] = scale * <q[h, i*dsub:(i+1)*dsub], C_K[i, c]>, float32,
 * stored centroid-major ([ksub][M] per head) -- the decode kernel's
 * shared-memory layout, so the kernel copies it without a transpose. */
int pqkv_build_lut(const float *q, int64_t n_heads, int d, const float *cb_k,
                   int M, int nbits, float scale, float *lut, void *stream);

/* One-time re-layouts of a layer's codebooks for the m64b8 fast path
 * (d=128, M=64, nbits=8), done at codebook load:
 *   key:   [256][64] float2 (centroid-major; the in-kernel LUT build reads it
 *          with coalesced 16-byte loads)
 *   value: [2][256][32] float2 (subspace half, centroid, subspace-in-half;
 *          the shared-memory image the value gather reads conflict-free)
 * Each output is 65536 float32.  Other geometries use the plain
 * (M, ksub, dsub) codebooks and need no call. */
int pqkv_prepare_key_codebook(const float *cb_k, int d, int M, int nbits,
                              float *out, void *stream);
int pqkv_prepare_value_codebook(const float *cb_v, int d, int M, int nbits,
                                float *out, void *stream);
/* The value codebook with fp16 entries ([256][2][32] half2, 64 KiB; round to
 * nearest) for decode launches with PQKV_DECODE_F16_VALUE_CODEBOOK: 4-byte
 * shared-memory gathers instead of 8 and fp16 softmax weights in mixed
 * f16 x f16 + f32 FMAs (no reference counterpart -- a stated-tolerance mode;
 * the sums stay fp32). */
int pqkv_prepare_value_codebook_f16(const float *cb_v, int d, int M, int nbits,
                                    void *out, void *stream);

/* Keep [base, base + bytes) -- e.g. every layer's codebook layouts in one
 * allocation -- resident in L2 for kernels launched on `stream` (and graphs
 * captured from it): sets the persisting-L2 carve-out and the stream's access
 * policy window (hitProp persisting, missProp streaming).  base == NULL
 * clears it.  No reference counterpart (a B200 memory-placement knob). */
int pqkv_l2_persist(const void *base, size_t bytes, float hit_ratio, void *stream);

/* Number of persistent CTAs pqkv_decode_partials uses on the current device
 * (one per SM for the fast path); needed to size the partials buffer. */
int pqkv_decode_grid(int d, int M, int nbits, int *num_ctas);

/* Floats needed for the partials workspace: (2*num_ctas + 2*B*Hq) * (d + 4)
 * (split records, then one dense-window record per head). */
int64_t pqkv_partials_floats(int num_ctas, int B, int Hq, int d);

/* Quantized-span softmax partials: the fused LUT-score + online softmax +
 * value accumulation of quantized_partial (attention.py:114-166), i.e.
 * build_key_lut (:70-83), score_codes (_kernels.py:27-34) and the value
 * aggregation (_kernels.py:37-43 + attention.py:103-111 / :155-157), for
 * every (batch b, query head hq) over tokens [0, n_q[b]) of KV head
 * hkv = hq / (Hq / Hkv).  The token space of all heads is split evenly over
 * num_ctas persistent CTAs; each (CTA, head) overlap emits one partial.
 *   q        [B*Hq][d] float32 queries, scores scaled by `scale`
 *   cb_k     fast path: pqkv_prepare_key_codebook output (the LUT is built
 *            in shared memory by the decode kernel itself);
 *            other geometries: the plain (M, ksub, dsub) codebook
 *   lut_ws   other geometries: [B*Hq][ksub][M] float32 scratch that receives
 *            the tables (pqkv_build_lut); unused (may be NULL) on the fast path
 *   codes_k/codes_v  [B][Hkv][ld_tok][M] cells; fast path: decode layout
 *   n_q      [B] int32 (device): quantized tokens per sequence
 *   cb_v     fast path: pqkv_prepare_value_codebook output; else (M,ksub,dsub)
 *   partials pqkv_partials_floats(num_ctas, B, Hq, d) floats */
int pqkv_decode_partials(const float *q, float scale, const float *cb_k,
                         float *lut_ws, int B, int Hq, int Hkv,
                         const void *codes_k, const void *codes_v,
                         int64_t ld_tok, const int32_t *n_q, const float *cb_v,
                         int d, int M, int nbits, int num_ctas,
                         float *partials, void *stream);

/* Same, from precomputed tables lut [B*Hq][ksub][M] (pqkv_build_lut) -- the
 * quantized_partial(lut, ...) form of the reference API. */
int pqkv_decode_partials_lut(const float *lut, int B, int Hq, int Hkv,
                             const void *codes_k, const void *codes_v,
                             int64_t ld_tok, const int32_t *n_q,
                             const float *cb_v, int d, int M, int nbits,
                             int num_ctas, float *partials, void *stream);

/* Finish one decode step for every (b, hq): merge that head's quantized
 * partials in a fixed order (merge_partials, attention.py:193-204), add the
 * dense partial over the full-precision recent rows plus the current token
 * (dense_partial :169-190, decode_step :264-267) and finalize (:207-211).
 *   q            [B*Hq][d] float32 (scores use `scale`)
 *   recent_k/v   [B][Hkv][ld_recent][d] float32, rows [0, n_recent[b])
 *   n_recent     [B] int32 (device) or NULL (no recent rows)
 *   k_cur/v_cur  [B][Hkv][d] float32 or NULL (no current token)
 *   out          [B*Hq][d] float32 (may be NULL)
 *   lse          [B*Hq] float32 m + log(l) (may be NULL)
 *   merged       [B*Hq][d+4] merged, un-normalised partial (may be NULL) --
 *                the record exchanged between ranks for a sequence split.
 * A head whose merged partial is empty (l == 0) gets NaN outputs (the
 * reference's finalize raises ValueError; the Python layer checks). */
int pqkv_decode_finish(const float *partials, int num_ctas, int B, int Hq,
                       int Hkv, int d, const int32_t *n_q, const float *q,
                       float scale, const float *recent_k,
                       const float *recent_v, int64_t ld_recent,
                       const int32_t *n_recent, const float *k_cur,
                       const float *v_cur, float *out, float *lse,
                       float *merged, void *stream);

/* Flags of pqkv_decode_attention. */
#define PQKV_DECODE_PDL 1 /* programmatic dependent launch: the grid may start
                             while the previous kernel on the stream drains;
                             it waits for it before touching q, lengths,
                             recent rows, counters, partials or outputs */
#define PQKV_DECODE_STATIC_CODEBOOKS 2 /* the codebooks were written before the
                             previous kernel on the stream started (e.g. at
                             load time), so they may be read before that
                             kernel finishes (with PQKV_DECODE_PDL) */
#define PQKV_DECODE_F16_VALUE_CODEBOOK 4 /* cb_v is the fp16 layout of
                             pqkv_prepare_value_codebook_f16 */
#define PQKV_DECODE_ONE_HEAD_PER_CTA 16 /* GQA: keep one query head per CTA.
                             By default the fp16 mode with an even group
                             serves two (or four) query heads of a KV head per
                             CTA, and the exact path with a group that is a
                             multiple of 4 runs clusters of two CTAs that
                             serve four query heads (each CTA one half of the
                             subspaces), sharing the value gathers */
#define PQKV_DECODE_F16_KEY_TABLE 32 /* with PQKV_DECODE_F16_VALUE_CODEBOOK
                             and an even GQA group: the query heads a CTA
                             serves keep one packed fp16 key table (entry
                             (c, i) = their scores in fp16), one gather per
                             key code for all of them; scores are summed in
                             fp32.  A group that is a multiple of 4: four
                             query heads per CTA (8-byte entries, the value
                             gathers shared by the four, fp32 weights);
                             otherwise two (4-byte entries).  Ignored for
                             odd groups. */
#define PQKV_DECODE_KEY_TABLE_PAIRS 64 /* with PQKV_DECODE_F16_KEY_TABLE: two
                             query heads per CTA even when the group is a
                             multiple of 4 */
#define PQKV_DECODE_APPEND_RECENT 128 /* one head (B = Hq = Hkv = 1, m64b8, fp32
                                      * values): after the merge the finishing CTA
                                      * appends (k_cur, v_cur) at row n_recent[0] of
                                      * recent_k / recent_v (ld_recent rows) and bumps
                                      * n_recent[0] -- pqkv_append_recent fused into
                                      * the launch (recent_k, recent_v, n_recent are
                                      * written) */
#define PQKV_DECODE_EARLY_CODES 8 /* the codes below n_q were written before
                             the previous kernel on the stream started (the
                             codes of a decode step are appended by an
                             earlier step), so the work split and the first
                             code loads may precede that kernel's end (with
                             PQKV_DECODE_PDL).  n_q itself is re-read after
                             the grid-dependency wait; if it changed, the
                             split and the loads are redone (B <= 256; larger
                             batches ignore this flag) */

/* One fused launch per layer: decode_step (attention.py:214-287) for every
 * (b, hq) -- pqkv_decode_partials' quantized span, the dense partial of the
 * recent rows + current token (dense_partial :169-190, computed by the CTA
 * holding the head's last quantized tokens), and, by the last CTA to finish
 * each head (an arrival counter), the fixed-order merge_partials (:193-204)
 * and finalize (:207-211).  Arguments as pqkv_decode_partials plus those of
 * pqkv_decode_finish, and
 *   counters  [B*Hq] int32, zero before the first call; every launch leaves
 *             them zero again (a launch must not be aborted midway)
 *   partials  pqkv_partials_floats(num_ctas, B, Hq, d) floats
 *   flags     PQKV_DECODE_* bits
 * Other geometries run pqkv_decode_partials + pqkv_decode_finish (counters
 * and flags unused). */
int pqkv_decode_attention(const float *q, float scale, const float *cb_k,
                          float *lut_ws, int B, int Hq, int Hkv,
                          const void *codes_k, const void *codes_v,
                          int64_t ld_tok, const int32_t *n_q,
                          const float *cb_v, int d, int M, int nbits,
                          const float *recent_k, const float *recent_v,
                          int64_t ld_recent, const int32_t *n_recent,
                          const float *k_cur, const float *v_cur, int num_ctas,
                          float *partials, int32_t *counters, float *out,
                          float *lse, float *merged, int flags, void *stream);

/* Merge n_parts partial records per head in index order (merge_partials,
 * attention.py:193-204; the cross-GPU log-sum-exp merge of a sequence
 * split) and optionally finalize.  parts: [n_parts][n_heads][d+4]. */
int pqkv_merge_partials(const float *parts, int n_parts, int64_t n_heads,
                        int d, float *out, float *lse, float *merged,
                        void *stream);

/* Lower seam of the reference (_kernels.py:46-53, 56-65), float32:
 *   scores[t] = sum_i lut[code[t,i], i]          (lut centroid-major [ksub][M])
 *   h[i, c]  += p[t] for code[t, i] == c          (h is zeroed first) */
int pqkv_score_codes(const float *lut, const void *codes, int64_t n, int M,
                     int nbits, float *scores, void *stream);
int pqkv_accumulate_mass(const void *codes, const float *p, int64_t n, int M,
                         int nbits, float *h, void *stream);

/* The same seam in float64 with the reference's loop orders, bit-identical
 * to _score_codes_jit / _accumulate_mass_jit (_kernels.py:27-43):
 *   scores[t] = sum over i = 0..M-1 of lut[i][code[t,i]]  (lut [M][ksub] f64,
 *               the reference Lut.table layout; summed in order from 0.0)
 *   h[i][c]   = sum over t = 0..n-1 of p[t] where code[t,i] == c  (in t order)
 * Used by the drop-in _kernels module (score_codes, accumulate_mass). */
int pqkv_score_codes_f64(const double *lut, const void *codes, int64_t n, int M,
                         int nbits, double *scores, void *stream);
int pqkv_accumulate_mass_f64(const void *codes, const double *p, int64_t n, int M,
                             int nbits, double *h, void *stream);

/* The reference API's float64 small ops on the GPU (the decode kernels keep
 * their float32 tables in shared memory):
 *   pqkv_build_lut_f64      build_key_lut (attention.py:70-83): out
 *                           [n_heads][M][ksub] f64 (the Lut.table layout),
 *                           (sum_j C[i][c][j] q[i dsub + j]) * scale
 *   pqkv_dense_partial_f64  dense_partial (:169-190) over r rows K, V
 *                           [r][d] f64 (d <= 1024): rec = (m, l, 0, 0,
 *                           acc[d]) f64 */
int pqkv_build_lut_f64(const double *q, int64_t n_heads, int d, const float *cb_k, int M,
                       int nbits, double scale, double *out, void *stream);
int pqkv_dense_partial_f64(const double *q, const double *K, const double *V, int64_t r,
                           int d, double scale, double *rec, void *stream);

/* ---- Binary formats at the boundary (fileio.py:71-160) ----------------
 * Unlike the entry points above these do file IO, allocate a pinned staging
 * buffer (and a device temporary for layout conversion) and synchronise
 * `stream` before returning.  Errors: PQKV_EFORMAT with the reference's
 * FormatError texts, PQKV_EIO for the file system.
 *
 * .pqkv codebook (read_codebook fileio.py:80-96, write_codebook :71-77):
 * "PQKV" + <IBIII (version 1, kind 0 key / 1 value, d, M, nbits), a 21-byte
 * header, then M * 2^nbits * dsub float32, subspace-major (unaligned body).
 *   pqkv_codebook_file_info  header + size check, no body read
 *   pqkv_read_codebook       body -> centroids [M][ksub][dsub] (device, or
 *                            host with PQKV_FILE_HOST) and/or, m64b8 only,
 *                            straight into the decode kernel's layout
 *                            (pqkv_prepare_key/value_codebook by the kind)
 *   pqkv_write_codebook      centroids (device, or host) -> file */
#define PQKV_FILE_HOST 1 /* the centroid pointer is host memory */
int pqkv_codebook_file_info(const char *path, int *kind, int *d, int *M, int *nbits);
int pqkv_read_codebook(const char *path, int flags, float *centroids, float *layout,
                       void *stream);
int pqkv_write_codebook(const char *path, int kind, int d, int M, int nbits,
                        const float *centroids, int flags, void *stream);

/* .pqkc cache dump (write_cache_dump fileio.py:99-114, read_cache_dump
 * :117-156): "PQKC" + <IIIIQI (version 1, d, M, nbits, n_q u64, recent_len),
 * K codes, V codes (reference row layout), recent K, recent V (float32).  A
 * file of `heads` caches (every layer x sequence x KV head of a serving
 * cache) is `heads` such records back to back.  Device buffers: head h's codes
 * at codes + h * code_stride cells (layout PQKV_CODES_ROWS, or
 * PQKV_CODES_DECODE for m64b8, converted on the device), its recent rows at
 * recent + h * recent_stride floats.  Reading checks every record's header
 * against the destination and, when a cell can hold one, out-of-range codes
 * ("corrupted dump").
 *   pqkv_cache_dump_info     header of the record at byte `offset` */
#define PQKV_CODES_ROWS 0
#define PQKV_CODES_DECODE 1
int pqkv_cache_dump_info(const char *path, int64_t offset, int *d, int *M, int *nbits,
                         int64_t *n_q, int *recent_len, int64_t *record_bytes);
int pqkv_write_cache_dumps(const char *path, int heads, int d, int M, int nbits,
                           int64_t n_q, int recent_len, const void *codes_k,
                           const void *codes_v, int64_t code_stride, int layout,
                           const float *recent_k, const float *recent_v,
                           int64_t recent_stride, void *stream);
int pqkv_read_cache_dumps(const char *path, int heads, int d, int M, int nbits,
                          int64_t n_q, int recent_len, void *codes_k, void *codes_v,
                          int64_t code_stride, int layout, float *recent_k,
                          float *recent_v, int64_t recent_stride, void *stream);

/* Test-only: one kernel that releases a following PDL launch immediately
 * (griddepcontrol.launch_dependents), waits ns nanoseconds, then writes v to
 * p[0..n).  Used to check that PQKV_DECODE_EARLY_CODES re-validates the
 * lengths it read before its grid-dependency wait. */
int pqkv_debug_delayed_fill(int32_t *p, int n, int32_t v, long long ns,
                            void *stream);

/* ---- per-token appends with device-resident lengths --------------------
 * A cache's (n_q, n_recent) as int32 lens[2] on the device, updated in stream
 * order, so that a decode step needs no host->device length transfer.
 * pqkv_append_recent replaces LayerKVCache.append_decode's row write
 * (kv_cache.py:188-200): rows n = lens[1] of rk / rv (row stride d) take the d
 * floats of k / v, then lens[1] = n + 1.  pqkv_publish_lengths is a flush's
 * single publication point (kv_cache.py:228) on the device: lens[0] += batch,
 * lens[1] -= batch (the recent base pointer the caller passes moves by batch
 * rows). */
int pqkv_append_recent(const float *k, const float *v, float *rk, float *rv,
                       int32_t *lens, int d, void *stream);

/* decode_step's per-token work for one head of a cache with device lengths
 * (attention.py:214-287 for a LayerKVCache): pqkv_decode_attention with B =
 * Hq = Hkv = 1 reading n_q = lens[0] and the recent length lens[1], then
 * pqkv_append_recent of (k_cur, v_cur) -- one call per token.  The plan holds
 * the per-cache constants (codebook layouts, code stores, lens, scale,
 * workspace); recent_k / recent_v point at the ring's first live row;
 * num_ctas > 0 caps the grid (<= the plan's; a short context wants few). */
int pqkv_step_plan_create(const float *cb_k, const float *cb_v,
                          const void *codes_k, const void *codes_v,
                          int64_t ld_tok, int32_t *lens, float scale, int d,
                          int M, int nbits, int num_ctas, float *partials,
                          int32_t *counters, void **plan);
int pqkv_step_run(void *plan, const float *q, const float *k_cur,
                  const float *v_cur, float *recent_k, float *recent_v,
                  int64_t ld_recent, int num_ctas, float *out, void *stream);
int pqkv_step_plan_destroy(void *plan);
int pqkv_publish_lengths(int32_t *lens, int batch, void *stream);

/* ---- paged code store (growth without copies) ---------------------------
 * Replaces the reference's grow-by-copy code store (kv_cache.py:74-76,
 * 217-228).  A store reserves n_regions * region_bytes of virtual address
 * space (region_bytes rounded up to the allocation granularity); region r
 * starts at base + r * region_bytes.  pqkv_vstore_ensure(bytes) maps physical
 * pages (CUDA VMM: cuMemCreate / cuMemMap, geometric growth) so that every
 * region has at least `bytes` mapped; mapped pages never move, so a head's
 * codes stay one contiguous run for the decode kernel (ld_tok = region_bytes
 * / row bytes) and the store grows without copying.  Pages are not zeroed.
 * pqkv_vstore_destroy synchronises the device, unmaps and frees. */
typedef struct pqkv_vstore pqkv_vstore;
int64_t pqkv_vstore_granularity(int device);
int pqkv_vstore_create(int device, int64_t n_regions, int64_t region_bytes,
                       pqkv_vstore **out, void **base);
int pqkv_vstore_ensure(pqkv_vstore *vs, int64_t bytes);
int64_t pqkv_vstore_mapped(const pqkv_vstore *vs);
int64_t pqkv_vstore_region_bytes(const pqkv_vstore *vs);
int pqkv_vstore_destroy(pqkv_vstore *vs);

#ifdef __cplusplus
}
#endif
#endif /* PQKV_SM100_H */
