/*
 * dessert_b200 -- C ABI of the B200-native DESSERT vector-set search hot path.
 *
 * Every entry point takes plain device pointers (caller-owned, e.g. torch
 * tensors' data_ptr()), sizes, and a cudaStream_t passed as void*.  Calls are
 * asynchronous on that stream unless stated otherwise.  Return value: 0 on
 * success, a DSRT_E* status otherwise; dsrt_last_error() returns a
 * thread-local message whose prefix matches the reference's ValueError text
 * ("invalid parameter", "dimension mismatch", ...), so a host shim can re-raise
 * the reference's exception types unchanged.  No C++ exception crosses the ABI.
 *
 * The reference (/root/reference/pkg/src/dessert) is pure Python/numpy and has
 * no FFI; each entry point below names the Python function it replaces.  The
 * ctypes binding a maintainer would add to the reference is in INTEGRATION.md.
 *
 * Device data layout ("plane records"): a vector's L codes of C
 * bits are stored bit-sliced -- W = ceil(L/32) words per bit plane, plane b of
 * word w holds bit b of codes 32w..32w+31 -- in a record of
 * R = dsrt_record_words(L, C) uint32 words (C*W rounded up to a multiple of 4,
 * i.e. 16-byte aligned records).  A set is a contiguous run of records;
 * set_off[N+1] (int64) gives the CSR boundaries.
 */
#ifndef DESSERT_B200_H
#define DESSERT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum dsrt_status {
    DSRT_OK = 0,
    DSRT_EINVAL = 1,       /* bad argument -> ValueError                */
    DSRT_ECUDA = 2,        /* CUDA runtime / launch error -> RuntimeError */
    DSRT_EUNSUPPORTED = 3, /* shape outside what the kernels implement   */
    DSRT_ERANGE = 4        /* index out of range -> IndexError           */
};

/* element types of vector inputs */
enum dsrt_dtype { DSRT_F32 = 0, DSRT_F64 = 1, DSRT_F16 = 2, DSRT_BF16 = 3 };

/* hashing arithmetic (K1) */
enum dsrt_hash_mode {
    DSRT_HASH_F64 = 0,      /* planes float64 (L*C, d); DFMA accumulation         */
    DSRT_HASH_F32 = 1,      /* planes float32 (L*C, d); FFMA accumulation         */
    DSRT_HASH_TC_FIX = 2,   /* tcgen05 kind::f16, one fp16 pass + exact fix-up of the bits
                               near zero; planes float64 (L*C, d) (the reference's);
                               X fp16 or bf16; d = 128, C <= 8, L*C <= ~600        */
    DSRT_HASH_TC_BF16X2 = 3, /* tcgen05 kind::f16; planes bf16 hi/lo (2, L*C, d), X bf16 */
    DSRT_HASH_TC_F16X2 = 4   /* tcgen05 kind::f16; planes fp16 hi/lo (2, L*C, d), X fp16 */
};

const char *dsrt_last_error(void);
int dsrt_version(void);
/* uint32 words per plane record for (L, C); 0 if out of range. */
int dsrt_record_words(int L, int C);
/* SM count etc. of the current device (host call, synchronous). */
int dsrt_device_info(int *sm_count, int *cc_major, int *cc_minor, size_t *free_bytes);
/* Stream-ordered copy between caller-owned buffers (device or page-locked host;
 * cudaMemcpyDefault).  The batched query path stages its query vectors and its
 * top-k results through pinned host buffers with this call, so those copies can
 * be captured into the same CUDA graph as the kernels (replaces the host-side
 * np.asarray / list building around index.py:264-319's device work). */
int dsrt_copy_async(void *dst, const void *src, size_t bytes, void *stream);
/* Concatenate up to four small device buffers (byte counts multiples of 4, each
 * segment placed at the next 16-byte boundary of dst) with one kernel; dst may be
 * page-locked host memory (written over the bus, visible after the stream is
 * synchronised).  Used to return a query's (scores, ids, zero-row flag, candidate
 * count) with one graph node instead of four device-to-host copies. */
int dsrt_pack4_async(void *dst, const void *src0, size_t n0, const void *src1, size_t n1,
                     const void *src2, size_t n2, const void *src3, size_t n3, void *stream);

/*
 * K1 -- replaces lsh.hash_matrix (lsh.py:90-106) and hash_vector (lsh.py:80-87).
 * X: (n, d) row-major of x_dtype.  planes: per mode above.  Outputs (either may
 * be NULL): codes (n, L) of width 1/2/4 bytes for C<=8/<=16/<=24, and plane
 * records (n, R).  zero_rows (may be NULL): device uint32 counter incremented
 * per all-zero row (the reference raises "zero vector").
 */
int dsrt_hash(const void *X, int x_dtype, int64_t n, int d, const void *planes, int mode, int L,
              int C, void *codes_out, uint32_t *records_out, uint32_t *zero_rows, void *stream);

/*
 * K2 -- replaces the per-set build_tiny_table loop (index.py:142-145,
 * sketch.py:51-80) by the device layout.
 *   dsrt_codes_to_records: (n, L) codes of width code_bytes -> plane records;
 *     bad_codes (may be NULL) counts codes >= 2^C ("code out of range").
 *   dsrt_sizes_to_offsets: exclusive scan of set sizes -> set_off (N+1);
 *     bad (may be NULL) counts sizes < 1 ("empty set") or > 65535 ("set too large").
 *   dsrt_counting_sort: vectors tagged with set ids (any order) -> set_off (N+1)
 *     and a stable permutation perm (n) grouping vectors by set (counting sort:
 *     histogram + scan for the offsets, stable LSD radix scatter for perm).
 *     workspace from dsrt_counting_sort_workspace.
 *   dsrt_gather_rows: dst[i] = src[perm[i]] for rows of row_bytes (multiple of 4).
 */
int dsrt_codes_to_records(const void *codes, int code_bytes, int64_t n, int L, int C,
                          uint32_t *records_out, uint32_t *bad_codes, void *stream);
int dsrt_sizes_to_offsets(const int64_t *sizes, int64_t n_sets, int64_t *set_off_out,
                          uint32_t *bad, void *workspace, size_t workspace_bytes, void *stream);
size_t dsrt_scan_workspace(int64_t n_sets);
int dsrt_counting_sort(const int64_t *set_of_vec, int64_t n, int64_t n_sets, int64_t *set_off_out,
                       int64_t *perm_out, void *workspace, size_t workspace_bytes, void *stream);
size_t dsrt_counting_sort_workspace(int64_t n, int64_t n_sets);
int dsrt_gather_rows(const void *src, int64_t row_bytes, const int64_t *perm, int64_t n, void *dst,
                     void *stream);
/*
 * TinyTable export (replaces build_tiny_table, sketch.py:51-80, for one set of
 * the device layout): offsets (L, 2^C + 1) and ids (L, m) as int32, with
 * bucket (t, h) = ids[t, offsets[t,h]:offsets[t,h+1]] in ascending vector id
 * (the reference's stable counting sort).  codes: (n_vec, L) of code_bytes.
 */
int dsrt_tinytable(const void *codes, int code_bytes, const int64_t *set_off, int64_t set, int L,
                   int C, int32_t *offsets_out, int32_t *ids_out, void *stream);

/*
 * accumulate_collisions(_batch) (sketch.py:92-153) on one TinyTable:
 * counts[q, j] = |{t : stored code of j in table t == qcodes[q, t]}|.
 * offsets (L, r+1), ids (L, m), qcodes (m_q, L) as int32 (codes validated by
 * the caller); counts (m_q, m) int32.
 */
int dsrt_collision_counts(const int32_t *offsets, const int32_t *ids, int L, int r, int m,
                          const int32_t *qcodes, int m_q, int32_t *counts, void *stream);

/*
 * K3 -- replaces _score_one/_score_chunk/score_candidate (index.py:183-261) for
 * sigma = max with default weights:
 *   score = pairwise_sum_f64(lut[c_q], q < m_q) / m_q,
 *   c_q   = max_j sum_t [code_q[t] == code_j[t]].
 * lut: (L+1) float64 from build_sim_lookup (host-computed bytes).
 *
 * dsrt_score_all: every query set against sets [set_begin, set_end):
 *   scores[q * ld + (s - set_begin)].
 * dsrt_score_candidates: query set q against cand[q * cand_ld + e] for
 *   e < n_cand[q] (n_cand may be NULL: all cand_ld; cand may be NULL: identity);
 *   scores[q * cand_ld + e].
 * maxcounts (may be NULL): uint16 c_q at [(q * ld_or_cand_ld + e) * m_q + qi].
 * qrecords: (n_qsets, m_q, R) plane records of the query codes.
 * Any C <= 24 and L: shapes outside the register-blocked kernels (C > 16 or
 * C * ceil(L/32) > 32) are scored by the general kernel (same bytes); maxcounts
 * must be NULL for them (DSRT_EUNSUPPORTED otherwise).
 */
int dsrt_score_all(const uint32_t *records, const int64_t *set_off, int64_t set_begin,
                   int64_t set_end, const uint32_t *qrecords, int64_t n_qsets, int m_q, int L,
                   int C, const double *lut, double *scores, int64_t ld, uint16_t *maxcounts,
                   void *stream);
int dsrt_score_candidates(const uint32_t *records, const int64_t *set_off, int64_t n_sets,
                          const int64_t *cand, const int32_t *n_cand, int64_t cand_ld,
                          const uint32_t *qrecords, int64_t n_qsets, int m_q, int L, int C,
                          const double *lut, double *scores, uint16_t *maxcounts, void *stream);

/*
 * K3g -- general aggregation (index.py:170-216 _sim_table_for/_score_one for
 * every Scorer): inner_kind 0 = sigma max, 1 = avg-phi; weights (m_q float64,
 * NULL = all ones, scoring.py:93-97 Scorer.weights).  table = (L+1) float64:
 * the lookup table for max, phi(lookup table) for avg-phi (host-computed).
 *   max:     per_query[q] = table[max_j c_qj]
 *   avg-phi: per_query[q] = reduceat-sum(table[c_qj] : c_qj > 0, j ascending) / m
 *   score    = mean(w * per_query)   (numpy pairwise order throughout)
 * Targets as dsrt_score_candidates (cand NULL: identity; n_cand NULL: all
 * cand_ld; entries e >= n_cand[q] unwritten; invalid set index -> NaN).
 * inner_kind 0 runs on the K3 kernels (weights folded into their epilogue);
 * avg-phi on a general kernel.  m_cap bounds the target set size for avg-phi
 * (its per-lane count scratch); L <= 128, C <= 16.
 */
size_t dsrt_score_agg_workspace(int64_t n_qsets, int64_t cand_ld, int m_q, int64_t m_cap);
int dsrt_score_agg(const uint32_t *records, const int64_t *set_off, int64_t n_sets,
                   const int64_t *cand, const int32_t *n_cand, int64_t cand_ld,
                   const uint32_t *qrecords, int64_t n_qsets, int m_q, int L, int C,
                   int inner_kind, const double *table, const double *weights, int64_t m_cap,
                   double *scores, void *workspace, size_t ws_bytes, void *stream);

/*
 * K4 -- replaces heapq.nsmallest(top_k, ..., key=(-score, doc_id)) (index.py:314-319).
 * Row r: scores[r * ld + i], i < n (n_valid[r] if given).  ids: doc id of
 * element i -- shared (ids[i]) if ids_ld == 0, else ids[r * ids_ld + i]; NULL
 * means id = i.  Outputs (k per row, padded with score -1 / id UINT64_MAX /
 * pos -1 when fewer are valid): out_scores, out_ids, out_pos (element index).
 */
int dsrt_topk(const double *scores, int64_t ld, const uint64_t *ids, int64_t ids_ld,
              const int32_t *n_valid, int64_t n, int64_t n_rows, int k, double *out_scores,
              uint64_t *out_ids, int64_t *out_pos, void *stream);
int dsrt_topk_max_k(void);
/*
 * dsrt_topk for candidate lists: the id of element i of row r is
 * ids[id_index[r * id_index_ld + i]] (doc ids of the candidate set indices),
 * read in the kernel instead of a separate gather.  Elements i < n_valid[r]
 * must hold valid indices.
 */
int dsrt_topk_indexed(const double *scores, int64_t ld, const uint64_t *ids, const int64_t *id_index,
                      int64_t id_index_ld, const int32_t *n_valid, int64_t n, int64_t n_rows, int k,
                      double *out_scores, uint64_t *out_ids, int64_t *out_pos, void *stream);

/*
 * Exhaustive search = K3 + K4 fused through survivor lists (search.cu):
 * replaces query()'s exhaustive branch, _score_chunk over every set plus
 * heapq.nsmallest(top_k, key=(-score, doc_id)) (index.py:250-261, 302-319),
 * for n_qsets query sets at once, without materialising the score matrix.
 * sigma = max with optional weights (m_q float64 or NULL).  Outputs
 * out_scores / out_ids (n_qsets, k) as dsrt_topk (padding -1.0 / UINT64_MAX).
 * mode 0: threshold rounds when profitable (K3 epilogue appends sets whose
 * score reaches the running k-th best); mode 1: materialised chunks of at most
 * score_buffer_bytes, merged by K4.  *overflow (device int32) is set when a
 * survivor list overflowed in mode 0: results are then invalid and the caller
 * reruns with mode 1.  No host synchronisation inside (graph-capturable).
 */
size_t dsrt_search_all_workspace(int64_t n_sets, int64_t n_qsets, int m_q, int k, int mode,
                                 size_t score_buffer_bytes);
int dsrt_search_all(const uint32_t *records, const int64_t *set_off, int64_t n_sets,
                    const uint64_t *doc_ids, const uint32_t *qrecords, int64_t n_qsets, int m_q,
                    int L, int C, const double *lut, const double *weights, int k, int mode,
                    size_t score_buffer_bytes, double *out_scores, uint64_t *out_ids,
                    int32_t *overflow, void *workspace, size_t ws_bytes, void *stream);
/*
 * Measurement hook: while enabled, every launch of dsrt_search_all is bracketed
 * by CUDA events on its stream; _read synchronises on them and returns the
 * summed milliseconds of the scoring launches and of the top-k / list launches
 * and the number of launch calls timed since the last read (then resets).
 */
void dsrt_search_profile(int enable);
int dsrt_search_profile_read(double *score_ms, double *other_ms, int64_t *launches);

/*
 * K5 -- replaces prefilter.filter_candidates (prefilter.py:111-144).
 * Q: (n_qsets * m_q, d) float64 query vectors; centroids (k_c, d) float64.
 * postings CSR: post_off (k_c + 1), post_docs (ascending doc indices).
 * Output per query set: cand[q * k_filter + e] (count desc, index asc) and
 * n_cand[q].  workspace from dsrt_prefilter_workspace.  Any probe and k_filter:
 * probe > 32, k_filter > 16384 or m_q * probe > 65535 run a general path
 * (float64 sims + K4 selections, temporaries allocated stream-ordered).
 */
int dsrt_prefilter(const double *Q, int64_t n_qsets, int m_q, int d, const double *centroids,
                   int64_t k_c, const int64_t *post_off, const int64_t *post_docs, int64_t n_docs,
                   const int64_t *chunk_bounds, int probe, int k_filter, int64_t *cand,
                   int32_t *n_cand, void *workspace, size_t workspace_bytes, void *stream);
size_t dsrt_prefilter_workspace(int64_t n_qsets, int m_q, int64_t k_c, int64_t n_docs, int probe);
/*
 * K5, tensor-core screen (same results as dsrt_prefilter): tcgen05 fp16 GEMM of
 * normalised Q rows against centroids_f16 = fp16(centroids / cent_max_norm).
 * The GEMM pass keeps each row's probe-th best 32-column chunk maximum A'_P and
 * records every chunk maximum; every centroid of a chunk reaching
 * A'_P - 2 eps (eps = the screen's rigorous error bound) is re-approximated
 * from the same fp16 operands and kept if >= A'_P - 2 eps (a second GEMM pass
 * collects them instead when the chunk-maximum buffer would exceed 1 GB).  The
 * kept centroids are re-ranked in float64 (ties -> lower centroid id); rows with
 * more than 32 fall back to the exact float64 scan.  Selection as
 * dsrt_prefilter.  d = 128; probe > 12 or k_filter > 16384 take the general path.
 */
int dsrt_prefilter_tc(const double *Q, int64_t n_qsets, int m_q, int d, const double *centroids,
                      const void *centroids_f16, double cent_max_norm, int64_t k_c,
                      const int64_t *post_off, const int64_t *post_docs, int64_t n_docs,
                      const int64_t *chunk_bounds, int probe, int k_filter, int64_t *cand,
                      int32_t *n_cand, void *workspace, size_t workspace_bytes, void *stream);
/*
 * Posting chunk boundaries for the counting pass (postings are doc-ascending):
 * out[c * (nch + 1) + j] = index in post_docs of the first doc >= j * D in
 * posting c, D = the counting chunk (64 KB of counters), nch = chunks of n_docs.
 * Depend only on the postings and the counter width (m_q * probe), so callers
 * compute them once per index and pass them as chunk_bounds (NULL: per call).
 */
int64_t dsrt_posting_chunk_bounds_size(int64_t k_c, int64_t n_docs, int m_q, int probe);
int dsrt_posting_chunk_bounds(const int64_t *post_off, const int64_t *post_docs, int64_t k_c,
                              int64_t n_docs, int m_q, int probe, int64_t *out, void *stream);
size_t dsrt_prefilter_tc_workspace(int64_t n_qsets, int m_q, int64_t k_c, int64_t n_docs, int probe);
/* rows of float64 -> fp16 (scale > 0: multiply by scale; scale <= 0: normalise each row) */
int dsrt_to_f16_rows(const double *src, int64_t n, int d, double scale, void *dst, void *stream);
/* rows of float64 -> bf16 times scale (> 0) */
int dsrt_to_bf16_rows(const double *src, int64_t n, int d, double scale, void *dst, void *stream);

/*
 * K7 -- train_centroids (prefilter.py:47-82): spherical Lloyd iterations in
 * float64, deterministic (no atomics), in the reference's operation order:
 * unit rows (numpy norm), init = unit rows[init_idx] (init_idx: k indices
 * from np.random.default_rng(seed).choice(n, k, replace=False), computed by
 * the caller), per iteration exact argmax assignment (K6 screen for d = 128,
 * SIMT scan otherwise), sequential per-centroid sums in sample order
 * (np.add.at), pairwise norms, dead clusters reseeded from the stable argsort
 * of the best similarities.  centroids_out: (k, d) float64.  d <= 1024.
 * Errors in the reference's order: zero vector, k < 1, n < k, iters < 1.
 */
size_t dsrt_train_centroids_workspace(int64_t n, int d, int64_t k);
int dsrt_train_centroids(const double *samples, int64_t n, int d, int64_t k, int iters,
                         const int64_t *init_idx, double *centroids_out, void *workspace,
                         size_t ws_bytes, void *stream);

/*
 * .dsri index files (storage.py:130-260, sketch.py:192-239) from / to the
 * device layout.
 * dsrt_dsri_write_sets: the sets section -- per set s at byte rec_off[s] of
 *   out: doc id u64, TinyTable header (m, L, r, flags u32, 0 u64), offsets
 *   (L, r+1) and ids (L, m), u8/u16 LE by m -- built from the plane records
 *   with a stable per-(set, table) counting sort.  C <= 12.
 * dsrt_postings_to_varints: prefilter postings CSR -> the varint stream
 *   (count, then doc-id deltas, per centroid); out NULL = length only.
 * dsrt_dsri_scan_sets (HOST memory, no GPU): walk the set headers of buf
 *   from pos; per set doc id, m and TinyTable position; stops at the first
 *   header failure (err_kind 1..6, see storage.cu).  Returns sets parsed.
 * dsrt_dsri_decode_sets: validate (offsets span 0..m, monotone, ids a
 *   permutation) and decode codes (n_vec, L) for the parsed sets;
 *   *first_bad = -1 or (set << 2 | kind) of the first failing set.
 * dsrt_varints_to_postings: varint stream -> postings CSR (ERANGE: truncated).
 */
int dsrt_dsri_write_sets(const uint32_t *records, const int64_t *set_off, const uint64_t *doc_ids,
                         int64_t n_sets, int L, int C, const int64_t *rec_off, uint8_t *out,
                         void *stream);
size_t dsrt_varint_workspace(int64_t n_vals);
int dsrt_postings_to_varints(const int64_t *post_off, const int64_t *post_docs, int64_t k,
                             int64_t total, uint8_t *out, int64_t *n_bytes, void *workspace,
                             size_t ws_bytes, void *stream);
int64_t dsrt_dsri_scan_sets(const uint8_t *buf, size_t len, size_t pos, int64_t n_sets, int L,
                            int C, uint64_t *doc_ids, int64_t *sizes, int64_t *tt_off,
                            uint32_t *hdr_out, int *err_kind, size_t *end_pos);
int dsrt_dsri_decode_sets(const uint8_t *buf, const int64_t *tt_off, const int64_t *set_off,
                          int64_t n_sets, int L, int C, int64_t m_max, void *codes,
                          int code_bytes, int64_t *first_bad, void *stream);
int dsrt_varints_to_postings(const uint8_t *bytes, int64_t n_bytes, int64_t k, int64_t *post_off,
                             int64_t *post_docs, int64_t *total_out, void *workspace,
                             size_t ws_bytes, void *stream);

/*
 * K6 -- centroid assignment for build_centroid_index (prefilter.py:85-108):
 * assign[i] = argmax_c <X[i], centroids[c]> (lowest c on ties, as np.argmax),
 * exact.  d = 128: tensor-core screen + float64 re-rank + exact fallback (X
 * of x_dtype: fp16/bf16 rows are read in place; f32/f64 are normalised into
 * an fp16 staging buffer; cents_lp = fp16 (bf16 for bf16 X) copy of
 * centroids / max_c |c|).  Other d (<= 1024): float64 unit rows in numpy's
 * order and a sequential-FMA SIMT scan (cents_lp unused); zero rows -> EINVAL.
 */
int dsrt_assign_centroids(const void *X, int x_dtype, int64_t n, int d, const double *centroids,
                          const void *cents_lp, int64_t k_c, int32_t *assign_out, void *workspace,
                          size_t workspace_bytes, void *stream);
size_t dsrt_assign_centroids_workspace(int64_t n, int d, int64_t k_c);
/*
 * Append postings of new documents (ids all >= those of the old postings) to
 * an existing CSR: posting c = old posting c followed by added posting c.
 * new_off (k_c + 1), new_docs (old_total + add_total).
 */
int dsrt_merge_postings(const int64_t *old_off, const int64_t *old_docs, const int64_t *add_off,
                        const int64_t *add_docs, int64_t k_c, int64_t *new_off, int64_t *new_docs,
                        void *stream);
/*
 * Postings from assignments: vectors grouped by document (set_off, N+1);
 * post_off (k_c + 1), post_docs (capacity n_vec), *n_post (device int64):
 * posting c = ascending, deduplicated documents having a vector assigned to c.
 */
int dsrt_postings_from_assign(const int32_t *assign, int64_t n_vec, const int64_t *set_off,
                              int64_t n_docs, int64_t k_c, int64_t *post_off, int64_t *post_docs,
                              int64_t *n_post, void *workspace, size_t workspace_bytes,
                              void *stream);
size_t dsrt_postings_workspace(int64_t n_vec, int64_t k_c);

/* Diagnostic: D(M,N) f32 = A(M,128) . B(N,128)^T on the tcgen05 path (TMA ->
 * 128B-swizzled smem -> UMMA -> TMEM -> tcgen05.ld); fp16 (0) or bf16 (1)
 * operands, 16 <= N <= 256.  Validates the tensor-core plumbing K1/K5 use. */
int dsrt_tc_selftest(const void *A, int a_bf16, const void *B, int b_bf16, float *D, int M, int N,
                     void *stream);

/* Microbenchmark of the INT pipe (LOP3 / POPC / IMNMX lane-ops per second);
 * host call, synchronous.  Writes ops/s for {lop3, popc, imnmx, mixed}. */
int dsrt_microbench_int(double *ops_per_s_out4, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* DESSERT_B200_H */
