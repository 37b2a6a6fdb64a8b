// K5 -- centroid prefilter: replaces prefilter.filter_candidates
// (prefilter.py:111-144).
//
//  A  probe_kernel:   sims = Q @ centroids^T in float64 (the reference computes
//                     the same product in float64), per query row the top
//                     `probe` centroids by (sim desc, id asc) -- the stable
//                     argsort tie rule of prefilter.py:136 -- per centroid chunk;
//  A2 merge_kernel:   merge the per-chunk winners of each row;
//  B  count_kernel:   counts[set, doc] += 1 for every (query vector, probed
//                     centroid, posting entry) (prefilter.py:138-141);
//  C  select_kernel:  touched docs by (count desc, index asc)[:k_filter]
//                     (prefilter.py:142-144): count histogram -> threshold
//                     count c*, all docs above it, the lowest-index docs at c*
//                     in one ordered pass, then a shared-memory bitonic sort.
#include "common.cuh"

namespace dsrt {

constexpr int kPRows = 32;      // query rows per CTA
constexpr int kPTile = 256;     // centroids per smem tile (= threads)
constexpr int kPDim = 16;       // dims per smem stage
constexpr int kPChunkTiles = 8; // tiles per CTA chunk (2048 centroids)
constexpr int kMaxProbe = 32;
constexpr int kSelThreads = 1024;
constexpr int kSelMax = 16384;  // max k_filter handled in shared memory

struct Cand {
    double s;
    int32_t id;
};

__device__ __forceinline__ bool better(double sa, int ia, double sb, int ib) {
    return sa > sb || (sa == sb && ia < ib);
}

// Warp-cooperative: insert (s, id) candidates held one per lane into a sorted
// top-P list kept in lanes 0..P-1 (lane i holds rank i).  P <= 32.
__device__ __forceinline__ void warp_topP_merge(double &ts, int &ti, double cs, int ci, int P) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    // repeatedly extract the best remaining candidate of the warp and insert
    for (int r = 0; r < P; ++r) {
        double bs = cs;
        int bi = ci, bl = lane;
        for (int o = 16; o > 0; o >>= 1) {
            const double os = __shfl_xor_sync(full, bs, o);
            const int oi = __shfl_xor_sync(full, bi, o);
            const int ol = __shfl_xor_sync(full, bl, o);
            if (better(os, oi, bs, bi)) {
                bs = os;
                bi = oi;
                bl = ol;
            }
        }
        // worst of current top list is at rank P-1
        const double ws = __shfl_sync(full, ts, P - 1);
        const int wi = __shfl_sync(full, ti, P - 1);
        if (!better(bs, bi, ws, wi)) break;  // nothing left improves the list
        if (lane == bl) {
            cs = -INFINITY;
            ci = 0x7fffffff;
        }
        // insert (bs, bi): find position pos = number of entries better than it
        const bool ahead = lane < P && better(ts, ti, bs, bi);
        const int pos = __popc(__ballot_sync(full, ahead));
        const double ps = __shfl_up_sync(full, ts, 1);
        const int pi = __shfl_up_sync(full, ti, 1);
        if (lane < P && lane > pos) {
            ts = ps;
            ti = pi;
        }
        if (lane == pos) {
            ts = bs;
            ti = bi;
        }
    }
}

// grid: (row tiles, centroid chunks).  256 threads; each thread owns one
// centroid of the current tile and accumulates its dot with 32 query rows.
__global__ void __launch_bounds__(kPTile)
    probe_kernel(const double *__restrict__ Q, int64_t n_rows, int d,
                 const double *__restrict__ cents, int64_t k_c, int P, Cand *__restrict__ out) {
    // dynamic smem: qs[kPDim][kPRows], then cs[kPDim][kPTile+1] aliased by sims[kPRows][kPTile+1]
    extern __shared__ __align__(16) double psm[];
    double (*qs)[kPRows] = reinterpret_cast<double (*)[kPRows]>(psm);
    double (*cs)[kPTile + 1] = reinterpret_cast<double (*)[kPTile + 1]>(psm + kPDim * kPRows);
    double (*sims)[kPTile + 1] = reinterpret_cast<double (*)[kPTile + 1]>(psm + kPDim * kPRows);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kPRows;
    const int64_t c_chunk0 = static_cast<int64_t>(blockIdx.y) * kPTile * kPChunkTiles;
    // per-warp running top-P for rows warp*4 .. warp*4+3 (lane i = rank i)
    double ts[4];
    int ti[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        ts[j] = -INFINITY;
        ti[j] = 0x7fffffff;
    }
    for (int tile = 0; tile < kPChunkTiles; ++tile) {
        const int64_t c0 = c_chunk0 + static_cast<int64_t>(tile) * kPTile;
        if (c0 >= k_c) break;
        double acc[kPRows];
#pragma unroll
        for (int r = 0; r < kPRows; ++r) acc[r] = 0.0;
        for (int k0 = 0; k0 < d; k0 += kPDim) {
            __syncthreads();
            for (int i = tid; i < kPDim * kPRows; i += kPTile) {
                const int kk = i % kPDim, r = i / kPDim;
                const int64_t gr = r0 + r;
                qs[kk][r] = (gr < n_rows && k0 + kk < d) ? Q[gr * d + k0 + kk] : 0.0;
            }
            for (int i = tid; i < kPDim * kPTile; i += kPTile) {
                const int kk = i % kPDim, c = i / kPDim;
                const int64_t gc = c0 + c;
                cs[kk][c] = (gc < k_c && k0 + kk < d) ? cents[gc * d + k0 + kk] : 0.0;
            }
            __syncthreads();
            const int kmax = min(kPDim, d - k0);
            for (int kk = 0; kk < kmax; ++kk) {
                const double cv = cs[kk][tid];
#pragma unroll
                for (int r = 0; r < kPRows; ++r) acc[r] = fma(qs[kk][r], cv, acc[r]);
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kPRows; ++r) sims[r][tid] = acc[r];
        __syncthreads();
        // warp w merges rows 4w..4w+3 over this tile's 256 centroids
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int r = warp * 4 + j;
            for (int c = lane; c < kPTile; c += 32) {
                const int64_t gc = c0 + c;
                const double s = gc < k_c ? sims[r][c] : -INFINITY;
                const int id = gc < k_c ? static_cast<int>(gc) : 0x7fffffff;
                warp_topP_merge(ts[j], ti[j], s, id, P);
            }
        }
    }
    const int64_t n_chunks = gridDim.y;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t gr = r0 + warp * 4 + j;
        if (gr < n_rows && lane < P) out[(gr * n_chunks + blockIdx.y) * P + lane] = Cand{ts[j], ti[j]};
    }
}

// one warp per row: merge n_chunks*P candidates into the final top-P ids
__global__ void merge_kernel(const Cand *__restrict__ in, int64_t n_rows, int n_chunks, int P,
                             int32_t *__restrict__ probed) {
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= n_rows) return;
    double ts = -INFINITY;
    int ti = 0x7fffffff;
    const int64_t total = static_cast<int64_t>(n_chunks) * P;
    for (int64_t b = 0; b < total; b += 32) {
        double s = -INFINITY;
        int id = 0x7fffffff;
        if (b + lane < total) {
            const Cand c = in[row * total + b + lane];
            s = c.s;
            id = c.id;
        }
        warp_topP_merge(ts, ti, s, id, P);
    }
    if (lane < P) probed[row * P + lane] = ti;
}

// one warp per (query set, query vector, probe slot): +1 per posting entry.
// counts: uint16 pairs packed in uint32 words, per query set a row of
// ceil(n_docs/2) words.
__global__ void count_kernel(const int32_t *__restrict__ probed, int64_t n_q, int m_q, int P,
                             const int64_t *__restrict__ post_off,
                             const int64_t *__restrict__ post_docs, int64_t row_words,
                             uint32_t *__restrict__ counts) {
    const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t total = n_q * m_q * P;
    if (w >= total) return;
    const int64_t qs = w / (static_cast<int64_t>(m_q) * P);
    const int c = probed[w];
    if (c < 0 || c == 0x7fffffff) return;
    const int64_t lo = post_off[c], hi = post_off[c + 1];
    uint32_t *row = counts + qs * row_words;
    for (int64_t i = lo + lane; i < hi; i += 32) {
        const int64_t doc = post_docs[i];
        atomicAdd(row + (doc >> 1), 1u << (16 * (doc & 1)));
    }
}

__device__ __forceinline__ uint32_t count_of(const uint32_t *row, int64_t doc) {
    return (row[doc >> 1] >> (16 * (doc & 1))) & 0xffffu;
}

// one CTA per query set
__global__ void __launch_bounds__(kSelThreads)
    select_kernel(const uint32_t *__restrict__ counts, int64_t row_words, int64_t n_docs,
                  int max_count, int k_filter, int64_t *__restrict__ cand,
                  int32_t *__restrict__ n_cand) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t *buf = reinterpret_cast<uint64_t *>(smem);                 // kSelMax keys
    uint32_t *hist = reinterpret_cast<uint32_t *>(buf + kSelMax);       // max_count+1
    __shared__ int s_cstar, s_need, s_slot, s_eq_run;
    __shared__ int warp_eq[32];
    const int64_t qs = blockIdx.x;
    const uint32_t *row = counts + qs * row_words;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i <= max_count; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int64_t doc = tid; doc < n_docs; doc += blockDim.x) {
        const uint32_t c = count_of(row, doc);
        if (c) atomicAdd(&hist[tmin<uint32_t>(c, static_cast<uint32_t>(max_count))], 1u);
    }
    __syncthreads();
    if (tid == 0) {
        // docs with count > c are `cum`; c* = largest c with cum(>c) + hist[c] >= k_filter
        int64_t cum = 0;
        bool found = false;
        for (int c = max_count; c >= 1; --c) {
            if (cum + hist[c] >= static_cast<uint32_t>(k_filter)) {
                s_cstar = c;
                s_need = static_cast<int>(k_filter - cum);
                found = true;
                break;
            }
            cum += hist[c];
        }
        if (!found) {  // fewer than k_filter touched docs: take all of them
            s_cstar = 1;
            s_need = static_cast<int>(hist[1]);
        }
        s_slot = 0;
        s_eq_run = 0;
    }
    __syncthreads();
    const uint32_t cstar = s_cstar;
    const int need = s_need;
    // ordered pass over docs in tiles of blockDim: take count > c*, and the
    // first `need` docs (ascending index) with count == c*.
    for (int64_t base = 0; base < n_docs; base += blockDim.x) {
        const int64_t doc = base + tid;
        const uint32_t c = doc < n_docs ? count_of(row, doc) : 0u;
        const bool gt = c > cstar;
        const bool eq = c == cstar && c > 0;
        const unsigned bal = __ballot_sync(0xffffffffu, eq);
        if (lane == 0) warp_eq[warp] = __popc(bal);
        __syncthreads();
        int before = __popc(bal & ((1u << lane) - 1u));
        for (int w = 0; w < warp; ++w) before += warp_eq[w];
        const int run = s_eq_run;
        bool take = gt || (eq && run + before < need);
        if (take) {
            const int slot = atomicAdd(&s_slot, 1);
            if (slot < kSelMax)
                buf[slot] = (static_cast<uint64_t>(c) << 40) | (0xffffffffffull - static_cast<uint64_t>(doc));
        }
        __syncthreads();
        if (tid == 0) {
            int tot = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += warp_eq[w];
            s_eq_run = run + tot;
        }
        __syncthreads();
    }
    const int m = min(s_slot, kSelMax);
    int p2 = 1;
    while (p2 < m) p2 <<= 1;
    for (int i = m + tid; i < p2; i += blockDim.x) buf[i] = 0;  // sentinels sort last
    __syncthreads();
    for (int size = 2; size <= p2; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < p2; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool desc = (i & size) == 0;
                    if ((buf[i] < buf[j]) == desc) {
                        const uint64_t t = buf[i];
                        buf[i] = buf[j];
                        buf[j] = t;
                    }
                }
            }
            __syncthreads();
        }
    const int outn = min(m, k_filter);
    for (int i = tid; i < k_filter; i += blockDim.x)
        cand[qs * k_filter + i] = i < outn ? static_cast<int64_t>(0xffffffffffull - (buf[i] & 0xffffffffffull)) : -1;
    if (tid == 0) n_cand[qs] = outn;
}

static size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

struct PrefilterWs {
    size_t cand_bytes, probed_bytes, counts_bytes, total;
    int64_t n_chunks, row_words;
};

static PrefilterWs ws_layout(int64_t n_q, int m_q, int64_t k_c, int64_t n_docs, int P) {
    PrefilterWs w{};
    const int64_t rows = n_q * m_q;
    w.n_chunks = (k_c + kPTile * kPChunkTiles - 1) / (kPTile * kPChunkTiles);
    w.row_words = (n_docs + 1) / 2;
    w.cand_bytes = align256(static_cast<size_t>(rows) * w.n_chunks * P * sizeof(Cand));
    w.probed_bytes = align256(static_cast<size_t>(rows) * P * sizeof(int32_t));
    w.counts_bytes = align256(static_cast<size_t>(n_q) * w.row_words * sizeof(uint32_t));
    w.total = w.cand_bytes + w.probed_bytes + w.counts_bytes;
    return w;
}

}  // namespace dsrt

using namespace dsrt;

extern "C" size_t dsrt_prefilter_workspace(int64_t n_q, int m_q, int64_t k_c, int64_t n_docs,
                                           int probe) {
    const int P = static_cast<int>(tmin<int64_t>(tmax(probe, 1), k_c));
    return ws_layout(n_q, m_q, k_c, n_docs, P).total;
}

extern "C" int dsrt_prefilter(const double *Q, int64_t n_q, int m_q, int d, const double *cents,
                              int64_t k_c, const int64_t *post_off, const int64_t *post_docs,
                              int64_t n_docs, int probe, int k_filter, int64_t *cand,
                              int32_t *n_cand, void *workspace, size_t ws_bytes, void *stream) {
    DSRT_REQUIRE(probe >= 1, DSRT_EINVAL, "invalid parameter: probe must be >= 1, got %d", probe);
    DSRT_REQUIRE(k_filter >= 1, DSRT_EINVAL, "invalid parameter: k_filter must be >= 1, got %d", k_filter);
    DSRT_REQUIRE(m_q >= 1 && n_q >= 0, DSRT_EINVAL, "Q must be a non-empty (m_q, d) matrix");
    DSRT_REQUIRE(k_c >= 1 && d >= 1, DSRT_EINVAL, "invalid parameter: k=%lld d=%d", (long long)k_c, d);
    const int P = static_cast<int>(tmin<int64_t>(probe, k_c));
    DSRT_REQUIRE(P <= kMaxProbe, DSRT_EUNSUPPORTED, "invalid parameter: probe=%d exceeds %d", P, kMaxProbe);
    DSRT_REQUIRE(k_filter <= kSelMax, DSRT_EUNSUPPORTED, "invalid parameter: k_filter=%d exceeds %d",
                 k_filter, kSelMax);
    const int max_count = m_q * P;
    DSRT_REQUIRE(max_count <= 65535, DSRT_EUNSUPPORTED, "invalid parameter: m_q*probe too large");
    DSRT_REQUIRE(k_c < (1LL << 31), DSRT_EUNSUPPORTED, "invalid parameter: too many centroids");
    if (n_q == 0) return DSRT_OK;
    const PrefilterWs w = ws_layout(n_q, m_q, k_c, n_docs, P);
    DSRT_REQUIRE(workspace != nullptr && ws_bytes >= w.total, DSRT_EINVAL,
                 "invalid parameter: prefilter workspace too small");
    cudaStream_t st = as_stream(stream);
    uint8_t *ws = static_cast<uint8_t *>(workspace);
    Cand *cands = reinterpret_cast<Cand *>(ws);
    int32_t *probed = reinterpret_cast<int32_t *>(ws + w.cand_bytes);
    uint32_t *counts = reinterpret_cast<uint32_t *>(ws + w.cand_bytes + w.probed_bytes);
    const int64_t rows = n_q * m_q;
    dim3 g1(static_cast<unsigned>((rows + kPRows - 1) / kPRows), static_cast<unsigned>(w.n_chunks));
    DSRT_REQUIRE(w.n_chunks < 65536, DSRT_EUNSUPPORTED, "too many centroid chunks");
    const size_t psmem = (kPDim * kPRows + kPRows * (kPTile + 1)) * sizeof(double);
    DSRT_CUDA(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem));
    probe_kernel<<<g1, kPTile, psmem, st>>>(Q, rows, d, cents, k_c, P, cands);
    merge_kernel<<<static_cast<unsigned>((rows * 32 + 255) / 256), 256, 0, st>>>(
        cands, rows, static_cast<int>(w.n_chunks), P, probed);
    DSRT_CUDA(cudaMemsetAsync(counts, 0, w.counts_bytes, st));
    const int64_t warps = rows * P;
    count_kernel<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, st>>>(
        probed, n_q, m_q, P, post_off, post_docs, w.row_words, counts);
    const size_t smem = kSelMax * sizeof(uint64_t) + (max_count + 1) * sizeof(uint32_t);
    DSRT_CUDA(cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    select_kernel<<<static_cast<unsigned>(n_q), kSelThreads, smem, st>>>(
        counts, w.row_words, n_docs, max_count, k_filter, cand, n_cand);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}
