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
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cooperative_groups.h>

#include "tc_common.cuh"

namespace cg = cooperative_groups;
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

// ---- chunked counting: CTA per (query set, doc chunk), counters in shared memory
constexpr int kChunkBytes = 64 * 1024;  // counters per CTA (3 CTAs per SM)
constexpr int kCntThreads = 512;
static int64_t chunk_docs(int cb) { return static_cast<int64_t>(kChunkBytes) * 8 / cb; }

// bnd[c * (nch + 1) + j] = index in post_docs of the first doc >= j * D of posting c
// (postings are doc-ascending); j = nch -> end of the posting
__global__ void chunk_bounds_kernel(const int64_t *__restrict__ post_off, const int64_t *__restrict__ post_docs,
                                    int64_t k_c, int nch, int64_t D, int64_t *__restrict__ bnd) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= k_c * (nch + 1)) return;
    const int64_t c = i / (nch + 1);
    const int j = static_cast<int>(i - c * (nch + 1));
    const int64_t lo = post_off[c], hi = post_off[c + 1];
    bnd[i] = j == nch ? hi : lo + lower_bound_i64(post_docs + lo, hi - lo, j * D);
}

// Counting walk of one (query set, doc chunk): warp w takes the probed rows
// w, w + NWARP, ...; lane j of the warp fetches row j's posting sub-range for
// the chunk (independent loads, not a dependent chain per posting), a warp scan
// turns the sub-range lengths into one flat index space, and the lanes then
// stream the doc ids 4 loads deep, each lane advancing its own segment cursor.
template <int CB, int NWARP>
__device__ __forceinline__ void count_postings(uint32_t *sc, const int32_t *__restrict__ prow, int MP,
                                               const int64_t *__restrict__ bnd, int nch, int ch,
                                               const int64_t *__restrict__ post_docs, int64_t doc0) {
    constexpr int DPW = 32 / CB;
    __shared__ int64_t seg_base[NWARP][32];  // flat index -> post_docs index offset
    __shared__ int32_t seg_end[NWARP][32];   // inclusive prefix of segment lengths
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int r0 = 0; r0 < MP; r0 += NWARP * 32) {
        const int r = r0 + warp + NWARP * lane;
        int64_t a = 0;
        int len = 0;
        if (r < MP) {
            const int c = prow[r];
            if (c >= 0 && c != 0x7fffffff) {
                const int64_t *bc = bnd + static_cast<int64_t>(c) * (nch + 1) + ch;
                a = bc[0];
                len = static_cast<int>(bc[1] - a);
            }
        }
        // pull the row's posting sub-range toward L2 now; the flattened loads below
        // then mostly hit L2 instead of waiting on HBM batch after batch
        for (int64_t ln = (a * 8) & ~int64_t(127); ln < (a + len) * 8; ln += 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char *>(post_docs) + ln));
        int incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        seg_base[warp][lane] = a - (incl - len);
        seg_end[warp][lane] = incl;
        __syncwarp();
        int seg = 0;
        for (int i0 = 0; i0 < total; i0 += 8 * 32) {
            int64_t dd[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * 32 + lane;
                dd[u] = -1;
                if (i < total) {
                    while (i >= seg_end[warp][seg]) ++seg;
                    dd[u] = post_docs[seg_base[warp][seg] + i] - doc0;
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (dd[u] >= 0) atomicAdd(&sc[dd[u] / DPW], 1u << (CB * static_cast<int>(dd[u] % DPW)));
        }
        __syncwarp();
    }
}

// Count histogram of a chunk of u8 counters in shared memory (NT threads).
// Words whose bytes are all <= 3 (nearly all) are tallied without compares:
// byte-lane sums of bit 0, bit 1 and bit0 & bit1 give n1 + n3, n2 + n3 and n3;
// the rare words holding a count >= 4 go byte by byte through shared atomics.
// sum_s (optional, W_CH / 128 words): bit g = 16-byte group g holds a count >= 2.
template <int NT>
__device__ __forceinline__ void chunk_hist8(const uint32_t *sc, uint32_t *hist, int max_count,
                                            uint32_t *sum_s = nullptr) {
    constexpr int W_CH = kChunkBytes / 4;
    constexpr uint32_t M = 0x01010101u;
    static_assert(W_CH / NT <= 64, "byte-lane sums must not overflow");
    uint32_t A = 0, B = 0, Cc = 0;
    const uint4 *s4 = reinterpret_cast<const uint4 *>(sc);
    for (int i = threadIdx.x; i < W_CH / 4; i += NT) {
        const uint4 v = s4[i];
        if (sum_s != nullptr) {
            const unsigned f = __ballot_sync(0xffffffffu, ((v.x | v.y | v.z | v.w) & 0xfefefefeu) != 0u);
            if ((threadIdx.x & 31) == 0) sum_s[i >> 5] = f;
        }
        const uint32_t xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            uint32_t x = xs[k];
            if (x & 0xfcfcfcfcu) {
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const uint32_t c = (x >> (8 * b)) & 0xffu;
                    if (c != 0u) atomicAdd(&hist[tmin<uint32_t>(c, static_cast<uint32_t>(max_count))], 1u);
                }
                x = 0u;
            }
            const uint32_t b0 = x & M, b1 = (x >> 1) & M;
            A += b0;
            B += b1;
            Cc += b0 & b1;
        }
    }
    const uint32_t n3 = (Cc * M) >> 24;
    uint32_t h1 = ((A * M) >> 24) - n3, h2 = ((B * M) >> 24) - n3, h3 = n3;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        h1 += __shfl_xor_sync(0xffffffffu, h1, o);
        h2 += __shfl_xor_sync(0xffffffffu, h2, o);
        h3 += __shfl_xor_sync(0xffffffffu, h3, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (max_count >= 1) atomicAdd(&hist[1], h1);
        if (max_count >= 2) atomicAdd(&hist[2], h2);
        if (max_count >= 3) atomicAdd(&hist[3], h3);
    }
}

// counts of one doc chunk for one query set in shared memory, then its count
// histogram (hist_bins = max_count + 1) and the counter words of the row
template <int CB>
__global__ void __launch_bounds__(kCntThreads)
    count_chunk_kernel(const int32_t *__restrict__ probed, int MP, const int64_t *__restrict__ bnd,
                       int nch, const int64_t *__restrict__ post_docs, int64_t row_words,
                       int max_count, uint32_t *__restrict__ counts, uint32_t *__restrict__ chist,
                       uint32_t *__restrict__ gsum) {
    constexpr int DPW = 32 / CB;
    constexpr uint32_t MASK = (1u << CB) - 1u;
    constexpr int W_CH = kChunkBytes / 4;          // counter words per chunk
    constexpr int64_t D = static_cast<int64_t>(W_CH) * DPW;  // docs per chunk
    extern __shared__ __align__(16) uint32_t sc[];  // W_CH counter words, then max_count+1 bins
    uint32_t *hist = sc + W_CH;
    const int ch = blockIdx.x;
    const int64_t qs = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31;
    for (int i = tid; i < W_CH / 4; i += kCntThreads) reinterpret_cast<uint4 *>(sc)[i] = make_uint4(0, 0, 0, 0);
    for (int i = tid; i <= max_count; i += kCntThreads) hist[i] = 0;
    __syncthreads();
    count_postings<CB, kCntThreads / 32>(sc, probed + qs * MP, MP, bnd, nch, ch, post_docs, ch * D);
    __syncthreads();
    // histogram of this chunk's counts: 1..3 by SIMD compares, >= 4 by shared atomics
    constexpr uint32_t ONE = CB == 8 ? 0x01010101u : 0x00010001u;
    uint32_t h1 = 0, h2 = 0, h3 = 0;
    if constexpr (CB == 8) {
        __shared__ uint32_t sum_s[kChunkBytes / 4 / 128];
        chunk_hist8<kCntThreads>(sc, hist, max_count, sum_s);
        __syncthreads();
        for (int i = tid; i < kChunkBytes / 4 / 128; i += kCntThreads)
            gsum[(qs * nch + ch) * (kChunkBytes / 4 / 128) + i] = sum_s[i];
    } else {
    for (int i = tid; i < W_CH; i += kCntThreads) {
        const uint32_t x = sc[i];
        if (x == 0u) continue;
        if (CB == 8) {
            h1 += __popc(__vcmpeq4(x, ONE) & ONE);
            h2 += __popc(__vcmpeq4(x, 2 * ONE) & ONE);
            h3 += __popc(__vcmpeq4(x, 3 * ONE) & ONE);
            if (__vcmpgeu4(x, 4 * ONE) == 0u) continue;
        } else {
            h1 += __popc(__vcmpeq2(x, ONE) & ONE);
            h2 += __popc(__vcmpeq2(x, 2 * ONE) & ONE);
            h3 += __popc(__vcmpeq2(x, 3 * ONE) & ONE);
            if (__vcmpgeu2(x, 4 * ONE) == 0u) continue;
        }
#pragma unroll
        for (int k = 0; k < DPW; ++k) {
            const uint32_t v = (x >> (CB * k)) & MASK;
            if (v >= 4) atomicAdd(&hist[tmin<uint32_t>(v, static_cast<uint32_t>(max_count))], 1u);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        h1 += __shfl_xor_sync(0xffffffffu, h1, o);
        h2 += __shfl_xor_sync(0xffffffffu, h2, o);
        h3 += __shfl_xor_sync(0xffffffffu, h3, o);
    }
    if (lane == 0) {
        if (max_count >= 1) atomicAdd(&hist[1], h1);
        if (max_count >= 2) atomicAdd(&hist[2], h2);
        if (max_count >= 3) atomicAdd(&hist[3], h3);
    }
    }
    __syncthreads();
    // chist[(qs * nb + bin) * nch + chunk]: one bin's chunk counts are contiguous
    for (int i = tid; i <= max_count; i += kCntThreads)
        chist[(qs * (max_count + 1) + i) * static_cast<int64_t>(nch) + ch] = hist[i];
    // counter words of the row (chunks tile the whole padded row)
    const int64_t w0 = static_cast<int64_t>(ch) * W_CH;
    const int64_t nw = tmin<int64_t>(W_CH, row_words - w0);
    uint32_t *row = counts + qs * row_words + w0;
    for (int64_t i = tid; i < nw / 4; i += kCntThreads)
        reinterpret_cast<uint4 *>(row)[i] = reinterpret_cast<const uint4 *>(sc)[i];
}

__device__ __forceinline__ uint32_t count_of(const uint32_t *row, int64_t doc) {
    return (row[doc >> 1] >> (16 * (doc & 1))) & 0xffffu;
}

// u16 counters (m_q * probe > 255), large batches: one CTA per query set.  Counters are u8 (u16) lanes of uint32
// words.  The count histogram is the sum of the counting pass's chunk
// histograms; c* = largest c with #(count > c) + hist[c] >= k_filter.  One
// ordered pass (ascending doc order, 4 x uint4 per thread per step) takes every
// doc with count > c* and the first `need` docs with count == c* (block-wide
// exclusive scan of the per-thread tie counts); then a bitonic sort by (count
// desc, index asc) in shared memory.

template <int CB>  // counter bits: 8 or 16
__global__ void __launch_bounds__(kSelThreads)
    select_kernel(const uint32_t *__restrict__ counts, int64_t row_words, int64_t n_docs,
                  int max_count, int k_filter, int64_t *__restrict__ cand,
                  int32_t *__restrict__ n_cand, const uint32_t *__restrict__ chist, int nch) {
    constexpr int DPG = 128 / CB;            // docs per uint4 group
    constexpr int DPW = 32 / CB;             // docs per word
    constexpr uint32_t MASK = (1u << CB) - 1u;
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t *buf = reinterpret_cast<uint64_t *>(smem);                    // kSelMax keys
    uint32_t *hist = reinterpret_cast<uint32_t *>(buf + kSelMax);          // max_count+1
    __shared__ int s_cstar, s_need, s_slot, s_eq_run, s_eq_step;
    __shared__ int warp_tot[32];
    const int64_t qs = blockIdx.x;
    const uint32_t *row = counts + qs * row_words;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // each thread owns 4 consecutive uint4 groups per step (4*DPG docs, 64 B):
    // four independent loads in flight, ascending doc order across threads
    constexpr int G = 4;
    const int64_t n_groups = (n_docs + DPG - 1) / DPG;
    const uint4 *row4 = reinterpret_cast<const uint4 *>(row);
    const int64_t row_words4 = row_words / 4;
    auto load_groups = [&](int64_t g0, uint32_t (&w)[4 * G]) {
#pragma unroll
        for (int u = 0; u < G; ++u) {
            const int64_t g = g0 + u;
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (g < row_words4) v = __ldg(row4 + g);
            w[4 * u] = v.x; w[4 * u + 1] = v.y; w[4 * u + 2] = v.z; w[4 * u + 3] = v.w;
        }
    };
    const int64_t per_step = static_cast<int64_t>(blockDim.x) * G;
    {  // global histogram = sum of the chunk histograms of the counting pass
        const uint32_t *gh = chist + qs * nch * static_cast<int64_t>(max_count + 1);
        for (int b = tid; b <= max_count; b += blockDim.x) {
            uint32_t t = 0;
            for (int c = 0; c < nch; ++c) t += gh[b * static_cast<int64_t>(nch) + c];
            hist[b] = t;
        }
        __syncthreads();
    }
    if (tid == 0) {
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
        if (!found) {
            s_cstar = 1;
            s_need = static_cast<int>(hist[1]);
        }
        s_slot = 0;
        s_eq_run = 0;
    }
    __syncthreads();
    const uint32_t cstar = s_cstar;
    const int need = s_need;
    for (int64_t base = 0; base < n_groups; base += per_step) {
        const int64_t g0 = base + static_cast<int64_t>(tid) * G;
        uint32_t w[4 * G];
        load_groups(g0, w);
        // SIMD per word: lanes equal to c* (ties) and >= c* (hits); c* >= 1
        const uint32_t cs = CB == 8 ? cstar * 0x01010101u : cstar * 0x00010001u;
        int eqn = 0;
        uint32_t hitmask = 0;  // bit q: word q has a doc with count >= c*
#pragma unroll
        for (int q = 0; q < 4 * G; ++q) {
            if (w[q] == 0u) continue;
            if (CB == 8) {
                eqn += __popc(__vcmpeq4(w[q], cs) & 0x01010101u);
                hitmask |= (__vcmpgeu4(w[q], cs) != 0u ? 1u : 0u) << q;
            } else {
                eqn += __popc(__vcmpeq2(w[q], cs) & 0x00010001u);
                hitmask |= (__vcmpgeu2(w[q], cs) != 0u ? 1u : 0u) << q;
            }
        }
        const int nhit = hitmask != 0u;
        // block exclusive scan of eqn (ascending doc order = ascending tid)
        int x = eqn;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_tot[warp] = x;
        __syncthreads();
        if (warp == 0) {  // scan of the 32 warp totals
            int t = warp_tot[lane];
            int sx = t;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, sx, o);
                if (lane >= o) sx += y;
            }
            warp_tot[lane] = sx - t;  // exclusive
            if (lane == 31) s_eq_step = sx;
        }
        __syncthreads();
        int run = s_eq_run + warp_tot[warp] + (x - eqn);
        if (nhit > 0) {
#pragma unroll
            for (int q = 0; q < 4 * G; ++q) {
                if (!((hitmask >> q) & 1u)) continue;
#pragma unroll
                for (int k = 0; k < DPW; ++k) {
                    const uint32_t c = (w[q] >> (CB * k)) & MASK;
                    if (c < cstar) continue;  // c* >= 1, so c == 0 is skipped
                    bool take = c > cstar;
                    if (c == cstar) {
                        take = run < need;
                        ++run;
                    }
                    if (take) {
                        const int64_t doc = g0 * DPG + q * DPW + k;
                        const int slot = atomicAdd(&s_slot, 1);
                        if (slot < kSelMax)
                            buf[slot] = (static_cast<uint64_t>(c) << 40) | (0xffffffffffull - static_cast<uint64_t>(doc));
                    }
                }
            }
        }
        __syncthreads();
        if (tid == 0) s_eq_run += s_eq_step;
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

// ---- small batches: chunk-parallel selection (the single-CTA ordered scan of
// select_kernel would scan a whole counter row alone):
//  plan:  per query set, c*/need from the summed chunk histograms and the
//         number of ties (count == c*) in earlier chunks;
//  scan:  CTA per (query set, chunk), 32-word strips per thread in doc order;
//         ties ranked by a block scan go straight to their final slot (they
//         follow all hits, ascending doc), hits (count > c*) are appended;
//  final: per query set, bitonic sort of the hits by (count desc, index asc).
struct SelPlan {
    int32_t cstar, need, pad0, pad1;
};

__global__ void sel_plan_kernel(const uint32_t *__restrict__ chist, int nch, int max_count, int k_filter,
                                SelPlan *__restrict__ plan, int32_t *__restrict__ tie_base,
                                int32_t *__restrict__ hits_n) {
    extern __shared__ uint32_t ph[];  // max_count + 1
    const int64_t qs = blockIdx.x;
    const uint32_t *gh = chist + qs * nch * static_cast<int64_t>(max_count + 1);
    for (int b = threadIdx.x; b <= max_count; b += blockDim.x) {
        uint32_t t = 0;
        for (int c = 0; c < nch; ++c) t += gh[b * static_cast<int64_t>(nch) + c];
        ph[b] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t cum = 0;
        int cstar = 1, need = static_cast<int>(ph[1]);
        for (int c = max_count; c >= 1; --c) {
            if (cum + ph[c] >= static_cast<uint32_t>(k_filter)) {
                cstar = c;
                need = static_cast<int>(k_filter - cum);
                break;
            }
            cum += ph[c];
        }
        plan[qs] = SelPlan{cstar, need, 0, 0};
        hits_n[qs] = 0;
        int32_t run = 0;
        for (int c = 0; c < nch; ++c) {
            tie_base[qs * nch + c] = run;
            run += static_cast<int32_t>(gh[cstar * static_cast<int64_t>(nch) + c]);
        }
    }
}

constexpr int kScanThreads = 512;

template <int CB>
__global__ void __launch_bounds__(kScanThreads)
    sel_scan_kernel(const uint32_t *__restrict__ counts, int64_t row_words, int nch, int k_filter,
                    const SelPlan *__restrict__ plan, const int32_t *__restrict__ tie_base,
                    int32_t *__restrict__ hits_n, uint64_t *__restrict__ hits,
                    int64_t *__restrict__ ties) {
    constexpr int DPW = 32 / CB;
    constexpr uint32_t MASK = (1u << CB) - 1u;
    constexpr uint32_t ONE = CB == 8 ? 0x01010101u : 0x00010001u;
    constexpr int W_CH = kChunkBytes / 4;
    constexpr int SW = W_CH / kScanThreads;  // words per thread strip
    __shared__ int warp_tot[kScanThreads / 32];
    const int ch = blockIdx.x;
    const int64_t qs = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const SelPlan pl = plan[qs];
    const uint32_t cstar = static_cast<uint32_t>(pl.cstar);
    const int64_t w0 = static_cast<int64_t>(ch) * W_CH + static_cast<int64_t>(tid) * SW;
    const uint32_t *row = counts + qs * row_words;
    const uint32_t ceq = cstar * ONE, cgt = (cstar + 1) * ONE;
    uint32_t w[SW];
#pragma unroll
    for (int q = 0; q < SW; q += 4) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (w0 + q + 4 <= row_words) v = *reinterpret_cast<const uint4 *>(row + w0 + q);
        w[q] = v.x; w[q + 1] = v.y; w[q + 2] = v.z; w[q + 3] = v.w;
    }
    int eqn = 0;
    uint32_t hitmask = 0;
#pragma unroll
    for (int q = 0; q < SW; ++q) {
        const uint32_t x = w[q];
        if (x == 0u) continue;
        if (CB == 8) {
            eqn += __popc(__vcmpeq4(x, ceq) & ONE);
            if (cstar < MASK && __vcmpgeu4(x, cgt) != 0u) hitmask |= 1u << q;
        } else {
            eqn += __popc(__vcmpeq2(x, ceq) & ONE);
            if (cstar < MASK && __vcmpgeu2(x, cgt) != 0u) hitmask |= 1u << q;
        }
    }
    int x = eqn;  // block exclusive scan of the tie counts (doc order = thread order)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const int t = lane < kScanThreads / 32 ? warp_tot[lane] : 0;
        int sx = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, sx, o);
            if (lane >= o) sx += y;
        }
        if (lane < kScanThreads / 32) warp_tot[lane] = sx - t;
    }
    __syncthreads();
    int rank = tie_base[qs * nch + ch] + warp_tot[warp] + (x - eqn);
    const int need = pl.need;
    int64_t *tout = ties + qs * k_filter;
    const int64_t doc_w0 = w0 * DPW;
    if (eqn > 0 && rank < need) {  // rare: rolled loops over the words (re-read via L1)
#pragma unroll 1
        for (int q = 0; q < SW && rank < need; ++q) {
            const uint32_t xw = row[w0 + q];
            if (xw == 0u) continue;
#pragma unroll 1
            for (int k = 0; k < DPW; ++k)
                if (((xw >> (CB * k)) & MASK) == cstar) {
                    if (rank < need) tout[rank] = doc_w0 + q * DPW + k;
                    ++rank;
                }
        }
    }
    if (hitmask != 0u) {
#pragma unroll 1
        for (int q = 0; q < SW; ++q) {
            if (!((hitmask >> q) & 1u)) continue;
            const uint32_t xw = row[w0 + q];
#pragma unroll 1
            for (int k = 0; k < DPW; ++k) {
                const uint32_t c = (xw >> (CB * k)) & MASK;
                if (c > cstar) {
                    const int slot = atomicAdd(hits_n + qs, 1);
                    if (slot < k_filter)
                        hits[qs * k_filter + slot] = (static_cast<uint64_t>(c) << 40) |
                                                     (0xffffffffffull - static_cast<uint64_t>(doc_w0 + q * DPW + k));
                }
            }
        }
    }
}

constexpr int kFinThreads = 1024;

// hits sorted by (count desc, index asc), then the ties (ascending doc)
__global__ void __launch_bounds__(kFinThreads)
    sel_final_kernel(const SelPlan *__restrict__ plan, const int32_t *__restrict__ hits_n,
                     const uint64_t *__restrict__ hits, const int64_t *__restrict__ ties, int k_filter,
                     int64_t *__restrict__ cand, int32_t *__restrict__ n_cand) {
    extern __shared__ uint64_t hb[];  // pow2 >= k_filter keys
    const int64_t qs = blockIdx.x;
    const int tid = threadIdx.x;
    const SelPlan pl = plan[qs];
    const int nh = tmin(hits_n[qs], k_filter);
    int p2 = 1;
    while (p2 < nh) p2 <<= 1;
    for (int i = tid; i < p2; i += blockDim.x) hb[i] = i < nh ? hits[qs * k_filter + i] : 0ull;
    __syncthreads();
    for (int size = 2; size <= p2; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < p2; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool desc = (i & size) == 0;
                    if ((hb[i] < hb[j]) == desc) {
                        const uint64_t t = hb[i];
                        hb[i] = hb[j];
                        hb[j] = t;
                    }
                }
            }
            __syncthreads();
        }
    const int nt = tmin(pl.need, k_filter - nh);
    const int outn = nh + nt;
    for (int i = tid; i < k_filter; i += blockDim.x) {
        int64_t v = -1;
        if (i < nh) v = static_cast<int64_t>(0xffffffffffull - (hb[i] & 0xffffffffffull));
        else if (i < outn) v = ties[qs * k_filter + (i - nh)];
        cand[qs * k_filter + i] = v;
    }
    if (tid == 0) n_cand[qs] = outn;
}

// ---- u8 counters (m_q * probe <= 255), any batch: sort-free placement.
// The output order (count desc, index asc) is a counting sort keyed by count,
// so every selected doc's final slot follows from histograms alone:
//   hit (count c > c*):  #(count > c, all chunks) + #(count == c, earlier
//                        chunks) + rank among count == c in this chunk;
//   tie (count == c*):   H + #(count == c*, earlier chunks) + rank in chunk,
//                        kept while < need  (H = #(count > c*) = k_filter - need).
// CTA per (query set, chunk): the plan (c*, H, need) and the bases come from
// the counting pass's chunk histograms; ties are ranked by a block scan in doc
// order; the chunk's hits (< k_filter of them) are compacted in doc order and
// ranked per count by one warp with __match_any_sync.  No atomics, no sort.
constexpr int kPlaceThreads = 512;
constexpr int kPlaceWarps = kPlaceThreads / 32;
static size_t place_smem(int max_count, int k_filter) {
    return kChunkBytes + 16 + static_cast<size_t>(2 * (max_count + 1)) * sizeof(uint32_t) +
           static_cast<size_t>(k_filter) * sizeof(uint32_t);
}

// Shared tail of the placement kernels: above[] holds the global count
// histogram and pre[] the counts of earlier chunks (both [max_count + 1], in
// shared memory, synced); cw the chunk's nw counter words (after `bar`, if any).
// plan (optional): (c*, H, need) precomputed by sel_plan8_kernel, in which case
// pre[] already holds this chunk's slot bases (pre[c*] = its first tie rank,
// pre[c] = #(count > c) + earlier chunks' count-c docs for c > c*) and above[]
// is unused.
__device__ __forceinline__ void place_chunk(const uint32_t *cw, int nw, uint64_t *bar, int ch, int64_t qs,
                                            int max_count, int k_filter, uint32_t *above, uint32_t *pre,
                                            uint32_t *hl, int64_t *__restrict__ cand,
                                            int32_t *__restrict__ n_cand, const int4 *plan = nullptr,
                                            uint32_t gmask2 = 0xffu) {
    constexpr int W_CH = kChunkBytes / 4;      // counter words per chunk
    constexpr int SW = W_CH / kPlaceThreads;   // words per thread strip (128 docs)
    constexpr uint32_t ONE = 0x01010101u;
    __shared__ uint32_t s_tot[2][kPlaceWarps];
    __shared__ int s_cstar, s_need, s_H;
    const int nb = max_count + 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (plan != nullptr) {
        if (tid == 0) {
            const int4 pl = *plan;
            s_cstar = pl.x;
            s_H = pl.y;
            s_need = pl.z;
        }
    } else if (warp == 0) {  // descending suffix scan of the histogram: c*, H, need; above[c] for c >= c*
        const uint32_t g1 = nb > 1 ? above[1] : 0u;
        uint32_t carry = 0;
        int cstar = -1;
        for (int top = max_count; top >= 1 && cstar < 0; top -= 32) {
            const int b = top - lane;
            const uint32_t g = b >= 1 ? above[b] : 0u;
            uint32_t incl = g;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const unsigned hit = __ballot_sync(0xffffffffu, b >= 1 && carry + incl >= static_cast<uint32_t>(k_filter));
            if (b >= 1) above[b] = carry + incl - g;
            if (hit != 0u) cstar = top - (__ffs(hit) - 1);
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        __syncwarp();
        if (lane == 0) {
            if (cstar >= 1) {
                s_cstar = cstar;
                s_H = static_cast<int>(above[cstar]);
                s_need = k_filter - s_H;
            } else {  // fewer than k_filter touched docs: take all of them
                s_cstar = 1;
                s_H = static_cast<int>(above[1]);
                s_need = static_cast<int>(g1);
            }
        }
    }
    __syncthreads();
    const uint32_t cstar = static_cast<uint32_t>(s_cstar);
    const int need = s_need, H = s_H;
    const uint32_t ceq = cstar * ONE;
    if (bar != nullptr) mbar_wait(bar, 0);
    // tie / hit counts of this thread's strip; 16-byte groups visited in a rotated
    // order so a warp's LDS.128 spread over all banks (counting is order-free)
    const uint4 *s4 = reinterpret_cast<const uint4 *>(cw) + tid * (SW / 4);
    const int ng = tmax(0, tmin(SW / 4, nw / 4 - tid * (SW / 4)));
    uint32_t le = 0, lg = 0;        // byte-lane sums (<= 32 per lane)
    uint32_t emask = 0, gmask = 0;  // bit q: word q of the strip holds a tie / a hit
    // with c* >= 2 only groups holding a count >= 2 can hold ties or hits
    const uint32_t gsel = cstar >= 2u ? gmask2 : 0xffu;
    if (gsel != 0xffu) {
        for (uint32_t gm = gsel; gm != 0u; gm &= gm - 1u) {
            const int g = __ffs(gm) - 1;
            if (g >= ng) break;
            const uint4 v = s4[g];
            const uint32_t xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t e = __vcmpeq4(xs[k], ceq) & ONE, t = __vcmpgtu4(xs[k], ceq) & ONE;
                le += e;
                lg += t;
                emask |= (e != 0u ? 1u : 0u) << (4 * g + k);
                gmask |= (t != 0u ? 1u : 0u) << (4 * g + k);
            }
        }
    } else
#pragma unroll
    for (int u = 0; u < SW / 4; ++u) {
        const int g = (u + tid) & (SW / 4 - 1);
        if (g < ng) {
            const uint4 v = s4[g];
            const uint32_t xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t e = __vcmpeq4(xs[k], ceq) & ONE, t = __vcmpgtu4(xs[k], ceq) & ONE;
                le += e;
                lg += t;
                emask |= (e != 0u ? 1u : 0u) << (4 * g + k);
                gmask |= (t != 0u ? 1u : 0u) << (4 * g + k);
            }
        }
    }
    const uint32_t eqn = (le * ONE) >> 24, gtn = (lg * ONE) >> 24;
    // block exclusive scans of (ties, hits) in thread = doc order
    uint32_t xe = eqn, xg = gtn;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t ye = __shfl_up_sync(0xffffffffu, xe, o);
        const uint32_t yg = __shfl_up_sync(0xffffffffu, xg, o);
        if (lane >= o) { xe += ye; xg += yg; }
    }
    if (lane == 31) { s_tot[0][warp] = xe; s_tot[1][warp] = xg; }
    __syncthreads();
    uint32_t be = 0, bg = 0, nh = 0;
#pragma unroll
    for (int i = 0; i < kPlaceWarps; ++i) {
        const uint32_t te = s_tot[0][i], tg = s_tot[1][i];
        be += i < warp ? te : 0u;
        bg += i < warp ? tg : 0u;
        nh += tg;
    }
    int64_t *out = cand + qs * k_filter;
    const uint32_t *sw = cw + tid * SW;
    const int64_t doc0 = static_cast<int64_t>(ch) * W_CH * 4;  // first doc of the chunk
    const int sdoc0 = tid * SW * 4;                               // first doc of the strip, in the chunk
    // ties: global tie rank = pre[c*] + rank in chunk; slot H + rank while rank < need
    int64_t trank = static_cast<int64_t>(pre[cstar]) + be + (xe - eqn);
    if (eqn > 0 && trank < need) {
        for (uint32_t wm = emask; wm != 0u && trank < need; wm &= wm - 1u) {
            const int q = __ffs(wm) - 1;
            uint32_t m = __vcmpeq4(sw[q], ceq) & 0x80808080u;
            while (m != 0u) {
                const int byte = (__ffs(m) - 1) >> 3;
                m &= m - 1u;
                if (trank < need) out[H + trank] = doc0 + sdoc0 + q * 4 + byte;
                ++trank;
            }
        }
    }
    // hits: compact (doc in chunk, count) in doc order
    if (gtn > 0) {
        uint32_t pos = bg + (xg - gtn);
        for (uint32_t wm = gmask; wm != 0u; wm &= wm - 1u) {
            const int q = __ffs(wm) - 1;
            const uint32_t x = sw[q];
            uint32_t m = __vcmpgtu4(x, ceq) & 0x80808080u;
            while (m != 0u) {
                const int byte = (__ffs(m) - 1) >> 3;
                m &= m - 1u;
                hl[pos++] = (static_cast<uint32_t>(sdoc0 + q * 4 + byte) << 8) | ((x >> (8 * byte)) & 0xffu);
            }
        }
    }
    __syncthreads();
    if (warp == 0 && nh > 0) {  // rank hits per count in doc order, 32 at a time
        // pre[c] becomes this chunk's running slot base for count c
        if (plan == nullptr)
            for (int b = lane + static_cast<int>(cstar) + 1; b < nb; b += 32) pre[b] += above[b];
        __syncwarp();
        for (uint32_t i0 = 0; i0 < nh; i0 += 32) {
            const uint32_t i = i0 + lane;
            const bool act = i < nh;
            const uint32_t e = act ? hl[i] : 0u;
            const uint32_t c = act ? (e & 0xffu) : 0x100u + lane;  // inactive lanes: unique keys
            const unsigned peers = __match_any_sync(0xffffffffu, c);
            const int rank = __popc(peers & ((1u << lane) - 1u));
            uint32_t base = 0;
            if (act) base = pre[c];
            __syncwarp();
            if (act) {
                out[base + rank] = doc0 + static_cast<int64_t>(e >> 8);
                if (rank == 0) pre[c] = base + __popc(peers);
            }
            __syncwarp();
        }
    }
    if (ch == 0) {
        const int total = H + need;  // == k_filter unless fewer docs were touched
        for (int i = total + tid; i < k_filter; i += kPlaceThreads) out[i] = -1;
        if (tid == 0) n_cand[qs] = total;
    }
}

// Placement plan per query set (u8 counters), computed once instead of by each
// of its chunk CTAs: c*, H, need from the summed chunk histograms, and per chunk
// the slot bases (tie base at c*, hit bases above it) -> plan[qs], bases[qs][ch][c].
__global__ void __launch_bounds__(256)
    sel_plan8_kernel(const uint32_t *__restrict__ chist, int nch, int max_count, int k_filter,
                     int4 *__restrict__ plan, uint32_t *__restrict__ bases) {
    extern __shared__ uint32_t pl_s[];  // [nb] histogram -> suffix counts
    __shared__ int s_cstar, s_H, s_need;
    const int nb = max_count + 1;
    const int64_t qs = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31;
    const uint32_t *gh = chist + qs * nch * static_cast<int64_t>(nb);
    for (int b = tid; b < nb; b += blockDim.x) {
        const uint32_t *gb = gh + b * static_cast<int64_t>(nch);
        uint32_t g = 0;
        for (int c = 0; c < nch; ++c) g += __ldg(gb + c);
        pl_s[b] = g;
    }
    __syncthreads();
    if (tid < 32) {
        const uint32_t g1 = nb > 1 ? pl_s[1] : 0u;
        uint32_t carry = 0;
        int cstar = -1;
        for (int top = max_count; top >= 1 && cstar < 0; top -= 32) {
            const int b = top - lane;
            const uint32_t g = b >= 1 ? pl_s[b] : 0u;
            uint32_t incl = g;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const unsigned hit = __ballot_sync(0xffffffffu, b >= 1 && carry + incl >= static_cast<uint32_t>(k_filter));
            if (b >= 1) pl_s[b] = carry + incl - g;
            if (hit != 0u) cstar = top - (__ffs(hit) - 1);
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        __syncwarp();
        if (lane == 0) {
            if (cstar >= 1) {
                s_cstar = cstar;
                s_H = static_cast<int>(pl_s[cstar]);
                s_need = k_filter - s_H;
            } else {
                s_cstar = 1;
                s_H = static_cast<int>(pl_s[1]);
                s_need = static_cast<int>(g1);
            }
            plan[qs] = make_int4(s_cstar, s_H, s_need, 0);
        }
    }
    __syncthreads();
    const int cstar = s_cstar;
    for (int b = tid; b < nb; b += blockDim.x) {
        if (b < cstar) continue;
        const uint32_t *gb = gh + b * static_cast<int64_t>(nch);
        uint32_t run = b == cstar ? 0u : pl_s[b];  // ties rank from 0; hits after #(count > b)
        for (int c = 0; c < nch; ++c) {
            bases[(qs * nch + c) * static_cast<int64_t>(nb) + b] = run;
            run += __ldg(gb + c);
        }
    }
}

// Separate counting pass (written counter rows + chunk histograms): the chunk's
// words stream into shared memory (bulk copy) while its slot bases are loaded.
__global__ void __launch_bounds__(kPlaceThreads, 2)
    sel_place_kernel(const uint32_t *__restrict__ counts, int64_t row_words, int nch, int max_count,
                     int k_filter, const int4 *__restrict__ plan, const uint32_t *__restrict__ bases,
                     const uint32_t *__restrict__ gsum, int64_t *__restrict__ cand,
                     int32_t *__restrict__ n_cand) {
    constexpr int W_CH = kChunkBytes / 4;
    extern __shared__ __align__(128) uint8_t psm_b[];
    uint32_t *cw = reinterpret_cast<uint32_t *>(psm_b);
    uint64_t *bar = reinterpret_cast<uint64_t *>(psm_b + kChunkBytes);
    const int nb = max_count + 1;
    uint32_t *above = reinterpret_cast<uint32_t *>(psm_b + kChunkBytes + 16);
    uint32_t *pre = above + nb;
    uint32_t *hl = pre + nb;
    const int ch = blockIdx.x;
    const int64_t qs = blockIdx.y;
    const int tid = threadIdx.x;
    const int64_t cw0 = static_cast<int64_t>(ch) * W_CH;
    const int nw = static_cast<int>(tmin<int64_t>(W_CH, row_words - cw0));  // multiple of 4
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(bar, static_cast<uint32_t>(nw) * 4u);
        bulk_g2s(cw, counts + qs * row_words + cw0, static_cast<uint32_t>(nw) * 4u, bar);
    }
    const uint32_t *bs = bases + (qs * nch + ch) * static_cast<int64_t>(nb);
    for (int b = tid; b < nb; b += kPlaceThreads) pre[b] = __ldg(bs + b);
    // this strip's 8 group flags (count >= 2) from the counting pass's summary
    static_assert(W_CH / 4 / kPlaceThreads == 8, "one summary byte per thread strip");
    const uint32_t sbits = (__ldg(gsum + (qs * nch + ch) * (W_CH / 128) + tid / 4) >> (8 * (tid & 3))) & 0xffu;
    __syncthreads();
    place_chunk(cw, nw, bar, ch, qs, max_count, k_filter, above, pre, hl, cand, n_cand, plan + qs, sbits);
}

// Fused counting + placement for n_docs <= kMaxFusedChunks * 64K (u8 counters):
// a thread-block cluster of the nch chunk CTAs of one query set counts in
// shared memory, exchanges the chunk histograms over distributed shared
// memory, and places straight from the shared counters -- no counter rows in
// HBM, one launch.
constexpr int kMaxFusedChunks = 16;
static size_t fused_smem(int max_count, int k_filter) {
    return place_smem(max_count, k_filter) + static_cast<size_t>(max_count + 1) * sizeof(uint32_t);
}

__global__ void __launch_bounds__(kPlaceThreads, 2)
    count_place_kernel(const int32_t *__restrict__ probed, int MP, const int64_t *__restrict__ bnd, int nch,
                       const int64_t *__restrict__ post_docs, int64_t row_words, int max_count, int k_filter,
                       int64_t *__restrict__ cand, int32_t *__restrict__ n_cand) {
    constexpr int W_CH = kChunkBytes / 4;
    extern __shared__ __align__(128) uint8_t psm_b[];
    uint32_t *cw = reinterpret_cast<uint32_t *>(psm_b);
    const int nb = max_count + 1;
    uint32_t *above = reinterpret_cast<uint32_t *>(psm_b + kChunkBytes + 16);
    uint32_t *pre = above + nb;
    uint32_t *hl = pre + nb;
    uint32_t *hist = hl + k_filter;  // this chunk's histogram (read by the cluster)
    cg::cluster_group cluster = cg::this_cluster();
    const int ch = static_cast<int>(cluster.block_rank());
    const int64_t qs = blockIdx.y;
    const int tid = threadIdx.x;
    for (int i = tid; i < W_CH / 4; i += kPlaceThreads) reinterpret_cast<uint4 *>(cw)[i] = make_uint4(0, 0, 0, 0);
    for (int i = tid; i < nb; i += kPlaceThreads) hist[i] = 0;
    __syncthreads();
    count_postings<8, kPlaceWarps>(cw, probed + qs * MP, MP, bnd, nch, ch, post_docs,
                                   static_cast<int64_t>(ch) * W_CH * 4);
    __syncthreads();
    chunk_hist8<kPlaceThreads>(cw, hist, max_count);
    cluster.sync();  // every chunk histogram complete
    for (int b = tid; b < nb; b += kPlaceThreads) {
        uint32_t g = 0, p = 0;
        for (int c = 0; c < nch; ++c) {
            const uint32_t v = cluster.map_shared_rank(hist, c)[b];
            g += v;
            p += c < ch ? v : 0u;
        }
        above[b] = g;
        pre[b] = p;
    }
    // the remote reads must finish before any CTA of the cluster exits
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    __syncthreads();
    const int nw = static_cast<int>(tmin<int64_t>(W_CH, row_words - static_cast<int64_t>(ch) * W_CH));
    place_chunk(cw, nw, nullptr, ch, qs, max_count, k_filter, above, pre, hl, cand, n_cand);
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

static size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }
// counters: uint8 when m_q*probe <= 255, else uint16; rows padded to 16 bytes
static int counter_bits(int max_count) { return max_count <= 255 ? 8 : 16; }
static int64_t row_words_for(int64_t n_docs, int max_count) {
    const int64_t dpg = 128 / counter_bits(max_count);
    return ((n_docs + dpg - 1) / dpg) * 4;  // 16-byte groups; the last chunk may be partial
}

// chunked counting workspace: posting chunk boundaries + per-chunk histograms
static int n_chunks_for(int64_t n_docs, int max_count) {
    return static_cast<int>((n_docs + chunk_docs(counter_bits(max_count)) - 1) / chunk_docs(counter_bits(max_count)));
}
// bounds (unless cached) | chunk histograms | placement plans | per-chunk slot bases
static size_t count_ws_chunks(int64_t n_q, int m_q, int P, int64_t k_c, int64_t n_docs) {
    const int mc = m_q * P, nch = n_chunks_for(n_docs, mc);
    return align256(static_cast<size_t>(k_c) * (nch + 1) * sizeof(int64_t)) +
           2 * align256(static_cast<size_t>(n_q) * nch * (mc + 1) * sizeof(uint32_t)) +
           align256(static_cast<size_t>(n_q) * sizeof(int4)) +
           align256(static_cast<size_t>(n_q) * nch * (kChunkBytes / 4 / 128) * sizeof(uint32_t));
}
static bool small_batch(int64_t n_q) { return n_q * 8 <= sm_count(); }
// + the small-batch selection buffers (plans, tie bases, hit counts, hits, ties)
static size_t count_ws_bytes(int64_t n_q, int m_q, int P, int64_t k_c, int64_t n_docs) {
    size_t b = count_ws_chunks(n_q, m_q, P, k_c, n_docs);
    if (small_batch(n_q)) {
        const int nch = n_chunks_for(n_docs, m_q * P);
        b += align256(static_cast<size_t>(n_q) * sizeof(SelPlan)) +
             align256(static_cast<size_t>(n_q) * nch * sizeof(int32_t)) +
             align256(static_cast<size_t>(n_q) * sizeof(int32_t)) +
             align256(static_cast<size_t>(n_q) * kSelMax * 16);
    }
    return b;
}

// The fused cluster kernel saves a launch and the counter round trip, which
// pays at small batches (latency); at large batches the 16-CTA clusters
// schedule worse than the two plain kernels (cfg3 batch 256: 0.95 vs 0.78 ms
// prefilter).  DSRT_FUSED_SELECT=0 / 1 forces either path (tests run both).
static bool fused_enabled(int64_t n_q) {
    const char *e = getenv("DSRT_FUSED_SELECT");
    if (e != nullptr && e[0] == '0') return false;
    if (e != nullptr && e[0] == '1') return true;
    return small_batch(n_q);
}

// counts (written whole by the chunked pass; no memset) -> candidates.  cws:
// count_ws_bytes workspace.
static int launch_count_select(const int32_t *probed, int64_t n_q, int m_q, int P, const int64_t *post_off,
                               const int64_t *post_docs, int64_t n_docs, int64_t k_c, int64_t row_words,
                               uint32_t *counts, int k_filter, int64_t *cand, int32_t *n_cand,
                               uint8_t *cws, const int64_t *bounds_in, cudaStream_t st) {
    const int max_count = m_q * P;
    const int cb = counter_bits(max_count);
    const int nch = n_chunks_for(n_docs, max_count);
    DSRT_REQUIRE(nch < 65536 && n_q < 65536, DSRT_EUNSUPPORTED, "invalid parameter: count grid too large");
    int64_t *bnd = reinterpret_cast<int64_t *>(cws);
    uint32_t *chist = reinterpret_cast<uint32_t *>(cws + align256(static_cast<size_t>(k_c) * (nch + 1) * sizeof(int64_t)));
    const int64_t nb = k_c * (nch + 1);
    if (bounds_in != nullptr) {  // cached by the caller (dsrt_posting_chunk_bounds)
        bnd = const_cast<int64_t *>(bounds_in);
    } else {
        chunk_bounds_kernel<<<static_cast<unsigned>((nb + 255) / 256), 256, 0, st>>>(post_off, post_docs, k_c,
                                                                                  nch, chunk_docs(cb), bnd);
    }
    if (cb == 8 && nch <= kMaxFusedChunks && fused_enabled(n_q)) {  // one cluster per query set
        const size_t fsmem = fused_smem(max_count, k_filter);
        DSRT_CUDA(cudaFuncSetAttribute(count_place_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem));
        DSRT_CUDA(cudaFuncSetAttribute(count_place_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(nch), static_cast<unsigned>(n_q));
        cfg.blockDim = dim3(kPlaceThreads);
        cfg.dynamicSmemBytes = fsmem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = static_cast<unsigned>(nch);
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        DSRT_CUDA(cudaLaunchKernelEx(&cfg, count_place_kernel, probed, m_q * P, static_cast<const int64_t *>(bnd), nch,
                                     post_docs, row_words, max_count, k_filter, cand, n_cand));
        DSRT_LAUNCH_CHECK();
        return DSRT_OK;
    }
    const size_t hb = align256(static_cast<size_t>(n_q) * nch * (max_count + 1) * sizeof(uint32_t));
    uint32_t *bases = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(chist) + hb);
    int4 *plan = reinterpret_cast<int4 *>(reinterpret_cast<uint8_t *>(bases) + hb);
    uint32_t *gsum = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(plan) +
                                                  align256(static_cast<size_t>(n_q) * sizeof(int4)));
    const size_t csmem = kChunkBytes + (max_count + 1) * sizeof(uint32_t);
    auto ck = cb == 8 ? count_chunk_kernel<8> : count_chunk_kernel<16>;
    DSRT_CUDA(cudaFuncSetAttribute(ck, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
    ck<<<dim3(static_cast<unsigned>(nch), static_cast<unsigned>(n_q)), kCntThreads, csmem, st>>>(
        probed, m_q * P, bnd, nch, post_docs, row_words, max_count, counts, chist, gsum);
    if (cb == 8) {  // sort-free placement (any batch): plan per query set, then place per chunk
        sel_plan8_kernel<<<static_cast<unsigned>(n_q), 256, (max_count + 1) * sizeof(uint32_t), st>>>(
            chist, nch, max_count, k_filter, plan, bases);
        const size_t psmem = place_smem(max_count, k_filter);
        DSRT_CUDA(cudaFuncSetAttribute(sel_place_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem));
        sel_place_kernel<<<dim3(static_cast<unsigned>(nch), static_cast<unsigned>(n_q)), kPlaceThreads, psmem, st>>>(
            counts, row_words, nch, max_count, k_filter, plan, bases, gsum, cand, n_cand);
        DSRT_LAUNCH_CHECK();
        return DSRT_OK;
    }
    if (small_batch(n_q)) {  // chunk-parallel selection: plan -> chunk scans -> final sort
        uint8_t *sws = cws + count_ws_chunks(n_q, m_q, P, k_c, n_docs);
        SelPlan *plan = reinterpret_cast<SelPlan *>(sws);
        sws += align256(static_cast<size_t>(n_q) * sizeof(SelPlan));
        int32_t *tie_base = reinterpret_cast<int32_t *>(sws);
        sws += align256(static_cast<size_t>(n_q) * nch * sizeof(int32_t));
        int32_t *hits_n = reinterpret_cast<int32_t *>(sws);
        sws += align256(static_cast<size_t>(n_q) * sizeof(int32_t));
        uint64_t *hits = reinterpret_cast<uint64_t *>(sws);
        int64_t *ties = reinterpret_cast<int64_t *>(hits + static_cast<size_t>(n_q) * k_filter);
        sel_plan_kernel<<<static_cast<unsigned>(n_q), 128, (max_count + 1) * sizeof(uint32_t), st>>>(
            chist, nch, max_count, k_filter, plan, tie_base, hits_n);
        // (u8 counters never get here: they are placed above)
        sel_scan_kernel<16><<<dim3(static_cast<unsigned>(nch), static_cast<unsigned>(n_q)), kScanThreads, 0, st>>>(
            counts, row_words, nch, k_filter, plan, tie_base, hits_n, hits, ties);
        int p2 = 1;
        while (p2 < k_filter) p2 <<= 1;
        const size_t fsmem = static_cast<size_t>(p2) * sizeof(uint64_t);
        DSRT_CUDA(cudaFuncSetAttribute(sel_final_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem));
        sel_final_kernel<<<static_cast<unsigned>(n_q), kFinThreads, fsmem, st>>>(plan, hits_n, hits, ties,
                                                                                  k_filter, cand, n_cand);
        DSRT_LAUNCH_CHECK();
        return DSRT_OK;
    }
    const size_t smem = kSelMax * sizeof(uint64_t) + (max_count + 1) * sizeof(uint32_t);
    DSRT_CUDA(cudaFuncSetAttribute(select_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    select_kernel<16><<<static_cast<unsigned>(n_q), kSelThreads, smem, st>>>(
        counts, row_words, n_docs, max_count, k_filter, cand, n_cand, chist, nch);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}

struct PrefilterWs {
    size_t cand_bytes, probed_bytes, counts_bytes, total;
    int64_t n_chunks, row_words;
};

static PrefilterWs ws_layout(int64_t n_q, int m_q, int64_t k_c, int64_t n_docs, int P) {
    PrefilterWs w{};
    const int64_t rows = n_q * m_q;
    w.n_chunks = (k_c + kPTile * kPChunkTiles - 1) / (kPTile * kPChunkTiles);
    w.row_words = row_words_for(n_docs, m_q * P);
    w.cand_bytes = align256(static_cast<size_t>(rows) * w.n_chunks * P * sizeof(Cand));
    w.probed_bytes = align256(static_cast<size_t>(rows) * P * sizeof(int32_t));
    w.counts_bytes = align256(static_cast<size_t>(n_q) * w.row_words * sizeof(uint32_t));
    w.total = w.cand_bytes + w.probed_bytes + w.counts_bytes + count_ws_bytes(n_q, m_q, P, k_c, n_docs);
    return w;
}


// ====================================================================
// Tensor-core screen (exact results): sims ~ fp16(q/|q|) . fp16(c*s) on
// tcgen05.  Pass 0 finds a lower bound A'_P <= A_P of each row's P-th best
// approx value: the P-th best of the 32-column chunk maxima (P real values of
// the row; one insertion per chunk instead of per value).  Every centroid with
// approx >= A'_P - 2 eps (found from the recorded half-chunk maxima, or by a
// second GEMM sweep) is re-ranked in float64 -- that set provably contains the
// exact top-P, ties included; rows
// with more than kCandMax such centroids fall back to the exact float64 scan.  eps bounds |approx - exact| for unit-bounded rows:
// fp16 operand rounding 2u(1+u) with u = 2^-11 plus fp32 accumulation.
// ====================================================================
constexpr int kSN = 128;         // centroids per N-tile
#ifndef DSRT_SSTAGES
#define DSRT_SSTAGES 4
#endif
constexpr int kSStages = DSRT_SSTAGES;
constexpr int kSEpi = 8;                     // epilogue warps: 2 per TMEM lane quarter
constexpr int kSThreads = 64 + 32 * kSEpi;   // + TMA producer warp + MMA warp
constexpr int kSHalves = kSEpi / 4;          // column halves of a tile per lane quarter
constexpr double kScreenEps = 1.2e-3;

struct ScreenCand {
    float s;
    int32_t id;
};

template <typename T>
__device__ __forceinline__ double as_f64(T v);
template <>
__device__ __forceinline__ double as_f64<double>(double v) { return v; }
template <>
__device__ __forceinline__ double as_f64<float>(float v) { return static_cast<double>(v); }
template <>
__device__ __forceinline__ double as_f64<__half>(__half v) { return static_cast<double>(__half2float(v)); }
template <>
__device__ __forceinline__ double as_f64<__nv_bfloat16>(__nv_bfloat16 v) {
    return static_cast<double>(__bfloat162float(v));
}

template <typename TS>
__global__ void to_f16_rows_kernel(const TS *__restrict__ src, int64_t n, int d, double scale,
                                   __half *__restrict__ dst) {
    const int64_t row = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const TS *x = src + row * d;
    double s = scale;
    if (scale <= 0.0) {  // per-row normalisation
        double ss = 0.0;
        for (int k = lane; k < d; k += 32) ss = fma(as_f64(x[k]), as_f64(x[k]), ss);
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        s = ss > 0.0 ? 1.0 / sqrt(ss) : 0.0;
    }
    for (int k = lane; k < d; k += 32) dst[row * d + k] = __double2half(as_f64(x[k]) * s);
}

__device__ __forceinline__ bool s_better(float sa, int ia, float sb, int ib) {
    return sa > sb || (sa == sb && ia < ib);
}

// grid: (row tiles of 128, splits).  A = 128 query rows (resident), B = 128-
// centroid tiles streamed by TMA; TMEM double-buffered; 4 epilogue warps, one
// query row per thread.  PASS 0: branch-free running top-P of approx values
// (only when some lane improves, via a warp vote) -> out_vals[row][split][P].
// PASS 1: append every centroid with approx >= theta[row] to the row's list
// (capped at kCandMax; overflow -> the row falls back to the exact scan).
constexpr int kCandMax = 32;
constexpr int kMaxPtc = 12;

// RT = query-row tiles per CTA sharing every streamed centroid tile (RT = 2 halves
// the B-tile stream per row; the pass is bound by that stream, not the MMA).
template <int PASS, int PT, int RT = 1>
__global__ void __launch_bounds__(kSThreads, 1)
    pf_screen_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_c,
                     int64_t n_rows, int64_t k_c, int64_t tiles_per_split, int P,
                     float *__restrict__ out_vals, const float *__restrict__ theta,
                     ScreenCand *__restrict__ lists, int32_t *__restrict__ list_n, uint32_t idesc,
                     float *__restrict__ cmaxes) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int kA = 2 * 128 * 128, kB = 2 * kSN * 128;
    uint8_t *sa = smem;           // RT x kA
    uint8_t *sb = smem + RT * kA;
    __shared__ uint64_t full[kSStages], empty[kSStages], tfull[2], tempty[2], bar_a;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t m0 = static_cast<int64_t>(blockIdx.x) * 128 * RT;
    const int64_t n_tiles_total = (k_c + kSN - 1) / kSN;
    const int64_t t_lo = blockIdx.y * tiles_per_split;
    const int64_t t_hi = tmin<int64_t>(t_lo + tiles_per_split, n_tiles_total);
    if (threadIdx.x == 0) {
        tma_prefetch(&map_q);
        tma_prefetch(&map_c);
        for (int s = 0; s < kSStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], kSEpi);
        }
        mbar_init(&bar_a, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(&tmem_base, 256 * RT);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    if (warp == 0) {
        if (lane == 0) {
            mbar_arrive_expect_tx(&bar_a, RT * kA);
#pragma unroll
            for (int r = 0; r < RT; ++r) {
                tma_load_2d(sa + r * kA, &map_q, 0, static_cast<int>(m0 + r * 128), &bar_a);
                tma_load_2d(sa + r * kA + 128 * 128, &map_q, 64, static_cast<int>(m0 + r * 128), &bar_a);
            }
            int it = 0;
            for (int64_t t = t_lo; t < t_hi; ++t, ++it) {
                const int st = it % kSStages;
                if (it >= kSStages) mbar_wait(&empty[st], ((it / kSStages) - 1) & 1);
                mbar_arrive_expect_tx(&full[st], kB);
                tma_load_2d(sb + st * kB, &map_c, 0, static_cast<int>(t * kSN), &full[st]);
                tma_load_2d(sb + st * kB + kSN * 128, &map_c, 64, static_cast<int>(t * kSN), &full[st]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            mbar_wait(&bar_a, 0);
            int it = 0;
            for (int64_t t = t_lo; t < t_hi; ++t, ++it) {
                const int st = it % kSStages, acc = it & 1;
                mbar_wait(&full[st], (it / kSStages) & 1);
                if (it >= 2) mbar_wait(&tempty[acc], ((it >> 1) - 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int r = 0; r < RT; ++r) {
                    const uint32_t d = tmem + (acc * RT + r) * kSN;
                    for (int kb = 0; kb < 2; ++kb) {
                        const uint64_t ad = umma_desc_sw128(sa + r * kA + kb * 128 * 128);
                        const uint64_t bd = umma_desc_sw128(sb + st * kB + kb * kSN * 128);
#pragma unroll
                        for (int k = 0; k < 4; ++k) umma_f16(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
                    }
                }
                umma_commit(&empty[st]);
                umma_commit(&tfull[acc]);
            }
        }
    } else {
        const int quarter = warp & 3;                // TMEM lanes 32*quarter .. +31
        const int half = (warp - 2) / 4;             // which column slice of each tile
        float tvs[RT][PT];
        float worsts[RT];  // tvs[r][P-1]
        int nsubs[RT];     // PASS 2: candidates of this (row, split, half)
#pragma unroll
        for (int r = 0; r < RT; ++r) {
#pragma unroll
            for (int j = 0; j < PT; ++j) tvs[r][j] = -INFINITY;
            worsts[r] = -INFINITY;
            nsubs[r] = 0;
        }
        int it = 0;
        for (int64_t t = t_lo; t < t_hi; ++t, ++it) {
            const int acc = it & 1;
            mbar_wait(&tfull[acc], (it >> 1) & 1);
            tc_fence_after();
            const int64_t id0 = t * kSN;
            const bool full_tile = id0 + kSN <= k_c;
#pragma unroll
            for (int r = 0; r < RT; ++r) {
            const int64_t row = m0 + r * 128 + quarter * 32 + lane;
            const bool row_ok = row < n_rows;
            float (&tv)[PT] = tvs[r];
            float &worst = worsts[r];
            int &nsub = nsubs[r];
            const float th = (PASS != 0 && row_ok) ? theta[row] : INFINITY;
            const uint32_t base = tmem + (acc * RT + r) * kSN + (static_cast<uint32_t>(quarter * 32) << 16);
            // one 32-column chunk of accumulators (values r) starting at column c0
            auto chunk = [&](uint32_t (&r)[32], const int c0) {
                if (!full_tile) {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (id0 + c0 + j >= k_c) r[j] = __float_as_uint(-INFINITY);
                }
                // chunk maximum (trees over the two 16-column halves, independent FMNMX)
                // -> one vote per 32 values
                float ma[8], mb[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    ma[j] = fmaxf(__uint_as_float(r[j]), __uint_as_float(r[j + 8]));
                    mb[j] = fmaxf(__uint_as_float(r[j + 16]), __uint_as_float(r[j + 24]));
                }
#pragma unroll
                for (int w = 4; w > 0; w >>= 1)
#pragma unroll
                    for (int j = 0; j < w; ++j) {
                        ma[j] = fmaxf(ma[j], ma[j + w]);
                        mb[j] = fmaxf(mb[j], mb[j + w]);
                    }
                const float cmax = fmaxf(ma[0], mb[0]);
                // half-chunk maxima for the chunk-driven candidate pass ([chunk][row]: coalesced),
                // as fp16 rounded UP (an upper bound: a half reaching theta is never missed)
                if (PASS == 0 && cmaxes != nullptr && row_ok)
                    reinterpret_cast<uint32_t *>(cmaxes)[((id0 + c0) >> 5) * n_rows + row] =
                        static_cast<uint32_t>(__half_as_ushort(__float2half_ru(ma[0]))) |
                        (static_cast<uint32_t>(__half_as_ushort(__float2half_ru(mb[0]))) << 16);
                if (PASS == 0) {
                    // top-P of the chunk maxima: P real values of the row, so their
                    // P-th best A'_P <= A_P and theta' = A'_P - 2 eps keeps pass 1 a
                    // superset of the exact top-P (one insertion per chunk, not 32)
                    if (__any_sync(0xffffffffu, cmax > worst)) {
                        float x = cmax;
                        if (x > worst) {
#pragma unroll
                            for (int q = 0; q < PT; ++q) {
                                const float hi = fmaxf(tv[q], x);
                                x = fminf(tv[q], x);
                                tv[q] = hi;
                            }
                            worst = tv[0];
#pragma unroll
                            for (int q = 1; q < PT; ++q)
                                if (q < P) worst = tv[q];
                        }
                    }
                } else {
                    if (__any_sync(0xffffffffu, cmax >= th)) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const float v = __uint_as_float(r[j]);
                            if (v >= th) {
                                if (PASS == 2) {  // own sub-list per (row, split, half): no atomics
                                    if (nsub < kCandMax)
                                        lists[(((row * gridDim.y + blockIdx.y) * kSHalves + half) * kCandMax) + nsub] =
                                            ScreenCand{v, static_cast<int32_t>(id0 + c0 + j)};
                                    ++nsub;
                                } else {
                                    const int slot = atomicAdd(list_n + row, 1);
                                    if (slot < kCandMax)
                                        lists[row * kCandMax + slot] = ScreenCand{v, static_cast<int32_t>(id0 + c0 + j)};
                                }
                            }
                        }
                    }
                }
                        };
            if constexpr (PASS == 0) {  // both chunks of this half in flight before one wait
                uint32_t va[32], vb[32];
                const int c0a = half * (kSN / kSHalves);
                static_assert(kSN / kSHalves == 64, "two 32-column chunks per half");
                tmem_ld32(base + c0a, va);
                tmem_ld32(base + c0a + 32, vb);
                tmem_wait_ld();
                chunk(va, c0a);
                chunk(vb, c0a + 32);
            } else {
#pragma unroll 1
                for (int c0 = half * (kSN / kSHalves); c0 < (half + 1) * (kSN / kSHalves); c0 += 32) {
                    uint32_t v[32];
                    tmem_ld32(base + c0, v);
                    tmem_wait_ld();
                    chunk(v, c0);
                }
            }
            }  // r
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
#pragma unroll
        for (int r = 0; r < RT; ++r) {
            const int64_t row = m0 + r * 128 + quarter * 32 + lane;
            if (row >= n_rows) continue;
            if (PASS == 2) list_n[(row * gridDim.y + blockIdx.y) * kSHalves + half] = nsubs[r];
            if (PASS == 0) {
                // one partial list per (split, column half): n_split * kSHalves lists per row
                float *o = out_vals + ((row * gridDim.y + blockIdx.y) * kSHalves + half) * kMaxPtc;
#pragma unroll
                for (int j = 0; j < kMaxPtc; ++j) o[j] = j < PT ? tvs[r][j < PT ? j : 0] : -INFINITY;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 256 * RT);
}

// theta = (P-th best approx over all splits) - 2 eps
// (theta scaled by |x| when the screen ran on raw, unnormalised rows Xraw)
template <typename TQ>
__global__ void pf_theta_kernel(const float *__restrict__ vals, int n_split, int64_t n_rows, int P,
                                float eps2, float *__restrict__ theta, int32_t *__restrict__ list_n,
                                const TQ *__restrict__ Xraw, int d) {
    // warp per row: lanes merge disjoint partial lists, then P rounds of a warp max
    const int64_t row = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= n_rows) return;
    if (Xraw != nullptr) {  // eps bound scales with |x| (the 1.0001 margin covers rounding)
        double ss = 0.0;
        for (int k = lane; k < d; k += 32) {
            const double v = as_f64(Xraw[row * d + k]);
            ss = fma(v, v, ss);
        }
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        eps2 = static_cast<float>(eps2 * sqrt(ss) * 1.0001);
    }
    float tv[kMaxPtc];
#pragma unroll
    for (int j = 0; j < kMaxPtc; ++j) tv[j] = -INFINITY;
    for (int s = lane; s < n_split; s += 32)
        for (int j = 0; j < P; ++j) {
            float x = vals[(row * n_split + s) * kMaxPtc + j];
#pragma unroll
            for (int q = 0; q < kMaxPtc; ++q) {
                const float hi = fmaxf(tv[q], x);
                x = fminf(tv[q], x);
                tv[q] = hi;
            }
        }
    float aP = -INFINITY;
    for (int q = 0; q < P; ++q) {  // pop the warp-wide maximum P times
        float wm = tv[0];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
        const int owner = __ffs(__ballot_sync(0xffffffffu, tv[0] == wm)) - 1;
        if (lane == owner) {
#pragma unroll
            for (int k = 0; k + 1 < kMaxPtc; ++k) tv[k] = tv[k + 1];
            tv[kMaxPtc - 1] = -INFINITY;
        }
        aP = wm;
    }
    if (lane == 0) {
        theta[row] = aP - eps2;
        list_n[row] = 0;
    }
}

// Candidate pass driven by the pass-0 chunk maxima (replaces a second GEMM):
// warp = (32 query rows, span of kCSpan 32-centroid chunks).  Lane l scans row
// l's chunk maxima (cmaxes is [chunk][row], so the warp's loads coalesce); for
// every (row, chunk) whose maximum reaches theta[row] the warp recomputes the
// chunk's 32 approximations (lane = centroid) from the screen's own fp16
// operands with fp32 FMA -- within eps of exact, like the tensor-core values --
// and appends those >= theta to the row's list (> kCandMax: exact fallback).
// Soundness: an exact top-P centroid has approx >= exact - eps >= theta under
// either rounding, so its chunk's maximum reaches theta and it is appended.
// span: chunks per warp (multiple of 8), sized by the host for enough warps.
// cmaxes holds per (chunk, row) the two 16-column half maxima as fp16 rounded up;
// only halves reaching theta are recomputed (2 lanes per centroid, 64 dims each).
__global__ void __launch_bounds__(256)
    pf_chunk_cand_kernel(const uint32_t *__restrict__ cmaxes, int64_t n_chunks, int span,
                         const float *__restrict__ theta, const __half *__restrict__ q16,
                         const __half *__restrict__ c16, int64_t k_c, int64_t n_rows,
                         ScreenCand *__restrict__ lists, int32_t *__restrict__ list_n) {
    __shared__ float qf[8][128];  // the current match's query row, as float
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32;
    const int64_t j0 = (static_cast<int64_t>(blockIdx.y) * 8 + warp) * span;
    if (j0 >= n_chunks) return;
    const int64_t j1 = tmin<int64_t>(j0 + span, n_chunks);
    const int64_t row = r0 + lane;
    const bool row_ok = row < n_rows;
    const float th = row_ok ? theta[row] : INFINITY;
    const int part = lane >> 4;  // which 64 dims of the centroid this lane sums
    // one (row, chunk half) match: lanes (c, c + 16) share centroid c of the half
    auto process = [&](int l, int64_t j, int hh) {
        const int64_t rr = r0 + l;
        const float thr = __shfl_sync(0xffffffffu, th, l);
        {  // stage the query row as float (lane k: dims 4k .. 4k+3)
            const uint2 h = __ldg(reinterpret_cast<const uint2 *>(q16 + rr * 128) + lane);
            const float2 a = __half22float2(*reinterpret_cast<const __half2 *>(&h.x));
            const float2 b = __half22float2(*reinterpret_cast<const __half2 *>(&h.y));
            reinterpret_cast<float4 *>(qf[warp])[lane] = make_float4(a.x, a.y, b.x, b.y);
        }
        __syncwarp();
        const int64_t cid = j * 32 + hh * 16 + (lane & 15);
        float acc = 0.f;
        if (cid < k_c) {
            const uint4 *cv = reinterpret_cast<const uint4 *>(c16 + cid * 128) + part * 8;
            uint4 c[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) c[k] = __ldg(cv + k);
            float a0 = 0.f, a1 = 0.f;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const __half2 *ch2 = reinterpret_cast<const __half2 *>(&c[k]);
                const float4 q0 = reinterpret_cast<const float4 *>(qf[warp])[part * 16 + 2 * k];
                const float4 q1 = reinterpret_cast<const float4 *>(qf[warp])[part * 16 + 2 * k + 1];
                const float2 c0 = __half22float2(ch2[0]), c1 = __half22float2(ch2[1]);
                const float2 c2 = __half22float2(ch2[2]), c3 = __half22float2(ch2[3]);
                a0 = fmaf(q0.x, c0.x, a0); a1 = fmaf(q0.y, c0.y, a1);
                a0 = fmaf(q0.z, c1.x, a0); a1 = fmaf(q0.w, c1.y, a1);
                a0 = fmaf(q1.x, c2.x, a0); a1 = fmaf(q1.y, c2.y, a1);
                a0 = fmaf(q1.z, c3.x, a0); a1 = fmaf(q1.w, c3.y, a1);
            }
            acc = a0 + a1;
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 16);
        __syncwarp();
        const bool ok = lane < 16 && cid < k_c && acc >= thr;
        const unsigned okm = __ballot_sync(0xffffffffu, ok);
        int base = 0;
        if (lane == 0 && okm != 0u) base = atomicAdd(list_n + rr, __popc(okm));
        base = __shfl_sync(0xffffffffu, base, 0);
        const int slot = base + __popc(okm & ((1u << lane) - 1u));
        if (ok && slot < kCandMax) lists[rr * kCandMax + slot] = ScreenCand{acc, static_cast<int32_t>(cid)};
    };
    __shared__ uint32_t mq[8][16];  // per warp: the match ballots of the 8 chunks x 2 halves
    for (int64_t jb = j0; jb < j1; jb += 8) {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            v[u] = (row_ok && jb + u < j1) ? __ldg(cmaxes + (jb + u) * n_rows + row) : 0xfc00fc00u;  // -inf
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const bool h0 = __half2float(__ushort_as_half(static_cast<unsigned short>(v[u] & 0xffffu))) >= th;
            const bool h1 = __half2float(__ushort_as_half(static_cast<unsigned short>(v[u] >> 16))) >= th;
            const unsigned m0 = __ballot_sync(0xffffffffu, h0), m1 = __ballot_sync(0xffffffffu, h1);
            if (lane == 0) {
                mq[warp][2 * u] = m0;
                mq[warp][2 * u + 1] = m1;
            }
        }
        __syncwarp();
        // one rolled loop over the matches keeps a single copy of process() (the
        // unrolled form thrashed the instruction cache)
#pragma unroll 1
        for (int k = 0; k < 16; ++k) {
            unsigned m = mq[warp][k];
            while (m != 0u) {
                const int l = __ffs(m) - 1;
                m &= m - 1u;
                process(l, jb + (k >> 1), k & 1);
            }
        }
        __syncwarp();
    }
}

// warp per row: exact float64 re-rank of the collected candidates -> probed ids;
// flags rows whose list overflowed (fallback to the exact scan).
template <typename TQ>
__global__ void pf_rerank_kernel(const ScreenCand *__restrict__ lists, const int32_t *__restrict__ list_n,
                                 const TQ *__restrict__ Q, const double *__restrict__ cents,
                                 int64_t n_rows, int d, int P, int32_t *__restrict__ probed,
                                 int32_t *__restrict__ fallback, double *__restrict__ best = nullptr) {
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= n_rows) return;
    const int n = list_n[row];
    if (n > kCandMax || n < P) {  // overflow (or fewer candidates than probes: degenerate)
        if (lane == 0) fallback[row] = 1;
        return;
    }
    if (lane == 0) fallback[row] = 0;
    double ex = -INFINITY;
    int eid = 0x7fffffff;
    if (lane < n) {
        const int c = lists[row * kCandMax + lane].id;
        const TQ *q = Q + row * d;
        const double *cv = cents + static_cast<int64_t>(c) * d;
        double acc = 0.0;
        for (int k = 0; k < d; ++k) acc = fma(as_f64(q[k]), cv[k], acc);
        ex = acc;
        eid = c;
    }
    double es = -INFINITY;
    int ei = 0x7fffffff;
    warp_topP_merge(es, ei, ex, eid, P);
    if (lane < P) probed[row * P + lane] = ei;
    if (best != nullptr && lane == 0) best[row] = es;  // P == 1: the exact top similarity
}

// as pf_rerank_kernel, for the prefilter's per-writer sub-lists (pass 2): a row's
// W = n_split * kSHalves sub-lists are compacted into a 32-entry staging row
// (overflow of the total -> exact fallback), then re-ranked in float64.
template <typename TQ>
__global__ void pf_rerank_sub_kernel(const ScreenCand *__restrict__ sub, const int32_t *__restrict__ sub_n, int W,
                                     const TQ *__restrict__ Q, const double *__restrict__ cents,
                                     int64_t n_rows, int d, int P, int32_t *__restrict__ probed,
                                     int32_t *__restrict__ fallback) {
    __shared__ ScreenCand stage[8][kCandMax];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (row >= n_rows) return;
    int total = 0;
    for (int w0 = 0; w0 < W; w0 += 32) {
        const int w = w0 + lane;
        const int cnt = w < W ? sub_n[row * W + w] : 0;
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int base = total + incl - cnt;
        for (int i = 0; i < cnt && base + i < kCandMax; ++i)
            stage[warp][base + i] = sub[(row * W + w) * static_cast<int64_t>(kCandMax) + i];
        total += __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncwarp();
    if (total > kCandMax || total < P) {
        if (lane == 0) fallback[row] = 1;
        return;
    }
    if (lane == 0) fallback[row] = 0;
    double ex = -INFINITY;
    int eid = 0x7fffffff;
    if (lane < total) {
        const int c = stage[warp][lane].id;
        const TQ *q = Q + row * d;
        const double *cv = cents + static_cast<int64_t>(c) * d;
        double acc = 0.0;
        for (int k = 0; k < d; ++k) acc = fma(as_f64(q[k]), cv[k], acc);
        ex = acc;
        eid = c;
    }
    double es = -INFINITY;
    int ei = 0x7fffffff;
    warp_topP_merge(es, ei, ex, eid, P);
    if (lane < P) probed[row * P + lane] = ei;
}

// exact float64 scan for flagged rows (one CTA per row; rare)
template <typename TQ>
__global__ void __launch_bounds__(256)
    pf_fallback_kernel(const int32_t *__restrict__ fallback, const TQ *__restrict__ Q,
                       const double *__restrict__ cents, int64_t n_rows, int64_t k_c, int d, int P,
                       int32_t *__restrict__ probed, double *__restrict__ best = nullptr) {
    const int64_t row = blockIdx.x;
    if (row >= n_rows || fallback[row] == 0) return;
    __shared__ double q[512];
    __shared__ double cs[8][32];
    __shared__ int ci[8][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int k = threadIdx.x; k < d && k < 512; k += blockDim.x) q[k] = as_f64(Q[row * d + k]);
    __syncthreads();
    double ts = -INFINITY;
    int ti = 0x7fffffff;
    for (int64_t c0 = static_cast<int64_t>(warp) * 32; c0 < k_c; c0 += 256) {
        const int64_t c = c0 + lane;
        double s = -INFINITY;
        int id = 0x7fffffff;
        if (c < k_c) {
            double acc = 0.0;
            for (int k = 0; k < d; ++k) acc = fma(q[k], cents[c * d + k], acc);
            s = acc;
            id = static_cast<int>(c);
        }
        warp_topP_merge(ts, ti, s, id, P);
    }
    cs[warp][lane] = ts;
    ci[warp][lane] = ti;
    __syncthreads();
    if (warp == 0) {
        double fs = -INFINITY;
        int fi = 0x7fffffff;
        for (int w = 0; w < 8; ++w) warp_topP_merge(fs, fi, lane < P ? cs[w][lane] : -INFINITY,
                                                    lane < P ? ci[w][lane] : 0x7fffffff, P);
        if (lane < P) probed[row * P + lane] = fi;
        if (best != nullptr && lane == 0) best[row] = fs;
    }
}

}  // namespace dsrt

using namespace dsrt;

extern "C" int64_t dsrt_posting_chunk_bounds_size(int64_t k_c, int64_t n_docs, int m_q, int probe) {
    return k_c * (n_chunks_for(n_docs, m_q * tmax(probe, 1)) + 1);
}

extern "C" int dsrt_posting_chunk_bounds(const int64_t *post_off, const int64_t *post_docs, int64_t k_c,
                                         int64_t n_docs, int m_q, int probe, int64_t *out, void *stream) {
    DSRT_REQUIRE(k_c >= 1 && n_docs >= 1 && m_q >= 1 && probe >= 1, DSRT_EINVAL, "invalid parameter: empty");
    const int P = static_cast<int>(tmin<int64_t>(probe, k_c));
    const int cb = counter_bits(m_q * P);
    const int nch = n_chunks_for(n_docs, m_q * P);
    const int64_t nb = k_c * (nch + 1);
    chunk_bounds_kernel<<<static_cast<unsigned>((nb + 255) / 256), 256, 0, as_stream(stream)>>>(
        post_off, post_docs, k_c, nch, chunk_docs(cb), out);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}


// ====================================================================
// General path: probe > kMaxProbe, k_filter > kSelMax or m_q*probe > 65535
// (the reference accepts any values, prefilter.py:111-144).  Same arithmetic as
// the fast path, with the per-row / per-query-set selections done by K4:
//   sims    thread per (row, centroid): the sequential-FMA float64 dot of
//           probe_kernel (bit-identical sims) -> rows x k_c
//   probe   K4 top-P per row by (sim desc, id asc) = argsort(-sims, stable)[:P]
//   count   warp per (query row, probed centroid) posting: u32 atomics per doc
//   select  K4 top-k_filter per query set over keys (count, or -1 untouched)
//           by (count desc, index asc); untouched docs never enter the list.
// Temporaries are stream-ordered allocations, processed in bounded batches.
namespace dsrt {
int topk_run_ext(const double *scores, int64_t ld, int64_t n, int k, double *out_s, uint64_t *out_id,
                 int64_t n_rows, cudaStream_t st);

__global__ void pfg_sims_kernel(const double *__restrict__ Q, int64_t rows, int d,
                                const double *__restrict__ cents, int64_t k_c, double *__restrict__ sims) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= rows * k_c) return;
    const int64_t r = i / k_c, c = i - r * k_c;
    const double *q = Q + r * d, *x = cents + c * d;
    double acc = 0.0;
    for (int k = 0; k < d; ++k) acc = fma(__ldg(q + k), __ldg(x + k), acc);
    sims[i] = acc;
}

__global__ void pfg_probed_kernel(const uint64_t *__restrict__ ids, int64_t n, int32_t *__restrict__ probed) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) probed[i] = static_cast<int32_t>(ids[i]);
}

// grid.x: (query row, probe rank) pairs of one query set batch, grid.y: query set
__global__ void pfg_count_kernel(const int32_t *__restrict__ probed, int mp, const int64_t *__restrict__ post_off,
                                 const int64_t *__restrict__ post_docs, int64_t n_docs,
                                 uint32_t *__restrict__ counts) {
    const int64_t qs = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t pr = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + warp;
    if (pr >= mp) return;
    const int64_t c = probed[qs * mp + pr];
    uint32_t *row = counts + qs * n_docs;
    for (int64_t e = post_off[c] + lane; e < post_off[c + 1]; e += 32) atomicAdd(row + post_docs[e], 1u);
}

__global__ void pfg_keys_kernel(const uint32_t *__restrict__ counts, int64_t n, double *__restrict__ keys) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) keys[i] = counts[i] > 0u ? static_cast<double>(counts[i]) : -1.0;
}

// row per query set: cand = selected doc indices (count >= 1), -1 after n_cand
__global__ void pfg_cand_kernel(const double *__restrict__ s, const uint64_t *__restrict__ ids, int k,
                                int64_t *__restrict__ cand, int32_t *__restrict__ n_cand) {
    const int64_t qs = blockIdx.x;
    __shared__ int n;
    if (threadIdx.x == 0) n = 0;
    __syncthreads();
    int mine = 0;
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        const bool ok = s[qs * k + i] >= 1.0;
        cand[qs * k + i] = ok ? static_cast<int64_t>(ids[qs * k + i]) : -1;
        mine += ok;
    }
    atomicAdd(&n, mine);
    __syncthreads();
    if (threadIdx.x == 0) n_cand[qs] = n;
}

static int prefilter_general(const double *Q, int64_t n_q, int m_q, int d, const double *cents, int64_t k_c,
                             const int64_t *post_off, const int64_t *post_docs, int64_t n_docs, int P,
                             int k_filter, int64_t *cand, int32_t *n_cand, cudaStream_t st) {
    const int64_t rows = n_q * m_q;
    int32_t *probed = nullptr;
    DSRT_CUDA(malloc_async(reinterpret_cast<void **>(&probed), static_cast<size_t>(rows) * P * 4, st));
    // ---- probe: sims in row batches of <= 256 MB, top-P per row
    const int64_t rb = tmax<int64_t>(1, tmin<int64_t>(rows, (int64_t(256) << 20) / (8 * k_c)));
    double *sims = nullptr, *ts = nullptr;
    uint64_t *ti = nullptr;
    DSRT_CUDA(malloc_async(reinterpret_cast<void **>(&sims), static_cast<size_t>(rb) * k_c * 8, st));
    DSRT_CUDA(malloc_async(reinterpret_cast<void **>(&ts), static_cast<size_t>(rb) * P * 8, st));
    DSRT_CUDA(malloc_async(reinterpret_cast<void **>(&ti), static_cast<size_t>(rb) * P * 8, st));
    int rc = DSRT_OK;
    for (int64_t r0 = 0; r0 < rows && rc == DSRT_OK; r0 += rb) {
        const int64_t nr = tmin(rb, rows - r0);
        pfg_sims_kernel<<<static_cast<unsigned>((nr * k_c + 255) / 256), 256, 0, st>>>(Q + r0 * d, nr, d, cents,
                                                                                      k_c, sims);
        rc = topk_run_ext(sims, k_c, k_c, P, ts, ti, nr, st);
        if (rc == DSRT_OK)
            pfg_probed_kernel<<<static_cast<unsigned>((nr * P + 255) / 256), 256, 0, st>>>(ti, nr * P, probed + r0 * P);
    }
    cudaFreeAsync(sims, st);
    cudaFreeAsync(ts, st);
    cudaFreeAsync(ti, st);
    if (rc) {
        cudaFreeAsync(probed, st);
        return rc;
    }
    // ---- count + select in query-set batches of <= 512 MB of counters and keys
    const int64_t qb = tmax<int64_t>(1, tmin<int64_t>(n_q, (int64_t(512) << 20) / (12 * tmax<int64_t>(1, n_docs))));
    uint32_t *counts = nullptr;
    double *keys = nullptr, *os = nullptr;
    uint64_t *oi = nullptr;
    DSRT_CUDA(malloc_async(reinterpret_cast<void **>(&counts), static_cast<size_t>(qb) * n_docs * 4, st));
    DSRT_CUDA(malloc_async(reinterpret_cast<void **>(&keys), static_cast<size_t>(qb) * n_docs * 8, st));
    DSRT_CUDA(malloc_async(reinterpret_cast<void **>(&os), static_cast<size_t>(qb) * k_filter * 8, st));
    DSRT_CUDA(malloc_async(reinterpret_cast<void **>(&oi), static_cast<size_t>(qb) * k_filter * 8, st));
    const int mp = m_q * P;
    for (int64_t q0 = 0; q0 < n_q && rc == DSRT_OK; q0 += qb) {
        const int64_t nq = tmin(qb, n_q - q0);
        if (cudaMemsetAsync(counts, 0, static_cast<size_t>(nq) * n_docs * 4, st) != cudaSuccess) {
            rc = DSRT_ECUDA;
            break;
        }
        pfg_count_kernel<<<dim3(static_cast<unsigned>((mp + 7) / 8), static_cast<unsigned>(nq)), 256, 0, st>>>(
            probed + q0 * mp, mp, post_off, post_docs, n_docs, counts);
        pfg_keys_kernel<<<static_cast<unsigned>((nq * n_docs + 255) / 256), 256, 0, st>>>(counts, nq * n_docs, keys);
        rc = topk_run_ext(keys, n_docs, n_docs, k_filter, os, oi, nq, st);
        if (rc == DSRT_OK)
            pfg_cand_kernel<<<static_cast<unsigned>(nq), 256, 0, st>>>(os, oi, k_filter, cand + q0 * k_filter,
                                                                      n_cand + q0);
    }
    cudaFreeAsync(counts, st);
    cudaFreeAsync(keys, st);
    cudaFreeAsync(os, st);
    cudaFreeAsync(oi, st);
    cudaFreeAsync(probed, st);
    if (rc) return rc;
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}
}  // namespace dsrt

extern "C" size_t dsrt_prefilter_workspace(int64_t n_q, int m_q, int64_t k_c, int64_t n_docs,
                                           int probe) {
    const int P = static_cast<int>(tmin<int64_t>(tmax(probe, 1), k_c));
    return ws_layout(n_q, m_q, k_c, n_docs, P).total;
}

extern "C" int dsrt_prefilter(const double *Q, int64_t n_q, int m_q, int d, const double *cents,
                              int64_t k_c, const int64_t *post_off, const int64_t *post_docs,
                              int64_t n_docs, const int64_t *chunk_bounds, int probe, int k_filter,
                              int64_t *cand, int32_t *n_cand, void *workspace, size_t ws_bytes,
                              void *stream) {
    DSRT_REQUIRE(probe >= 1, DSRT_EINVAL, "invalid parameter: probe must be >= 1, got %d", probe);
    DSRT_REQUIRE(k_filter >= 1, DSRT_EINVAL, "invalid parameter: k_filter must be >= 1, got %d", k_filter);
    DSRT_REQUIRE(m_q >= 1 && n_q >= 0, DSRT_EINVAL, "Q must be a non-empty (m_q, d) matrix");
    DSRT_REQUIRE(k_c >= 1 && d >= 1, DSRT_EINVAL, "invalid parameter: k=%lld d=%d", (long long)k_c, d);
    const int P = static_cast<int>(tmin<int64_t>(probe, k_c));
    const int max_count = m_q * P;
    DSRT_REQUIRE(k_c < (1LL << 31), DSRT_EUNSUPPORTED, "invalid parameter: too many centroids");
    if (n_q == 0) return DSRT_OK;
    if (P > kMaxProbe || k_filter > kSelMax || max_count > 65535)
        return prefilter_general(Q, n_q, m_q, d, cents, k_c, post_off, post_docs, n_docs, P, k_filter, cand,
                                 n_cand, as_stream(stream));
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
    int rc2 = launch_count_select(probed, n_q, m_q, P, post_off, post_docs, n_docs, k_c, w.row_words, counts,
                                  k_filter, cand, n_cand, ws + w.cand_bytes + w.probed_bytes + w.counts_bytes,
                                  chunk_bounds, st);
    if (rc2) return rc2;
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}

// ---------------------------------------------------------- TC entry points
namespace dsrt {
template <int PASS, int PT, int RT = 1>
static int launch_screen(dim3 g, size_t smem, cudaStream_t st, const CUtensorMap &mq, const CUtensorMap &mc,
                         int64_t rows, int64_t k_c, int64_t tps, int P, float *vals, const float *theta,
                         ScreenCand *lists, int32_t *listn, uint32_t idesc, float *cmaxes = nullptr) {
    DSRT_CUDA(cudaFuncSetAttribute(pf_screen_kernel<PASS, PT, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    pf_screen_kernel<PASS, PT, RT><<<g, kSThreads, smem, st>>>(mq, mc, rows, k_c, tps, P, vals, theta, lists,
                                                               listn, idesc, cmaxes);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}
}  // namespace dsrt
extern "C" int dsrt_to_f16_rows(const double *src, int64_t n, int d, double scale, void *dst,
                                void *stream) {
    DSRT_REQUIRE(n >= 0 && d >= 1, DSRT_EINVAL, "invalid parameter: n=%lld d=%d", (long long)n, d);
    if (n == 0) return DSRT_OK;
    to_f16_rows_kernel<double><<<static_cast<unsigned>((n + 7) / 8), 256, 0, as_stream(stream)>>>(
        src, n, d, scale, static_cast<__half *>(dst));
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}

namespace dsrt {
struct TcWs {
    size_t q16, screen, theta, lists, listn, probed, fallback, counts, cnt_ws, cmax, total;
    int64_t n_split, row_words, tiles_per_split;
};
constexpr size_t kCmaxCap = size_t(1) << 30;
// Query-row tiles per screen CTA: 2 once there are enough rows to fill the GPU
// with 256-row CTAs (each streamed centroid tile then feeds two MMAs).
static int screen_rt(int64_t rows) {
    if (const char *e = getenv("DSRT_SCREEN_RT")) return atoi(e) >= 2 ? 2 : 1;
    return (rows + 255) / 256 >= 8 ? 2 : 1;
}
static TcWs tc_ws_layout(int64_t n_q, int m_q, int64_t k_c, int64_t n_docs, int P) {
    TcWs w{};
    const int64_t rows = n_q * m_q;
    const int rt = screen_rt(rows);
    const int64_t m_tiles = (rows + 128 * rt - 1) / (128 * rt);  // CTA row tiles
    const int64_t n_tiles = (k_c + kSN - 1) / kSN;
    const int sms = sm_count();
    // about one wave of CTAs: fewer splits amortise each row's list warm-up
    int64_t bs = rt == 1 ? (sms + m_tiles / 2) / m_tiles : sms / m_tiles;
    bs = tmax<int64_t>(1, tmin<int64_t>(n_tiles, bs));
    if (const char *e = getenv("DSRT_SCREEN_SPLIT")) bs = tmax<int64_t>(1, tmin<int64_t>(n_tiles, atoi(e)));
    w.n_split = bs;
    w.tiles_per_split = (n_tiles + bs - 1) / bs;
    w.n_split = (n_tiles + w.tiles_per_split - 1) / w.tiles_per_split;
    w.row_words = row_words_for(n_docs, m_q * P);
    w.q16 = align256(static_cast<size_t>(m_tiles * 128 * rt) * 128 * 2);
    w.screen = align256(static_cast<size_t>(rows) * w.n_split * kSHalves * kMaxPtc * sizeof(float));
    w.theta = align256(static_cast<size_t>(rows) * sizeof(float));
    // per-writer candidate sub-lists: (row, split, column half) x kCandMax
    w.lists = align256(static_cast<size_t>(rows) * w.n_split * kSHalves * kCandMax * sizeof(ScreenCand));
    w.listn = align256(static_cast<size_t>(rows) * w.n_split * kSHalves * sizeof(int32_t));
    w.probed = align256(static_cast<size_t>(rows) * P * sizeof(int32_t));
    w.fallback = align256(static_cast<size_t>(rows) * sizeof(int32_t));
    w.counts = align256(static_cast<size_t>(n_q) * w.row_words * sizeof(uint32_t));
    w.cnt_ws = count_ws_bytes(n_q, m_q, P, k_c, n_docs);
    // pass-0 chunk maxima for the chunk-driven candidate pass (else a second GEMM pass)
    const size_t cmax = static_cast<size_t>(n_tiles) * (kSN / 32) * rows * sizeof(float);
    const char *g2 = getenv("DSRT_SCREEN_GEMM2");  // tests: force the second-GEMM candidate pass
    w.cmax = (cmax <= kCmaxCap && !(g2 != nullptr && g2[0] == '1')) ? align256(cmax) : 0;
    w.total = w.q16 + w.screen + w.theta + w.lists + w.listn + w.probed + w.fallback + w.counts + w.cnt_ws +
              w.cmax;
    return w;
}
}  // namespace dsrt

extern "C" size_t dsrt_prefilter_tc_workspace(int64_t n_q, int m_q, int64_t k_c, int64_t n_docs,
                                              int probe) {
    const int P = static_cast<int>(tmin<int64_t>(tmax(probe, 1), k_c));
    return tc_ws_layout(n_q, m_q, k_c, n_docs, P).total;
}

extern "C" int dsrt_prefilter_tc(const double *Q, int64_t n_q, int m_q, int d, const double *cents,
                                 const void *cents_f16, double cent_max_norm, int64_t k_c,
                                 const int64_t *post_off, const int64_t *post_docs, int64_t n_docs,
                                 const int64_t *chunk_bounds,
                                 int probe, int k_filter, int64_t *cand, int32_t *n_cand,
                                 void *workspace, size_t ws_bytes, void *stream) {
    DSRT_REQUIRE(probe >= 1, DSRT_EINVAL, "invalid parameter: probe must be >= 1, got %d", probe);
    DSRT_REQUIRE(k_filter >= 1, DSRT_EINVAL, "invalid parameter: k_filter must be >= 1, got %d", k_filter);
    DSRT_REQUIRE(m_q >= 1 && n_q >= 0, DSRT_EINVAL, "Q must be a non-empty (m_q, d) matrix");
    DSRT_REQUIRE(d == 128, DSRT_EUNSUPPORTED, "invalid parameter: tensor-core prefilter needs d=128");
    const int P = static_cast<int>(tmin<int64_t>(probe, k_c));
    const int max_count = m_q * P;
    DSRT_REQUIRE(k_c < (1LL << 31) && cent_max_norm > 0, DSRT_EINVAL, "invalid parameter: centroids");
    if (n_q == 0) return DSRT_OK;
    if (P > kMaxPtc || k_filter > kSelMax || max_count > 65535)  // outside the screen's envelope
        return prefilter_general(Q, n_q, m_q, d, cents, k_c, post_off, post_docs, n_docs, P, k_filter, cand,
                                 n_cand, as_stream(stream));
    const TcWs w = tc_ws_layout(n_q, m_q, k_c, n_docs, P);
    DSRT_REQUIRE(workspace != nullptr && ws_bytes >= w.total, DSRT_EINVAL,
                 "invalid parameter: prefilter workspace too small");
    cudaStream_t st = as_stream(stream);
    uint8_t *ws = static_cast<uint8_t *>(workspace);
    size_t o = 0;
    __half *q16 = reinterpret_cast<__half *>(ws + o); o += w.q16;
    float *vals = reinterpret_cast<float *>(ws + o); o += w.screen;
    float *theta = reinterpret_cast<float *>(ws + o); o += w.theta;
    ScreenCand *lists = reinterpret_cast<ScreenCand *>(ws + o); o += w.lists;
    int32_t *listn = reinterpret_cast<int32_t *>(ws + o); o += w.listn;
    int32_t *probed = reinterpret_cast<int32_t *>(ws + o); o += w.probed;
    int32_t *fallback = reinterpret_cast<int32_t *>(ws + o); o += w.fallback;
    uint32_t *counts = reinterpret_cast<uint32_t *>(ws + o); o += w.counts;
    uint8_t *cnt_ws = ws + o; o += w.cnt_ws;
    float *cmaxes = w.cmax > 0 ? reinterpret_cast<float *>(ws + o) : nullptr;
    const int64_t rows = n_q * m_q;
    const int rt = screen_rt(rows);
    const int64_t m_tiles = (rows + 127) / 128;
    const int64_t q_rows = ((rows + 128 * rt - 1) / (128 * rt)) * 128 * rt;  // padded, zero-filled
    DSRT_CUDA(cudaMemsetAsync(q16, 0, w.q16, st));
    to_f16_rows_kernel<double><<<static_cast<unsigned>((rows + 7) / 8), 256, 0, st>>>(Q, rows, d, 0.0, q16);
    CUtensorMap mq, mc;
    int rc = make_tmap_2d(&mq, q16, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 128, q_rows, 256, 64, 128,
                          CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    rc = make_tmap_2d(&mc, cents_f16, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 128, k_c, 256, 64, kSN,
                      CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    const size_t smem = 1024 + 2 * 128 * 128 + kSStages * 2 * kSN * 128;
    dim3 g(static_cast<unsigned>(m_tiles), static_cast<unsigned>(w.n_split));
    const uint32_t idesc = idesc_f16(128, kSN, 0, 0);
    if (rt == 2 && P <= 4) {  // two row tiles per CTA share each centroid tile
        const dim3 g2(static_cast<unsigned>(q_rows / 256), static_cast<unsigned>(w.n_split));
        rc = launch_screen<0, 4, 2>(g2, smem + 2 * 128 * 128, st, mq, mc, rows, k_c, w.tiles_per_split, P, vals,
                                    nullptr, nullptr, nullptr, idesc, cmaxes);
    } else {
        rc = P <= 4 ? launch_screen<0, 4>(g, smem, st, mq, mc, rows, k_c, w.tiles_per_split, P, vals, nullptr, nullptr, nullptr, idesc, cmaxes)
           : P <= 8 ? launch_screen<0, 8>(g, smem, st, mq, mc, rows, k_c, w.tiles_per_split, P, vals, nullptr, nullptr, nullptr, idesc, cmaxes)
                    : launch_screen<0, 12>(g, smem, st, mq, mc, rows, k_c, w.tiles_per_split, P, vals, nullptr, nullptr, nullptr, idesc, cmaxes);
    }
    if (rc) return rc;
    // eps in normalised units (|q^| = 1, |c*s| <= 1)
    pf_theta_kernel<double><<<static_cast<unsigned>((rows * 32 + 255) / 256), 256, 0, st>>>(
        vals, static_cast<int>(w.n_split * kSHalves), rows, P, static_cast<float>(2.0 * kScreenEps), theta, listn,
        nullptr, d);
    if (cmaxes != nullptr) {  // candidates from the chunk maxima + fp16 SIMT recompute
        const int64_t n_chunks = ((k_c + kSN - 1) / kSN) * (kSN / 32);
        const int64_t rgroups = (rows + 31) / 32;
        // ~32 warps per SM of work, spans of 8..64 chunks
        const int64_t want = 512LL * sm_count();  // many short spans: matches are latency-bound
        const int span = static_cast<int>(tmax<int64_t>(8, tmin<int64_t>(64, ((n_chunks * rgroups / want) + 7) / 8 * 8)));
        const dim3 gc(static_cast<unsigned>(rgroups), static_cast<unsigned>((n_chunks + 8LL * span - 1) / (8LL * span)));
        pf_chunk_cand_kernel<<<gc, 256, 0, st>>>(reinterpret_cast<const uint32_t *>(cmaxes), n_chunks, span, theta, q16,
                                                  static_cast<const __half *>(cents_f16), k_c, rows, lists, listn);
        pf_rerank_kernel<double><<<static_cast<unsigned>((rows * 32 + 255) / 256), 256, 0, st>>>(
            lists, listn, Q, cents, rows, d, P, probed, fallback);
    } else {  // second GEMM pass collecting approx >= theta
        rc = launch_screen<2, 4>(g, smem, st, mq, mc, rows, k_c, w.tiles_per_split, P, nullptr, theta, lists,
                                 listn, idesc);
        if (rc) return rc;
        pf_rerank_sub_kernel<double><<<static_cast<unsigned>((rows * 32 + 255) / 256), 256, 0, st>>>(
            lists, listn, static_cast<int>(w.n_split * kSHalves), Q, cents, rows, d, P, probed, fallback);
    }
    pf_fallback_kernel<double><<<static_cast<unsigned>(rows), 256, 0, st>>>(fallback, Q, cents, rows, k_c, d,
                                                                           P, probed);
    rc = launch_count_select(probed, n_q, m_q, P, post_off, post_docs, n_docs, k_c, w.row_words, counts,
                             k_filter, cand, n_cand, cnt_ws, chunk_bounds, st);
    if (rc) return rc;
    DSRT_LAUNCH_CHECK();
    (void)cent_max_norm;
    return DSRT_OK;
}

// ===================================================================
// Exact centroid assignment (build_centroid_index, prefilter.py:85-108):
// argmax_c <x, c> with np.argmax's first-index tie rule, via the same
// tensor-core screen (P = 1) + float64 re-rank + exact fallback.  fp16/bf16
// rows feed TMA directly (no copy; the screen error then scales with |x|);
// float32/float64 rows are normalised into an fp16 staging buffer.
// ===================================================================
namespace dsrt {
constexpr int64_t kAssignChunk = 1 << 22;

static size_t assign_ws_layout(int64_t n, size_t *parts) {
    const int64_t ch = tmin<int64_t>(n, kAssignChunk);
    const int64_t tiles = (ch + 127) / 128;
    parts[0] = align256(static_cast<size_t>(tiles * 128) * 128 * 2);        // q16 staging
    parts[1] = align256(static_cast<size_t>(ch) * kSHalves * kMaxPtc * sizeof(float));  // pass-0 values (1 split)
    parts[2] = align256(static_cast<size_t>(ch) * sizeof(float));            // theta
    parts[3] = align256(static_cast<size_t>(ch) * kCandMax * sizeof(ScreenCand));
    parts[4] = align256(static_cast<size_t>(ch) * sizeof(int32_t));          // list counts
    parts[5] = align256(static_cast<size_t>(ch) * sizeof(int32_t));          // fallback flags
    size_t t = 0;
    for (int i = 0; i < 6; ++i) t += parts[i];
    return t;
}

template <typename TQ>
static int assign_impl(const TQ *X, int64_t n, int d, const double *cents, const void *cents_lp,
                       int64_t k_c, bool raw, bool bf16, int32_t *assign_out, void *ws,
                       cudaStream_t st, double *best = nullptr) {
    size_t part[6];
    assign_ws_layout(n, part);
    uint8_t *w = static_cast<uint8_t *>(ws);
    __half *q16 = reinterpret_cast<__half *>(w);
    float *vals = reinterpret_cast<float *>(w + part[0]);
    float *theta = reinterpret_cast<float *>(w + part[0] + part[1]);
    ScreenCand *lists = reinterpret_cast<ScreenCand *>(w + part[0] + part[1] + part[2]);
    int32_t *listn = reinterpret_cast<int32_t *>(w + part[0] + part[1] + part[2] + part[3]);
    int32_t *fallback = reinterpret_cast<int32_t *>(w + part[0] + part[1] + part[2] + part[3] + part[4]);
    const CUtensorMapDataType dt = bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    CUtensorMap mc;
    int rc = make_tmap_2d(&mc, cents_lp, dt, 128, k_c, 256, 64, kSN, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    const size_t smem = 1024 + 2 * 128 * 128 + kSStages * 2 * kSN * 128;
    const uint32_t idesc = idesc_f16(128, kSN, bf16, bf16);
    const int64_t n_tiles_c = (k_c + kSN - 1) / kSN;
    const double eps = raw ? (bf16 ? 8e-3 : 1.2e-3) : kScreenEps;
    for (int64_t r0 = 0; r0 < n; r0 += kAssignChunk) {
        const int64_t rows = tmin<int64_t>(kAssignChunk, n - r0);
        const int64_t m_tiles = (rows + 127) / 128;
        CUtensorMap mq;
        if (raw) {
            rc = make_tmap_2d(&mq, X + r0 * d, dt, 128, rows, 256, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
        } else {
            DSRT_CUDA(cudaMemsetAsync(q16, 0, part[0], st));
            to_f16_rows_kernel<TQ><<<static_cast<unsigned>((rows + 7) / 8), 256, 0, st>>>(X + r0 * d, rows, d, 0.0, q16);
            rc = make_tmap_2d(&mq, q16, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 128, m_tiles * 128, 256, 64, 128,
                              CU_TENSOR_MAP_SWIZZLE_128B);
        }
        if (rc) return rc;
        const int sms = sm_count();
        int64_t n_split = tmax<int64_t>(1, tmin<int64_t>(n_tiles_c, (sms + m_tiles / 2) / m_tiles));
        const int64_t tps = (n_tiles_c + n_split - 1) / n_split;
        n_split = (n_tiles_c + tps - 1) / tps;
        dim3 g(static_cast<unsigned>(m_tiles), static_cast<unsigned>(n_split));
        // vals is sized for one split; more splits only happen for small chunks
        float *v = vals;
        float *vtmp = nullptr;
        if (n_split > 1) {
            DSRT_CUDA(malloc_async(reinterpret_cast<void **>(&vtmp), rows * n_split * kSHalves * kMaxPtc * sizeof(float), st));
            v = vtmp;
        }
        rc = launch_screen<0, 4>(g, smem, st, mq, mc, rows, k_c, tps, 1, v, nullptr, nullptr, nullptr, idesc);
        if (rc) return rc;
        pf_theta_kernel<TQ><<<static_cast<unsigned>((rows * 32 + 255) / 256), 256, 0, st>>>(
            v, static_cast<int>(n_split * kSHalves), rows, 1, static_cast<float>(2.0 * eps), theta, listn,
            raw ? X + r0 * d : nullptr, d);
        rc = launch_screen<1, 4>(g, smem, st, mq, mc, rows, k_c, tps, 1, nullptr, theta, lists, listn, idesc);
        if (rc) return rc;
        pf_rerank_kernel<TQ><<<static_cast<unsigned>((rows * 32 + 255) / 256), 256, 0, st>>>(
            lists, listn, X + r0 * d, cents, rows, d, 1, assign_out + r0, fallback,
            best ? best + r0 : nullptr);
        pf_fallback_kernel<TQ><<<static_cast<unsigned>(rows), 256, 0, st>>>(fallback, X + r0 * d, cents, rows,
                                                                             k_c, d, 1, assign_out + r0,
                                                                             best ? best + r0 : nullptr);
        if (vtmp) cudaFreeAsync(vtmp, st);
        DSRT_LAUNCH_CHECK();
    }
    return DSRT_OK;
}
size_t assign_simt_ws(int64_t n, int d);
int assign_simt(const void *X, int dtype, int64_t n, int d, const double *cents, int64_t k,
                int32_t *assign, void *ws, cudaStream_t st);

// k-means assignment step: float64 unit rows, exact argmax and its similarity.
int assign_unit_rows_f64(const double *X, int64_t n, const double *cents, const void *cents_f16,
                         int64_t k_c, int32_t *assign_out, double *best, void *ws, cudaStream_t st) {
    return assign_impl<double>(X, n, 128, cents, cents_f16, k_c, false, false, assign_out, ws, st, best);
}

}  // namespace dsrt

extern "C" size_t dsrt_assign_centroids_workspace(int64_t n, int d, int64_t k_c) {
    size_t parts[6];
    (void)k_c;
    if (d != 128) return assign_simt_ws(n, d);
    return assign_ws_layout(tmax<int64_t>(n, 1), parts);
}

extern "C" int dsrt_assign_centroids(const void *X, int x_dtype, int64_t n, int d, const double *cents,
                                     const void *cents_lp, int64_t k_c, int32_t *assign_out,
                                     void *workspace, size_t ws_bytes, void *stream) {
    DSRT_REQUIRE(k_c >= 1 && k_c < (1LL << 31), DSRT_EINVAL, "invalid parameter: k=%lld", (long long)k_c);
    DSRT_REQUIRE(ws_bytes >= dsrt_assign_centroids_workspace(n, d, k_c), DSRT_EINVAL,
                 "invalid parameter: assignment workspace too small");
    if (n == 0) return DSRT_OK;
    cudaStream_t st = as_stream(stream);
    if (d != 128) return assign_simt(X, x_dtype, n, d, cents, k_c, assign_out, workspace, st);
    switch (x_dtype) {
        case DSRT_F16: return assign_impl<__half>(static_cast<const __half *>(X), n, d, cents, cents_lp, k_c, true, false, assign_out, workspace, st);
        case DSRT_BF16: return assign_impl<__nv_bfloat16>(static_cast<const __nv_bfloat16 *>(X), n, d, cents, cents_lp, k_c, true, true, assign_out, workspace, st);
        case DSRT_F32: return assign_impl<float>(static_cast<const float *>(X), n, d, cents, cents_lp, k_c, false, false, assign_out, workspace, st);
        case DSRT_F64: return assign_impl<double>(static_cast<const double *>(X), n, d, cents, cents_lp, k_c, false, false, assign_out, workspace, st);
        default: break;
    }
    set_error("invalid parameter: x dtype %d", x_dtype);
    return DSRT_EINVAL;
}

__global__ void to_bf16_rows_kernel(const double *__restrict__ src, int64_t n, int d, double scale,
                                    __nv_bfloat16 *__restrict__ dst) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n * d) dst[i] = __double2bfloat16(src[i] * scale);
}

extern "C" int dsrt_to_bf16_rows(const double *src, int64_t n, int d, double scale, void *dst, void *stream) {
    DSRT_REQUIRE(n >= 0 && d >= 1 && scale > 0, DSRT_EINVAL, "invalid parameter: n=%lld d=%d", (long long)n, d);
    if (n == 0) return DSRT_OK;
    to_bf16_rows_kernel<<<static_cast<unsigned>((n * d + 255) / 256), 256, 0, as_stream(stream)>>>(
        src, n, d, scale, static_cast<__nv_bfloat16 *>(dst));
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}
