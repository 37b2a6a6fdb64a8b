// K3 -- DESSERT set scoring (sigma = max, A = mean with default weights).
//
// Replaces the reference's per-candidate Python loop
//   _score_chunk / _score_one / score_candidate   (index.py:183-261)
// which sorts collision keys gathered from TinyTables (sketch.py:156-178).
// The dense form computed here is the same integer count
//   c_q = max_j sum_t [code_q[t] == code_j[t]]
// (pinned by the reference's own tests: sketch.py oracle equivalence,
// test_index.py:130-144), followed by the float64 LUT and numpy's pairwise
// mean (index.py:216), reproduced bit-for-bit in lane_score() below.
//
// Compare arithmetic is bit-sliced: per 32 tables and C code bits, the
// mismatch mask is OR_b (q_b XOR x_b) -- C LOP3 + 1 POPC per 32 table
// compares -- and the running max of matches is a running min of mismatches
// (POPC + add + min fuse into VIADDMNMX for L = 64).
//
// Mapping: one warp = one query set, lane = query vector, so max_j needs no
// cross-lane reduction; set vectors are read from shared memory with
// broadcast LDS.128.  When a set ends, each lane parks its c_q byte in a
// per-warp shared "slot" row; after 32 sets every lane turns one slot row
// into one set score (LUT + numpy pairwise order) -- the float64 epilogue is
// thus spread over lanes instead of being a warp-wide reduction per set.
#pragma once
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace dsrt {

constexpr unsigned kFull = 0xffffffffu;


template <int QPL>
struct SlotGeom {
    static constexpr int kRow = 32 * QPL + 4;  // bytes per slot row (+4: bank skew)
    static constexpr int kBytes = 32 * kRow;   // 32 slots per warp
};

// numpy pairwise_sum_DOUBLE for one leaf (n <= 128): 8 strided accumulators,
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), sequential remainder; n < 8 sums
// sequentially from 0.0.  Then the reduction identity 0.0 and / n (np.mean).
// w_s: per-query-vector weights in shared memory (all 1.0 for the default
// scorer: 1.0 * v == v exactly, so one code path serves both, index.py:216).
__device__ __forceinline__ double lane_score(const uint8_t *__restrict__ row, int n,
                                             const double *__restrict__ lut_s,
                                             const double *__restrict__ w_s) {
    double res;
    if (n < 8) {
        res = 0.0;
        for (int i = 0; i < n; ++i) res = __dadd_rn(res, __dmul_rn(w_s[i], lut_s[row[i]]));
    } else {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dmul_rn(w_s[j], lut_s[row[j]]);
        const int n8 = n - (n & 7);
        for (int i = 8; i < n8; i += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], __dmul_rn(w_s[i + j], lut_s[row[i + j]]));
        }
        res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                        __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (int i = n8; i < n; ++i) res = __dadd_rn(res, __dmul_rn(w_s[i], lut_s[row[i]]));
    }
    return __ddiv_rn(__dadd_rn(0.0, res), static_cast<double>(n));
}

// Threshold-append epilogue (exhaustive search, search.cu): instead of
// storing every score, a set whose score reaches the query set's current
// threshold tau[q] (the k-th best score so far) is appended as (score, doc id)
// to the query set's survivor list at cnt[q]++ (one atomic per warp flush).
// Appends past `cap` are counted but not stored (overflow -> caller reruns).
struct AppendOut {
    const double *tau;        // (n_qsets) thresholds; nullptr = append mode off
    int32_t *cnt;             // (n_qsets) list fill
    double *cs;               // (n_qsets, cap) scores
    uint64_t *cid;            // (n_qsets, cap) doc ids
    const uint64_t *doc_ids;  // (n_sets) doc id of each set
    int64_t cap;
};

// Per-warp deferred epilogue: 32 slot rows of c_q bytes.
template <int QPL>
struct Slots {
    uint8_t *buf;        // this warp's SlotGeom<QPL>::kBytes
    int n = 0;           // filled slots (warp-uniform)
    uint32_t valid = 0;  // bit i: slot i holds a valid set

    // park the finished set's c_q (= L - min mismatches) in slot n
    __device__ __forceinline__ void push(const int (&rmin)[QPL], int L, int m_q, bool ok) {
        const int lane = threadIdx.x & 31;
        uint8_t *row = buf + n * SlotGeom<QPL>::kRow;
#pragma unroll
        for (int s = 0; s < QPL; ++s) {
            const int qi = lane + 32 * s;
            if (qi < m_q) row[qi] = static_cast<uint8_t>(L - rmin[s]);
        }
        valid |= (ok ? 1u : 0u) << n;
        ++n;
    }

    // write slot row idx without touching the counters (exhaustive kernel: the
    // QS query sets of a warp share one slot counter; every pushed set is valid)
    __device__ __forceinline__ void put(const int (&rmin)[QPL], int L, int m_q, int idx) const {
        const int lane = threadIdx.x & 31;
        uint8_t *row = buf + idx * SlotGeom<QPL>::kRow;
#pragma unroll
        for (int s = 0; s < QPL; ++s) {
            const int qi = lane + 32 * s;
            if (qi < m_q) row[qi] = static_cast<uint8_t>(L - rmin[s]);
        }
    }

    // split-lane layout (QPL == 1): lanes l and l + 16 hold queries l and
    // l + 16 after the half-warp combine; lanes < 16 write both
    __device__ __forceinline__ void push_split(const int (&rmin)[2], int L, int m_q, bool ok) {
        const int lane = threadIdx.x & 31;
        uint8_t *row = buf + n * SlotGeom<QPL>::kRow;
        if (lane < 16) {
            if (lane < m_q) row[lane] = static_cast<uint8_t>(L - rmin[0]);
            if (lane + 16 < m_q) row[lane + 16] = static_cast<uint8_t>(L - rmin[1]);
        }
        valid |= (ok ? 1u : 0u) << n;
        ++n;
    }

    // lane i < n scores slot i -> out[col0 + i]; optional uint16 max counts
    __device__ __forceinline__ void flush(int m_q, const double *__restrict__ lut_s,
                                          const double *__restrict__ w_s,
                                          double *__restrict__ out_row, int64_t col0,
                                          uint16_t *__restrict__ mc, int64_t mc_row0,
                                          int mc_stride, int mc_q0) {
        const int lane = threadIdx.x & 31;
        __syncwarp();
        if (lane < n) {
            const uint8_t *row = buf + lane * SlotGeom<QPL>::kRow;
            const bool ok = (valid >> lane) & 1u;
            if (out_row != nullptr)
                out_row[col0 + lane] =
                    ok ? lane_score(row, m_q, lut_s, w_s) : __longlong_as_double(0x7ff8000000000000ll);
            if (mc != nullptr && ok) {
                uint16_t *dst = mc + (mc_row0 + col0 + lane) * mc_stride + mc_q0;
                for (int i = 0; i < m_q; ++i) dst[i] = row[i];
            }
        }
        __syncwarp();
        n = 0;
        valid = 0;
    }

    // append-mode flush: lane i < n scores slot i (set index set0 + i) and
    // appends it when score >= tau[qs]
    __device__ __forceinline__ void flush_append(int m_q, const double *__restrict__ lut_s,
                                                 const double *__restrict__ w_s,
                                                 const AppendOut &app, int64_t qs, int64_t set0) {
        const int lane = threadIdx.x & 31;
        __syncwarp();
        double sc = 0.0;
        bool keep = false;
        if (lane < n && ((valid >> lane) & 1u)) {
            sc = lane_score(buf + lane * SlotGeom<QPL>::kRow, m_q, lut_s, w_s);
            keep = sc >= __ldg(app.tau + qs);
        }
        const unsigned bal = __ballot_sync(kFull, keep);
        if (bal != 0u) {
            int base = 0;
            if (lane == 0) base = atomicAdd(app.cnt + qs, __popc(bal));
            base = __shfl_sync(kFull, base, 0);
            const int64_t pos = base + __popc(bal & ((1u << lane) - 1u));
            if (keep && pos < app.cap) {
                app.cs[qs * app.cap + pos] = sc;
                app.cid[qs * app.cap + pos] = __ldg(app.doc_ids + set0 + lane);
            }
        }
        __syncwarp();
        n = 0;
        valid = 0;
    }
};

template <int K, int W, int QPL>
__device__ __forceinline__ void load_queries(uint32_t (&q)[QPL][K * W],
                                             const uint32_t *__restrict__ qrecs, int64_t qset,
                                             int m_q, bool active) {
    constexpr int R = ((K * W) + 3) & ~3;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int s = 0; s < QPL; ++s) {
        const int qi = lane + 32 * s;
        const bool ok = active && qi < m_q;
        const uint32_t *src = qrecs + (qset * m_q + (ok ? qi : 0)) * R;
#pragma unroll
        for (int i = 0; i < K * W; ++i) q[s][i] = ok ? __ldg(src + i) : 0u;
    }
}

// Mismatch count of one query (registers) vs one record (uint32 words).
template <int K, int W>
__device__ __forceinline__ int mismatches(const uint32_t (&q)[K * W], const uint32_t *x) {
    int mm = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
        uint32_t acc = q[w] ^ x[w];
#pragma unroll
        for (int b = 1; b < K; ++b) acc |= q[b * W + w] ^ x[b * W + w];
        mm += __popc(acc);
    }
    return mm;
}

// Split-lane candidate mapping (m_q in (16, 32]): lane l holds queries
// (l & 15) and (l & 15) + 16, and half-warp h = l >> 4 scans the set vectors
// 2p + h, so every broadcast LDS feeds two pairs per lane; the halves are
// combined (shfl_xor 16) when the set ends.
template <int K, int W>
__device__ __forceinline__ void load_queries_split(uint32_t (&q)[2][K * W],
                                                   const uint32_t *__restrict__ qrecs, int64_t qset,
                                                   int m_q) {
    constexpr int R = ((K * W) + 3) & ~3;
    const int l = threadIdx.x & 15;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const int qi = l + 16 * s;
        const bool ok = qi < m_q;
        const uint32_t *src = qrecs + (qset * m_q + (ok ? qi : 0)) * R;
#pragma unroll
        for (int i = 0; i < K * W; ++i) q[s][i] = ok ? __ldg(src + i) : 0u;
    }
}

template <int K, int W>
__device__ __forceinline__ int min3(int a, int b, int c) {
    if constexpr (W == 1) return __vimin3_s32(a, b, c);
    else return min(a, min(b, c));
}

// The pair loop is written with explicit trip counts (16 vectors per trip, then 0-3
// groups of 4, then one clamped block for the last 1-3 vectors): the counts are three
// shifts of nv, where the compiler's own unroll-by-4 prologue took ~20 instructions per
// piece (cfg3 candidate scoring: x4 unroll 1.377 -> 1.336 ms; explicit trips: see DESIGN).
template <int K, int W>
__device__ __forceinline__ void scan_split(const uint32_t (&q)[2][K * W], int (&rmin)[2],
                                           const uint32_t *xs, int nv) {
    constexpr int R = ((K * W) + 3) & ~3;
    constexpr int V = R / 4;  // uint4 per vector
    const int h = (threadIdx.x >> 4) & 1;
    // group of 4 vectors at px: half h takes vectors h and 2 + h
    auto group = [&](const uint4 *px) {
        uint4 xa[V], xb[V];
#pragma unroll
        for (int u = 0; u < V; ++u) {
            xa[u] = px[u];
            xb[u] = px[2 * V + u];
        }
#pragma unroll
        for (int s = 0; s < 2; ++s)
            rmin[s] = min3<K, W>(rmin[s], mismatches<K, W>(q[s], reinterpret_cast<const uint32_t *>(xa)),
                                 mismatches<K, W>(q[s], reinterpret_cast<const uint32_t *>(xb)));
    };
    const uint4 *px = reinterpret_cast<const uint4 *>(xs) + h * V;
    for (int t = nv >> 4; t > 0; --t) {
        group(px);
        group(px + 4 * V);
        group(px + 8 * V);
        group(px + 12 * V);
        px += 16 * V;
    }
    for (int r = (nv >> 2) & 3; r > 0; --r) {
        group(px);
        px += 4 * V;
    }
    // one tail block for the last 1-3 vectors: half h takes 4g + h and 4g + 2 + h,
    // indices clamped to nv - 1 (a repeated vector leaves the minimum unchanged)
    if (nv & 3) {
        const int g4 = nv & ~3;
        const int va = min(g4 + h, nv - 1), vb = min(g4 + 2 + h, nv - 1);
        const uint4 *xr = reinterpret_cast<const uint4 *>(xs);
        uint4 xa[V], xb[V];
#pragma unroll
        for (int u = 0; u < V; ++u) {
            xa[u] = xr[va * V + u];
            xb[u] = xr[vb * V + u];
        }
#pragma unroll
        for (int s = 0; s < 2; ++s)
            rmin[s] = min3<K, W>(rmin[s], mismatches<K, W>(q[s], reinterpret_cast<const uint32_t *>(xa)),
                                 mismatches<K, W>(q[s], reinterpret_cast<const uint32_t *>(xb)));
    }
}

// Process vectors [0, nv) of a shared-memory record array.  For W = 1 two
// vectors share one 3-input min (VIMNMX3): 8 LOP3 + 0.5 min per (query,
// vector) at C = 8 instead of 8 + 1; for W = 2 ptxas already fuses the
// two-word add with the min (VIADDMNMX).
// PU: unroll of the W = 1 pair loop (4 in candidate mode: one query set per
// warp needs more vectors in flight; 2 in exhaustive mode, where register
// blocking of several query sets already provides them)
template <int K, int W, int QPL, int PU = 2>
__device__ __forceinline__ void scan_vectors(const uint32_t (&q)[QPL][K * W], int (&rmin)[QPL],
                                             const uint32_t *xs, int nv) {
    constexpr int R = ((K * W) + 3) & ~3;
    const uint4 *x4 = reinterpret_cast<const uint4 *>(xs);
    int i = 0;
    if constexpr (W == 1 && PU == 4) {
        // pointer-walked groups of 4 vectors: loads at immediate offsets, one
        // add + compare per group instead of re-deriving the address from i
        const uint4 *p = x4;
        const uint4 *const pend = x4 + (nv & ~3) * (R / 4);
        for (; p != pend; p += 4 * (R / 4)) {
            uint4 xv[4][R / 4];
#pragma unroll
            for (int g = 0; g < 4; ++g)
#pragma unroll
                for (int u = 0; u < R / 4; ++u) xv[g][u] = p[g * (R / 4) + u];
#pragma unroll
            for (int s = 0; s < QPL; ++s) {
                const int m0 = __vimin3_s32(rmin[s], mismatches<K, W>(q[s], reinterpret_cast<const uint32_t *>(xv[0])),
                                            mismatches<K, W>(q[s], reinterpret_cast<const uint32_t *>(xv[1])));
                rmin[s] = __vimin3_s32(m0, mismatches<K, W>(q[s], reinterpret_cast<const uint32_t *>(xv[2])),
                                       mismatches<K, W>(q[s], reinterpret_cast<const uint32_t *>(xv[3])));
            }
        }
        i = nv & ~3;
        if (nv & 2) {
            uint4 xa[R / 4], xb[R / 4];
#pragma unroll
            for (int u = 0; u < R / 4; ++u) {
                xa[u] = x4[i * (R / 4) + u];
                xb[u] = x4[(i + 1) * (R / 4) + u];
            }
#pragma unroll
            for (int s = 0; s < QPL; ++s)
                rmin[s] = __vimin3_s32(rmin[s], mismatches<K, W>(q[s], reinterpret_cast<const uint32_t *>(xa)),
                                       mismatches<K, W>(q[s], reinterpret_cast<const uint32_t *>(xb)));
            i += 2;
        }
    } else if constexpr (W == 1) {
        // explicit trip counts (shifts of nv) and a walking pointer: the compiler's own
        // unroll prologue cost ~20 instructions per call, i.e. per set
        constexpr int V = R / 4;
        auto pair = [&](const uint4 *px) {
            uint4 xa[V], xb[V];
#pragma unroll
            for (int u = 0; u < V; ++u) {
                xa[u] = px[u];
                xb[u] = px[V + u];
            }
            const uint32_t *a = reinterpret_cast<const uint32_t *>(xa);
            const uint32_t *b = reinterpret_cast<const uint32_t *>(xb);
#pragma unroll
            for (int s = 0; s < QPL; ++s)
                rmin[s] = __vimin3_s32(rmin[s], mismatches<K, W>(q[s], a), mismatches<K, W>(q[s], b));
        };
        const uint4 *px = x4;
        if constexpr (PU >= 2) {
            for (int t = nv >> 2; t > 0; --t) {
                pair(px);
                pair(px + 2 * V);
                px += 4 * V;
            }
            if (nv & 2) pair(px);
        } else {
            for (int t = nv >> 1; t > 0; --t) {
                pair(px);
                px += 2 * V;
            }
        }
        if (nv & 1) {  // odd last vector
            uint4 xv[V];
#pragma unroll
            for (int u = 0; u < V; ++u) xv[u] = x4[(nv - 1) * V + u];
            const uint32_t *x = reinterpret_cast<const uint32_t *>(xv);
#pragma unroll
            for (int s = 0; s < QPL; ++s) rmin[s] = min(rmin[s], mismatches<K, W>(q[s], x));
        }
        i = nv;
    }
    // one vector at a time: the W >= 2 path (4 per trip, explicit counts as above) and the
    // odd last vector of the 4-vector W = 1 groups
    constexpr int V1 = R / 4;
    auto single = [&](const uint4 *px) {
        uint4 xv[V1];
#pragma unroll
        for (int u = 0; u < V1; ++u) xv[u] = px[u];
        const uint32_t *x = reinterpret_cast<const uint32_t *>(xv);
#pragma unroll
        for (int s = 0; s < QPL; ++s) rmin[s] = min(rmin[s], mismatches<K, W>(q[s], x));
    };
    const uint4 *p1 = x4 + i * V1;
    const int left = nv - i;
    for (int t = left >> 2; t > 0; --t) {
        single(p1);
        single(p1 + V1);
        single(p1 + 2 * V1);
        single(p1 + 3 * V1);
        p1 += 4 * V1;
    }
    for (int r = left & 3; r > 0; --r) {
        single(p1);
        p1 += V1;
    }
}

// Lane-distributed window of set_off: lane l holds set_off[base + l] (absolute 64-bit
// indices), or -- OffWindowRel -- set_off[s_lo + base + l] - vbeg as an int: the window is
// then built on set_off + s_lo with vbase = the chunk's first vector, so the consumer loop
// runs on chunk-relative 32-bit indices (launch_all keeps a chunk below 2^31 vectors and sets).
struct OffWindow {
    const int64_t *off;
    int64_t base, limit;  // valid indices <= limit
    int64_t v;
    __device__ __forceinline__ void load(int64_t b) {
        base = b;
        const int64_t i = b + (threadIdx.x & 31);
        v = i <= limit ? __ldg(off + i) : INT64_MAX;
    }
    __device__ __forceinline__ int64_t get(int64_t i) {  // warp-uniform i
        if (i - base >= 32) load(i);
        return __shfl_sync(kFull, v, static_cast<int>(i - base));
    }
};
struct OffWindowRel {
    const int64_t *off;  // set_off + s_lo
    int base, limit;
    int v;
    int64_t vbase;
    __device__ __forceinline__ void load(int b) {
        base = b;
        const int i = b + (threadIdx.x & 31);
        v = i <= limit ? static_cast<int>(__ldg(off + i) - vbase) : INT32_MAX;
    }
    __device__ __forceinline__ int get(int i) {  // warp-uniform i
        if (i - base >= 32) load(i);
        return __shfl_sync(kFull, v, i - base);
    }
};

// ------------------------------------------------------- exhaustive (shared)
// Exhaustive-mode tiles: 16 KB of records per TMA bulk copy (256 vectors at L=64 C=7,
// 512 at L=32 C=8): fewer ring waits and fewer sets split across tiles than
// 128-vector tiles (cfg1 0.906 -> 0.914, cfg4 0.809 -> 0.82 of the INT roofline)
// while 4 stages + slots keep 2 CTAs per SM.
#ifndef DSRT_TILE_BYTES
#define DSRT_TILE_BYTES 16384
#endif
template <int K, int W>
constexpr int tile_vec() {
    constexpr int rb = ((((K * W) + 3) & ~3) * 4);  // record bytes
    return DSRT_TILE_BYTES / rb > 128 ? DSRT_TILE_BYTES / rb : 128;
}
constexpr int kStages = 4;     // smem ring depth

template <int K, int W>
constexpr int tile_bytes() {
    return tile_vec<K, W>() * (((K * W) + 3) & ~3) * 4;
}
template <int K, int W, int QPL, int NW, int QS>
constexpr size_t all_smem_static() {
    return kStages * tile_bytes<K, W>() + 2 * kStages * sizeof(uint64_t) +
           NW * QS * SlotGeom<QPL>::kBytes;
}

#ifndef DSRT_ALL_MINB
#define DSRT_ALL_MINB 2
#endif
// grid: (query-set groups of NW*QS, set chunks).  One producer warp streams the
// chunk's plane records through a kStages ring with cp.async.bulk (TMA);
// NW consumer warps share every tile, each register-blocking QS query sets
// (lane l holds query l of each), so one broadcast LDS feeds QS pairs.
//
// CL = 2: the grid's x (query-set groups) is clustered in pairs that score the same
// chunk; every record tile is fetched once per pair -- tile t by CTA t % 2 with a
// multicast bulk copy into both CTAs' ring -- and each consumer warp releases the
// stage on both CTAs' barriers (count NW * CL), so each record byte crosses the L2
// -> SM path once per pair instead of twice.
template <int K, int W, int QPL, int NW, int QS, int CL = 1>
__global__ void __launch_bounds__((NW + 1) * 32, DSRT_ALL_MINB)
    score_all_kernel(const uint32_t *__restrict__ recs, const int64_t *__restrict__ set_off,
                     int64_t set_begin, int64_t set_end, const uint32_t *__restrict__ qrecs,
                     int64_t n_qsets, int m_q, int L, const double *__restrict__ lut,
                     const double *__restrict__ weights, double *__restrict__ scores, int64_t ld,
                     uint16_t *__restrict__ maxcounts, int mc_stride, int mc_q0, int n_chunks,
                     AppendOut app) {
    constexpr int R = ((K * W) + 3) & ~3;
    constexpr int S = QS * QPL;  // register slots per lane
    constexpr int kTileVec = tile_vec<K, W>();
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t *tiles = reinterpret_cast<uint32_t *>(smem);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + kStages * tile_bytes<K, W>());
    uint64_t *empty = full + kStages;
    uint8_t *slot_mem = reinterpret_cast<uint8_t *>(empty + kStages);
    double *lut_s = reinterpret_cast<double *>(slot_mem + NW * QS * SlotGeom<QPL>::kBytes);
    double *w_s = lut_s + (L + 1);  // m_q weights (1.0 when none); used only when m_q <= 128
    __shared__ int64_t bounds[2];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int chunk = blockIdx.y;
    if (threadIdx.x == 0) {
        const int64_t nset = set_end - set_begin;
        const int64_t v0 = __ldg(set_off + set_begin), v1 = __ldg(set_off + set_end);
        const int64_t tv = v1 - v0;
        const int64_t t_lo = v0 + (tv * chunk) / n_chunks;
        const int64_t t_hi = v0 + (tv * (chunk + 1)) / n_chunks;
        bounds[0] = chunk == 0 ? set_begin : set_begin + lower_bound_i64(set_off + set_begin, nset, t_lo);
        bounds[1] = chunk == n_chunks - 1 ? set_end
                                          : set_begin + lower_bound_i64(set_off + set_begin, nset, t_hi);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW * CL);
        }
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i <= L; i += blockDim.x) lut_s[i] = __ldg(lut + i);
    for (int i = threadIdx.x; i < m_q; i += blockDim.x) w_s[i] = weights ? __ldg(weights + i) : 1.0;
    __syncthreads();
    if constexpr (CL > 1) cluster_sync_threads();  // peers' barriers exist before any multicast
    const int64_t s_lo = bounds[0], s_hi = bounds[1];
    if (s_lo >= s_hi) return;  // the whole cluster (same chunk) leaves together
    const int64_t vbeg = __ldg(set_off + s_lo), vend = __ldg(set_off + s_hi);
    const int64_t n_tiles = (vend - vbeg + kTileVec - 1) / kTileVec;
    [[maybe_unused]] const uint32_t crank = CL > 1 ? static_cast<uint32_t>(blockIdx.x % CL) : 0u;

    if (warp == NW) {  // ---------------- producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_last();
            for (int64_t t = 0; t < n_tiles; ++t) {
                const int st = static_cast<int>(t % kStages);
                const uint32_t n = static_cast<uint32_t>(t / kStages);
                if (t >= kStages) mbar_wait_suspend(&empty[st], (n - 1) & 1);
                const int64_t tv0 = vbeg + t * kTileVec;
                const int64_t nvec = tmin<int64_t>(kTileVec, vend - tv0);
                const uint32_t bytes = static_cast<uint32_t>(nvec * R * 4);
                mbar_arrive_expect_tx(&full[st], bytes);
                if constexpr (CL > 1) {
                    if (static_cast<uint32_t>(t % CL) == crank)
                        bulk_g2s_keep_mc(tiles + st * (kTileVec * R), recs + tv0 * R, bytes, &full[st], pol,
                                         static_cast<uint16_t>((1u << CL) - 1u));
                } else {
                    bulk_g2s_keep(tiles + st * (kTileVec * R), recs + tv0 * R, bytes, &full[st], pol);
                }
            }
        }
        if constexpr (CL > 1) {
            __syncwarp();  // the .aligned cluster barrier needs the whole warp converged
            cluster_sync_threads();  // stay until the peers are done with our ring
        }
        return;
    }

    // ------------------------- consumers: QS query sets per warp, lane = query
    const int64_t qset0 = (static_cast<int64_t>(blockIdx.x) * NW + warp) * QS;
    const bool any_active = qset0 < n_qsets;
    uint32_t q[S][K * W];
#pragma unroll
    for (int j = 0; j < QS; ++j) {
        const bool act = qset0 + j < n_qsets;
        load_queries<K, W, QPL>(*reinterpret_cast<uint32_t(*)[QPL][K * W]>(&q[j * QPL][0]), qrecs,
                                act ? qset0 + j : 0, m_q, act);
    }
    int rmin[S];
#pragma unroll
    for (int s = 0; s < S; ++s) rmin[s] = L;
    Slots<QPL> slots[QS];
#pragma unroll
    for (int j = 0; j < QS; ++j) slots[j].buf = slot_mem + (warp * QS + j) * SlotGeom<QPL>::kBytes;
    // Set and vector indices of the consumer loop.  Two-word records (L = 64, cfg1) run on
    // chunk-relative 32-bit indices (fewer instructions per set: 205.2 -> 201.2 ms at cfg1
    // shape); for one-word records the same change re-scheduled the hot loop for the worse
    // (226.8 -> 230.4 ms at cfg4 shape), so they keep absolute 64-bit indices.
    using I = std::conditional_t<(W >= 2), int, int64_t>;
    constexpr bool REL = sizeof(I) == 4;
    const I s1 = static_cast<I>(REL ? s_hi - s_lo : s_hi);
    const I v0 = static_cast<I>(REL ? 0 : vbeg), v1 = static_cast<I>(REL ? vend - vbeg : vend);
    using Win = std::conditional_t<REL, OffWindowRel, OffWindow>;
    Win win;
    if constexpr (REL) win = Win{set_off + s_lo, 0, static_cast<int>(s1), 0, vbeg};
    else win = Win{set_off, 0, s_hi, 0};
    I s = static_cast<I>(REL ? 0 : s_lo);
    win.load(s + 1);

    int64_t slot_col = s_lo - set_begin;
    I s_end_v = win.get(s + 1);
    I v = v0;
    int nslot = 0;  // filled slot rows, shared by the QS query sets (all valid)
    auto flush_all = [&]() {
#pragma unroll
        for (int j = 0; j < QS; ++j) {
            const int64_t qs = qset0 + j;
            slots[j].n = nslot;
            slots[j].valid = nslot == 32 ? 0xffffffffu : ((1u << nslot) - 1u);
            if (qs < n_qsets) {
                if (app.tau != nullptr)
                    slots[j].flush_append(m_q, lut_s, w_s, app, qs, set_begin + slot_col);
                else
                    slots[j].flush(m_q, lut_s, w_s, scores ? scores + qs * ld : nullptr, slot_col,
                                   maxcounts, qs * ld, mc_stride, mc_q0);
            }
            slots[j].n = 0;
            slots[j].valid = 0;
        }
    };
    // slot-row stores (Slots::put for the QS query sets): per-lane predicates and one
    // running offset, the row of query set j at a compile-time distance
    bool st_ok[QPL];
#pragma unroll
    for (int i = 0; i < QPL; ++i) st_ok[i] = lane + 32 * i < m_q;
    uint8_t *const wbase = slot_mem + warp * QS * SlotGeom<QPL>::kBytes + lane;
    int wro = 0;  // nslot * kRow
    auto finish_set = [&]() {
#pragma unroll
        for (int j = 0; j < QS; ++j)
#pragma unroll
            for (int i = 0; i < QPL; ++i)
                if (st_ok[i])
                    wbase[wro + j * SlotGeom<QPL>::kBytes + 32 * i] = static_cast<uint8_t>(L - rmin[j * QPL + i]);
        wro += SlotGeom<QPL>::kRow;
#pragma unroll
        for (int i = 0; i < S; ++i) rmin[i] = L;
        ++s;
        if (++nslot == 32) {
            if (any_active) flush_all();
            nslot = 0;
            wro = 0;
            slot_col += 32;
        }
        if (s < s1) s_end_v = win.get(s + 1);
    };

    for (int64_t t = 0; t < n_tiles; ++t) {
        const int st = static_cast<int>(t % kStages);
        mbar_wait(&full[st], static_cast<uint32_t>(t / kStages) & 1);
        const uint32_t *tile = tiles + st * (kTileVec * R);
        const I tv0 = v0 + static_cast<I>(t) * kTileVec;
        const I tv1 = tmin<I>(tv0 + kTileVec, v1);
        while (v < tv1) {
            const I stop = tmin<I>(s_end_v, tv1);
            if (any_active && stop > v)
                scan_vectors<K, W, S>(q, rmin, tile + (v - tv0) * R, static_cast<int>(stop - v));
            v = stop;
            while (s < s1 && v == s_end_v) finish_set();
        }
        __syncwarp();
        if (lane == 0) {
            if constexpr (CL > 1) {
#pragma unroll
                for (int r = 0; r < CL; ++r) mbar_arrive_rank(&empty[st], static_cast<uint32_t>(r));
            } else {
                mbar_arrive(&empty[st]);
            }
        }
    }
    while (s < s1) finish_set();  // trailing empty sets (validated away upstream)
    if (any_active && nslot > 0) flush_all();
    if constexpr (CL > 1) {
        __syncwarp();
        cluster_sync_threads();
    }
}

// --------------------------------------------------------- candidate lists
#ifndef DSRT_PIECE_BYTES
#define DSRT_PIECE_BYTES 3072
#endif
#ifndef DSRT_CAND_BUFS
#define DSRT_CAND_BUFS 3
#endif
constexpr int kPieceBytes = DSRT_PIECE_BYTES;  // per-warp staging piece
constexpr int kBufs = DSRT_CAND_BUFS;          // per-warp ring depth
#ifndef DSRT_CAND_WARPS
#define DSRT_CAND_WARPS 8
#endif
constexpr int kCandWarps = DSRT_CAND_WARPS;       // warps per candidate-mode CTA (16 warps per SM)

// Candidate-mode pieces: 4 KB when one query vector per lane (the smallest slot
// rows) still fits 2 CTAs per SM -- fewer, larger pieces cut the per-piece ring
// bookkeeping (cfg3 scoring 1.595 -> 1.567 ms); 3 KB otherwise.
template <int QPL>
constexpr int cand_piece_bytes() {
    return QPL == 1 ? (kPieceBytes > 4096 ? kPieceBytes : 4096) : kPieceBytes;
}
template <int K, int W, int PB = kPieceBytes>
constexpr int piece_vec() {
    return PB / ((((K * W) + 3) & ~3) * 4);
}
template <int QPL>
constexpr size_t cand_smem_static() {
    return kCandWarps * (kBufs * cand_piece_bytes<QPL>() + kBufs * sizeof(uint64_t) + SlotGeom<QPL>::kBytes);
}

// Candidate metadata through a lane window: lane l holds (vbeg, vend) of
// candidate base + l (vend = -1 for an invalid set index), loaded in one batch
// per 32 candidates instead of a dependent load chain per candidate.
struct CandWin {
    int32_t base = -(1 << 30), len = 0;  // base: candidate index of lane 0
    int64_t vb = 0;
    __device__ __forceinline__ void load(int64_t b, int64_t e_hi, const int64_t *cand_row,
                                         const int64_t *set_off, int64_t n_sets) {
        base = static_cast<int32_t>(b);
        const int64_t e = b + (threadIdx.x & 31);
        int64_t sidx = -1;
        if (e < e_hi) sidx = cand_row ? __ldg(cand_row + e) : e;
        const bool ok = sidx >= 0 && sidx < n_sets;
        vb = ok ? __ldg(set_off + sidx) : 0;
        len = ok ? static_cast<int32_t>(__ldg(set_off + sidx + 1) - vb) : -1;
    }
    // (vbeg, vend) of candidate e; vend = -1 marks an invalid set index
    __device__ __forceinline__ void get(int64_t e, int64_t e_hi, const int64_t *cand_row,
                                        const int64_t *set_off, int64_t n_sets, int64_t &ovb,
                                        int64_t &ove) {
        if (e - base >= 32) load(e, e_hi, cand_row, set_off, n_sets);
        const int l = static_cast<int>(e - base);
        ovb = __shfl_sync(0xffffffffu, vb, l);
        const int32_t n = __shfl_sync(0xffffffffu, len, l);
        ove = n < 0 ? -1 : ovb + n;
    }
};

// Piece window of the candidate kernel: lane l holds, for candidate base + l of the
// run, the byte address of its records and the metadata word of its (single) piece --
// nvec | kPieceDone | kPieceValid -- or kPieceMulti when the set is longer than one piece
// (then len is used).  One batch of loads per 32 candidates; issuing a piece is three
// shuffles and the bulk copy.
constexpr uint32_t kPieceDone = 1u << 16, kPieceValid = 1u << 17, kPieceMulti = 0xffffffffu;
static_assert(kPieceValid == 1u << 17, "the slot valid bit is taken from bit 17 of the piece word");
struct PieceWin {
    int32_t base = -(1 << 30), len = 0;  // base: run-relative candidate index of lane 0
    uint32_t meta = 0;
    const uint32_t *src = nullptr;
    template <int PV, int R>
    __device__ __forceinline__ void load(int32_t k, int64_t e_lo, int64_t e_hi, const int64_t *cand_row,
                                         const int64_t *set_off, int64_t n_sets,
                                         const uint32_t *recs) {
        base = k;
        const int64_t e = e_lo + k + (threadIdx.x & 31);
        int64_t sidx = -1;
        if (e < e_hi) sidx = cand_row ? __ldg(cand_row + e) : e;
        const bool ok = sidx >= 0 && sidx < n_sets;
        const int64_t vb = ok ? __ldg(set_off + sidx) : 0;
        len = ok ? static_cast<int32_t>(__ldg(set_off + sidx + 1) - vb) : 0;
        src = recs + vb * R;
        meta = len > PV ? kPieceMulti
                        : (static_cast<uint32_t>(len) | kPieceDone | (ok ? kPieceValid : 0u));
    }
};

// One warp = (query set, run of candidate slots).  Each warp streams its
// candidates' records through a private kBufs-deep ring filled by
// cp.async.bulk issued from lane 0.
#ifndef DSRT_CAND_MINB
#define DSRT_CAND_MINB (16 / DSRT_CAND_WARPS)
#endif
#ifndef DSRT_CAND_WAVES
#define DSRT_CAND_WAVES 4  // candidate-mode grid: waves of warps (sets the run length)
#endif
template <int K, int W, int QPL, bool SPLIT = false>
__global__ void __launch_bounds__(kCandWarps * 32, DSRT_CAND_MINB)
    score_cand_kernel(const uint32_t *__restrict__ recs, const int64_t *__restrict__ set_off,
                      int64_t n_sets, const int64_t *__restrict__ cand,
                      const int32_t *__restrict__ n_cand, int64_t cand_ld,
                      const uint32_t *__restrict__ qrecs, int64_t n_qsets, int m_q, int L,
                      const double *__restrict__ lut, const double *__restrict__ weights,
                      double *__restrict__ scores,
                      uint16_t *__restrict__ maxcounts, int mc_stride, int mc_q0, int64_t run_len,
                      int64_t runs_per_q) {
    constexpr int R = ((K * W) + 3) & ~3;
    constexpr int PB = cand_piece_bytes<QPL>();
    constexpr int PV = piece_vec<K, W, PB>();
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t *bufs = reinterpret_cast<uint32_t *>(smem) + warp * (kBufs * PB / 4);
    uint8_t *after_bufs = smem + kCandWarps * kBufs * PB;
    uint64_t *bars = reinterpret_cast<uint64_t *>(after_bufs) + warp * kBufs;
    uint8_t *slot_mem = after_bufs + kCandWarps * kBufs * sizeof(uint64_t);
    double *lut_s = reinterpret_cast<double *>(slot_mem + kCandWarps * SlotGeom<QPL>::kBytes);
    double *w_s = lut_s + (L + 1);  // m_q weights (1.0 when none)

    if (lane == 0) {
        for (int b = 0; b < kBufs; ++b) mbar_init(&bars[b], 1);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i <= L; i += blockDim.x) lut_s[i] = __ldg(lut + i);
    for (int i = threadIdx.x; i < m_q; i += blockDim.x) w_s[i] = weights ? __ldg(weights + i) : 1.0;
    __syncthreads();

    const int64_t gw = static_cast<int64_t>(blockIdx.x) * kCandWarps + warp;
    const int64_t qset = gw / runs_per_q;
    if (qset >= n_qsets) return;
    const int64_t nc = n_cand ? tmin<int64_t>(__ldg(n_cand + qset), cand_ld) : cand_ld;
    const int64_t e_lo = (gw % runs_per_q) * run_len;
    const int64_t e_hi = tmin(e_lo + run_len, nc);
    if (e_lo >= e_hi) return;

    static_assert(!SPLIT || QPL == 1, "split-lane mapping covers m_q <= 32");
    constexpr int QR = SPLIT ? 2 : QPL;  // query vectors held per lane
    uint32_t q[QR][K * W];
    if constexpr (SPLIT) load_queries_split<K, W>(q, qrecs, qset, m_q);
    else load_queries<K, W, QPL>(q, qrecs, qset, m_q, true);
    int rmin[QR];
#pragma unroll
    for (int s = 0; s < QR; ++s) rmin[s] = L;
    Slots<QPL> slots{slot_mem + warp * SlotGeom<QPL>::kBytes};
    double *out_row = scores != nullptr ? scores + qset * cand_ld : nullptr;

    // candidate metadata through a lane window (PieceWin): one batch of loads per 32
    // candidates instead of a dependent load chain per set.
    const int64_t *cand_row = cand ? cand + qset * cand_ld : nullptr;
    PieceWin pwin;
    // producer iterator (lane-uniform state; lane 0 issues the copies): pk = candidates of
    // the run already issued; a set longer than one piece is continued from (mp_src, mp_rem)
    const int nrun = static_cast<int>(e_hi - e_lo);
    int pk = 0, mp_rem = 0;
    const uint32_t *mp_src = nullptr;
    constexpr uint32_t kDone = kPieceDone, kValid = kPieceValid;
    // The buffer being refilled was last read by this warp's LDS, complete before
    // the __syncwarp that precedes every refill, so no proxy fence is needed for
    // the bulk copy's write-after-read.
    // The ring is refilled in consumption order, so the buffer to fill is always the one
    // just consumed (b), and kBufs pieces are outstanding whenever the loop is left.
    auto issue = [&](int b) -> uint32_t {  // next piece into buffer b; returns its metadata
        uint32_t meta = 0;
        const uint32_t *src = nullptr;
        if (mp_rem > 0) {  // continue a multi-piece set (rare: longer than PV vectors)
            const int nvec = min(PV, mp_rem);
            src = mp_src;
            mp_src += static_cast<int64_t>(nvec) * R;
            mp_rem -= nvec;
            meta = static_cast<uint32_t>(nvec);
            if (mp_rem == 0) {
                meta |= kDone | kValid;
                ++pk;
            }
        } else if (pk < nrun) {
            int l = pk - pwin.base;
            if (l >= 32) {
                pwin.load<PV, R>(pk, e_lo, e_hi, cand_row, set_off, n_sets, recs);
                l = 0;
            }
            meta = __shfl_sync(kFull, pwin.meta, l);
            src = reinterpret_cast<const uint32_t *>(
                __shfl_sync(kFull, reinterpret_cast<unsigned long long>(pwin.src), l));
            if (meta == kPieceMulti) {
                mp_rem = __shfl_sync(kFull, pwin.len, l) - PV;
                mp_src = src + static_cast<int64_t>(PV) * R;
                meta = static_cast<uint32_t>(PV);
            } else {
                ++pk;
            }
        }
        if (lane == 0) {
            const uint32_t bytes = (meta & 0xffffu) * static_cast<uint32_t>(R * 4);
            if (bytes > 0) {
                mbar_arrive_expect_tx(&bars[b], bytes);
                bulk_g2s(bufs + b * (PV * R), src, bytes, &bars[b]);
            } else {
                mbar_arrive(&bars[b]);
            }
        }
        return meta;
    };
    // Consumer: replays the producer's piece sequence from metadata the
    // producer recorded at issue time (meta[0] = the oldest outstanding
    // piece: nvec | kDone | kValid), so the per-piece bookkeeping is a
    // register rotation instead of a second walk over the candidate list.
    int ck = 0;  // consumed candidates of the run
    int64_t slot_col = e_lo;
    uint32_t meta[kBufs];
#pragma unroll
    for (int i = 0; i < kBufs; ++i) meta[i] = issue(i);
    int b = 0;
    uint32_t phase = 0;
    // split-lane slot stores: per-lane predicates and a running row pointer, set up once
    const bool st0 = SPLIT && lane < 16 && lane < m_q, st1 = SPLIT && lane < 16 && lane + 16 < m_q;
    uint8_t *wr = slots.buf + lane;
    while (ck < nrun) {
        mbar_wait(&bars[b], phase);
        const uint32_t m0 = meta[0];
        const int nvec = static_cast<int>(m0 & 0xffffu);
        if (nvec > 0) {
            if constexpr (SPLIT) scan_split<K, W>(q, rmin, bufs + b * (PV * R), nvec);
            else scan_vectors<K, W, QPL, 4>(q, rmin, bufs + b * (PV * R), nvec);
        }
        if (m0 & kDone) {  // candidate complete
            if constexpr (SPLIT) {
#pragma unroll
                for (int i = 0; i < 2; ++i) rmin[i] = min(rmin[i], __shfl_xor_sync(kFull, rmin[i], 16));
                // Slots::push_split with the address and predicate arithmetic hoisted
                if (st0) wr[0] = static_cast<uint8_t>(L - rmin[0]);
                if (st1) wr[16] = static_cast<uint8_t>(L - rmin[1]);
                wr += SlotGeom<QPL>::kRow;
                slots.valid |= ((m0 >> 17) & 1u) << slots.n;  // kValid
                ++slots.n;
            } else {
                slots.push(rmin, L, m_q, (m0 & kValid) != 0);
            }
#pragma unroll
            for (int i = 0; i < QR; ++i) rmin[i] = L;
            if (slots.n == 32) {
                slots.flush(m_q, lut_s, w_s, out_row, slot_col, maxcounts, qset * cand_ld, mc_stride, mc_q0);
                slot_col += 32;
                wr = slots.buf + lane;
            }
            ++ck;
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i + 1 < kBufs; ++i) meta[i] = meta[i + 1];
        meta[kBufs - 1] = issue(b);  // refill the buffer just consumed
        if (++b == kBufs) { b = 0; phase ^= 1u; }
    }
    if (slots.n > 0)
        slots.flush(m_q, lut_s, w_s, out_row, slot_col, maxcounts, qset * cand_ld, mc_stride, mc_q0);
    // drain: wait for outstanding pieces so no bulk copy outlives the CTA
    for (int i = 0; i < kBufs; ++i) {
        mbar_wait(&bars[b], phase);
        if (++b == kBufs) { b = 0; phase ^= 1u; }
    }
}

// ------------------------------------------------------------- dispatch
template <int K, int W, int QPL, int QS>
static int launch_all(const uint32_t *recs, const int64_t *set_off, int64_t sb, int64_t se,
                      const uint32_t *qrecs, int64_t n_qsets, int m_q, int L, const double *lut,
                      const double *weights, double *scores, int64_t ld, uint16_t *mc,
                      int mc_stride, int mc_q0, const AppendOut &app, cudaStream_t st) {
#ifndef DSRT_ALL_NW
#define DSRT_ALL_NW 8
#endif
    constexpr int NW = DSRT_ALL_NW;  // consumer warps per CTA (+1 producer warp)
    const size_t smem = all_smem_static<K, W, QPL, NW, QS>() + (L + 1 + m_q) * sizeof(double);
    // query-set groups in cluster pairs sharing each record tile: opt-in (DSRT_ALL_CLUSTER=1).
    // Measured at cfg4 shape (1M sets x 1024 query sets): L2 -> SM bytes 88 -> 59 GB, DRAM
    // reads unchanged (2.88 -> 2.84 GB), kernel 1.176 -> 1.193 s -- the pairing costs more
    // than it saves in this INT-bound kernel, so it is off by default.
    const char *ce = getenv("DSRT_ALL_CLUSTER");
    const bool pair = (ce && ce[0] == '1') && n_qsets > NW * QS;
    auto kern = pair ? score_all_kernel<K, W, QPL, NW, QS, 2> : score_all_kernel<K, W, QPL, NW, QS, 1>;
    DSRT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int64_t groups = (n_qsets + NW * QS - 1) / (NW * QS);
    if (pair) groups += groups & 1;  // whole pairs (an extra CTA with no query sets still streams)
    int occ = 0;
    DSRT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, (NW + 1) * 32, smem));
    occ = occ < 1 ? 1 : occ;
    const int64_t nset = se - sb;
    // ~8 waves of CTAs; each chunk keeps >= 64 sets so tile pipelines stay full
#ifndef DSRT_ALL_WAVES
#define DSRT_ALL_WAVES 64  // measured at cfg4 shape: 8 -> 64 waves: 0.843 -> 0.852 of INT, DRAM 1.28x -> 1.13x (smaller chunks keep the 32 groups of a chunk within L2)
#endif
    int64_t waves = DSRT_ALL_WAVES;
    if (const char *e = getenv("DSRT_ALL_WAVES")) waves = tmax(1, atoi(e));  // tuning knob
    int64_t chunks = (waves * sm_count() * occ + groups - 1) / groups;
    chunks = tmax<int64_t>(1, tmin<int64_t>(chunks, (nset + 63) / 64));
    chunks = tmin<int64_t>(chunks, 65535);
    // the consumers index a chunk's sets and vectors with 32-bit relative offsets: chunks are cut
    // by equal vector counts and a set has <= 65535 vectors, so <= 32767 sets per chunk on
    // average keeps every chunk below 2^31 vectors (and sets)
    chunks = tmax<int64_t>(chunks, (nset + 32766) / 32767);
    DSRT_REQUIRE(chunks <= 65535, DSRT_EUNSUPPORTED, "invalid parameter: too many sets for one scoring launch");
    dim3 grid(static_cast<unsigned>(groups), static_cast<unsigned>(chunks));
    DSRT_REQUIRE(groups < (1LL << 31), DSRT_EUNSUPPORTED, "invalid parameter: too many query sets");
    if (pair) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3((NW + 1) * 32);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        DSRT_CUDA(cudaLaunchKernelEx(&cfg, kern, recs, set_off, sb, se, qrecs, n_qsets, m_q, L, lut, weights,
                                     scores, ld, mc, mc_stride, mc_q0, static_cast<int>(chunks), app));
    } else {
        kern<<<grid, (NW + 1) * 32, smem, st>>>(recs, set_off, sb, se, qrecs, n_qsets, m_q, L, lut,
                                               weights, scores, ld, mc, mc_stride, mc_q0,
                                               static_cast<int>(chunks), app);
    }
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}

template <int K, int W, int QPL, bool SPLIT = false>
static int launch_cand(const uint32_t *recs, const int64_t *set_off, int64_t n_sets,
                       const int64_t *cand, const int32_t *n_cand, int64_t cand_ld,
                       const uint32_t *qrecs, int64_t n_qsets, int m_q, int L, const double *lut,
                       const double *weights, double *scores, uint16_t *mc, int mc_stride,
                       int mc_q0, cudaStream_t st) {
    const size_t smem = cand_smem_static<QPL>() + (L + 1 + m_q) * sizeof(double);
    auto kern = score_cand_kernel<K, W, QPL, SPLIT>;
    DSRT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    DSRT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kCandWarps * 32, smem));
    occ = occ < 1 ? 1 : occ;
    // enough warps for ~4 waves, but runs of >= 4 candidates
    const int64_t want_warps = static_cast<int64_t>(DSRT_CAND_WAVES) * sm_count() * occ * kCandWarps;
    int64_t runs = (want_warps + n_qsets - 1) / n_qsets;
    runs = tmax<int64_t>(1, tmin<int64_t>(runs, (cand_ld + 3) / 4));
    const int64_t run_len = (cand_ld + runs - 1) / runs;
    runs = (cand_ld + run_len - 1) / run_len;
    const int64_t warps = n_qsets * runs;
    const int64_t blocks = (warps + kCandWarps - 1) / kCandWarps;
    DSRT_REQUIRE(blocks < (1LL << 31), DSRT_EUNSUPPORTED, "invalid parameter: grid too large");
    kern<<<static_cast<unsigned>(blocks), kCandWarps * 32, smem, st>>>(
        recs, set_off, n_sets, cand, n_cand, cand_ld, qrecs, n_qsets, m_q, L, lut, weights, scores,
        mc, mc_stride, mc_q0, run_len, runs);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}

// Dispatch on (C, W, QPL) template instances.
struct ScoreArgs {
    bool cand_mode;
    const uint32_t *recs;
    const int64_t *set_off;
    int64_t sb, se, n_sets;
    const int64_t *cand;
    const int32_t *n_cand;
    int64_t cand_ld;
    const uint32_t *qrecs;
    int64_t n_qsets;
    int m_q, L;
    const double *lut;
    const double *weights;  // (m_q) or nullptr = all ones
    double *scores;
    int64_t ld;
    uint16_t *mc;
    int mc_stride, mc_q0;
    int qs_override;  // 0 = heuristic; else query sets per warp (1/2/4)
    AppendOut app;    // exhaustive threshold-append epilogue (app.tau == nullptr: off)
};

// K3 entry (score.cu): dispatch on (C, W, QPL, QS); m_q > 128 via slices + finalize.
int score_dispatch(ScoreArgs a, int C, cudaStream_t st);

template <int K, int W, int QPL>
static int run_one(const ScoreArgs &a, cudaStream_t st) {
    if (a.cand_mode) {
        if constexpr (QPL == 1 && W <= 2 && K <= 8) {
            if (a.m_q > 16 && a.qs_override != -1)  // split-lane mapping (-1 forces the plain one)
                return launch_cand<K, W, QPL, true>(a.recs, a.set_off, a.n_sets, a.cand, a.n_cand,
                                                    a.cand_ld, a.qrecs, a.n_qsets, a.m_q, a.L, a.lut,
                                                    a.weights, a.scores, a.mc, a.mc_stride, a.mc_q0, st);
        }
        return launch_cand<K, W, QPL>(a.recs, a.set_off, a.n_sets, a.cand, a.n_cand, a.cand_ld,
                                      a.qrecs, a.n_qsets, a.m_q, a.L, a.lut, a.weights, a.scores, a.mc,
                                      a.mc_stride, a.mc_q0, st);
    }
    // register-block several query sets per warp when there are enough of them
    if constexpr (QPL == 1 && W <= 2 && K <= 8) {
        const int qs = a.qs_override > 0 ? a.qs_override : (a.n_qsets >= 256 ? (W == 1 ? 4 : 2) : 1);
        if (qs == 4)
            return launch_all<K, W, QPL, 4>(a.recs, a.set_off, a.sb, a.se, a.qrecs, a.n_qsets, a.m_q,
                                            a.L, a.lut, a.weights, a.scores, a.ld, a.mc, a.mc_stride, a.mc_q0,
                                            a.app, st);
        if (qs == 2)
            return launch_all<K, W, QPL, 2>(a.recs, a.set_off, a.sb, a.se, a.qrecs, a.n_qsets, a.m_q,
                                            a.L, a.lut, a.weights, a.scores, a.ld, a.mc, a.mc_stride, a.mc_q0,
                                            a.app, st);
    }
    return launch_all<K, W, QPL, 1>(a.recs, a.set_off, a.sb, a.se, a.qrecs, a.n_qsets, a.m_q, a.L,
                                    a.lut, a.weights, a.scores, a.ld, a.mc, a.mc_stride, a.mc_q0, a.app, st);
}

template <int K, int W>
static int run_qpl(const ScoreArgs &a, int qpl, cudaStream_t st) {
    switch (qpl) {
        case 1: return run_one<K, W, 1>(a, st);
        case 2: return run_one<K, W, 2>(a, st);
        default: return run_one<K, W, 4>(a, st);
    }
}

template <int K>
int run_w(const ScoreArgs &a, int W, int qpl, cudaStream_t st) {
    switch (W) {
        case 1: return run_qpl<K, 1>(a, qpl, st);
        case 2: return run_qpl<K, 2>(a, qpl, st);
        case 3: return run_qpl<K, 3>(a, qpl, st);
        case 4: return run_qpl<K, 4>(a, qpl, st);
        default: break;
    }
    set_error("invalid parameter: L=%d unsupported by the scoring kernel (L <= 128)", a.L);
    return DSRT_EUNSUPPORTED;
}

}  // namespace dsrt
