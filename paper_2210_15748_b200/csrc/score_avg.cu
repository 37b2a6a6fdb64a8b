// K3a -- avg-phi scoring on the K3 pipeline.
//
// Same mapping as score_cand_kernel (warp = (query set, run of targets), lane
// = query vector, per-warp cp.async.bulk ring of plane records, broadcast
// LDS.128), with the running min of mismatches replaced by a streaming form
// of the reference's avg-phi inner aggregation (index.py:207-214):
//
//   per_query[q] = reduceat-sum(table[c_qj] : c_qj > 0, j ascending) / m
//
// numpy's reduceat seeds the segment with its first element and adds
// pairwise_sum(rest).  For n = |rest| <= 128 pairwise_sum is one leaf -- 8
// strided accumulators over the first n - n%8 values, combined
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n%8 remaining values in order
// (n < 8: plain sequence from 0.0) -- which streams: completed groups of 8
// go into r[0..7], the <= 7 pending counts wait as bytes in two registers.
// n > 128 (a set with > 129 colliding vectors for one query) needs the
// recursive split; such (query set, target) items are appended to an
// overflow list and recomputed by the general kernel (score_agg.cu).
//
// The per-query values (times the weights) are parked in a per-warp shared
// row per target; every 32 targets lane i sums row i in numpy order
// (np.mean: 0.0 + pairwise, / m_q).
#include "score_kernels.cuh"

namespace dsrt {

constexpr int kAvgRow = 33;  // doubles per slot row (32 + 1 skew)

// Per-lane streaming state.  Counts enter a 16-entry per-lane ring in shared
// memory unconditionally (the slot is reused when c == 0), and maintain()
// -- called at warp-uniform points at least every 8 adds -- takes the first
// element and folds complete groups of 8 into r[].  The divergent work thus
// runs once per 8 vectors instead of whenever some lane fills a group.
struct AvgStream {
    double first, r[8];
    uint8_t *ring;  // this lane's ring: element k at ring[(k & 15) * 32]
    int h, np, ng;  // ring head, pending count, folded groups
    bool hf;        // first element taken

    __device__ __forceinline__ void reset() {
        h = np = ng = 0;
        hf = false;
        first = 0.0;
    }
    __device__ __forceinline__ void add(int c) {
        ring[((h + np) & 15) * 32] = static_cast<uint8_t>(c);
        np += c > 0 ? 1 : 0;
    }
    __device__ __forceinline__ double at(int k, const double *__restrict__ tab) const {
        return tab[ring[((h + k) & 15) * 32]];
    }
    __device__ __forceinline__ void maintain(const double *__restrict__ tab) {
        if (!hf && np > 0) {
            first = at(0, tab);
            h = (h + 1) & 15;
            --np;
            hf = true;
        }
        if (np >= 8) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const double v = at(k, tab);
                r[k] = ng == 0 ? v : __dadd_rn(r[k], v);
            }
            h = (h + 8) & 15;
            np -= 8;
            ++ng;
        }
    }
    // per_query value after the last add; overflow (|rest| > 128) -> ovf = true
    __device__ __forceinline__ double finish(int64_t m, const double *__restrict__ tab, bool &ovf) {
        maintain(tab);
        if (!hf) return 0.0;
        if (8 * ng + np > 128) {
            ovf = true;
            return 0.0;
        }
        double res = 0.0;
        if (ng > 0)
            res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                            __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (int k = 0; k < np; ++k) res = __dadd_rn(res, at(k, tab));
        return __ddiv_rn(__dadd_rn(first, res), static_cast<double>(m));
    }
};

// numpy pairwise mean of a shared row of n <= 32 doubles
__device__ __forceinline__ double row_mean(const double *row, int n) {
    double res;
    if (n < 8) {
        res = 0.0;
        for (int i = 0; i < n; ++i) res = __dadd_rn(res, row[i]);
    } else {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = row[j];
        const int n8 = n - (n & 7);
        for (int i = 8; i < n8; i += 8)
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], row[i + j]);
        res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                        __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (int i = n8; i < n; ++i) res = __dadd_rn(res, row[i]);
    }
    return __ddiv_rn(__dadd_rn(0.0, res), static_cast<double>(n));
}

struct AvgArgs {
    const uint32_t *recs;
    const int64_t *set_off;
    int64_t n_sets;
    const int64_t *cand;
    const int32_t *n_cand;
    int64_t cand_ld;
    const uint32_t *qrecs;
    int64_t n_qsets;
    int m_q, L;
    const double *table;
    const double *weights;
    double *scores;
    int64_t *ovf_items;   // (qset * cand_ld + e) of overflowed targets
    unsigned long long *ovf_count;
    int64_t ovf_cap;
};

constexpr size_t avg_smem_static() {
    return kCandWarps * (kBufs * kPieceBytes + kBufs * sizeof(uint64_t) +
                         32 * kAvgRow * sizeof(double) + 16 * 32);
}

template <int K, int W>
__global__ void __launch_bounds__(kCandWarps * 32, 16 / kCandWarps)
    score_avg_kernel(const AvgArgs a, int64_t run_len, int64_t runs_per_q) {
    constexpr int R = ((K * W) + 3) & ~3;
    constexpr int PV = piece_vec<K, W>();
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t *bufs = reinterpret_cast<uint32_t *>(smem) + warp * (kBufs * PV * R);
    uint8_t *after_bufs = smem + kCandWarps * kBufs * kPieceBytes;
    uint64_t *bars = reinterpret_cast<uint64_t *>(after_bufs) + warp * kBufs;
    double *rows_all = reinterpret_cast<double *>(after_bufs + kCandWarps * kBufs * sizeof(uint64_t));
    double *rows = rows_all + warp * 32 * kAvgRow;
    uint8_t *rings = reinterpret_cast<uint8_t *>(rows_all + kCandWarps * 32 * kAvgRow);
    double *tab_s = reinterpret_cast<double *>(rings + kCandWarps * 16 * 32);
    double *w_s = a.weights != nullptr ? tab_s + (a.L + 1) : nullptr;

    if (lane == 0) {
        for (int b = 0; b < kBufs; ++b) mbar_init(&bars[b], 1);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i <= a.L; i += blockDim.x) tab_s[i] = __ldg(a.table + i);
    if (w_s != nullptr)
        for (int i = threadIdx.x; i < a.m_q; i += blockDim.x) w_s[i] = __ldg(a.weights + i);
    __syncthreads();

    const int64_t gw = static_cast<int64_t>(blockIdx.x) * kCandWarps + warp;
    const int64_t qset = gw / runs_per_q;
    if (qset >= a.n_qsets) return;
    const int64_t cand_ld = a.cand_ld;
    const int64_t nc = a.n_cand ? tmin<int64_t>(__ldg(a.n_cand + qset), cand_ld) : cand_ld;
    const int64_t e_lo = (gw % runs_per_q) * run_len;
    const int64_t e_hi = tmin(e_lo + run_len, nc);
    if (e_lo >= e_hi) return;

    uint32_t q[1][K * W];
    load_queries<K, W, 1>(q, a.qrecs, qset, a.m_q, true);
    const bool act = lane < a.m_q;
    AvgStream acc;
    acc.ring = rings + warp * (16 * 32) + lane;
    acc.reset();
    double *out_row = a.scores + qset * cand_ld;
    const int64_t *cand_row = a.cand ? a.cand + qset * cand_ld : nullptr;
    const double nan = __longlong_as_double(0x7ff8000000000000ll);

    CandWin pwin, cwin;
    int64_t pe = e_lo, pv, pvend;
    pwin.get(pe, e_hi, cand_row, a.set_off, a.n_sets, pv, pvend);
    if (pvend < 0) { pv = 0; pvend = 0; }
    int64_t issued = 0;
    auto issue = [&]() {
        const int b = static_cast<int>(issued % kBufs);
        const int64_t nvec = pe < e_hi ? tmin<int64_t>(PV, pvend - pv) : 0;
        if (lane == 0) {
            const uint32_t bytes = static_cast<uint32_t>(nvec * R * 4);
            fence_proxy_async_smem();
            if (bytes > 0) {
                mbar_arrive_expect_tx(&bars[b], bytes);
                bulk_g2s(bufs + b * (PV * R), a.recs + pv * R, bytes, &bars[b]);
            } else {
                mbar_arrive(&bars[b]);
            }
        }
        ++issued;
        pv += nvec;
        if (pe < e_hi && pv >= pvend) {
            ++pe;
            if (pe < e_hi) {
                pwin.get(pe, e_hi, cand_row, a.set_off, a.n_sets, pv, pvend);
                if (pvend < 0) { pv = 0; pvend = 0; }
            }
        }
    };
    int64_t ce = e_lo, cv, cvend, slot_col = e_lo;
    cwin.get(ce, e_hi, cand_row, a.set_off, a.n_sets, cv, cvend);
    bool cvalid = cvend >= 0;
    if (!cvalid) { cv = 0; cvend = 0; }
    int64_t m = cvend - cv;
    int n_slots = 0;
    uint32_t bad = 0;  // bit i: slot i is invalid or overflowed (NaN / recomputed)
    auto flush = [&]() {
        __syncwarp();
        if (lane < n_slots)
            out_row[slot_col + lane] = ((bad >> lane) & 1u) ? nan : row_mean(rows + lane * kAvgRow, a.m_q);
        __syncwarp();
        slot_col += n_slots;
        n_slots = 0;
        bad = 0;
    };
    int64_t consumed = 0;
    for (int i = 0; i < kBufs; ++i) issue();
    while (ce < e_hi) {
        const int b = static_cast<int>(consumed % kBufs);
        mbar_wait(&bars[b], static_cast<uint32_t>(consumed / kBufs) & 1);
        const int64_t nvec = tmin<int64_t>(PV, cvend - cv);
        const uint4 *x4 = reinterpret_cast<const uint4 *>(bufs + b * (PV * R));
        const int nv = static_cast<int>(nvec);
        int i = 0;
        for (; i + 8 <= nv; i += 8) {  // blocks of 8 adds, then one maintain
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                uint4 xv[R / 4];
#pragma unroll
                for (int u = 0; u < R / 4; ++u) xv[u] = x4[(i + k) * (R / 4) + u];
                acc.add(a.L - mismatches<K, W>(q[0], reinterpret_cast<const uint32_t *>(xv)));
            }
            acc.maintain(tab_s);
        }
        for (; i < nv; ++i) {
            uint4 xv[R / 4];
#pragma unroll
            for (int u = 0; u < R / 4; ++u) xv[u] = x4[i * (R / 4) + u];
            acc.add(a.L - mismatches<K, W>(q[0], reinterpret_cast<const uint32_t *>(xv)));
        }
        acc.maintain(tab_s);
        ++consumed;
        cv += nvec;
        if (cv >= cvend) {  // target complete
            bool ovf = false;
            double v = acc.finish(m, tab_s, ovf);
            ovf = __any_sync(0xffffffffu, ovf && act) != 0;
            if (act) rows[n_slots * kAvgRow + lane] = w_s != nullptr ? __dmul_rn(w_s[lane], v) : v;
            if (ovf && cvalid && lane == 0) {
                const unsigned long long k = atomicAdd(a.ovf_count, 1ull);
                if (static_cast<int64_t>(k) < a.ovf_cap) a.ovf_items[k] = qset * cand_ld + ce;
            }
            bad |= ((ovf || !cvalid) ? 1u : 0u) << n_slots;
            ++n_slots;
            acc.reset();
            if (n_slots == 32) flush();
            ++ce;
            if (ce < e_hi) {
                cwin.get(ce, e_hi, cand_row, a.set_off, a.n_sets, cv, cvend);
                cvalid = cvend >= 0;
                if (!cvalid) { cv = 0; cvend = 0; }
                m = cvend - cv;
            }
        }
        __syncwarp();
        issue();
    }
    if (n_slots > 0) flush();
    while (consumed < issued) {
        const int b = static_cast<int>(consumed % kBufs);
        mbar_wait(&bars[b], static_cast<uint32_t>(consumed / kBufs) & 1);
        ++consumed;
    }
}

template <int K, int W>
static int launch_avg(const AvgArgs &a, cudaStream_t st) {
    const size_t smem = avg_smem_static() + (a.L + 1) * sizeof(double) +
                        (a.weights != nullptr ? a.m_q * sizeof(double) : 0);
    auto kern = score_avg_kernel<K, W>;
    DSRT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    DSRT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kCandWarps * 32, smem));
    occ = occ < 1 ? 1 : occ;
    const int64_t want_warps = 4LL * sm_count() * occ * kCandWarps;
    int64_t runs = (want_warps + a.n_qsets - 1) / a.n_qsets;
    runs = tmax<int64_t>(1, tmin<int64_t>(runs, (a.cand_ld + 3) / 4));
    const int64_t run_len = (a.cand_ld + runs - 1) / runs;
    runs = (a.cand_ld + run_len - 1) / run_len;
    const int64_t blocks = (a.n_qsets * runs + kCandWarps - 1) / kCandWarps;
    DSRT_REQUIRE(blocks < (1LL << 31), DSRT_EUNSUPPORTED, "invalid parameter: grid too large");
    kern<<<static_cast<unsigned>(blocks), kCandWarps * 32, smem, st>>>(a, run_len, runs);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}

bool score_avg_supported(int L, int C, int m_q) {
    return m_q >= 1 && m_q <= 32 && C >= 1 && C <= 8 && L >= 1 && L <= 64;
}

int score_avg_fast(const uint32_t *records, const int64_t *set_off, int64_t n_sets,
                   const int64_t *cand, const int32_t *n_cand, int64_t cand_ld,
                   const uint32_t *qrecs, int64_t n_qsets, int m_q, int L, int C,
                   const double *table, const double *weights, double *scores,
                   int64_t *ovf_items, unsigned long long *ovf_count, int64_t ovf_cap,
                   cudaStream_t st) {
    AvgArgs a{records, set_off, n_sets, cand, n_cand, cand_ld, qrecs, n_qsets, m_q, L,
              table, weights, scores, ovf_items, ovf_count, ovf_cap};
    const int W = plane_words(L);
    switch (C * 4 + W) {
#define DSRT_AVG(k)                                              \
    case k * 4 + 1: return launch_avg<k, 1>(a, st);              \
    case k * 4 + 2: return launch_avg<k, 2>(a, st);
        DSRT_AVG(1) DSRT_AVG(2) DSRT_AVG(3) DSRT_AVG(4)
        DSRT_AVG(5) DSRT_AVG(6) DSRT_AVG(7) DSRT_AVG(8)
#undef DSRT_AVG
        default: break;
    }
    set_error("invalid parameter: avg-phi fast kernel does not cover L=%d C=%d", L, C);
    return DSRT_EUNSUPPORTED;
}

}  // namespace dsrt
