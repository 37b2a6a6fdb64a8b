// K3g -- general inner/outer aggregation: sigma = max
// or avg-phi, optional per-query-vector weights.  Follows _score_one
// (index.py:183-216) with _sim_table_for (index.py:170-180):
//
//   max:     per_query[q] = table[max_j c_qj]
//   avg-phi: per_query[q] = add.reduceat(table[c_qj] for c_qj > 0, j ascending) / m
//            (numpy reduceat segment = first element + pairwise(rest))
//   score  = mean(w * per_query) = (0.0 + pairwise(w_q * per_query[q])) / m_q
//
// with table = lut (max) or phi(lut) (avg-phi), host-computed bytes.  The
// sigma = max, unit-weight north-star path stays on the register-blocked
// kernels in score_kernels.cuh; this kernel is the general path.
//
// Work item = (query set, target).  One warp per item, persistent grid; lane
// = query vector (32-wide slices of m_q).  Target records are warp-uniform
// (broadcast loads); the avg-phi counts c_qj > 0 are compacted per lane into
// warp scratch [k][lane] (uint16, c <= L) and summed in the reference's order
// afterwards.  Any L (runtime plane-word loop above 128 tables) and C <= 24:
// this kernel is also the sigma = max path for shapes outside the K3 kernels'
// register envelope (C > 16 or C * ceil(L/32) > 32), see score_general in score.cu.
#include "common.cuh"

namespace dsrt {

int score_max_fast(const uint32_t *records, const int64_t *set_off, int64_t n_sets,
                   const int64_t *cand, const int32_t *n_cand, int64_t cand_ld,
                   const uint32_t *qrecs, int64_t n_qsets, int m_q, int L, int C,
                   const double *lut, const double *weights, double *scores, cudaStream_t st);
bool score_max_fast_supported(int L, int C);
bool score_avg_supported(int L, int C, int m_q);
int score_avg_fast(const uint32_t *records, const int64_t *set_off, int64_t n_sets,
                   const int64_t *cand, const int32_t *n_cand, int64_t cand_ld,
                   const uint32_t *qrecs, int64_t n_qsets, int m_q, int L, int C,
                   const double *table, const double *weights, double *scores,
                   int64_t *ovf_items, unsigned long long *ovf_count, int64_t ovf_cap,
                   cudaStream_t st);
constexpr int64_t kOvfCap = 1 << 20;  // overflow items recomputed from a list

constexpr int kAggWarps = 8;
constexpr int kAggMaxC = 24;

// numpy pairwise_sum_DOUBLE over v(start..start+n) where v(k) = table[s[k * 32]]
__device__ double pw_counts(const uint16_t *s, int n, const double *__restrict__ table) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r = __dadd_rn(r, __ldg(table + s[i * 32]));
        return r;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __ldg(table + s[j * 32]);
        int i;
        for (i = 8; i < n - (n % 8); i += 8)
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], __ldg(table + s[(i + j) * 32]));
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; ++i) res = __dadd_rn(res, __ldg(table + s[i * 32]));
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(pw_counts(s, n2, table), pw_counts(s + n2 * 32, n - n2, table));
}

// numpy pairwise_sum_DOUBLE over a contiguous double array
__device__ double pw_doubles(const double *a, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
        return r;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int i;
        for (i = 8; i < n - (n % 8); i += 8)
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; ++i) res = __dadd_rn(res, a[i]);
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(pw_doubles(a, n2), pw_doubles(a + n2, n - n2));
}

struct AggArgs {
    const uint32_t *records;
    const int64_t *set_off;
    int64_t n_sets;
    const int64_t *cand;    // NULL: identity
    const int32_t *n_cand;  // NULL: all cand_ld
    int64_t cand_ld;
    const uint32_t *qrecs;
    int64_t n_qsets;
    int m_q, L, C, R;
    int kind;               // 0 max, 1 avg-phi
    const double *table;    // (L+1)
    const double *weights;  // (m_q) or NULL
    double *scores;         // (n_qsets, cand_ld)
    uint8_t *scratch;       // per warp: 32 * m_cap uint16 counts, then m_q doubles
    int64_t m_cap;
    size_t warp_bytes;
    uint32_t *status;       // bit 0: target set larger than m_cap
    const int64_t *items;   // list mode: item indices (qset * cand_ld + e); NULL = all
    int64_t n_items;
};

// WT = plane words per table bit held in registers (1..4); WT = 0: any W, query
// words re-read through L1 for every set vector (L > 128, the rare shapes).
template <int WT>
__global__ void __launch_bounds__(kAggWarps * 32)
    score_agg_kernel(const AggArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = blockIdx.x * static_cast<int64_t>(kAggWarps) + (threadIdx.x >> 5);
    const int64_t n_warps = static_cast<int64_t>(gridDim.x) * kAggWarps;
    uint16_t *cnt = reinterpret_cast<uint16_t *>(a.scratch + gw * a.warp_bytes);
    double *pq = reinterpret_cast<double *>(a.scratch + gw * a.warp_bytes + 64 * a.m_cap);
    const int W = WT > 0 ? WT : plane_words(a.L);
    const int64_t items = a.items ? a.n_items : a.n_qsets * a.cand_ld;
    const uint32_t tail = (a.L % 32) ? ((1u << (a.L % 32)) - 1u) : 0xffffffffu;
    for (int64_t ii = gw; ii < items; ii += n_warps) {
        const int64_t it = a.items ? a.items[ii] : ii;
        const int64_t qs = it / a.cand_ld, e = it - qs * a.cand_ld;
        double *out = a.scores + qs * a.cand_ld + e;
        if (a.n_cand != nullptr && e >= tmin<int64_t>(a.n_cand[qs], a.cand_ld)) continue;
        const int64_t s = a.cand ? a.cand[qs * a.cand_ld + e] : e;
        if (s < 0 || s >= a.n_sets) {  // invalid set index: NaN, as score_cand_kernel
            if (lane == 0) *out = __longlong_as_double(0x7ff8000000000000ll);
            continue;
        }
        const int64_t v0 = a.set_off[s], m = a.set_off[s + 1] - v0;
        if (a.kind == 1 && m > a.m_cap) {
            if (lane == 0) {
                atomicOr(a.status, 1u);
                *out = -1.0;
            }
            continue;
        }
        const uint32_t *xr = a.records + v0 * a.R;
        for (int q0 = 0; q0 < a.m_q; q0 += 32) {
            const int q = q0 + lane;
            const bool act = q < a.m_q;
            constexpr int WR = WT > 0 ? WT : 1;
            uint32_t qw[kAggMaxC][WR];
            const uint32_t *qr = a.qrecs + (qs * a.m_q + (act ? q : 0)) * static_cast<int64_t>(a.R);
            if constexpr (WT > 0) {
#pragma unroll
                for (int b = 0; b < kAggMaxC; ++b)
#pragma unroll
                    for (int w = 0; w < WT; ++w) qw[b][w] = (b < a.C) ? __ldg(qr + b * WT + w) : 0u;
            }
            int cmax = 0, nz = 0;
            for (int64_t j = 0; j < m; ++j) {
                const uint32_t *x = xr + j * a.R;
                int mm = 0;
                if constexpr (WT > 0) {
#pragma unroll
                    for (int w = 0; w < WT; ++w) {
                        uint32_t acc = 0;
#pragma unroll
                        for (int b = 0; b < kAggMaxC; ++b)
                            if (b < a.C) acc |= qw[b][w] ^ __ldg(x + b * WT + w);
                        if (w == WT - 1) acc &= tail;
                        mm += __popc(acc);
                    }
                } else {
                    for (int w = 0; w < W; ++w) {
                        uint32_t acc = 0;
                        for (int b = 0; b < a.C; ++b) acc |= __ldg(qr + b * W + w) ^ __ldg(x + b * W + w);
                        if (w == W - 1) acc &= tail;
                        mm += __popc(acc);
                    }
                }
                const int c = a.L - mm;
                cmax = tmax(cmax, c);
                if (a.kind == 1 && c > 0 && act) {
                    cnt[nz * 32 + lane] = static_cast<uint16_t>(c);
                    ++nz;
                }
            }
            __syncwarp();
            if (act) {
                double v;
                if (a.kind == 0) {
                    v = __ldg(a.table + cmax);
                } else if (nz == 0) {
                    v = 0.0;
                } else {  // reduceat: first + pairwise(rest), then / m
                    const double first = __ldg(a.table + cnt[lane]);
                    v = __ddiv_rn(__dadd_rn(first, pw_counts(cnt + 32 + lane, nz - 1, a.table)),
                                  static_cast<double>(m));
                }
                pq[q] = a.weights ? __dmul_rn(__ldg(a.weights + q), v) : v;
            }
            __syncwarp();
        }
        if (lane == 0)
            *out = __ddiv_rn(__dadd_rn(0.0, pw_doubles(pq, a.m_q)), static_cast<double>(a.m_q));
        __syncwarp();
    }
}

static int64_t agg_warps(int64_t items) {
    return tmax<int64_t>(1, tmin<int64_t>(items, 148LL * 4 * kAggWarps));
}

static size_t agg_warp_bytes(int m_q, int64_t m_cap) {
    return static_cast<size_t>(64 * m_cap) + static_cast<size_t>(m_q) * 8;
}

}  // namespace dsrt

using namespace dsrt;

static size_t ovf_bytes(int64_t items) {
    return static_cast<size_t>(tmin<int64_t>(items, kOvfCap)) * 8 + 256;
}

extern "C" size_t dsrt_score_agg_workspace(int64_t n_qsets, int64_t cand_ld, int m_q, int64_t m_cap) {
    if (n_qsets < 0 || cand_ld < 0 || m_q < 1 || m_cap < 0) return 0;
    const int64_t warps = (agg_warps(n_qsets * cand_ld) + kAggWarps - 1) / kAggWarps * kAggWarps;
    return static_cast<size_t>(warps) * agg_warp_bytes(m_q, m_cap) + 256 + ovf_bytes(n_qsets * cand_ld);
}

extern "C" int dsrt_score_agg(const uint32_t *records, const int64_t *set_off, int64_t n_sets,
                              const int64_t *cand, const int32_t *n_cand, int64_t cand_ld,
                              const uint32_t *qrecords, int64_t n_qsets, int m_q, int L, int C,
                              int inner_kind, const double *table, const double *weights,
                              int64_t m_cap, double *scores, void *workspace, size_t ws_bytes,
                              void *stream) {
    DSRT_REQUIRE(m_q >= 1, DSRT_EINVAL, "empty query: need at least one query vector");
    DSRT_REQUIRE(L >= 1 && L <= 65535 && C >= 1, DSRT_EINVAL, "invalid parameter: L=%d C=%d", L, C);
    DSRT_REQUIRE(C <= kAggMaxC, DSRT_EUNSUPPORTED, "invalid parameter: C=%d > %d", C, kAggMaxC);
    DSRT_REQUIRE(inner_kind == 0 || inner_kind == 1, DSRT_EINVAL,
                 "invalid parameter: inner_kind=%d (0 max, 1 avg-phi)", inner_kind);
    DSRT_REQUIRE(n_qsets >= 0 && cand_ld >= 0 && n_sets >= 0 && m_cap >= 0, DSRT_EINVAL,
                 "invalid parameter: negative size");
    DSRT_REQUIRE(cand != nullptr || cand_ld <= n_sets, DSRT_EINVAL,
                 "invalid parameter: cand_ld > n_sets without a candidate list");
    const int W = plane_words(L);
    const int64_t items = n_qsets * cand_ld;
    if (items == 0) return DSRT_OK;
    if (inner_kind == 0 && score_max_fast_supported(L, C))  // weighted max: the K3 kernels
        return score_max_fast(records, set_off, n_sets, cand, n_cand, cand_ld, qrecords, n_qsets,
                              m_q, L, C, table, weights, scores, as_stream(stream));
    DSRT_REQUIRE(ws_bytes >= dsrt_score_agg_workspace(n_qsets, cand_ld, m_q, m_cap), DSRT_EINVAL,
                 "invalid parameter: aggregation workspace too small");
    cudaStream_t st = as_stream(stream);
    AggArgs a{};
    a.records = records;
    a.set_off = set_off;
    a.n_sets = n_sets;
    a.cand = cand;
    a.n_cand = n_cand;
    a.cand_ld = cand_ld;
    a.qrecs = qrecords;
    a.n_qsets = n_qsets;
    a.m_q = m_q;
    a.L = L;
    a.C = C;
    a.R = record_words(L, C);
    a.kind = inner_kind;
    a.table = table;
    a.weights = weights;
    a.scores = scores;
    a.m_cap = m_cap;
    a.warp_bytes = agg_warp_bytes(m_q, m_cap);
    uint8_t *w = static_cast<uint8_t *>(workspace);
    a.status = reinterpret_cast<uint32_t *>(w);
    unsigned long long *ovf_count = reinterpret_cast<unsigned long long *>(w + 8);
    int64_t *ovf_items = reinterpret_cast<int64_t *>(w + 256);
    a.scratch = w + ovf_bytes(items) + 256;
    DSRT_CUDA(cudaMemsetAsync(w, 0, 16, st));
    int64_t work = items;
    if (inner_kind == 1 && score_avg_supported(L, C, m_q)) {
        // streaming kernel; targets with > 129 colliding vectors come back as a list
        const int64_t cap = tmin<int64_t>(items, kOvfCap);
        int rc = score_avg_fast(records, set_off, n_sets, cand, n_cand, cand_ld, qrecords, n_qsets,
                                m_q, L, C, table, weights, scores, ovf_items, ovf_count, cap, st);
        if (rc) return rc;
        unsigned long long n_ovf = 0;
        DSRT_CUDA(cudaMemcpyAsync(&n_ovf, ovf_count, 8, cudaMemcpyDeviceToHost, st));
        DSRT_CUDA(cudaStreamSynchronize(st));
        if (n_ovf == 0) return DSRT_OK;
        if (static_cast<int64_t>(n_ovf) <= cap) {
            a.items = ovf_items;
            a.n_items = static_cast<int64_t>(n_ovf);
            work = a.n_items;
        }
    }
    const unsigned blocks = static_cast<unsigned>((agg_warps(work) + kAggWarps - 1) / kAggWarps);
    switch (W) {
        case 1: score_agg_kernel<1><<<blocks, kAggWarps * 32, 0, st>>>(a); break;
        case 2: score_agg_kernel<2><<<blocks, kAggWarps * 32, 0, st>>>(a); break;
        case 3: score_agg_kernel<3><<<blocks, kAggWarps * 32, 0, st>>>(a); break;
        case 4: score_agg_kernel<4><<<blocks, kAggWarps * 32, 0, st>>>(a); break;
        default: score_agg_kernel<0><<<blocks, kAggWarps * 32, 0, st>>>(a); break;
    }
    DSRT_LAUNCH_CHECK();
    uint32_t h = 0;
    DSRT_CUDA(cudaMemcpyAsync(&h, a.status, 4, cudaMemcpyDeviceToHost, st));
    DSRT_CUDA(cudaStreamSynchronize(st));
    DSRT_REQUIRE((h & 1u) == 0, DSRT_EINVAL, "invalid parameter: set larger than m_cap=%lld",
                 static_cast<long long>(m_cap));
    return DSRT_OK;
}

namespace dsrt {
// sigma = max (kind 0) on the general kernel with its own stream-ordered workspace:
// the K3 entry points' path for shapes outside the register-blocked kernels.
int score_general_max(const uint32_t *records, const int64_t *set_off, int64_t n_sets,
                      const int64_t *cand, const int32_t *n_cand, int64_t cand_ld,
                      const uint32_t *qrecs, int64_t n_qsets, int m_q, int L, int C, const double *lut,
                      const double *weights, double *scores, cudaStream_t st) {
    const size_t ws = dsrt_score_agg_workspace(n_qsets, cand_ld, m_q, 0);
    void *w = nullptr;
    DSRT_CUDA(malloc_async(&w, ws, st));
    const int rc = dsrt_score_agg(records, set_off, n_sets, cand, n_cand, cand_ld, qrecs, n_qsets, m_q, L, C,
                                  0, lut, weights, 0, scores, w, ws, st);
    cudaFreeAsync(w, st);
    return rc;
}
}  // namespace dsrt
