// K3 dispatch + C ABI (kernels in score_kernels.cuh, instantiated in score_inst_*.cu).
#include <cstdlib>

#include "score_kernels.cuh"

namespace dsrt {

// ----------------------------------------------- m_q > 128: finalize pass
// per-query value w[i] * LUT[c_q] of one (query set, set) row
struct McRow {
    const uint16_t *mc;
    const double *lut, *w;
    __device__ __forceinline__ double operator()(int i) const {
        const double v = __ldg(lut + mc[i]);
        return __dmul_rn(w != nullptr ? __ldg(w + i) : 1.0, v);
    }
};

// numpy pairwise_sum_DOUBLE of f(lo .. lo + n - 1): 8 strided accumulators per
// <= 128 leaf, recursive split n2 = n/2 - (n/2 mod 8) above (no scratch).
template <class F>
__device__ double pw_rec(const F &f, int lo, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r = __dadd_rn(r, f(lo + i));
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = f(lo + j);
        int i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], f(lo + i + j));
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; ++i) res = __dadd_rn(res, f(lo + i));
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(pw_rec(f, lo, n2), pw_rec(f, lo + n2, n - n2));
}

// One thread per target e < w of one query set: LUT[maxcounts] -> weighted
// numpy pairwise mean -> out[e].  Candidate lists: entries e >= n_cand stay
// unwritten and invalid set indices get NaN, as on the m_q <= 128 path (their
// maxcount rows were never written and are not read).
__global__ void finalize_kernel(const uint16_t *__restrict__ mc, int64_t w, int m_q,
                                const double *__restrict__ lut, const double *__restrict__ weights,
                                double *__restrict__ out, const int64_t *__restrict__ cand_row,
                                const int32_t *__restrict__ n_cand_q, int64_t n_sets) {
    const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (e >= w) return;
    if (n_cand_q != nullptr && e >= tmin<int64_t>(w, tmax<int32_t>(0, __ldg(n_cand_q)))) return;
    if (cand_row != nullptr) {
        const int64_t s = __ldg(cand_row + e);
        if (s < 0 || s >= n_sets) {
            out[e] = __longlong_as_double(0x7ff8000000000000ll);
            return;
        }
    }
    const McRow f{mc + e * m_q, lut, weights};
    const double sum = __dadd_rn(0.0, pw_rec(f, 0, m_q));
    out[e] = __ddiv_rn(sum, static_cast<double>(m_q));
}

extern template int run_w<1>(const ScoreArgs &, int, int, cudaStream_t);
extern template int run_w<2>(const ScoreArgs &, int, int, cudaStream_t);
extern template int run_w<3>(const ScoreArgs &, int, int, cudaStream_t);
extern template int run_w<4>(const ScoreArgs &, int, int, cudaStream_t);
extern template int run_w<5>(const ScoreArgs &, int, int, cudaStream_t);
extern template int run_w<6>(const ScoreArgs &, int, int, cudaStream_t);
extern template int run_w<7>(const ScoreArgs &, int, int, cudaStream_t);
extern template int run_w<8>(const ScoreArgs &, int, int, cudaStream_t);
extern template int run_w<9>(const ScoreArgs &, int, int, cudaStream_t);
extern template int run_w<10>(const ScoreArgs &, int, int, cudaStream_t);
extern template int run_w<11>(const ScoreArgs &, int, int, cudaStream_t);
extern template int run_w<12>(const ScoreArgs &, int, int, cudaStream_t);
extern template int run_w<13>(const ScoreArgs &, int, int, cudaStream_t);
extern template int run_w<14>(const ScoreArgs &, int, int, cudaStream_t);
extern template int run_w<15>(const ScoreArgs &, int, int, cudaStream_t);
extern template int run_w<16>(const ScoreArgs &, int, int, cudaStream_t);

static int run_k(const ScoreArgs &a, int C, int qpl, cudaStream_t st) {
    const int W = plane_words(a.L);
    if (C * W > 32) {  // keep query planes within a register budget
        set_error("invalid parameter: C*ceil(L/32)=%d exceeds the kernel register budget (32)", C * W);
        return DSRT_EUNSUPPORTED;
    }
    switch (C) {
#define DSRT_CASE(k) \
    case k: return run_w<k>(a, W, qpl, st);
        DSRT_CASE(1) DSRT_CASE(2) DSRT_CASE(3) DSRT_CASE(4) DSRT_CASE(5) DSRT_CASE(6)
        DSRT_CASE(7) DSRT_CASE(8) DSRT_CASE(9) DSRT_CASE(10) DSRT_CASE(11) DSRT_CASE(12)
        DSRT_CASE(13) DSRT_CASE(14) DSRT_CASE(15) DSRT_CASE(16)
#undef DSRT_CASE
        default: break;
    }
    set_error("invalid parameter: C=%d unsupported by the scoring kernel (C <= 16)", C);
    return DSRT_EUNSUPPORTED;
}

// m_q <= 128 runs in one pass; larger m_q runs 128-query slices writing
// uint16 maxcounts, then finalize_kernel applies numpy's recursive pairwise sum.
// The maxcount scratch is bounded: set ranges are processed in sub-ranges of
// at most kMcBudget bytes per query set.
constexpr size_t kMcBudget = size_t(256) << 20;

bool score_max_fast_supported(int L, int C);
int score_general_max(const uint32_t *records, const int64_t *set_off, int64_t n_sets,
                      const int64_t *cand, const int32_t *n_cand, int64_t cand_ld,
                      const uint32_t *qrecs, int64_t n_qsets, int m_q, int L, int C, const double *lut,
                      const double *weights, double *scores, cudaStream_t st);

// Shapes outside the register-blocked kernels (C > 16 or C * ceil(L/32) > 32;
// the reference allows C <= 24 and any L, lsh.py:17, 54-66): scores through the
// general kernel K3g (score_agg.cu) with sigma = max -- same arithmetic, no
// register blocking.  Integer max counts and the threshold-append epilogue
// stay with the fast kernels.
static int score_general(const ScoreArgs &a, int C, cudaStream_t st) {
    DSRT_REQUIRE(a.mc == nullptr && a.app.tau == nullptr, DSRT_EUNSUPPORTED,
                 "invalid parameter: max counts / threshold search need C <= 16 and "
                 "C*ceil(L/32) <= 32 (L=%d, C=%d)", a.L, C);
    if (a.scores == nullptr) return DSRT_OK;
    const int R = record_words(a.L, C);
    const int64_t width = a.cand_mode ? a.cand_ld : (a.se - a.sb);
    if (width == 0) return DSRT_OK;
    // exhaustive ranges: identity candidates over the shifted set window
    const int64_t *off = a.cand_mode ? a.set_off : a.set_off + a.sb;
    const int64_t ns = a.cand_mode ? a.n_sets : width;
    const int64_t ld = a.ld > 0 ? a.ld : width;
    if (ld == width)
        return score_general_max(a.recs, off, ns, a.cand_mode ? a.cand : nullptr,
                                 a.cand_mode ? a.n_cand : nullptr, width, a.qrecs, a.n_qsets, a.m_q,
                                 a.L, C, a.lut, a.weights, a.scores, st);
    for (int64_t qs = 0; qs < a.n_qsets; ++qs) {  // strided output rows: one query set per call
        const int64_t *cq = a.cand_mode && a.cand ? a.cand + qs * a.cand_ld : nullptr;
        const int32_t *nq = a.cand_mode && a.n_cand ? a.n_cand + qs : nullptr;
        const int rc = score_general_max(a.recs, off, ns, cq, nq, width,
                                         a.qrecs + qs * a.m_q * static_cast<int64_t>(R), 1, a.m_q, a.L,
                                         C, a.lut, a.weights, a.scores + qs * ld, st);
        if (rc) return rc;
    }
    return DSRT_OK;
}

int score_dispatch(ScoreArgs a, int C, cudaStream_t st) {
    if (const char *e = getenv("DSRT_QS")) a.qs_override = atoi(e);
    DSRT_REQUIRE(a.m_q >= 1, DSRT_EINVAL, "empty query: need at least one query vector");
    DSRT_REQUIRE(a.L >= 1 && C >= 1, DSRT_EINVAL, "invalid parameter: L=%d C=%d", a.L, C);
    if (a.n_qsets == 0) return DSRT_OK;
    if (!score_max_fast_supported(a.L, C)) return score_general(a, C, st);
    const int R = record_words(a.L, C);
    if (a.m_q <= 128) {
        const int qpl = (a.m_q + 31) / 32;
        a.mc_stride = a.m_q;
        a.mc_q0 = 0;
        return run_k(a, C, qpl == 3 ? 4 : qpl, st);
    }
    DSRT_REQUIRE(a.app.tau == nullptr, DSRT_EUNSUPPORTED,
                 "invalid parameter: threshold append needs m_q <= 128");
    // targets of one query set: [t0, t1) = set range (exhaustive), identity
    // candidates [0, cand_ld) (cand == nullptr) or one candidate list (unsplit)
    const bool split = !a.cand_mode || a.cand == nullptr;
    const int64_t width = a.cand_mode ? a.cand_ld : (a.se - a.sb);
    if (width == 0) return DSRT_OK;
    const int64_t sub = split ? tmax<int64_t>(1, static_cast<int64_t>(kMcBudget / (2 * a.m_q))) : width;
    uint16_t *own = nullptr;
    if (a.mc == nullptr)
        DSRT_CUDA(malloc_async(reinterpret_cast<void **>(&own),
                               static_cast<size_t>(tmin(sub, width)) * a.m_q * sizeof(uint16_t), st));
    const int64_t ld = a.cand_mode ? a.cand_ld : a.ld;
    int rc = DSRT_OK;
    for (int64_t qs = 0; qs < a.n_qsets && rc == DSRT_OK; ++qs) {
        for (int64_t e0 = 0; e0 < width && rc == DSRT_OK; e0 += sub) {
            const int64_t e1 = tmin(width, e0 + sub);
            // maxcounts of (qs, e0 .. e1): the caller's array or the scratch
            uint16_t *mc = own ? own : a.mc + (qs * ld + e0) * a.m_q;
            for (int q0 = 0; q0 < a.m_q && rc == DSRT_OK; q0 += 128) {
                // Each 128-query slice is a pseudo query set (n_qsets = 1) whose
                // records start at qrecs + (qs*m_q + q0)*R; it writes uint16 counts
                // at mc[e*m_q + q0 + qi].
                ScoreArgs b = a;
                b.n_qsets = 1;
                b.m_q = min(128, a.m_q - q0);
                b.qrecs = a.qrecs + (qs * a.m_q + q0) * static_cast<int64_t>(R);
                b.scores = nullptr;
                b.weights = nullptr;
                b.mc = mc;
                b.mc_stride = a.m_q;
                b.mc_q0 = q0;
                b.ld = e1 - e0;
                if (!b.cand_mode) {
                    b.sb = a.sb + e0;
                    b.se = a.sb + e1;
                } else if (b.cand == nullptr) {  // identity candidates: shift the set window
                    b.set_off = a.set_off + e0;
                    b.n_sets = tmin<int64_t>(a.n_sets - e0, e1 - e0);
                    b.cand_ld = e1 - e0;
                    b.n_cand = nullptr;  // entries >= n_cand may be written (they are unspecified)
                } else {
                    b.cand = a.cand + qs * a.cand_ld;
                    if (a.n_cand) b.n_cand = a.n_cand + qs;
                }
                const int qpl = (b.m_q + 31) / 32;
                rc = run_k(b, C, qpl == 3 ? 4 : qpl, st);
            }
            if (rc == DSRT_OK && a.scores != nullptr) {
                const int64_t w = e1 - e0;
                const bool list = a.cand_mode && a.cand != nullptr;
                const int32_t *nc = list && a.n_cand ? a.n_cand + qs : nullptr;
                finalize_kernel<<<static_cast<unsigned>((w + 127) / 128), 128, 0, st>>>(
                    mc, w, a.m_q, a.lut, a.weights, a.scores + qs * ld + e0,
                    list ? a.cand + qs * a.cand_ld : nullptr, nc, a.n_sets);
                if (cudaGetLastError() != cudaSuccess) rc = DSRT_ECUDA;
            }
        }
    }
    if (own) cudaFreeAsync(own, st);
    return rc;
}

// sigma = max with optional weights for dsrt_score_agg: the exhaustive kernel
// when every set is scored by >= 8 query sets, else the candidate kernel.
int score_max_fast(const uint32_t *records, const int64_t *set_off, int64_t n_sets,
                   const int64_t *cand, const int32_t *n_cand, int64_t cand_ld,
                   const uint32_t *qrecs, int64_t n_qsets, int m_q, int L, int C,
                   const double *lut, const double *weights, double *scores, cudaStream_t st) {
    ScoreArgs a{};
    a.recs = records; a.set_off = set_off; a.n_sets = n_sets; a.qrecs = qrecs;
    a.n_qsets = n_qsets; a.m_q = m_q; a.L = L; a.lut = lut; a.weights = weights;
    a.scores = scores;
    if (cand == nullptr && n_cand == nullptr && n_qsets >= 8 && cand_ld <= n_sets) {
        a.cand_mode = false;
        a.sb = 0; a.se = cand_ld; a.ld = cand_ld;
    } else {
        a.cand_mode = true;
        a.cand = cand; a.n_cand = n_cand; a.cand_ld = cand_ld; a.ld = cand_ld;
    }
    return score_dispatch(a, C, st);
}

bool score_max_fast_supported(int L, int C) {
    return L >= 1 && L <= 128 && C >= 1 && C <= 16 && C * plane_words(L) <= 32;
}

}  // namespace dsrt

using namespace dsrt;

extern "C" int dsrt_score_all(const uint32_t *records, const int64_t *set_off, int64_t set_begin,
                              int64_t set_end, const uint32_t *qrecords, int64_t n_qsets, int m_q,
                              int L, int C, const double *lut, double *scores, int64_t ld,
                              uint16_t *maxcounts, void *stream) {
    DSRT_REQUIRE(set_begin >= 0 && set_end >= set_begin, DSRT_EINVAL,
                 "invalid parameter: set range [%lld, %lld)", (long long)set_begin,
                 (long long)set_end);
    DSRT_REQUIRE(ld >= set_end - set_begin, DSRT_EINVAL, "invalid parameter: ld < set count");
    if (set_end == set_begin) return DSRT_OK;
    ScoreArgs a{};
    a.cand_mode = false;
    a.recs = records; a.set_off = set_off; a.sb = set_begin; a.se = set_end;
    a.n_sets = set_end; a.qrecs = qrecords; a.n_qsets = n_qsets; a.m_q = m_q; a.L = L;
    a.lut = lut; a.scores = scores; a.ld = ld; a.mc = maxcounts;
    return score_dispatch(a, C, as_stream(stream));
}

extern "C" int dsrt_score_candidates(const uint32_t *records, const int64_t *set_off,
                                     int64_t n_sets, const int64_t *cand, const int32_t *n_cand,
                                     int64_t cand_ld, const uint32_t *qrecords, int64_t n_qsets,
                                     int m_q, int L, int C, const double *lut, double *scores,
                                     uint16_t *maxcounts, void *stream) {
    DSRT_REQUIRE(cand_ld >= 0, DSRT_EINVAL, "invalid parameter: cand_ld < 0");
    if (cand_ld == 0) return DSRT_OK;
    ScoreArgs a{};
    a.cand_mode = true;
    a.recs = records; a.set_off = set_off; a.n_sets = n_sets; a.cand = cand; a.n_cand = n_cand;
    a.cand_ld = cand_ld; a.qrecs = qrecords; a.n_qsets = n_qsets; a.m_q = m_q; a.L = L;
    a.lut = lut; a.scores = scores; a.ld = cand_ld; a.mc = maxcounts;
    return score_dispatch(a, C, as_stream(stream));
}
