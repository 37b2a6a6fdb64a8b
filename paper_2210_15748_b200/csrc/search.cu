// Exhaustive search: K3 scoring of every set fused with the K4 top-k.
//
// Replaces query()'s exhaustive branch -- _score_chunk over np.arange(N)
// (index.py:250-261, 302-310) followed by heapq.nsmallest with key
// (-score, doc_id) (index.py:314-319) -- for a batch of query sets, without
// materialising the n_qsets x N float64 score matrix in HBM.
//
// Threshold mode (m_q <= 128, n_qsets >= 8, large N):
//   seed   sets [0, s0): scores into a buffer, top-k -> head of list A,
//          tau[q] = k-th best score so far (-1.0 while fewer than k sets);
//   rounds sets [s_r, s_r+1), ranges growing 8x: the K3 epilogue appends each
//          set whose score >= tau[q] to list A as (score, doc id); top-k over A
//          -> head of list B, tau = its k-th score; swap A and B.
// Correctness: tau is the k-th best score of a subset of the sets, so it is
// <= the final k-th best; every global winner therefore has score >= tau when
// its set is scored and is appended.  Sets below tau cannot enter the top-k of
// the sets scored so far (the head holds k entries >= tau).  Ties with tau are
// kept, so the final top-k applies the reference key (score desc, doc id asc)
// to a superset of the winners: results equal the materialised ranking.
// With ~8x growth per round about 7k sets survive per round; a list that
// exceeds its capacity raises *overflow and the caller reruns in mode 1.
//
// Materialised mode (mode 1, m_q > 128, n_qsets < 8, or a small score
// matrix): chunks of sets are scored into the buffer, each chunk's top-k is
// merged into a running top-k (list columns [0, k) running, [k, 2k) chunk).
#include <cstdlib>
#include <mutex>
#include <utility>
#include <vector>

#include "score_kernels.cuh"
#include "topk.cuh"

namespace dsrt {

namespace {

constexpr int64_t kGrowth = 8;         // round length ratio
constexpr int64_t kSeedDiv = 512;      // seed = N / 512 sets (at least kSeedMinK * k): its scores are materialised
constexpr int64_t kSeedMinK = 4;
constexpr size_t kThresholdMinBytes = size_t(512) << 20;  // score matrix size that switches modes

// DSRT_SEARCH_MIN_BYTES (test knob): score-matrix size above which mode 0 uses
// threshold rounds (default 512 MB; tests lower it to cover the path at small N)
size_t threshold_min_bytes() {
    const char *e = getenv("DSRT_SEARCH_MIN_BYTES");
    return e ? static_cast<size_t>(strtoull(e, nullptr, 10)) : kThresholdMinBytes;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct Plan {
    bool threshold = false;
    int64_t chunk = 0;  // materialised: sets per chunk; threshold: seed sets s0
    int64_t cap = 0;    // list row capacity
    size_t off_lists = 0, off_cnt = 0, off_tau = 0, total = 0;
};

}  // namespace
bool score_max_fast_supported(int L, int C);
namespace {

Plan make_plan(int64_t N, int64_t n_q, int m_q, int k, int mode, size_t buf_bytes, bool fast = true) {
    Plan p;
    const int64_t per_set = 8 * tmax<int64_t>(1, n_q);
    const int64_t chunk_w = tmax<int64_t>(1, tmin<int64_t>(N, static_cast<int64_t>(buf_bytes) / per_set));
    const int64_t s0 = tmin<int64_t>(chunk_w, tmax<int64_t>(N / kSeedDiv, kSeedMinK * k));
    p.threshold = mode == 0 && fast && m_q <= 128 && n_q >= 8 && s0 < N && s0 >= 2 * static_cast<int64_t>(k) &&
                  static_cast<size_t>(n_q) * N * 8 > threshold_min_bytes();
    if (p.threshold) {
        p.chunk = s0;
        p.cap = tmin<int64_t>(k + N, 17 * static_cast<int64_t>(k) + 4096);
    } else {
        p.chunk = chunk_w;
        p.cap = 2 * static_cast<int64_t>(k);
    }
    const size_t buf = align256(static_cast<size_t>(n_q) * p.chunk * 8);
    const size_t list = align256(static_cast<size_t>(n_q) * p.cap * 16);
    p.off_lists = buf;
    p.off_cnt = buf + 2 * list;
    p.off_tau = p.off_cnt + align256(static_cast<size_t>(n_q) * 4 * 2);
    p.total = p.off_tau + align256(static_cast<size_t>(n_q) * 8) + 256;
    return p;
}

// Optional CUDA-event timing of every launch (bench.py: the dominant kernel's
// time measured on the launching stream).  Off by default; not thread-safe
// beyond the mutex around the event lists.
struct Prof {
    std::mutex mu;
    bool on = false;
    std::vector<cudaEvent_t> ev[2];  // [0] scoring launches, [1] top-k / list kernels (pairs)
    int64_t launches = 0;
};
Prof &prof() {
    static Prof p;
    return p;
}
struct ProfScope {  // records a (start, stop) pair around one launch when profiling
    cudaEvent_t a = nullptr, b = nullptr;
    int cls;
    cudaStream_t st;
    ProfScope(int c, cudaStream_t s) : cls(c), st(s) {
        Prof &p = prof();
        std::lock_guard<std::mutex> g(p.mu);
        if (!p.on) return;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, st);
    }
    ~ProfScope() {
        if (a == nullptr) return;
        cudaEventRecord(b, st);
        Prof &p = prof();
        std::lock_guard<std::mutex> g(p.mu);
        p.ev[cls].push_back(a);
        p.ev[cls].push_back(b);
    }
};

struct List {
    double *s;
    uint64_t *id;
    int32_t *cnt;
};

// cnt_prev > cap_prev -> overflow; next list: k head entries, tau = k-th score
__global__ void list_next_kernel(const int32_t *__restrict__ cnt_prev, int64_t cap_prev,
                                 int32_t *__restrict__ cnt_next, double *__restrict__ tau,
                                 const double *__restrict__ s_next, int64_t cap_next, int k,
                                 int64_t n_q, int32_t *__restrict__ overflow) {
    const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (q >= n_q) return;
    if (cnt_prev != nullptr && cnt_prev[q] > cap_prev) atomicOr(overflow, 1);
    if (cnt_next != nullptr) {
        cnt_next[q] = k;
        tau[q] = s_next[q * cap_next + k - 1];
    }
}

struct Search {
    const uint32_t *records;
    const int64_t *set_off;
    int64_t N;
    const uint64_t *doc_ids;
    const uint32_t *qrecs;
    int64_t n_q;
    int m_q, L, C;
    const double *lut, *weights;
    int k;
    cudaStream_t st;

    // scores of sets [c0, c1) for every query set -> buf (n_q, c1 - c0)
    int score_range(int64_t c0, int64_t c1, double *buf, const AppendOut *app) const {
        ScoreArgs a{};
        a.recs = records; a.qrecs = qrecs; a.n_qsets = n_q; a.m_q = m_q; a.L = L;
        a.lut = lut; a.weights = weights;
        if (app != nullptr || n_q >= 8) {  // exhaustive kernel
            a.cand_mode = false;
            a.set_off = set_off; a.n_sets = N; a.sb = c0; a.se = c1;
            a.scores = app ? nullptr : buf; a.ld = c1 - c0;
            if (app) a.app = *app;
        } else {                           // few query sets: candidate kernel over the window
            a.cand_mode = true;
            a.set_off = set_off + c0; a.n_sets = c1 - c0; a.cand_ld = c1 - c0; a.ld = c1 - c0;
            a.scores = buf;
        }
        ProfScope ps(0, st);
        return score_dispatch(a, C, st);
    }

    // top-k of rows (n entries, stride ld) -> (out_s, out_id) rows at out_ld
    int topk(const double *s, int64_t ld, int64_t n, const uint64_t *ids, int64_t ids_ld,
             const int32_t *n_valid, double *out_s, uint64_t *out_id, int64_t out_ld) const {
        TopkArgs t{};
        t.scores = s; t.ld = ld; t.n = n; t.ids = ids; t.ids_ld = ids_ld; t.n_valid = n_valid;
        t.k = k; t.out_s = out_s; t.out_id = out_id; t.out_ld = out_ld;
        ProfScope ps(1, st);
        return topk_run(t, n_q, st);
    }
};

int list_next(const Search &S, const List *prev, int64_t cap_prev, const List *next,
              int64_t cap_next, double *tau, int32_t *overflow) {
    const unsigned blocks = static_cast<unsigned>((S.n_q + 255) / 256);
    ProfScope ps(1, S.st);
    list_next_kernel<<<blocks, 256, 0, S.st>>>(prev ? prev->cnt : nullptr, cap_prev,
                                               next ? next->cnt : nullptr, tau,
                                               next ? next->s : nullptr, cap_next, S.k, S.n_q,
                                               overflow);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}

#define DSRT_TRY(x)                    \
    do {                               \
        const int _rc = (x);           \
        if (_rc != DSRT_OK) return _rc; \
    } while (0)

int run_materialised(const Search &S, const Plan &p, double *buf, List A, List B,
                     double *out_s, uint64_t *out_id) {
    const int64_t k = S.k;
    for (int64_t c0 = 0; c0 < S.N; c0 += p.chunk) {
        const int64_t c1 = tmin(S.N, c0 + p.chunk), w = c1 - c0;
        const bool first = c0 == 0, last = c1 == S.N;
        DSRT_TRY(S.score_range(c0, c1, buf, nullptr));
        if (first) {  // running top-k = this chunk's (or the answer)
            DSRT_TRY(S.topk(buf, w, w, S.doc_ids + c0, 0, nullptr, last ? out_s : A.s,
                            last ? out_id : A.id, last ? k : p.cap));
            continue;
        }
        DSRT_TRY(S.topk(buf, w, w, S.doc_ids + c0, 0, nullptr, A.s + k, A.id + k, p.cap));
        DSRT_TRY(S.topk(A.s, p.cap, 2 * k, A.id, p.cap, nullptr, last ? out_s : B.s,
                        last ? out_id : B.id, last ? k : p.cap));
        std::swap(A, B);
    }
    return DSRT_OK;
}

int run_threshold(const Search &S, const Plan &p, double *buf, List A, List B, double *tau,
                  double *out_s, uint64_t *out_id, int32_t *overflow) {
    const int64_t s0 = p.chunk;
    DSRT_TRY(S.score_range(0, s0, buf, nullptr));
    DSRT_TRY(S.topk(buf, s0, s0, S.doc_ids, 0, nullptr, A.s, A.id, p.cap));
    DSRT_TRY(list_next(S, nullptr, 0, &A, p.cap, tau, overflow));
    for (int64_t r0 = s0; r0 < S.N;) {
        const int64_t r1 = tmin(S.N, r0 * kGrowth);
        const bool last = r1 == S.N;
        const AppendOut app{tau, A.cnt, A.s, A.id, S.doc_ids, p.cap};
        DSRT_TRY(S.score_range(r0, r1, nullptr, &app));
        DSRT_TRY(S.topk(A.s, p.cap, p.cap, A.id, p.cap, A.cnt, last ? out_s : B.s,
                        last ? out_id : B.id, last ? S.k : p.cap));
        DSRT_TRY(list_next(S, &A, p.cap, last ? nullptr : &B, p.cap, tau, overflow));
        std::swap(A, B);
        r0 = r1;
    }
    return DSRT_OK;
}

}  // namespace

}  // namespace dsrt

using namespace dsrt;

extern "C" size_t dsrt_search_all_workspace(int64_t n_sets, int64_t n_qsets, int m_q, int k, int mode,
                                            size_t score_buffer_bytes) {
    if (n_sets <= 0 || n_qsets <= 0 || k < 1) return 256;
    // either plan (threshold rounds need fast-kernel shapes; others run materialised)
    return tmax(make_plan(n_sets, n_qsets, m_q, k, mode, score_buffer_bytes, true).total,
                make_plan(n_sets, n_qsets, m_q, k, mode, score_buffer_bytes, false).total);
}

extern "C" int dsrt_search_all(const uint32_t *records, const int64_t *set_off, int64_t n_sets,
                               const uint64_t *doc_ids, const uint32_t *qrecords, int64_t n_qsets,
                               int m_q, int L, int C, const double *lut, const double *weights, int k,
                               int mode, size_t score_buffer_bytes, double *out_scores,
                               uint64_t *out_ids, int32_t *overflow, void *workspace, size_t ws_bytes,
                               void *stream) {
    DSRT_REQUIRE(k >= 1, DSRT_EINVAL, "invalid parameter: top_k must be >= 1, got %d", k);
    DSRT_REQUIRE(m_q >= 1, DSRT_EINVAL, "empty query: need at least one query vector");
    DSRT_REQUIRE(n_sets >= 0 && n_qsets >= 0, DSRT_EINVAL, "invalid parameter: negative size");
    DSRT_REQUIRE(mode == 0 || mode == 1, DSRT_EINVAL, "invalid parameter: mode=%d", mode);
    DSRT_REQUIRE(doc_ids != nullptr && overflow != nullptr, DSRT_EINVAL,
                 "invalid parameter: doc_ids and overflow are required");
    const cudaStream_t st = as_stream(stream);
    DSRT_CUDA(cudaMemsetAsync(overflow, 0, sizeof(int32_t), st));
    if (n_qsets == 0) return DSRT_OK;
    if (n_sets == 0) {  // every row is padding
        TopkArgs t{};
        t.scores = nullptr; t.ld = 0; t.n = 0; t.k = k; t.out_s = out_scores; t.out_id = out_ids;
        return topk_run(t, n_qsets, st);
    }
    const Plan p = make_plan(n_sets, n_qsets, m_q, k, mode, score_buffer_bytes, score_max_fast_supported(L, C));
    DSRT_REQUIRE(workspace != nullptr && ws_bytes >= p.total, DSRT_EINVAL,
                 "invalid parameter: search workspace %zu < %zu bytes", ws_bytes, p.total);
    uint8_t *ws = static_cast<uint8_t *>(workspace);
    double *buf = reinterpret_cast<double *>(ws);
    const size_t list_bytes = align256(static_cast<size_t>(n_qsets) * p.cap * 16);
    List A{reinterpret_cast<double *>(ws + p.off_lists), nullptr,
           reinterpret_cast<int32_t *>(ws + p.off_cnt)};
    A.id = reinterpret_cast<uint64_t *>(A.s + n_qsets * p.cap);
    List B{reinterpret_cast<double *>(ws + p.off_lists + list_bytes), nullptr, A.cnt + n_qsets};
    B.id = reinterpret_cast<uint64_t *>(B.s + n_qsets * p.cap);
    double *tau = reinterpret_cast<double *>(ws + p.off_tau);
    const Search S{records, set_off, n_sets, doc_ids, qrecords, n_qsets, m_q, L, C, lut, weights, k, st};
    if (p.threshold) return run_threshold(S, p, buf, A, B, tau, out_scores, out_ids, overflow);
    return run_materialised(S, p, buf, A, B, out_scores, out_ids);
}

extern "C" void dsrt_search_profile(int enable) {
    Prof &p = prof();
    std::lock_guard<std::mutex> g(p.mu);
    p.on = enable != 0;
}

extern "C" int dsrt_search_profile_read(double *score_ms, double *other_ms, int64_t *launches) {
    Prof &p = prof();
    std::lock_guard<std::mutex> g(p.mu);
    double tot[2] = {0.0, 0.0};
    int64_t n = 0;
    for (int c = 0; c < 2; ++c) {
        for (size_t i = 0; i + 1 < p.ev[c].size(); i += 2) {
            float ms = 0.f;
            DSRT_CUDA(cudaEventSynchronize(p.ev[c][i + 1]));
            DSRT_CUDA(cudaEventElapsedTime(&ms, p.ev[c][i], p.ev[c][i + 1]));
            tot[c] += ms;
            ++n;
        }
        for (cudaEvent_t e : p.ev[c]) cudaEventDestroy(e);
        p.ev[c].clear();
    }
    if (score_ms) *score_ms = tot[0];
    if (other_ms) *other_ms = tot[1];
    if (launches) *launches = n;
    return DSRT_OK;
}
