// K4 -- batched top-k by (score desc, doc_id asc).
//
// Replaces heapq.nsmallest(top_k, ((score, doc_id) ...), key=lambda e:
// (-e[0], e[1])) in query() (index.py:314-319).  One CTA per row (query set):
//  1. MSB radix select (8-bit digits) on an order-preserving 64-bit key of the
//     float64 score (sign-flipped IEEE pattern: negative padding such as the
//     -1.0 of short rows sorts below every score) -> threshold prefix T and
//     the number of T-ties still needed;
//  2. if more ties than needed: radix select on doc_id (ascending) among the
//     ties (reference tie-break: lower doc id first);
//  3. k <= 4096: compact the k winners into shared memory and bitonic-sort
//     them by (score desc, doc_id asc);
//     k > 4096 (topk_large_kernel): compact the winners into a global scratch
//     row, bitonic-sort 4096-element runs in shared memory, then merge runs
//     pairwise (merge path, every thread merging its own output span) until
//     one run remains -- any k, no host sort.
#include "common.cuh"
#include "topk.cuh"

namespace dsrt {

constexpr int kTopkThreads = 1024;
constexpr int kTopkRun = 4096;      // large k: shared-memory sorted run length

// order-preserving key of a double (total order of the IEEE values)
__device__ __forceinline__ uint64_t okey(double d) {
    const uint64_t u = static_cast<uint64_t>(__double_as_longlong(d));
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_okey(uint64_t k) {
    const uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double(static_cast<long long>(u));
}

struct RowView {
    const double *s;
    const uint64_t *ids;
    int64_t row, ids_ld;
    const int64_t *ix = nullptr;  // optional per-row index into ids (candidate lists)
    int64_t ix_ld = 0;
    __device__ __forceinline__ uint64_t key(int64_t i) const { return okey(__ldg(s + i)); }
    __device__ __forceinline__ uint64_t id(int64_t i) const {
        if (ix != nullptr) return __ldg(ids + __ldg(ix + row * ix_ld + i));
        if (ids == nullptr) return static_cast<uint64_t>(i);
        return ids_ld ? __ldg(ids + row * ids_ld + i) : __ldg(ids + i);
    }
};

// Block-wide MSB radix select.  Among elements with pred(i), find the value
// prefix such that exactly `need` elements are >= (descending) or <=
// (ascending) it, counting ties into the last bin.  Returns (prefix, mask,
// remaining) through shared memory.
// Leading bytes shared by every candidate key are skipped: one pass ORs and
// ANDs the keys and the select starts at the first byte where they differ
// (scores in [0, 1] share their sign/exponent byte).  The digit of each pass
// is chosen by a warp-wide scan of the 256 bins (8 per lane), not a serial loop.
template <bool DESC, typename KeyF, typename PredF>
__device__ void radix_select(int64_t n, int64_t need, KeyF keyf, PredF pred, uint32_t *hist,
                             uint64_t *out_prefix, uint64_t *out_mask, int64_t *out_rem) {
    __shared__ uint64_t s_prefix, s_mask, s_or, s_and;
    __shared__ int64_t s_rem;
    __shared__ int s_done;
    if (threadIdx.x == 0) {
        s_prefix = 0;
        s_mask = 0;
        s_rem = need;
        s_done = 0;
        s_or = 0;
        s_and = ~0ull;
    }
    __syncthreads();
    {
        uint64_t o = 0, a = ~0ull;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            if (!pred(i)) continue;
            const uint64_t k = keyf(i);
            o |= k;
            a &= k;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            o |= __shfl_xor_sync(0xffffffffu, o, off);
            a &= __shfl_xor_sync(0xffffffffu, a, off);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicOr(reinterpret_cast<unsigned long long *>(&s_or), o);
            atomicAnd(reinterpret_cast<unsigned long long *>(&s_and), a);
        }
    }
    __syncthreads();
    const uint64_t diff = s_or ^ s_and;  // bits that differ between candidates
    int top = 56;
    while (top > 0 && ((diff >> top) & 255u) == 0u) top -= 8;
    if (threadIdx.x == 0) {  // the common leading bytes are part of every prefix
        const uint64_t lead = top >= 56 ? 0ull : (~0ull << (top + 8));
        s_prefix = s_and & lead;
        s_mask = lead;
    }
    __syncthreads();
    for (int shift = top; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        const uint64_t prefix = s_prefix, mask = s_mask;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            if (!pred(i)) continue;
            const uint64_t k = keyf(i);
            if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) {  // warp 0: bins in selection order, 8 per lane
            const int lane = threadIdx.x;
            uint32_t h[8];
            int64_t loc = 0;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const int dgt = DESC ? 255 - (lane * 8 + t) : lane * 8 + t;
                h[t] = hist[dgt];
                loc += h[t];
            }
            int64_t incl = loc;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int64_t y = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += y;
            }
            const int64_t rem = s_rem;
            const unsigned hitm = __ballot_sync(0xffffffffu, incl >= rem);
            const int owner = hitm ? __ffs(hitm) - 1 : 31;
            if (lane == owner) {
                int64_t cum = incl - loc;
                int t = 0;
                for (; t < 7; ++t) {
                    if (cum + h[t] >= rem) break;
                    cum += h[t];
                }
                const int sel = DESC ? 255 - (lane * 8 + t) : lane * 8 + t;
                s_rem = rem - cum;
                s_prefix = prefix | (static_cast<uint64_t>(sel) << shift);
                s_mask = mask | (255ull << shift);
                if (static_cast<int64_t>(h[t]) == rem - cum) s_done = 1;  // take the whole bin
            }
        }
        __syncthreads();
        if (s_done) break;
    }
    if (threadIdx.x == 0) {
        *out_prefix = s_prefix;
        *out_mask = s_mask;
        *out_rem = s_rem;
    }
    __syncthreads();
}

// (score desc, id asc); invalid entries (pos < 0, padding) last
__device__ __forceinline__ bool before(uint64_t ka, uint64_t ia, int64_t pa, uint64_t kb,
                                       uint64_t ib, int64_t pb) {
    if ((pa >= 0) != (pb >= 0)) return pa >= 0;
    return ka > kb || (ka == kb && ia < ib);
}

struct Threshold {
    uint64_t tp, tm, ip, im;
    int64_t id_rem;  // elements still needed from the boundary class (key and id prefix ties)
    bool use_id;
};

// Steps 1-2: the (score prefix, id prefix) threshold that admits exactly
// kk = min(k, nr) elements of the row.  Block-uniform result in *th.
__device__ void row_threshold(const RowView &rv, int64_t nr, int64_t kk, uint32_t *hist,
                              Threshold *th) {
    __shared__ uint64_t t_prefix, t_mask, i_prefix, i_mask;
    __shared__ int64_t t_rem, i_rem;
    __shared__ unsigned long long cnt;
    __shared__ int use_id;
    if (threadIdx.x == 0) {
        use_id = 0;
        i_prefix = 0;
        i_mask = 0;
    }
    if (kk > 0 && kk < nr) {
        radix_select<true>(
            nr, kk, [&](int64_t i) { return rv.key(i); }, [](int64_t) { return true; }, hist,
            &t_prefix, &t_mask, &t_rem);
        if (threadIdx.x == 0) cnt = 0;
        __syncthreads();
        const uint64_t tp = t_prefix, tm = t_mask;
        unsigned long long local = 0;
        for (int64_t i = threadIdx.x; i < nr; i += blockDim.x) local += ((rv.key(i) & tm) == tp);
        atomicAdd(&cnt, local);
        __syncthreads();
        if (static_cast<int64_t>(cnt) > t_rem) {  // more threshold ties than needed: lowest ids
            radix_select<false>(
                nr, t_rem, [&](int64_t i) { return rv.id(i); },
                [&](int64_t i) { return (rv.key(i) & tm) == tp; }, hist, &i_prefix, &i_mask,
                &i_rem);
            if (threadIdx.x == 0) use_id = 1;
        }
    } else if (threadIdx.x == 0) {
        t_prefix = 0;
        t_mask = 0;  // everything matches (key & 0) == 0 -> take all
        t_rem = nr;
    }
    __syncthreads();
    th->tp = t_prefix;
    th->tm = t_mask;
    th->ip = i_prefix;
    th->im = i_mask;
    th->use_id = use_id != 0;
    th->id_rem = use_id ? i_rem : 0;
}

// 0: out, 1: in, 2: boundary class -- same score prefix and same id prefix as
// the k-th element.  Boundary elements are admitted up to th.id_rem by a ticket
// counter: they are either exactly id_rem (the id select ended on a whole bin)
// or identical (key, id) duplicates (e.g. padding rows), so the pick among
// them does not change the output, and never more than k elements enter.
__device__ __forceinline__ int admitted(const Threshold &th, uint64_t key, const RowView &rv,
                                        int64_t i) {
    const uint64_t km = key & th.tm;
    if (km != th.tp) return km > th.tp ? 1 : 0;
    if (!th.use_id) return 1;
    const uint64_t idm = rv.id(i) & th.im;
    return idm < th.ip ? 1 : (idm == th.ip ? 2 : 0);
}

// Bitonic sort of p2 (power of two) triples in shared memory, "before" order.
__device__ void bitonic_smem(uint64_t *bkey, uint64_t *bid, int64_t *bpos, int p2) {
    for (int size = 2; size <= p2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < p2; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const bool i_first = before(bkey[i], bid[i], bpos[i], bkey[j], bid[j], bpos[j]);
                    if (i_first != up) {
                        const uint64_t tk = bkey[i], ti = bid[i];
                        const int64_t tpz = bpos[i];
                        bkey[i] = bkey[j]; bid[i] = bid[j]; bpos[i] = bpos[j];
                        bkey[j] = tk; bid[j] = ti; bpos[j] = tpz;
                    }
                }
            }
            __syncthreads();
        }
    }
}

__device__ __forceinline__ void write_out(const TopkArgs &a, int64_t row, int64_t i, bool valid,
                                          uint64_t key, uint64_t id, int64_t pos) {
    const int64_t o = row * a.out_ld + i;
    if (a.out_s) a.out_s[o] = valid ? from_okey(key) : -1.0;
    if (a.out_id) a.out_id[o] = valid ? id : ~0ull;
    if (a.out_pos) a.out_pos[o] = valid ? pos : -1;
}

__global__ void __launch_bounds__(kTopkThreads) topk_kernel(TopkArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    int cap = 1;  // winner buffer: pow2 >= k (at most k winners are collected)
    while (cap < a.k) cap <<= 1;
    uint64_t *bkey = reinterpret_cast<uint64_t *>(smem);
    uint64_t *bid = bkey + cap;
    int64_t *bpos = reinterpret_cast<int64_t *>(bid + cap);
    __shared__ uint32_t hist[256];
    __shared__ int cnt;
    __shared__ unsigned long long tickets;

    const int64_t row = blockIdx.x;
    RowView rv{a.scores + row * a.ld, a.ids, row, a.ids_ld, a.ix, a.ix_ld};
    int64_t nr = a.n;
    if (a.n_valid) nr = tmin<int64_t>(a.n, tmax<int64_t>(0, __ldg(a.n_valid + row)));
    const int64_t kk = tmin<int64_t>(a.k, nr);
    Threshold th;
    row_threshold(rv, nr, kk, hist, &th);
    if (threadIdx.x == 0) {
        cnt = 0;
        tickets = 0;
    }
    __syncthreads();
    if (kk > 0) {
        for (int64_t i = threadIdx.x; i < nr; i += blockDim.x) {
            const uint64_t key = rv.key(i);
            const int adm = admitted(th, key, rv, i);
            if (adm == 1 || (adm == 2 && static_cast<int64_t>(atomicAdd(&tickets, 1ull)) < th.id_rem)) {
                const int slot = atomicAdd(&cnt, 1);
                if (slot < cap) {
                    bkey[slot] = key;
                    bid[slot] = rv.id(i);
                    bpos[slot] = i;
                }
            }
        }
    }
    __syncthreads();
    const int m = tmin(cnt, cap);
    int p2 = 1;
    while (p2 < m) p2 <<= 1;
    for (int i = m + threadIdx.x; i < p2; i += blockDim.x) {  // sentinels sort last
        bkey[i] = 0;
        bid[i] = ~0ull;
        bpos[i] = -1;
    }
    __syncthreads();
    bitonic_smem(bkey, bid, bpos, p2);
    for (int i = threadIdx.x; i < a.k; i += blockDim.x) {
        const bool v = i < m;
        write_out(a, row, i, v, v ? bkey[i] : 0, v ? bid[i] : 0, v ? bpos[i] : -1);
    }
}

// Merge-path split: number of elements taken from run A among the first
// `diag` outputs of merge(A[0, na), B[0, nb)) ("before" order, A first on ties).
__device__ __forceinline__ int64_t merge_split(const uint64_t *ak, const uint64_t *ai,
                                               const int64_t *ap, int64_t na, const uint64_t *bk,
                                               const uint64_t *bi, const int64_t *bp, int64_t nb,
                                               int64_t diag) {
    int64_t lo = tmax<int64_t>(0, diag - nb), hi = tmin<int64_t>(diag, na);
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;  // take mid + 1 from A?  needs A[mid] <= B[diag-mid-1]
        const int64_t j = diag - mid - 1;
        if (!before(bk[j], bi[j], bp[j], ak[mid], ai[mid], ap[mid])) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(kTopkThreads) topk_large_kernel(TopkArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t *bkey = reinterpret_cast<uint64_t *>(smem);
    uint64_t *bid = bkey + kTopkRun;
    int64_t *bpos = reinterpret_cast<int64_t *>(bid + kTopkRun);
    __shared__ uint32_t hist[256];
    __shared__ unsigned long long cnt, tickets;

    const int64_t row = blockIdx.x;
    RowView rv{a.scores + row * a.ld, a.ids, row, a.ids_ld, a.ix, a.ix_ld};
    int64_t nr = a.n;
    if (a.n_valid) nr = tmin<int64_t>(a.n, tmax<int64_t>(0, __ldg(a.n_valid + row)));
    const int64_t kk = tmin<int64_t>(a.k, nr);
    Threshold th;
    row_threshold(rv, nr, kk, hist, &th);
    uint64_t *k0 = a.sk + row * 2 * a.run_cap, *k1 = k0 + a.run_cap;
    uint64_t *i0 = a.si + row * 2 * a.run_cap, *i1 = i0 + a.run_cap;
    int64_t *p0 = a.sp + row * 2 * a.run_cap, *p1 = p0 + a.run_cap;
    if (threadIdx.x == 0) {
        cnt = 0;
        tickets = 0;
    }
    __syncthreads();
    if (kk > 0) {
        for (int64_t i = threadIdx.x; i < nr; i += blockDim.x) {
            const uint64_t key = rv.key(i);
            const int adm = admitted(th, key, rv, i);
            if (adm == 1 || (adm == 2 && static_cast<int64_t>(atomicAdd(&tickets, 1ull)) < th.id_rem)) {
                const int64_t slot = static_cast<int64_t>(atomicAdd(&cnt, 1ull));
                if (slot < a.run_cap) {
                    k0[slot] = key;
                    i0[slot] = rv.id(i);
                    p0[slot] = i;
                }
            }
        }
    }
    __syncthreads();
    const int64_t m = tmin<int64_t>(static_cast<int64_t>(cnt), a.run_cap);
    // sorted runs of kTopkRun in shared memory
    for (int64_t r0 = 0; r0 < m; r0 += kTopkRun) {
        const int len = static_cast<int>(tmin<int64_t>(kTopkRun, m - r0));
        int p2 = 1;
        while (p2 < len) p2 <<= 1;
        for (int i = threadIdx.x; i < p2; i += blockDim.x) {
            const bool v = i < len;
            bkey[i] = v ? k0[r0 + i] : 0;
            bid[i] = v ? i0[r0 + i] : ~0ull;
            bpos[i] = v ? p0[r0 + i] : -1;
        }
        __syncthreads();
        bitonic_smem(bkey, bid, bpos, p2);
        for (int i = threadIdx.x; i < len; i += blockDim.x) {
            k0[r0 + i] = bkey[i];
            i0[r0 + i] = bid[i];
            p0[r0 + i] = bpos[i];
        }
        __syncthreads();
    }
    // pairwise merges of runs (ping-pong between the two scratch halves)
    for (int64_t w = kTopkRun; w < m; w <<= 1) {
        for (int64_t base = 0; base < m; base += 2 * w) {
            const int64_t na = tmin<int64_t>(w, m - base);
            const int64_t nb = tmin<int64_t>(w, tmax<int64_t>(0, m - base - w));
            const int64_t tot = na + nb;
            const int64_t per = (tot + blockDim.x - 1) / blockDim.x;
            const int64_t d0 = tmin<int64_t>(tot, threadIdx.x * per);
            const int64_t d1 = tmin<int64_t>(tot, d0 + per);
            const uint64_t *ak = k0 + base, *ai = i0 + base, *bk = k0 + base + w, *bi = i0 + base + w;
            const int64_t *ap = p0 + base, *bp = p0 + base + w;
            int64_t x = merge_split(ak, ai, ap, na, bk, bi, bp, nb, d0);
            int64_t y = d0 - x;
            for (int64_t o = d0; o < d1; ++o) {
                bool takeA;
                if (x >= na) takeA = false;
                else if (y >= nb) takeA = true;
                else takeA = !before(bk[y], bi[y], bp[y], ak[x], ai[x], ap[x]);
                const int64_t dst = base + o;
                if (takeA) {
                    k1[dst] = ak[x]; i1[dst] = ai[x]; p1[dst] = ap[x]; ++x;
                } else {
                    k1[dst] = bk[y]; i1[dst] = bi[y]; p1[dst] = bp[y]; ++y;
                }
            }
        }
        __syncthreads();
        uint64_t *tk = k0; k0 = k1; k1 = tk;
        uint64_t *ti = i0; i0 = i1; i1 = ti;
        int64_t *tq = p0; p0 = p1; p1 = tq;
    }
    for (int64_t i = threadIdx.x; i < a.k; i += blockDim.x) {
        const bool v = i < m;
        write_out(a, row, i, v, v ? k0[i] : 0, v ? i0[i] : 0, v ? p0[i] : -1);
    }
}

int topk_run(const TopkArgs &in, int64_t n_rows, cudaStream_t st) {
    TopkArgs a = in;
    DSRT_REQUIRE(a.k >= 1, DSRT_EINVAL, "invalid parameter: top_k must be >= 1, got %d", a.k);
    DSRT_REQUIRE(a.n >= 0 && a.ld >= a.n, DSRT_EINVAL, "invalid parameter: n=%lld ld=%lld",
                 (long long)a.n, (long long)a.ld);
    if (a.out_ld == 0) a.out_ld = a.k;
    DSRT_REQUIRE(a.out_ld >= a.k, DSRT_EINVAL, "invalid parameter: out_ld < k");
    if (n_rows == 0) return DSRT_OK;
    DSRT_REQUIRE(n_rows < (1LL << 31), DSRT_EUNSUPPORTED, "invalid parameter: too many rows");
    const size_t trip = 2 * sizeof(uint64_t) + sizeof(int64_t);
    if (a.k <= kTopkMax) {
        int cap = 1;
        while (cap < a.k) cap <<= 1;
        const size_t smem = static_cast<size_t>(cap) * trip;
        DSRT_CUDA(cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(kTopkMax * trip)));
        // short rows (candidate lists) in a large batch: small CTAs, several per SM; a small
        // batch keeps 1024 threads per row (latency)
        const int threads = (a.n <= 8192 && n_rows >= sm_count()) ? 256 : kTopkThreads;
        topk_kernel<<<static_cast<unsigned>(n_rows), threads, smem, st>>>(a);
        DSRT_LAUNCH_CHECK();
        return DSRT_OK;
    }
    // large k: the <= min(k, n) winners of a row in a global scratch (two halves)
    a.run_cap = tmax<int64_t>(1, tmin<int64_t>(a.k, a.n));
    const size_t elems = static_cast<size_t>(2 * a.run_cap) * static_cast<size_t>(n_rows);
    uint8_t *scratch = nullptr;
    DSRT_CUDA(malloc_async(reinterpret_cast<void **>(&scratch), elems * trip, st));
    a.sk = reinterpret_cast<uint64_t *>(scratch);
    a.si = a.sk + elems;
    a.sp = reinterpret_cast<int64_t *>(a.si + elems);
    DSRT_CUDA(cudaFuncSetAttribute(topk_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(kTopkRun * trip)));
    topk_large_kernel<<<static_cast<unsigned>(n_rows), kTopkThreads, kTopkRun * trip, st>>>(a);
    const cudaError_t e = cudaGetLastError();
    cudaFreeAsync(scratch, st);
    DSRT_CUDA(e);
    return DSRT_OK;
}

// plain rows (id = element index) for internal callers without the header struct
int topk_run_ext(const double *scores, int64_t ld, int64_t n, int k, double *out_s, uint64_t *out_id,
                 int64_t n_rows, cudaStream_t st) {
    TopkArgs a{};
    a.scores = scores;
    a.ld = ld;
    a.n = n;
    a.k = k;
    a.out_s = out_s;
    a.out_id = out_id;
    return topk_run(a, n_rows, st);
}

}  // namespace dsrt

using namespace dsrt;

extern "C" int dsrt_topk_max_k(void) { return kTopkMax; }

extern "C" int dsrt_topk(const double *scores, int64_t ld, const uint64_t *ids, int64_t ids_ld,
                         const int32_t *n_valid, int64_t n, int64_t n_rows, int k,
                         double *out_scores, uint64_t *out_ids, int64_t *out_pos, void *stream) {
    TopkArgs a{};
    a.scores = scores; a.ld = ld; a.ids = ids; a.ids_ld = ids_ld; a.n_valid = n_valid; a.n = n;
    a.k = k; a.out_s = out_scores; a.out_id = out_ids; a.out_pos = out_pos; a.out_ld = k;
    return topk_run(a, n_rows, as_stream(stream));
}

extern "C" int dsrt_topk_indexed(const double *scores, int64_t ld, const uint64_t *ids,
                                 const int64_t *id_index, int64_t id_index_ld, const int32_t *n_valid,
                                 int64_t n, int64_t n_rows, int k, double *out_scores, uint64_t *out_ids,
                                 int64_t *out_pos, void *stream) {
    DSRT_REQUIRE(ids != nullptr && id_index != nullptr, DSRT_EINVAL,
                 "invalid parameter: dsrt_topk_indexed needs ids and id_index");
    TopkArgs a{};
    a.scores = scores; a.ld = ld; a.ids = ids; a.ids_ld = 0; a.ix = id_index; a.ix_ld = id_index_ld;
    a.n_valid = n_valid; a.n = n; a.k = k; a.out_s = out_scores; a.out_id = out_ids;
    a.out_pos = out_pos; a.out_ld = k;
    return topk_run(a, n_rows, as_stream(stream));
}
