// K4 -- batched top-k by (score desc, doc_id asc).
//
// Replaces heapq.nsmallest(top_k, ((score, doc_id) ...), key=lambda e:
// (-e[0], e[1])) in query() (index.py:314-319).  One CTA per row (query set):
//  1. MSB radix select (8-bit digits) on the float64 bit pattern (scores are
//     >= 0, so the IEEE pattern is monotone) -> threshold prefix T and the
//     number of T-ties still needed;
//  2. if more ties than needed: radix select on doc_id (ascending) among the
//     ties (reference tie-break: lower doc id first);
//  3. compact the k winners into shared memory and bitonic-sort them by
//     (score desc, doc_id asc).
#include "common.cuh"

namespace dsrt {

constexpr int kTopkThreads = 1024;
constexpr int kTopkMax = 4096;

struct RowView {
    const double *s;
    const uint64_t *ids;
    int64_t row, ids_ld;
    const int64_t *ix = nullptr;  // optional per-row index into ids (candidate lists)
    int64_t ix_ld = 0;
    __device__ __forceinline__ uint64_t key(int64_t i) const {
        return static_cast<uint64_t>(__double_as_longlong(__ldg(s + i)));
    }
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

__device__ __forceinline__ bool before(uint64_t ka, uint64_t ia, uint64_t kb, uint64_t ib) {
    // (score desc, id asc)
    return ka > kb || (ka == kb && ia < ib);
}

__global__ void __launch_bounds__(kTopkThreads)
    topk_kernel(const double *__restrict__ scores, int64_t ld, const uint64_t *__restrict__ ids,
                int64_t ids_ld, const int32_t *__restrict__ n_valid, int64_t n, int k,
                double *__restrict__ out_s, uint64_t *__restrict__ out_id,
                int64_t *__restrict__ out_pos, const int64_t *__restrict__ ix, int64_t ix_ld) {
    extern __shared__ __align__(16) uint8_t smem[];
    int cap = 1;  // winner buffer: pow2 >= k (at most k winners are collected)
    while (cap < k) cap <<= 1;
    uint64_t *bkey = reinterpret_cast<uint64_t *>(smem);
    uint64_t *bid = bkey + cap;
    int64_t *bpos = reinterpret_cast<int64_t *>(bid + cap);
    __shared__ uint32_t hist[256];
    __shared__ uint64_t t_prefix, t_mask, i_prefix, i_mask;
    __shared__ int64_t t_rem, i_rem;
    __shared__ int cnt;

    const int64_t row = blockIdx.x;
    RowView rv{scores + row * ld, ids, row, ids_ld, ix, ix_ld};
    int64_t nr = n;
    if (n_valid) nr = tmin<int64_t>(n, tmax<int64_t>(0, __ldg(n_valid + row)));
    const int64_t kk = tmin<int64_t>(k, nr);

    bool use_id_filter = false;
    if (kk > 0 && kk < nr) {
        radix_select<true>(
            nr, kk, [&](int64_t i) { return rv.key(i); }, [](int64_t) { return true; }, hist,
            &t_prefix, &t_mask, &t_rem);
        // how many elements tie with the threshold bin?
        if (threadIdx.x == 0) cnt = 0;
        __syncthreads();
        const uint64_t tp = t_prefix, tm = t_mask;
        int local = 0;
        for (int64_t i = threadIdx.x; i < nr; i += blockDim.x) local += ((rv.key(i) & tm) == tp);
        atomicAdd(&cnt, local);
        __syncthreads();
        if (cnt > t_rem) {
            use_id_filter = true;
            radix_select<false>(
                nr, t_rem, [&](int64_t i) { return rv.id(i); },
                [&](int64_t i) { return (rv.key(i) & tm) == tp; }, hist, &i_prefix, &i_mask,
                &i_rem);
        }
    } else if (threadIdx.x == 0) {
        t_prefix = 0;
        t_mask = 0;  // everything matches (key & 0) == 0 -> take all
        t_rem = nr;
    }
    __syncthreads();
    // collect winners
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    const uint64_t tp = t_prefix, tm = t_mask, ip = i_prefix, im = i_mask;
    if (kk > 0) {
        for (int64_t i = threadIdx.x; i < nr; i += blockDim.x) {
            const uint64_t key = rv.key(i);
            const uint64_t km = key & tm;
            bool take = km > tp;
            if (km == tp) {
                if (!use_id_filter) {
                    take = true;
                } else {
                    const uint64_t idm = rv.id(i) & im;
                    take = idm <= ip;
                }
            }
            if (take) {
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
    // bitonic sort, "before" order; sentinel pos -1 forced last
    for (int size = 2; size <= p2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < p2; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const bool vi = bpos[i] >= 0, vj = bpos[j] >= 0;
                    bool i_first;
                    if (vi != vj)
                        i_first = vi;
                    else
                        i_first = before(bkey[i], bid[i], bkey[j], bid[j]);
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
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        const int64_t o = row * static_cast<int64_t>(k) + i;
        if (i < m) {
            if (out_s) out_s[o] = __longlong_as_double(static_cast<long long>(bkey[i]));
            if (out_id) out_id[o] = bid[i];
            if (out_pos) out_pos[o] = bpos[i];
        } else {
            if (out_s) out_s[o] = -1.0;
            if (out_id) out_id[o] = ~0ull;
            if (out_pos) out_pos[o] = -1;
        }
    }
}

}  // namespace dsrt

using namespace dsrt;

extern "C" int dsrt_topk_max_k(void) { return kTopkMax; }

static int topk_launch(const double *scores, int64_t ld, const uint64_t *ids, int64_t ids_ld,
                       const int64_t *ix, int64_t ix_ld, const int32_t *n_valid, int64_t n, int64_t n_rows,
                       int k, double *out_scores, uint64_t *out_ids, int64_t *out_pos, void *stream) {
    DSRT_REQUIRE(k >= 1, DSRT_EINVAL, "invalid parameter: top_k must be >= 1, got %d", k);
    DSRT_REQUIRE(k <= kTopkMax, DSRT_EUNSUPPORTED,
                 "invalid parameter: top_k=%d exceeds the device top-k limit %d", k, kTopkMax);
    DSRT_REQUIRE(n >= 0 && ld >= n, DSRT_EINVAL, "invalid parameter: n=%lld ld=%lld",
                 (long long)n, (long long)ld);
    if (n_rows == 0) return DSRT_OK;
    DSRT_REQUIRE(n_rows < (1LL << 31), DSRT_EUNSUPPORTED, "invalid parameter: too many rows");
    int cap = 1;
    while (cap < k) cap <<= 1;
    const size_t smem = static_cast<size_t>(cap) * (2 * sizeof(uint64_t) + sizeof(int64_t));
    DSRT_CUDA(cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(kTopkMax * (2 * sizeof(uint64_t) + sizeof(int64_t)))));
    // short rows (candidate lists) in a large batch: small CTAs, several per SM; a small
    // batch keeps 1024 threads per row (latency)
    const int threads = (n <= 8192 && n_rows >= sm_count()) ? 256 : kTopkThreads;
    topk_kernel<<<static_cast<unsigned>(n_rows), threads, smem, as_stream(stream)>>>(
        scores, ld, ids, ids_ld, n_valid, n, k, out_scores, out_ids, out_pos, ix, ix_ld);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}

extern "C" int dsrt_topk(const double *scores, int64_t ld, const uint64_t *ids, int64_t ids_ld,
                         const int32_t *n_valid, int64_t n, int64_t n_rows, int k,
                         double *out_scores, uint64_t *out_ids, int64_t *out_pos, void *stream) {
    return topk_launch(scores, ld, ids, ids_ld, nullptr, 0, n_valid, n, n_rows, k, out_scores, out_ids,
                       out_pos, stream);
}

extern "C" int dsrt_topk_indexed(const double *scores, int64_t ld, const uint64_t *ids,
                                 const int64_t *id_index, int64_t id_index_ld, const int32_t *n_valid,
                                 int64_t n, int64_t n_rows, int k, double *out_scores, uint64_t *out_ids,
                                 int64_t *out_pos, void *stream) {
    DSRT_REQUIRE(ids != nullptr && id_index != nullptr, DSRT_EINVAL,
                 "invalid parameter: dsrt_topk_indexed needs ids and id_index");
    return topk_launch(scores, ld, ids, 0, id_index, id_index_ld, n_valid, n, n_rows, k, out_scores, out_ids,
                       out_pos, stream);
}
