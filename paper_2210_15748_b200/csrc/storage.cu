// .dsri index files from / to the device layout.
//
// The reference serialises an index as a header, then per set its doc id
// and TinyTable bytes (sketch.py:192-239: 24-byte header m,L,r,flags,0;
// offsets (L, r+1) and ids (L, m), u8 or u16 little-endian by m), then the
// optional prefilter block: k, d, n_docs, float64 centroids, and per
// centroid a varint count followed by varint doc-id deltas
// (storage.py:130-173).
//
// Export: the sets section is written by one CTA per set; warp w builds
// table t = w, w+8, ... with a stable counting sort straight from the plane
// records (histogram in shared memory, warp scan, __match_any_sync ranking so
// ids stay ascending within a bucket) -- byte-identical to build_tiny_table.
// Postings are varint-encoded in parallel (length pass, scan, byte pass).
//
// Import: a host walk over the set headers (sizes only; sequential by
// nature), then device passes that validate every (set, table) -- offsets
// span 0..m and are monotone, ids are a permutation -- and decode the codes
// (code[ids[p]][t] = bucket of position p), and a parallel varint decoder
// for the postings.
#include <cstring>

#include "common.cuh"

namespace dsrt {

int exclusive_scan_i64(const int64_t *in, int64_t n, int64_t *out, void *ws, size_t ws_bytes,
                       cudaStream_t st);
size_t scan_ws_bytes(int64_t n);

constexpr int kStWarps = 8;
constexpr int kStMaxC = 12;  // counting-sort counters in shared memory: (r + 1) per warp

__device__ __forceinline__ void put_le(uint8_t *p, uint32_t v, int width) {
    p[0] = static_cast<uint8_t>(v);
    if (width == 2) p[1] = static_cast<uint8_t>(v >> 8);
}

__device__ __forceinline__ uint32_t get_le(const uint8_t *p, int width) {
    return width == 2 ? (static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8)) : p[0];
}

// code of vector v at table t from its plane record
__device__ __forceinline__ uint32_t record_code(const uint32_t *rec, int W, int C, int t) {
    uint32_t c = 0;
    for (int b = 0; b < C; ++b) c |= ((rec[b * W + (t >> 5)] >> (t & 31)) & 1u) << b;
    return c;
}

// warp-wide in-place inclusive scan of cnt[0..n), 32 entries per step
__device__ __forceinline__ void warp_inclusive_scan(uint32_t *cnt, int n) {
    const int lane = threadIdx.x & 31;
    uint32_t carry = 0;
    for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        uint32_t x = i < n ? cnt[i] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (i < n) cnt[i] = carry + x;
        carry += __shfl_sync(0xffffffffu, x, 31);
    }
    __syncwarp();
}

__global__ void __launch_bounds__(kStWarps * 32)
    dsri_sets_kernel(const uint32_t *__restrict__ recs, const int64_t *__restrict__ set_off,
                     const uint64_t *__restrict__ doc_ids, int64_t n_sets, int L, int C,
                     const int64_t *__restrict__ rec_off, uint8_t *__restrict__ out) {
    extern __shared__ uint32_t st_cnt[];
    const int64_t s = blockIdx.x;
    if (s >= n_sets) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = 1 << C, W = plane_words(L), R = record_words(L, C);
    const int64_t v0 = set_off[s];
    const int m = static_cast<int>(set_off[s + 1] - v0);
    const int ow = m <= 255 ? 1 : 2, iw = m <= 256 ? 1 : 2;
    uint8_t *base = out + rec_off[s];
    if (threadIdx.x == 0) {
        const uint64_t id = doc_ids[s];
        for (int i = 0; i < 8; ++i) base[i] = static_cast<uint8_t>(id >> (8 * i));
        const uint32_t hdr[4] = {static_cast<uint32_t>(m), static_cast<uint32_t>(L),
                                 static_cast<uint32_t>(r),
                                 static_cast<uint32_t>((ow == 2 ? 1 : 0) | (iw == 2 ? 2 : 0))};
        for (int f = 0; f < 4; ++f)
            for (int i = 0; i < 4; ++i) base[8 + 4 * f + i] = static_cast<uint8_t>(hdr[f] >> (8 * i));
        for (int i = 0; i < 8; ++i) base[24 + i] = 0;
    }
    uint8_t *offs = base + 32;
    uint8_t *ids = offs + static_cast<int64_t>(L) * (r + 1) * ow;
    uint32_t *cnt = st_cnt + warp * (r + 1);
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t *srec = recs + v0 * R;
    for (int t = warp; t < L; t += kStWarps) {
        for (int h = lane; h <= r; h += 32) cnt[h] = 0;
        __syncwarp();
        for (int j = lane; j < m; j += 32)
            atomicAdd(&cnt[record_code(srec + static_cast<int64_t>(j) * R, W, C, t) + 1], 1u);
        __syncwarp();
        // counts are shifted by one (code c at c + 1): the inclusive scan gives
        // cnt[h] = #codes < h = offsets[h], h = 0..r; cnt[c] is then c's cursor
        warp_inclusive_scan(cnt, r + 1);
        for (int h = lane; h <= r; h += 32)
            put_le(offs + (static_cast<int64_t>(t) * (r + 1) + h) * ow, cnt[h], ow);
        __syncwarp();
        // stable placement: ascending j in chunks of 32, rank by __match_any_sync
        for (int j0 = 0; j0 < m; j0 += 32) {
            const int j = j0 + lane;
            const bool ok = j < m;
            const uint32_t code = ok ? record_code(srec + static_cast<int64_t>(j) * R, W, C, t)
                                     : static_cast<uint32_t>(r) + 1u + lane;
            const unsigned peers = __match_any_sync(0xffffffffu, code);
            uint32_t before = 0;
            if (ok) before = cnt[code];
            __syncwarp();
            if (ok && (peers & lt) == 0) cnt[code] = before + __popc(peers);
            __syncwarp();
            if (ok)
                put_le(ids + (static_cast<int64_t>(t) * m + before + __popc(peers & lt)) * iw,
                       static_cast<uint32_t>(j), iw);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- import
// status codes of the device validation (the reference's checks, in order)
enum : int { kOkSet = 0, kBadSpan = 1, kBadMonotone = 2, kBadPerm = 3 };

// warp per (set, table): validate and decode codes.  first_bad: atomicMin of
// (set << 2 | kind) over failing sets.
__global__ void __launch_bounds__(kStWarps * 32)
    dsri_decode_kernel(const uint8_t *__restrict__ buf, const int64_t *__restrict__ tt_off,
                       const int64_t *__restrict__ set_off, int64_t n_sets, int L, int r,
                       uint8_t *__restrict__ codes, int code_bytes, int words_per_warp,
                       unsigned long long *__restrict__ first_bad) {
    extern __shared__ uint32_t st_seen[];  // per warp: ceil(m_max / 32) words
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t item = static_cast<int64_t>(blockIdx.x) * kStWarps + warp;
    if (item >= n_sets * L) return;
    const int64_t s = item / L;
    const int t = static_cast<int>(item - s * L);
    const int64_t v0 = set_off[s];
    const int m = static_cast<int>(set_off[s + 1] - v0);
    const int ow = m <= 255 ? 1 : 2, iw = m <= 256 ? 1 : 2;
    const uint8_t *offs = buf + tt_off[s] + 24 + static_cast<int64_t>(t) * (r + 1) * ow;
    const uint8_t *ids = buf + tt_off[s] + 24 + static_cast<int64_t>(L) * (r + 1) * ow +
                         static_cast<int64_t>(t) * m * iw;
    // offsets span 0..m (all tables are checked before monotonicity in the
    // reference; per-table kinds are merged by taking the smallest kind)
    int kind = kOkSet;
    if (get_le(offs, ow) != 0 || get_le(offs + static_cast<int64_t>(r) * ow, ow) != static_cast<uint32_t>(m))
        kind = kBadSpan;
    bool mono = true;
    for (int h = lane; h < r; h += 32)
        if (get_le(offs + static_cast<int64_t>(h + 1) * ow, ow) < get_le(offs + static_cast<int64_t>(h) * ow, ow))
            mono = false;
    if (!__all_sync(0xffffffffu, mono) && kind == kOkSet) kind = kBadMonotone;
    // permutation: bitmap of seen ids
    const int nw = (m + 31) / 32;
    uint32_t *seen = st_seen + static_cast<int64_t>(warp) * words_per_warp;
    bool perm_ok = true;
    if (kind == kOkSet) {
        for (int i = lane; i < nw; i += 32) seen[i] = 0;
        __syncwarp();
        for (int p = lane; p < m; p += 32) {
            const uint32_t id = get_le(ids + static_cast<int64_t>(p) * iw, iw);
            if (id >= static_cast<uint32_t>(m)) {
                perm_ok = false;
            } else {
                const uint32_t old = atomicOr(&seen[id >> 5], 1u << (id & 31));
                if (old & (1u << (id & 31))) perm_ok = false;
            }
        }
        if (!__all_sync(0xffffffffu, perm_ok)) kind = kBadPerm;
    }
    if (kind != kOkSet) {
        if (lane == 0) atomicMin(first_bad, (static_cast<unsigned long long>(s) << 2) | kind);
        return;
    }
    // decode: position p lies in bucket h with offs[h] <= p < offs[h+1]
    for (int p = lane; p < m; p += 32) {
        int lo = 0, hi = r;  // find the last h with offs[h] <= p
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (get_le(offs + static_cast<int64_t>(mid) * ow, ow) <= static_cast<uint32_t>(p)) lo = mid;
            else hi = mid;
        }
        const uint32_t id = get_le(ids + static_cast<int64_t>(p) * iw, iw);
        uint8_t *dst = codes + ((v0 + id) * L + t) * code_bytes;
        for (int b = 0; b < code_bytes; ++b) dst[b] = static_cast<uint8_t>(lo >> (8 * b));
    }
}

// ---------------------------------------------------------------- varints
__device__ __forceinline__ int varint_len(uint64_t v) {
    int n = 1;
    while (v >= 0x80) {
        v >>= 7;
        ++n;
    }
    return n;
}

// values of the postings block: [count_c, deltas of c ...] per centroid
__global__ void post_values_kernel(const int64_t *__restrict__ post_off, const int64_t *__restrict__ docs,
                                   int64_t k, int64_t total, int64_t *__restrict__ vals) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= k + total) return;
    // element i of the value stream: find centroid c with post_off[c] + c <= i
    int64_t lo = 0, hi = k;  // last c with post_off[c] + c <= i
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (post_off[mid] + mid <= i) lo = mid;
        else hi = mid;
    }
    const int64_t c = lo, start = post_off[c] + c;
    if (i == start) {
        vals[i] = post_off[c + 1] - post_off[c];
    } else {
        const int64_t e = post_off[c] + (i - start - 1);
        vals[i] = docs[e] - (e > post_off[c] ? docs[e - 1] : 0);
    }
}

__global__ void varint_len_kernel(const int64_t *__restrict__ vals, int64_t n, int64_t *__restrict__ lens,
                                  uint32_t *__restrict__ neg) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    if (vals[i] < 0) atomicOr(neg, 1u);
    lens[i] = varint_len(static_cast<uint64_t>(vals[i]));
}

__global__ void varint_write_kernel(const int64_t *__restrict__ vals, const int64_t *__restrict__ pos,
                                    int64_t n, uint8_t *__restrict__ out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    uint64_t v = static_cast<uint64_t>(vals[i]);
    uint8_t *p = out + pos[i];
    while (v >= 0x80) {
        *p++ = static_cast<uint8_t>((v & 0x7f) | 0x80);
        v >>= 7;
    }
    *p = static_cast<uint8_t>(v);
}

// decode: is_end[i] = byte i terminates a varint
__global__ void varint_ends_kernel(const uint8_t *__restrict__ b, int64_t n, int64_t *__restrict__ is_end) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) is_end[i] = (b[i] & 0x80) ? 0 : 1;
}

// value of the varint ending at byte i -> vals[rank[i]]; overflow (> 63 bits) flagged
__global__ void varint_decode_kernel(const uint8_t *__restrict__ b, int64_t n, const int64_t *__restrict__ rank,
                                     int64_t *__restrict__ vals, uint32_t *__restrict__ bad) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n || (b[i] & 0x80)) return;
    int64_t s = i;
    while (s > 0 && (b[s - 1] & 0x80)) --s;
    if (i - s >= 9) {
        atomicOr(bad, 1u);
        vals[rank[i]] = 0;
        return;
    }
    uint64_t v = 0;
    for (int64_t j = i; j >= s; --j) v = (v << 7) | (b[j] & 0x7f);
    vals[rank[i]] = static_cast<int64_t>(v);
}

// sequential walk of the counts: seg[c] = start of centroid c's values
__global__ void post_walk_kernel(const int64_t *__restrict__ vals, int64_t n_vals, int64_t k,
                                 int64_t *__restrict__ seg, int64_t *__restrict__ status) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    int64_t s = 0;
    for (int64_t c = 0; c < k; ++c) {
        if (s >= n_vals) {
            status[0] = 1;  // truncated
            return;
        }
        const int64_t cnt = vals[s];
        seg[c] = s;
        if (cnt < 0 || s + 1 + cnt > n_vals) {
            status[0] = 1;
            return;
        }
        s += 1 + cnt;
    }
    seg[k] = s;
    status[0] = 0;
}

__global__ void post_off_kernel(const int64_t *__restrict__ seg, int64_t k, int64_t *__restrict__ post_off) {
    const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (c <= k) post_off[c] = seg[c] - c;
}

// deltas of centroid c sit at vals[seg[c] + 1 ...]; docs = running sums per centroid
__global__ void post_docs_kernel(const int64_t *__restrict__ vals, const int64_t *__restrict__ seg,
                                 const int64_t *__restrict__ post_off, int64_t k, int64_t *__restrict__ docs) {
    const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (c >= k) return;
    int64_t prev = 0;
    const int64_t n = post_off[c + 1] - post_off[c];
    for (int64_t j = 0; j < n; ++j) {
        prev += vals[seg[c] + 1 + j];
        docs[post_off[c] + j] = prev;
    }
}

}  // namespace dsrt

using namespace dsrt;

// ----------------------------------------------------------------- export ABI
extern "C" int dsrt_dsri_write_sets(const uint32_t *records, const int64_t *set_off,
                                    const uint64_t *doc_ids, int64_t n_sets, int L, int C,
                                    const int64_t *rec_off, uint8_t *out, void *stream) {
    DSRT_REQUIRE(L >= 1 && C >= 1, DSRT_EINVAL, "invalid parameter: L=%d C=%d", L, C);
    DSRT_REQUIRE(C <= kStMaxC, DSRT_EUNSUPPORTED, "invalid parameter: device TinyTable export needs C <= %d",
                 kStMaxC);
    if (n_sets == 0) return DSRT_OK;
    cudaStream_t st = as_stream(stream);
    const size_t smem = static_cast<size_t>(kStWarps) * ((1 << C) + 1) * sizeof(uint32_t);
    DSRT_CUDA(cudaFuncSetAttribute(dsri_sets_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    DSRT_REQUIRE(n_sets < (1LL << 31), DSRT_EUNSUPPORTED, "invalid parameter: too many sets");
    dsri_sets_kernel<<<static_cast<unsigned>(n_sets), kStWarps * 32, smem, st>>>(records, set_off, doc_ids,
                                                                              n_sets, L, C, rec_off, out);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}

// workspace for n values: vals (n), lens/positions (n + 1), scan tiles, flags
extern "C" size_t dsrt_varint_workspace(int64_t n_vals) {
    return static_cast<size_t>(2 * n_vals + 2) * 8 + scan_ws_bytes(n_vals + 1) + 256;
}

// postings CSR -> varint bytes; *n_bytes (host) = encoded length.  out may be
// NULL to query the length only.
extern "C" int dsrt_postings_to_varints(const int64_t *post_off, const int64_t *post_docs, int64_t k,
                                        int64_t total, uint8_t *out, int64_t *n_bytes, void *workspace,
                                        size_t ws_bytes, void *stream) {
    DSRT_REQUIRE(k >= 0 && total >= 0, DSRT_EINVAL, "invalid parameter: negative size");
    const int64_t n = k + total;
    DSRT_REQUIRE(ws_bytes >= dsrt_varint_workspace(n), DSRT_EINVAL, "invalid parameter: workspace too small");
    *n_bytes = 0;
    if (n == 0) return DSRT_OK;
    cudaStream_t st = as_stream(stream);
    uint8_t *w = static_cast<uint8_t *>(workspace);
    int64_t *vals = reinterpret_cast<int64_t *>(w);
    int64_t *pos = vals + n;  // lengths, then (in place) byte positions; n + 1 entries
    void *sws = pos + n + 1;
    uint32_t *neg = reinterpret_cast<uint32_t *>(static_cast<uint8_t *>(sws) + scan_ws_bytes(n + 1));
    DSRT_CUDA(cudaMemsetAsync(neg, 0, 4, st));
    const unsigned b = static_cast<unsigned>((n + 255) / 256);
    post_values_kernel<<<b, 256, 0, st>>>(post_off, post_docs, k, total, vals);
    varint_len_kernel<<<b, 256, 0, st>>>(vals, n, pos, neg);
    DSRT_LAUNCH_CHECK();
    int rc = exclusive_scan_i64(pos, n, pos, sws, scan_ws_bytes(n + 1), st);
    if (rc) return rc;
    int64_t tot = 0;
    uint32_t hneg = 0;
    DSRT_CUDA(cudaMemcpyAsync(&tot, pos + n, 8, cudaMemcpyDeviceToHost, st));
    DSRT_CUDA(cudaMemcpyAsync(&hneg, neg, 4, cudaMemcpyDeviceToHost, st));
    DSRT_CUDA(cudaStreamSynchronize(st));
    DSRT_REQUIRE(hneg == 0, DSRT_EINVAL, "invalid parameter: postings not ascending");
    *n_bytes = tot;
    if (out == nullptr) return DSRT_OK;
    varint_write_kernel<<<b, 256, 0, st>>>(vals, pos, n, out);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}

// ----------------------------------------------------------------- import ABI
// Host walk over the sets section (no GPU): per set its doc id, m, and the
// byte offset of its TinyTable; stops at the first set whose header fails a
// check (the reference's order, storage.py:222-235 + sketch.py:209-223).
// Returns the number of sets parsed; *err_kind: 0 ok, 1 doc id truncated,
// 2 header truncated, 3 payload truncated, 4 bad dimensions, 5 width flags,
// 6 shape differs from the config (payload complete; the caller validates it
// first, as the reference does).  hdr_out: (m, L, r, flags) of the failing
// set; *end_pos: the failing set's TinyTable position, or the section end.
extern "C" int64_t dsrt_dsri_scan_sets(const uint8_t *buf, size_t len, size_t pos, int64_t n_sets,
                                       int L, int C, uint64_t *doc_ids, int64_t *sizes,
                                       int64_t *tt_off, uint32_t *hdr_out, int *err_kind,
                                       size_t *end_pos) {
    const uint32_t r_cfg = 1u << C;
    *err_kind = 0;
    for (int64_t i = 0; i < n_sets; ++i) {
        if (len - pos < 8) { *err_kind = 1; *end_pos = pos; return i; }
        uint64_t id;
        std::memcpy(&id, buf + pos, 8);  // little-endian host
        doc_ids[i] = id;
        pos += 8;
        *end_pos = pos;
        if (len - pos < 24) { *err_kind = 2; return i; }
        uint32_t h[4];
        std::memcpy(h, buf + pos, 16);
        for (int f = 0; f < 4; ++f) hdr_out[f] = h[f];
        const uint32_t m = h[0], l = h[1], r = h[2], flags = h[3];
        if (m < 1 || l < 1 || r < 1) { *err_kind = 4; return i; }
        const int ow = (flags & 1) ? 2 : 1, iw = (flags & 2) ? 2 : 1;
        if (ow != (m <= 255 ? 1 : 2) || iw != (m <= 256 ? 1 : 2)) { *err_kind = 5; return i; }
        const size_t payload = static_cast<size_t>(l) * (static_cast<size_t>(r) + 1) * ow +
                               static_cast<size_t>(l) * m * iw;
        if (len - pos - 24 < payload) { *err_kind = 3; return i; }
        if (l != static_cast<uint32_t>(L) || r != r_cfg) { *err_kind = 6; return i; }
        tt_off[i] = static_cast<int64_t>(pos);
        sizes[i] = m;
        pos += 24 + payload;
    }
    *end_pos = pos;
    return n_sets;
}

extern "C" int dsrt_dsri_decode_sets(const uint8_t *buf, const int64_t *tt_off, const int64_t *set_off,
                                     int64_t n_sets, int L, int C, int64_t m_max, void *codes,
                                     int code_bytes, int64_t *first_bad, void *stream) {
    DSRT_REQUIRE(L >= 1 && C >= 1 && C <= 24, DSRT_EINVAL, "invalid parameter: L=%d C=%d", L, C);
    DSRT_REQUIRE(code_bytes == 1 || code_bytes == 2 || code_bytes == 4, DSRT_EINVAL,
                 "invalid parameter: code width %d", code_bytes);
    *first_bad = -1;
    if (n_sets == 0) return DSRT_OK;
    cudaStream_t st = as_stream(stream);
    unsigned long long *fb = nullptr;
    DSRT_CUDA(malloc_async(reinterpret_cast<void **>(&fb), 8, st));
    DSRT_CUDA(cudaMemsetAsync(fb, 0xff, 8, st));
    const int wpw = static_cast<int>((m_max + 31) / 32);
    const size_t smem = static_cast<size_t>(kStWarps) * wpw * 4;
    DSRT_REQUIRE(smem <= 200 * 1024, DSRT_EUNSUPPORTED, "invalid parameter: set too large to decode");
    DSRT_CUDA(cudaFuncSetAttribute(dsri_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t items = n_sets * L;
    dsri_decode_kernel<<<static_cast<unsigned>((items + kStWarps - 1) / kStWarps), kStWarps * 32, smem, st>>>(
        buf, tt_off, set_off, n_sets, L, 1 << C, static_cast<uint8_t *>(codes), code_bytes, wpw, fb);
    DSRT_LAUNCH_CHECK();
    unsigned long long h = 0;
    DSRT_CUDA(cudaMemcpyAsync(&h, fb, 8, cudaMemcpyDeviceToHost, st));
    DSRT_CUDA(cudaStreamSynchronize(st));
    cudaFreeAsync(fb, st);
    *first_bad = h == ~0ull ? -1 : static_cast<int64_t>(h);
    return DSRT_OK;
}

// varint bytes -> postings CSR (k centroids).  post_off (k+1); post_docs must
// hold the total (<= n_bytes).  *total_out = number of postings; truncated
// streams return DSRT_ERANGE.
extern "C" int dsrt_varints_to_postings(const uint8_t *bytes, int64_t n_bytes, int64_t k, int64_t *post_off,
                                        int64_t *post_docs, int64_t *total_out, void *workspace,
                                        size_t ws_bytes, void *stream) {
    DSRT_REQUIRE(ws_bytes >= dsrt_varint_workspace(n_bytes) + static_cast<size_t>(k + 2) * 8, DSRT_EINVAL,
                 "invalid parameter: workspace too small");
    cudaStream_t st = as_stream(stream);
    uint8_t *w = static_cast<uint8_t *>(workspace);
    int64_t *vals = reinterpret_cast<int64_t *>(w);       // <= n_bytes values
    int64_t *is_end = vals + n_bytes;                       // n_bytes + 1 (scanned in place)
    void *sws = is_end + n_bytes + 1;
    uint32_t *bad = reinterpret_cast<uint32_t *>(static_cast<uint8_t *>(sws) + scan_ws_bytes(n_bytes + 1));
    int64_t *status = reinterpret_cast<int64_t *>(bad + 2);
    int64_t *seg = reinterpret_cast<int64_t *>(w + dsrt_varint_workspace(n_bytes));
    DSRT_CUDA(cudaMemsetAsync(bad, 0, 16, st));
    const unsigned b = static_cast<unsigned>((n_bytes + 255) / 256 + 1);
    int64_t n_vals = 0;
    if (n_bytes > 0) {
        varint_ends_kernel<<<b, 256, 0, st>>>(bytes, n_bytes, is_end);
        DSRT_LAUNCH_CHECK();
        int rc = exclusive_scan_i64(is_end, n_bytes, is_end, sws, scan_ws_bytes(n_bytes + 1), st);
        if (rc) return rc;
        varint_decode_kernel<<<b, 256, 0, st>>>(bytes, n_bytes, is_end, vals, bad);
        DSRT_LAUNCH_CHECK();
        DSRT_CUDA(cudaMemcpyAsync(&n_vals, is_end + n_bytes, 8, cudaMemcpyDeviceToHost, st));
    }
    post_walk_kernel<<<1, 1, 0, st>>>(vals, n_vals, k, seg, status);
    int64_t hs = 1;
    uint32_t hb = 0;
    DSRT_CUDA(cudaMemcpyAsync(&hs, status, 8, cudaMemcpyDeviceToHost, st));
    DSRT_CUDA(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, st));
    DSRT_CUDA(cudaStreamSynchronize(st));
    DSRT_REQUIRE(hb == 0, DSRT_EINVAL, "corrupt postings: varint too long");
    DSRT_REQUIRE(hs == 0, DSRT_ERANGE, "truncated postings");
    const unsigned bk = static_cast<unsigned>((k + 256) / 256);
    post_off_kernel<<<bk, 256, 0, st>>>(seg, k, post_off);
    post_docs_kernel<<<bk, 256, 0, st>>>(vals, seg, post_off, k, post_docs);
    DSRT_LAUNCH_CHECK();
    DSRT_CUDA(cudaMemcpyAsync(total_out, post_off + k, 8, cudaMemcpyDeviceToHost, st));
    DSRT_CUDA(cudaStreamSynchronize(st));
    return DSRT_OK;
}
