// Centroid -> document postings from per-vector assignments (the inversion
// step of build_centroid_index, prefilter.py:85-108): posting c lists each
// document with a vector assigned to c exactly once, in ascending document
// index.  Device counting sort: stable radix sort of vectors by centroid
// (vector order is document order, so each bucket is document-ascending),
// drop repeats of the same document inside a bucket, compact with a scan.
#include "common.cuh"

namespace dsrt {

int exclusive_scan_i64(const int64_t *in, int64_t n, int64_t *out, void *ws, size_t ws_bytes,
                       cudaStream_t st);
size_t scan_ws_bytes(int64_t n);
size_t radix_sort_ws(int64_t n);
int radix_sort_perm(const int64_t *keys, int64_t n, int key_bits, int64_t *perm_out, void *ws,
                    size_t ws_bytes, cudaStream_t st);

__global__ void doc_of_vec_kernel(const int64_t *__restrict__ set_off, int64_t n_docs,
                                  int64_t *__restrict__ doc_of) {
    const int64_t doc = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
    if (doc >= n_docs) return;
    for (int64_t v = set_off[doc] + (threadIdx.x & 31); v < set_off[doc + 1]; v += 32) doc_of[v] = doc;
}

__global__ void keys_from_assign_kernel(const int32_t *__restrict__ assign, int64_t n, int64_t k_c,
                                        int64_t *__restrict__ keys, uint32_t *bad) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int32_t c = assign[i];
    if (c < 0 || c >= k_c) {
        atomicAdd(bad, 1u);
        keys[i] = 0;
    } else {
        keys[i] = c;
    }
}

// keep[i] = first occurrence of (centroid, doc) in sorted order; per-centroid unique counts
__global__ void keep_kernel(const int64_t *__restrict__ keys, const int64_t *__restrict__ perm,
                            const int64_t *__restrict__ doc_of, int64_t n, int64_t *__restrict__ keep,
                            unsigned long long *__restrict__ ucount) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int64_t v = perm[i];
    const int64_t c = keys[v], doc = doc_of[v];
    bool k = true;
    if (i > 0) {
        const int64_t pv = perm[i - 1];
        k = keys[pv] != c || doc_of[pv] != doc;
    }
    keep[i] = k ? 1 : 0;
    if (k) atomicAdd(ucount + c, 1ull);
}

__global__ void compact_kernel(const int64_t *__restrict__ perm, const int64_t *__restrict__ doc_of,
                               const int64_t *__restrict__ keep, const int64_t *__restrict__ pos,
                               int64_t n, int64_t *__restrict__ post_docs, int64_t *__restrict__ n_post) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    if (keep[i]) post_docs[pos[i]] = doc_of[perm[i]];
    if (i == n - 1) *n_post = pos[i] + keep[i];
}

static size_t al(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

// block per centroid: old posting, then the added one (add ids > old ids)
__global__ void merge_postings_kernel(const int64_t *__restrict__ old_off, const int64_t *__restrict__ old_docs,
                                      const int64_t *__restrict__ add_off, const int64_t *__restrict__ add_docs,
                                      int64_t k_c, int64_t *__restrict__ new_off, int64_t *__restrict__ new_docs) {
    const int64_t c = blockIdx.x;
    if (c >= k_c) return;
    const int64_t o0 = old_off[c], o1 = old_off[c + 1], a0 = add_off[c], a1 = add_off[c + 1];
    const int64_t dst = o0 + a0;  // (old start) + (added start) = merged start
    if (threadIdx.x == 0) {
        new_off[c] = dst;
        if (c == k_c - 1) new_off[k_c] = o1 + a1;
    }
    for (int64_t i = threadIdx.x; i < o1 - o0; i += blockDim.x) new_docs[dst + i] = old_docs[o0 + i];
    for (int64_t i = threadIdx.x; i < a1 - a0; i += blockDim.x) new_docs[dst + (o1 - o0) + i] = add_docs[a0 + i];
}

}  // namespace dsrt

using namespace dsrt;

extern "C" int dsrt_merge_postings(const int64_t *old_off, const int64_t *old_docs, const int64_t *add_off,
                                   const int64_t *add_docs, int64_t k_c, int64_t *new_off, int64_t *new_docs,
                                   void *stream) {
    DSRT_REQUIRE(k_c >= 1 && k_c < (1LL << 31), DSRT_EINVAL, "invalid parameter: k=%lld", (long long)k_c);
    merge_postings_kernel<<<static_cast<unsigned>(k_c), 128, 0, as_stream(stream)>>>(
        old_off, old_docs, add_off, add_docs, k_c, new_off, new_docs);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}

extern "C" size_t dsrt_postings_workspace(int64_t n_vec, int64_t k_c) {
    const size_t n8 = al(static_cast<size_t>(n_vec + 1) * 8);
    return 5 * n8 + al(static_cast<size_t>(k_c) * 8) + al(scan_ws_bytes(n_vec + 1)) +
           al(scan_ws_bytes(k_c + 1)) + radix_sort_ws(n_vec) + 256;
}

extern "C" int dsrt_postings_from_assign(const int32_t *assign, int64_t n_vec, const int64_t *set_off,
                                         int64_t n_docs, int64_t k_c, int64_t *post_off,
                                         int64_t *post_docs, int64_t *n_post, void *workspace,
                                         size_t ws_bytes, void *stream) {
    DSRT_REQUIRE(n_vec >= 1 && n_docs >= 1 && k_c >= 1, DSRT_EINVAL, "invalid parameter: empty input");
    DSRT_REQUIRE(ws_bytes >= dsrt_postings_workspace(n_vec, k_c), DSRT_EINVAL,
                 "invalid parameter: postings workspace too small");
    cudaStream_t st = as_stream(stream);
    uint8_t *w = static_cast<uint8_t *>(workspace);
    const size_t n8 = al(static_cast<size_t>(n_vec + 1) * 8);
    int64_t *keys = reinterpret_cast<int64_t *>(w);
    int64_t *doc_of = reinterpret_cast<int64_t *>(w + n8);
    int64_t *perm = reinterpret_cast<int64_t *>(w + 2 * n8);
    int64_t *keep = reinterpret_cast<int64_t *>(w + 3 * n8);
    int64_t *pos = reinterpret_cast<int64_t *>(w + 4 * n8);
    unsigned long long *ucount = reinterpret_cast<unsigned long long *>(w + 5 * n8);
    uint8_t *scan1 = w + 5 * n8 + al(static_cast<size_t>(k_c) * 8);
    uint8_t *scan2 = scan1 + al(scan_ws_bytes(n_vec + 1));
    uint8_t *rws = scan2 + al(scan_ws_bytes(k_c + 1));
    uint32_t *bad = reinterpret_cast<uint32_t *>(rws + radix_sort_ws(n_vec));
    DSRT_CUDA(cudaMemsetAsync(bad, 0, 4, st));
    DSRT_CUDA(cudaMemsetAsync(ucount, 0, k_c * 8, st));
    const unsigned b256 = static_cast<unsigned>((n_vec + 255) / 256);
    keys_from_assign_kernel<<<b256, 256, 0, st>>>(assign, n_vec, k_c, keys, bad);
    doc_of_vec_kernel<<<static_cast<unsigned>((n_docs + 7) / 8), 256, 0, st>>>(set_off, n_docs, doc_of);
    DSRT_LAUNCH_CHECK();
    int bits = 1;
    while (bits < 62 && (1LL << bits) < k_c) ++bits;
    int rc = radix_sort_perm(keys, n_vec, bits, perm, rws, radix_sort_ws(n_vec), st);
    if (rc) return rc;
    keep_kernel<<<b256, 256, 0, st>>>(keys, perm, doc_of, n_vec, keep, ucount);
    rc = exclusive_scan_i64(keep, n_vec, pos, scan1, scan_ws_bytes(n_vec + 1), st);
    if (rc) return rc;
    compact_kernel<<<b256, 256, 0, st>>>(perm, doc_of, keep, pos, n_vec, post_docs, n_post);
    rc = exclusive_scan_i64(reinterpret_cast<const int64_t *>(ucount), k_c, post_off, scan2,
                            scan_ws_bytes(k_c + 1), st);
    if (rc) return rc;
    DSRT_LAUNCH_CHECK();
    uint32_t h = 0;
    DSRT_CUDA(cudaMemcpyAsync(&h, bad, 4, cudaMemcpyDeviceToHost, st));
    DSRT_CUDA(cudaStreamSynchronize(st));
    DSRT_REQUIRE(h == 0, DSRT_ERANGE, "centroid index out of range: %u assignments", h);
    return DSRT_OK;
}
