// K2 -- device code layout (replaces the per-set TinyTable build).
//
// The reference sketches every set separately (index.py:142-145 ->
// build_tiny_table, sketch.py:51-80: per table bincount + cumsum + stable
// argsort).  On the device the same information is kept as one CSR stream:
//   set_off[N+1]  (exclusive scan of set sizes -- the counting sort's scan)
//   records[sum m_i][R]  (bit-sliced codes, set-contiguous)
// A TinyTable is a per-(set, table) counting sort of these codes; the scorer
// needs only the codes themselves (dense compare == bucket walk,
// sketch.py:92-153), so no bucket arrays are materialised.
//
// dsrt_counting_sort builds the CSR from vectors tagged with arbitrary set ids:
// histogram -> exclusive scan -> atomic scatter -> per-set stabilisation
// (ascending original index, i.e. the order build_index would see).
#include "common.cuh"

namespace dsrt {

// ------------------------------------------------------ codes -> records
template <typename TC>
__global__ void codes_to_records_kernel(const TC *__restrict__ codes, int64_t n, int L, int C,
                                        uint32_t *__restrict__ recs, uint32_t *bad) {
    const int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (v >= n) return;
    const int W = plane_words(L), R = record_words(L, C);
    const uint32_t lim = C >= 32 ? 0xffffffffu : ((1u << C) - 1u);
    uint32_t *out = recs + v * R;
    int nbad = 0;
    for (int w = 0; w < W; ++w) {
        uint32_t planes[24];
        for (int b = 0; b < C; ++b) planes[b] = 0;
        const int t1 = min(L, 32 * (w + 1));
        for (int t = 32 * w; t < t1; ++t) {
            const uint32_t code = static_cast<uint32_t>(codes[v * L + t]);
            nbad += code > lim;
            for (int b = 0; b < C; ++b) planes[b] |= ((code >> b) & 1u) << (t & 31);
        }
        for (int b = 0; b < C; ++b) out[b * W + w] = planes[b];
    }
    for (int i = C * W; i < R; ++i) out[i] = 0;
    if (nbad && bad) atomicAdd(bad, static_cast<uint32_t>(nbad));
}

// ------------------------------------------------------------- scan
constexpr int kScanBlock = 1024;
constexpr int kScanItems = 8;  // per thread
constexpr int64_t kScanTile = kScanBlock * kScanItems;

__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t *warp_sums,
                                                        int64_t *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int64_t s = lane < (blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        warp_sums[lane] = s;  // inclusive
    }
    __syncthreads();
    const int64_t before = (warp > 0 ? warp_sums[warp - 1] : 0) + x - v;
    if (total) *total = warp_sums[(blockDim.x >> 5) - 1];
    __syncthreads();
    return before;
}

// pass 1: per-tile sums (and size validation)
__global__ void scan_reduce_kernel(const int64_t *__restrict__ in, int64_t n,
                                   int64_t *__restrict__ tile_sums, uint32_t *bad, int check) {
    __shared__ int64_t ws[32];
    __shared__ int64_t tot;
    const int64_t base = blockIdx.x * kScanTile;
    int64_t s = 0;
    int nbad = 0;
    for (int i = 0; i < kScanItems; ++i) {
        const int64_t idx = base + static_cast<int64_t>(threadIdx.x) * kScanItems + i;
        if (idx < n) {
            const int64_t v = in[idx];
            s += v;
            if (check) nbad += (v < 1) || (v > 65535);
        }
    }
    if (nbad && bad) atomicAdd(bad, static_cast<uint32_t>(nbad));
    block_exclusive_scan(s, ws, &tot);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

// pass 2: exclusive scan of tile sums (single block, loops)
__global__ void scan_tiles_kernel(int64_t *tile_sums, int64_t n_tiles) {
    __shared__ int64_t ws[32];
    __shared__ int64_t tot;
    int64_t carry = 0;
    for (int64_t b = 0; b < n_tiles; b += blockDim.x) {
        const int64_t i = b + threadIdx.x;
        const int64_t v = i < n_tiles ? tile_sums[i] : 0;
        const int64_t ex = block_exclusive_scan(v, ws, &tot);
        if (i < n_tiles) tile_sums[i] = carry + ex;
        carry += tot;
    }
}

// pass 3: out[i] = exclusive prefix (out has n+1 entries; out[n] = total)
__global__ void scan_apply_kernel(const int64_t *__restrict__ in, int64_t n,
                                  const int64_t *__restrict__ tile_off, int64_t *__restrict__ out) {
    __shared__ int64_t ws[32];
    const int64_t base = blockIdx.x * kScanTile;
    int64_t v[kScanItems];
    int64_t s = 0;
    for (int i = 0; i < kScanItems; ++i) {
        const int64_t idx = base + static_cast<int64_t>(threadIdx.x) * kScanItems + i;
        v[i] = idx < n ? in[idx] : 0;
        s += v[i];
    }
    int64_t run = tile_off[blockIdx.x] + block_exclusive_scan(s, ws, nullptr);
    for (int i = 0; i < kScanItems; ++i) {
        const int64_t idx = base + static_cast<int64_t>(threadIdx.x) * kScanItems + i;
        if (idx < n) out[idx] = run;
        run += v[i];
        if (idx == n - 1) out[n] = run;
    }
}

static int exclusive_scan(const int64_t *in, int64_t n, int64_t *out, uint32_t *bad, int check,
                          void *ws, size_t ws_bytes, cudaStream_t st) {
    const int64_t tiles = (n + kScanTile - 1) / kScanTile;
    DSRT_REQUIRE(ws != nullptr && ws_bytes >= static_cast<size_t>(tiles) * 8, DSRT_EINVAL,
                 "invalid parameter: scan workspace too small");
    int64_t *tile_sums = static_cast<int64_t *>(ws);
    if (n == 0) {
        DSRT_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), st));
        return DSRT_OK;
    }
    scan_reduce_kernel<<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(in, n, tile_sums, bad, check);
    scan_tiles_kernel<<<1, kScanBlock, 0, st>>>(tile_sums, tiles);
    scan_apply_kernel<<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(in, n, tile_sums, out);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}

int exclusive_scan_i64(const int64_t *in, int64_t n, int64_t *out, void *ws, size_t ws_bytes,
                       cudaStream_t st) {
    return exclusive_scan(in, n, out, nullptr, 0, ws, ws_bytes, st);
}
size_t scan_ws_bytes(int64_t n) {
    return static_cast<size_t>((n + kScanTile - 1) / kScanTile + 1) * sizeof(int64_t);
}
size_t radix_sort_ws(int64_t n);
int radix_sort_perm(const int64_t *keys, int64_t n, int key_bits, int64_t *perm_out, void *ws,
                    size_t ws_bytes, cudaStream_t st);

// ---------------------------------------------------------- counting sort
__global__ void histogram_kernel(const int64_t *__restrict__ set_of, int64_t n, int64_t n_sets,
                                 unsigned long long *__restrict__ counts, uint32_t *bad) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int64_t s = set_of[i];
    if (s < 0 || s >= n_sets) {
        atomicAdd(bad, 1u);
        return;
    }
    atomicAdd(counts + s, 1ull);
}

__global__ void gather_rows_kernel(const uint32_t *__restrict__ src, int64_t row_words,
                                   const int64_t *__restrict__ perm, int64_t n,
                                   uint32_t *__restrict__ dst) {
    const int64_t total = n * row_words;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / row_words, w = i % row_words;
        dst[i] = src[perm[r] * row_words + w];
    }
}

// One thread per table: counting sort of the set's codes in table t
// (histogram -> exclusive scan -> stable scatter in ascending j).
template <typename TC>
__global__ void tinytable_kernel(const TC *__restrict__ codes, const int64_t *__restrict__ set_off,
                                 int64_t set, int L, int r, int32_t *__restrict__ offsets,
                                 int32_t *__restrict__ ids) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= L) return;
    const int64_t v0 = set_off[set], m = set_off[set + 1] - v0;
    int32_t *off = offsets + static_cast<int64_t>(t) * (r + 1);
    for (int h = 0; h <= r; ++h) off[h] = 0;
    for (int64_t j = 0; j < m; ++j) off[static_cast<uint32_t>(codes[(v0 + j) * L + t]) + 1] += 1;
    for (int h = 0; h < r; ++h) off[h + 1] += off[h];
    // scatter with a cursor per bucket: reuse off[h] as the cursor, then restore
    for (int64_t j = 0; j < m; ++j) {
        const uint32_t h = static_cast<uint32_t>(codes[(v0 + j) * L + t]);
        ids[static_cast<int64_t>(t) * m + off[h]++] = static_cast<int32_t>(j);
    }
    for (int h = r; h > 0; --h) off[h] = off[h - 1];
    off[0] = 0;
}

}  // namespace dsrt

using namespace dsrt;

namespace dsrt {
// accumulate_collisions_batch (sketch.py:118-153) on a TinyTable: thread per
// (query row, table) adds 1 to every stored vector in bucket (t, code).
__global__ void collision_counts_kernel(const int32_t *__restrict__ offsets, const int32_t *__restrict__ ids,
                                        int L, int r, int m, const int32_t *__restrict__ qcodes, int m_q,
                                        int32_t *__restrict__ counts) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<int64_t>(m_q) * L) return;
    const int q = static_cast<int>(i / L), t = static_cast<int>(i % L);
    const int h = qcodes[static_cast<int64_t>(q) * L + t];
    const int lo = offsets[static_cast<int64_t>(t) * (r + 1) + h];
    const int hi = offsets[static_cast<int64_t>(t) * (r + 1) + h + 1];
    for (int p = lo; p < hi; ++p) atomicAdd(counts + static_cast<int64_t>(q) * m + ids[static_cast<int64_t>(t) * m + p], 1);
}
}  // namespace dsrt

extern "C" int dsrt_collision_counts(const int32_t *offsets, const int32_t *ids, int L, int r, int m,
                                     const int32_t *qcodes, int m_q, int32_t *counts, void *stream) {
    DSRT_REQUIRE(L >= 1 && r >= 1 && m >= 1 && m_q >= 0, DSRT_EINVAL, "invalid parameter: L=%d r=%d m=%d", L, r, m);
    if (m_q == 0) return DSRT_OK;
    cudaStream_t st = as_stream(stream);
    DSRT_CUDA(cudaMemsetAsync(counts, 0, static_cast<size_t>(m_q) * m * sizeof(int32_t), st));
    const int64_t n = static_cast<int64_t>(m_q) * L;
    collision_counts_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(offsets, ids, L, r, m, qcodes,
                                                                                 m_q, counts);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}

extern "C" int dsrt_tinytable(const void *codes, int code_bytes, const int64_t *set_off, int64_t set,
                              int L, int C, int32_t *offsets_out, int32_t *ids_out, void *stream) {
    DSRT_REQUIRE(L >= 1 && C >= 1 && C <= 24, DSRT_EINVAL, "invalid parameter: L=%d C=%d", L, C);
    const int r = 1 << C;
    const unsigned blocks = static_cast<unsigned>((L + 127) / 128);
    cudaStream_t st = as_stream(stream);
    if (code_bytes == 1)
        tinytable_kernel<uint8_t><<<blocks, 128, 0, st>>>(static_cast<const uint8_t *>(codes), set_off, set, L, r, offsets_out, ids_out);
    else if (code_bytes == 2)
        tinytable_kernel<uint16_t><<<blocks, 128, 0, st>>>(static_cast<const uint16_t *>(codes), set_off, set, L, r, offsets_out, ids_out);
    else if (code_bytes == 4)
        tinytable_kernel<uint32_t><<<blocks, 128, 0, st>>>(static_cast<const uint32_t *>(codes), set_off, set, L, r, offsets_out, ids_out);
    else
        DSRT_REQUIRE(false, DSRT_EINVAL, "invalid parameter: code width %d", code_bytes);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}

extern "C" int dsrt_codes_to_records(const void *codes, int code_bytes, int64_t n, int L, int C,
                                     uint32_t *records_out, uint32_t *bad_codes, void *stream) {
    DSRT_REQUIRE(L >= 1 && C >= 1 && C <= 24, DSRT_EINVAL, "invalid parameter: L=%d C=%d", L, C);
    DSRT_REQUIRE(code_bytes == 1 || code_bytes == 2 || code_bytes == 4, DSRT_EINVAL,
                 "invalid parameter: code width %d", code_bytes);
    if (n == 0) return DSRT_OK;
    cudaStream_t st = as_stream(stream);
    const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
    if (code_bytes == 1)
        codes_to_records_kernel<uint8_t><<<blocks, 256, 0, st>>>(static_cast<const uint8_t *>(codes), n, L, C, records_out, bad_codes);
    else if (code_bytes == 2)
        codes_to_records_kernel<uint16_t><<<blocks, 256, 0, st>>>(static_cast<const uint16_t *>(codes), n, L, C, records_out, bad_codes);
    else
        codes_to_records_kernel<uint32_t><<<blocks, 256, 0, st>>>(static_cast<const uint32_t *>(codes), n, L, C, records_out, bad_codes);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}

extern "C" size_t dsrt_scan_workspace(int64_t n_sets) {
    return static_cast<size_t>((n_sets + kScanTile - 1) / kScanTile + 1) * sizeof(int64_t);
}

extern "C" int dsrt_sizes_to_offsets(const int64_t *sizes, int64_t n_sets, int64_t *set_off_out,
                                     uint32_t *bad, void *workspace, size_t workspace_bytes,
                                     void *stream) {
    DSRT_REQUIRE(n_sets >= 0, DSRT_EINVAL, "invalid parameter: n_sets < 0");
    return exclusive_scan(sizes, n_sets, set_off_out, bad, 1, workspace, workspace_bytes,
                          as_stream(stream));
}

extern "C" size_t dsrt_counting_sort_workspace(int64_t n, int64_t n_sets) {
    // counts (n_sets u64) + scan tiles + flags + radix sort workspace
    return static_cast<size_t>(n_sets) * 8 + dsrt_scan_workspace(n_sets) + 256 + radix_sort_ws(n);
}

extern "C" int dsrt_counting_sort(const int64_t *set_of_vec, int64_t n, int64_t n_sets,
                                  int64_t *set_off_out, int64_t *perm_out, void *workspace,
                                  size_t workspace_bytes, void *stream) {
    DSRT_REQUIRE(n >= 0 && n_sets >= 1, DSRT_EINVAL, "invalid parameter: n=%lld n_sets=%lld",
                 (long long)n, (long long)n_sets);
    DSRT_REQUIRE(workspace_bytes >= dsrt_counting_sort_workspace(n, n_sets), DSRT_EINVAL,
                 "invalid parameter: counting-sort workspace too small");
    cudaStream_t st = as_stream(stream);
    uint8_t *ws = static_cast<uint8_t *>(workspace);
    unsigned long long *counts = reinterpret_cast<unsigned long long *>(ws);
    uint8_t *scan_ws = ws + n_sets * 8;
    uint32_t *flags = reinterpret_cast<uint32_t *>(scan_ws + dsrt_scan_workspace(n_sets));
    void *rws = scan_ws + dsrt_scan_workspace(n_sets) + 256;
    DSRT_CUDA(cudaMemsetAsync(ws, 0, n_sets * 8, st));
    DSRT_CUDA(cudaMemsetAsync(flags, 0, 16, st));
    const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
    if (n > 0) histogram_kernel<<<blocks, 256, 0, st>>>(set_of_vec, n, n_sets, counts, flags);
    DSRT_LAUNCH_CHECK();
    int rc = exclusive_scan(reinterpret_cast<const int64_t *>(counts), n_sets, set_off_out, nullptr,
                            0, scan_ws, dsrt_scan_workspace(n_sets), st);
    if (rc != DSRT_OK) return rc;
    uint32_t h = 0;
    DSRT_CUDA(cudaMemcpyAsync(&h, flags, sizeof(h), cudaMemcpyDeviceToHost, st));
    DSRT_CUDA(cudaStreamSynchronize(st));
    DSRT_REQUIRE(h == 0, DSRT_ERANGE, "set index out of range: %u vectors name a set outside [0, %lld)",
                 h, (long long)n_sets);
    int bits = 1;
    while (bits < 63 && (1LL << bits) < n_sets) ++bits;
    return radix_sort_perm(set_of_vec, n, bits, perm_out, rws, radix_sort_ws(n), st);
}

extern "C" int dsrt_gather_rows(const void *src, int64_t row_bytes, const int64_t *perm, int64_t n,
                                void *dst, void *stream) {
    DSRT_REQUIRE(row_bytes > 0 && row_bytes % 4 == 0, DSRT_EINVAL,
                 "invalid parameter: row_bytes %lld", (long long)row_bytes);
    if (n == 0) return DSRT_OK;
    gather_rows_kernel<<<4 * 148 * 4, 256, 0, as_stream(stream)>>>(
        static_cast<const uint32_t *>(src), row_bytes / 4, perm, n, static_cast<uint32_t *>(dst));
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}
