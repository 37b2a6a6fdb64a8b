// Stable LSD radix sort of int64 keys (8-bit digits) returning the sorted
// permutation -- the scatter stage of the counting sorts that build the CSR
// layouts (vectors by set, postings by centroid).  Stable by construction:
// per 4096-element tile, warp w ranks its 512 consecutive elements step by
// step with __match_any_sync, warps are combined by an exclusive scan per
// digit, tiles by a device-wide exclusive scan of the (digit, tile) counts.
#include "common.cuh"

namespace dsrt {

constexpr int kRThreads = 256;
constexpr int kRWarps = kRThreads / 32;
constexpr int kRSteps = 16;                       // 32-element steps per warp
constexpr int kRTile = kRThreads * kRSteps;       // 4096

int exclusive_scan_i64(const int64_t *in, int64_t n, int64_t *out, void *ws, size_t ws_bytes,
                       cudaStream_t st);
size_t scan_ws_bytes(int64_t n);

__global__ void __launch_bounds__(kRThreads)
    rs_hist_kernel(const int64_t *__restrict__ keys, int64_t n, int shift, int64_t n_tiles,
                   int64_t *__restrict__ hist) {
    __shared__ uint32_t cnt[256];
    cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kRTile;
    for (int i = threadIdx.x; i < kRTile; i += kRThreads) {
        const int64_t e = base + i;
        if (e < n) atomicAdd(&cnt[(keys[e] >> shift) & 255], 1u);
    }
    __syncthreads();
    hist[static_cast<int64_t>(threadIdx.x) * n_tiles + blockIdx.x] = cnt[threadIdx.x];
}

__global__ void __launch_bounds__(kRThreads)
    rs_scatter_kernel(const int64_t *__restrict__ keys_in, const int64_t *__restrict__ vals_in,
                      int64_t n, int shift, int64_t n_tiles, const int64_t *__restrict__ offsets,
                      int64_t *__restrict__ keys_out, int64_t *__restrict__ vals_out) {
    __shared__ int wcount[kRWarps][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < kRWarps * 256; i += kRThreads) (&wcount[0][0])[i] = 0;
    __syncthreads();
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kRTile + warp * (32 * kRSteps);
    int dg[kRSteps], lr[kRSteps];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int s = 0; s < kRSteps; ++s) {
        const int64_t e = base + s * 32 + lane;
        const bool ok = e < n;
        const int d = ok ? static_cast<int>((keys_in[e] >> shift) & 255) : 256 + lane;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int before = ok ? wcount[warp][d] : 0;
        __syncwarp();
        if (ok && (peers & lt) == 0) wcount[warp][d] = before + __popc(peers);
        __syncwarp();
        dg[s] = d;
        lr[s] = before + __popc(peers & lt);
    }
    __syncthreads();
    {  // exclusive scan over warps, one digit per thread
        const int d = threadIdx.x;
        int run = 0;
#pragma unroll
        for (int w = 0; w < kRWarps; ++w) {
            const int t = wcount[w][d];
            wcount[w][d] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < kRSteps; ++s) {
        const int64_t e = base + s * 32 + lane;
        if (e < n) {
            const int d = dg[s];
            const int64_t pos = offsets[static_cast<int64_t>(d) * n_tiles + blockIdx.x] + wcount[warp][d] + lr[s];
            keys_out[pos] = keys_in[e];
            vals_out[pos] = vals_in ? vals_in[e] : e;
        }
    }
}

size_t radix_sort_ws(int64_t n) {
    const int64_t tiles = (n + kRTile - 1) / kRTile;
    return 4 * static_cast<size_t>(n) * 8 + static_cast<size_t>(256 * tiles) * 16 +
           scan_ws_bytes(256 * tiles) + 1024;
}

// perm_out[i] = index of the i-th smallest key (ties in index order).
int radix_sort_perm(const int64_t *keys, int64_t n, int key_bits, int64_t *perm_out, void *ws,
                    size_t ws_bytes, cudaStream_t st) {
    DSRT_REQUIRE(ws_bytes >= radix_sort_ws(n), DSRT_EINVAL, "invalid parameter: radix workspace too small");
    if (n == 0) return DSRT_OK;
    const int64_t tiles = (n + kRTile - 1) / kRTile;
    DSRT_REQUIRE(tiles < (1LL << 31), DSRT_EUNSUPPORTED, "invalid parameter: too many elements");
    uint8_t *w = static_cast<uint8_t *>(ws);
    int64_t *ka = reinterpret_cast<int64_t *>(w);
    int64_t *kb = ka + n;
    int64_t *va = kb + n;
    int64_t *vb = va + n;
    int64_t *hist = vb + n;
    int64_t *offs = hist + 256 * tiles;
    void *scan_ws = offs + 256 * tiles + 1;
    const size_t scan_bytes = scan_ws_bytes(256 * tiles);
    const int passes = tmax(1, (key_bits + 7) / 8);
    const int64_t *kin = keys;
    const int64_t *vin = nullptr;
    for (int p = 0; p < passes; ++p) {
        int64_t *kout = (p & 1) ? kb : ka;
        int64_t *vout = (p == passes - 1) ? perm_out : ((p & 1) ? vb : va);
        rs_hist_kernel<<<static_cast<unsigned>(tiles), kRThreads, 0, st>>>(kin, n, 8 * p, tiles, hist);
        int rc = exclusive_scan_i64(hist, 256 * tiles, offs, scan_ws, scan_bytes, st);
        if (rc) return rc;
        rs_scatter_kernel<<<static_cast<unsigned>(tiles), kRThreads, 0, st>>>(kin, vin, n, 8 * p, tiles,
                                                                               offs, kout, vout);
        DSRT_LAUNCH_CHECK();
        kin = kout;
        vin = vout;
    }
    return DSRT_OK;
}

}  // namespace dsrt
