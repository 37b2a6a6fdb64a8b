// K7 -- spherical k-means (train_centroids, prefilter.py:47-82) on the device,
// deterministic and in the reference's float64 operation order:
//
//   X      = rows / np.linalg.norm(rows)       norm = sqrt(pairwise(x*x))
//   init   = X[rng.choice(n, k, replace=False)] (indices from the host rng)
//   repeat iters:
//     assign[i] = argmax_c <X_i, c>  (first index on ties); best[i] = that value
//                 -- tcgen05 screen + float64 re-rank as K6, dot = sequential
//                    FMA chain over d (OpenBLAS dgemm's per-element order for
//                    full tiles); d != 128: exact SIMT scan
//     sums[c]   = sum of X_i over assign[i] = c in ascending i  (np.add.at)
//     norms[c]  = sqrt(pairwise(sums[c]^2));  dead = count == 0 | norm < 1e-12
//     dead c (ascending) <- X[argsort(best, stable)[r]], norm 1
//     cents     = sums / norms
//
// Members of a centroid are found with the stable counting sort of K2, so
// the per-centroid sums run sequentially in sample order (no atomics: the
// result is deterministic, unlike a scatter-add).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cmath>

#include "common.cuh"

extern "C" int dsrt_counting_sort(const int64_t *set_of_vec, int64_t n, int64_t n_sets,
                                  int64_t *set_off_out, int64_t *perm_out, void *workspace,
                                  size_t ws_bytes, void *stream);
extern "C" size_t dsrt_counting_sort_workspace(int64_t n, int64_t n_sets);
extern "C" size_t dsrt_assign_centroids_workspace(int64_t n, int d, int64_t k_c);
extern "C" int dsrt_to_f16_rows(const double *src, int64_t n, int d, double scale, void *dst,
                                void *stream);

namespace dsrt {

int assign_unit_rows_f64(const double *X, int64_t n, const double *cents, const void *cents_f16,
                         int64_t k_c, int32_t *assign_out, double *best, void *ws, cudaStream_t st);
size_t radix_sort_ws(int64_t n);
int radix_sort_perm(const int64_t *keys, int64_t n, int key_bits, int64_t *perm_out, void *ws,
                    size_t ws_bytes, cudaStream_t st);
int exclusive_scan_i64(const int64_t *in, int64_t n, int64_t *out, void *ws, size_t ws_bytes,
                       cudaStream_t st);
size_t scan_ws_bytes(int64_t n);

constexpr int kKmMaxD = 1024;

static size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

// numpy pairwise_sum_DOUBLE of (a[i] * a[i]) over a[0..n) with stride s
__device__ double pw_sq(const double *a, int n, int s) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r = __dadd_rn(r, __dmul_rn(a[i * s], a[i * s]));
        return r;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dmul_rn(a[j * s], a[j * s]);
        int i;
        for (i = 8; i < n - (n % 8); i += 8)
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], __dmul_rn(a[(i + j) * s], a[(i + j) * s]));
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; ++i) res = __dadd_rn(res, __dmul_rn(a[i * s], a[i * s]));
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(pw_sq(a, n2, s), pw_sq(a + n2 * s, n - n2, s));
}

// np.linalg.norm(row) = sqrt(0.0 + pairwise(x*x))
__device__ __forceinline__ double row_norm(const double *a, int n) {
    return __dsqrt_rn(__dadd_rn(0.0, pw_sq(a, n, 1)));
}

__device__ __forceinline__ double km_f64(double v) { return v; }
__device__ __forceinline__ double km_f64(float v) { return static_cast<double>(v); }
__device__ __forceinline__ double km_f64(__half v) { return static_cast<double>(__half2float(v)); }
__device__ __forceinline__ double km_f64(__nv_bfloat16 v) { return static_cast<double>(__bfloat162float(v)); }

// _unit_rows (prefilter.py:37-44): rows as float64 (exact for every input
// dtype), X / norm in numpy's order; zero rows flagged
template <typename TQ>
__global__ void km_unit_rows_kernel(const TQ *__restrict__ X, int64_t n, int d,
                                    double *__restrict__ out, uint32_t *__restrict__ zero) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    double *o = out + i * d;
    for (int k = 0; k < d; ++k) o[k] = km_f64(X[i * d + k]);
    const double nrm = row_norm(o, d);
    if (nrm == 0.0) atomicOr(zero, 1u);
    for (int k = 0; k < d; ++k) o[k] = __ddiv_rn(o[k], nrm);
}

__global__ void km_gather_rows_kernel(const double *__restrict__ X, const int64_t *__restrict__ idx,
                                      int64_t k, int d, double *__restrict__ out) {
    const int64_t c = blockIdx.x;
    if (c >= k) return;
    const int64_t src = idx[c];
    for (int t = threadIdx.x; t < d; t += blockDim.x) out[c * d + t] = X[src * d + t];
}

// exact SIMT assignment for d != 128: warp per row, lanes over centroids
__global__ void __launch_bounds__(128)
    km_assign_simt_kernel(const double *__restrict__ X, int64_t n, int d,
                          const double *__restrict__ cents, int64_t k, int32_t *__restrict__ assign,
                          double *__restrict__ best) {
    extern __shared__ double xs[];  // 4 warps x d
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = blockIdx.x * 4LL + warp;
    if (i >= n) return;
    double *x = xs + warp * d;
    for (int t = lane; t < d; t += 32) x[t] = X[i * d + t];
    __syncwarp();
    double bs = -INFINITY;
    int64_t bi = INT64_MAX;
    for (int64_t c = lane; c < k; c += 32) {
        const double *cv = cents + c * d;
        double acc = 0.0;
        for (int t = 0; t < d; ++t) acc = fma(x[t], cv[t], acc);
        if (acc > bs) { bs = acc; bi = c; }  // ascending c per lane: first max kept
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, bs, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (os > bs || (os == bs && oi < bi)) { bs = os; bi = oi; }
    }
    if (lane == 0) {
        assign[i] = static_cast<int32_t>(bi);
        best[i] = bs;
    }
}

__global__ void km_keys_kernel(const int32_t *__restrict__ assign, int64_t n, int64_t *__restrict__ keys) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) keys[i] = assign[i];
}

// block per centroid, thread per dimension: sequential sum in sample order,
// then the row norm (pairwise) and the dead flag
__global__ void km_sums_kernel(const double *__restrict__ X, int d, const int64_t *__restrict__ off,
                               const int64_t *__restrict__ perm, int64_t k, double *__restrict__ sums,
                               double *__restrict__ norms, int64_t *__restrict__ dead,
                               unsigned long long *__restrict__ n_dead) {
    const int64_t c = blockIdx.x;
    if (c >= k) return;
    const int64_t b = off[c], e = off[c + 1];
    double *srow = sums + c * d;
    for (int t = threadIdx.x; t < d; t += blockDim.x) {
        double s = 0.0;
        for (int64_t m = b; m < e; ++m) s = __dadd_rn(s, X[perm[m] * d + t]);
        srow[t] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const double nrm = row_norm(srow, d);
        const bool dd = (e == b) || (nrm < 1e-12);
        norms[c] = nrm;
        dead[c] = dd ? 1 : 0;
        if (dd) atomicAdd(n_dead, 1ull);
    }
}

// order-preserving int64 key of a double (ascending)
__global__ void km_best_keys_kernel(const double *__restrict__ best, int64_t n, int64_t *__restrict__ keys) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint64_t u = static_cast<uint64_t>(__double_as_longlong(best[i]));
    keys[i] = static_cast<int64_t>((u >> 63) ? ~u : (u | 0x8000000000000000ull));
}

// dead slot r (ascending centroid id) <- X[order[r]], norm 1
__global__ void km_reseed_kernel(const int64_t *__restrict__ dead, const int64_t *__restrict__ rank,
                                 int64_t k, const int64_t *__restrict__ order, const double *__restrict__ X,
                                 int d, double *__restrict__ sums, double *__restrict__ norms) {
    const int64_t c = blockIdx.x;
    if (c >= k || dead[c] == 0) return;
    const int64_t p = order[rank[c]];
    for (int t = threadIdx.x; t < d; t += blockDim.x) sums[c * d + t] = X[p * d + t];
    if (threadIdx.x == 0) norms[c] = 1.0;
}

__global__ void km_divide_kernel(const double *__restrict__ sums, const double *__restrict__ norms,
                                 int64_t k, int d, double *__restrict__ cents) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= k * d) return;
    cents[i] = __ddiv_rn(sums[i], norms[i / d]);
}

// Exact assignment for any d <= kKmMaxD (K6 for d != 128): unit rows in
// numpy's order, sequential FMA dots, np.argmax's first-index rule.  Rows go
// in chunks of kKmChunk through a float64 staging buffer (ws: kKmChunk*d*8
// bytes + 64).  Zero rows are reported through *zero_rows (host).
constexpr int64_t kKmChunk = 1 << 18;
size_t assign_simt_ws(int64_t n, int d) {
    return static_cast<size_t>(tmin<int64_t>(tmax<int64_t>(n, 1), kKmChunk)) * d * 8 + 256;
}
int assign_simt(const void *X, int dtype, int64_t n, int d, const double *cents, int64_t k,
                int32_t *assign, void *ws, cudaStream_t st) {
    DSRT_REQUIRE(d >= 1 && d <= kKmMaxD, DSRT_EUNSUPPORTED, "invalid parameter: d=%d > %d", d, kKmMaxD);
    uint8_t *w = static_cast<uint8_t *>(ws);
    uint32_t *zero = reinterpret_cast<uint32_t *>(w);
    double *xu = reinterpret_cast<double *>(w + 256);
    double *best = nullptr;
    DSRT_CUDA(malloc_async(reinterpret_cast<void **>(&best), tmin<int64_t>(n, kKmChunk) * 8, st));
    DSRT_CUDA(cudaMemsetAsync(zero, 0, 4, st));
    const size_t smem = 4 * static_cast<size_t>(d) * 8;
    for (int64_t r0 = 0; r0 < n; r0 += kKmChunk) {
        const int64_t rows = tmin<int64_t>(kKmChunk, n - r0);
        const unsigned nb = static_cast<unsigned>((rows + 127) / 128);
        switch (dtype) {
            case DSRT_F64: km_unit_rows_kernel<double><<<nb, 128, 0, st>>>(static_cast<const double *>(X) + r0 * d, rows, d, xu, zero); break;
            case DSRT_F32: km_unit_rows_kernel<float><<<nb, 128, 0, st>>>(static_cast<const float *>(X) + r0 * d, rows, d, xu, zero); break;
            case DSRT_F16: km_unit_rows_kernel<__half><<<nb, 128, 0, st>>>(static_cast<const __half *>(X) + r0 * d, rows, d, xu, zero); break;
            case DSRT_BF16: km_unit_rows_kernel<__nv_bfloat16><<<nb, 128, 0, st>>>(static_cast<const __nv_bfloat16 *>(X) + r0 * d, rows, d, xu, zero); break;
            default:
                cudaFreeAsync(best, st);
                set_error("invalid parameter: x dtype %d", dtype);
                return DSRT_EINVAL;
        }
        km_assign_simt_kernel<<<static_cast<unsigned>((rows + 3) / 4), 128, smem, st>>>(
            xu, rows, d, cents, k, assign + r0, best);
        DSRT_LAUNCH_CHECK();
    }
    cudaFreeAsync(best, st);
    uint32_t hz = 0;
    DSRT_CUDA(cudaMemcpyAsync(&hz, zero, 4, cudaMemcpyDeviceToHost, st));
    DSRT_CUDA(cudaStreamSynchronize(st));
    DSRT_REQUIRE(hz == 0, DSRT_EINVAL, "zero vector in documents: cannot assign to a centroid");
    return DSRT_OK;
}

struct KmLayout {
    size_t xu, assign, best, keys, off, perm, sums, norms, dead, rank, c16, misc, sort, aws, rws, sws;
    size_t total;
};

static KmLayout km_layout(int64_t n, int d, int64_t k) {
    KmLayout L{};
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o += align256(bytes);
        return at;
    };
    L.xu = take(static_cast<size_t>(n) * d * 8);
    L.assign = take(static_cast<size_t>(n) * 4);
    L.best = take(static_cast<size_t>(n) * 8);
    L.keys = take(static_cast<size_t>(n) * 8);
    L.off = take(static_cast<size_t>(k + 1) * 8);
    L.perm = take(static_cast<size_t>(n) * 8);
    L.sums = take(static_cast<size_t>(k) * d * 8);
    L.norms = take(static_cast<size_t>(k) * 8);
    L.dead = take(static_cast<size_t>(k + 1) * 8);
    L.rank = take(static_cast<size_t>(k + 1) * 8);
    L.c16 = take(static_cast<size_t>(k) * d * 2);
    L.misc = take(64);
    L.sort = take(dsrt_counting_sort_workspace(n, k));
    L.aws = take(d == 128 ? dsrt_assign_centroids_workspace(n, d, k) : 0);
    L.rws = take(radix_sort_ws(n));
    L.sws = take(scan_ws_bytes(k + 1));
    L.total = o;
    return L;
}

}  // namespace dsrt

using namespace dsrt;

extern "C" size_t dsrt_train_centroids_workspace(int64_t n, int d, int64_t k) {
    if (n < 1 || d < 1) return 0;
    return km_layout(n, d, tmax<int64_t>(k, 1)).total;
}

extern "C" int dsrt_train_centroids(const double *samples, int64_t n, int d, int64_t k, int iters,
                                    const int64_t *init_idx, double *centroids_out, void *workspace,
                                    size_t ws_bytes, void *stream) {
    // validation order of train_centroids: _unit_rows (shape, zero rows), then k / iters
    DSRT_REQUIRE(n >= 1 && d >= 1, DSRT_EINVAL, "samples must be a non-empty (n, d) matrix");
    DSRT_REQUIRE(d <= kKmMaxD, DSRT_EUNSUPPORTED, "invalid parameter: d=%d > %d", d, kKmMaxD);
    const int64_t k_ws = tmax<int64_t>(k, 1);
    const KmLayout L = km_layout(n, d, k_ws);
    DSRT_REQUIRE(ws_bytes >= L.total, DSRT_EINVAL, "invalid parameter: k-means workspace too small");
    cudaStream_t st = as_stream(stream);
    uint8_t *w = static_cast<uint8_t *>(workspace);
    double *xu = reinterpret_cast<double *>(w + L.xu);
    int32_t *assign = reinterpret_cast<int32_t *>(w + L.assign);
    double *best = reinterpret_cast<double *>(w + L.best);
    int64_t *keys = reinterpret_cast<int64_t *>(w + L.keys);
    int64_t *off = reinterpret_cast<int64_t *>(w + L.off);
    int64_t *perm = reinterpret_cast<int64_t *>(w + L.perm);
    double *sums = reinterpret_cast<double *>(w + L.sums);
    double *norms = reinterpret_cast<double *>(w + L.norms);
    int64_t *dead = reinterpret_cast<int64_t *>(w + L.dead);
    int64_t *rank = reinterpret_cast<int64_t *>(w + L.rank);
    void *c16 = w + L.c16;
    uint32_t *zero = reinterpret_cast<uint32_t *>(w + L.misc);
    unsigned long long *n_dead = reinterpret_cast<unsigned long long *>(w + L.misc + 8);
    double *cents = centroids_out;

    DSRT_CUDA(cudaMemsetAsync(w + L.misc, 0, 64, st));
    const unsigned nb = static_cast<unsigned>((n + 127) / 128);
    km_unit_rows_kernel<double><<<nb, 128, 0, st>>>(samples, n, d, xu, zero);
    DSRT_LAUNCH_CHECK();
    uint32_t hz = 0;
    DSRT_CUDA(cudaMemcpyAsync(&hz, zero, 4, cudaMemcpyDeviceToHost, st));
    DSRT_CUDA(cudaStreamSynchronize(st));
    DSRT_REQUIRE(hz == 0, DSRT_EINVAL, "zero vector in samples: cannot assign to a centroid");
    DSRT_REQUIRE(k >= 1, DSRT_EINVAL, "invalid parameter: k must be >= 1, got %lld", (long long)k);
    DSRT_REQUIRE(n >= k, DSRT_EINVAL, "too few samples: need at least k=%lld, got %lld",
                 (long long)k, (long long)n);
    DSRT_REQUIRE(iters >= 1, DSRT_EINVAL, "invalid parameter: iters must be >= 1, got %d", iters);
    DSRT_REQUIRE(k < (1LL << 31), DSRT_EUNSUPPORTED, "invalid parameter: k too large");
    DSRT_REQUIRE(init_idx != nullptr, DSRT_EINVAL, "invalid parameter: init indices missing");
    km_gather_rows_kernel<<<static_cast<unsigned>(k), 128, 0, st>>>(xu, init_idx, k, d, cents);
    DSRT_LAUNCH_CHECK();
    const int tpb = d < 128 ? 32 * ((d + 31) / 32) : 128;
    for (int it = 0; it < iters; ++it) {
        if (d == 128) {
            int rc = dsrt_to_f16_rows(cents, k, d, 1.0, c16, st);
            if (rc) return rc;
            rc = assign_unit_rows_f64(xu, n, cents, c16, k, assign, best, w + L.aws, st);
            if (rc) return rc;
        } else {
            const size_t smem = 4 * static_cast<size_t>(d) * 8;
            km_assign_simt_kernel<<<static_cast<unsigned>((n + 3) / 4), 128, smem, st>>>(
                xu, n, d, cents, k, assign, best);
            DSRT_LAUNCH_CHECK();
        }
        km_keys_kernel<<<nb, 128, 0, st>>>(assign, n, keys);
        int rc = dsrt_counting_sort(keys, n, k, off, perm, w + L.sort, dsrt_counting_sort_workspace(n, k), st);
        if (rc) return rc;
        DSRT_CUDA(cudaMemsetAsync(n_dead, 0, 8, st));
        km_sums_kernel<<<static_cast<unsigned>(k), tpb, 0, st>>>(xu, d, off, perm, k, sums, norms, dead, n_dead);
        DSRT_LAUNCH_CHECK();
        unsigned long long hd = 0;
        DSRT_CUDA(cudaMemcpyAsync(&hd, n_dead, 8, cudaMemcpyDeviceToHost, st));
        DSRT_CUDA(cudaStreamSynchronize(st));
        if (hd > 0) {  // farthest-assigned points, one per dead cluster (ascending ids)
            km_best_keys_kernel<<<nb, 128, 0, st>>>(best, n, keys);
            rc = radix_sort_perm(keys, n, 64, perm, w + L.rws, radix_sort_ws(n), st);
            if (rc) return rc;
            rc = exclusive_scan_i64(dead, k, rank, w + L.sws, scan_ws_bytes(k + 1), st);
            if (rc) return rc;
            km_reseed_kernel<<<static_cast<unsigned>(k), tpb, 0, st>>>(dead, rank, k, perm, xu, d, sums, norms);
            DSRT_LAUNCH_CHECK();
        }
        km_divide_kernel<<<static_cast<unsigned>((k * d + 255) / 256), 256, 0, st>>>(sums, norms, k, d, cents);
        DSRT_LAUNCH_CHECK();
    }
    return DSRT_OK;
}
