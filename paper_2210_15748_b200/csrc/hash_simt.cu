// K1 (SIMT modes) -- SRP hashing with a fused sign-and-pack epilogue.
//
// Replaces lsh.hash_matrix (lsh.py:90-106): bits = (X @ planes.T) > 0.0,
// code_t = sum_c bit[t*C + c] << c.  DSRT_HASH_F64 accumulates in float64
// against the reference's float64 planes (flips only where BLAS and this
// kernel round a near-zero projection differently); DSRT_HASH_F32 uses
// float32 planes.  The tensor-core modes (the cfg-2 throughput path) live in
// hash_tc.cu.
//
// CTA = 64 rows; planes are consumed in 32-plane x 64-dim tiles staged in
// shared memory ([dim][plane] so each thread's 32 accumulators read 8
// broadcast LDS.128 per dimension); sign bits are gathered per row in shared
// memory and packed into codes and plane records at the end.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace dsrt {

constexpr int kHRows = 64;
constexpr int kHPlanes = 32;
constexpr int kHDim = 32;
constexpr int kMaxBitWords = 128;  // L*C <= 4096

template <typename T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f32<__half>(__half v) { return __half2float(v); }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T, typename A>
__device__ __forceinline__ A to_acc(T v) {
    return static_cast<A>(to_f32<T>(v));
}
template <>
__device__ __forceinline__ double to_acc<double, double>(double v) { return v; }
template <>
__device__ __forceinline__ float to_acc<double, float>(double v) { return static_cast<float>(v); }

// Pack the sign bits of one row into codes and plane records.
__device__ __forceinline__ void pack_row(const uint32_t *bits, int L, int C, int64_t row,
                                         void *codes_out, uint32_t *recs_out) {
    const int W = plane_words(L), R = record_words(L, C);
    const int code_bytes = C <= 8 ? 1 : (C <= 16 ? 2 : 4);
    uint32_t rec[128];
    const bool want_rec = recs_out != nullptr && R <= 128;
    if (want_rec)
        for (int i = 0; i < R; ++i) rec[i] = 0;
    for (int t = 0; t < L; ++t) {
        uint32_t code = 0;
        for (int c = 0; c < C; ++c) {
            const int p = t * C + c;
            code |= ((bits[p >> 5] >> (p & 31)) & 1u) << c;
        }
        if (codes_out) {
            if (code_bytes == 1)
                static_cast<uint8_t *>(codes_out)[row * L + t] = static_cast<uint8_t>(code);
            else if (code_bytes == 2)
                static_cast<uint16_t *>(codes_out)[row * L + t] = static_cast<uint16_t>(code);
            else
                static_cast<uint32_t *>(codes_out)[row * L + t] = code;
        }
        if (want_rec)
            for (int b = 0; b < C; ++b) rec[b * W + (t >> 5)] |= ((code >> b) & 1u) << (t & 31);
    }
    if (want_rec)
        for (int i = 0; i < R; ++i) recs_out[row * R + i] = rec[i];
}

template <typename TX, typename A>
__global__ void __launch_bounds__(kHRows)
    hash_simt_kernel(const TX *__restrict__ X, int64_t n, int d, const A *__restrict__ planes,
                     int L, int C, void *codes_out, uint32_t *recs_out, uint32_t *zero_rows) {
    __shared__ A xs[kHDim][kHRows + 1];
    __shared__ __align__(16) A ps[kHDim][kHPlanes];
    extern __shared__ uint32_t bits_dyn[];  // [kHRows][bw]
    const int tid = threadIdx.x;
    const int bw = (L * C + 31) / 32 + 1;
    uint32_t *my_bits = bits_dyn + tid * bw;
    const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kHRows;
    const int64_t row = row0 + tid;
    const int P = L * C;
    bool nonzero = false;
    for (int w = 0; w < (P + 31) / 32; ++w) my_bits[w] = 0;

    for (int p0 = 0; p0 < P; p0 += kHPlanes) {
        A acc[kHPlanes];
#pragma unroll
        for (int j = 0; j < kHPlanes; ++j) acc[j] = A(0);
        for (int k0 = 0; k0 < d; k0 += kHDim) {
            __syncthreads();
            // stage X tile (64 rows x 64 dims), transposed
            for (int i = tid; i < kHRows * kHDim; i += kHRows) {
                const int r = i / kHDim, kk = i % kHDim;
                const int64_t gr = row0 + r;
                A v = A(0);
                if (gr < n && k0 + kk < d) v = to_acc<TX, A>(X[gr * d + k0 + kk]);
                xs[kk][r] = v;
            }
            // stage planes tile (32 planes x 64 dims) as [dim][plane]
            for (int i = tid; i < kHPlanes * kHDim; i += kHRows) {
                const int pp = i / kHDim, kk = i % kHDim;
                A v = A(0);
                if (p0 + pp < P && k0 + kk < d) v = planes[static_cast<int64_t>(p0 + pp) * d + k0 + kk];
                ps[kk][pp] = v;
            }
            __syncthreads();
            const int kmax = min(kHDim, d - k0);
            for (int kk = 0; kk < kmax; ++kk) {
                const A xv = xs[kk][tid];
                if (p0 == 0) nonzero |= (xv != A(0));
#pragma unroll
                for (int j = 0; j < kHPlanes; ++j) acc[j] = fma(xv, ps[kk][j], acc[j]);
            }
        }
        uint32_t word = 0;
#pragma unroll
        for (int j = 0; j < kHPlanes; ++j) word |= (acc[j] > A(0) ? 1u : 0u) << j;
        my_bits[p0 >> 5] = word;  // p0 is a multiple of 32
    }
    if (row < n) {
        if (!nonzero && zero_rows) atomicAdd(zero_rows, 1u);
        pack_row(my_bits, L, C, row, codes_out, recs_out);
    }
}

// Small batches (too few 64-row blocks to fill the GPU): the 32-plane chunk
// becomes a grid dimension; each CTA writes one sign word per row (same
// per-(row, plane) sequential FMA as above, so bits are identical) and a
// per-row pass packs the words into codes and records.
template <typename TX, typename A, int NPL>
__global__ void __launch_bounds__(kHRows)
    hash_simt_chunk_kernel(const TX *__restrict__ X, int64_t n, int d, const A *__restrict__ planes, int P,
                           uint32_t *__restrict__ bits, int bw, uint32_t *zero_rows) {
    // NPL planes per CTA: 32 (one sign word per row) or 8 (one sign byte; tiny
    // batches, where 32-plane CTAs leave most SMs idle)
    static_assert(NPL == 32 || NPL == 8, "sign word or byte");
    __shared__ A xs[kHDim][kHRows + 1];
    __shared__ __align__(16) A ps[kHDim][NPL];
    const int tid = threadIdx.x;
    const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kHRows;
    const int64_t row = row0 + tid;
    const int p0 = blockIdx.y * NPL;
    bool nonzero = false;
    A acc[NPL];
#pragma unroll
    for (int j = 0; j < NPL; ++j) acc[j] = A(0);
    for (int k0 = 0; k0 < d; k0 += kHDim) {
        __syncthreads();
        for (int i = tid; i < kHRows * kHDim; i += kHRows) {
            const int r = i / kHDim, kk = i % kHDim;
            const int64_t gr = row0 + r;
            A v = A(0);
            if (gr < n && k0 + kk < d) v = to_acc<TX, A>(X[gr * d + k0 + kk]);
            xs[kk][r] = v;
        }
        for (int i = tid; i < NPL * kHDim; i += kHRows) {
            const int pp = i / kHDim, kk = i % kHDim;
            A v = A(0);
            if (p0 + pp < P && k0 + kk < d) v = planes[static_cast<int64_t>(p0 + pp) * d + k0 + kk];
            ps[kk][pp] = v;
        }
        __syncthreads();
        const int kmax = min(kHDim, d - k0);
        for (int kk = 0; kk < kmax; ++kk) {
            const A xv = xs[kk][tid];
            nonzero |= (xv != A(0));
#pragma unroll
            for (int j = 0; j < NPL; ++j) acc[j] = fma(xv, ps[kk][j], acc[j]);
        }
    }
    uint32_t word = 0;
#pragma unroll
    for (int j = 0; j < NPL; ++j) word |= (acc[j] > A(0) ? 1u : 0u) << j;
    if (row < n) {
        if (NPL == 32) bits[row * bw + blockIdx.y] = word;
        else reinterpret_cast<uint8_t *>(bits + row * bw)[blockIdx.y] = static_cast<uint8_t>(word);
        if (blockIdx.y == 0 && !nonzero && zero_rows) atomicAdd(zero_rows, 1u);
    }
}

// Small-batch pack: one thread per (row, output item) -- item i < max(L, R) is
// code i (if i < L) and record word i (if i < R) -- instead of a thread per row
// walking all L * C bits through a local-memory record (the batch-1 latency path).
__global__ void hash_pack_kernel(const uint32_t *__restrict__ bits, int bw, int64_t n, int L, int C,
                                 void *codes_out, uint32_t *recs_out) {
    const int W = plane_words(L), R = record_words(L, C);
    const int items = L > R ? L : R;
    const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t row = g / items;
    const int i = static_cast<int>(g - row * items);
    if (row >= n) return;
    const uint32_t *b = bits + row * bw;
    auto bit = [&](int p) { return (__ldg(b + (p >> 5)) >> (p & 31)) & 1u; };
    if (codes_out != nullptr && i < L) {
        uint32_t code = 0;
        for (int c = 0; c < C; ++c) code |= bit(i * C + c) << c;
        const int code_bytes = C <= 8 ? 1 : (C <= 16 ? 2 : 4);
        if (code_bytes == 1) static_cast<uint8_t *>(codes_out)[row * L + i] = static_cast<uint8_t>(code);
        else if (code_bytes == 2) static_cast<uint16_t *>(codes_out)[row * L + i] = static_cast<uint16_t>(code);
        else static_cast<uint32_t *>(codes_out)[row * L + i] = code;
    }
    if (recs_out != nullptr && i < R) {  // word i = plane bit (i / W) of tables 32 (i % W) ..
        uint32_t word = 0;
        if (i < C * W) {
            const int pb = i / W, t0 = 32 * (i % W);
            for (int j = 0; j < 32 && t0 + j < L; ++j) word |= bit((t0 + j) * C + pb) << j;
        }
        recs_out[row * R + i] = word;
    }
}

template <typename TX, typename A>
static int launch_hash(const void *X, int64_t n, int d, const void *planes, int L, int C,
                       void *codes, uint32_t *recs, uint32_t *zero_rows, cudaStream_t st) {
    const int64_t blocks = (n + kHRows - 1) / kHRows;
    if (blocks < sm_count()) {  // small batch: split the planes across CTAs
        const int bw = (L * C + 31) / 32;
        uint32_t *bits = nullptr;
        DSRT_CUDA(malloc_async(reinterpret_cast<void **>(&bits), static_cast<size_t>(n) * bw * 4, st));
        if (blocks * bw * 4 <= sm_count()) {  // tiny batch: 8-plane CTAs (sign bytes)
            // (bytes past the last plane stay unwritten: the pack reads only plane bits)
            hash_simt_chunk_kernel<TX, A, 8><<<dim3(static_cast<unsigned>(blocks), static_cast<unsigned>((L * C + 7) / 8)),
                                               kHRows, 0, st>>>(
                static_cast<const TX *>(X), n, d, static_cast<const A *>(planes), L * C, bits, bw, zero_rows);
        } else {
            hash_simt_chunk_kernel<TX, A, 32><<<dim3(static_cast<unsigned>(blocks), static_cast<unsigned>(bw)), kHRows, 0,
                                                st>>>(
                static_cast<const TX *>(X), n, d, static_cast<const A *>(planes), L * C, bits, bw, zero_rows);
        }
        const int64_t items = n * static_cast<int64_t>(tmax(L, record_words(L, C)));
        hash_pack_kernel<<<static_cast<unsigned>((items + 127) / 128), 128, 0, st>>>(bits, bw, n, L, C, codes,
                                                                                   recs);
        cudaFreeAsync(bits, st);
        DSRT_LAUNCH_CHECK();
        return DSRT_OK;
    }
    const size_t smem = static_cast<size_t>(kHRows) * ((L * C + 31) / 32 + 1) * sizeof(uint32_t);
    DSRT_CUDA(cudaFuncSetAttribute(hash_simt_kernel<TX, A>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    hash_simt_kernel<TX, A><<<static_cast<unsigned>(blocks), kHRows, smem, st>>>(
        static_cast<const TX *>(X), n, d, static_cast<const A *>(planes), L, C, codes, recs,
        zero_rows);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}

int hash_tc(const void *X, int x_dtype, int64_t n, int d, const void *planes, int mode, int L,
            int C, void *codes_out, uint32_t *records_out, uint32_t *zero_rows, cudaStream_t st);
int hash_fix(const void *X, int x_dtype, int64_t n, int d, const void *planes, int L, int C,
             void *codes_out, uint32_t *records_out, uint32_t *zero_rows, cudaStream_t st);

}  // namespace dsrt

using namespace dsrt;

extern "C" int dsrt_hash(const void *X, int x_dtype, int64_t n, int d, const void *planes,
                         int mode, int L, int C, void *codes_out, uint32_t *records_out,
                         uint32_t *zero_rows, void *stream) {
    DSRT_REQUIRE(d >= 1, DSRT_EINVAL, "invalid parameter: d must be >= 1, got %d", d);
    DSRT_REQUIRE(C >= 1 && C <= 24, DSRT_EINVAL, "invalid parameter: C must be in [1, 24], got %d", C);
    DSRT_REQUIRE(L >= 1, DSRT_EINVAL, "invalid parameter: L must be >= 1, got %d", L);
    DSRT_REQUIRE(n >= 0, DSRT_EINVAL, "invalid parameter: n < 0");
    DSRT_REQUIRE(L * C <= 32 * kMaxBitWords, DSRT_EUNSUPPORTED,
                 "invalid parameter: L*C=%d exceeds %d hash bits per vector", L * C, 32 * kMaxBitWords);
    if (n == 0) return DSRT_OK;
    cudaStream_t st = as_stream(stream);
    if (mode == DSRT_HASH_TC_FIX)
        return hash_fix(X, x_dtype, n, d, planes, L, C, codes_out, records_out, zero_rows, st);
    if (mode == DSRT_HASH_TC_BF16X2 || mode == DSRT_HASH_TC_F16X2)
        return hash_tc(X, x_dtype, n, d, planes, mode, L, C, codes_out, records_out, zero_rows, st);
    DSRT_REQUIRE(mode == DSRT_HASH_F64 || mode == DSRT_HASH_F32, DSRT_EINVAL,
                 "invalid parameter: hash mode %d", mode);
    const bool f64 = mode == DSRT_HASH_F64;
    switch (x_dtype) {
        case DSRT_F32:
            return f64 ? launch_hash<float, double>(X, n, d, planes, L, C, codes_out, records_out, zero_rows, st)
                       : launch_hash<float, float>(X, n, d, planes, L, C, codes_out, records_out, zero_rows, st);
        case DSRT_F64:
            return f64 ? launch_hash<double, double>(X, n, d, planes, L, C, codes_out, records_out, zero_rows, st)
                       : launch_hash<double, float>(X, n, d, planes, L, C, codes_out, records_out, zero_rows, st);
        case DSRT_F16:
            return f64 ? launch_hash<__half, double>(X, n, d, planes, L, C, codes_out, records_out, zero_rows, st)
                       : launch_hash<__half, float>(X, n, d, planes, L, C, codes_out, records_out, zero_rows, st);
        case DSRT_BF16:
            return f64 ? launch_hash<__nv_bfloat16, double>(X, n, d, planes, L, C, codes_out, records_out, zero_rows, st)
                       : launch_hash<__nv_bfloat16, float>(X, n, d, planes, L, C, codes_out, records_out, zero_rows, st);
        default: break;
    }
    set_error("invalid parameter: x dtype %d", x_dtype);
    return DSRT_EINVAL;
}
