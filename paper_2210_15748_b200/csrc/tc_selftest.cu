// tcgen05 plumbing: tensor-map creation and a diagnostic GEMM
// D(M,N) = A(M,128) . B(N,128)^T (fp16/bf16 in, fp32 out) that exercises
// exactly the TMA -> SWIZZLE_128B smem -> UMMA descriptor -> TMEM -> tcgen05.ld
// chain used by the hashing and prefilter kernels (dsrt_tc_selftest).
#include <mutex>

#include "tc_common.cuh"

namespace dsrt {

typedef CUresult (*PFN_tmapEncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                        const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                        const cuuint32_t *, CUtensorMapInterleave,
                                        CUtensorMapSwizzle, CUtensorMapL2promotion,
                                        CUtensorMapFloatOOBfill);

static PFN_tmapEncodeTiled encode_fn() {
    static PFN_tmapEncodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_tmapEncodeTiled>(p);
    });
    return fn;
}

int make_tmap_2d(CUtensorMap *map, const void *base, CUtensorMapDataType dtype, uint64_t inner,
                 uint64_t outer, uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer,
                 CUtensorMapSwizzle swizzle) {
    PFN_tmapEncodeTiled fn = encode_fn();
    DSRT_REQUIRE(fn != nullptr, DSRT_ECUDA, "cuda error: cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_stride_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, dtype, 2, const_cast<void *>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    DSRT_REQUIRE(r == CUDA_SUCCESS, DSRT_ECUDA, "cuda error: cuTensorMapEncodeTiled failed (%d)", (int)r);
    return DSRT_OK;
}

// One CTA per 128-row tile of A; B (N <= 256 rows) loaded whole.  128 threads.
__global__ void __launch_bounds__(128)
    tc_selftest_kernel(const __grid_constant__ CUtensorMap map_a,
                       const __grid_constant__ CUtensorMap map_b, float *__restrict__ D, int M,
                       int N, uint32_t idesc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sa = smem;                   // 2 x (128 x 128 B)
    uint8_t *sb = smem + 2 * 128 * 128;   // 2 x (N x 128 B)
    __shared__ uint64_t bar_load, bar_mma;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * 128;
    if (threadIdx.x == 0) {
        tma_prefetch(&map_a);
        tma_prefetch(&map_b);
        mbar_init(&bar_load, 1);
        mbar_init(&bar_mma, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(&tmem_base, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar_load, 2 * 128 * 128 + 2 * N * 128);
        tma_load_2d(sa, &map_a, 0, m0, &bar_load);
        tma_load_2d(sa + 128 * 128, &map_a, 64, m0, &bar_load);
        tma_load_2d(sb, &map_b, 0, 0, &bar_load);
        tma_load_2d(sb + N * 128, &map_b, 64, 0, &bar_load);
        mbar_wait(&bar_load, 0);
        tc_fence_after();
        for (int kb = 0; kb < 2; ++kb) {
            const uint64_t ad = umma_desc_sw128(sa + kb * 128 * 128);
            const uint64_t bd = umma_desc_sw128(sb + kb * N * 128);
            for (int k = 0; k < 4; ++k)
                umma_f16(tmem, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
        }
        umma_commit(&bar_mma);
    }
    __syncwarp();
    mbar_wait(&bar_mma, 0);
    tc_fence_after();
    const int row = m0 + warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, r);
        tmem_wait_ld();
        if (row < M)
            for (int j = 0; j < 32 && c0 + j < N; ++j) D[static_cast<int64_t>(row) * N + c0 + j] = __uint_as_float(r[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 256);
}

}  // namespace dsrt

using namespace dsrt;

extern "C" int dsrt_tc_selftest(const void *A, int a_bf16, const void *B, int b_bf16, float *D,
                                int M, int N, void *stream) {
    DSRT_REQUIRE(M >= 1 && N >= 16 && N <= 256 && N % 16 == 0, DSRT_EINVAL,
                 "invalid parameter: M=%d N=%d (N in [16,256], multiple of 16)", M, N);
    // kind::f16 needs matching A/B formats (mixed fp16 x bf16 traps on sm_100a)
    DSRT_REQUIRE(a_bf16 == b_bf16, DSRT_EINVAL, "invalid parameter: A and B must share fp16/bf16");
    CUtensorMap ma, mb;
    const CUtensorMapDataType ta = a_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    const CUtensorMapDataType tb = b_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    int rc = make_tmap_2d(&ma, A, ta, 128, M, 256, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    rc = make_tmap_2d(&mb, B, tb, 128, N, 256, 64, N, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    const size_t smem = 1024 + 2 * 128 * 128 + 2 * 256 * 128;
    DSRT_CUDA(cudaFuncSetAttribute(tc_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    tc_selftest_kernel<<<(M + 127) / 128, 128, smem, as_stream(stream)>>>(
        ma, mb, D, M, N, idesc_f16(128, N, a_bf16, b_bf16));
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}
