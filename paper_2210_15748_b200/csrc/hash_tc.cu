// K1 tensor-core modes -- SRP hashing as a tcgen05 GEMM with a fused
// sign-and-pack epilogue (replaces lsh.hash_matrix, lsh.py:90-106, for
// fp16/bf16 inputs; the cfg-2 index-build throughput path).
//
//   D[row, p] = sum_k X[row, k] * W[p, k]      (fp32 accumulate in TMEM)
//   bit[row, p] = D > 0;  code_t = sum_c bit[t*C + c] << c
//
// Planes are split into "parts" (hi/lo) so the fp16/bf16 operand rounding of
// the float64 reference planes stays far inside the allowed band
// |w.x| < 1e-4 |w||x|:  W = W_hi + W_lo, D = X.W_hi^T + X.W_lo^T (two MMA
// chains into the same accumulator).  fp16/bf16 X is exact (the reference
// hashes the same values cast to float64).
//
// Decomposition: the L tables split into column groups of 32 tables (one
// plane word each, N_g = 32*C <= 256 MMA columns, plane-major: column
// b*32 + t = bit b of table t, so one 32-column TMEM load is one plane word;
// the planes are permuted into that order per call).  CTA c handles
// group c % G for the 128-row tiles c/G, c/G + n_cta/G, ...  -- consecutive
// CTAs share each X tile through L2.  Warp roles (320 threads):
//   warp 0: TMA producer (3-stage ring of X tiles, planes loaded once),
//   warp 1: MMA issuer (one thread, 8 K-steps x parts per tile),
//   warps 2-5: epilogue (TMEM -> registers -> sign bits -> codes + plane
//              records), TMEM double-buffered so it overlaps the next MMAs; the
//              load of plane word b + 1 is in flight while word b is packed.
//              The planes are stored negated, so the accumulator's sign bit is
//              the hash bit (one funnel shift per value).
// Measured bounds at cfg2 (10M bf16 rows, codes + records): 1.60 ms; the MMA/TMA
// pipeline alone (no accumulator read-out) 1.42-1.49 ms at the ~1.4 GHz the SMs
// hold under this tensor load, so the kernel is tensor-bound on its two chains.
// One chain with the same epilogue (timing build DSRT_HASH_EXP_PARTS1, wrong
// bits) takes 1.37 ms: reading 128 x 32C fp32 accumulators out of TMEM and the
// bit transposes then pace it, so halving the MMA work cannot halve the time.
// A second epilogue warp set on alternate tiles (DSRT_HASH_ESETS=2) is slower
// (1.84 ms: 10 warps cap the kernel at 168 registers and it spills).
#include <cstdlib>

#include "tc_common.cuh"

namespace dsrt {

#ifndef DSRT_HASH_ESETS
#define DSRT_HASH_ESETS 1  // 2 (measured): 10 warps cap the kernel at 168 registers, it spills, 1.60 -> 2.20 ms
#endif
constexpr int kHESets = DSRT_HASH_ESETS;         // epilogue warp sets (4 warps each)
constexpr int kHThreads = 64 + 128 * kHESets;

struct HashTcParams {
    int64_t n_rows;
    int L, Cr, groups, n_pad;  // n_pad = padded MMA N per group (multiple of 16)
    int parts;
    void *codes_out;          // uint8 (n, L)   (C <= 8)
    uint32_t *recs_out;       // (n, R)
    uint32_t *zero_rows;
    int mc;  // > 1: the `groups` CTAs of a cluster share every X tile by TMA multicast
};

template <int PARTS, int C, int kHStages>
__global__ void __launch_bounds__(kHThreads, 1)
    hash_tc_kernel(const __grid_constant__ CUtensorMap map_x,
                   const __grid_constant__ CUtensorMap map_w, HashTcParams p, uint32_t idesc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int NP = p.n_pad;
    constexpr int kTileA = 2 * 128 * 128;                 // two 64-column blocks
    uint8_t *sa = smem;                                    // kHStages x kTileA
    uint8_t *sb = smem + kHStages * kTileA;                // PARTS x 2 x (NP x 128 B)
    __shared__ uint64_t full[kHStages], empty[kHStages], tfull[2], tempty[2], bar_b;
    __shared__ uint32_t tmem_base;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int group = blockIdx.x % p.groups;
    const int cta_in_group = blockIdx.x / p.groups;
    const int ctas_per_group = gridDim.x / p.groups;
    const int64_t n_tiles = (p.n_rows + 127) / 128;

    if (threadIdx.x == 0) {
        tma_prefetch(&map_x);
        tma_prefetch(&map_w);
        for (int s = 0; s < kHStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], p.mc > 1 ? p.mc : 1);  // multicast: every CTA's MMA frees the stage
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);  // 4 epilogue warps
        }
        mbar_init(&bar_b, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(&tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    if (p.mc > 1) cluster_sync_all();  // peers' barriers are initialised before any multicast
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    const uint16_t cmask = static_cast<uint16_t>((1u << p.mc) - 1u);

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            const int prow = group * 32 * C;  // first plane row of this group
            mbar_arrive_expect_tx(&bar_b, PARTS * 2 * NP * 128);
            for (int part = 0; part < PARTS; ++part)
                for (int kb = 0; kb < 2; ++kb)
                    tma_load_2d(sb + (part * 2 + kb) * NP * 128, &map_w, kb * 64,
                                part * (p.groups * 32 * C) + prow, &bar_b);
            int it = 0;
            for (int64_t tile = cta_in_group; tile < n_tiles; tile += ctas_per_group, ++it) {
                const int st = it % kHStages;
                if (it >= kHStages) mbar_wait(&empty[st], ((it / kHStages) - 1) & 1);
                mbar_arrive_expect_tx(&full[st], kTileA);
                if (p.mc > 1) {  // X read once: CTA (group) g multicasts the 64-column boxes kb = g mod G
                    for (int kb = group; kb < 2; kb += p.mc)
                        tma_load_2d_mc(sa + st * kTileA + kb * 128 * 128, &map_x, kb * 64,
                                       static_cast<int>(tile * 128), &full[st], cmask);
                } else {
                    tma_load_2d(sa + st * kTileA, &map_x, 0, static_cast<int>(tile * 128), &full[st]);
                    tma_load_2d(sa + st * kTileA + 128 * 128, &map_x, 64, static_cast<int>(tile * 128),
                                &full[st]);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            mbar_wait(&bar_b, 0);
            int it = 0;
            for (int64_t tile = cta_in_group; tile < n_tiles; tile += ctas_per_group, ++it) {
                const int st = it % kHStages, acc = it & 1;
                mbar_wait(&full[st], (it / kHStages) & 1);
                if (it >= 2) mbar_wait(&tempty[acc], ((it >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t d = tmem + acc * 256;
#ifdef DSRT_HASH_EXP_PARTS1  // timing experiment only (wrong bits): one MMA chain instead of hi + lo
                constexpr int kParts = 1;
#else
                constexpr int kParts = PARTS;
#endif
                for (int part = 0; part < kParts; ++part)
                    for (int kb = 0; kb < 2; ++kb) {
                        const uint64_t ad = umma_desc_sw128(sa + st * kTileA + kb * 128 * 128);
                        const uint64_t bd = umma_desc_sw128(sb + (part * 2 + kb) * NP * 128);
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            umma_f16(d, ad + 2 * k, bd + 2 * k, idesc, (part | kb | k) != 0);
                    }
                if (p.mc > 1)
                    umma_commit_mc(&empty[st], cmask);
                else
                    umma_commit(&empty[st]);
                umma_commit(&tfull[acc]);
            }
        }
    } else {
        // ------------------------------------------------ epilogue (warps 2..5 and 6..9)
        const int quarter = warp & 3;   // TMEM lanes 32*quarter .. +31
        const int eset = (warp - 2) >> 2;  // set 0: even tiles (accumulator 0), set 1: odd tiles
        const int L = p.L;
        const int t0 = group * 32;
        const int nt = min(32, L - t0);
        const uint32_t tmask = nt == 32 ? 0xffffffffu : ((1u << nt) - 1u);
        const int W = (L + 31) >> 5, R = ((C * W) + 3) & ~3;
        int it = 0;
        constexpr int NB = kHESets == 1 ? 2 : 1;
        uint32_t r[NB][32];
        for (int64_t tile = cta_in_group; tile < n_tiles; tile += ctas_per_group, ++it) {
            const int acc = it & 1;
            if (kHESets == 2 && acc != eset) continue;
            mbar_wait(&tfull[acc], (it >> 1) & 1);
            tc_fence_after();
            const int64_t row = tile * 128 + quarter * 32 + lane;
            uint32_t plane[C];
#pragma unroll
            for (int b = 0; b < C; ++b) plane[b] = 0;
            uint32_t codes_w[8];  // 32 tables x 8-bit codes
            uint32_t any_nonzero = 0;
            const uint32_t base = tmem + acc * 256 + (static_cast<uint32_t>(quarter * 32) << 16);
            // chunk b = plane word b (32 tables); sign bits gathered by funnel shifts
            bool want_zero = group == 0 && p.zero_rows != nullptr;
            // The planes are stored negated (permute_planes_kernel), so the accumulator
            // holds -w.x and its sign bit is the hash bit: one funnel shift per value.
            // The load of plane word b + 1 is in flight while word b is packed.
            // one set: double-buffered, the next word's load is in flight while this one is
            // packed; two sets would hide the load latency behind each other and use one
            // buffer (10 warps leave 168 registers per thread)
#ifdef DSRT_HASH_EXP_NOLD  // timing experiment only: no accumulator read-out at all
#pragma unroll
            for (int j = 0; j < 32; ++j) r[0][j] = r[NB - 1][j] = 0;
#else
            tmem_ld32(base, r[0]);
#endif
#pragma unroll
            for (int b = 0; b < C; ++b) {
                uint32_t(&rb)[32] = r[b % NB];
#ifndef DSRT_HASH_EXP_NOLD
                tmem_wait_ld_dep(rb);
                if (NB == 2 && b + 1 < C) tmem_ld32(base + (b + 1) * 32, r[(b + 1) % NB]);
#endif
                uint32_t pw = 0;
#ifdef DSRT_HASH_EXP_NOPACK  // timing experiment only: TMEM loads without the sign packing
                pw = rb[0] ^ rb[31];
#else
#pragma unroll
                for (int j = 31; j >= 0; --j) pw = __funnelshift_l(rb[j], pw, 1);
#endif
                plane[b] = pw & tmask;
                if (want_zero) {  // rows whose first word is all +-0 check every column (rare)
#pragma unroll
                    for (int j = 0; j < 32; ++j) any_nonzero |= rb[j];
                    if (b == 0) want_zero = __any_sync(0xffffffffu, (any_nonzero & 0x7fffffffu) == 0u);
                }
#ifndef DSRT_HASH_EXP_NOLD
                if (NB == 1 && b + 1 < C) tmem_ld32(base + (b + 1) * 32, rb);
#endif
            }
            any_nonzero &= 0x7fffffffu;
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (p.codes_out) codes_from_planes<C>(plane, codes_w);  // 8x8 bit transposes
            if (row < p.n_rows) {
                if (p.codes_out) {
                    uint8_t *dst = static_cast<uint8_t *>(p.codes_out) + row * L + t0;
                    if (nt == 32 && (L & 15) == 0) {
                        uint4 *d4 = reinterpret_cast<uint4 *>(dst);
                        d4[0] = make_uint4(codes_w[0], codes_w[1], codes_w[2], codes_w[3]);
                        d4[1] = make_uint4(codes_w[4], codes_w[5], codes_w[6], codes_w[7]);
                    } else {
#pragma unroll
                        for (int t = 0; t < 32; ++t)
                            if (t < nt) dst[t] = (codes_w[t >> 2] >> (8 * (t & 3))) & 0xffu;
                    }
                }
                if (p.recs_out) {
                    uint32_t *rec = p.recs_out + row * R;
#pragma unroll
                    for (int b = 0; b < C; ++b) rec[b * W + group] = plane[b];
                    if (group == 0)
                        for (int i = C * W; i < R; ++i) rec[i] = 0;
                }
                if (group == 0 && p.zero_rows && any_nonzero == 0) atomicAdd(p.zero_rows, 1u);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (p.mc > 1) cluster_sync_all();  // no CTA leaves while peers may still multicast into it
    if (warp == 1) tmem_dealloc(tmem, 512);
}

template <int PARTS, int C, int STAGES>
static int launch_hash_tc(const CUtensorMap &mx, const CUtensorMap &mw, const HashTcParams &hp,
                          uint32_t idesc, size_t smem, int ctas, cudaStream_t st);

// reference plane order (row t*C + b per part) -> plane-major groups (row
// g*32*C + b*32 + t), negated, zero planes for tables >= L.  16-bit elements.
__global__ void permute_planes_kernel(const uint16_t *__restrict__ src, int parts, int L, int C,
                                      int groups, uint16_t *__restrict__ dst) {
    const int64_t rows = static_cast<int64_t>(parts) * groups * 32 * C;
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= rows * 128) return;
    const int64_t row = i >> 7;
    const int k = static_cast<int>(i & 127);
    const int per_part = groups * 32 * C;
    const int part = static_cast<int>(row / per_part);
    const int rem = static_cast<int>(row % per_part);
    const int g = rem / (32 * C), b = (rem % (32 * C)) / 32, t = rem % 32;
    const int tg = g * 32 + t;
    // sign bit flipped (fp16 and bf16 alike): the MMA accumulates -w.x, whose sign bit is the hash bit
    dst[i] = tg < L ? uint16_t(src[(static_cast<int64_t>(part) * L * C + tg * C + b) * 128 + k] ^ 0x8000u)
                    : uint16_t(0);
}

static int launch_hash_tc_c(int C, int /*parts: always 2 (hi/lo)*/, int stages, const CUtensorMap &mx,
                            const CUtensorMap &mw, const HashTcParams &hp, uint32_t idesc,
                            size_t smem, int ctas, cudaStream_t st) {
#define DSRT_HC(c)                                                                            \
    case c:                                                                                   \
        return stages == 3 ? launch_hash_tc<2, c, 3>(mx, mw, hp, idesc, smem, ctas, st)       \
                           : launch_hash_tc<2, c, 2>(mx, mw, hp, idesc, smem, ctas, st);
    switch (C) {
        DSRT_HC(1) DSRT_HC(2) DSRT_HC(3) DSRT_HC(4) DSRT_HC(5) DSRT_HC(6) DSRT_HC(7) DSRT_HC(8)
        default: break;
    }
#undef DSRT_HC
    set_error("invalid parameter: tensor-core hash needs C <= 8, got %d", C);
    return DSRT_EUNSUPPORTED;
}

int hash_tc(const void *X, int x_dtype, int64_t n, int d, const void *planes, int mode, int L,
            int C, void *codes_out, uint32_t *records_out, uint32_t *zero_rows, cudaStream_t st) {
    const bool bf16 = mode == DSRT_HASH_TC_BF16X2;
    const int parts = 2;
    DSRT_REQUIRE(x_dtype == (bf16 ? DSRT_BF16 : DSRT_F16), DSRT_EINVAL,
                 "invalid parameter: tensor-core hash mode %d needs %s vectors", mode,
                 bf16 ? "bf16" : "fp16");
    DSRT_REQUIRE(d == 128, DSRT_EUNSUPPORTED, "invalid parameter: tensor-core hash needs d=128, got %d", d);
    DSRT_REQUIRE(C <= 8, DSRT_EUNSUPPORTED, "invalid parameter: tensor-core hash needs C <= 8, got %d", C);
    DSRT_REQUIRE(n < (1LL << 31), DSRT_EUNSUPPORTED, "invalid parameter: too many rows for one call");
    const int groups = (L + 31) / 32;
    const int n_pad = 32 * C;  // plane-major group: 32 tables per plane word
    DSRT_REQUIRE(n_pad <= 256, DSRT_EUNSUPPORTED, "invalid parameter: MMA N too large");
    const CUtensorMapDataType dt = bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    const int64_t prow = static_cast<int64_t>(parts) * groups * 32 * C;
    uint16_t *pp = nullptr;
    DSRT_CUDA(malloc_async(reinterpret_cast<void **>(&pp), prow * 128 * sizeof(uint16_t), st));
    permute_planes_kernel<<<static_cast<unsigned>((prow * 128 + 255) / 256), 256, 0, st>>>(
        static_cast<const uint16_t *>(planes), parts, L, C, groups, pp);
    DSRT_LAUNCH_CHECK();
    CUtensorMap mx, mw;
    int rc = make_tmap_2d(&mx, X, dt, 128, static_cast<uint64_t>(n), 256, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc == DSRT_OK)
        rc = make_tmap_2d(&mw, pp, dt, 128, static_cast<uint64_t>(prow), 256, 64, n_pad,
                          CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) {
        cudaFreeAsync(pp, st);
        return rc;
    }
    // X tiles are shared by the groups' CTAs through a cluster + TMA multicast (each X
    // byte read from HBM once); DSRT_HASH_MC=0 restores independent loads (A/B timing)
    const char *mce = getenv("DSRT_HASH_MC");
    const int mc = (groups >= 2 && groups <= 8 && !(mce && mce[0] == '0')) ? groups : 1;
    HashTcParams hp{n, L, C, groups, n_pad, parts, codes_out, records_out, zero_rows, mc};
    const size_t b_bytes = static_cast<size_t>(parts) * 2 * n_pad * 128;
    const int stages = (1024 + 3 * 2 * 128 * 128 + b_bytes <= 227 * 1024) ? 3 : 2;
    const size_t smem = 1024 + stages * 2 * 128 * 128 + b_bytes;
    const int64_t n_tiles = (n + 127) / 128;
    int ctas = sm_count() * 1;
    ctas = ctas - ctas % groups;
    ctas = static_cast<int>(tmin<int64_t>(ctas, n_tiles * groups));
    ctas = tmax(ctas, groups);
    const uint32_t idesc = idesc_f16(128, n_pad, bf16, bf16);
    rc = launch_hash_tc_c(C, parts, stages, mx, mw, hp, idesc, smem, ctas, st);
    cudaFreeAsync(pp, st);  // stream-ordered: freed after the kernel
    return rc;
}

template <int PARTS, int C, int STAGES>
static int launch_hash_tc(const CUtensorMap &mx, const CUtensorMap &mw, const HashTcParams &hp,
                          uint32_t idesc, size_t smem, int ctas, cudaStream_t st) {
    auto kern = hash_tc_kernel<PARTS, C, STAGES>;
    DSRT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (hp.mc > 1) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(ctas));
        cfg.blockDim = dim3(kHThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = static_cast<unsigned>(hp.mc);
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        DSRT_CUDA(cudaLaunchKernelEx(&cfg, kern, mx, mw, hp, idesc));
    } else {
        kern<<<ctas, kHThreads, smem, st>>>(mx, mw, hp, idesc);
    }
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}

}  // namespace dsrt
