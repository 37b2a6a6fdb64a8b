// K1 tensor-core mode DSRT_HASH_TC_FIX -- SRP hashing (lsh.hash_matrix,
// lsh.py:90-106) as ONE fp16 tcgen05 GEMM per tile with an exact fix-up of the
// few sign bits the fp16 rounding of the planes can change.  The cfg-2
// index-build path (fp16 or bf16 vectors, d = 128, C <= 8).
//
//   planes  w (float64, the reference's own, lsh.py:64-65) are multiplied by a
//           per-plane positive scale s_p = 2^-6 (1 + j/64), j chosen to minimise
//           the relative fp16 rounding error of that plane (a positive scale never
//           changes a sign), and split on the device into hi = fp16(s_p w) (the MMA
//           operand, resident in shared memory) and lo = s_p w - hi (stored as
//           e4m3(lo 2^E) with one power-of-two scale, read by the fix-up).
//   vectors x: fp16 rows are used as they are; bf16 rows are scaled by a power of
//           two that puts their largest |element| in [0.5, 1) and rounded to fp16
//           in shared memory (exact except for elements below 2^-14, whose error
//           is at most 2^-25 each) -- again a positive scale per row.
//   D = x^ . hi  (fp32 accumulate in TMEM).  For plane p in plane word (g, b):
//     |D - x.w| <= t = |x^| c_gb + 128 * 2^-25 max|hi|,
//     c_gb = 1.001 max_{p in word} (|lo_p| + 2e-5 |hi_p|)
//     (Cauchy-Schwarz on the lo part; <= 128 * 2^-23 * sum |x^_i hi_i| for the
//     tensor-core fp32 accumulation; the conversion term for bf16 rows).
//   |D| >= t  ->  sign(D) is the sign of x.w: the bit is ~MSB(D).
//   |D| <  t  ->  "flagged": the bit is recomputed as
//                 v = sum x^_i hi_i + 2^-E sum x^_i lo8_i  (fp32 FHFMA chains; the
//                 e4m3 lo adds <= 2^-4 |x^||lo_p| <= 3.1e-5 |x||w|), so a GPU bit can
//                 differ from the float64 reference only where |x.w| < 5e-5 |w||x|
//                 -- inside the north star's 1e-4 band.  ~0.3 % of the bits are
//                 flagged for unit-norm data (about 1.3 per 448-bit row).
//
// vs the hi/lo kernel (hash_tc.cu, modes 3/4): half the MMA work (one operand
// pass instead of two) and every X tile is read once (all table groups' hi
// planes are resident in one CTA), at the cost of the flag test (a third
// instruction per accumulator value) and the fix-ups.  Measured on cfg2
// (10M bf16 rows, L=64 C=7): 3.2-3.8 ms vs 1.82 ms for hi/lo -- the epilogue,
// not the tensor pipe, bounds this kernel (0.91 ms with the epilogue removed),
// so hi/lo stays the default and this mode is opt-in (K1).
//
// Warp roles (448 threads, one persistent CTA per SM):
//   warp 0       TMA producer: hi planes once, then a ring of 128-row X tiles
//   warp 1       MMA issuer: per (tile, 32-table group g) one N = 32C chain of
//                8 K-steps into TMEM buffer g % 2 (256 columns each)
//   warps 2-5    converters: thread per row; bf16 -> scaled fp16 in place, row
//                norm, zero-row count
//   warps 6-13   epilogue: thread per row (TMEM lane quarter = warp % 4); warp
//                set h = 0 / 1 takes the groups g = h (mod 2) of every tile;
//                sign and flag words per 32 columns (funnel shifts of MSB(D) and
//                of MSB(2 bits(D) - 2 bits(t))), a per-warp queue of flagged
//                (row, plane) items recomputed lane-per-item, then records and
//                u8 codes (8x8 bit transposes) staged in the quarter's freed X
//                rows and written with coalesced 16-byte stores.
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include "tc_common.cuh"

namespace dsrt {

namespace {

constexpr int kFThreads = 448;
constexpr int kTileX = 2 * 128 * 128;  // one 128-row x 128-dim fp16/bf16 tile (two 64-col blocks)
constexpr int kQCap = 128;             // per-warp fix-up queue entries
constexpr int kEpi = 8;                // epilogue warps
constexpr unsigned kFull32 = 0xffffffffu;
constexpr int kStatWords = 8;          // header words of the stats block

struct FixParams {
    int64_t n_rows;
    int L, G, NP;             // tables, 32-table groups, MMA N per group (= 32 C)
    void *codes_out;          // uint8 (n, L)
    uint32_t *recs_out;       // (n, R)
    uint32_t *zero_rows;
    const uint8_t *lo8;       // (G * NP, 128) e4m3(lo 2^E), plane-major group order
    const float *stats;       // [0] max|hi_i|, [1] E, [2] max|lo_i|, [8 + g*8 + b] c_gb
};

__device__ __forceinline__ float fhfma(uint32_t a, uint32_t b, float c) {
    // c + a.lo * b.lo + a.hi * b.hi, fp16 inputs, fp32 accumulation (FHFMA)
    asm("{.reg .b16 al, ah, bl, bh;\n\t"
        "mov.b32 {al, ah}, %1;\n\tmov.b32 {bl, bh}, %2;\n\t"
        "fma.rn.f32.f16 %0, al, bl, %0;\n\tfma.rn.f32.f16 %0, ah, bh, %0;}"
        : "+f"(c)
        : "r"(a), "r"(b));
    return c;
}

// 2 x - t on the FMA pipe (IMAD) rather than the ALU pipe, which the sign and
// flag funnel shifts already load
__device__ __forceinline__ uint32_t mad2(uint32_t x, uint32_t neg_t) {
    uint32_t y;
    asm("mad.lo.u32 %0, %1, 2, %2;" : "=r"(y) : "r"(x), "r"(neg_t));
    return y;
}

// mbarrier wait with a short sleep between polls: the single-thread producer and
// issuer loops would otherwise take issue slots from the epilogue warps
// (try_wait with a suspend-time hint: the warp is descheduled until the phase
// completes or the hint expires, instead of re-issuing the poll)
__device__ __forceinline__ void mbar_wait_backoff(uint64_t *bar, uint32_t parity, int /*unused*/) {
    uint32_t ok;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity), "r"(0x989680u)
            : "memory");
    } while (!ok);
}

// named barrier of the two epilogue warps sharing a TMEM lane quarter
__device__ __forceinline__ void pair_sync(int id) {
    asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}

// 4 e4m3 values (bytes of w, lowest first) -> two f16x2 words
__device__ __forceinline__ void e4m3x4_to_f16x2(uint32_t w, uint32_t &a, uint32_t &b) {
    asm("{.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\t"
        "cvt.rn.f16x2.e4m3x2 %0, l;\n\tcvt.rn.f16x2.e4m3x2 %1, h;}"
        : "=r"(a), "=r"(b)
        : "r"(w));
}

// 16-byte chunk c (0..15) of row r in a SWIZZLE_128B K-major tile of `rows` rows
// stored as two 64-column blocks (block stride rows * 128 B).
__device__ __forceinline__ const uint4 *sw_chunk(const uint8_t *tile, int rows, int r, int c) {
    return reinterpret_cast<const uint4 *>(tile + (c >> 3) * rows * 128 + r * 128 +
                                           (((c & 7) ^ (r & 7)) << 4));
}

template <int C, int S, bool BF16>
__global__ void __launch_bounds__(kFThreads, 1)
    hash_fix_kernel(const __grid_constant__ CUtensorMap map_x,
                    const __grid_constant__ CUtensorMap map_w, FixParams p, uint32_t idesc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment by pointer arithmetic (keeps the shared address space
    // visible to the compiler: LDS, not generic loads)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int NP = p.NP, G = p.G;
    uint8_t *sa = smem;                        // S x kTileX
    uint8_t *sb = smem + S * kTileX;           // G x 2 x (NP x 128 B)
    // rowinfo: S x 128 x {|x^| (float, rounded up), mode 0 normal / 1 flag all / 2 none}
    uint32_t *rowinfo = reinterpret_cast<uint32_t *>(sb + static_cast<size_t>(G) * 2 * NP * 128);
    uint16_t *queue = reinterpret_cast<uint16_t *>(rowinfo + S * 256);  // kEpi x kQCap
    uint32_t *corr = reinterpret_cast<uint32_t *>(queue + kEpi * kQCap);  // kEpi x 32 rows x 8 words
    float *coef_s = reinterpret_cast<float *>(corr + kEpi * 32 * 8);      // G x 8 (c_gb)
    __shared__ uint64_t full[S], conv[S], xempty[S], tfull[2], tempty[2], bar_b;
    __shared__ uint32_t tmem_base;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t n_tiles = (p.n_rows + 127) / 128;

    if (threadIdx.x == 0) {
        tma_prefetch(&map_x);
        tma_prefetch(&map_w);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&conv[s], 4);
            mbar_init(&xempty[s], kEpi);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], kEpi / 2);
        }
        mbar_init(&bar_b, 1);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < kEpi * 32 * 8; i += kFThreads) corr[i] = 0;
    for (int i = threadIdx.x; i < G * 8; i += kFThreads) coef_s[i] = p.stats[kStatWords + i];
    if (warp == 1) tmem_alloc(&tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            mbar_arrive_expect_tx(&bar_b, G * 2 * NP * 128);
            for (int g = 0; g < G; ++g)
                for (int kb = 0; kb < 2; ++kb)
                    tma_load_2d(sb + (g * 2 + kb) * NP * 128, &map_w, kb * 64, g * NP, &bar_b);
            int it = 0;
            for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
                const int st = it % S;
                if (it >= S) mbar_wait_backoff(&xempty[st], ((it / S) - 1) & 1, 128);
                mbar_arrive_expect_tx(&full[st], kTileX);
                tma_load_2d(sa + st * kTileX, &map_x, 0, static_cast<int>(tile * 128), &full[st]);
                tma_load_2d(sa + st * kTileX + 128 * 128, &map_x, 64, static_cast<int>(tile * 128),
                            &full[st]);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            mbar_wait(&bar_b, 0);
            int it = 0;
            uint32_t uses[2] = {0u, 0u};  // buffer b serves the groups g = b (mod 2)
            for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
                const int st = it % S;
                mbar_wait_backoff(&conv[st], (it / S) & 1, 32);
                tc_fence_after();
                for (int g = 0; g < G; ++g) {
                    const int buf = g & 1;
                    if (uses[buf] >= 1) mbar_wait_backoff(&tempty[buf], (uses[buf] - 1) & 1, 32);
                    ++uses[buf];
                    tc_fence_after();
                    const uint32_t d = tmem + buf * 256;
#pragma unroll
                    for (int kb = 0; kb < 2; ++kb) {
                        const uint64_t ad = umma_desc_sw128(sa + st * kTileX + kb * 128 * 128);
                        const uint64_t bd = umma_desc_sw128(sb + (g * 2 + kb) * NP * 128);
#pragma unroll
                        for (int k = 0; k < 4; ++k) umma_f16(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
                    }
                    umma_commit(&tfull[buf]);
                }
            }
        }
    } else if (warp < 6) {
        // ------------------------------------------------ converters (thread per row)
        const int r = (warp - 2) * 32 + lane;
        int it = 0;
        for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
            const int st = it % S;
            mbar_wait_backoff(&full[st], (it / S) & 1, 32);
            uint8_t *xt = sa + st * kTileX;
            uint4 v[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) v[c] = *sw_chunk(xt, 128, r, c);
            float n4[4] = {0.0f, 0.0f, 0.0f, 0.0f};  // four partial sums of squares (ILP)
            bool nonfinite = false, zero = false;
#ifdef DSRT_FIX_NOCONV  // timing experiment only: no bf16 conversion (wrong bits)
            if constexpr (false) {
#else
            if constexpr (BF16) {
#endif
                uint32_t m = 0;
#pragma unroll
                for (int c = 0; c < 16; ++c)
                    m = max(m, __vmaxu2(__vmaxu2(v[c].x & 0x7fff7fffu, v[c].y & 0x7fff7fffu),
                                        __vmaxu2(v[c].z & 0x7fff7fffu, v[c].w & 0x7fff7fffu)));
                m = max(m & 0xffffu, m >> 16);
                nonfinite = m >= 0x7f80u;
                zero = m == 0u;
                float s1 = 1.0f, s2 = 1.0f;
                if (!nonfinite && !zero) {
                    int e;
                    frexpf(__uint_as_float(m << 16), &e);  // max = f 2^e, f in [0.5, 1)
                    if (e > -120 && e < 120) {
                        s1 = ldexpf(1.0f, -e);
                    } else {  // two factors: 2^-e may exceed the float range
                        const int k1 = (-e) / 2;
                        s1 = ldexpf(1.0f, k1);
                        s2 = ldexpf(1.0f, -e - k1);
                    }
                }
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    uint32_t w4[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float a = __uint_as_float(w4[j] << 16) * s1 * s2;
                        const float b = __uint_as_float(w4[j] & 0xffff0000u) * s1 * s2;
                        const __half2 hh = __floats2half2_rn(a, b);
                        w4[j] = *reinterpret_cast<const uint32_t *>(&hh);
                        n4[j] = fhfma(w4[j], w4[j], n4[j]);
                    }
                    *const_cast<uint4 *>(sw_chunk(xt, 128, r, c)) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
                }
                fence_proxy_async_smem();  // generic-proxy writes -> tcgen05.mma operand reads
            } else {
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    n4[0] = fhfma(v[c].x, v[c].x, n4[0]);
                    n4[1] = fhfma(v[c].y, v[c].y, n4[1]);
                    n4[2] = fhfma(v[c].z, v[c].z, n4[2]);
                    n4[3] = fhfma(v[c].w, v[c].w, n4[3]);
                }
            }
            const float nrm = (n4[0] + n4[1]) + (n4[2] + n4[3]);
            if constexpr (!BF16) {
                nonfinite = !(nrm <= 3.0e38f);
                zero = nrm == 0.0f;
            }
            const int64_t row = tile * 128 + r;
            // zero rows (an error upstream) and the TMA zero fill past n: no fix-ups
            const bool none = zero || row >= p.n_rows;
            const uint32_t mode = none ? 2u : (nonfinite ? 1u : 0u);
            // |x^| rounded up; the fp32 sum of squares is within 64 ulp (absorbed
            // by the 1.001 factor in c_gb)
            rowinfo[(st * 128 + r) * 2 + 0] = __float_as_uint(mode == 0 ? __fsqrt_ru(nrm) : 0.0f);
            rowinfo[(st * 128 + r) * 2 + 1] = mode;
            if (zero && row < p.n_rows && p.zero_rows) atomicAdd(p.zero_rows, 1u);
            __syncwarp();
            if (lane == 0) mbar_arrive(&conv[st]);
        }
    } else {
        // ------------------------------------------------ epilogue (thread per row)
        // Warp set h (warps 6-9: h = 0, 10-13: h = 1) takes the table groups g = h,
        // h + 2, ... of every tile, all C plane words each, in TMEM buffer h; so the
        // two sets work on different groups at once and need no exchange.
        const int quarter = warp & 3;        // TMEM lanes 32 * quarter .. + 31
        const int ew = warp - 6;             // 0 .. 7
        const int h = ew >> 2;
        const int rloc = quarter * 32 + lane;
        uint16_t *q = queue + ew * kQCap;
        uint32_t *cw = corr + ew * 32 * 8;
        const int L = p.L;
        const int W = (L + 31) >> 5, R = ((C * W) + 3) & ~3;
        const float lo_scale = __int_as_float((127 - static_cast<int>(p.stats[1])) << 23);  // 2^-E
        const float conv_err = BF16 ? __fmul_ru(3.814697265625e-06f, p.stats[0]) : 0.0f;  // 128 * 2^-25
        const uint8_t *lo8 = p.lo8;
        // staged outputs: one group per warp set and a quarter's records / codes fit
        // in its 32 x 128 B slice of a 64-column block
        const bool stage = G <= 2 && 32 * R * 4 <= 32 * 128 && L <= 128;
        uint32_t use = 0;  // uses of TMEM buffer h so far
        int it = 0;
        for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
            const int st = it % S;
            mbar_wait_backoff(&conv[st], (it / S) & 1, 20);
            const float xn = __uint_as_float(rowinfo[(st * 128 + rloc) * 2 + 0]);
            const uint32_t rmode = rowinfo[(st * 128 + rloc) * 2 + 1];
            const uint8_t *xt = sa + st * kTileX;
            const int64_t row = tile * 128 + rloc;
            uint32_t sw[C] = {};  // plane words of this warp's (last) group of the tile
            int gk = -1;          // that group (staged outputs)
            for (int g = h; g < G; g += 2, ++use) {
                const int t0 = g * 32;
                const int nt = min(32, L - t0);
                const uint32_t tmask = nt == 32 ? 0xffffffffu : ((1u << nt) - 1u);
                const uint8_t *lo_g = lo8 + static_cast<int64_t>(g) * NP * 128;
                // per-word thresholds t = |x^| c_gb + conv_err as -2 bits(t) (0: none),
                // parked in this lane's shared row so the rolled word loop reads them
                // with one load instead of a select chain
                uint32_t *nt_s = cw + lane * 8;  // this lane's fix-up row, free until the fix-ups
                uint32_t allm[C];
#pragma unroll
                for (int b = 0; b < C; ++b) {
                    const float t = __fmaf_ru(xn, coef_s[g * 8 + b], conv_err);
                    const uint32_t tb = __float_as_uint(t);
                    allm[b] = (rmode == 1u || (rmode == 0u && tb >= 0x40000000u)) ? kFull32 : 0u;
                    nt_s[b] = rmode == 0u ? 0u - 2u * tb : 0u;
                }
                if (C < 8) nt_s[C] = 0u;
                mbar_wait_backoff(&tfull[h], use & 1, 20);
                tc_fence_after();
                const uint32_t base = tmem + h * 256 + (static_cast<uint32_t>(quarter * 32) << 16);
                uint32_t fw[C] = {};
                // two 32-column TMEM loads in flight per wait, four packing chains
                // interleaved; rolled over word pairs (ptxas would otherwise hoist
                // every load ahead of the first use), words shifting through sw / fw
#ifdef DSRT_FIX_EPI_NONE  // timing experiment only: release TMEM without reading it
                if (false)
#endif
#pragma unroll 1
                for (int b0 = 0; b0 < C; b0 += 2) {
                    uint32_t ra[32], rb[32];
                    const bool two = b0 + 1 < C;
                    tmem_ld32(base + b0 * 32, ra);
                    if (two) tmem_ld32(base + (b0 + 1) * 32, rb);
                    tmem_wait_ld();
                    const uint32_t ta = nt_s[b0], tb2 = nt_s[b0 + 1];
                    uint32_t sa_ = 0, fa = 0, sb_ = 0, fb = 0;
#pragma unroll
                    for (int j = 31; j >= 0; --j) {
                        sa_ = __funnelshift_l(ra[j], sa_, 1);              // MSB(D): D < 0 or -0
                        fa = __funnelshift_l(mad2(ra[j], ta), fa, 1);      // 2 bits(|D|) < 2 bits(t)
                        sb_ = __funnelshift_l(rb[j], sb_, 1);
                        fb = __funnelshift_l(mad2(rb[j], tb2), fb, 1);
                    }
                    // shift the pair in (C is a compile-time constant: register arrays)
                    if (two) {
#pragma unroll
                        for (int k = 0; k + 2 < C; ++k) {
                            sw[k] = sw[k + 2];
                            fw[k] = fw[k + 2];
                        }
                        sw[C - 2] = ~sa_;
                        fw[C - 2] = fa;
                        sw[C - 1] = ~sb_;
                        fw[C - 1] = fb;
                    } else {  // odd C, last word: everything moves down by one
#pragma unroll
                        for (int k = 0; k + 1 < C; ++k) {
                            sw[k] = sw[k + 1];
                            fw[k] = fw[k + 1];
                        }
                        sw[C - 1] = ~sa_;
                        fw[C - 1] = fa;
                    }
                }
                tc_fence_before();
#pragma unroll
                for (int b = 0; b < 8; ++b) nt_s[b] = 0u;  // back to the zeroed fix-up row
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[h]);
                int cnt = 0;
#pragma unroll
                for (int b = 0; b < C; ++b) {
                    sw[b] &= tmask;
                    fw[b] = (fw[b] | allm[b]) & tmask;
                    cnt += __popc(fw[b]);
                    // warm L1 with the flagged planes' lo rows (128 B each) for the fix-ups
                    uint32_t pf = fw[b];
                    while (pf != 0u) {
                        const int t = __ffs(pf) - 1;
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(lo_g + (b * 32 + t) * 128));
                        pf &= pf - 1u;
                    }
                }
#ifdef DSRT_FIX_NOFIX  // timing experiment only: skip the fix-ups (wrong bits)
                cnt = 0;
#endif
                // ---- fix-ups of flagged (row, plane) items, lane per item
                if (__any_sync(kFull32, cnt != 0)) {
                    uint32_t pend[C];
#pragma unroll
                    for (int b = 0; b < C; ++b) pend[b] = fw[b];
                    const uint8_t *hb = sb + static_cast<size_t>(g) * 2 * NP * 128;
                    while (true) {
                        int mine = 0;
#pragma unroll
                        for (int b = 0; b < C; ++b) mine += __popc(pend[b]);
                        int incl = mine;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const int y = __shfl_up_sync(kFull32, incl, o);
                            if (lane >= o) incl += y;
                        }
                        const int total = __shfl_sync(kFull32, incl, 31);
                        if (total == 0) break;
                        int idx = incl - mine;
#pragma unroll
                        for (int b = 0; b < C; ++b) {
                            uint32_t w = pend[b];
                            while (w != 0u && idx < kQCap) {
                                const int t = __ffs(w) - 1;
                                q[idx++] = static_cast<uint16_t>(lane | (b << 5) | (t << 8));
                                w &= w - 1u;
                            }
                            pend[b] = w;
                        }
                        __syncwarp();
                        const int take = min(total, kQCap);
#pragma unroll 1
                        for (int i0 = 0; i0 < take; i0 += 32) {
                            const int ii = i0 + lane;
                            if (ii < take) {
                                const uint32_t e = q[ii];
                                const int r5 = e & 31, b = (e >> 5) & 7, t = e >> 8;
                                const int xr = quarter * 32 + r5, col = b * 32 + t;
                                const uint4 *lg = reinterpret_cast<const uint4 *>(lo_g + col * 128);
                                uint4 lv[8];
#pragma unroll
                                for (int c = 0; c < 8; ++c) lv[c] = __ldg(lg + c);
                                float ah = 0.0f, al = 0.0f;
#pragma unroll
                                for (int c = 0; c < 16; ++c) {  // hi part from shared memory first
                                    const uint4 xv = *sw_chunk(xt, 128, xr, c);
                                    const uint4 hv = *sw_chunk(hb, NP, col, c);
                                    ah = fhfma(xv.x, hv.x, ah);
                                    ah = fhfma(xv.y, hv.y, ah);
                                    ah = fhfma(xv.z, hv.z, ah);
                                    ah = fhfma(xv.w, hv.w, ah);
                                }
#pragma unroll
                                for (int c = 0; c < 8; ++c) {  // 16 fp8 lo values per uint4 = 2 x chunks
                                    const uint4 x0 = *sw_chunk(xt, 128, xr, 2 * c);
                                    const uint4 x1 = *sw_chunk(xt, 128, xr, 2 * c + 1);
                                    uint32_t l0, l1;
                                    e4m3x4_to_f16x2(lv[c].x, l0, l1);
                                    al = fhfma(x0.x, l0, al);
                                    al = fhfma(x0.y, l1, al);
                                    e4m3x4_to_f16x2(lv[c].y, l0, l1);
                                    al = fhfma(x0.z, l0, al);
                                    al = fhfma(x0.w, l1, al);
                                    e4m3x4_to_f16x2(lv[c].z, l0, l1);
                                    al = fhfma(x1.x, l0, al);
                                    al = fhfma(x1.y, l1, al);
                                    e4m3x4_to_f16x2(lv[c].w, l0, l1);
                                    al = fhfma(x1.z, l0, al);
                                    al = fhfma(x1.w, l1, al);
                                }
                                const float vv = fmaf(al, lo_scale, ah);
                                if (vv > 0.0f) atomicOr(&cw[r5 * 8 + b], 1u << t);
                            }
                        }
                        __syncwarp();
                        if (total <= kQCap) break;
                    }
#pragma unroll
                    for (int b = 0; b < C; ++b) {
                        sw[b] = (sw[b] & ~fw[b]) | cw[lane * 8 + b];
                        cw[lane * 8 + b] = 0u;
                    }
                    __syncwarp();
                }

                // ---- outputs
                if (stage) {  // sw is kept for the quarter's staged, coalesced store below
                    gk = g;
                } else if (row < p.n_rows) {  // G > 2: direct stores per group
                    if (p.recs_out) {
                        uint32_t *rec = p.recs_out + row * R;
#pragma unroll
                        for (int b = 0; b < C; ++b) rec[b * W + g] = sw[b];
                        if (g == 0)
                            for (int k = C * W; k < R; ++k) rec[k] = 0;
                    }
                    if (p.codes_out) {
                        uint32_t cwd[8];
                        codes_from_planes<C>(sw, cwd);
                        uint8_t *dst = static_cast<uint8_t *>(p.codes_out) + row * L + t0;
#pragma unroll
                        for (int tt = 0; tt < 32; ++tt)
                            if (tt < nt) dst[tt] = (cwd[tt >> 2] >> (8 * (tt & 3))) & 0xffu;
                    }
                }
            }
            if (stage) {
                // The quarter's x^ rows (32 x 128 B in each 64-column block) are free once
                // both warps of the pair are past their fix-ups (and every MMA of the tile
                // has completed): block 0's rows stage the records, block 1's the u8 codes,
                // laid out as in global memory, then the pair writes both with 16-byte
                // coalesced stores (instead of C scattered 4-byte stores per row).
                uint8_t *xq = sa + st * kTileX + quarter * 32 * 128;
                uint32_t *rs = reinterpret_cast<uint32_t *>(xq);
                uint8_t *cs = xq + 128 * 128;
                pair_sync(1 + quarter);
                if (gk >= 0) {
                    if (p.recs_out) {
#pragma unroll
                        for (int b = 0; b < C; ++b) rs[lane * R + b * W + gk] = sw[b];
                        if (gk == 0)
                            for (int k = C * W; k < R; ++k) rs[lane * R + k] = 0u;
                    }
                    if (p.codes_out) {
                        uint32_t cwd[8];
                        codes_from_planes<C>(sw, cwd);
                        const int t0 = gk * 32, nt = min(32, L - t0);
                        uint8_t *dst = cs + lane * L + t0;
                        if (nt == 32 && (L & 15) == 0) {
                            reinterpret_cast<uint4 *>(dst)[0] = make_uint4(cwd[0], cwd[1], cwd[2], cwd[3]);
                            reinterpret_cast<uint4 *>(dst)[1] = make_uint4(cwd[4], cwd[5], cwd[6], cwd[7]);
                        } else {
#pragma unroll
                            for (int tt = 0; tt < 32; ++tt)
                                if (tt < nt) dst[tt] = (cwd[tt >> 2] >> (8 * (tt & 3))) & 0xffu;
                        }
                    }
                }
                pair_sync(1 + quarter);
#ifndef DSRT_FIX_NOOUT
                const int64_t row0 = tile * 128 + quarter * 32;
                const int nv = static_cast<int>(tmin<int64_t>(32, p.n_rows - row0));
                const int tid = h * 32 + lane;
                if (nv > 0 && p.recs_out) {
                    const int n16 = nv * R / 4;
                    uint4 *dst = reinterpret_cast<uint4 *>(p.recs_out + row0 * R);
                    for (int i = tid; i < n16; i += 64) dst[i] = reinterpret_cast<const uint4 *>(rs)[i];
                }
                if (nv > 0 && p.codes_out) {
                    uint8_t *dst = static_cast<uint8_t *>(p.codes_out) + row0 * L;
                    if ((L & 15) == 0) {
                        const int n16 = nv * L / 16;
                        for (int i = tid; i < n16; i += 64)
                            reinterpret_cast<uint4 *>(dst)[i] = reinterpret_cast<const uint4 *>(cs)[i];
                    } else {
                        for (int i = tid; i < nv * L; i += 64) dst[i] = cs[i];
                    }
                }
#endif
                fence_proxy_async_smem();  // generic writes before the next TMA fill of this stage
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&xempty[st]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

// f64 planes (reference order: row t*C + b) -> hi fp16 and lo (float) in
// plane-major group order (row g*NP + b*32 + t; zero rows for tables >= L) and
// the bound statistics.  Block per output row, thread per dimension (d = 128).
// The plane's scale 2^-6 (1 + j/64) is the j in [0, 64) with the smallest
// relative rounding error.
__global__ void fix_planes_kernel(const double *__restrict__ planes, int L, int C, int NP,
                                  __half *__restrict__ hi, float *__restrict__ lo32,
                                  float *__restrict__ stats) {
    const int orow = blockIdx.x, k = threadIdx.x, wp = k >> 5;
    const int g = orow / NP, rem = orow % NP, b = rem / 32, t = rem % 32;
    const int tg = g * 32 + t;
    double w = 0.0;
    if (tg < L && b < C) w = planes[(static_cast<int64_t>(tg) * C + b) * 128 + k] * 0.015625;
    __shared__ double red[64][4];
    __shared__ double best_s;
#pragma unroll 1
    for (int j = 0; j < 64; ++j) {
        const double ws = w * (1.0 + j / 64.0);
        const double e = ws - static_cast<double>(__half2float(__double2half(ws)));
        double e2 = e * e;
        for (int o = 16; o > 0; o >>= 1) e2 += __shfl_xor_sync(0xffffffffu, e2, o);
        if ((k & 31) == 0) red[j][wp] = e2;
    }
    __syncthreads();
    if (k == 0) {
        int bj = 0;
        double br = 0.0;
        for (int j = 0; j < 64; ++j) {
            const double s = 1.0 + j / 64.0;
            const double r = (red[j][0] + red[j][1] + red[j][2] + red[j][3]) / (s * s);
            if (j == 0 || r < br) {
                br = r;
                bj = j;
            }
        }
        best_s = 1.0 + bj / 64.0;
    }
    __syncthreads();
    const double ws = w * best_s;
    const __half hh = __double2half(ws);
    const double hd = static_cast<double>(__half2float(hh));
    const double l = ws - hd;  // exact in float: |l| <= 2^-11 |hd| and 11 + 24 bits suffice
    hi[static_cast<int64_t>(orow) * 128 + k] = hh;
    lo32[static_cast<int64_t>(orow) * 128 + k] = static_cast<float>(l);
    __shared__ double s_lo[4], s_hi[4];
    __shared__ float s_abs[4], s_loabs[4];
    double ll = l * l, h2 = hd * hd;
    float aa = fabsf(__half2float(hh)), la = fabsf(static_cast<float>(l));
    for (int o = 16; o > 0; o >>= 1) {
        ll += __shfl_xor_sync(0xffffffffu, ll, o);
        h2 += __shfl_xor_sync(0xffffffffu, h2, o);
        aa = fmaxf(aa, __shfl_xor_sync(0xffffffffu, aa, o));
        la = fmaxf(la, __shfl_xor_sync(0xffffffffu, la, o));
    }
    if ((k & 31) == 0) {
        s_lo[wp] = ll;
        s_hi[wp] = h2;
        s_abs[wp] = aa;
        s_loabs[wp] = la;
    }
    __syncthreads();
    if (k == 0) {
        const double nl = sqrt(s_lo[0] + s_lo[1] + s_lo[2] + s_lo[3]);
        const double nh = sqrt(s_hi[0] + s_hi[1] + s_hi[2] + s_hi[3]);
        const double c = (nl + 2e-5 * nh) * 1.001;
        const float am = fmaxf(fmaxf(s_abs[0], s_abs[1]), fmaxf(s_abs[2], s_abs[3]));
        const float lm = fmaxf(fmaxf(s_loabs[0], s_loabs[1]), fmaxf(s_loabs[2], s_loabs[3]));
        // non-negative floats order like their bit patterns: integer atomicMax
        atomicMax(reinterpret_cast<unsigned *>(stats + 0), __float_as_uint(am));
        atomicMax(reinterpret_cast<unsigned *>(stats + 2), __float_as_uint(lm));
        atomicMax(reinterpret_cast<unsigned *>(stats + kStatWords + g * 8 + b),
                  __float_as_uint(__double2float_ru(c)));
    }
}

// lo (float) -> e4m3(lo 2^E) with one power-of-two scale putting max |lo| in
// [128, 256); stats[1] = E (as a float).  The fix-up error this adds is at most
// 2^-4 |x^| |lo_p| + 2^-10-E |x^|_1, far inside the band (see the header).
__global__ void fix_lo8_kernel(const float *__restrict__ lo32, int64_t n, float *__restrict__ stats,
                               uint8_t *__restrict__ lo8) {
    const float lm = stats[2];
    int e = 0;
    if (lm > 0.0f) frexpf(lm, &e);  // lm in [2^(e-1), 2^e)
    const int E = 8 - e;            // lm 2^E in [128, 256)
    if (blockIdx.x == 0 && threadIdx.x == 0) stats[1] = static_cast<float>(E);
    const float sc = ldexpf(1.0f, E);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const __nv_fp8_e4m3 v(lo32[i] * sc);
        lo8[i] = *reinterpret_cast<const uint8_t *>(&v);
    }
}

template <int C, int S, bool BF16>
int launch_fix(const CUtensorMap &mx, const CUtensorMap &mw, const FixParams &fp, uint32_t idesc,
               size_t smem, int ctas, cudaStream_t st) {
    auto kern = hash_fix_kernel<C, S, BF16>;
    DSRT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<ctas, kFThreads, smem, st>>>(mx, mw, fp, idesc);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}

template <int C>
int launch_fix_c(int S, bool bf16, const CUtensorMap &mx, const CUtensorMap &mw, const FixParams &fp,
                 uint32_t idesc, size_t smem, int ctas, cudaStream_t st) {
    if (S == 3)
        return bf16 ? launch_fix<C, 3, true>(mx, mw, fp, idesc, smem, ctas, st)
                    : launch_fix<C, 3, false>(mx, mw, fp, idesc, smem, ctas, st);
    return bf16 ? launch_fix<C, 2, true>(mx, mw, fp, idesc, smem, ctas, st)
                : launch_fix<C, 2, false>(mx, mw, fp, idesc, smem, ctas, st);
}

}  // namespace

size_t hash_fix_smem(int L, int C, int stages) {
    const int G = (L + 31) / 32, NP = 32 * C;
    return 1024 + static_cast<size_t>(stages) * kTileX + static_cast<size_t>(G) * 2 * NP * 128 +
           static_cast<size_t>(stages) * 256 * 4 + kEpi * kQCap * 2 + kEpi * 32 * 8 * 4 +
           static_cast<size_t>(G) * 8 * 4;
}

bool hash_fix_supported(int d, int L, int C) {
    return d == 128 && C >= 1 && C <= 8 && hash_fix_smem(L, C, 2) <= 227 * 1024;
}

int hash_fix(const void *X, int x_dtype, int64_t n, int d, const void *planes, int L, int C,
             void *codes_out, uint32_t *records_out, uint32_t *zero_rows, cudaStream_t st) {
    DSRT_REQUIRE(x_dtype == DSRT_F16 || x_dtype == DSRT_BF16, DSRT_EINVAL,
                 "invalid parameter: hash mode %d needs fp16 or bf16 vectors", DSRT_HASH_TC_FIX);
    DSRT_REQUIRE(hash_fix_supported(d, L, C), DSRT_EUNSUPPORTED,
                 "invalid parameter: tensor-core hash (fix-up mode) needs d=128, C<=8 and "
                 "L*C planes resident in shared memory (d=%d, L=%d, C=%d)", d, L, C);
    DSRT_REQUIRE(n < (1LL << 31), DSRT_EUNSUPPORTED, "invalid parameter: too many rows for one call");
    const bool bf16 = x_dtype == DSRT_BF16;
    const int G = (L + 31) / 32, NP = 32 * C;
    const int64_t prow = static_cast<int64_t>(G) * NP;
    const int64_t nel = prow * 128;
    uint8_t *ws = nullptr;
    const size_t hi_bytes = static_cast<size_t>(nel) * sizeof(__half);
    const size_t lo32_bytes = static_cast<size_t>(nel) * sizeof(float);
    const size_t stat_bytes = (kStatWords + 8 * static_cast<size_t>(G)) * sizeof(float);
    DSRT_CUDA(malloc_async(reinterpret_cast<void **>(&ws), hi_bytes + lo32_bytes + nel + stat_bytes, st));
    __half *hi = reinterpret_cast<__half *>(ws);
    float *lo32 = reinterpret_cast<float *>(ws + hi_bytes);
    uint8_t *lo8 = ws + hi_bytes + lo32_bytes;
    float *stats = reinterpret_cast<float *>(ws + hi_bytes + lo32_bytes + nel);
    DSRT_CUDA(cudaMemsetAsync(stats, 0, stat_bytes, st));
    fix_planes_kernel<<<static_cast<unsigned>(prow), 128, 0, st>>>(static_cast<const double *>(planes), L,
                                                                   C, NP, hi, lo32, stats);
    DSRT_LAUNCH_CHECK();
    fix_lo8_kernel<<<static_cast<unsigned>((nel + 255) / 256), 256, 0, st>>>(lo32, nel, stats, lo8);
    DSRT_LAUNCH_CHECK();
    CUtensorMap mx, mw;
    const CUtensorMapDataType dt = bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    int rc = make_tmap_2d(&mx, X, dt, 128, static_cast<uint64_t>(n), 256, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc == DSRT_OK)
        rc = make_tmap_2d(&mw, hi, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 128, static_cast<uint64_t>(prow), 256,
                          64, NP, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc == DSRT_OK) {
        FixParams fp{n, L, G, NP, codes_out, records_out, zero_rows, lo8, stats};
        const int S = hash_fix_smem(L, C, 3) <= 227 * 1024 ? 3 : 2;
        const size_t smem = hash_fix_smem(L, C, S);
        const int64_t n_tiles = (n + 127) / 128;
        const int ctas = static_cast<int>(tmax<int64_t>(1, tmin<int64_t>(sm_count(), n_tiles)));
        const uint32_t idesc = idesc_f16(128, NP, 0, 0);
        switch (C) {
            case 1: rc = launch_fix_c<1>(S, bf16, mx, mw, fp, idesc, smem, ctas, st); break;
            case 2: rc = launch_fix_c<2>(S, bf16, mx, mw, fp, idesc, smem, ctas, st); break;
            case 3: rc = launch_fix_c<3>(S, bf16, mx, mw, fp, idesc, smem, ctas, st); break;
            case 4: rc = launch_fix_c<4>(S, bf16, mx, mw, fp, idesc, smem, ctas, st); break;
            case 5: rc = launch_fix_c<5>(S, bf16, mx, mw, fp, idesc, smem, ctas, st); break;
            case 6: rc = launch_fix_c<6>(S, bf16, mx, mw, fp, idesc, smem, ctas, st); break;
            case 7: rc = launch_fix_c<7>(S, bf16, mx, mw, fp, idesc, smem, ctas, st); break;
            default: rc = launch_fix_c<8>(S, bf16, mx, mw, fp, idesc, smem, ctas, st); break;
        }
    }
    cudaFreeAsync(ws, st);  // stream-ordered: released after the kernel
    return rc;
}

}  // namespace dsrt
