// C-ABI plumbing: thread-local error text, version, device queries.
#include <mutex>

#include "common.cuh"

namespace dsrt {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

// Stream-ordered scratch allocations.  The device's default memory pool keeps
// its memory across synchronisations (release threshold = max), otherwise
// every synchronising call would unmap and re-map its scratch (~0.4 ms).
cudaError_t malloc_async(void **p, size_t bytes, cudaStream_t st) {
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    });
    return cudaMallocAsync(p, bytes, st);
}

int sm_count() {
    static int cached = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        cached = n;
    });
    return cached;
}

}  // namespace dsrt

using namespace dsrt;

extern "C" const char *dsrt_last_error(void) { return g_err; }

extern "C" int dsrt_version(void) { return 100; }  // 0.1.0

extern "C" int dsrt_record_words(int L, int C) {
    if (L < 1 || C < 1 || C > 24) return 0;
    return record_words(L, C);
}

extern "C" int dsrt_device_info(int *sms, int *major, int *minor, size_t *free_bytes) {
    int dev = 0;
    DSRT_CUDA(cudaGetDevice(&dev));
    cudaDeviceProp p;
    DSRT_CUDA(cudaGetDeviceProperties(&p, dev));
    if (sms) *sms = p.multiProcessorCount;
    if (major) *major = p.major;
    if (minor) *minor = p.minor;
    if (free_bytes) {
        size_t fr = 0, tot = 0;
        DSRT_CUDA(cudaMemGetInfo(&fr, &tot));
        *free_bytes = fr;
    }
    return DSRT_OK;
}

extern "C" int dsrt_copy_async(void *dst, const void *src, size_t bytes, void *stream) {
    if (bytes == 0) return DSRT_OK;
    DSRT_REQUIRE(dst != nullptr && src != nullptr, DSRT_EINVAL, "invalid parameter: null buffer");
    DSRT_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
    return DSRT_OK;
}

namespace {
struct Pack4 {
    const uint32_t *src[4];
    uint32_t words[4], dst_word[4];
};
__global__ void pack4_kernel(uint32_t *__restrict__ dst, Pack4 p) {
#pragma unroll
    for (int s = 0; s < 4; ++s)
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < p.words[s]; i += gridDim.x * blockDim.x)
            dst[p.dst_word[s] + i] = p.src[s][i];
}
}  // namespace

extern "C" int dsrt_pack4_async(void *dst, const void *src0, size_t n0, const void *src1, size_t n1,
                                const void *src2, size_t n2, const void *src3, size_t n3, void *stream) {
    const void *src[4] = {src0, src1, src2, src3};
    const size_t n[4] = {n0, n1, n2, n3};
    Pack4 p;
    size_t off = 0, most = 0;
    for (int s = 0; s < 4; ++s) {
        DSRT_REQUIRE(n[s] % 4 == 0 && n[s] < (size_t(1) << 31), DSRT_EINVAL,
                     "invalid parameter: pack segment sizes must be multiples of 4 bytes");
        DSRT_REQUIRE(n[s] == 0 || src[s] != nullptr, DSRT_EINVAL, "invalid parameter: null segment");
        p.src[s] = static_cast<const uint32_t *>(src[s]);
        p.words[s] = static_cast<uint32_t>(n[s] / 4);
        p.dst_word[s] = static_cast<uint32_t>(off / 4);
        off += (n[s] + 15) & ~size_t(15);
        most = n[s] > most ? n[s] : most;
    }
    if (most == 0) return DSRT_OK;
    DSRT_REQUIRE(dst != nullptr, DSRT_EINVAL, "invalid parameter: null buffer");
    const unsigned blocks = static_cast<unsigned>(tmin<size_t>(64, (most / 4 + 255) / 256));
    pack4_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<uint32_t *>(dst), p);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}
