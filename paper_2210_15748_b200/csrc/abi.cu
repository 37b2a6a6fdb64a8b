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
