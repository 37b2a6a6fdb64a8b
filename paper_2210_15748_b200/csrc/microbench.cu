// INT-pipe microbenchmark: lane-ops/s of LOP3, POPC and IMNMX on this B200,
// the denominator of the scoring roofline (P_int must be
// measured on the box).  8 independent chains per thread, 148*16 CTAs x 256.
#include "common.cuh"

namespace dsrt {

constexpr int kIters = 4096;

template <int OP>
__global__ void __launch_bounds__(256) int_pipe_kernel(uint32_t seed, uint32_t *sink) {
    uint32_t a[8], b = seed ^ threadIdx.x, c = seed * 2654435761u + blockIdx.x;
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = seed + i * 7919u + threadIdx.x;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) {
                asm volatile("lop3.b32 %0, %0, %1, %2, 0xF6;" : "+r"(a[i]) : "r"(b), "r"(c));
            } else if (OP == 1) {
                uint32_t t;
                asm volatile("popc.b32 %0, %1;" : "=r"(t) : "r"(a[i]));
                a[i] = t ^ a[i];  // keep the chain (adds one LOP)
            } else if (OP == 2) {
                asm volatile("min.s32 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
            } else {
                // the scoring inner-loop mix: 7 LOP3 + 1 POPC + 1 min per chain step
                uint32_t acc = a[i] ^ b;
#pragma unroll
                for (int k = 0; k < 6; ++k)
                    asm volatile("lop3.b32 %0, %0, %1, %2, 0xF6;" : "+r"(acc) : "r"(b + k), "r"(c));
                uint32_t p;
                asm volatile("popc.b32 %0, %1;" : "=r"(p) : "r"(acc));
                asm volatile("min.s32 %0, %0, %1;" : "+r"(a[i]) : "r"(p));
            }
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r ^= a[i];
    if (r == 0x12345678u) sink[0] = r;
}

template <int OP>
static double time_op(cudaStream_t st, uint32_t *sink, double ops_per_thread_iter) {
    const int blocks = sm_count() * 16, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int_pipe_kernel<OP><<<blocks, threads, 0, st>>>(1u, sink);  // warm-up
    cudaEventRecord(e0, st);
    for (int r = 0; r < 5; ++r) int_pipe_kernel<OP><<<blocks, threads, 0, st>>>(r + 2u, sink);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double ops = 5.0 * blocks * threads * static_cast<double>(kIters) * 8.0 * ops_per_thread_iter;
    return ops / (ms * 1e-3);
}

}  // namespace dsrt

using namespace dsrt;

extern "C" int dsrt_microbench_int(double *out4, void *stream) {
    cudaStream_t st = as_stream(stream);
    uint32_t *sink = nullptr;
    DSRT_CUDA(cudaMalloc(&sink, 4));
    out4[0] = time_op<0>(st, sink, 1.0);  // LOP3 lane-ops/s
    out4[1] = time_op<1>(st, sink, 1.0);  // POPC (+1 LOP) pairs/s
    out4[2] = time_op<2>(st, sink, 1.0);  // IMNMX lane-ops/s
    out4[3] = time_op<3>(st, sink, 32.0); // compares/s of the 7-plane scoring mix
    cudaFree(sink);
    DSRT_LAUNCH_CHECK();
    return DSRT_OK;
}
