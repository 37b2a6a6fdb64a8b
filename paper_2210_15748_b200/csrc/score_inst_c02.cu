// Explicit instantiation of the scoring kernels for C = 2.
#include "score_kernels.cuh"

namespace dsrt {
template int run_w<2>(const ScoreArgs &, int, int, cudaStream_t);
}  // namespace dsrt
