// Explicit instantiation of the scoring kernels for C = 6.
#include "score_kernels.cuh"

namespace dsrt {
template int run_w<6>(const ScoreArgs &, int, int, cudaStream_t);
}  // namespace dsrt
