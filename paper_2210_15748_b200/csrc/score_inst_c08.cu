// Explicit instantiation of the scoring kernels for C = 8.
#include "score_kernels.cuh"

namespace dsrt {
template int run_w<8>(const ScoreArgs &, int, int, cudaStream_t);
}  // namespace dsrt
