// Explicit instantiation of the scoring kernels for C = 13.
#include "score_kernels.cuh"

namespace dsrt {
template int run_w<13>(const ScoreArgs &, int, int, cudaStream_t);
}  // namespace dsrt
