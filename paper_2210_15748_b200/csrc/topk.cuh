// K4 top-k: internal C++ interface shared by topk.cu and the search pipeline.
#pragma once
#include "common.cuh"

namespace dsrt {

constexpr int kTopkMax = 4096;  // k above this runs the large-k (global merge) kernel

struct TopkArgs {
    const double *scores;
    int64_t ld;
    const uint64_t *ids;     // nullptr: id = element index
    int64_t ids_ld;          // 0: ids shared by every row
    const int32_t *n_valid;  // nullptr: n per row
    int64_t n;
    int k;
    double *out_s;
    uint64_t *out_id;
    int64_t *out_pos;
    int64_t out_ld;          // output row stride (>= k; 0 = k)
    const int64_t *ix;       // optional id index (candidate lists): id = ids[ix[row*ix_ld + i]]
    int64_t ix_ld;
    // large k only (set by topk_run): per-row scratch of 2 * run_cap triples
    uint64_t *sk;
    uint64_t *si;
    int64_t *sp;
    int64_t run_cap;
};

// Row-wise top-k by (score desc, id asc) on `st`; rows padded with
// (-1.0, UINT64_MAX, -1) when fewer than k are valid.
int topk_run(const TopkArgs &a, int64_t n_rows, cudaStream_t st);

}  // namespace dsrt
