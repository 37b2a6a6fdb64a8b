// K1 tensor-core modes (tcgen05) -- see DESIGN.md.  Placeholder until the
// tcgen05 kernel lands: reports EUNSUPPORTED so the host selects a SIMT mode.
#include "common.cuh"

namespace dsrt {
int hash_tc(const void *, int, int64_t, int, const void *, int, int, int, void *, uint32_t *,
            uint32_t *, cudaStream_t) {
    set_error("unsupported: tensor-core hash mode not built");
    return DSRT_EUNSUPPORTED;
}
}  // namespace dsrt
