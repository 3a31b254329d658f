// FAST mode (tcgen05) launchers — placeholder until the tensor-core path lands.
#include "frs_common.cuh"

namespace frs {

int launch_fast_draft(frs_ctx *, const float *, int, int, const void *, int, const int32_t *, int, float, int32_t *,
                      int32_t *, float *, float *, double *, uint32_t *, cudaStream_t) {
    return fail(FRS_ENOTSUP, "FAST draft head not built yet");
}
int launch_fast_verify(frs_ctx *, const float *, int, int, const void *, int, int32_t, int32_t *, float *, uint32_t *,
                       cudaStream_t) {
    return fail(FRS_ENOTSUP, "FAST verify head not built yet");
}

}  // namespace frs
