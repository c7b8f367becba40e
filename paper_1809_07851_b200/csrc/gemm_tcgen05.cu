// NK3 on tcgen05 (placeholder until the tensor-core kernel lands).
#include "common.h"

int fc_tcgen05_available() { return 0; }

cudaError_t fc_launch_gemm_tcgen05(const Geometry &, const float *, const float *, const float *, float *,
                                   cudaStream_t) {
    return cudaErrorNotSupported;
}
