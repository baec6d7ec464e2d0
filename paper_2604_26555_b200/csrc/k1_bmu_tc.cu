// k1_bmu_tc.cu — tcgen05 3xTF32 BMU kernel (placeholder until the tensor-core path lands).
#include <cuda_runtime.h>

#include "engine.h"

namespace tsom {

bool tc_supported(uint32_t, uint32_t) { return false; }

cudaError_t launch_bmu_tc(const float*, uint64_t, uint32_t, const float*, float*, int,
                          cudaStream_t) {
    return cudaErrorNotSupported;
}

}  // namespace tsom
