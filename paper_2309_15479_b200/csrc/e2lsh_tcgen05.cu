// e2lsh_tcgen05.cu — K4: dense E2LSH baseline on tcgen05 tensor cores.
// (placeholder until the tcgen05 GEMM lands)
#include "internal.h"

namespace fastlsh {

fastlsh_status launch_e2lsh(const fastlsh_params*, DeviceCopy&, const float*, int64_t, int32_t*,
                            float*, int, cudaStream_t) {
    return FASTLSH_EUNSUPPORTED;
}

}  // namespace fastlsh
