// gather_inst3.cu — instantiations of the K1 kernel template (gather_impl.cuh) for MS in
// {50, 52, 54, 56, 58, 60, 62, 64}; split across translation units so nvcc builds them in parallel.
#include "gather_impl.cuh"

namespace fastlsh {
namespace k1 {

KernelFn kernel_for_ms_3(int MS, int shape, bool fused) {
    switch (MS) {
        case 50: return fused ? kernel_for<50, true>(shape) : kernel_for<50, false>(shape);
        case 52: return fused ? kernel_for<52, true>(shape) : kernel_for<52, false>(shape);
        case 54: return fused ? kernel_for<54, true>(shape) : kernel_for<54, false>(shape);
        case 56: return fused ? kernel_for<56, true>(shape) : kernel_for<56, false>(shape);
        case 58: return fused ? kernel_for<58, true>(shape) : kernel_for<58, false>(shape);
        case 60: return fused ? kernel_for<60, true>(shape) : kernel_for<60, false>(shape);
        case 62: return fused ? kernel_for<62, true>(shape) : kernel_for<62, false>(shape);
        case 64: return fused ? kernel_for<64, true>(shape) : kernel_for<64, false>(shape);
        default: return nullptr;
    }
}

}  // namespace k1
}  // namespace fastlsh
