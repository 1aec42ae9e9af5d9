// gather_inst2.cu — instantiations of the K1 kernel template (gather_impl.cuh) for MS in
// {34, 36, 38, 40, 42, 44, 46, 48}; split across translation units so nvcc builds them in parallel.
#include "gather_impl.cuh"

namespace fastlsh {
namespace k1 {

KernelFn kernel_for_ms_2(int MS, int shape, bool fused) {
    switch (MS) {
        case 34: return fused ? kernel_for<34, true>(shape) : kernel_for<34, false>(shape);
        case 36: return fused ? kernel_for<36, true>(shape) : kernel_for<36, false>(shape);
        case 38: return fused ? kernel_for<38, true>(shape) : kernel_for<38, false>(shape);
        case 40: return fused ? kernel_for<40, true>(shape) : kernel_for<40, false>(shape);
        case 42: return fused ? kernel_for<42, true>(shape) : kernel_for<42, false>(shape);
        case 44: return fused ? kernel_for<44, true>(shape) : kernel_for<44, false>(shape);
        case 46: return fused ? kernel_for<46, true>(shape) : kernel_for<46, false>(shape);
        case 48: return fused ? kernel_for<48, true>(shape) : kernel_for<48, false>(shape);
        default: return nullptr;
    }
}

}  // namespace k1
}  // namespace fastlsh
