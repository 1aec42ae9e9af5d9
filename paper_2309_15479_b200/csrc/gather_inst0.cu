// gather_inst0.cu — instantiations of the K1 kernel template (gather_impl.cuh) for MS in
// {2, 4, 6, 8, 10, 12, 14, 16}; split across translation units so nvcc builds them in parallel.
#include "gather_impl.cuh"

namespace fastlsh {
namespace k1 {

KernelFn kernel_for_ms_0(int MS, int shape, bool fused) {
    switch (MS) {
        case 2: return fused ? kernel_for<2, true>(shape) : kernel_for<2, false>(shape);
        case 4: return fused ? kernel_for<4, true>(shape) : kernel_for<4, false>(shape);
        case 6: return fused ? kernel_for<6, true>(shape) : kernel_for<6, false>(shape);
        case 8: return fused ? kernel_for<8, true>(shape) : kernel_for<8, false>(shape);
        case 10: return fused ? kernel_for<10, true>(shape) : kernel_for<10, false>(shape);
        case 12: return fused ? kernel_for<12, true>(shape) : kernel_for<12, false>(shape);
        case 14: return fused ? kernel_for<14, true>(shape) : kernel_for<14, false>(shape);
        case 16: return fused ? kernel_for<16, true>(shape) : kernel_for<16, false>(shape);
        default: return nullptr;
    }
}

}  // namespace k1
}  // namespace fastlsh
