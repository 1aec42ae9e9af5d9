// gather_inst1.cu — instantiations of the K1 kernel template (gather_impl.cuh) for MS in
// {18, 20, 22, 24, 26, 28, 30, 32}; split across translation units so nvcc builds them in parallel.
#include "gather_impl.cuh"

namespace fastlsh {
namespace k1 {

KernelFn kernel_for_ms_1(int MS, int shape, bool fused) {
    switch (MS) {
        case 18: return fused ? kernel_for<18, true>(shape) : kernel_for<18, false>(shape);
        case 20: return fused ? kernel_for<20, true>(shape) : kernel_for<20, false>(shape);
        case 22: return fused ? kernel_for<22, true>(shape) : kernel_for<22, false>(shape);
        case 24: return fused ? kernel_for<24, true>(shape) : kernel_for<24, false>(shape);
        case 26: return fused ? kernel_for<26, true>(shape) : kernel_for<26, false>(shape);
        case 28: return fused ? kernel_for<28, true>(shape) : kernel_for<28, false>(shape);
        case 30: return fused ? kernel_for<30, true>(shape) : kernel_for<30, false>(shape);
        case 32: return fused ? kernel_for<32, true>(shape) : kernel_for<32, false>(shape);
        default: return nullptr;
    }
}

}  // namespace k1
}  // namespace fastlsh
