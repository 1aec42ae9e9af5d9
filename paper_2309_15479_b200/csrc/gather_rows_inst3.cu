// gather_rows_inst3.cu — instantiations of the K1r kernel template (gather_rows.cuh) for MS in
// {8, 10, 32, 38, 56, 64, 104}; split across translation units so nvcc builds them in parallel.
#include "gather_rows.cuh"

namespace fastlsh {
namespace k1r {

RowKernelFn row_kernel_ms_3(int MS, int cls) {
    switch (MS) {
        case 8: return row_kernel_for<8>(cls);
        case 10: return row_kernel_for<10>(cls);
        case 32: return row_kernel_for<32>(cls);
        case 38: return row_kernel_for<38>(cls);
        case 56: return row_kernel_for<56>(cls);
        case 64: return row_kernel_for<64>(cls);
        case 104: return row_kernel_for<104>(cls);
        default: return nullptr;
    }
}

}  // namespace k1r
}  // namespace fastlsh
