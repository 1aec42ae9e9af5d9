// gather_rows_inst4.cu — instantiations of the K1r kernel template (gather_rows.cuh) for MS in
// {2, 16, 26, 42, 54, 72, 96}; split across translation units so nvcc builds them in parallel.
#include "gather_rows.cuh"

namespace fastlsh {
namespace k1r {

RowKernelFn row_kernel_ms_4(int MS, int cls) {
    switch (MS) {
        case 2: return row_kernel_for<2>(cls);
        case 16: return row_kernel_for<16>(cls);
        case 26: return row_kernel_for<26>(cls);
        case 42: return row_kernel_for<42>(cls);
        case 54: return row_kernel_for<54>(cls);
        case 72: return row_kernel_for<72>(cls);
        case 96: return row_kernel_for<96>(cls);
        default: return nullptr;
    }
}

}  // namespace k1r
}  // namespace fastlsh
