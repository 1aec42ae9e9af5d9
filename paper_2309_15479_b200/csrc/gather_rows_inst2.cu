// gather_rows_inst2.cu — instantiations of the K1r kernel template (gather_rows.cuh) for MS in
// {4, 14, 28, 40, 50, 62, 112}; split across translation units so nvcc builds them in parallel.
#include "gather_rows.cuh"

namespace fastlsh {
namespace k1r {

RowKernelFn row_kernel_ms_2(int MS, int cls) {
    switch (MS) {
        case 4: return row_kernel_for<4>(cls);
        case 14: return row_kernel_for<14>(cls);
        case 28: return row_kernel_for<28>(cls);
        case 40: return row_kernel_for<40>(cls);
        case 50: return row_kernel_for<50>(cls);
        case 62: return row_kernel_for<62>(cls);
        case 112: return row_kernel_for<112>(cls);
        default: return nullptr;
    }
}

}  // namespace k1r
}  // namespace fastlsh
