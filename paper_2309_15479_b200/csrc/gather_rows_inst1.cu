// gather_rows_inst1.cu — instantiations of the K1r kernel template (gather_rows.cuh) for MS in
// {6, 12, 30, 36, 48, 60, 120}; split across translation units so nvcc builds them in parallel.
#include "gather_rows.cuh"

namespace fastlsh {
namespace k1r {

RowKernelFn row_kernel_ms_1(int MS, int cls) {
    switch (MS) {
        case 6: return row_kernel_for<6>(cls);
        case 12: return row_kernel_for<12>(cls);
        case 30: return row_kernel_for<30>(cls);
        case 36: return row_kernel_for<36>(cls);
        case 48: return row_kernel_for<48>(cls);
        case 60: return row_kernel_for<60>(cls);
        case 120: return row_kernel_for<120>(cls);
        default: return nullptr;
    }
}

}  // namespace k1r
}  // namespace fastlsh
