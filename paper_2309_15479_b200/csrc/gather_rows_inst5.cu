// gather_rows_inst5.cu — instantiations of the K1r kernel template (gather_rows.cuh) for MS in
// {18, 24, 44, 52, 80, 88}; split across translation units so nvcc builds them in parallel.
#include "gather_rows.cuh"

namespace fastlsh {
namespace k1r {

RowKernelFn row_kernel_ms_5(int MS, int cls) {
    switch (MS) {
        case 18: return row_kernel_for<18>(cls);
        case 24: return row_kernel_for<24>(cls);
        case 44: return row_kernel_for<44>(cls);
        case 52: return row_kernel_for<52>(cls);
        case 80: return row_kernel_for<80>(cls);
        case 88: return row_kernel_for<88>(cls);
        default: return nullptr;
    }
}

}  // namespace k1r
}  // namespace fastlsh
