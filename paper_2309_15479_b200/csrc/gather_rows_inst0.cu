// gather_rows_inst0.cu — instantiations of the K1r kernel template (gather_rows.cuh) for MS in
// {20, 22, 34, 46, 58, 128}; split across translation units so nvcc builds them in parallel.
#include "gather_rows.cuh"

namespace fastlsh {
namespace k1r {

RowKernelFn row_kernel_ms_0(int MS, int cls) {
    switch (MS) {
        case 20: return row_kernel_for<20>(cls);
        case 22: return row_kernel_for<22>(cls);
        case 34: return row_kernel_for<34>(cls);
        case 46: return row_kernel_for<46>(cls);
        case 58: return row_kernel_for<58>(cls);
        case 128: return row_kernel_for<128>(cls);
        default: return nullptr;
    }
}

}  // namespace k1r
}  // namespace fastlsh
