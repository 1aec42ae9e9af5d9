// mc.cpp — NVLS multicast allocations for the fused key all-gather (DESIGN.md
// "Multi-GPU"). K1j can store every compound key with multimem.st into a table mapped through an
// NVSwitch multicast object, so each GPU of the group receives the key while the kernel runs
// (fastlsh_hash_keys_multicast). In a multi-process job the table comes from torch symmetric memory
// (its multicast_ptr). This file creates the same kind of mapping for the CURRENT device alone
// (driver API: cuMulticastCreate / AddDevice / BindMem + cuMemMap of both the physical memory and
// the multicast object), so the multimem store path can be exercised and parity-tested on one GPU.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <new>

#include "internal.h"

namespace fastlsh {
namespace {

struct Drv {
    bool ok = false;
    CUresult (*getAttr)(int*, CUdevice_attribute, CUdevice) = nullptr;
    CUresult (*mcGran)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
    CUresult (*mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
    CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
    CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                          unsigned long long) = nullptr;
    CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
    CUresult (*memRelease)(CUmemGenericAllocationHandle) = nullptr;
    CUresult (*addrReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
    CUresult (*addrFree)(CUdeviceptr, size_t) = nullptr;
    CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
    CUresult (*memUnmap)(CUdeviceptr, size_t) = nullptr;
    CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
    CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
};

template <typename F>
bool sym(const char* name, F& f) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        return false;
    f = reinterpret_cast<F>(p);
    return true;
}

const Drv& drv() {
    static Drv d = [] {
        Drv r;
        r.ok = sym("cuDeviceGetAttribute", r.getAttr) && sym("cuMulticastGetGranularity", r.mcGran) &&
               sym("cuMulticastCreate", r.mcCreate) && sym("cuMulticastAddDevice", r.mcAddDevice) &&
               sym("cuMulticastBindMem", r.mcBindMem) && sym("cuMemCreate", r.memCreate) &&
               sym("cuMemRelease", r.memRelease) && sym("cuMemAddressReserve", r.addrReserve) &&
               sym("cuMemAddressFree", r.addrFree) && sym("cuMemMap", r.memMap) && sym("cuMemUnmap", r.memUnmap) &&
               sym("cuMemSetAccess", r.setAccess) && sym("cuMulticastUnbind", r.mcUnbind);
        return r;
    }();
    return d;
}

struct McTable {
    int dev = 0;
    size_t size = 0;
    CUmemGenericAllocationHandle mem = 0, mc = 0;
    CUdeviceptr uc_va = 0, mc_va = 0;
    bool bound = false;
};

void release(const Drv& d, McTable* t) {
    if (t->mc_va) { d.memUnmap(t->mc_va, t->size); d.addrFree(t->mc_va, t->size); }
    if (t->uc_va) { d.memUnmap(t->uc_va, t->size); d.addrFree(t->uc_va, t->size); }
    if (t->bound) d.mcUnbind(t->mc, (CUdevice)t->dev, 0, t->size);
    if (t->mc) d.memRelease(t->mc);
    if (t->mem) d.memRelease(t->mem);
    delete t;
}

}  // namespace
}  // namespace fastlsh

using namespace fastlsh;

extern "C" {

fastlsh_status fastlsh_multicast_alloc(size_t bytes, void** unicast_ptr, void** multicast_ptr, void** handle) {
    if (!bytes || !unicast_ptr || !multicast_ptr || !handle) return FASTLSH_EINVAL;
    *unicast_ptr = *multicast_ptr = *handle = nullptr;
    const Drv& d = drv();
    if (!d.ok) return FASTLSH_EUNSUPPORTED;
    int dev = 0;
    cudaError_t ce = cudaGetDevice(&dev);
    if (ce != cudaSuccess) return set_cuda_error(ce);
    cudaFree(nullptr);  // the primary context exists before driver calls
    int supported = 0;
    if (d.getAttr(&supported, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, (CUdevice)dev) != CUDA_SUCCESS || !supported)
        return FASTLSH_EUNSUPPORTED;
    McTable* t = new (std::nothrow) McTable();
    if (!t) return FASTLSH_ENOMEM;
    t->dev = dev;
    CUmulticastObjectProp mp = {};
    mp.numDevices = 1;
    mp.size = bytes;
    size_t gran = 0;
    if (d.mcGran(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || !gran) {
        delete t;
        return FASTLSH_EUNSUPPORTED;
    }
    t->size = (bytes + gran - 1) / gran * gran;
    mp.size = t->size;
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = dev;
    CUmemAccessDesc acc = {};
    acc.location = ap.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    const bool ok = d.mcCreate(&t->mc, &mp) == CUDA_SUCCESS && d.mcAddDevice(t->mc, (CUdevice)dev) == CUDA_SUCCESS &&
                    d.memCreate(&t->mem, t->size, &ap, 0) == CUDA_SUCCESS &&
                    (t->bound = d.mcBindMem(t->mc, 0, t->mem, 0, t->size, 0) == CUDA_SUCCESS) &&
                    d.addrReserve(&t->uc_va, t->size, gran, 0, 0) == CUDA_SUCCESS &&
                    d.memMap(t->uc_va, t->size, 0, t->mem, 0) == CUDA_SUCCESS &&
                    d.setAccess(t->uc_va, t->size, &acc, 1) == CUDA_SUCCESS &&
                    d.addrReserve(&t->mc_va, t->size, gran, 0, 0) == CUDA_SUCCESS &&
                    d.memMap(t->mc_va, t->size, 0, t->mc, 0) == CUDA_SUCCESS &&
                    d.setAccess(t->mc_va, t->size, &acc, 1) == CUDA_SUCCESS;
    if (!ok) {
        release(d, t);
        return FASTLSH_EUNSUPPORTED;
    }
    *unicast_ptr = reinterpret_cast<void*>(t->uc_va);
    *multicast_ptr = reinterpret_cast<void*>(t->mc_va);
    *handle = t;
    return FASTLSH_OK;
}

void fastlsh_multicast_free(void* handle) {
    if (!handle) return;
    const Drv& d = drv();
    if (d.ok) release(d, static_cast<McTable*>(handle));
}

}  // extern "C"
