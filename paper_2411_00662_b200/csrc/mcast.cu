// NVSwitch multicast (NVLS) for the intra-node AllGather (SURVEY.md §8(f)
// item 3; the AllGather being replaced is dataplane.hpp:243-256, the
// "gather" of the TP shards into full rows).  With unicast stores a TP rank
// sends its slice t - 1 times (once per peer); through a multicast object one
// multimem.st leaves the GPU once and the switch replicates it to every
// bound device, so the AllGather's egress drops from (t - 1) slices to one.
//
// Setup (one group of `ndev` processes, one GPU each; the caller moves the
// POSIX file descriptor between processes, e.g. over a Unix socket):
//   leader:  moe_mc_create  -> fd          others: moe_mc_import(fd)
//   all:     moe_mc_add_device (then a group barrier: binding needs every device)
//   all:     moe_mc_bind -> this device's physical buffer (unicast VA) and the
//            multicast VA; a store through the multicast VA lands in every
//            device's buffer at the same offset.
// Driver entry points are resolved at run time (no libcuda link), at the
// runtime's own version: the multicast API appeared in 12.1.
#include <cuda.h>

#include <mutex>

#include "common.cuh"

struct moe_mc {
  CUmemGenericAllocationHandle mc = 0;
  CUmemGenericAllocationHandle mem = 0;
  CUdeviceptr uc_va = 0, mc_va = 0;
  size_t bytes = 0;
  int ndev = 0;
  int device = -1;
  bool mem_mapped = false, mc_mapped = false;
};

namespace monta {
namespace {

struct Drv {
  CUresult (*mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                        unsigned long long) = nullptr;
  CUresult (*mcGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) =
      nullptr;
  CUresult (*memRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*memExport)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long) = nullptr;
  CUresult (*memImport)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
  CUresult (*addrReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*addrFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*memUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*allocGranularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*devAttr)(int*, CUdevice_attribute, CUdevice) = nullptr;
  bool ok = false;
};

const Drv& drv() {
  static Drv d;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* name, auto& fn) {
      void* p = nullptr;
      cudaDriverEntryPointQueryResult q{};
      if (cudaGetDriverEntryPointByVersion(name, &p, CUDART_VERSION, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(p);
      return p != nullptr;
    };
    bool ok = true;
    ok &= get("cuMulticastCreate", d.mcCreate);
    ok &= get("cuMulticastAddDevice", d.mcAddDevice);
    ok &= get("cuMulticastBindMem", d.mcBindMem);
    ok &= get("cuMulticastGetGranularity", d.mcGranularity);
    ok &= get("cuMulticastUnbind", d.mcUnbind);
    ok &= get("cuMemCreate", d.memCreate);
    ok &= get("cuMemRelease", d.memRelease);
    ok &= get("cuMemExportToShareableHandle", d.memExport);
    ok &= get("cuMemImportFromShareableHandle", d.memImport);
    ok &= get("cuMemAddressReserve", d.addrReserve);
    ok &= get("cuMemAddressFree", d.addrFree);
    ok &= get("cuMemMap", d.memMap);
    ok &= get("cuMemUnmap", d.memUnmap);
    ok &= get("cuMemSetAccess", d.setAccess);
    ok &= get("cuMemGetAllocationGranularity", d.allocGranularity);
    ok &= get("cuDeviceGetAttribute", d.devAttr);
    d.ok = ok;
  });
  return d;
}

moe_status cu_fail(CUresult r, const char* what) { return fail(MOE_ERR_CUDA, "%s: CUresult %d", what, int(r)); }
#define MONTA_CU(expr, what)                       \
  do {                                             \
    const CUresult _r = (expr);                    \
    if (_r != CUDA_SUCCESS) return cu_fail(_r, what); \
  } while (0)

CUmulticastObjectProp mc_prop(int ndev, size_t bytes) {
  CUmulticastObjectProp p{};
  p.numDevices = unsigned(ndev);
  p.size = bytes;
  p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return p;
}

// AllGather store: this rank's `bytes` (16-byte multiple) from src to the
// multicast VA at `dst_off`: one multimem.st per 16 bytes, replicated by the
// switch into every bound device's buffer; a system fence at the end so the
// stores are visible before the stream moves on.
__global__ void __launch_bounds__(256) k_mc_store(const uint4* __restrict__ src, uint4* mc_dst, int64_t nvec) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nvec; i += int64_t(gridDim.x) * blockDim.x) {
    const uint4 v = __ldg(src + i);
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc_dst + i), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
  }
  __threadfence_system();
}

}  // namespace
}  // namespace monta

using namespace monta;

extern "C" moe_status moe_mc_supported(int device, int* supported) {
  if (!supported) return fail(MOE_ERR_INVALID_ARGUMENT, "mc_supported: null output");
  *supported = 0;
  int v = 0;
  cudaFree(nullptr);
  if (!drv().ok) return fail(MOE_ERR_UNSUPPORTED, "multicast driver entry points unavailable");
  MONTA_CU(drv().devAttr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, CUdevice(device)), "cuDeviceGetAttribute");
  *supported = v ? 1 : 0;
  return MOE_OK;
}

extern "C" moe_status moe_mc_granularity(int ndev, size_t bytes, size_t* granularity) {
  if (!granularity || ndev < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "mc_granularity: bad argument");
  if (!drv().ok) return fail(MOE_ERR_UNSUPPORTED, "multicast driver entry points unavailable");
  const CUmulticastObjectProp p = mc_prop(ndev, bytes);
  MONTA_CU(drv().mcGranularity(granularity, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
  return MOE_OK;
}

extern "C" moe_status moe_mc_create(int ndev, size_t bytes, int* fd_out, moe_mc** out) {
  if (!fd_out || !out || ndev < 1 || bytes == 0) return fail(MOE_ERR_INVALID_ARGUMENT, "mc_create: bad argument");
  if (!drv().ok) return fail(MOE_ERR_UNSUPPORTED, "multicast driver entry points unavailable");
  cudaFree(nullptr);  // a current context for the driver calls
  moe_mc* m = new moe_mc;
  m->bytes = bytes;
  m->ndev = ndev;
  const CUmulticastObjectProp p = mc_prop(ndev, bytes);
  CUresult r = drv().mcCreate(&m->mc, &p);
  if (r != CUDA_SUCCESS) {
    delete m;
    return cu_fail(r, "cuMulticastCreate");
  }
  int fd = -1;
  r = drv().memExport(&fd, m->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
  if (r != CUDA_SUCCESS) {
    drv().memRelease(m->mc);
    delete m;
    return cu_fail(r, "cuMemExportToShareableHandle(multicast)");
  }
  *fd_out = fd;
  *out = m;
  return MOE_OK;
}

extern "C" moe_status moe_mc_import(int fd, int ndev, size_t bytes, moe_mc** out) {
  if (!out || fd < 0 || ndev < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "mc_import: bad argument");
  if (!drv().ok) return fail(MOE_ERR_UNSUPPORTED, "multicast driver entry points unavailable");
  cudaFree(nullptr);
  moe_mc* m = new moe_mc;
  m->bytes = bytes;
  m->ndev = ndev;
  const CUresult r =
      drv().memImport(&m->mc, reinterpret_cast<void*>(intptr_t(fd)), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  if (r != CUDA_SUCCESS) {
    delete m;
    return cu_fail(r, "cuMemImportFromShareableHandle(multicast)");
  }
  *out = m;
  return MOE_OK;
}

extern "C" moe_status moe_mc_add_device(moe_mc* m, int device) {
  if (!m) return fail(MOE_ERR_INVALID_ARGUMENT, "mc_add_device: null object");
  CUdevice dev = device;
  MONTA_CUDA(cudaSetDevice(device));
  MONTA_CU(drv().mcAddDevice(m->mc, dev), "cuMulticastAddDevice");
  m->device = device;
  return MOE_OK;
}

extern "C" moe_status moe_mc_bind(moe_mc* m, void** local_va, void** mc_va) {
  if (!m || !local_va || !mc_va || m->device < 0) return fail(MOE_ERR_INVALID_ARGUMENT, "mc_bind: add the device first");
  const Drv& d = drv();
  MONTA_CUDA(cudaSetDevice(m->device));
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = m->device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  MONTA_CU(d.allocGranularity(&gran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity");
  if (m->bytes % gran) return fail(MOE_ERR_INVALID_ARGUMENT, "mc_bind: size not a multiple of %zu", gran);
  MONTA_CU(d.memCreate(&m->mem, m->bytes, &ap, 0), "cuMemCreate");
  MONTA_CU(d.mcBindMem(m->mc, 0, m->mem, 0, m->bytes, 0), "cuMulticastBindMem");
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = m->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  MONTA_CU(d.addrReserve(&m->uc_va, m->bytes, gran, 0, 0), "cuMemAddressReserve");
  MONTA_CU(d.memMap(m->uc_va, m->bytes, 0, m->mem, 0), "cuMemMap(unicast)");
  m->mem_mapped = true;
  MONTA_CU(d.setAccess(m->uc_va, m->bytes, &acc, 1), "cuMemSetAccess(unicast)");
  MONTA_CU(d.addrReserve(&m->mc_va, m->bytes, gran, 0, 0), "cuMemAddressReserve(multicast)");
  MONTA_CU(d.memMap(m->mc_va, m->bytes, 0, m->mc, 0), "cuMemMap(multicast)");
  m->mc_mapped = true;
  MONTA_CU(d.setAccess(m->mc_va, m->bytes, &acc, 1), "cuMemSetAccess(multicast)");
  *local_va = reinterpret_cast<void*>(m->uc_va);
  *mc_va = reinterpret_cast<void*>(m->mc_va);
  return MOE_OK;
}

extern "C" moe_status moe_mc_store(const void* src, void* mc_dst, size_t bytes, int32_t grid_req, void* stream) {
  if (!src || !mc_dst || bytes % 16 || (reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(mc_dst)) % 16)
    return fail(MOE_ERR_INVALID_ARGUMENT, "mc_store: 16-byte aligned buffers and sizes only");
  if (bytes == 0) return MOE_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t nvec = int64_t(bytes / 16);
  const int64_t cap = grid_req > 0 ? int64_t(grid_req) : int64_t(sms) * 4;
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>((nvec + 255) / 256, cap)));
  k_mc_store<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const uint4*>(src),
                                                                  static_cast<uint4*>(mc_dst), nvec);
  MONTA_CHECK_LAUNCH("mc_store launch");
  return MOE_OK;
}

extern "C" moe_status moe_mc_destroy(moe_mc* m) {
  if (!m) return MOE_OK;
  const Drv& d = drv();
  cudaDeviceSynchronize();
  if (m->mc_mapped) d.memUnmap(m->mc_va, m->bytes);
  if (m->mc_va) d.addrFree(m->mc_va, m->bytes);
  if (m->mem_mapped) d.memUnmap(m->uc_va, m->bytes);
  if (m->uc_va) d.addrFree(m->uc_va, m->bytes);
  if (m->mem && m->device >= 0) d.mcUnbind(m->mc, CUdevice(m->device), 0, m->bytes);
  if (m->mem) d.memRelease(m->mem);
  if (m->mc) d.memRelease(m->mc);
  delete m;
  return MOE_OK;
}
