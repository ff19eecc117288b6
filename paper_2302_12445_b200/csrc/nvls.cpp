// Symmetric heap for the NVLS (NVLink SHARP) backend: on every rank one
// physical allocation (cuMemCreate) mapped twice — at a local (unicast)
// address and through ONE multicast object spanning all P GPUs, so a store to
// the multicast alias lands on every rank and multimem.ld_reduce returns the
// sum over ranks, reduced in the NVSwitch.
//
// Setup (collective, the caller moves one (pid, fd) pair between processes):
//   dear_symm_create   every rank: physical memory + local mapping; rank 0
//                      also creates the multicast object and exports it as a
//                      POSIX file descriptor
//   dear_symm_join     ranks != 0: pidfd_getfd() the descriptor out of rank
//                      0's process, import it, add this GPU
//   (barrier: every GPU added before any memory is bound, cuda.h)
//   dear_symm_bind     bind the physical memory, map the multicast alias
//   (barrier)
// The first kFlagBytes of the heap hold the runtime's per-bucket counters
// (dear_nvls_connect carves them in call order, identical on every rank);
// the rest is handed out to the caller (dear_symm_ptr).
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "dear.h"
#include "dear_internal.h"

struct dear_symm {
  int rank = 0, P = 1, device = 0;
  size_t size = 0;  // bytes mapped (granularity multiple)
  CUmemGenericAllocationHandle mem = 0, mc = 0;
  bool have_mem = false, have_mc = false, bound = false;
  CUdeviceptr uc = 0, mcp = 0;
  bool uc_mapped = false, mc_mapped = false, uc_reserved = false, mc_reserved = false;
  int fd = -1;
  size_t flag_next = 0;
};

namespace dear {
namespace {

constexpr size_t kFlagBytes = 1 << 20;

struct Driver {
  decltype(&cuMemCreate) memCreate = nullptr;
  decltype(&cuMemRelease) memRelease = nullptr;
  decltype(&cuMemAddressReserve) addrReserve = nullptr;
  decltype(&cuMemAddressFree) addrFree = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) setAccess = nullptr;
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  decltype(&cuMemExportToShareableHandle) exportHandle = nullptr;
  decltype(&cuMemImportFromShareableHandle) importHandle = nullptr;
  decltype(&cuMulticastCreate) mcCreate = nullptr;
  decltype(&cuMulticastAddDevice) mcAddDevice = nullptr;
  decltype(&cuMulticastBindMem) mcBindMem = nullptr;
  decltype(&cuMulticastUnbind) mcUnbind = nullptr;
  decltype(&cuMulticastGetGranularity) mcGranularity = nullptr;
  decltype(&cuDeviceGet) deviceGet = nullptr;
  decltype(&cuDeviceGetAttribute) deviceAttr = nullptr;
  decltype(&cuGetErrorString) errorString = nullptr;
  bool ok = false;
};

template <typename F>
void load(F& f, const char* name, bool& ok) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p) {
    ok = false;
    return;
  }
  f = reinterpret_cast<F>(p);
}

const Driver& drv() {
  static Driver d = [] {
    Driver x;
    bool ok = true;
    load(x.memCreate, "cuMemCreate", ok);
    load(x.memRelease, "cuMemRelease", ok);
    load(x.addrReserve, "cuMemAddressReserve", ok);
    load(x.addrFree, "cuMemAddressFree", ok);
    load(x.map, "cuMemMap", ok);
    load(x.unmap, "cuMemUnmap", ok);
    load(x.setAccess, "cuMemSetAccess", ok);
    load(x.granularity, "cuMemGetAllocationGranularity", ok);
    load(x.exportHandle, "cuMemExportToShareableHandle", ok);
    load(x.importHandle, "cuMemImportFromShareableHandle", ok);
    load(x.mcCreate, "cuMulticastCreate", ok);
    load(x.mcAddDevice, "cuMulticastAddDevice", ok);
    load(x.mcBindMem, "cuMulticastBindMem", ok);
    load(x.mcUnbind, "cuMulticastUnbind", ok);
    load(x.mcGranularity, "cuMulticastGetGranularity", ok);
    load(x.deviceGet, "cuDeviceGet", ok);
    load(x.deviceAttr, "cuDeviceGetAttribute", ok);
    load(x.errorString, "cuGetErrorString", ok);
    x.ok = ok;
    return x;
  }();
  if (!d.ok) throw Error(DEAR_EINTERNAL, "NVLS: CUDA driver entry points unavailable");
  return d;
}

void cu_check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) {
    const char* s = nullptr;
    if (drv().errorString) drv().errorString(r, &s);
    throw Error(DEAR_EINTERNAL, std::string(what) + ": " + (s ? s : "CUDA driver error"));
  }
}

bool multicast_supported(int device) {
  const Driver& d = drv();
  CUdevice dev = 0;
  int v = 0;
  if (d.deviceGet(&dev, device) != CUDA_SUCCESS) return false;
  return d.deviceAttr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) == CUDA_SUCCESS && v != 0;
}

void rt_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(DEAR_EINTERNAL, std::string(what) + ": " + cudaGetErrorString(e));
}

[[noreturn]] void bad(const std::string& m) { throw Error(DEAR_EINVAL, m); }

CUmulticastObjectProp mc_prop(int P, size_t size) {
  CUmulticastObjectProp p{};
  p.numDevices = static_cast<unsigned>(P);
  p.size = size;
  p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  p.flags = 0;
  return p;
}

void map_rw(CUdeviceptr* va, bool* reserved, bool* mapped, size_t size, size_t align,
            CUmemGenericAllocationHandle h, int device) {
  const Driver& d = drv();
  cu_check(d.addrReserve(va, size, align, 0, 0), "cuMemAddressReserve");
  *reserved = true;
  cu_check(d.map(*va, size, 0, h, 0), "cuMemMap");
  *mapped = true;
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  cu_check(d.setAccess(*va, size, &acc, 1), "cuMemSetAccess");
}

void release(dear_symm* h) {
  const Driver& d = drv();
  if (h->mc_mapped) d.unmap(h->mcp, h->size);
  if (h->mc_reserved) d.addrFree(h->mcp, h->size);
  if (h->bound) {
    CUdevice dev = 0;
    d.deviceGet(&dev, h->device);
    d.mcUnbind(h->mc, dev, 0, h->size);
  }
  if (h->uc_mapped) d.unmap(h->uc, h->size);
  if (h->uc_reserved) d.addrFree(h->uc, h->size);
  if (h->have_mem) d.memRelease(h->mem);
  if (h->have_mc) d.memRelease(h->mc);
  if (h->fd >= 0) close(h->fd);
}

}  // namespace

// Used by runtime.cpp (dear_nvls_connect).
bool symm_contains(const dear_symm* h, const void* p, size_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uintptr_t lo = static_cast<uintptr_t>(h->uc) + kFlagBytes;
  return a >= lo && a + bytes <= static_cast<uintptr_t>(h->uc) + h->size;
}
int symm_rank(const dear_symm* h) { return h->rank; }
int symm_size(const dear_symm* h) { return h->P; }
int symm_bound(const dear_symm* h) { return h->bound && h->mc_mapped ? 1 : 0; }
int64_t symm_mc_delta(const dear_symm* h) {
  return static_cast<int64_t>(h->mcp) - static_cast<int64_t>(h->uc);
}
uintptr_t symm_base(const dear_symm* h) { return static_cast<uintptr_t>(h->uc); }
// Carves `bytes` of the counter region (64 B aligned); throws when full.
size_t symm_take_flags(dear_symm* h, size_t bytes) {
  const size_t at = h->flag_next;
  const size_t n = (bytes + 63) / 64 * 64;
  if (at + n > kFlagBytes) bad("dear_nvls_connect: the symmetric heap's counter region is full");
  h->flag_next = at + n;
  return at;
}

}  // namespace dear

using namespace dear;

extern "C" {

int dear_nvls_supported(int32_t device, int32_t* ok) {
  DEAR_API_BEGIN
  if (!ok) bad("dear_nvls_supported: null output");
  rt_check(cudaFree(nullptr), "cudaFree(0)");
  *ok = multicast_supported(device) ? 1 : 0;
  DEAR_API_END
}

int dear_symm_create(int32_t rank, int32_t P, int64_t bytes, dear_symm** out, int64_t* pid,
                     int64_t* fd) {
  DEAR_API_BEGIN
  if (!out || P < 1 || rank < 0 || rank >= P || bytes < 0) bad("dear_symm_create: bad arguments");
  if (P < 2) bad("dear_symm_create: a multicast team needs at least 2 GPUs");
  const Driver& d = drv();
  auto* h = new dear_symm();
  try {
    h->rank = rank;
    h->P = P;
    rt_check(cudaGetDevice(&h->device), "cudaGetDevice");
    rt_check(cudaFree(nullptr), "cudaFree(0)");  // primary context current
    if (!multicast_supported(h->device)) throw Error(DEAR_EINTERNAL, "NVLS: this GPU does not support multicast objects");
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = h->device;
    // An exported / imported multicast object binds only externally
    // shareable memory.
    prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t g1 = 0, g2 = 0;
    cu_check(d.granularity(&g1, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED),
             "cuMemGetAllocationGranularity");
    const size_t want = kFlagBytes + static_cast<size_t>(bytes);
    CUmulticastObjectProp mp = mc_prop(P, want);
    cu_check(d.mcGranularity(&g2, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED),
             "cuMulticastGetGranularity");
    const size_t gran = g1 > g2 ? g1 : g2;
    h->size = (want + gran - 1) / gran * gran;
    cu_check(d.memCreate(&h->mem, h->size, &prop, 0), "cuMemCreate");
    h->have_mem = true;
    map_rw(&h->uc, &h->uc_reserved, &h->uc_mapped, h->size, gran, h->mem, h->device);
    rt_check(cudaMemset(reinterpret_cast<void*>(h->uc), 0, h->size), "cudaMemset(heap)");
    rt_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    if (rank == 0) {
      mp = mc_prop(P, h->size);
      cu_check(d.mcCreate(&h->mc, &mp), "cuMulticastCreate");
      h->have_mc = true;
      CUdevice dev = 0;
      cu_check(d.deviceGet(&dev, h->device), "cuDeviceGet");
      cu_check(d.mcAddDevice(h->mc, dev), "cuMulticastAddDevice");
      int f = -1;
      cu_check(d.exportHandle(&f, h->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
               "cuMemExportToShareableHandle");
      h->fd = f;
      if (pid) *pid = static_cast<int64_t>(getpid());
      if (fd) *fd = f;
    } else {
      if (pid) *pid = -1;
      if (fd) *fd = -1;
    }
  } catch (...) {
    release(h);
    delete h;
    throw;
  }
  *out = h;
  DEAR_API_END
}

int dear_symm_join(dear_symm* h, int64_t pid, int64_t fd) {
  DEAR_API_BEGIN
  if (!h) bad("dear_symm_join: null heap");
  if (h->rank == 0) return DEAR_OK;
  if (h->have_mc) bad("dear_symm_join: already joined");
  const Driver& d = drv();
  // Take a duplicate of rank 0's descriptor out of its process (same user).
  const long pidfd = syscall(SYS_pidfd_open, static_cast<pid_t>(pid), 0);
  if (pidfd < 0) throw Error(DEAR_EINTERNAL, "NVLS: pidfd_open of rank 0 failed");
  const long local = syscall(SYS_pidfd_getfd, static_cast<int>(pidfd), static_cast<int>(fd), 0);
  close(static_cast<int>(pidfd));
  if (local < 0) throw Error(DEAR_EINTERNAL, "NVLS: pidfd_getfd of the multicast handle failed");
  h->fd = static_cast<int>(local);
  cu_check(d.importHandle(&h->mc, reinterpret_cast<void*>(static_cast<intptr_t>(h->fd)),
                          CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
           "cuMemImportFromShareableHandle");
  h->have_mc = true;
  CUdevice dev = 0;
  cu_check(d.deviceGet(&dev, h->device), "cuDeviceGet");
  cu_check(d.mcAddDevice(h->mc, dev), "cuMulticastAddDevice");
  DEAR_API_END
}

int dear_symm_bind(dear_symm* h) {
  DEAR_API_BEGIN
  if (!h || !h->have_mc) bad("dear_symm_bind: create / join first");
  if (h->bound) bad("dear_symm_bind: already bound");
  const Driver& d = drv();
  cu_check(d.mcBindMem(h->mc, 0, h->mem, 0, h->size, 0), "cuMulticastBindMem");
  h->bound = true;
  size_t gran = 0;
  CUmulticastObjectProp mp = mc_prop(h->P, h->size);
  cu_check(d.mcGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED),
           "cuMulticastGetGranularity");
  map_rw(&h->mcp, &h->mc_reserved, &h->mc_mapped, h->size, gran, h->mc, h->device);
  DEAR_API_END
}

int dear_symm_ptr(dear_symm* h, void** local, void** multicast, int64_t* bytes) {
  DEAR_API_BEGIN
  if (!h) bad("dear_symm_ptr: null heap");
  if (local) *local = reinterpret_cast<void*>(h->uc + kFlagBytes);
  if (multicast) *multicast = h->mc_mapped ? reinterpret_cast<void*>(h->mcp + kFlagBytes) : nullptr;
  if (bytes) *bytes = static_cast<int64_t>(h->size - kFlagBytes);
  DEAR_API_END
}

int dear_symm_destroy(dear_symm* h) {
  DEAR_API_BEGIN
  if (h) {
    cudaDeviceSynchronize();
    release(h);
    delete h;
  }
  DEAR_API_END
}

}  // extern "C"
