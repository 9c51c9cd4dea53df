// Per-donor peer-memory pool, host tier, device/stream/event plumbing.
//
// The reference models a peer device as a DeviceSpec row plus a segment free
// list (memalloc.py:24-79; profiles.py:165-178) and never touches memory.
// Here a pool is real donor-resident memory mapped into every reader's
// address space:
//   HV_POOL_VMM — cuMemAddressReserve for the whole harvestable range, then
//     physical chunks are created on the donor (cuMemCreate, location=donor),
//     mapped (cuMemMap) and opened to the readers (cuMemSetAccess) only while
//     a live segment overlaps them.  Memory goes back to the donor the moment
//     the last overlapping segment is released, which is what "harvest" means
//     on a shared box (runtime.py:396-411).
//   HV_POOL_IPC — one cudaMalloc slab exportable with cudaIpcGetMemHandle, for
//     the one-process-per-GPU launch (torchrun) where readers live in other
//     processes.
// Driver entry points are resolved at run time through cudart, so the
// library loads on a machine without a GPU driver (the CPU test tier).
#include <cuda.h>
#include <string.h>

#include <map>
#include <mutex>
#include <new>
#include <shared_mutex>
#include <vector>

#include "hv_common.h"

namespace hv {
namespace {
std::shared_mutex g_host_mu;
std::map<uint64_t, uint64_t> g_host_ranges;  // base -> end (exclusive)
}  // namespace

void host_range_add(uint64_t base, uint64_t bytes) {
  std::unique_lock<std::shared_mutex> lk(g_host_mu);
  g_host_ranges[base] = base + bytes;
}

void host_range_remove(uint64_t base) {
  std::unique_lock<std::shared_mutex> lk(g_host_mu);
  g_host_ranges.erase(base);
}

bool host_range_contains(uint64_t p, uint64_t bytes) {
  std::shared_lock<std::shared_mutex> lk(g_host_mu);
  auto it = g_host_ranges.upper_bound(p);
  if (it == g_host_ranges.begin()) return false;
  --it;
  return p >= it->first && p + bytes <= it->second;
}
}  // namespace hv

namespace {

struct DriverApi {
  bool loaded = false;
  int status = HV_OK;
  decltype(&cuMemGetAllocationGranularity) getGranularity = nullptr;
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) addressFree = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) setAccess = nullptr;
  decltype(&cuMemExportToShareableHandle) exportHandle = nullptr;
  decltype(&cuMemImportFromShareableHandle) importHandle = nullptr;
};

std::once_flag g_driver_once;
DriverApi g_driver;

template <typename F>
int resolve(const char* name, F* fn) {
  cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
  void* p = nullptr;
  cudaError_t e = cudaGetDriverEntryPointByVersion(name, &p, 12000, cudaEnableDefault, &q);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return hv_cuda_status(e);
  }
  if (q != cudaDriverEntryPointSuccess || !p) return HV_E_UNSUPPORTED;
  *fn = reinterpret_cast<F>(p);
  return HV_OK;
}

int driver() {
  std::call_once(g_driver_once, [] {
    DriverApi d;
    int st = HV_OK;
    if (!st) st = resolve("cuMemGetAllocationGranularity", &d.getGranularity);
    if (!st) st = resolve("cuMemCreate", &d.create);
    if (!st) st = resolve("cuMemRelease", &d.release);
    if (!st) st = resolve("cuMemAddressReserve", &d.reserve);
    if (!st) st = resolve("cuMemAddressFree", &d.addressFree);
    if (!st) st = resolve("cuMemMap", &d.map);
    if (!st) st = resolve("cuMemUnmap", &d.unmap);
    if (!st) st = resolve("cuMemSetAccess", &d.setAccess);
    if (!st) st = resolve("cuMemExportToShareableHandle", &d.exportHandle);
    if (!st) st = resolve("cuMemImportFromShareableHandle", &d.importHandle);
    d.status = st;
    d.loaded = (st == HV_OK);
    g_driver = d;
  });
  return g_driver.status;
}

inline int cu_status(CUresult r) { return r == CUDA_SUCCESS ? HV_OK : (HV_E_CU_BASE - (int)r); }

#define HV_CU(expr)                      \
  do {                                   \
    CUresult hv_r_ = (expr);             \
    if (hv_r_ != CUDA_SUCCESS) return cu_status(hv_r_); \
  } while (0)

}  // namespace

struct hv_pool {
  unsigned flags = 0;
  int donor = 0;
  std::vector<int> readers;
  uint64_t bytes = 0;        // harvestable range
  uint64_t chunk = 0;        // physical chunk (VMM)
  CUdeviceptr va = 0;
  bool imported = false;     // IPC import (close, don't free)
  // VMM bookkeeping
  std::vector<CUmemGenericAllocationHandle> handles;
  std::vector<uint32_t> refs;
  uint64_t committed = 0;
};

namespace {

int map_chunk(hv_pool* p, uint64_t ci) {
  CUmemAllocationProp prop;
  memset(&prop, 0, sizeof(prop));
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = p->donor;
  CUmemGenericAllocationHandle h = 0;
  HV_CU(g_driver.create(&h, p->chunk, &prop, 0));
  CUdeviceptr at = p->va + ci * p->chunk;
  CUresult r = g_driver.map(at, p->chunk, 0, h, 0);
  if (r != CUDA_SUCCESS) {
    g_driver.release(h);
    return cu_status(r);
  }
  std::vector<CUmemAccessDesc> acc;
  CUmemAccessDesc d;
  memset(&d, 0, sizeof(d));
  d.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  d.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  d.location.id = p->donor;
  acc.push_back(d);
  for (int rd : p->readers) {
    if (rd == p->donor) continue;
    d.location.id = rd;
    acc.push_back(d);
  }
  r = g_driver.setAccess(at, p->chunk, acc.data(), acc.size());
  if (r != CUDA_SUCCESS) {
    g_driver.unmap(at, p->chunk);
    g_driver.release(h);
    return cu_status(r);
  }
  p->handles[ci] = h;
  p->committed += p->chunk;
  return HV_OK;
}

int unmap_chunk(hv_pool* p, uint64_t ci) {
  CUdeviceptr at = p->va + ci * p->chunk;
  HV_CU(g_driver.unmap(at, p->chunk));
  HV_CU(g_driver.release(p->handles[ci]));
  p->handles[ci] = 0;
  p->committed -= p->chunk;
  return HV_OK;
}

}  // namespace

HV_EXPORT int hv_pool_create(int donor_dev, uint64_t bytes, uint64_t chunk_bytes,
                             const int* reader_devs, int n_readers, unsigned flags,
                             hv_pool** out) {
  HV_CHECK_ARG(out != nullptr && bytes > 0 && n_readers >= 0);
  HV_CHECK_ARG(n_readers == 0 || reader_devs != nullptr);
  int ndev = 0;
  HV_CUDA(cudaGetDeviceCount(&ndev));
  HV_CHECK_ARG(donor_dev >= 0 && donor_dev < ndev);
  for (int i = 0; i < n_readers; ++i) HV_CHECK_ARG(reader_devs[i] >= 0 && reader_devs[i] < ndev);
  hv_pool* p = new (std::nothrow) hv_pool();
  if (!p) return HV_E_NOMEM;
  p->flags = flags;
  p->donor = donor_dev;
  p->readers.assign(reader_devs, reader_devs + n_readers);
  // every reader that is not the donor must be able to reach it over P2P
  for (int rd : p->readers) {
    if (rd == donor_dev) continue;
    int ok = 0;
    cudaError_t e = cudaDeviceCanAccessPeer(&ok, rd, donor_dev);
    if (e != cudaSuccess || !ok) {
      delete p;
      (void)cudaGetLastError();
      return HV_E_UNSUPPORTED;
    }
  }
  if (flags & HV_POOL_IPC) {
    hv::DeviceGuard dg;
    int gs = dg.set(donor_dev);
    if (gs) {
      delete p;
      return gs;
    }
    void* ptr = nullptr;
    cudaError_t e = cudaMalloc(&ptr, bytes);
    if (e != cudaSuccess) {
      delete p;
      (void)cudaGetLastError();
      return hv_cuda_status(e);
    }
    for (int rd : p->readers) {
      if (rd == donor_dev) continue;
      if (dg.set(rd)) continue;
      e = cudaDeviceEnablePeerAccess(donor_dev, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) e = cudaSuccess;
      (void)cudaGetLastError();
    }
    p->va = (CUdeviceptr)ptr;
    p->bytes = bytes;
    p->chunk = bytes;
    p->committed = bytes;
    *out = p;
    return HV_OK;
  }
  int st = driver();
  if (st) {
    delete p;
    return st;
  }
  CUmemAllocationProp prop;
  memset(&prop, 0, sizeof(prop));
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = donor_dev;
  if (flags & HV_POOL_REMOTE) prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  CUresult r = g_driver.getGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  if (r != CUDA_SUCCESS || gran == 0) {
    delete p;
    return r != CUDA_SUCCESS ? cu_status(r) : HV_E_UNSUPPORTED;
  }
  uint64_t chunk = chunk_bytes ? chunk_bytes : (uint64_t)gran;
  chunk = (chunk + gran - 1) / gran * gran;
  const uint64_t nchunks = (bytes + chunk - 1) / chunk;
  p->chunk = chunk;
  p->bytes = bytes;
  p->handles.assign(nchunks, 0);
  p->refs.assign(nchunks, 0);
  r = g_driver.reserve(&p->va, nchunks * chunk, chunk, 0, 0);
  if (r != CUDA_SUCCESS) {
    delete p;
    return cu_status(r);
  }
  if ((flags & HV_POOL_EAGER) && !(flags & HV_POOL_REMOTE)) {
    st = hv_pool_commit(p, 0, bytes);
    if (st) {
      hv_pool_destroy(p);
      return st;
    }
  }
  *out = p;
  return HV_OK;
}

HV_EXPORT int hv_pool_commit(hv_pool* p, uint64_t offset, uint64_t bytes) {
  HV_CHECK_ARG(p != nullptr);
  HV_CHECK_ARG(offset <= p->bytes && bytes <= p->bytes - offset);
  if ((p->flags & HV_POOL_IPC) || p->imported || bytes == 0) return HV_OK;
  if (p->flags & HV_POOL_REMOTE) return HV_E_INVALID;   // chunks arrive as FDs (hv_pool_map_fd)
  const uint64_t c0 = offset / p->chunk, c1 = (offset + bytes - 1) / p->chunk;
  for (uint64_t ci = c0; ci <= c1; ++ci) {
    if (p->refs[ci] == 0) {
      int st = map_chunk(p, ci);
      if (st) {  // roll back what this call took
        for (uint64_t cj = c0; cj < ci; ++cj)
          if (--p->refs[cj] == 0) unmap_chunk(p, cj);
        return st;
      }
    }
    ++p->refs[ci];
  }
  return HV_OK;
}

HV_EXPORT int hv_pool_decommit(hv_pool* p, uint64_t offset, uint64_t bytes) {
  HV_CHECK_ARG(p != nullptr);
  HV_CHECK_ARG(offset <= p->bytes && bytes <= p->bytes - offset);
  if ((p->flags & HV_POOL_IPC) || p->imported || bytes == 0) return HV_OK;
  if (p->flags & HV_POOL_REMOTE) return HV_E_INVALID;
  const uint64_t c0 = offset / p->chunk, c1 = (offset + bytes - 1) / p->chunk;
  for (uint64_t ci = c0; ci <= c1; ++ci) HV_CHECK_ARG(p->refs[ci] > 0);
  int st = HV_OK;
  for (uint64_t ci = c0; ci <= c1; ++ci) {
    if (--p->refs[ci] == 0) {
      int s2 = unmap_chunk(p, ci);
      if (s2 && !st) st = s2;
    }
  }
  return st;
}

HV_EXPORT int hv_pool_committed_bytes(const hv_pool* p, uint64_t* out) {
  HV_CHECK_ARG(p && out);
  *out = p->committed;
  return HV_OK;
}

HV_EXPORT int hv_pool_info(const hv_pool* p, uint64_t* va, uint64_t* bytes,
                           uint64_t* chunk_bytes, int* donor_dev) {
  HV_CHECK_ARG(p != nullptr);
  if (va) *va = (uint64_t)p->va;
  if (bytes) *bytes = p->bytes;
  if (chunk_bytes) *chunk_bytes = p->chunk;
  if (donor_dev) *donor_dev = p->donor;
  return HV_OK;
}

HV_EXPORT int hv_pool_destroy(hv_pool* p) {
  if (!p) return HV_OK;
  int st = HV_OK;
  if (p->imported) {
    cudaError_t e = cudaIpcCloseMemHandle((void*)p->va);
    if (e != cudaSuccess) st = hv_cuda_status(e);
  } else if (p->flags & HV_POOL_IPC) {
    hv::DeviceGuard dg;
    dg.set(p->donor);
    cudaError_t e = cudaFree((void*)p->va);
    if (e != cudaSuccess) st = hv_cuda_status(e);
  } else if (p->va) {
    for (uint64_t ci = 0; ci < p->handles.size(); ++ci)
      if (p->refs[ci] > 0 || p->handles[ci] != 0) {
        int s2 = unmap_chunk(p, ci);
        if (s2 && !st) st = s2;
      }
    CUresult r = g_driver.addressFree(p->va, p->handles.size() * p->chunk);
    if (r != CUDA_SUCCESS && !st) st = cu_status(r);
  }
  (void)cudaGetLastError();
  delete p;
  return st;
}

HV_EXPORT int hv_pool_export_ipc(const hv_pool* p, void* handle64) {
  HV_CHECK_ARG(p && handle64 && (p->flags & HV_POOL_IPC) && !p->imported);
  hv::DeviceGuard dg;
  {
    int gs = dg.set(p->donor);
    if (gs) return gs;
  }
  cudaIpcMemHandle_t h;
  HV_CUDA(cudaIpcGetMemHandle(&h, (void*)p->va));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle64, &h, sizeof(h));
  return HV_OK;
}

HV_EXPORT int hv_pool_import_ipc(const void* handle64, int donor_dev, uint64_t bytes,
                                 int reader_dev, hv_pool** out) {
  HV_CHECK_ARG(handle64 && out && bytes > 0);
  hv::DeviceGuard dg;
  {
    int gs = dg.set(reader_dev);
    if (gs) return gs;
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  void* ptr = nullptr;
  HV_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
  hv_pool* p = new (std::nothrow) hv_pool();
  if (!p) {
    cudaIpcCloseMemHandle(ptr);
    return HV_E_NOMEM;
  }
  p->flags = HV_POOL_IPC;
  p->imported = true;
  p->donor = donor_dev;
  p->readers.push_back(reader_dev);
  p->va = (CUdeviceptr)ptr;
  p->bytes = bytes;
  p->chunk = bytes;
  p->committed = bytes;
  *out = p;
  return HV_OK;
}

// ---- cross-process VMM donation (POSIX file descriptors) -------------------
//
// One process per GPU: a donor process creates each physical chunk on its
// own GPU with a shareable handle and passes the file descriptor to the
// reader over a Unix socket (pool.DonorServer, SCM_RIGHTS); the reader maps
// it into a VA range it reserved (HV_POOL_REMOTE) and opens it to its own
// device.  Releasing is the reverse: the reader unmaps and drops its handle,
// the donor drops its own, and the HBM goes back to the donor GPU -- the
// multi-process form of the single-process commit/decommit above.

HV_EXPORT int hv_chunk_granularity(int device, uint64_t* out) {
  HV_CHECK_ARG(out);
  int st = driver();
  if (st) return st;
  CUmemAllocationProp prop;
  memset(&prop, 0, sizeof(prop));
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g = 0;
  HV_CU(g_driver.getGranularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  *out = g;
  return HV_OK;
}

HV_EXPORT int hv_chunk_create_shareable(int device, uint64_t bytes, uint64_t* handle_out, int* fd_out) {
  HV_CHECK_ARG(handle_out && fd_out && bytes > 0);
  int st = driver();
  if (st) return st;
  hv::DeviceGuard dg;
  if ((st = dg.set(device))) return st;
  CUmemAllocationProp prop;
  memset(&prop, 0, sizeof(prop));
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle h = 0;
  HV_CU(g_driver.create(&h, bytes, &prop, 0));
  int fd = -1;
  CUresult r = g_driver.exportHandle(&fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
  if (r != CUDA_SUCCESS) {
    g_driver.release(h);
    return cu_status(r);
  }
  *handle_out = (uint64_t)h;
  *fd_out = fd;
  return HV_OK;
}

HV_EXPORT int hv_chunk_release(uint64_t handle) {
  int st = driver();
  if (st) return st;
  HV_CU(g_driver.release((CUmemGenericAllocationHandle)handle));
  return HV_OK;
}

HV_EXPORT int hv_pool_map_fd(hv_pool* p, uint64_t chunk_index, int fd) {
  HV_CHECK_ARG(p && (p->flags & HV_POOL_REMOTE) && fd >= 0);
  HV_CHECK_ARG(chunk_index < p->handles.size() && p->handles[chunk_index] == 0);
  int st = driver();
  if (st) return st;
  CUmemGenericAllocationHandle h = 0;
  HV_CU(g_driver.importHandle(&h, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
  CUdeviceptr at = p->va + chunk_index * p->chunk;
  CUresult r = g_driver.map(at, p->chunk, 0, h, 0);
  if (r != CUDA_SUCCESS) {
    g_driver.release(h);
    return cu_status(r);
  }
  std::vector<CUmemAccessDesc> acc;
  CUmemAccessDesc d;
  memset(&d, 0, sizeof(d));
  d.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  d.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  for (int rd : p->readers) {
    d.location.id = rd;
    acc.push_back(d);
  }
  r = g_driver.setAccess(at, p->chunk, acc.data(), acc.size());
  if (r != CUDA_SUCCESS) {
    g_driver.unmap(at, p->chunk);
    g_driver.release(h);
    return cu_status(r);
  }
  p->handles[chunk_index] = h;
  p->refs[chunk_index] = 1;
  p->committed += p->chunk;
  return HV_OK;
}

HV_EXPORT int hv_pool_unmap_chunk(hv_pool* p, uint64_t chunk_index) {
  HV_CHECK_ARG(p && (p->flags & HV_POOL_REMOTE) && chunk_index < p->handles.size());
  HV_CHECK_ARG(p->handles[chunk_index] != 0);
  int st = unmap_chunk(p, chunk_index);
  p->refs[chunk_index] = 0;
  return st;
}

// ---- host tier ------------------------------------------------------------

HV_EXPORT int hv_host_alloc(uint64_t bytes, void** h_ptr, uint64_t* d_alias) {
  HV_CHECK_ARG(h_ptr && bytes > 0);
  void* p = nullptr;
  HV_CUDA(cudaHostAlloc(&p, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  void* d = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(&d, p, 0);
  if (e != cudaSuccess) {
    cudaFreeHost(p);
    (void)cudaGetLastError();
    return hv_cuda_status(e);
  }
  *h_ptr = p;
  if (d_alias) *d_alias = (uint64_t)d;
  hv::host_range_add((uint64_t)p, bytes);
  if (d != p) hv::host_range_add((uint64_t)d, bytes);
  return HV_OK;
}

HV_EXPORT int hv_host_alloc_flags(uint64_t bytes, unsigned flags, void** h_ptr, uint64_t* d_alias) {
  HV_CHECK_ARG(h_ptr && bytes > 0);
  unsigned f = cudaHostAllocPortable | cudaHostAllocMapped;
  if (flags & HV_HOST_WRITE_COMBINED) f |= cudaHostAllocWriteCombined;
  void* p = nullptr;
  HV_CUDA(cudaHostAlloc(&p, bytes, f));
  void* d = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(&d, p, 0);
  if (e != cudaSuccess) {
    cudaFreeHost(p);
    (void)cudaGetLastError();
    return hv_cuda_status(e);
  }
  *h_ptr = p;
  if (d_alias) *d_alias = (uint64_t)d;
  hv::host_range_add((uint64_t)p, bytes);
  if (d != p) hv::host_range_add((uint64_t)d, bytes);
  return HV_OK;
}

HV_EXPORT int hv_host_free(void* h_ptr) {
  if (!h_ptr) return HV_OK;
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, h_ptr, 0) != cudaSuccess) {
    (void)cudaGetLastError();
    d = nullptr;
  }
  hv::host_range_remove((uint64_t)h_ptr);
  if (d && d != h_ptr) hv::host_range_remove((uint64_t)d);
  HV_CUDA(cudaFreeHost(h_ptr));
  return HV_OK;
}

HV_EXPORT int hv_host_register(void* h_ptr, uint64_t bytes, uint64_t* d_alias) {
  HV_CHECK_ARG(h_ptr && bytes > 0);
  HV_CUDA(cudaHostRegister(h_ptr, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped));
  void* d = nullptr;
  HV_CUDA(cudaHostGetDevicePointer(&d, h_ptr, 0));
  if (d_alias) *d_alias = (uint64_t)d;
  hv::host_range_add((uint64_t)h_ptr, bytes);
  if (d != h_ptr) hv::host_range_add((uint64_t)d, bytes);
  return HV_OK;
}

HV_EXPORT int hv_host_unregister(void* h_ptr) {
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, h_ptr, 0) != cudaSuccess) {
    (void)cudaGetLastError();
    d = nullptr;
  }
  hv::host_range_remove((uint64_t)h_ptr);
  if (d && d != h_ptr) hv::host_range_remove((uint64_t)d);
  HV_CUDA(cudaHostUnregister(h_ptr));
  return HV_OK;
}

// ---- devices, scratch, streams, events -------------------------------------

HV_EXPORT int hv_device_count(int* n) {
  HV_CHECK_ARG(n);
  cudaError_t e = cudaGetDeviceCount(n);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
    (void)cudaGetLastError();
    *n = 0;
    return HV_OK;
  }
  HV_CUDA(e);
  return HV_OK;
}

HV_EXPORT int hv_mem_get_info(int device, uint64_t* free_bytes, uint64_t* total_bytes) {
  HV_CHECK_ARG(free_bytes && total_bytes);
  hv::DeviceGuard dg;
  {
    int gs = dg.set(device);
    if (gs) return gs;
  }
  size_t f = 0, t = 0;
  HV_CUDA(cudaMemGetInfo(&f, &t));
  *free_bytes = f;
  *total_bytes = t;
  return HV_OK;
}

HV_EXPORT int hv_sm_count(int device, int* n) {
  HV_CHECK_ARG(n);
  HV_CUDA(cudaDeviceGetAttribute(n, cudaDevAttrMultiProcessorCount, device));
  return HV_OK;
}

HV_EXPORT int hv_can_access_peer(int reader, int donor, int* ok) {
  HV_CHECK_ARG(ok);
  if (reader == donor) {
    *ok = 1;
    return HV_OK;
  }
  HV_CUDA(cudaDeviceCanAccessPeer(ok, reader, donor));
  return HV_OK;
}

HV_EXPORT int hv_enable_peer_access(int reader, int donor) {
  if (reader == donor) return HV_OK;
  hv::DeviceGuard dg;
  {
    int gs = dg.set(reader);
    if (gs) return gs;
  }
  cudaError_t e = cudaDeviceEnablePeerAccess(donor, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    (void)cudaGetLastError();
    return HV_OK;
  }
  HV_CUDA(e);
  return HV_OK;
}

HV_EXPORT int hv_device_synchronize(int device) {
  hv::DeviceGuard dg;
  {
    int gs = dg.set(device);
    if (gs) return gs;
  }
  HV_CUDA(cudaDeviceSynchronize());
  return HV_OK;
}

HV_EXPORT int hv_dev_alloc(int device, uint64_t bytes, uint64_t* d_ptr) {
  HV_CHECK_ARG(d_ptr && bytes > 0);
  hv::DeviceGuard dg;
  {
    int gs = dg.set(device);
    if (gs) return gs;
  }
  void* p = nullptr;
  HV_CUDA(cudaMalloc(&p, bytes));
  *d_ptr = (uint64_t)p;
  return HV_OK;
}

HV_EXPORT int hv_dev_free(int device, uint64_t d_ptr) {
  hv::DeviceGuard dg;
  {
    int gs = dg.set(device);
    if (gs) return gs;
  }
  HV_CUDA(cudaFree((void*)d_ptr));
  return HV_OK;
}

HV_EXPORT int hv_memcpy_h2d(uint64_t d_dst, const void* h_src, uint64_t bytes, void* stream) {
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  HV_CUDA(cudaMemcpyAsync((void*)d_dst, h_src, bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream));
  return HV_OK;
}

HV_EXPORT int hv_memcpy_d2h(void* h_dst, uint64_t d_src, uint64_t bytes, void* stream) {
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  HV_CUDA(cudaMemcpyAsync(h_dst, (const void*)d_src, bytes, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  return HV_OK;
}

HV_EXPORT int hv_memset_d8(uint64_t d_dst, int value, uint64_t bytes, void* stream) {
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  HV_CUDA(cudaMemsetAsync((void*)d_dst, value, bytes, (cudaStream_t)stream));
  return HV_OK;
}

HV_EXPORT int hv_stream_create(int device, int priority, void** stream) {
  HV_CHECK_ARG(stream);
  hv::DeviceGuard dg;
  {
    int gs = dg.set(device);
    if (gs) return gs;
  }
  cudaStream_t s = nullptr;
  HV_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, priority));
  *stream = (void*)s;
  return HV_OK;
}

HV_EXPORT int hv_stream_destroy(void* stream) {
  if (stream) HV_CUDA(cudaStreamDestroy((cudaStream_t)stream));
  return HV_OK;
}

HV_EXPORT int hv_stream_synchronize(void* stream) {
  HV_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return HV_OK;
}

HV_EXPORT int hv_event_create(int device, unsigned timing, void** event) {
  HV_CHECK_ARG(event);
  hv::DeviceGuard dg;
  {
    int gs = dg.set(device);
    if (gs) return gs;
  }
  cudaEvent_t e = nullptr;
  HV_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
  *event = (void*)e;
  return HV_OK;
}

HV_EXPORT int hv_event_destroy(void* event) {
  if (event) HV_CUDA(cudaEventDestroy((cudaEvent_t)event));
  return HV_OK;
}

HV_EXPORT int hv_event_record(void* event, void* stream) {
  HV_CHECK_ARG(event);
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  HV_CUDA(cudaEventRecord((cudaEvent_t)event, (cudaStream_t)stream));
  return HV_OK;
}

HV_EXPORT int hv_event_query(void* event, int* done) {
  HV_CHECK_ARG(event && done);
  cudaError_t e = cudaEventQuery((cudaEvent_t)event);
  if (e == cudaErrorNotReady) {
    (void)cudaGetLastError();
    *done = 0;
    return HV_OK;
  }
  HV_CUDA(e);
  *done = 1;
  return HV_OK;
}

HV_EXPORT int hv_event_synchronize(void* event) {
  HV_CHECK_ARG(event);
  HV_CUDA(cudaEventSynchronize((cudaEvent_t)event));
  return HV_OK;
}

HV_EXPORT int hv_event_elapsed_ms(void* start, void* stop, float* ms) {
  HV_CHECK_ARG(start && stop && ms);
  HV_CUDA(cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)stop));
  return HV_OK;
}

HV_EXPORT int hv_stream_wait_event(void* stream, void* event) {
  HV_CHECK_ARG(event);
  HV_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)event, 0));
  return HV_OK;
}

// Stream priorities: [greatest, least] for `device` (greatest is the most
// urgent, a negative number on B200).
HV_EXPORT int hv_stream_priority_range(int device, int* least, int* greatest) {
  HV_CHECK_ARG(least && greatest);
  hv::DeviceGuard dg;
  {
    int gs = dg.set(device);
    if (gs) return gs;
  }
  HV_CUDA(cudaDeviceGetStreamPriorityRange(least, greatest));
  return HV_OK;
}

// Instantiate a captured graph so that each kernel node keeps the priority of
// the stream it was captured from (cudaGraphInstantiateFlagUseNodePriority):
// a fetch stream created urgent stays urgent inside the replay, so its CTAs
// are dispatched ahead of the compute stream's when SMs free up.
HV_EXPORT int hv_graph_instantiate(void* graph, unsigned flags, void** exec_out) {
  HV_CHECK_ARG(graph && exec_out);
  unsigned long long f = 0;
  if (flags & HV_GRAPH_NODE_PRIORITY) f |= cudaGraphInstantiateFlagUseNodePriority;
  cudaGraphExec_t e = nullptr;
  HV_CUDA(cudaGraphInstantiateWithFlags(&e, (cudaGraph_t)graph, f));
  *exec_out = (void*)e;
  return HV_OK;
}

HV_EXPORT int hv_graph_launch(void* exec, void* stream) {
  HV_CHECK_ARG(exec);
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  HV_CUDA(cudaGraphLaunch((cudaGraphExec_t)exec, (cudaStream_t)stream));
  return HV_OK;
}

HV_EXPORT int hv_graph_exec_destroy(void* exec) {
  if (exec) HV_CUDA(cudaGraphExecDestroy((cudaGraphExec_t)exec));
  return HV_OK;
}
