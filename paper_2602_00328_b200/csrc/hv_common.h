// Internal helpers shared by the translation units of libharvest_b200.so.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/harvest_b200.h"

#define HV_EXPORT extern "C" __attribute__((visibility("default")))

static inline int hv_cuda_status(cudaError_t e) {
  return e == cudaSuccess ? HV_OK : (HV_E_CUDA_BASE - (int)e);
}

#define HV_CUDA(expr)                                  \
  do {                                                 \
    cudaError_t hv_e_ = (expr);                        \
    if (hv_e_ != cudaSuccess) {                        \
      (void)cudaGetLastError();                        \
      return hv_cuda_status(hv_e_);                    \
    }                                                  \
  } while (0)

#define HV_CHECK_ARG(cond)         \
  do {                             \
    if (!(cond)) return HV_E_INVALID; \
  } while (0)

namespace hv {
// Switches the calling thread's current device for the duration of one ABI
// call and restores the caller's on return: the library never leaves a
// different device current behind (torch and the caller keep theirs).
struct DeviceGuard {
  int prev = -1;
  bool changed = false;
  int set(int dev) {
    if (prev < 0 && cudaGetDevice(&prev) != cudaSuccess) {
      (void)cudaGetLastError();
      prev = -1;
    }
    if (dev == (changed ? -2 : prev)) return HV_OK;
    HV_CUDA(cudaSetDevice(dev));
    changed = dev != prev;
    return HV_OK;
  }
  ~DeviceGuard() {
    if (changed && prev >= 0) cudaSetDevice(prev);
  }
};

// Make the device that owns `stream` current (static cudart keeps its own
// notion of the current device, so never rely on the caller's); `g` restores
// the caller's device when the ABI call returns.
int bind_stream_device(void* stream, int* device_out, DeviceGuard& g);
void note_launch(uint64_t n = 1);
// Host-tier address ranges (pinned allocations made or registered through
// this library).  The AUTO fetch engine routes large objects whose source
// lies in one of them to the copy engine (PCIe reads by the DMA engine are
// ~8% more efficient than SM-issued sysmem loads).
void host_range_add(uint64_t base, uint64_t bytes);
void host_range_remove(uint64_t base);
bool host_range_contains(uint64_t p, uint64_t bytes);
int sm_count(int device);

// Function attributes belong to a kernel in one device's context, so they
// are set once per (kernel, device).  `Fn` is the kernel; the caller has made
// `dev` current.
template <auto Fn>
int kernel_attr(int dev, cudaFuncAttribute attr, int value) {
  static std::atomic<uint64_t> done{0};
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return HV_OK;
  HV_CUDA(cudaFuncSetAttribute(Fn, attr, value));
  done.fetch_or(bit, std::memory_order_acq_rel);
  return HV_OK;
}

}  // namespace hv
