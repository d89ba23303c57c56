// Per-device one-time kernel attributes. cudaFuncSetAttribute acts on the
// calling thread's current device, so "set once per process" would leave a
// second GPU of the same process without the dynamic shared-memory opt-in;
// one bit per device ordinal, set atomically (engines may run in threads).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

namespace hc {

template <class Kernel>
inline void max_dynamic_smem_once(Kernel kern, int bytes, std::atomic<uint64_t>& done) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = uint64_t(1) << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done.fetch_or(bit, std::memory_order_acq_rel);
}

}  // namespace hc
