// C-ABI: library-level entry points (error reporting, device info).
#include <cuda_runtime.h>

#include <string>

#include "capi_util.hpp"

namespace hc {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace hc

extern "C" {

const char* hc_last_error(void) { return hc::g_last_error.c_str(); }

int hc_abi_version(void) { return 1; }

// Number of visible CUDA devices (0 when no GPU / driver).
int hc_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// PCI bus id ("0000:18:00.0") of a visible device — for NUMA-local pinning
// of the host pools (bench.py binds each rank to its GPU's NUMA node).
int hc_device_pci_bus_id(int dev, char* buf, int len) {
    return hc_guard([&] { HC_CUDA(cudaDeviceGetPCIBusId(buf, len, dev)); });
}

int hc_set_device(int dev) {
    return hc_guard([&] { HC_CUDA(cudaSetDevice(dev)); });
}

}  // extern "C"
