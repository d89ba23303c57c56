// Error plumbing for the C ABI: exceptions -> int status + thread-local
// message. Status codes mirror the reference's exception types
// (errors.hpp:9-21): 1 InputError, 2 CapacityError, 3 ConfigError, 4 CUDA /
// runtime failure.
#pragma once
#include <cuda_runtime.h>

#include <cmath>
#include <stdexcept>
#include <string>

#include "host/errors.hpp"

namespace hc {
void set_last_error(const std::string& msg);
}

using hc_input_error = hc::InputError;

#define HC_CUDA(expr)                                                                                  \
    do {                                                                                               \
        cudaError_t _e = (expr);                                                                       \
        if (_e != cudaSuccess) {                                                                       \
            (void)cudaGetLastError(); /* reported here: do not resurface it at the next check */      \
            throw hc::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e) + " @" __FILE__ ":" + \
                                std::to_string(__LINE__));                                             \
        }                                                                                              \
    } while (0)

template <class F>
int hc_guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const hc::InputError& e) {
        hc::set_last_error(e.what());
        return 1;
    } catch (const hc::CapacityError& e) {
        hc::set_last_error(e.what());
        return 2;
    } catch (const hc::ConfigError& e) {
        hc::set_last_error(e.what());
        return 3;
    } catch (const std::exception& e) {
        hc::set_last_error(e.what());
        return 4;
    }
}
