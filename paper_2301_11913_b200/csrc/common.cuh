// Shared helpers for the sm_100a kernels behind include/swarm_b200.h.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <string>

#include "swarm_b200.h"

namespace swarm {

void set_error(const std::string& msg);
std::atomic<uint64_t>& launch_counter();

inline void count_launch(uint64_t n = 1) { launch_counter().fetch_add(n, std::memory_order_relaxed); }

inline int cuda_fail(cudaError_t e, const char* what) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return SWARM_E_CUDA;
}

inline int invalid(const std::string& msg) {
    set_error(msg);
    return SWARM_E_INVALID;
}

#define SWARM_CUDA_TRY(expr)                                        \
    do {                                                            \
        cudaError_t _e = (expr);                                    \
        if (_e != cudaSuccess) return ::swarm::cuda_fail(_e, #expr); \
    } while (0)

// Check the launch that was just enqueued.
#define SWARM_LAUNCH_CHECK(name)                                     \
    do {                                                             \
        ::swarm::count_launch();                                     \
        cudaError_t _e = cudaGetLastError();                         \
        if (_e != cudaSuccess) return ::swarm::cuda_fail(_e, name);  \
    } while (0)

inline cudaStream_t as_stream(swarm_stream_t s) { return static_cast<cudaStream_t>(s); }

constexpr int kNumSMs = 148;

}  // namespace swarm
