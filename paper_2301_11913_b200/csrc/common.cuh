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

// Programmatic dependent launch.  Kernels of the per-layer chain (GEMMs,
// attention, LayerNorm) are launched with programmatic stream serialization, so
// a kernel's CTAs can be scheduled — and run their prologue (barrier init, TMEM
// allocation, descriptor prefetch) on SMs the previous kernel's tail leaves
// idle — before that kernel finishes.  Every such kernel calls pdl_trigger()
// first and pdl_wait() before its first global-memory access; both are no-ops
// for a kernel launched without the attribute.  Off unless SWARM_PDL=1 (csrc/lib.cu).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();

inline int pdl_attr(cudaLaunchAttribute* a) {
    if (!pdl_enabled()) return 0;
    a->id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a->val.programmaticStreamSerializationAllowed = 1;
    return 1;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    cfg.numAttrs = static_cast<unsigned>(pdl_attr(&attr[0]));
    cfg.attrs = attr;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace swarm
