// Library-wide state of libswarm_b200.so: per-thread error text and the
// launch counter bench.py reports as gpu_launches.
#include <cstdlib>
#include <string>

#include "common.cuh"

namespace swarm {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }

// Off by default since round 2c: with several peers' streams sharing a GPU, dependents launched
// early hold SM slots other streams' kernels could use -- the engine headline measured +0.7% at
// 1 GPU and +1% at 4 GPUs without it (scripts/gpu_ab_multi.sh, gpu_scale_env_ab.sh).  SWARM_PDL=1
// turns it on (a single-stream caller may prefer it).
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("SWARM_PDL");
        return e && e[0] == '1';
    }();
    return on;
}

namespace {
// Busy-wait on the global timer (one thread): keeps a stream occupied so the
// kernels a host thread issues behind it queue up back to back.
__global__ void k_spin(uint64_t ns) {
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        __nanosleep(1000);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
}
}  // namespace
std::atomic<uint64_t>& launch_counter() { return g_launches; }

}  // namespace swarm

extern "C" {

const char* swarm_last_error(void) { return swarm::g_last_error.c_str(); }
int swarm_version(void) { return 1; }
uint64_t swarm_launch_count(void) { return swarm::launch_counter().load(); }

int swarm_gpu_spin(uint64_t ns, swarm_stream_t stream) {
    swarm::k_spin<<<1, 1, 0, swarm::as_stream(stream)>>>(ns);
    SWARM_LAUNCH_CHECK("k_spin");
    return SWARM_OK;
}

}  // extern "C"
