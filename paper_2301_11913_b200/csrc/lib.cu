// Library-wide state of libswarm_b200.so: per-thread error text and the
// launch counter bench.py reports as gpu_launches.
#include <string>

#include "common.cuh"

namespace swarm {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }
std::atomic<uint64_t>& launch_counter() { return g_launches; }

}  // namespace swarm

extern "C" {

const char* swarm_last_error(void) { return swarm::g_last_error.c_str(); }
int swarm_version(void) { return 1; }
uint64_t swarm_launch_count(void) { return swarm::launch_counter().load(); }

}  // extern "C"
