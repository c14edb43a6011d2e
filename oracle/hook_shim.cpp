// TEST INFRASTRUCTURE ONLY — the other half of the additive engine hook:
// the reference's own sim::run, compiled from P/src/sim.cpp patched by hook_patch.py (one
// swarm_hook_emit call per record point; nothing else changed), forwards every record to a C
// callback.  Pointing that callback at swarm_driver_on_record (include/swarm_b200.h) makes the
// unmodified reference engine drive the B200 executor without Python in the loop
// (tests/test_reference_hook.py).
#include <cstdint>
#include <string>

#include "swarm_b200.h"
#include "swarmsim/errors.hpp"
#include "swarmsim/sim.hpp"
#include "swarmsim/trace.hpp"

typedef int (*swarm_record_fn)(void* ctx, const swarm_engine_record* record);

namespace {
thread_local swarm_record_fn g_fn = nullptr;
thread_local void* g_ctx = nullptr;
thread_local int g_rc = 0;
thread_local uint64_t g_records = 0;
}  // namespace

extern "C" void swarm_hook_emit(int kind, std::size_t trainer, std::size_t stage, int backward, long long worker,
                                long long from, double time, double end_time) {
    if (!g_fn || g_rc) return;
    swarm_engine_record r{};
    r.time = time;
    r.end_time = end_time;
    r.kind = kind;
    r.backward = backward;
    r.trainer = static_cast<uint32_t>(trainer);
    r.stage = static_cast<uint32_t>(stage);
    r.worker = worker;
    r.from_worker = from;
    g_records += 1;
    g_rc = g_fn(g_ctx, &r);
}

// sim::run(SimConfig::from_json(json) + churn trace, seed) with the hook on; returns 0, 1 ConfigError,
// 3 other exception, or 100 + the callback's first non-zero return code
extern "C" int hooked_sim_run(const char* json, const double* churn_t, const int64_t* churn_delta, size_t n_churn,
                              uint64_t seed, swarm_record_fn fn, void* ctx, uint64_t* completed, uint64_t* records) {
    try {
        auto cfg = swarmsim::sim::SimConfig::from_json(std::string(json));
        for (size_t i = 0; i < n_churn; ++i) cfg.churn.push_back(swarmsim::trace::TraceEvent{churn_t[i], churn_delta[i]});
        g_fn = fn;
        g_ctx = ctx;
        g_rc = 0;
        g_records = 0;
        const auto r = swarmsim::sim::run(cfg, seed);
        g_fn = nullptr;
        if (completed) *completed = r.completed;
        if (records) *records = g_records;
        return g_rc ? 100 + g_rc : 0;
    } catch (const swarmsim::ConfigError&) {
        g_fn = nullptr;
        return 1;
    } catch (const std::exception&) {
        g_fn = nullptr;
        return 3;
    }
}
