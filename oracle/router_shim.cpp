// TEST INFRASTRUCTURE ONLY — extern "C" shim over the UNMODIFIED reference
// router (P/src/wiring.cpp) and rebalancer (P/src/rebalancer.cpp), so tests can
// check that the B200 build's host router makes pick-for-pick identical
// decisions on the same call sequence.
#include <cstdint>
#include <set>

#include "swarmsim/errors.hpp"
#include "swarmsim/rebalancer.hpp"
#include "swarmsim/wiring.hpp"
#include "swarmsim/sim.hpp"
#include "swarmsim/trace.hpp"
#include <algorithm>
#include <cstring>
#include <string>

using namespace swarmsim;

extern "C" {

void* ref_router_new(size_t n_stages, double gamma, double epsilon) {
    try {
        return new wiring::RoutingState(n_stages, gamma, epsilon);
    } catch (...) {
        return nullptr;
    }
}

void ref_router_free(void* r) { delete static_cast<wiring::RoutingState*>(r); }

int ref_router_add_server(void* r, uint64_t peer, const size_t* stages, size_t n, double phase) {
    try {
        std::set<size_t> s(stages, stages + n);
        static_cast<wiring::RoutingState*>(r)->add_server(PeerId{peer}, s, phase);
        return 0;
    } catch (const ConfigError&) {
        return 1;
    } catch (...) {
        return 3;
    }
}

int ref_router_ban_server(void* r, uint64_t peer) {
    try {
        static_cast<wiring::RoutingState*>(r)->ban_server(PeerId{peer});
        return 0;
    } catch (const ConfigError&) {
        return 1;
    }
}

void ref_router_remove_server(void* r, uint64_t peer) {
    static_cast<wiring::RoutingState*>(r)->remove_server(PeerId{peer});
}

// 0 ok (peer in *out), 1 ConfigError, 2 NoPeerAvailable
int ref_router_choose_server(void* r, size_t stage, uint64_t* out) {
    try {
        *out = static_cast<wiring::RoutingState*>(r)->choose_server(stage).value;
        return 0;
    } catch (const ConfigError&) {
        return 1;
    } catch (const NoPeerAvailable&) {
        return 2;
    }
}

int ref_router_record_response(void* r, uint64_t peer, double elapsed) {
    try {
        static_cast<wiring::RoutingState*>(r)->record_response(PeerId{peer}, elapsed);
        return 0;
    } catch (const ConfigError&) {
        return 1;
    }
}

double ref_router_ema_of(void* r, uint64_t peer) {
    return static_cast<wiring::RoutingState*>(r)->ema_of(PeerId{peer});
}

double ref_router_priority_of(void* r, uint64_t peer) {
    return static_cast<wiring::RoutingState*>(r)->priority_of(PeerId{peer});
}

// Table in CSR form: stage s owns members [offsets[s], offsets[s+1]).
// Returns 0 and fills mover (or -1 as UINT64_MAX), from, to.
int ref_rebalance_decide(size_t n_stages, const size_t* offsets, const uint64_t* peers,
                         const double* queues, uint64_t* mover, size_t* from_stage,
                         size_t* to_stage, size_t* ops) {
    try {
        rebalancer::StageLoadTable t;
        t.loads.assign(n_stages, 0.0);
        t.members.resize(n_stages);
        for (size_t s = 0; s < n_stages; ++s) {
            for (size_t i = offsets[s]; i < offsets[s + 1]; ++i) {
                t.members[s][PeerId{peers[i]}] = queues[i];
                t.loads[s] += queues[i];
            }
        }
        size_t n_ops = 0;
        const auto d = rebalancer::decide(t, &n_ops);
        *mover = d.mover ? d.mover->value : UINT64_MAX;
        *from_stage = d.from_stage;
        *to_stage = d.to_stage;
        if (ops) *ops = n_ops;
        return 0;
    } catch (const ConfigError&) {
        return 1;
    }
}

}  // extern "C"

// The reference's best-case pipeline rate for `total_peers` peers given per-peer
// rates per stage (P/src/sim.cpp:88-116) — the CPU prediction for config E.
#include "swarmsim/sim.hpp"
extern "C" double ref_oracle_throughput(const double* rates, size_t n_stages, int64_t total_peers) {
    try {
        return swarmsim::sim::oracle_throughput(std::vector<double>(rates, rates + n_stages), total_peers);
    } catch (...) {
        return -1.0;
    }
}

// The reference's analytic stage cost (P/src/cost_model.cpp:50-70) for the
// cost-model compatibility test: out = {compute, comm, total, idle, utilization, square_cube}.
#include "swarmsim/cost_model.hpp"
extern "C" int ref_stage_cost(const int64_t* shape6, double act_bytes, const double* dev4, int overlap, double* out) {
    try {
        swarmsim::cost_model::LayerShape s{shape6[0], shape6[1], shape6[2], shape6[3], shape6[4], shape6[5], act_bytes};
        swarmsim::cost_model::DeviceProfile d{dev4[0], dev4[1], dev4[2], dev4[3]};
        const auto c = swarmsim::cost_model::stage_cost(s, d, overlap != 0);
        out[0] = c.compute_seconds;
        out[1] = c.comm_seconds;
        out[2] = c.total_seconds;
        out[3] = c.idle_fraction;
        out[4] = c.utilization;
        out[5] = swarmsim::cost_model::square_cube_ratio(s);
        return 0;
    } catch (...) {
        return 1;
    }
}

// The reference's discrete-event engine, unmodified (P/src/sim.cpp:811-830):
// SimConfig from the reference's own JSON schema (SimConfig::from_json,
// sim.cpp:920-992), one sim::run(config, seed).  Used by tests/test_engine.py to
// pin the B200 executor schedule (csrc/engine.cpp) decision-for-decision.
// Returns 0 ok, 1 ConfigError/ParseError, 3 other; buckets gets up to n_buckets.
#include <string>
extern "C" int ref_sim_run(const char* json, uint64_t seed, uint64_t* dispatched, uint64_t* completed,
                           double* buckets, size_t n_buckets, size_t* n_buckets_out) {
    try {
        const auto cfg = swarmsim::sim::SimConfig::from_json(std::string(json));
        const auto r = swarmsim::sim::run(cfg, seed);
        *dispatched = r.dispatched;
        *completed = r.completed;
        *n_buckets_out = r.throughput.completed.size();
        for (size_t i = 0; i < n_buckets && i < r.throughput.completed.size(); ++i) buckets[i] = r.throughput.completed[i];
        return 0;
    } catch (const swarmsim::ConfigError&) {
        return 1;
    } catch (const std::exception&) {
        return 3;
    }
}

// sim::run with a churn trace (SimConfig::from_json has no trace; the CLI loads it separately,
// P/tools/swarmsim_main.cpp) returning the counters and the event log (JSON lines, '\n'-joined).
extern "C" int ref_sim_run_churn(const char* json, const double* churn_t, const int64_t* churn_delta, size_t n_churn,
                                 uint64_t seed, uint64_t* counts /* dispatched, completed, requeued, abandoned */,
                                 double* buckets, size_t n_buckets, size_t* n_buckets_out, char* log, size_t log_cap) {
    try {
        auto cfg = swarmsim::sim::SimConfig::from_json(std::string(json));
        for (size_t i = 0; i < n_churn; ++i) cfg.churn.push_back(swarmsim::trace::TraceEvent{churn_t[i], churn_delta[i]});
        const auto r = swarmsim::sim::run(cfg, seed);
        counts[0] = r.dispatched;
        counts[1] = r.completed;
        counts[2] = r.requeued;
        counts[3] = r.abandoned;
        *n_buckets_out = r.throughput.completed.size();
        for (size_t i = 0; i < n_buckets && i < r.throughput.completed.size(); ++i) buckets[i] = r.throughput.completed[i];
        std::string all;
        for (const auto& line : r.event_log) all += line + "\n";
        if (log && log_cap) {
            const size_t n = std::min(all.size(), log_cap - 1);
            std::memcpy(log, all.data(), n);
            log[n] = 0;
        }
        return 0;
    } catch (const swarmsim::ConfigError&) {
        return 1;
    } catch (const std::exception&) {
        return 3;
    }
}
