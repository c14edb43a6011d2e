// Host-side control plane of the B200 SWARM pipeline: the per-trainer
// stochastic-wiring router (interleaved weighted round-robin, PAPER Alg. 1,
// PAPER:599-643) and the adaptive-rebalancing decision (Alg. 2).
//
// Decisions must be identical to the reference's on the same call sequence
// (SURVEY.md §8(a) a13/a14): the same keys (accumulated-time priority, then
// lowest peer id), the same EMA update gamma*dt + (1-gamma)*ema, the same
// stage-mate EMA seeding and virtual-time entry for newcomers, and the same
// floating-point operation order (P/src/wiring.cpp:33-120,
// P/src/rebalancer.cpp:25-69).  The data structure differs: each stage keeps an
// ordered set of (priority, peer) holding exactly one live entry per serving
// peer, instead of a lazily-pruned heap; the minimum is the same element.
#include <algorithm>
#include <cstdint>
#include <limits>
#include <map>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "swarm_b200.h"

namespace {

struct Peer {
    double ema = 0.0;
    double priority = 0.0;
    bool banned = false;
    std::vector<size_t> stages;  // ascending, unique
};

using Key = std::pair<double, uint64_t>;  // (priority, peer id): min = next pick

}  // namespace

struct swarm_router {
    double gamma = 0.1, epsilon = 1.0;
    std::unordered_map<uint64_t, Peer> peers;
    std::vector<std::set<Key>> ready;  // per stage: unbanned serving peers
    std::vector<double> ema_sum;       // per stage, over unbanned peers
    std::vector<size_t> ema_count;
    std::vector<double> vtime;         // priority of the latest pick per stage

    void unlist(uint64_t id, const Peer& p) {
        for (size_t s : p.stages) ready[s].erase({p.priority, id});
    }
    void list(uint64_t id, const Peer& p) {
        for (size_t s : p.stages) ready[s].insert({p.priority, id});
    }
    void leave_aggregates(const Peer& p) {
        if (p.banned) return;
        for (size_t s : p.stages) {
            ema_sum[s] -= p.ema;
            ema_count[s] -= 1;
        }
    }
};

namespace {
thread_local std::string g_err;
int bad(const std::string& m) {
    g_err = m;
    return SWARM_E_INVALID;
}
}  // namespace

extern "C" {

const char* swarm_router_last_error(void) { return g_err.c_str(); }

int swarm_router_create(size_t n_stages, double gamma, double epsilon, swarm_router_t* out) {
    if (n_stages == 0) return bad("RoutingState: need at least one stage");
    if (gamma <= 0.0 || gamma > 1.0) return bad("RoutingState: gamma must be in (0,1]");
    if (epsilon <= 0.0) return bad("RoutingState: epsilon must be positive");
    auto* r = new swarm_router;
    r->gamma = gamma;
    r->epsilon = epsilon;
    r->ready.resize(n_stages);
    r->ema_sum.assign(n_stages, 0.0);
    r->ema_count.assign(n_stages, 0);
    r->vtime.assign(n_stages, 0.0);
    *out = r;
    return SWARM_OK;
}

void swarm_router_destroy(swarm_router_t r) { delete r; }

int swarm_router_add_server(swarm_router_t r, uint64_t id, const size_t* stages, size_t n, double phase) {
    std::vector<size_t> st(stages, stages + n);
    std::sort(st.begin(), st.end());
    st.erase(std::unique(st.begin(), st.end()), st.end());
    for (size_t s : st)
        if (s >= r->ready.size()) return bad("add_server: stage index out of range");
    if (phase < 0.0 || phase > 1.0) return bad("add_server: phase must be in [0,1]");
    Peer& p = r->peers[id];
    if (!p.banned) r->unlist(id, p);
    r->leave_aggregates(p);
    // newcomer weight: mean EMA of its unbanned stage-mates, else epsilon
    double sum = 0.0;
    size_t cnt = 0;
    for (size_t s : st) {
        sum += r->ema_sum[s];
        cnt += r->ema_count[s];
    }
    p.ema = cnt > 0 ? sum / static_cast<double>(cnt) : r->epsilon;
    // enter `phase` of a round behind the latest pick of any stage it serves
    double vmax = 0.0;
    for (size_t s : st) vmax = std::max(vmax, r->vtime[s]);
    p.priority = std::max(r->epsilon, vmax + phase * p.ema);
    p.banned = false;
    p.stages = st;
    for (size_t s : p.stages) {
        r->ema_sum[s] += p.ema;
        r->ema_count[s] += 1;
    }
    r->list(id, p);
    return SWARM_OK;
}

int swarm_router_ban_server(swarm_router_t r, uint64_t id) {
    auto it = r->peers.find(id);
    if (it == r->peers.end()) return bad("ban_server: unknown peer");
    if (!it->second.banned) r->unlist(id, it->second);
    r->leave_aggregates(it->second);
    it->second.banned = true;
    return SWARM_OK;
}

void swarm_router_remove_server(swarm_router_t r, uint64_t id) {
    auto it = r->peers.find(id);
    if (it == r->peers.end()) return;
    if (!it->second.banned) r->unlist(id, it->second);
    r->leave_aggregates(it->second);
    r->peers.erase(it);
}

int swarm_router_is_banned(swarm_router_t r, uint64_t id) {
    auto it = r->peers.find(id);
    return it != r->peers.end() && it->second.banned;
}

int swarm_router_choose_server(swarm_router_t r, size_t stage, uint64_t* out) {
    if (stage >= r->ready.size()) return bad("choose_server: stage index out of range");
    auto& q = r->ready[stage];
    if (q.empty()) {
        g_err = "no unbanned peer serves stage " + std::to_string(stage);
        return SWARM_E_NO_PEER;
    }
    const uint64_t id = q.begin()->second;
    Peer& p = r->peers[id];
    r->unlist(id, p);
    r->vtime[stage] = p.priority;
    p.priority += p.ema;
    r->list(id, p);
    *out = id;
    return SWARM_OK;
}

int swarm_router_record_response(swarm_router_t r, uint64_t id, double elapsed) {
    if (elapsed <= 0.0) return bad("record_response: elapsed must be positive");
    auto it = r->peers.find(id);
    if (it == r->peers.end()) return bad("record_response: unknown peer");
    Peer& p = it->second;
    const double updated = r->gamma * elapsed + (1.0 - r->gamma) * p.ema;
    if (!p.banned)
        for (size_t s : p.stages) r->ema_sum[s] += updated - p.ema;
    p.ema = updated;
    return SWARM_OK;
}

int swarm_router_peer_state(swarm_router_t r, uint64_t id, double* ema, double* priority) {
    auto it = r->peers.find(id);
    if (it == r->peers.end()) return bad("peer_state: unknown peer");
    if (ema) *ema = it->second.ema;
    if (priority) *priority = it->second.priority;
    return SWARM_OK;
}

// Alg. 2 decision on a CSR load table (members of stage s: [offsets[s], offsets[s+1]),
// ascending peer id).  mover = UINT64_MAX when nobody moves.
int swarm_rebalance_decide(size_t n_stages, const size_t* offsets, const uint64_t* peers, const double* queues,
                           uint64_t* mover, size_t* from_stage, size_t* to_stage, size_t* op_count) {
    if (n_stages == 0) return bad("decide: empty load table");
    size_t ops = 0, s_min = 0, s_max = 0;
    double l_min = std::numeric_limits<double>::infinity(), l_max = -std::numeric_limits<double>::infinity();
    for (size_t s = 0; s < n_stages; ++s) {
        double load = 0.0;
        for (size_t i = offsets[s]; i < offsets[s + 1]; ++i, ++ops) load += queues[i];
        ++ops;
        if (load > l_max) l_max = load, s_max = s;  // first stage wins ties
        if (load < l_min) l_min = load, s_min = s;
    }
    *mover = UINT64_MAX;
    *from_stage = s_min;
    *to_stage = s_max;
    const size_t members = offsets[s_min + 1] - offsets[s_min];
    if (s_min != s_max && members > 1) {  // a stage keeps its last peer
        double q_min = std::numeric_limits<double>::infinity();
        for (size_t i = offsets[s_min]; i < offsets[s_min + 1]; ++i, ++ops)
            if (queues[i] < q_min) q_min = queues[i], *mover = peers[i];
    }
    if (op_count) *op_count += ops;
    return SWARM_OK;
}

}  // extern "C"
