// Engine-driven executor schedule: the reference's
// discrete-event engine (P/src/sim.cpp:209-759, class Engine) restated in full
// -- trainers, per-peer FIFO queues, IWRR dispatch, backward retracing the
// forward route (or re-routing when that peer is gone), periodic all-reduce
// stalls, churn (peer leave / join from a trace), starvation, and Alg. 2
// rebalancing over the DHT stand-in (announce / publish_load with propagation
// delay and TTL, straggler timeout, migration downtime) -- emitting, in
// event-processing order, the records a real executor needs to run the same
// work on GPUs: START (a peer begins a visit), HOP (a trainer's activation or
// gradient is dispatched to a peer's queue; from_worker = the peer that
// produced it), DONE, ALLREDUCE, and the membership records LEAVE, JOIN,
// MIGRATE, MIGRATED and the REBALANCE decision log.
//
// Every rank runs the same engine on the same seed, so all ranks see one total
// order of records; each issues its own visits in START order and its
// point-to-point halves at the records both ranks share.  Every dependency points
// backwards in that order, which is what makes the NCCL sequence deadlock-free.
//
// Decisions equal the reference's on the same SimConfig, churn trace and seed:
// the same mt19937_64 draw sequence (spawn-time round-robin phases sim.cpp:327-334,
// newcomer phases :310-314 and :545-547, victim choice :556-581, staggered
// trainer starts :254-258), the same event ordering key (time, kind, seq;
// sim.cpp:145-151), the same router calls (the host C++ RoutingState of
// csrc/router.cpp, decision-identical to wiring.cpp), the same registry
// visibility rules (peer_registry.cpp:25-72) and Alg. 2 (rebalancer.cpp:25-69,
// swarm_rebalance_decide) -- tests/test_engine.py compares dispatched /
// completed / requeued / abandoned, the per-bucket throughput and the
// membership + rebalance-decision log with the reference's sim::run compiled in
// oracle/_ref, on random configurations and churn traces.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <deque>
#include <limits>
#include <map>
#include <queue>
#include <random>
#include <string>
#include <vector>

#include "swarm_b200.h"

namespace {

// sim.cpp:127-136
enum Kind : int {
    kPeerLeave = 0,
    kPeerJoin = 1,
    kStageComplete = 2,
    kMigrationComplete = 3,
    kRebalanceTick = 4,
    kRebalanceDecide = 5,
    kAllReduceTick = 6,
    kTrainerStart = 7
};

struct Event {
    double time;
    int kind;
    uint64_t seq;
    size_t worker;
    uint64_t token;
};
struct EventLater {
    bool operator()(const Event& a, const Event& b) const {
        if (a.time != b.time) return a.time > b.time;
        if (a.kind != b.kind) return a.kind > b.kind;
        return a.seq > b.seq;
    }
};

struct Job {
    size_t trainer;
    bool backward;
};

struct Worker {
    size_t stage = 0;
    double speed = 1.0;
    bool alive = true;
    bool migrating = false;
    bool in_service = false;
    uint64_t token = 0;
    std::deque<Job> queue;
    double q_integral = 0.0, q_since = 0.0, window_start = 0.0;
    std::vector<double> recent_loads;
};

struct Trainer {
    size_t owner = 0;
    bool active = true;
    bool starving = false;
    bool backward = false;
    size_t next_stage = 0;
    size_t in_flight_worker = 0;
    int64_t prev_worker = -1;  // the peer that produced the trainer's pending input (-1: tokens)
    uint64_t microbatch = 0;
    std::vector<uint64_t> route;
    swarm_router_t routing = nullptr;
};

// peer_registry.cpp: (stage -> peer -> entry), last write wins, propagation delay, TTL
struct Entry {
    double value = 0.0, visible_at = 0.0, expires_at = 0.0;
};
struct RegStage {
    std::map<uint64_t, Entry> announcements, loads;
};
bool visible(const Entry& e, double now) { return e.visible_at <= now && now < e.expires_at; }

thread_local std::string g_err;
int bad(const std::string& m) {
    g_err = m;
    return SWARM_E_INVALID;
}

}  // namespace

struct swarm_engine {
    swarm_sim_config cfg{};
    size_t n_stages = 0;
    double fwd = 0.0, bwd_mult = 2.0, load_tau = 0.0;
    size_t load_windows = 1;
    std::mt19937_64 rng;
    std::vector<Worker> workers;
    std::vector<Trainer> trainers;
    std::vector<int64_t> serving;          // serving_count_ per stage
    std::vector<std::vector<size_t>> starving;
    std::vector<char> starvation_logged;
    std::vector<RegStage> registry;
    std::vector<double> tick_times;
    std::priority_queue<Event, std::vector<Event>, EventLater> events;
    uint64_t next_seq = 0;
    int64_t alive_total = 0;
    double now = 0.0, stall_until = 0.0;
    double tick_next = std::numeric_limits<double>::infinity();  // next AllReduceTick (infinite: none)
    uint64_t dispatched = 0, completed = 0, requeued = 0, abandoned = 0;
    std::vector<double> buckets;
    std::deque<swarm_engine_record> out;
    bool finished = false;

    ~swarm_engine() {
        for (auto& t : trainers) swarm_router_destroy(t.routing);
    }

    uint64_t draw(uint64_t n) { return rng() % n; }                              // sim.cpp:523
    double uniform01() { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }  // sim.cpp:525
    void push(double t, int kind, size_t w, uint64_t tok) { events.push(Event{t, kind, next_seq++, w, tok}); }

    double visit_seconds(const Worker& w, bool backward) const {  // sim.cpp:361-364
        return (backward ? fwd * bwd_mult : fwd) / w.speed;
    }

    void emit(int kind, size_t trainer, size_t stage, bool backward, int64_t worker, int64_t from, double t,
              double t_end) {
        swarm_engine_record r{};
        r.time = t;
        r.end_time = t_end;
        r.kind = kind;
        r.backward = backward ? 1 : 0;
        r.trainer = static_cast<uint32_t>(trainer);
        r.stage = static_cast<uint32_t>(stage);
        r.worker = worker;
        r.from_worker = from;
        r.microbatch = trainer < trainers.size() ? trainers[trainer].microbatch : 0;
        out.push_back(r);
    }

    // -- registry (peer_registry.cpp:25-46) ------------------------------------
    void reg_announce(uint64_t peer, size_t stage, double t) {
        registry[stage].announcements[peer] = Entry{0.0, t + cfg.propagation_delay, t + cfg.announce_ttl};
    }
    void reg_withdraw(uint64_t peer, size_t stage) {
        registry[stage].announcements.erase(peer);
        registry[stage].loads.erase(peer);
    }
    void reg_publish_load(uint64_t peer, size_t stage, double q, double t) {
        auto it = registry[stage].announcements.find(peer);
        if (it == registry[stage].announcements.end()) return;  // (the engine only publishes announced peers)
        registry[stage].loads[peer] = Entry{q, t + cfg.propagation_delay, it->second.expires_at};
    }

    // -- population (sim.cpp:300-336) -------------------------------------------
    int add_server(Trainer& tr, size_t peer, size_t stage, double phase) {
        if (swarm_router_add_server(tr.routing, peer, &stage, 1, phase) != SWARM_OK)
            return bad(swarm_router_last_error());
        return SWARM_OK;
    }

    int add_worker(size_t stage, double speed, double t) {
        const size_t idx = workers.size();
        Worker w;
        w.stage = stage;
        w.speed = speed;
        w.q_since = w.window_start = t;
        workers.push_back(std::move(w));
        serving[stage] += 1;
        reg_announce(idx, stage, t);
        for (Trainer& tr : trainers)
            if (tr.active && add_server(tr, idx, stage, uniform01()) != SWARM_OK) return SWARM_E_INVALID;
        return SWARM_OK;
    }

    int spawn_trainer(size_t owner) {
        Trainer tr;
        tr.owner = owner;
        if (swarm_router_create(n_stages, 0.1, 0.5 * (1.0 + bwd_mult) * fwd, &tr.routing) != SWARM_OK)
            return bad(swarm_router_last_error());
        tr.route.assign(n_stages, 0);
        for (size_t v = 0; v < workers.size(); ++v)
            if (workers[v].alive && !workers[v].migrating && add_server(tr, v, workers[v].stage, 1.0) != SWARM_OK) {
                swarm_router_destroy(tr.routing);
                return SWARM_E_INVALID;
            }
        for (size_t s = 0; s < n_stages; ++s) {
            const uint64_t n = static_cast<uint64_t>(std::max<int64_t>(serving[s], 0));
            if (n < 2) continue;
            uint64_t pick = 0;
            for (uint64_t c = draw(n); c > 0; --c) swarm_router_choose_server(tr.routing, s, &pick);
        }
        trainers.push_back(std::move(tr));
        return SWARM_OK;
    }

    // -- queue load (sim.cpp:368-393) --------------------------------------------
    void touch_queue(Worker& w) {
        w.q_integral += static_cast<double>(w.queue.size()) * (now - w.q_since);
        w.q_since = now;
    }
    double average_load(Worker& w) {
        touch_queue(w);
        const double span = now - w.window_start;
        const double avg = span > 0.0 ? w.q_integral / span : static_cast<double>(w.queue.size());
        w.q_integral = 0.0;
        w.window_start = now;
        w.recent_loads.push_back(avg);
        if (w.recent_loads.size() > load_windows)
            w.recent_loads.erase(w.recent_loads.begin(), w.recent_loads.end() - load_windows);
        double sum = 0.0;
        for (double v : w.recent_loads) sum += v;
        return sum / static_cast<double>(w.recent_loads.size());
    }

    // -- dispatch / service (sim.cpp:395-519) ----------------------------------------
    void start_service(size_t widx) {
        Worker& w = workers[widx];
        if (!w.alive || w.migrating || w.in_service || w.queue.empty()) return;
        const double start = std::max(now, stall_until);
        w.in_service = true;
        w.token += 1;
        const Job& job = w.queue.front();
        const double end = start + visit_seconds(w, job.backward);
        emit(SWARM_ENG_START, job.trainer, w.stage, job.backward, static_cast<int64_t>(widx), -1, start, end);
        push(end, kStageComplete, widx, w.token);
    }

    int dispatch_current(size_t tidx) {
        Trainer& tr = trainers[tidx];
        const size_t stage = tr.next_stage;
        uint64_t peer = 0;
        bool picked = false;
        if (tr.backward) {  // retrace the recorded forward route where possible
            const uint64_t cand = tr.route[stage];
            const Worker& cw = workers[cand];
            double e = 0, p = 0;
            const bool knows = swarm_router_peer_state(tr.routing, cand, &e, &p) == SWARM_OK;
            if (cw.alive && !cw.migrating && cw.stage == stage && knows && !swarm_router_is_banned(tr.routing, cand)) {
                peer = cand;
                picked = true;
            }
        }
        if (!picked) {
            const int rc = swarm_router_choose_server(tr.routing, stage, &peer);
            if (rc == SWARM_E_NO_PEER) {
                mark_starving(tidx, stage);
                return SWARM_OK;
            }
            if (rc != SWARM_OK) return bad(swarm_router_last_error());
        }
        Worker& w = workers[peer];
        tr.in_flight_worker = static_cast<size_t>(peer);
        dispatched += 1;
        emit(SWARM_ENG_HOP, tidx, stage, tr.backward, static_cast<int64_t>(peer), tr.prev_worker, now, now);
        touch_queue(w);
        w.queue.push_back(Job{tidx, tr.backward});
        start_service(static_cast<size_t>(peer));
        return SWARM_OK;
    }

    int start_microbatch(size_t tidx) {  // sim.cpp:438-444
        Trainer& tr = trainers[tidx];
        tr.backward = false;
        tr.next_stage = 0;
        tr.prev_worker = -1;
        tr.route.assign(n_stages, 0);
        return dispatch_current(tidx);
    }

    void mark_starving(size_t tidx, size_t stage) {  // sim.cpp:446-459
        trainers[tidx].starving = true;
        starving[stage].push_back(tidx);
        if (serving[stage] == 0) starvation_logged[stage] = 1;
    }

    int wake_starving(size_t stage) {  // sim.cpp:461-471
        starvation_logged[stage] = 0;
        auto waiting = std::move(starving[stage]);
        starving[stage].clear();
        for (size_t tidx : waiting) {
            Trainer& tr = trainers[tidx];
            if (!tr.active || !tr.starving) continue;
            tr.starving = false;
            if (dispatch_current(tidx) != SWARM_OK) return SWARM_E_INVALID;
        }
        return SWARM_OK;
    }

    int advance_trainer(size_t tidx) {  // sim.cpp:493-510
        Trainer& tr = trainers[tidx];
        const int64_t from = static_cast<int64_t>(tr.in_flight_worker);
        tr.prev_worker = from;
        if (!tr.backward) {
            tr.route[tr.next_stage] = tr.in_flight_worker;
            if (tr.next_stage + 1 < n_stages) tr.next_stage += 1;
            else tr.backward = true;  // turn around at the last stage
            return dispatch_current(tidx);
        }
        if (tr.next_stage > 0) {
            tr.next_stage -= 1;
            return dispatch_current(tidx);
        }
        completed += 1;  // record_completion, sim.cpp:512-518
        auto b = static_cast<size_t>(now / cfg.bucket_seconds);
        if (b >= buckets.size()) b = buckets.size() - 1;
        buckets[b] += 1.0;
        emit(SWARM_ENG_DONE, tidx, 0, true, from, from, now, now);
        tr.microbatch += 1;
        return start_microbatch(tidx);
    }

    int on_stage_complete(const Event& ev) {  // sim.cpp:472-491
        Worker& w = workers[ev.worker];
        if (!w.alive || ev.token != w.token || w.queue.empty()) return SWARM_OK;  // stale
        const Job job = w.queue.front();
        touch_queue(w);
        w.queue.pop_front();
        w.in_service = false;
        Trainer& tr = trainers[job.trainer];
        if (!tr.active) {
            abandoned += 1;
        } else {
            if (swarm_router_record_response(tr.routing, ev.worker, visit_seconds(w, job.backward)) != SWARM_OK)
                return bad(swarm_router_last_error());
            if (advance_trainer(job.trainer) != SWARM_OK) return SWARM_E_INVALID;
        }
        start_service(ev.worker);
        return SWARM_OK;
    }

    int requeue(std::deque<Job>& orphans) {  // sim.cpp:608-624, 687-697
        for (const Job& job : orphans) {
            if (!trainers[job.trainer].active) {
                abandoned += 1;
                continue;
            }
            requeued += 1;
            if (dispatch_current(job.trainer) != SWARM_OK) return SWARM_E_INVALID;
        }
        return SWARM_OK;
    }

    // -- churn (sim.cpp:527-625) ---------------------------------------------------
    int on_peer_join() {
        size_t stage = 0;
        if (cfg.rebalance_periodic) {  // fill the short-staffed stage
            for (size_t s = 1; s < n_stages; ++s)
                if (serving[s] < serving[stage]) stage = s;
        } else {
            stage = static_cast<size_t>(draw(n_stages));
        }
        const size_t widx = workers.size();
        if (add_worker(stage, 1.0, now) != SWARM_OK) return SWARM_E_INVALID;
        alive_total += 1;
        for (Trainer& tr : trainers)
            if (tr.active && add_server(tr, widx, stage, uniform01()) != SWARM_OK) return SWARM_E_INVALID;
        emit(SWARM_ENG_JOIN, 0, stage, false, static_cast<int64_t>(widx), -1, now, now);
        for (size_t t = 0; t < cfg.trainers_per_peer; ++t) {
            if (spawn_trainer(widx) != SWARM_OK) return SWARM_E_INVALID;
            if (start_microbatch(trainers.size() - 1) != SWARM_OK) return SWARM_E_INVALID;
        }
        return wake_starving(stage);
    }

    int on_peer_leave() {
        if (alive_total <= static_cast<int64_t>(n_stages)) return SWARM_OK;  // population floor
        std::vector<std::vector<size_t>> by_stage(n_stages);
        std::vector<size_t> movers;
        for (size_t i = 0; i < workers.size(); ++i) {
            const Worker& w = workers[i];
            if (!w.alive) continue;
            if (w.migrating) movers.push_back(i);
            else if (serving[w.stage] >= 2) by_stage[w.stage].push_back(i);
        }
        std::vector<size_t> stages;
        for (size_t s = 0; s < n_stages; ++s)
            if (!by_stage[s].empty()) stages.push_back(s);
        if (stages.empty()) {
            if (movers.empty()) return SWARM_OK;
            return kill_worker(movers[draw(movers.size())]);
        }
        const auto& pool = by_stage[stages[draw(stages.size())]];
        return kill_worker(pool[draw(pool.size())]);
    }

    int kill_worker(size_t widx) {
        Worker& w = workers[widx];
        const bool was_migrating = w.migrating;
        w.alive = false;
        w.token += 1;
        alive_total -= 1;
        if (!was_migrating) {
            serving[w.stage] -= 1;
            reg_withdraw(widx, w.stage);
        }
        emit(SWARM_ENG_LEAVE, 0, w.stage, was_migrating, static_cast<int64_t>(widx), -1, now, now);
        for (Trainer& tr : trainers)  // this peer's trainers stop; their in-flight work is abandoned
            if (tr.owner == widx && tr.active) {
                tr.active = false;
                swarm_router_destroy(tr.routing);
                swarm_router_create(n_stages, 0.1, 1.0, &tr.routing);
            }
        for (Trainer& tr : trainers)
            if (tr.active) swarm_router_remove_server(tr.routing, widx);
        std::deque<Job> orphans;
        touch_queue(w);
        orphans.swap(w.queue);
        w.in_service = false;
        return requeue(orphans);
    }

    // -- rebalancing (sim.cpp:629-719) ---------------------------------------------
    void on_rebalance_tick() {
        for (size_t i = 0; i < workers.size(); ++i) {
            Worker& w = workers[i];
            if (!w.alive || w.migrating) continue;
            reg_announce(i, w.stage, now);
            reg_publish_load(i, w.stage, average_load(w), now);
        }
        push(now + cfg.straggler_timeout, kRebalanceDecide, 0, 0);
        tick_times.push_back(now);
    }

    int on_rebalance_decide() {
        const double tick_time = tick_times.empty() ? now : tick_times.front();
        if (!tick_times.empty()) tick_times.erase(tick_times.begin());
        // rebalancer::collect_loads (rebalancer.cpp:10-23): the table as visible at tick + timeout
        const double read_time = tick_time + cfg.straggler_timeout;
        std::vector<size_t> offsets{0};
        std::vector<uint64_t> peers;
        std::vector<double> queues;
        for (size_t s = 0; s < n_stages; ++s) {
            const RegStage& rs = registry[s];
            for (const auto& [peer, e] : rs.loads) {
                auto ann = rs.announcements.find(peer);
                if (ann == rs.announcements.end() || !visible(ann->second, read_time)) continue;
                if (!visible(e, read_time)) continue;
                peers.push_back(peer);
                queues.push_back(e.value);
            }
            offsets.push_back(peers.size());
        }
        uint64_t mover = 0;
        size_t from = 0, to = 0;
        if (swarm_rebalance_decide(n_stages, offsets.data(), peers.data(), queues.data(), &mover, &from, &to,
                                   nullptr) != SWARM_OK)
            return bad(swarm_router_last_error());
        if (mover == UINT64_MAX) {
            emit(SWARM_ENG_REBALANCE, 0, to, false, -1, static_cast<int64_t>(from), now, now);
            return SWARM_OK;
        }
        Worker& w = workers[mover];
        if (!w.alive || w.migrating || w.stage != from || serving[w.stage] < 2) {  // stale table
            emit(SWARM_ENG_REBALANCE, 0, to, true, -1, static_cast<int64_t>(from), now, now);
            return SWARM_OK;
        }
        emit(SWARM_ENG_REBALANCE, 0, to, false, static_cast<int64_t>(mover), static_cast<int64_t>(from), now, now);
        return begin_migration(mover, to);
    }

    int begin_migration(size_t widx, size_t to_stage) {
        Worker& w = workers[widx];
        const size_t from = w.stage;
        serving[w.stage] -= 1;
        reg_withdraw(widx, w.stage);
        w.migrating = true;
        w.stage = to_stage;  // destination; not serving until the download ends
        w.token += 1;
        for (Trainer& tr : trainers) {
            double e = 0, p = 0;
            if (swarm_router_peer_state(tr.routing, widx, &e, &p) == SWARM_OK &&
                !swarm_router_is_banned(tr.routing, widx))
                swarm_router_ban_server(tr.routing, widx);
        }
        const double downtime = static_cast<double>(cfg.state_transfer_bytes) * 8.0 / cfg.download_bps;
        emit(SWARM_ENG_MIGRATE, 0, to_stage, false, static_cast<int64_t>(widx), static_cast<int64_t>(from), now,
             now + downtime);
        std::deque<Job> orphans;
        touch_queue(w);
        orphans.swap(w.queue);
        w.in_service = false;
        if (requeue(orphans) != SWARM_OK) return SWARM_E_INVALID;
        push(now + downtime, kMigrationComplete, widx, w.token);
        return SWARM_OK;
    }

    int on_migration_complete(const Event& ev) {
        Worker& w = workers[ev.worker];
        if (!w.alive || ev.token != w.token) return SWARM_OK;  // preempted mid-transfer
        w.migrating = false;
        serving[w.stage] += 1;
        w.q_integral = 0.0;
        w.q_since = w.window_start = now;
        w.recent_loads.clear();
        reg_announce(ev.worker, w.stage, now);
        for (Trainer& tr : trainers)
            if (tr.active && add_server(tr, ev.worker, w.stage, uniform01()) != SWARM_OK) return SWARM_E_INVALID;
        emit(SWARM_ENG_MIGRATED, 0, w.stage, false, static_cast<int64_t>(ev.worker), -1, now, now);
        return wake_starving(w.stage);
    }

    int handle(const Event& ev) {  // sim.cpp:345-357
        switch (ev.kind) {
            case kStageComplete: return on_stage_complete(ev);
            case kPeerLeave: return on_peer_leave();
            case kPeerJoin: return on_peer_join();
            case kRebalanceTick: on_rebalance_tick(); return SWARM_OK;
            case kRebalanceDecide: return on_rebalance_decide();
            case kMigrationComplete: return on_migration_complete(ev);
            case kAllReduceTick:
                stall_until = now + cfg.allreduce_stall;
                emit(SWARM_ENG_ALLREDUCE, 0, 0, false, -1, -1, now, stall_until);
                return SWARM_OK;
            case kTrainerStart:
                if (trainers[ev.worker].active) return start_microbatch(ev.worker);
                return SWARM_OK;
        }
        return SWARM_OK;
    }

    // process events until `want` records are buffered or the run ends
    int pump(size_t want) {
        while (!finished && out.size() < want) {
            // all-reduce ticks are generated lazily: the reference pushes them all up
            // front (sim.cpp:245-250), but a tick only ever ties another event on time,
            // where the kind decides, so its sequence number never matters
            const bool tick = tick_next < cfg.duration_seconds &&
                              (events.empty() || tick_next < events.top().time ||
                               (tick_next == events.top().time && kAllReduceTick < events.top().kind));
            if (!tick && events.empty()) {
                finished = true;
                break;
            }
            Event ev{};
            if (tick) {
                ev = Event{tick_next, kAllReduceTick, 0, 0, 0};
                tick_next += cfg.allreduce_period;
            } else {
                ev = events.top();
                events.pop();
            }
            if (ev.time > cfg.duration_seconds) {  // sim.cpp:262
                finished = true;
                break;
            }
            now = ev.time;
            const int rc = handle(ev);
            if (rc != SWARM_OK) return rc;
        }
        return SWARM_OK;
    }

    int create(uint64_t seed) {
        const swarm_sim_config& c = cfg;
        // SimConfig::validate (sim.cpp:48-83)
        if (c.n_stages == 0) return bad("SimConfig: need at least one stage");
        if (!(c.duration_seconds > 0.0) || !(c.bucket_seconds > 0.0))
            return bad("SimConfig: duration and bucket width must be positive");
        if (c.trainers_per_peer == 0) return bad("SimConfig: trainers_per_peer must be >= 1");
        if (!(c.backward_multiplier > 0.0)) return bad("SimConfig: backward_multiplier must be > 0");
        if (c.rebalance_periodic && !(c.rebalance_period > 0.0))
            return bad("SimConfig: rebalance period must be positive");
        if (!(c.forward_seconds > 0.0)) return bad("SimConfig: forward service time must be positive");
        if (!c.worker_stage || c.n_workers == 0) return bad("SimConfig: every stage needs an initial peer");
        if (c.rebalance_periodic && !(c.download_bps > 0.0)) return bad("apply: download_bps must be positive");
        if (c.propagation_delay < 0.0) return bad("PeerRegistry: negative propagation delay");
        if (!(c.announce_ttl > 0.0)) return bad("announce: ttl must be positive");
        n_stages = c.n_stages;
        std::vector<size_t> per_stage(n_stages, 0);
        for (size_t i = 0; i < c.n_workers; ++i) {
            if (c.worker_stage[i] >= n_stages) return bad("engine: worker stage out of range");
            if (i > 0 && c.worker_stage[i] < c.worker_stage[i - 1])
                return bad("engine: workers must be listed stage by stage (SimConfig::initial_peers order)");
            if (c.worker_speed && !(c.worker_speed[i] > 0.0)) return bad("engine: peer speed must be positive");
            per_stage[c.worker_stage[i]] += 1;
        }
        for (size_t s = 0; s < n_stages; ++s)
            if (per_stage[s] == 0) return bad("SimConfig: every stage needs an initial peer");
        fwd = c.forward_seconds;
        bwd_mult = c.backward_multiplier;
        load_tau = static_cast<double>(c.trainers_per_peer) * static_cast<double>(n_stages) * (1.0 + bwd_mult) * fwd;
        if (c.rebalance_periodic)
            load_windows = static_cast<size_t>(std::max(1.0, std::ceil(load_tau / c.rebalance_period)));
        rng.seed(seed);
        buckets.assign(static_cast<size_t>(std::ceil(c.duration_seconds / c.bucket_seconds)), 0.0);
        serving.assign(n_stages, 0);
        starving.resize(n_stages);
        starvation_logged.assign(n_stages, 0);
        registry.resize(n_stages);
        // seed_initial_population (sim.cpp:274-290)
        for (size_t i = 0; i < c.n_workers; ++i)
            if (add_worker(c.worker_stage[i], c.worker_speed ? c.worker_speed[i] : 1.0, 0.0) != SWARM_OK)
                return SWARM_E_INVALID;
        for (size_t w = 0; w < workers.size(); ++w)
            for (size_t k = 0; k < c.trainers_per_peer; ++k)
                if (spawn_trainer(w) != SWARM_OK) return SWARM_E_INVALID;
        alive_total = static_cast<int64_t>(workers.size());
        // schedule_churn (sim.cpp:292-298): the trace expanded into single-peer steps (initial_peers is set,
        // so a t=0 join is churn, not the initial population)
        for (size_t i = 0; i < c.n_churn; ++i) {
            const int64_t n = std::llabs(c.churn_delta[i]);
            for (int64_t k = 0; k < n; ++k)
                if (c.churn_t[i] < c.duration_seconds)
                    push(c.churn_t[i], c.churn_delta[i] < 0 ? kPeerLeave : kPeerJoin, 0, 0);
        }
        // Engine::run (sim.cpp:231-259): rebalance ticks past the warm-up, all-reduce ticks, staggered starts
        if (c.rebalance_periodic) {
            const double warmup = 2.0 * load_tau;
            for (double t = c.rebalance_period; t < c.duration_seconds; t += c.rebalance_period)
                if (t >= warmup) push(t, kRebalanceTick, 0, 0);
        }
        if (c.allreduce_period > 0.0 && c.allreduce_stall > 0.0) tick_next = c.allreduce_period;
        const double stagger = static_cast<double>(n_stages) * (1.0 + bwd_mult) * fwd;
        for (size_t i = 0; i < trainers.size(); ++i) push(uniform01() * stagger, kTrainerStart, i, 0);
        return SWARM_OK;
    }
};

extern "C" {

const char* swarm_engine_last_error(void) { return g_err.c_str(); }

int swarm_engine_create_ex(const swarm_sim_config* cfg, uint64_t seed, swarm_engine_t* out) {
    if (!out || !cfg) return bad("engine: null argument");
    *out = nullptr;
    auto* e = new swarm_engine;
    e->cfg = *cfg;
    // own copies of the caller's arrays
    static_assert(sizeof(size_t) == 8, "");
    const int rc = e->create(seed);
    e->cfg.worker_stage = nullptr;
    e->cfg.worker_speed = nullptr;
    e->cfg.churn_t = nullptr;
    e->cfg.churn_delta = nullptr;
    if (rc != SWARM_OK) {
        delete e;
        return rc;
    }
    *out = e;
    return SWARM_OK;
}

int swarm_engine_create(size_t n_stages, size_t n_workers, const size_t* worker_stage, const double* worker_speed,
                        double forward_seconds, double backward_multiplier, size_t trainers_per_peer,
                        double allreduce_period, double allreduce_stall, double duration_seconds,
                        double bucket_seconds, uint64_t seed, swarm_engine_t* out) {
    swarm_sim_config c = swarm_sim_config_default();
    c.n_stages = n_stages;
    c.n_workers = n_workers;
    c.worker_stage = worker_stage;
    c.worker_speed = worker_speed;
    c.forward_seconds = forward_seconds;
    c.backward_multiplier = backward_multiplier;
    c.trainers_per_peer = trainers_per_peer;
    c.allreduce_period = allreduce_period;
    c.allreduce_stall = allreduce_stall;
    c.duration_seconds = duration_seconds;
    c.bucket_seconds = bucket_seconds;
    return swarm_engine_create_ex(&c, seed, out);
}

swarm_sim_config swarm_sim_config_default(void) {  // the reference's SimConfig defaults (sim.hpp:21-54)
    swarm_sim_config c{};
    c.n_stages = 4;
    c.forward_seconds = 1.0;
    c.backward_multiplier = 2.0;
    c.trainers_per_peer = 1;
    c.rebalance_periodic = 0;
    c.rebalance_period = 300.0;
    c.straggler_timeout = 5.0;
    c.propagation_delay = 1.0;
    c.announce_ttl = 300.0;
    c.state_transfer_bytes = 0;
    c.download_bps = 500e6;
    c.duration_seconds = 3600.0;
    c.bucket_seconds = 60.0;
    return c;
}

void swarm_engine_destroy(swarm_engine_t e) { delete e; }

size_t swarm_engine_n_trainers(swarm_engine_t e) { return e ? e->trainers.size() : 0; }

int swarm_engine_next(swarm_engine_t e, swarm_engine_record* records, size_t cap, size_t* n) {
    if (!e || !n || (cap > 0 && !records)) return bad("engine: null argument");
    *n = 0;
    const int rc = e->pump(cap);
    if (rc != SWARM_OK) return rc;
    while (*n < cap && !e->out.empty()) {
        records[(*n)++] = e->out.front();
        e->out.pop_front();
    }
    return SWARM_OK;
}

int swarm_engine_summary(swarm_engine_t e, uint64_t* dispatched, uint64_t* completed, double* buckets,
                         size_t n_buckets, double* now) {
    if (!e) return bad("engine: null handle");
    if (dispatched) *dispatched = e->dispatched;
    if (completed) *completed = e->completed;
    if (now) *now = e->now;
    if (buckets)
        for (size_t i = 0; i < n_buckets && i < e->buckets.size(); ++i) buckets[i] = e->buckets[i];
    return SWARM_OK;
}

int swarm_engine_counts(swarm_engine_t e, uint64_t* requeued, uint64_t* abandoned, size_t* n_workers,
                        int64_t* alive) {
    if (!e) return bad("engine: null handle");
    if (requeued) *requeued = e->requeued;
    if (abandoned) *abandoned = e->abandoned;
    if (n_workers) *n_workers = e->workers.size();
    if (alive) *alive = e->alive_total;
    return SWARM_OK;
}

int swarm_engine_worker(swarm_engine_t e, size_t worker, size_t* stage, int* alive, int* migrating) {
    if (!e || worker >= e->workers.size()) return bad("engine: bad worker");
    const Worker& w = e->workers[worker];
    if (stage) *stage = w.stage;
    if (alive) *alive = w.alive;
    if (migrating) *migrating = w.migrating;
    return SWARM_OK;
}

}  // extern "C"
