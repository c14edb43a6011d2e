// Engine-driven executor schedule: the reference's
// discrete-event engine (P/src/sim.cpp:199-761) restated for a static
// population -- trainers, per-peer FIFO queues, IWRR dispatch, backward
// retracing the forward route, periodic all-reduce stalls -- emitting, in
// event-processing order, the records a real executor needs to run the same
// visits on GPUs: START (a peer begins a visit), HOP (a trainer's activation or
// gradient is dispatched to the next peer's queue), DONE (a microbatch
// finished its backward at stage 0) and ALLREDUCE (the stage-wide tick).
//
// Every rank runs the same engine on the same seed, so all ranks see one total
// order of records; each issues its own visits in START order and its
// point-to-point halves at the HOP's position.  Every dependency (a visit on
// its input HOP, a HOP on the visit that produced it) points backwards in that
// order, which is what makes the NCCL send/recv sequence deadlock-free.
//
// Decisions equal the reference's on the same SimConfig and seed: the same
// mt19937_64 draw sequence (spawn-time round-robin phases sim.cpp:327-334,
// staggered trainer starts :254-258), the same event ordering key (time, kind,
// seq; sim.cpp:145-151), the same router calls (choose_server on forward hops,
// route retrace on backward :405-436, record_response with the modeled visit
// time :486) -- tests/test_engine.py compares dispatched / completed / the
// per-bucket throughput with the reference's sim::run compiled in oracle/_ref.
// Churn, rebalancing and migration are the control plane's (out of scope for
// this schedule; swarm.py handles membership changes step-synchronously).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <deque>
#include <limits>
#include <queue>
#include <random>
#include <string>
#include <vector>

#include "swarm_b200.h"

namespace {

enum Kind : int { kStageComplete = 2, kAllReduceTick = 6, kTrainerStart = 7 };  // sim.cpp:127-136

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
    bool in_service = false;
    uint64_t token = 0;
    std::deque<Job> queue;
};

struct Trainer {
    size_t owner = 0;
    bool backward = false;
    size_t next_stage = 0;
    size_t in_flight_worker = 0;
    uint64_t microbatch = 0;
    std::vector<uint64_t> route;
    swarm_router_t routing = nullptr;
};

thread_local std::string g_err;
int bad(const std::string& m) {
    g_err = m;
    return SWARM_E_INVALID;
}

}  // namespace

struct swarm_engine {
    size_t n_stages = 0;
    double fwd = 0.0, bwd_mult = 2.0;
    double duration = 0.0, bucket = 60.0;
    double ar_period = 0.0, ar_stall = 0.0;
    std::mt19937_64 rng;
    std::vector<Worker> workers;
    std::vector<Trainer> trainers;
    std::priority_queue<Event, std::vector<Event>, EventLater> events;
    uint64_t next_seq = 0;
    double now = 0.0, stall_until = 0.0;
    double tick_next = std::numeric_limits<double>::infinity();  // next AllReduceTick (infinite: none)
    uint64_t dispatched = 0, completed = 0;
    std::vector<double> buckets;
    std::deque<swarm_engine_record> out;
    bool finished = false;

    ~swarm_engine() {
        for (auto& t : trainers) swarm_router_destroy(t.routing);
    }

    uint64_t draw(uint64_t n) { return rng() % n; }                                         // sim.cpp:523
    double uniform01() { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }             // sim.cpp:525
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

    void start_service(size_t widx) {  // sim.cpp:395-403
        Worker& w = workers[widx];
        if (w.in_service || w.queue.empty()) return;
        const double start = std::max(now, stall_until);
        w.in_service = true;
        w.token += 1;
        const Job& job = w.queue.front();
        const double end = start + visit_seconds(w, job.backward);
        emit(SWARM_ENG_START, job.trainer, w.stage, job.backward, static_cast<int64_t>(widx), -1, start, end);
        push(end, kStageComplete, widx, w.token);
    }

    int dispatch_current(size_t tidx, int64_t from) {  // sim.cpp:405-436 (static population)
        Trainer& tr = trainers[tidx];
        const size_t stage = tr.next_stage;
        uint64_t peer = 0;
        if (tr.backward) {
            peer = tr.route[stage];  // alive, serving `stage`, known and unbanned in a static run
        } else {
            const int rc = swarm_router_choose_server(tr.routing, stage, &peer);
            if (rc != SWARM_OK) return bad("engine: no peer serves stage " + std::to_string(stage));
        }
        tr.in_flight_worker = static_cast<size_t>(peer);
        dispatched += 1;
        emit(SWARM_ENG_HOP, tidx, stage, tr.backward, static_cast<int64_t>(peer), from, now, now);
        workers[peer].queue.push_back(Job{tidx, tr.backward});
        start_service(static_cast<size_t>(peer));
        return SWARM_OK;
    }

    int start_microbatch(size_t tidx) {  // sim.cpp:438-444
        Trainer& tr = trainers[tidx];
        tr.backward = false;
        tr.next_stage = 0;
        tr.route.assign(n_stages, 0);
        return dispatch_current(tidx, -1);
    }

    int advance_trainer(size_t tidx) {  // sim.cpp:493-510
        Trainer& tr = trainers[tidx];
        const int64_t from = static_cast<int64_t>(tr.in_flight_worker);
        if (!tr.backward) {
            tr.route[tr.next_stage] = tr.in_flight_worker;
            if (tr.next_stage + 1 < n_stages) tr.next_stage += 1;
            else tr.backward = true;  // turn around at the last stage
            return dispatch_current(tidx, from);
        }
        if (tr.next_stage > 0) {
            tr.next_stage -= 1;
            return dispatch_current(tidx, from);
        }
        completed += 1;  // record_completion, sim.cpp:512-518
        auto b = static_cast<size_t>(now / bucket);
        if (b >= buckets.size()) b = buckets.size() - 1;
        buckets[b] += 1.0;
        emit(SWARM_ENG_DONE, tidx, 0, true, from, from, now, now);
        tr.microbatch += 1;
        return start_microbatch(tidx);
    }

    int on_stage_complete(const Event& ev) {  // sim.cpp:472-491
        Worker& w = workers[ev.worker];
        if (ev.token != w.token || w.queue.empty()) return SWARM_OK;  // stale
        const Job job = w.queue.front();
        w.queue.pop_front();
        w.in_service = false;
        const int rc = swarm_router_record_response(trainers[job.trainer].routing, ev.worker,
                                                    visit_seconds(w, job.backward));
        if (rc != SWARM_OK) return rc;
        const int rc2 = advance_trainer(job.trainer);
        if (rc2 != SWARM_OK) return rc2;
        start_service(ev.worker);
        return SWARM_OK;
    }

    int handle(const Event& ev) {  // sim.cpp:345-357
        switch (ev.kind) {
            case kStageComplete: return on_stage_complete(ev);
            case kAllReduceTick:
                stall_until = now + ar_stall;
                emit(SWARM_ENG_ALLREDUCE, 0, 0, false, -1, -1, now, stall_until);
                return SWARM_OK;
            case kTrainerStart: return start_microbatch(ev.worker);
        }
        return SWARM_OK;
    }

    // process events until `want` records are buffered or the run ends
    int pump(size_t want) {
        while (!finished && out.size() < want) {
            // all-reduce ticks are generated lazily: the reference pushes them all up
            // front (sim.cpp:245-250), but a tick only ever ties another event on time,
            // where the kind decides, so its sequence number never matters
            const bool tick = tick_next < duration &&
                              (events.empty() || tick_next < events.top().time ||
                               (tick_next == events.top().time && kAllReduceTick < events.top().kind));
            if (!tick && events.empty()) {
                finished = true;
                break;
            }
            Event ev{};
            if (tick) {
                ev = Event{tick_next, kAllReduceTick, 0, 0, 0};
                tick_next += ar_period;
            } else {
                ev = events.top();
                events.pop();
            }
            if (ev.time > duration) {  // sim.cpp:262
                finished = true;
                break;
            }
            now = ev.time;
            const int rc = handle(ev);
            if (rc != SWARM_OK) return rc;
        }
        return SWARM_OK;
    }
};

extern "C" {

const char* swarm_engine_last_error(void) { return g_err.c_str(); }

int swarm_engine_create(size_t n_stages, size_t n_workers, const size_t* worker_stage, const double* worker_speed,
                        double forward_seconds, double backward_multiplier, size_t trainers_per_peer,
                        double allreduce_period, double allreduce_stall, double duration_seconds,
                        double bucket_seconds, uint64_t seed, swarm_engine_t* out) {
    // SimConfig::validate (sim.cpp:48-83), static-population subset
    if (!out) return bad("engine: null output handle");
    *out = nullptr;
    if (n_stages == 0) return bad("SimConfig: need at least one stage");
    if (!(duration_seconds > 0.0) || !(bucket_seconds > 0.0))
        return bad("SimConfig: duration and bucket width must be positive");
    if (trainers_per_peer == 0) return bad("SimConfig: trainers_per_peer must be >= 1");
    if (!(backward_multiplier > 0.0)) return bad("SimConfig: backward_multiplier must be > 0");
    if (!(forward_seconds > 0.0)) return bad("SimConfig: forward service time must be positive");
    if (!worker_stage || n_workers == 0) return bad("SimConfig: every stage needs an initial peer");
    std::vector<size_t> per_stage(n_stages, 0);
    for (size_t i = 0; i < n_workers; ++i) {
        if (worker_stage[i] >= n_stages) return bad("engine: worker stage out of range");
        if (i > 0 && worker_stage[i] < worker_stage[i - 1])
            return bad("engine: workers must be listed stage by stage (SimConfig::initial_peers order)");
        if (worker_speed && !(worker_speed[i] > 0.0)) return bad("engine: peer speed must be positive");
        per_stage[worker_stage[i]] += 1;
    }
    for (size_t s = 0; s < n_stages; ++s)
        if (per_stage[s] == 0) return bad("SimConfig: every stage needs an initial peer");

    auto* e = new swarm_engine;
    e->n_stages = n_stages;
    e->fwd = forward_seconds;
    e->bwd_mult = backward_multiplier;
    e->duration = duration_seconds;
    e->bucket = bucket_seconds;
    e->ar_period = allreduce_period;
    e->ar_stall = allreduce_stall;
    e->rng.seed(seed);
    e->buckets.assign(static_cast<size_t>(std::ceil(duration_seconds / bucket_seconds)), 0.0);
    e->workers.resize(n_workers);
    for (size_t i = 0; i < n_workers; ++i) {
        e->workers[i].stage = worker_stage[i];
        e->workers[i].speed = worker_speed ? worker_speed[i] : 1.0;
    }
    // spawn_trainer (sim.cpp:319-336): trainers_per_peer per worker, in worker order
    const double eps = 0.5 * (1.0 + backward_multiplier) * forward_seconds;
    for (size_t w = 0; w < n_workers; ++w) {
        for (size_t k = 0; k < trainers_per_peer; ++k) {
            Trainer tr;
            tr.owner = w;
            if (swarm_router_create(n_stages, 0.1, eps, &tr.routing) != SWARM_OK) {
                g_err = swarm_router_last_error();
                delete e;
                return SWARM_E_INVALID;
            }
            for (size_t v = 0; v < n_workers; ++v) {
                const size_t st = e->workers[v].stage;
                swarm_router_add_server(tr.routing, v, &st, 1, 1.0);
            }
            for (size_t s = 0; s < n_stages; ++s) {
                const uint64_t n = per_stage[s];
                if (n < 2) continue;
                uint64_t pick = 0;
                for (uint64_t c = e->draw(n); c > 0; --c) swarm_router_choose_server(tr.routing, s, &pick);
            }
            e->trainers.push_back(std::move(tr));
        }
    }
    // Engine::run (sim.cpp:235-259): all-reduce ticks, then staggered trainer starts
    if (allreduce_period > 0.0 && allreduce_stall > 0.0) e->tick_next = allreduce_period;
    const double stagger = static_cast<double>(n_stages) * (1.0 + backward_multiplier) * forward_seconds;
    for (size_t i = 0; i < e->trainers.size(); ++i) e->push(e->uniform01() * stagger, kTrainerStart, i, 0);
    *out = e;
    return SWARM_OK;
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

}  // extern "C"
