// Host driver: the engine-driven SWARM executor in C++ (SURVEY.md §8(f)1,
// §8(b) "host code stays in C++").  The reference's discrete-event engine decides
// (csrc/engine.cpp restates P/src/sim.cpp:209-759), the GPUs execute; the driver
// attaches real work at exactly the points where the reference advances
// simulated time:
//
//   START     (Engine::start_service, sim.cpp:395-403)  the serving peer runs the
//             stage visit on its stream (CUDA-graph replay per (peer, kind,
//             trainer, paired trainer, lane)).  A backward visit on a peer other
//             than the one that ran the microbatch's forward (the forward peer died
//             or migrated: dispatch_current re-routes, sim.cpp:405-436) first
//             recomputes the stage's forward from the trainer's stage input --
//             activation checkpointing, PAPER.md:206;
//   HOP       (Engine::dispatch_current)  the trainer's wire message [int8 codes |
//             fp32 scales | header] moves to the chosen peer: across ranks both
//             halves of the NCCL transfer are issued at the consuming visit's START
//             record (swarm_send/recv_compressed on the rank pair's communicator and
//             stream); on one GPU an event;
//   ALLREDUCE (AllReduceTick, sim.cpp:245-250, :352)  each stage's live peers sum
//             their fp32 gradient arenas (swarm_add_f32 among the peers a GPU
//             hosts, swarm_stage_allreduce across GPUs) and take an AdamW step over
//             the microbatches the stage served since the last tick;
//   DONE      (record_completion, sim.cpp:512-518);
//   LEAVE     (kill_worker, sim.cpp:583-625)  the peer stops serving; pending
//             transfers to it are dropped (its jobs come back as HOPs to others);
//             the stage communicators are rebuilt without it;
//   MIGRATE   (begin_migration, sim.cpp:673-702)  the mover drops its stage and
//             allocates the destination stage;
//   MIGRATED  (on_migration_complete, :704-719)  the mover downloads params + AdamW
//             m, v, step from a live stage-mate (the bytes rebalancer.cpp:71-75
//             counts) over NCCL and serves again; communicators rebuilt;
//   JOIN      (on_peer_join, :527-552)  a new peer (a spare GPU, or a shared one)
//             downloads its stage's state the same way and serves at once.
//
// swarm_driver_on_record() is the one entry point: swarm_driver_run() feeds it
// the driver's own engine, and the reference Engine can feed it the same records
// through an additive hook.  Every dependency points to an
// earlier record and every rank issues both halves of a transfer at the same
// record, so the NCCL sequence of every rank pair matches and cannot deadlock.
//
// Placement: peer pid (the reference's PeerId: initial peers stage by stage,
// joiners after them) lives on rank pid * world / n_initial (world >= peers: one
// peer per GPU; fewer GPUs: consecutive peers share one); a joiner beyond the
// initial peers goes to rank pid % world (a spare GPU when there is one).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "swarm_b200.h"

namespace {

thread_local std::string g_err;

int fail(const std::string& m, int rc = SWARM_E_INVALID) {
    g_err = m;
    return rc;
}

int cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return SWARM_OK;
    return fail(std::string(what) + ": " + cudaGetErrorString(e), SWARM_E_CUDA);
}

#define TRY(expr)                        \
    do {                                 \
        const int _rc = (expr);          \
        if (_rc != SWARM_OK) return _rc; \
    } while (0)
#define CU(expr) TRY(cuda((expr), #expr))

// one wire message buffer and the state of its producer / readers / transfers
struct Buf {
    void* p = nullptr;
    cudaEvent_t done = nullptr, read = nullptr, sent = nullptr, recvd = nullptr;
    bool has_done = false, has_read = false, has_sent = false, has_recvd = false;
    int xfer_op = -1;    // pending cross-rank half noted at the HOP: 0 send, 1 receive
    int xfer_rank = -1;  // the other rank
    int xfer_peer = -1;  // the consuming peer
};

struct Peer {
    int pid = 0, stage = 0;
    bool dead = false, migrating = false;
    swarm_stage_t st = nullptr;
    std::vector<cudaStream_t> lanes;
    int rr = 0, cur = 0;  // next lane (round robin), lane of the visit being issued
    int pend = -1;        // trainer whose deferred weight gradients are pending
    std::vector<cudaEvent_t> slot_ev;
    std::vector<char> has_slot;
    cudaEvent_t lane_ev = nullptr;
    // delayed parameter updates: the all-reduce + AdamW of bank b run on `upd` while the visits
    // continue on the other bank; upd_ev[b] marks that update's end
    cudaStream_t upd = nullptr;
    cudaEvent_t upd_ev[2] = {nullptr, nullptr};
    bool upd_pending[2] = {false, false};
    bool upd_fresh[2] = {false, false};  // the bank's update was issued at the last tick and not yet waited for
};

struct Graph {
    cudaGraphExec_t exec = nullptr;
    uint64_t kernels = 0;
};

struct VisitLog {
    uint32_t trainer, stage;
    uint64_t microbatch;
    int backward;
    int64_t peer;
};

uint64_t splitmix(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

}  // namespace

struct swarm_driver {
    swarm_driver_config cfg{};
    swarm_sim_config sim{};
    int S = 0, W = 1, R = 0, T = 0, Tmax = 0, tokens = 0, n0 = 0;
    // global membership, identical on every rank (it follows the records)
    std::vector<int> peer_stage, peer_alive, peer_migrating, peer_epoch, peer_steps;
    swarm_engine_t engine = nullptr;
    std::vector<std::unique_ptr<Peer>> peers;  // local peers
    std::vector<cudaStream_t> streams;         // owned (peers may share one: stream_per_peer = 0)
    std::unordered_map<int, Peer*> local;      // peer id -> local peer
    std::vector<Buf> bufs;                     // (kind, trainer, boundary): act = kind 0, grad = kind 1
    size_t wire_bytes = 0;
    void* scratch_wire = nullptr;  // the output of a recompute forward (not sent anywhere)
    float* scratch_loss = nullptr;
    // synthetic token pool (device), per-trainer token / target buffers, optional pinned host pool
    int32_t *pool_tok = nullptr, *pool_tgt = nullptr;
    const int32_t *host_tok = nullptr, *host_tgt = nullptr;
    int n_pool = 0;
    std::vector<int32_t*> tok, tgt;
    float* loss_sum = nullptr;
    std::vector<void*> allocs;
    // forward peer of each (trainer, stage) visit of the current microbatch (and its epoch)
    std::vector<int> fwd_peer, fwd_epoch;
    // per trainer, derived from the records alone (so any engine emitting START / HOP / DONE
    // drives the executor, e.g. the reference Engine through the hook of INTEGRATION.md §4):
    // its current job (stage, direction), the peer of that job's latest START and the peer that
    // ran the job before it (the producer of a requeued job's input), and its microbatch count
    std::vector<int> job_key, job_peer, prev_peer;
    std::vector<uint64_t> mb_count;
    // NCCL: one communicator + stream per rank pair, one per stage whose live peers span ranks
    std::vector<swarm_comm_t> pair_comm;
    std::vector<cudaStream_t> pair_stream;
    std::vector<swarm_comm_t> stage_comm;
    std::vector<swarm_comm_t> owned_comms;  // kept until destruction (a rebuilt stage's old one too)
    std::vector<int> served;                // backward visits per stage since the last tick (a global count)
    std::vector<VisitLog> log;
    std::unordered_map<uint64_t, Graph> graphs;
    std::unordered_set<uint64_t> warm;
    uint64_t records = 0, visits = 0, ticks = 0, optimizer_steps = 0, completed = 0, captures = 0;
    uint64_t captured_kernels = 0, replayed_kernels = 0, recomputes = 0, migrations = 0, state_bytes = 0;
    cudaEvent_t ev_tmp = nullptr;
    // tick cost on the compute streams: a (pre, post) timing-event pair around every stretch a
    // peer's stream spends in, or blocked on, a tick (the stage all-reduce + AdamW; with DPU the
    // first visit after a tick waiting for its bank's update); resolved into tick_ms
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tick_open;
    std::vector<cudaEvent_t> tick_pool;
    double tick_ms = 0.0;
    uint64_t tick_spans = 0;
    // profiled region: every visit eager (no graph) on one stream with the stages' kernel
    // profiling on, so the events around each kernel time it alone (the live roofline)
    bool prof = false;
    cudaStream_t prof_stream = nullptr;
    std::string prof_table;  // per-shape GEMM lines of the last profiled region (all local stages)
    swarm_engine_record pending{};  // run_until(-2): the membership record it stopped in front of
    bool has_pending = false;
    int bank = 0;  // DPU: the bank (weights shadow + gradient arena) the current interval's visits use

    cudaStream_t lane_stream(const Peer& p) const { return prof ? prof_stream : p.lanes[p.cur]; }

    std::vector<int> peer_rank0;  // optional explicit rank of each initial peer (swarm_driver_config.peer_rank)
    int rank_of_peer(int pid) const {
        if (pid < n0 && !peer_rank0.empty()) return peer_rank0[pid];
        if (pid < n0) return static_cast<int>(static_cast<int64_t>(pid) * W / n0);
        return pid % W;
    }

    Buf* buf_for(int t, int stage, bool backward) {  // the wire message the visit (t, stage, backward) reads
        if (backward) return stage == S - 1 ? nullptr : &bufs[(size_t(Tmax) + t) * (S - 1) + stage];
        return stage == 0 ? nullptr : &bufs[size_t(t) * (S - 1) + stage - 1];
    }
    Buf* out_for(int t, int stage, bool backward) {  // the message it writes
        if (backward) return stage == 0 ? nullptr : &bufs[(size_t(Tmax) + t) * (S - 1) + stage - 1];
        return stage == S - 1 ? nullptr : &bufs[size_t(t) * (S - 1) + stage];
    }

    int dalloc(void** p, size_t bytes) {
        CU(cudaMalloc(p, std::max<size_t>(bytes, 16)));
        allocs.push_back(*p);
        return cudaMemset(*p, 0, bytes) == cudaSuccess ? SWARM_OK : fail("driver: memset failed", SWARM_E_CUDA);
    }

    // ------------------------------------------------------------- graphs
    uint64_t gkey(int pid, int kind, int t, int p, int lane) const {  // + the DPU bank: graphs bake its pointers
        return (uint64_t(pid) << 48) | (uint64_t(kind) << 44) | (uint64_t(t & 0xFFFF) << 28) |
               (uint64_t((p + 1) & 0xFFFF) << 12) | (uint64_t(bank & 1) << 11) | uint64_t(lane & 0x7FF);
    }

    // paired-backward graphs (kind 2) per peer beyond SWARM_PAIR_GRAPH_CAP (default 48; 0 = no cap)
    // run eagerly: with several peers per stage the (trainer, partner) combinations keep appearing,
    // each capture + instantiation costs milliseconds, and an ever-growing graph set measured slower
    // (4 GPUs, 2 peers per stage, 16 trainers: 291k tokens/s uncapped, 321-322k capped at 32-64;
    // one GPU unchanged)
    std::unordered_map<int, int> pair_graphs;
    int pair_graph_cap() const {
        static const int cap = [] {
            const char* e = getenv("SWARM_PAIR_GRAPH_CAP");
            return e ? atoi(e) : 48;
        }();
        return cap;
    }
    int replay(uint64_t key, cudaStream_t st, const std::function<int()>& fn) {
        if (!cfg.use_graphs || !warm.count(key) || prof) {  // first use runs eagerly (lazy init, tensor-map caches)
            TRY(fn());
            if (!prof) warm.insert(key);
            return SWARM_OK;
        }
        auto it = graphs.find(key);
        if (it == graphs.end() && ((key >> 44) & 0xF) == 2 && pair_graph_cap() > 0) {
            const int pid = static_cast<int>(key >> 48);
            if (pair_graphs[pid] >= pair_graph_cap()) return fn();
            pair_graphs[pid] += 1;
        }
        if (it == graphs.end()) {
            const uint64_t k0 = swarm_launch_count();
            CU(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            const int rc = fn();
            cudaGraph_t g = nullptr;
            const cudaError_t e = cudaStreamEndCapture(st, &g);
            if (rc != SWARM_OK) return rc;
            CU(e);
            Graph gr;
            const cudaError_t ei = cudaGraphInstantiate(&gr.exec, g, 0);
            cudaGraphDestroy(g);
            CU(ei);
            gr.kernels = swarm_launch_count() - k0;
            captures += 1;
            captured_kernels += gr.kernels;
            it = graphs.emplace(key, gr).first;
        }
        CU(cudaGraphLaunch(it->second.exec, st));
        replayed_kernels += it->second.kernels;
        return SWARM_OK;
    }

    void forget_graphs(int pid) {  // the peer's stage object changed: its captured visits are invalid
        pair_graphs.erase(pid);
        for (auto it = graphs.begin(); it != graphs.end();) {
            if ((it->first >> 48) == uint64_t(pid)) {
                cudaGraphExecDestroy(it->second.exec);
                it = graphs.erase(it);
            } else {
                ++it;
            }
        }
        for (auto it = warm.begin(); it != warm.end();) it = ((*it >> 48) == uint64_t(pid)) ? warm.erase(it) : ++it;
    }

    // ------------------------------------------------------------- helpers
    int wait(cudaStream_t st, cudaEvent_t ev) { return cuda(cudaStreamWaitEvent(st, ev, 0), "cudaStreamWaitEvent"); }
    int timing_event(cudaEvent_t* e) {
        if (!tick_pool.empty()) {
            *e = tick_pool.back();
            tick_pool.pop_back();
            return SWARM_OK;
        }
        return cuda(cudaEventCreate(e), "cudaEventCreate");
    }
    int tick_begin(cudaStream_t st, cudaEvent_t* pre) {
        *pre = nullptr;
        if (prof) return SWARM_OK;
        TRY(timing_event(pre));
        return mark(*pre, st);
    }
    int tick_end(cudaStream_t st, cudaEvent_t pre) {
        if (!pre) return SWARM_OK;
        cudaEvent_t post = nullptr;
        TRY(timing_event(&post));
        TRY(mark(post, st));
        tick_open.emplace_back(pre, post);
        tick_spans += 1;
        if (tick_open.size() > 256) tick_resolve(false);
        return SWARM_OK;
    }
    // fold the completed pairs into tick_ms (block: wait for every open pair)
    void tick_resolve(bool block) {
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> keep;
        for (auto& [a, b] : tick_open) {
            if (block) cudaEventSynchronize(b);
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, a, b) == cudaSuccess) {
                tick_ms += ms;
                tick_pool.push_back(a);
                tick_pool.push_back(b);
            } else {
                cudaGetLastError();  // not ready yet
                keep.emplace_back(a, b);
            }
        }
        tick_open.swap(keep);
    }
    int mark(cudaEvent_t ev, cudaStream_t st) { return cuda(cudaEventRecord(ev, st), "cudaEventRecord"); }
    // `st` waits for everything issued so far on every lane of `p`
    int after_peer(cudaStream_t st, Peer& p) {
        for (cudaStream_t s : p.lanes) {
            if (s == st) continue;
            TRY(mark(ev_tmp, s));
            TRY(wait(st, ev_tmp));
        }
        return SWARM_OK;
    }

    int after_slot(Peer& p, int t) {
        if (!p.has_slot[t]) return SWARM_OK;
        return wait(lane_stream(p), p.slot_ev[t]);
    }
    int mark_slot(Peer& p, int t) {
        p.has_slot[t] = 1;
        return mark(p.slot_ev[t], lane_stream(p));
    }

    int pool_index(int t, uint64_t k) const { return static_cast<int>((uint64_t(t) * 7 + k) % uint64_t(n_pool)); }

    swarm_stage_config stage_cfg(int stage) const {
        swarm_stage_config sc = cfg.model;
        sc.is_first = stage == 0;
        sc.is_last = stage == S - 1;
        sc.max_slots = Tmax;
        sc.seed = cfg.seed * 1000 + stage;  // replicas of a stage start identical
        return sc;
    }

    int make_stage(Peer& p) {
        const swarm_stage_config sc = stage_cfg(p.stage);
        if (swarm_stage_create(&sc, &p.st) != SWARM_OK) return fail(std::string("driver: ") + swarm_last_error());
        if (cfg.pair_wgrad && swarm_stage_enable_wgrad_pairing_sets(p.st, std::max(2, Tmax)) != SWARM_OK)
            return fail(std::string("driver: ") + swarm_last_error());
        if (cfg.lanes > 1 && swarm_stage_enable_lanes(p.st, cfg.lanes) != SWARM_OK)
            return fail(std::string("driver: ") + swarm_last_error());
        if (cfg.dpu) {
            if (swarm_stage_enable_banks(p.st, nullptr) != SWARM_OK || swarm_stage_set_bank(p.st, bank) != SWARM_OK)
                return fail(std::string("driver: ") + swarm_last_error());
            CU(cudaDeviceSynchronize());
        }
        std::fill(p.has_slot.begin(), p.has_slot.end(), 0);
        p.pend = -1;
        p.rr = p.cur = 0;
        return SWARM_OK;
    }

    int add_local_peer(int pid, int stage) {
        auto p = std::make_unique<Peer>();
        p->pid = pid;
        p->stage = stage;
        TRY(make_stage(*p));
        if (!cfg.stream_per_peer && cfg.lanes > 1) return fail("driver: lanes need a stream per peer");
        for (int l = 0; l < cfg.lanes; ++l) {
            if (!cfg.stream_per_peer && !streams.empty()) {  // one stream per GPU, shared by its peers
                p->lanes.push_back(streams[0]);
                continue;
            }
            cudaStream_t s = nullptr;
            CU(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            streams.push_back(s);
            p->lanes.push_back(s);
        }
        p->slot_ev.resize(Tmax);
        p->has_slot.assign(Tmax, 0);
        for (auto& e : p->slot_ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&p->lane_ev, cudaEventDisableTiming));
        if (cfg.dpu) {
            CU(cudaStreamCreateWithFlags(&p->upd, cudaStreamNonBlocking));
            for (auto& e : p->upd_ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        local[pid] = p.get();
        peers.push_back(std::move(p));
        return SWARM_OK;
    }

    // ------------------------------------------------------------- visits
    int flush(Peer& p) {  // the peer's pending deferred weight gradients, alone, on its current lane
        const int t = p.pend;
        p.pend = -1;
        cudaStream_t st = lane_stream(p);
        if (cfg.lanes > 1) {
            TRY(swarm_stage_set_lane(p.st, p.cur));
            TRY(after_slot(p, t));
        }
        TRY(replay(gkey(p.pid, 3, t, -1, p.cur), st, [&] { return swarm_stage_flush_wgrad(p.st, t, t, st); }));
        if (cfg.lanes > 1) TRY(mark_slot(p, t));
        return SWARM_OK;
    }

    int load_tokens(int t, uint64_t k, int s, cudaStream_t st) {
        const int i = pool_index(t, k);
        const int32_t* src_tok = host_tok ? host_tok : pool_tok;
        const int32_t* src_tgt = host_tgt ? host_tgt : pool_tgt;
        const cudaMemcpyKind kind = host_tok ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        const size_t nb = size_t(tokens) * sizeof(int32_t);
        if (s == 0) CU(cudaMemcpyAsync(tok[t], src_tok + size_t(i) * tokens, nb, kind, st));
        if (s == S - 1) CU(cudaMemcpyAsync(tgt[t], src_tgt + size_t(i) * tokens, nb, kind, st));
        return SWARM_OK;
    }

    int visit(Peer& p, const swarm_engine_record& r, int s, int t, bool bwd, bool recompute, int* paired) {
        *paired = -1;
        cudaStream_t st = lane_stream(p);
        Buf* in = buf_for(t, s, bwd);
        Buf* out = out_for(t, s, bwd);
        Buf* fin = recompute ? buf_for(t, s, false) : nullptr;  // the stage input the recompute reads
        for (Buf* b : {in, fin}) {
            if (b && b->has_recvd) {  // the transfer into this buffer (pair stream)
                TRY(wait(st, b->recvd));
                b->has_recvd = false;
            }
            if (b && b->has_done) {  // produced by a peer on this GPU (another stream)
                TRY(wait(st, b->done));
                b->has_done = false;
            }
        }
        if (out && out->has_sent) {  // the previous message from this buffer has left
            TRY(wait(st, out->sent));
            out->has_sent = false;
        }
        if (out && out->has_read) {  // its previous local reader is done
            TRY(wait(st, out->read));
            out->has_read = false;
        }
        if ((!bwd || recompute) && p.pend == t) TRY(flush(p));  // a forward reuses the slot the pending wgrads read
        const float scale = 1.0f / static_cast<float>(tokens);
        if (recompute) {
            // backward on a peer that did not run this microbatch's forward: rebuild the slot's
            // activations from the trainer's stage input (activation checkpointing);
            // the output and the loss go to scratch (the pipeline already used them), the last
            // stage's LM-head gradient is accumulated here as the backward needs
            TRY(load_tokens(t, mb_count[t], s, st));
            const void* inp = s == 0 ? static_cast<const void*>(tok[t]) : fin->p;
            const int32_t* tg = s == S - 1 ? tgt[t] : nullptr;
            TRY(swarm_stage_forward(p.st, t, inp, tg, s == S - 1 ? nullptr : scratch_wire, scratch_loss, scale, st));
            recomputes += 1;
            if (fin) {
                TRY(mark(fin->read, st));
                fin->has_read = true;
            }
        }
        if (!bwd) {
            TRY(load_tokens(t, mb_count[t], s, st));
            const void* inp = s == 0 ? static_cast<const void*>(tok[t]) : in->p;
            void* o = out ? out->p : nullptr;
            const int32_t* tg = s == S - 1 ? tgt[t] : nullptr;
            TRY(replay(gkey(p.pid, 0, t, -1, p.cur), st,
                       [&] { return swarm_stage_forward(p.st, t, inp, tg, o, loss_sum, scale, st); }));
        } else {
            const void* gin = in ? in->p : nullptr;
            void* gout = out ? out->p : nullptr;
            if (!cfg.pair_wgrad) {
                TRY(replay(gkey(p.pid, 1, t, -1, p.cur), st,
                           [&] { return swarm_stage_backward(p.st, t, gin, gout, st); }));
            } else if (p.pend < 0) {  // first of a pair: data gradients now, dY kept in stash set t
                TRY(replay(gkey(p.pid, 1, t, -2, p.cur), st, [&] {
                    return swarm_stage_backward_ex(p.st, t, gin, gout, SWARM_WGRAD_DEFER, t, -1, 0, st);
                }));
                p.pend = t;
            } else {  // second: both visits' weight gradients as K = 2T GEMMs
                const int q = p.pend;
                p.pend = -1;
                *paired = q;
                if (cfg.lanes > 1) TRY(after_slot(p, q));  // the deferred visit's stash is complete
                TRY(replay(gkey(p.pid, 2, t, q, p.cur), st, [&] {
                    return swarm_stage_backward_ex(p.st, t, gin, gout, SWARM_WGRAD_PAIR, t, q, q, st);
                }));
            }
        }
        if (in) {
            TRY(mark(in->read, st));
            in->has_read = true;
        }
        if (out) {
            TRY(mark(out->done, st));
            out->has_done = true;
        }
        return SWARM_OK;
    }

    // issue this rank's half of a cross-rank transfer of buffer `b` (noted at the HOP, or a recompute input)
    int transfer(Buf& b, int op, int peer_rank, Peer* producer) {
        cudaStream_t ps = pair_stream[peer_rank];
        swarm_comm_t c = pair_comm[peer_rank];
        if (!c) return fail("driver: no communicator to rank " + std::to_string(peer_rank));
        const int other = R < peer_rank ? 1 : 0;  // ranks of a pair communicator are ordered by world rank
        if (op == 0) {
            if (b.has_done) {
                TRY(wait(ps, b.done));  // the producing visit (on its peer's stream)
                b.has_done = false;
            }
            if (producer) TRY(after_peer(ps, *producer));  // a resend: after everything the producer issued
            TRY(swarm_send_compressed(c, b.p, wire_bytes, other, ps));
            TRY(mark(b.sent, ps));
            b.has_sent = true;
        } else {
            if (b.has_read) {
                TRY(wait(ps, b.read));  // the previous reader of this buffer is done
                b.has_read = false;
            }
            TRY(swarm_recv_compressed(c, b.p, wire_bytes, other, ps));
            TRY(mark(b.recvd, ps));
            b.has_recvd = true;
        }
        return SWARM_OK;
    }

    int on_start(const swarm_engine_record& r) {
        const int s = static_cast<int>(r.stage), t = static_cast<int>(r.trainer), pid = static_cast<int>(r.worker);
        const bool bwd = r.backward != 0;
        if (t >= Tmax) return fail("driver: trainer beyond the driver's capacity");
        if (bwd) served[s] += 1;
        const int key = 2 * s + (bwd ? 1 : 0);
        if (job_key[t] != key) {
            prev_peer[t] = job_peer[t];
            job_key[t] = key;
        }
        job_peer[t] = pid;
        log.push_back(VisitLog{r.trainer, r.stage, mb_count[t], r.backward, r.worker});
        Buf* in = buf_for(t, s, bwd);
        if (in && in->xfer_op >= 0) {  // both ranks of a cross-rank hop, at the same record
            const int op = in->xfer_op;
            in->xfer_op = -1;
            TRY(transfer(*in, op, in->xfer_rank, nullptr));
        }
        // a backward on another peer than the forward's: its rank needs the trainer's stage input
        bool recompute = false;
        if (bwd) {
            const size_t k = size_t(t) * S + s;
            recompute = fwd_peer[k] != pid || fwd_epoch[k] != peer_epoch[pid];
            if (recompute && s > 0) {
                const int producer = fwd_peer[size_t(t) * S + s - 1];
                const int rp = rank_of_peer(producer), rc = rank_of_peer(pid);
                Buf* fin = buf_for(t, s, false);
                if (rp != rc && (rp == R || rc == R)) {
                    auto pit = local.find(producer);
                    TRY(transfer(*fin, rp == R ? 0 : 1, rp == R ? rc : rp, pit != local.end() ? pit->second : nullptr));
                }
            }
        } else {
            fwd_peer[size_t(t) * S + s] = pid;
            fwd_epoch[size_t(t) * S + s] = peer_epoch[pid];
        }
        auto it = local.find(pid);
        if (it == local.end()) return SWARM_OK;
        Peer& p = *it->second;
        p.cur = p.rr;
        p.rr = (p.rr + 1) % cfg.lanes;
        if (cfg.lanes > 1) {
            TRY(swarm_stage_set_lane(p.st, p.cur));
            TRY(after_slot(p, t));  // this slot's previous visit (e.g. the last stage's forward)
        }
        if (p.upd_pending[bank]) {  // DPU: this bank's weights are ready
            cudaEvent_t pre = nullptr;
            const bool first = p.upd_fresh[bank];  // (the first visit after the tick is the one that can stall)
            if (first) TRY(tick_begin(lane_stream(p), &pre));
            TRY(wait(lane_stream(p), p.upd_ev[bank]));
            if (first) TRY(tick_end(lane_stream(p), pre));
            p.upd_fresh[bank] = false;
        }
        int paired = -1;
        TRY(visit(p, r, s, t, bwd, recompute, &paired));
        if (cfg.lanes > 1) {
            TRY(mark_slot(p, t));
            if (paired >= 0) TRY(mark_slot(p, paired));  // the pair read that slot's activations and stash
        }
        visits += 1;
        return SWARM_OK;
    }

    int on_hop(const swarm_engine_record& r) {
        // same-rank hops need nothing: the consumer reads the producer's buffer in stream order
        // (an event orders two peers' streams on one GPU).  A cross-rank transfer is noted here and
        // issued by both ranks at the consuming visit's START: a receive posted at dispatch time
        // would spin an NCCL kernel on the SMs through the whole producing visit.
        const int t = static_cast<int>(r.trainer);
        if (t >= Tmax) return fail("driver: trainer beyond the driver's capacity");
        // the producer of the job's input: the peer that ran the trainer's previous job (a requeued
        // job's predecessor); engines that know it (csrc/engine.cpp) give the same value
        const int key = 2 * static_cast<int>(r.stage) + (r.backward ? 1 : 0);
        const int64_t src = r.from_worker >= -1 ? r.from_worker : (job_key[t] == key ? prev_peer[t] : job_peer[t]);
        const int64_t dst = r.worker;
        Buf* b = buf_for(t, static_cast<int>(r.stage), r.backward != 0);
        if (!b) return SWARM_OK;
        if (b->xfer_op >= 0 && b->xfer_peer != dst) b->xfer_op = -1;  // a requeue replaces an older route
        if (src < 0 || src == dst) return SWARM_OK;
        const int rs = rank_of_peer(static_cast<int>(src)), rd = rank_of_peer(static_cast<int>(dst));
        if (rs == rd || (rs != R && rd != R)) return SWARM_OK;
        b->xfer_op = rs == R ? 0 : 1;
        b->xfer_rank = rs == R ? rd : rs;
        b->xfer_peer = static_cast<int>(dst);
        return SWARM_OK;
    }

    int join_lanes(Peer& p) {  // lane 0 waits for every other lane
        p.cur = 0;
        if (prof) return SWARM_OK;  // one stream while profiling
        for (size_t i = 1; i < p.lanes.size(); ++i) {
            TRY(mark(p.lane_ev, p.lanes[i]));
            TRY(wait(p.lanes[0], p.lane_ev));
        }
        return SWARM_OK;
    }

    bool serving(const Peer& p) const { return !p.dead && !p.migrating; }

    // DPU tick: the interval's gradients (bank b) are all-reduced and applied by AdamW on each
    // stage lead's update stream, overlapped with the next interval, which computes on bank 1 - b (the
    // weights of the previous update: one step of delay) after that bank's own update has finished
    int on_allreduce_dpu() {
        ticks += 1;
        for (auto& p : peers) TRY(join_lanes(*p));
        for (auto& p : peers)
            if (p->pend >= 0 && serving(*p)) TRY(flush(*p));
        const int b = bank;
        for (int s = 0; s < S; ++s) {
            const int n = served[s];
            std::vector<Peer*> mine;
            for (auto& p : peers)
                if (serving(*p) && p->stage == s) mine.push_back(p.get());
            if (mine.empty() || n == 0) continue;
            Peer& lead = *mine[0];
            cudaStream_t u = lead.upd;
            for (Peer* q : mine) TRY(after_peer(u, *q));
            if (prof) {  // the profiled region's visits ran on the profile stream
                TRY(mark(ev_tmp, prof_stream));
                TRY(wait(u, ev_tmp));
            }
            const size_t np = swarm_stage_num_params(lead.st);
            float* lg = swarm_stage_grads_bank(lead.st, b);
            for (size_t i = 1; i < mine.size(); ++i) TRY(swarm_add_f32(lg, swarm_stage_grads_bank(mine[i]->st, b), np, u));
            if (stage_comm[s]) TRY(swarm_allreduce_sum(stage_comm[s], lg, np, SWARM_DTYPE_F32, u));
            for (size_t i = 1; i < mine.size(); ++i)
                CU(cudaMemcpyAsync(swarm_stage_grads_bank(mine[i]->st, b), lg, np * sizeof(float),
                                   cudaMemcpyDeviceToDevice, u));
            for (Peer* q : mine) TRY(swarm_stage_optimizer_step_bank(q->st, b, 1.0f / static_cast<float>(n), u));
            for (Peer* q : mine) {
                TRY(mark(q->upd_ev[b], u));
                q->upd_pending[b] = true;
                q->upd_fresh[b] = true;
            }
            optimizer_steps += mine.size();
        }
        for (int pid = 0; pid < static_cast<int>(peer_stage.size()); ++pid)
            if (peer_alive[pid] && !peer_migrating[pid] && served[peer_stage[pid]] > 0) peer_steps[pid] += 1;
        bank ^= 1;
        for (auto& p : peers)
            if (p->st) TRY(swarm_stage_set_bank(p->st, bank));
        for (auto& p : peers) {  // every lane of the peer continues after the join
            TRY(mark(p->lane_ev, p->lanes[0]));
            for (size_t i = 1; i < p->lanes.size(); ++i) TRY(wait(p->lanes[i], p->lane_ev));
        }
        std::fill(served.begin(), served.end(), 0);
        return SWARM_OK;
    }

    int on_allreduce() {
        if (cfg.dpu) return on_allreduce_dpu();
        ticks += 1;
        for (auto& p : peers) TRY(join_lanes(*p));  // the tick follows every visit on every lane
        for (auto& p : peers)
            if (p->pend >= 0 && serving(*p)) TRY(flush(*p));
        for (int s = 0; s < S; ++s) {
            const int n = served[s];
            if (n == 0) continue;
            std::vector<Peer*> mine;
            for (auto& p : peers)
                if (serving(*p) && p->stage == s) mine.push_back(p.get());
            if (mine.empty()) continue;
            Peer& lead = *mine[0];
            cudaStream_t st = lane_stream(lead);
            const size_t np = swarm_stage_num_params(lead.st);
            cudaEvent_t pre = nullptr;
            TRY(tick_begin(st, &pre));
            // the stage's gradient sum: peers sharing this GPU first, then across GPUs
            for (size_t i = 1; i < mine.size(); ++i) {
                TRY(after_peer(st, *mine[i]));
                TRY(swarm_add_f32(swarm_stage_grads(lead.st), swarm_stage_grads(mine[i]->st), np, st));
            }
            TRY(swarm_stage_allreduce(lead.st, stage_comm[s], st));
            for (size_t i = 1; i < mine.size(); ++i)
                CU(cudaMemcpyAsync(swarm_stage_grads(mine[i]->st), swarm_stage_grads(lead.st), np * sizeof(float),
                                   cudaMemcpyDeviceToDevice, st));
            for (Peer* q : mine)  // mean over the stage's microbatches since the last tick
                TRY(swarm_stage_optimizer_step(q->st, 1.0f / static_cast<float>(n), st));
            TRY(tick_end(st, pre));
            if (mine.size() > 1 && !prof) {
                TRY(mark(ev_tmp, st));
                for (size_t i = 1; i < mine.size(); ++i) {
                    cudaEvent_t q0 = nullptr;
                    TRY(tick_begin(mine[i]->lanes[0], &q0));
                    TRY(wait(mine[i]->lanes[0], ev_tmp));
                    TRY(tick_end(mine[i]->lanes[0], q0));
                }
            }
            optimizer_steps += mine.size();
        }
        for (int pid = 0; pid < static_cast<int>(peer_stage.size()); ++pid)
            if (peer_alive[pid] && !peer_migrating[pid] && served[peer_stage[pid]] > 0) peer_steps[pid] += 1;
        for (auto& p : peers) {  // every lane's next visit sees the updated weights
            if (prof) break;
            TRY(mark(p->lane_ev, p->lanes[0]));
            for (size_t i = 1; i < p->lanes.size(); ++i) TRY(wait(p->lanes[i], p->lane_ev));
        }
        std::fill(served.begin(), served.end(), 0);
        return SWARM_OK;
    }

    // ---------------------------------------------------------- membership
    int rebuild_stage_comms() {  // collective over the world: every rank makes the same S calls
        if (W == 1) return SWARM_OK;
        for (int s = 0; s < S; ++s) {
            std::vector<char> has(W, 0);
            for (int pid = 0; pid < static_cast<int>(peer_stage.size()); ++pid)
                if (peer_alive[pid] && !peer_migrating[pid] && peer_stage[pid] == s) has[rank_of_peer(pid)] = 1;
            int n = 0;
            for (char h : has) n += h;
            const int color = (n > 1 && has[R]) ? s : -1;
            swarm_comm_t c = nullptr;
            if (swarm_comm_split(cfg.comm, color, R, &c) != SWARM_OK)
                return fail(std::string("driver: ") + swarm_comm_last_error());
            if (c) owned_comms.push_back(c);
            stage_comm[s] = c;
        }
        return SWARM_OK;
    }

    void drop_transfers_to(int pid) {  // its jobs come back as HOPs to other peers
        for (Buf& b : bufs)
            if (b.xfer_op >= 0 && b.xfer_peer == pid) b.xfer_op = -1;
    }

    // a live stage-mate to download params + AdamW state from (lowest peer id), or -1
    int state_source(int stage, int except) const {
        for (int pid = 0; pid < static_cast<int>(peer_stage.size()); ++pid)
            if (pid != except && peer_alive[pid] && !peer_migrating[pid] && peer_stage[pid] == stage) return pid;
        return -1;
    }

    // copy params, AdamW m / v and the step count from `src` to `dst` (either may be remote)
    int copy_state(int src, int dst) {
        const int rs = rank_of_peer(src), rd = rank_of_peer(dst);
        if (rs != R && rd != R) return SWARM_OK;
        Peer* ps = rs == R ? local.at(src) : nullptr;
        Peer* pd = rd == R ? local.at(dst) : nullptr;
        swarm_stage_t any = ps ? ps->st : pd->st;
        const size_t np = swarm_stage_num_params(any);
        float *sp = nullptr, *sm = nullptr, *sv = nullptr, *dp = nullptr, *dm = nullptr, *dv = nullptr;
        int step = 0;
        if (ps) {
            sp = swarm_stage_params(ps->st);
            swarm_stage_optimizer_state(ps->st, &sm, &sv, &step);
        }
        if (pd) {
            dp = swarm_stage_params(pd->st);
            swarm_stage_optimizer_state(pd->st, &dm, &dv, nullptr);
        }
        state_bytes += np * 12;
        if (ps && ps->upd) {  // DPU: the source's update in flight lands first
            TRY(mark(ev_tmp, ps->upd));
            for (cudaStream_t s : ps->lanes) TRY(wait(s, ev_tmp));
        }
        if (rs == rd) {  // both on this GPU
            cudaStream_t st = pd->lanes[0];
            TRY(after_peer(st, *ps));
            for (auto [a, b] : {std::pair{dp, sp}, std::pair{dm, sm}, std::pair{dv, sv}})
                CU(cudaMemcpyAsync(a, b, np * sizeof(float), cudaMemcpyDeviceToDevice, st));
        } else {
            const int other = rs == R ? rd : rs;
            cudaStream_t ps_ = pair_stream[other];
            swarm_comm_t c = pair_comm[other];
            const int peer_in_pair = R < other ? 1 : 0;
            TRY(after_peer(ps_, ps ? *ps : *pd));
            TRY(swarm_comm_group_start());
            if (ps) {
                for (float* a : {sp, sm, sv}) TRY(swarm_send_compressed(c, a, np * sizeof(float), peer_in_pair, ps_));
            } else {
                for (float* a : {dp, dm, dv}) TRY(swarm_recv_compressed(c, a, np * sizeof(float), peer_in_pair, ps_));
            }
            TRY(swarm_comm_group_end());
            if (pd) {  // the new peer's lanes start after the download
                TRY(mark(ev_tmp, ps_));
                for (cudaStream_t s : pd->lanes) TRY(wait(s, ev_tmp));
            }
        }
        if (pd) {
            TRY(swarm_stage_set_step(pd->st, peer_steps[src]));
            TRY(swarm_stage_sync_shadow(pd->st, pd->lanes[0]));
            TRY(mark(ev_tmp, pd->lanes[0]));
            for (cudaStream_t s : pd->lanes) TRY(wait(s, ev_tmp));
        }
        return SWARM_OK;
    }

    int on_leave(const swarm_engine_record& r) {
        const int pid = static_cast<int>(r.worker);
        peer_alive[pid] = 0;
        drop_transfers_to(pid);
        auto it = local.find(pid);
        if (it != local.end()) it->second->dead = true;  // its GPU stops serving (memory kept)
        if (!r.backward) TRY(rebuild_stage_comms());  // a migrating peer was not in any group
        return SWARM_OK;
    }

    int on_migrate(const swarm_engine_record& r) {
        const int pid = static_cast<int>(r.worker), to = static_cast<int>(r.stage);
        peer_migrating[pid] = 1;
        peer_stage[pid] = to;
        peer_epoch[pid] += 1;
        migrations += 1;
        drop_transfers_to(pid);
        auto it = local.find(pid);
        if (it != local.end()) {  // drop the old stage, allocate the destination's (filled at MIGRATED)
            Peer& p = *it->second;
            for (cudaStream_t s : p.lanes) CU(cudaStreamSynchronize(s));
            forget_graphs(pid);
            swarm_stage_destroy(p.st);
            p.st = nullptr;
            p.stage = to;
            p.migrating = true;
            TRY(make_stage(p));
        }
        return rebuild_stage_comms();
    }

    int on_migrated(const swarm_engine_record& r) {
        const int pid = static_cast<int>(r.worker);
        const int src = state_source(static_cast<int>(r.stage), pid);
        peer_migrating[pid] = 0;
        if (src >= 0) {
            TRY(copy_state(src, pid));
            peer_steps[pid] = peer_steps[src];
        }
        auto it = local.find(pid);
        if (it != local.end()) it->second->migrating = false;
        return rebuild_stage_comms();
    }

    int on_join(const swarm_engine_record& r) {
        const int pid = static_cast<int>(r.worker), stage = static_cast<int>(r.stage);
        if (pid != static_cast<int>(peer_stage.size())) return fail("driver: join out of order");
        const int src = state_source(stage, -1);
        peer_stage.push_back(stage);
        peer_alive.push_back(1);
        peer_migrating.push_back(0);
        peer_epoch.push_back(0);
        peer_steps.push_back(0);
        if (rank_of_peer(pid) == R) TRY(add_local_peer(pid, stage));
        if (src >= 0) {
            TRY(copy_state(src, pid));
            peer_steps[pid] = peer_steps[src];
        }
        return rebuild_stage_comms();
    }

    int on_record(const swarm_engine_record& r) {
        records += 1;
        switch (r.kind) {
            case SWARM_ENG_START: return on_start(r);
            case SWARM_ENG_HOP: return on_hop(r);
            case SWARM_ENG_ALLREDUCE: return on_allreduce();
            case SWARM_ENG_DONE:
                completed += 1;
                if (r.trainer < mb_count.size()) {
                    mb_count[r.trainer] += 1;
                    job_key[r.trainer] = -1;  // the next microbatch starts from the tokens
                }
                return SWARM_OK;
            case SWARM_ENG_LEAVE: return on_leave(r);
            case SWARM_ENG_JOIN: return on_join(r);
            case SWARM_ENG_MIGRATE: return on_migrate(r);
            case SWARM_ENG_MIGRATED: return on_migrated(r);
            case SWARM_ENG_REBALANCE: return SWARM_OK;
        }
        return fail("driver: unknown record kind");
    }

    ~swarm_driver() {
        cudaDeviceSynchronize();
        for (auto& [a, b] : tick_open) {
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
        for (cudaEvent_t e : tick_pool) cudaEventDestroy(e);
        for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.exec);
        for (auto& p : peers) {
            for (cudaEvent_t e : p->slot_ev) cudaEventDestroy(e);
            if (p->lane_ev) cudaEventDestroy(p->lane_ev);
            for (cudaEvent_t e : p->upd_ev)
                if (e) cudaEventDestroy(e);
            if (p->upd) cudaStreamDestroy(p->upd);
            if (p->st) swarm_stage_destroy(p->st);
        }
        for (cudaStream_t s : streams) cudaStreamDestroy(s);
        for (Buf& b : bufs)
            for (cudaEvent_t e : {b.done, b.read, b.sent, b.recvd})
                if (e) cudaEventDestroy(e);
        for (cudaStream_t s : pair_stream)
            if (s) cudaStreamDestroy(s);
        for (swarm_comm_t c : owned_comms) swarm_comm_destroy(c);
        if (ev_tmp) cudaEventDestroy(ev_tmp);
        if (prof_stream) cudaStreamDestroy(prof_stream);
        for (void* p : allocs) cudaFree(p);
        if (engine) swarm_engine_destroy(engine);
    }

    int create(const swarm_sim_config* user_sim, const int* layout_in) {
        const swarm_driver_config& c = cfg;
        S = c.n_stages;
        W = c.world;
        R = c.rank;
        if (S < 1 || W < 1 || R < 0 || R >= W) return fail("driver: bad stage count / world / rank");
        if (c.lanes < 1) return fail("driver: lanes must be >= 1");
        if (c.n_pool < 1) return fail("driver: n_pool must be >= 1");
        if (W > 1 && !c.comm) return fail("driver: world > 1 needs a world communicator");
        // the engine's SimConfig: the caller's, or the static one the simple fields describe
        std::vector<size_t> wst;
        if (user_sim) {
            sim = *user_sim;
            if (static_cast<int>(sim.n_stages) != S) return fail("driver: sim.n_stages != n_stages");
            wst.assign(sim.worker_stage, sim.worker_stage + sim.n_workers);
        } else {
            std::vector<int> layout(S, 1);
            if (layout_in) {
                for (int s = 0; s < S; ++s) layout[s] = layout_in[s];
            } else if (W > S) {
                if (W % S) return fail("driver: world must be a multiple of the stage count");
                std::fill(layout.begin(), layout.end(), W / S);
            } else if (S % W) {
                return fail("driver: stage count must be a multiple of world");
            }
            for (int s = 0; s < S; ++s) {
                if (layout[s] < 1) return fail("driver: every stage needs a peer");
                for (int k = 0; k < layout[s]; ++k) wst.push_back(s);
            }
            sim = swarm_sim_config_default();
            sim.n_stages = S;
            sim.forward_seconds = c.forward_seconds;
            sim.backward_multiplier = c.backward_multiplier;
            sim.trainers_per_peer = c.trainers_per_peer;
            sim.allreduce_period = c.allreduce_period;
            sim.allreduce_stall = c.allreduce_stall;
            sim.duration_seconds = c.duration_seconds;
            sim.bucket_seconds = std::max(c.duration_seconds / 64, 1e-9);
            sim.worker_speed = nullptr;
        }
        n0 = static_cast<int>(wst.size());
        if (c.peer_rank) {
            peer_rank0.assign(c.peer_rank, c.peer_rank + n0);
            for (int r : peer_rank0)
                if (r < 0 || r >= W) return fail("driver: peer_rank entries must lie in [0, world)");
        }
        sim.n_workers = wst.size();
        sim.worker_stage = wst.data();
        const int rc_e = swarm_engine_create_ex(&sim, c.seed, &engine);
        if (rc_e != SWARM_OK) return fail(std::string("driver: ") + swarm_engine_last_error());
        int joins = 0;  // peers the churn trace can add (each brings trainers_per_peer trainers)
        for (size_t i = 0; i < sim.n_churn; ++i) joins += sim.churn_delta[i] > 0 ? int(sim.churn_delta[i]) : 0;
        sim.worker_stage = nullptr;
        sim.worker_speed = nullptr;
        sim.churn_t = nullptr;
        sim.churn_delta = nullptr;
        T = static_cast<int>(swarm_engine_n_trainers(engine));
        Tmax = T + joins * static_cast<int>(sim.trainers_per_peer);
        served.assign(S, 0);
        for (int pid = 0; pid < n0; ++pid) {
            peer_stage.push_back(static_cast<int>(wst[pid]));
            peer_alive.push_back(1);
            peer_migrating.push_back(0);
            peer_epoch.push_back(0);
            peer_steps.push_back(0);
        }
        fwd_peer.assign(size_t(Tmax) * S, -1);
        fwd_epoch.assign(size_t(Tmax) * S, 0);
        job_key.assign(Tmax, -1);
        job_peer.assign(Tmax, -1);
        prev_peer.assign(Tmax, -1);
        mb_count.assign(Tmax, 0);
        const swarm_stage_config& m = c.model;
        tokens = m.seq_len * m.micro_batch;
        for (int pid = 0; pid < n0; ++pid)
            if (rank_of_peer(pid) == R) TRY(add_local_peer(pid, peer_stage[pid]));
        // wire messages: size from the model (every stage's wire has the same size)
        {
            swarm_stage_t probe = peers.empty() ? nullptr : peers[0]->st;
            swarm_stage_config sc = m;
            sc.n_layers = 1;
            sc.max_slots = 1;
            sc.is_first = 0;
            sc.is_last = 0;
            if (!probe && swarm_stage_create(&sc, &probe) != SWARM_OK)
                return fail(std::string("driver: ") + swarm_last_error());
            wire_bytes = swarm_stage_wire_bytes(probe);
            if (peers.empty()) swarm_stage_destroy(probe);
        }
        bufs.resize(size_t(2) * Tmax * std::max(S - 1, 0));
        for (Buf& b : bufs) {
            TRY(dalloc(&b.p, wire_bytes));
            for (cudaEvent_t* e : {&b.done, &b.read, &b.sent, &b.recvd})
                CU(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        }
        TRY(dalloc(&scratch_wire, wire_bytes));
        TRY(dalloc(reinterpret_cast<void**>(&scratch_loss), sizeof(float)));
        // synthetic pool (identical on every rank): tokens uniform over the vocab, targets the next token
        n_pool = c.n_pool;
        {
            std::vector<int32_t> ht(size_t(n_pool) * tokens), hg(ht.size());
            uint64_t x = c.seed + 17;
            for (auto& v : ht) v = static_cast<int32_t>(splitmix(x) % uint64_t(std::max(m.vocab, 1)));
            for (int i = 0; i < n_pool; ++i)
                for (int j = 0; j < tokens; ++j) hg[size_t(i) * tokens + j] = ht[size_t(i) * tokens + (j + 1) % tokens];
            TRY(dalloc(reinterpret_cast<void**>(&pool_tok), ht.size() * 4));
            TRY(dalloc(reinterpret_cast<void**>(&pool_tgt), hg.size() * 4));
            CU(cudaMemcpy(pool_tok, ht.data(), ht.size() * 4, cudaMemcpyHostToDevice));
            CU(cudaMemcpy(pool_tgt, hg.data(), hg.size() * 4, cudaMemcpyHostToDevice));
        }
        tok.resize(Tmax);
        tgt.resize(Tmax);
        for (int t = 0; t < Tmax; ++t) {
            TRY(dalloc(reinterpret_cast<void**>(&tok[t]), size_t(tokens) * 4));
            TRY(dalloc(reinterpret_cast<void**>(&tgt[t]), size_t(tokens) * 4));
        }
        TRY(dalloc(reinterpret_cast<void**>(&loss_sum), sizeof(float)));
        CU(cudaEventCreateWithFlags(&ev_tmp, cudaEventDisableTiming));
        // communicators (collective over the world: every rank makes the same calls in the same order)
        pair_comm.assign(W, nullptr);
        pair_stream.assign(W, nullptr);
        stage_comm.assign(S, nullptr);
        if (W > 1) {
            // one communicator per rank pair: W - 1 (or W) rounds of a round-robin pairing, each a
            // split of the world
            const int n = W % 2 ? W + 1 : W;
            for (int round = 0; round < n - 1; ++round) {
                int partner = -1, color = -1;
                for (int i = 0; i < n / 2; ++i) {  // circle method: position 0 fixed, the rest rotate
                    auto at = [&](int k) { return k == 0 ? 0 : 1 + (k - 1 + round) % (n - 1); };
                    const int a = at(i), b = at(n - 1 - i);
                    if (a >= W || b >= W) continue;
                    if (a == R) partner = b, color = i;
                    if (b == R) partner = a, color = i;
                }
                // the pair communicators carry single wire messages: a few CTAs suffice, and a receive
                // posted ahead of its sender spins fewer SMs away from the stage's GEMMs (measured at
                // 4 x 1: the profiled GEMMs 247 -> 179 ms/step with 4 instead of NCCL's default channels)
                swarm_comm_t pc = nullptr;
                const char* mc = getenv("SWARM_P2P_MAX_CTAS");
                if (swarm_comm_split_ex(c.comm, color, R, mc ? atoi(mc) : 4, &pc) != SWARM_OK)
                    return fail(std::string("driver: ") + swarm_comm_last_error());
                if (pc) {
                    owned_comms.push_back(pc);
                    pair_comm[partner] = pc;
                    CU(cudaStreamCreateWithFlags(&pair_stream[partner], cudaStreamNonBlocking));
                }
            }
            TRY(rebuild_stage_comms());
        }
        CU(cudaDeviceSynchronize());  // stage initialisation ran on the legacy stream; peer streams do not wait on it
        return SWARM_OK;
    }
};

extern "C" {

const char* swarm_driver_last_error(void) { return g_err.c_str(); }

int swarm_driver_create(const swarm_driver_config* cfg, swarm_driver_t* out) {
    if (!cfg || !out) return fail("driver: null argument");
    *out = nullptr;
    auto d = std::make_unique<swarm_driver>();
    d->cfg = *cfg;
    d->cfg.sim = nullptr;  // read once by create(): the driver keeps no caller pointer
    d->cfg.layout = nullptr;
    const int rc = d->create(cfg->sim, cfg->layout);
    if (rc != SWARM_OK) return rc;
    *out = d.release();
    return SWARM_OK;
}

void swarm_driver_destroy(swarm_driver_t d) { delete d; }

int swarm_driver_on_record(swarm_driver_t d, const swarm_engine_record* r) {
    if (!d || !r) return fail("driver: null argument");
    return d->on_record(*r);
}

int swarm_driver_run_until(swarm_driver_t d, uint64_t n_microbatches, int stop_kind, uint64_t* completed) {
    if (!d) return fail("driver: null handle");
    const uint64_t target = d->completed + n_microbatches, start = d->completed;
    swarm_engine_record rec;
    while (d->completed < target) {
        size_t n = 0;
        if (d->has_pending) {  // a membership record held back by the previous call
            rec = d->pending;
            d->has_pending = false;
            n = 1;
        } else if (swarm_engine_next(d->engine, &rec, 1, &n) != SWARM_OK) {
            return fail(std::string("driver: ") + swarm_engine_last_error());
        }
        if (n == 0) break;  // the engine reached duration_seconds
        const bool membership = rec.kind >= SWARM_ENG_LEAVE && rec.kind != SWARM_ENG_REBALANCE;
        if (stop_kind == -2 && membership && d->completed > start) {
            // stop *before* it: its work (a stage re-created, communicators re-split) belongs to the next region
            d->pending = rec;
            d->has_pending = true;
            break;
        }
        TRY(d->on_record(rec));
        if (stop_kind >= 0 && rec.kind == stop_kind) break;
    }
    if (completed) *completed = d->completed - start;
    return SWARM_OK;
}

int swarm_driver_run(swarm_driver_t d, uint64_t n_microbatches, uint64_t* completed) {
    return swarm_driver_run_until(d, n_microbatches, -1, completed);
}

int swarm_driver_fork(swarm_driver_t d, swarm_stream_t stream) {
    if (!d) return fail("driver: null handle");
    cudaStream_t cur = static_cast<cudaStream_t>(stream);
    CU(cudaEventRecord(d->ev_tmp, cur));
    for (auto& p : d->peers)
        for (cudaStream_t s : p->lanes)
            if (s != cur) CU(cudaStreamWaitEvent(s, d->ev_tmp, 0));
    return SWARM_OK;
}

int swarm_driver_finish(swarm_driver_t d, swarm_stream_t stream) {
    if (!d) return fail("driver: null handle");
    cudaStream_t cur = static_cast<cudaStream_t>(stream);
    for (Buf& b : d->bufs) {  // outstanding transfers
        if (b.has_sent) {
            CU(cudaStreamWaitEvent(cur, b.sent, 0));
            b.has_sent = false;
        }
        if (b.has_recvd) {
            CU(cudaStreamWaitEvent(cur, b.recvd, 0));
            b.has_recvd = false;
        }
    }
    for (auto& p : d->peers)  // delayed parameter updates in flight
        if (p->upd) {
            CU(cudaEventRecord(d->ev_tmp, p->upd));
            CU(cudaStreamWaitEvent(cur, d->ev_tmp, 0));
        }
    for (cudaStream_t s : d->pair_stream)  // state downloads
        if (s) {
            CU(cudaEventRecord(d->ev_tmp, s));
            CU(cudaStreamWaitEvent(cur, d->ev_tmp, 0));
        }
    for (auto& p : d->peers)
        for (cudaStream_t s : p->lanes)
            if (s != cur) {
                CU(cudaEventRecord(d->ev_tmp, s));
                CU(cudaStreamWaitEvent(cur, d->ev_tmp, 0));
            }
    return SWARM_OK;
}

int swarm_driver_flush_wgrad(swarm_driver_t d) {
    if (!d) return fail("driver: null handle");
    for (auto& p : d->peers)
        if (p->pend >= 0 && d->serving(*p)) TRY(d->flush(*p));
    return SWARM_OK;
}

int swarm_driver_set_pool(swarm_driver_t d, const int32_t* tokens, const int32_t* targets, int n_pool, int host) {
    if (!d || n_pool < 1) return fail("driver: bad pool");
    if (host) {  // pinned host pool: every microbatch's tokens / targets cross PCIe in its consuming visit
        d->host_tok = tokens;
        d->host_tgt = targets;
        if (!tokens || !targets) d->host_tok = d->host_tgt = nullptr;
        return SWARM_OK;
    }
    if (n_pool > d->n_pool) return fail("driver: device pool larger than the driver's");
    const size_t nb = size_t(n_pool) * d->tokens * sizeof(int32_t);
    CU(cudaMemcpy(d->pool_tok, tokens, nb, cudaMemcpyDefault));
    CU(cudaMemcpy(d->pool_tgt, targets, nb, cudaMemcpyDefault));
    d->n_pool = n_pool;
    return SWARM_OK;
}

int swarm_driver_pool(swarm_driver_t d, int32_t** tokens, int32_t** targets, int* n_pool, int* tokens_per_mb) {
    if (!d) return fail("driver: null handle");
    if (tokens) *tokens = d->pool_tok;
    if (targets) *targets = d->pool_tgt;
    if (n_pool) *n_pool = d->n_pool;
    if (tokens_per_mb) *tokens_per_mb = d->tokens;
    return SWARM_OK;
}

float* swarm_driver_loss_sum(swarm_driver_t d) { return d ? d->loss_sum : nullptr; }

swarm_stage_t swarm_driver_stage(swarm_driver_t d, int peer) {
    if (!d) return nullptr;
    auto it = d->local.find(peer);
    return it == d->local.end() ? nullptr : it->second->st;
}

swarm_stream_t swarm_driver_peer_stream(swarm_driver_t d, int peer) {
    if (!d) return nullptr;
    auto it = d->local.find(peer);
    if (it == d->local.end()) return nullptr;
    Peer& p = *it->second;
    if (d->join_lanes(p) != SWARM_OK) return nullptr;
    return p.lanes[0];
}

swarm_engine_t swarm_driver_engine(swarm_driver_t d) { return d ? d->engine : nullptr; }

int swarm_driver_stats(swarm_driver_t d, swarm_driver_counters* s) {
    if (!d || !s) return fail("driver: null argument");
    s->records = d->records;
    s->visits = d->visits;
    s->ticks = d->ticks;
    s->optimizer_steps = d->optimizer_steps;
    s->completed = d->completed;
    s->captures = d->captures;
    s->kernels = swarm_launch_count() - d->captured_kernels + d->replayed_kernels;
    s->n_trainers = static_cast<uint32_t>(d->T);
    s->wire_bytes = d->wire_bytes;
    s->visit_log_size = d->log.size();
    s->recomputes = d->recomputes;
    s->migrations = d->migrations;
    s->state_bytes = d->state_bytes;
    s->n_peers = d->peer_stage.size();
    return SWARM_OK;
}

int swarm_driver_tick_time(swarm_driver_t d, double* ms, uint64_t* spans) {
    if (!d) return fail("driver: null argument");
    d->tick_resolve(true);
    if (ms) *ms = d->tick_ms;
    if (spans) *spans = d->tick_spans;
    return SWARM_OK;
}

int swarm_driver_peer_info(swarm_driver_t d, int peer, int* stage, int* alive, int* migrating, int* rank) {
    if (!d || peer < 0 || peer >= static_cast<int>(d->peer_stage.size())) return fail("driver: bad peer");
    if (stage) *stage = d->peer_stage[peer];
    if (alive) *alive = d->peer_alive[peer];
    if (migrating) *migrating = d->peer_migrating[peer];
    if (rank) *rank = d->rank_of_peer(peer);
    return SWARM_OK;
}

int swarm_driver_visit_log(swarm_driver_t d, size_t i, uint32_t* trainer, uint64_t* microbatch, uint32_t* stage,
                           int* backward, int64_t* peer) {
    if (!d || i >= d->log.size()) return fail("driver: visit log index out of range");
    const VisitLog& v = d->log[i];
    if (trainer) *trainer = v.trainer;
    if (microbatch) *microbatch = v.microbatch;
    if (stage) *stage = v.stage;
    if (backward) *backward = v.backward;
    if (peer) *peer = v.peer;
    return SWARM_OK;
}

int swarm_driver_profile_begin(swarm_driver_t d, uint64_t spin_ns) {
    if (!d) return fail("driver: null handle");
    if (d->prof) return fail("driver: profiling already on");
    if (!d->prof_stream) CU(cudaStreamCreateWithFlags(&d->prof_stream, cudaStreamNonBlocking));
    for (auto& p : d->peers) TRY(d->after_peer(d->prof_stream, *p));  // the profile stream starts after every lane
    // queue the profiled kernels behind a GPU spin so host launch gaps fall outside their events
    if (spin_ns) TRY(swarm_gpu_spin(spin_ns, d->prof_stream));
    for (auto& p : d->peers) {
        swarm_stage_profile(p->st, 1);
        swarm_stage_profile_weight(p->st, 1.0);
    }
    d->prof = true;
    return SWARM_OK;
}

int swarm_driver_profile_end(swarm_driver_t d, double* gemm_ms, double* gemm_flops, uint64_t* gemm_launches,
                             double* cat_ms, uint64_t* cat_launches) {
    if (!d || !d->prof) return fail("driver: profiling is off");
    d->prof = false;
    CU(cudaEventRecord(d->ev_tmp, d->prof_stream));
    for (auto& p : d->peers) {  // every lane continues after the profiled region
        swarm_stage_profile(p->st, 0);
        for (cudaStream_t s : p->lanes) CU(cudaStreamWaitEvent(s, d->ev_tmp, 0));
    }
    double ms = 0, fl = 0;
    uint64_t n = 0;
    double cm[SWARM_PROF_CATEGORIES] = {};
    uint64_t cn[SWARM_PROF_CATEGORIES] = {};
    for (auto& p : d->peers) {
        double a = 0, b = 0;
        uint64_t c = 0;
        TRY(swarm_stage_profile_read(p->st, &a, &b, &c));
        ms += a;
        fl += b;
        n += c;
        double pm[SWARM_PROF_CATEGORIES];
        uint64_t pn[SWARM_PROF_CATEGORIES];
        swarm_stage_profile_breakdown(p->st, pm, pn);
        for (int k = 0; k < SWARM_PROF_CATEGORIES; ++k) cm[k] += pm[k], cn[k] += pn[k];
    }
    if (gemm_ms) *gemm_ms = ms;
    if (gemm_flops) *gemm_flops = fl;
    if (gemm_launches) *gemm_launches = n;
    for (int k = 0; k < SWARM_PROF_CATEGORIES; ++k) {
        if (cat_ms) cat_ms[k] = cm[k];
        if (cat_launches) cat_launches[k] = cn[k];
    }
    d->prof_table.clear();
    for (auto& p : d->peers) d->prof_table += swarm_stage_profile_shapes(p->st);
    return SWARM_OK;
}

const char* swarm_driver_profile_shapes(swarm_driver_t d) { return d ? d->prof_table.c_str() : ""; }

int swarm_driver_peer_of_rank(swarm_driver_t d, int peer) { return d ? d->rank_of_peer(peer) : -1; }

}  // extern "C"
