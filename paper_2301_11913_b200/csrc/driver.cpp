// Host driver: the engine-driven SWARM executor in C++ (SURVEY.md §8(f)1,
// §8(b) "host code stays in C++").  The reference's discrete-event engine decides
// (csrc/engine.cpp restates P/src/sim.cpp:199-761), the GPUs execute; the driver
// attaches real work at exactly the points where the reference advances
// simulated time:
//
//   START     (Engine::start_service, sim.cpp:395-403)  the serving peer runs the
//             stage visit on its stream (CUDA-graph replay per (peer, kind,
//             trainer, paired trainer, lane));
//   HOP       (Engine::dispatch_current, sim.cpp:405-436)  the trainer's wire
//             message [int8 codes | fp32 scales | header] moves to the chosen
//             peer: across ranks both halves of the NCCL transfer are issued at
//             the consuming visit's START record (swarm_send/recv_compressed on
//             the rank pair's communicator and stream), on one GPU an event;
//   ALLREDUCE (AllReduceTick, sim.cpp:245-250, :352)  each stage's peers
//             all-reduce their fp32 gradient arena (swarm_stage_allreduce) and
//             take an AdamW step over the microbatches the stage served since the
//             last tick;
//   DONE      (record_completion, sim.cpp:512-518).
//
// swarm_driver_on_record() is the one entry point: swarm_driver_run() feeds it
// the driver's own engine, and the reference Engine can feed it the same records
// through an additive hook (tests/test_reference_hook.py).
// Every dependency points to an earlier record and every rank issues both
// halves of a transfer at the same record, so the NCCL p2p sequence of every
// rank pair matches and cannot deadlock (tests/test_executor_host.py).
#include <cuda_runtime.h>

#include <algorithm>
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
    int xfer_op = -1;  // pending cross-rank half noted at the HOP: 0 send, 1 receive
    int xfer_rank = -1;
};

struct Peer {
    int pid = 0, stage = 0;
    swarm_stage_t st = nullptr;
    std::vector<cudaStream_t> lanes;
    int rr = 0, cur = 0;  // next lane (round robin), lane of the visit being issued
    int pend = -1;        // trainer whose deferred weight gradients are pending
    std::vector<cudaEvent_t> slot_ev;
    std::vector<char> has_slot;
    cudaEvent_t lane_ev = nullptr;
    swarm_comm_t stage_comm = nullptr;
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
    int S = 0, W = 1, R = 0, T = 0, tokens = 0;
    // placement: world >= S -> peer id == rank, layout[s] peers on stage s;
    // world < S -> rank r hosts stages [r*S/W, (r+1)*S/W), one peer each (peer id == stage)
    std::vector<int> stage_of;
    int per_rank = 1;
    swarm_engine_t engine = nullptr;
    std::vector<Peer> peers;  // local peers
    std::vector<cudaStream_t> streams;  // owned (peers may share one: stream_per_peer = 0)
    std::unordered_map<int, size_t> local;  // peer id -> index into peers
    std::vector<Buf> bufs;  // (kind, trainer, boundary): act = kind 0, grad = kind 1
    size_t wire_bytes = 0;
    // synthetic token pool (device), per-trainer token / target buffers, optional pinned host pool
    int32_t *pool_tok = nullptr, *pool_tgt = nullptr;
    const int32_t *host_tok = nullptr, *host_tgt = nullptr;
    int n_pool = 0;
    std::vector<int32_t*> tok, tgt;
    float* loss_sum = nullptr;
    std::vector<void*> allocs;
    // NCCL: one communicator + stream per rank pair that exchanges messages, one per multi-peer stage
    std::vector<swarm_comm_t> pair_comm;  // indexed by peer rank (nullptr: none / self)
    std::vector<cudaStream_t> pair_stream;
    std::vector<swarm_comm_t> owned_comms;
    std::vector<int> served;  // backward visits per stage since the last tick (a global count)
    std::vector<VisitLog> log;
    std::unordered_map<uint64_t, Graph> graphs;
    std::unordered_set<uint64_t> warm;
    uint64_t records = 0, visits = 0, ticks = 0, optimizer_steps = 0, completed = 0, captures = 0;
    uint64_t captured_kernels = 0, replayed_kernels = 0;
    cudaEvent_t ev_tmp = nullptr;
    // profiled region: every visit eager (no graph) on one stream with the stages' kernel
    // profiling on, so the events around each kernel time it alone (the live roofline)
    bool prof = false;
    cudaStream_t prof_stream = nullptr;

    cudaStream_t lane_stream(const Peer& p) const { return prof ? prof_stream : p.lanes[p.cur]; }

    int rank_of_peer(int pid) const { return W >= S ? pid : stage_of[pid] / per_rank; }

    Buf* buf_for(int t, int stage, bool backward) {  // the wire message the visit (t, stage, backward) reads
        if (backward) return stage == S - 1 ? nullptr : &bufs[(size_t(1) * T + t) * (S - 1) + stage];
        return stage == 0 ? nullptr : &bufs[(size_t(0) * T + t) * (S - 1) + stage - 1];
    }
    Buf* out_for(int t, int stage, bool backward) {  // the message it writes
        if (backward) return stage == 0 ? nullptr : &bufs[(size_t(1) * T + t) * (S - 1) + stage - 1];
        return stage == S - 1 ? nullptr : &bufs[(size_t(0) * T + t) * (S - 1) + stage];
    }

    int dalloc(void** p, size_t bytes) {
        CU(cudaMalloc(p, std::max<size_t>(bytes, 16)));
        allocs.push_back(*p);
        return cudaMemset(*p, 0, bytes) == cudaSuccess ? SWARM_OK : fail("driver: memset failed", SWARM_E_CUDA);
    }

    // ------------------------------------------------------------- graphs
    static uint64_t gkey(int pid, int kind, int t, int p, int lane) {
        return (uint64_t(pid) << 48) | (uint64_t(kind) << 44) | (uint64_t(t & 0xFFFF) << 28) |
               (uint64_t((p + 1) & 0xFFFF) << 12) | uint64_t(lane & 0xFFF);
    }

    int replay(uint64_t key, cudaStream_t st, const std::function<int()>& fn) {
        if (!cfg.use_graphs || !warm.count(key) || prof) {  // first use runs eagerly (lazy init, tensor-map caches)
            TRY(fn());
            if (!prof) warm.insert(key);
            return SWARM_OK;
        }
        auto it = graphs.find(key);
        if (it == graphs.end()) {
            const uint64_t n0 = swarm_launch_count();
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
            gr.kernels = swarm_launch_count() - n0;
            captures += 1;
            captured_kernels += gr.kernels;
            it = graphs.emplace(key, gr).first;
        }
        CU(cudaGraphLaunch(it->second.exec, st));
        replayed_kernels += it->second.kernels;
        return SWARM_OK;
    }

    // ------------------------------------------------------------- helpers
    int wait(cudaStream_t st, cudaEvent_t ev) { return cuda(cudaStreamWaitEvent(st, ev, 0), "cudaStreamWaitEvent"); }
    int mark(cudaEvent_t ev, cudaStream_t st) { return cuda(cudaEventRecord(ev, st), "cudaEventRecord"); }

    int after_slot(Peer& p, int t) {
        if (!p.has_slot[t]) return SWARM_OK;
        return wait(lane_stream(p), p.slot_ev[t]);
    }
    int mark_slot(Peer& p, int t) {
        p.has_slot[t] = 1;
        return mark(p.slot_ev[t], lane_stream(p));
    }

    int pool_index(int t, uint64_t k) const { return static_cast<int>((uint64_t(t) * 7 + k) % uint64_t(n_pool)); }

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

    int visit(Peer& p, const swarm_engine_record& r, int s, int t, bool bwd, int* paired) {
        *paired = -1;
        cudaStream_t st = lane_stream(p);
        Buf* in = buf_for(t, s, bwd);
        Buf* out = out_for(t, s, bwd);
        if (in && in->has_recvd) {  // the transfer into this buffer (pair stream)
            TRY(wait(st, in->recvd));
            in->has_recvd = false;
        }
        if (in && in->has_done) {  // produced by a peer on this GPU (another stream)
            TRY(wait(st, in->done));
            in->has_done = false;
        }
        if (out && out->has_sent) {  // the previous message from this buffer has left
            TRY(wait(st, out->sent));
            out->has_sent = false;
        }
        if (out && out->has_read) {  // its previous local reader is done
            TRY(wait(st, out->read));
            out->has_read = false;
        }
        if (!bwd && p.pend == t) TRY(flush(p));  // this forward reuses the slot the pending weight gradients read
        if (!bwd) {
            const int i = pool_index(t, r.microbatch);
            const int32_t* src_tok = host_tok ? host_tok : pool_tok;
            const int32_t* src_tgt = host_tgt ? host_tgt : pool_tgt;
            const cudaMemcpyKind kind = host_tok ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
            const size_t nb = size_t(tokens) * sizeof(int32_t);
            if (s == 0) CU(cudaMemcpyAsync(tok[t], src_tok + size_t(i) * tokens, nb, kind, st));
            if (s == S - 1) CU(cudaMemcpyAsync(tgt[t], src_tgt + size_t(i) * tokens, nb, kind, st));
            const void* inp = s == 0 ? static_cast<const void*>(tok[t]) : in->p;
            void* o = out ? out->p : nullptr;
            const int32_t* tg = s == S - 1 ? tgt[t] : nullptr;
            const float scale = 1.0f / static_cast<float>(tokens);
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

    int transfer(Buf& b) {
        const int op = b.xfer_op, peer = b.xfer_rank;
        b.xfer_op = -1;
        cudaStream_t ps = pair_stream[peer];
        swarm_comm_t c = pair_comm[peer];
        if (!c) return fail("driver: no communicator to rank " + std::to_string(peer));
        const int other = R < peer ? 1 : 0;  // ranks of a pair communicator are ordered by world rank
        if (op == 0) {
            if (b.has_done) {
                TRY(wait(ps, b.done));  // the producing visit (on its peer's stream)
                b.has_done = false;
            }
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
        if (bwd) served[s] += 1;
        log.push_back(VisitLog{r.trainer, r.stage, r.microbatch, r.backward, r.worker});
        Buf* in = buf_for(t, s, bwd);
        if (in && in->xfer_op >= 0) TRY(transfer(*in));  // both ranks of a cross-rank hop, at the same record
        auto it = local.find(pid);
        if (it == local.end()) return SWARM_OK;
        Peer& p = peers[it->second];
        p.cur = p.rr;
        p.rr = (p.rr + 1) % cfg.lanes;
        if (cfg.lanes > 1) {
            TRY(swarm_stage_set_lane(p.st, p.cur));
            TRY(after_slot(p, t));  // this slot's previous visit (e.g. the last stage's forward)
        }
        int paired = -1;
        TRY(visit(p, r, s, t, bwd, &paired));
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
        const int64_t src = r.from_worker, dst = r.worker;
        if (src < 0 || src == dst) return SWARM_OK;
        const int rs = rank_of_peer(static_cast<int>(src)), rd = rank_of_peer(static_cast<int>(dst));
        if (rs == rd || (rs != R && rd != R)) return SWARM_OK;
        Buf* b = buf_for(static_cast<int>(r.trainer), static_cast<int>(r.stage), r.backward != 0);
        if (!b) return SWARM_OK;
        b->xfer_op = rs == R ? 0 : 1;
        b->xfer_rank = rs == R ? rd : rs;
        return SWARM_OK;
    }

    int join_lanes(Peer& p) {  // lane 0 waits for every other lane
        p.cur = 0;
        if (prof) return SWARM_OK;  // one stream while profiling
        for (size_t i = 1; i < p.lanes.size(); ++i) {
            TRY(mark(p.lane_ev, p.lanes[i]));
            TRY(wait(p.lanes[0], p.lane_ev));
        }
        p.cur = 0;
        return SWARM_OK;
    }

    int on_allreduce() {
        ticks += 1;
        for (Peer& p : peers) TRY(join_lanes(p));  // the tick follows every visit on every lane
        for (Peer& p : peers)
            if (p.pend >= 0) TRY(flush(p));
        for (Peer& p : peers) {
            const int n = served[p.stage];
            if (n == 0) continue;
            cudaStream_t st = lane_stream(p);
            TRY(swarm_stage_allreduce(p.st, p.stage_comm, st));
            TRY(swarm_stage_optimizer_step(p.st, 1.0f / static_cast<float>(n), st));  // mean over the stage's microbatches
            optimizer_steps += 1;
        }
        for (Peer& p : peers) {  // every lane's next visit sees the updated weights
            if (prof) break;
            TRY(mark(p.lane_ev, p.lanes[0]));
            for (size_t i = 1; i < p.lanes.size(); ++i) TRY(wait(p.lanes[i], p.lane_ev));
        }
        std::fill(served.begin(), served.end(), 0);
        return SWARM_OK;
    }

    int on_record(const swarm_engine_record& r) {
        records += 1;
        switch (r.kind) {
            case SWARM_ENG_START: return on_start(r);
            case SWARM_ENG_HOP: return on_hop(r);
            case SWARM_ENG_ALLREDUCE: return on_allreduce();
            case SWARM_ENG_DONE: completed += 1; return SWARM_OK;
        }
        return fail("driver: unknown record kind");
    }

    ~swarm_driver() {
        cudaDeviceSynchronize();
        for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.exec);
        for (Peer& p : peers) {
            for (cudaEvent_t e : p.slot_ev) cudaEventDestroy(e);
            if (p.lane_ev) cudaEventDestroy(p.lane_ev);
            if (p.st) swarm_stage_destroy(p.st);
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

    int create() {
        const swarm_driver_config& c = cfg;
        S = c.n_stages;
        W = c.world;
        R = c.rank;
        if (S < 1 || W < 1 || R < 0 || R >= W) return fail("driver: bad stage count / world / rank");
        if (c.lanes < 1) return fail("driver: lanes must be >= 1");
        if (c.n_pool < 1) return fail("driver: n_pool must be >= 1");
        if (W > 1 && !c.comm) return fail("driver: world > 1 needs a world communicator");
        // placement
        std::vector<int> layout(S, 1);
        if (W >= S) {
            if (c.layout) {
                int sum = 0;
                for (int s = 0; s < S; ++s) {
                    layout[s] = c.layout[s];
                    if (layout[s] < 1) return fail("driver: every stage needs a peer");
                    sum += layout[s];
                }
                if (sum != W) return fail("driver: layout must sum to the world size");
            } else {
                if (W % S) return fail("driver: world must be a multiple of the stage count");
                std::fill(layout.begin(), layout.end(), W / S);
            }
            for (int s = 0; s < S; ++s)
                for (int k = 0; k < layout[s]; ++k) stage_of.push_back(s);
        } else {
            if (S % W) return fail("driver: stage count must be a multiple of world");
            per_rank = S / W;
            for (int s = 0; s < S; ++s) stage_of.push_back(s);
        }
        // engine: SimConfig initial_peers = layout, speeds 1
        std::vector<size_t> wst(stage_of.begin(), stage_of.end());
        TRY(swarm_engine_create(S, wst.size(), wst.data(), nullptr, c.forward_seconds, c.backward_multiplier,
                                c.trainers_per_peer, c.allreduce_period, c.allreduce_stall, c.duration_seconds,
                                std::max(c.duration_seconds / 64, 1e-9), c.seed, &engine) == SWARM_OK
                ? SWARM_OK
                : fail(std::string("driver: ") + swarm_engine_last_error()));
        T = static_cast<int>(swarm_engine_n_trainers(engine));
        served.assign(S, 0);
        const swarm_stage_config& m = c.model;
        tokens = m.seq_len * m.micro_batch;
        // local peers and their stages (replicas of a stage start identical: seed * 1000 + stage)
        for (int pid = 0; pid < static_cast<int>(stage_of.size()); ++pid) {
            if (rank_of_peer(pid) != R) continue;
            Peer p;
            p.pid = pid;
            p.stage = stage_of[pid];
            swarm_stage_config sc = m;
            sc.is_first = p.stage == 0;
            sc.is_last = p.stage == S - 1;
            sc.max_slots = T;
            sc.seed = c.seed * 1000 + p.stage;
            if (swarm_stage_create(&sc, &p.st) != SWARM_OK) return fail(std::string("driver: ") + swarm_last_error());
            if (c.pair_wgrad && swarm_stage_enable_wgrad_pairing_sets(p.st, std::max(2, T)) != SWARM_OK)
                return fail(std::string("driver: ") + swarm_last_error());
            if (c.lanes > 1 && swarm_stage_enable_lanes(p.st, c.lanes) != SWARM_OK)
                return fail(std::string("driver: ") + swarm_last_error());
            if (!c.stream_per_peer && c.lanes > 1) return fail("driver: lanes need a stream per peer");
            for (int l = 0; l < c.lanes; ++l) {
                if (!c.stream_per_peer && !streams.empty()) {  // one stream per GPU, shared by its peers
                    p.lanes.push_back(streams[0]);
                    continue;
                }
                cudaStream_t s = nullptr;
                CU(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
                streams.push_back(s);
                p.lanes.push_back(s);
            }
            p.slot_ev.resize(T);
            p.has_slot.assign(T, 0);
            for (auto& e : p.slot_ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&p.lane_ev, cudaEventDisableTiming));
            local[pid] = peers.size();
            peers.push_back(std::move(p));
        }
        // wire messages: size from the model (every stage's wire has the same size)
        {
            swarm_stage_t probe = peers.empty() ? nullptr : peers[0].st;
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
        bufs.resize(size_t(2) * T * std::max(S - 1, 0));
        for (Buf& b : bufs) {
            TRY(dalloc(&b.p, wire_bytes));
            for (cudaEvent_t* e : {&b.done, &b.read, &b.sent, &b.recvd})
                CU(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        }
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
        tok.resize(T);
        tgt.resize(T);
        for (int t = 0; t < T; ++t) {
            TRY(dalloc(reinterpret_cast<void**>(&tok[t]), size_t(tokens) * 4));
            TRY(dalloc(reinterpret_cast<void**>(&tgt[t]), size_t(tokens) * 4));
        }
        TRY(dalloc(reinterpret_cast<void**>(&loss_sum), sizeof(float)));
        CU(cudaEventCreateWithFlags(&ev_tmp, cudaEventDisableTiming));
        // communicators (collective over the world: every rank makes the same calls in the same order)
        pair_comm.assign(W, nullptr);
        pair_stream.assign(W, nullptr);
        if (W > 1) {
            // one communicator per rank pair, W - 1 (or W) rounds of a round-robin pairing, each a
            // split of the world; plus one per multi-peer stage
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
                swarm_comm_t pc = nullptr;
                if (swarm_comm_split(c.comm, color, R, &pc) != SWARM_OK)
                    return fail(std::string("driver: ") + swarm_comm_last_error());
                if (pc) {
                    owned_comms.push_back(pc);
                    pair_comm[partner] = pc;
                    CU(cudaStreamCreateWithFlags(&pair_stream[partner], cudaStreamNonBlocking));
                }
            }
            if (W >= S) {
                const int color = layout[stage_of[R]] > 1 ? stage_of[R] : -1;
                swarm_comm_t sc = nullptr;
                if (swarm_comm_split(c.comm, color, R, &sc) != SWARM_OK)
                    return fail(std::string("driver: ") + swarm_comm_last_error());
                if (sc) {
                    owned_comms.push_back(sc);
                    for (Peer& p : peers) p.stage_comm = sc;
                }
            }
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
    const int rc = d->create();
    if (rc != SWARM_OK) return rc;
    *out = d.release();
    return SWARM_OK;
}

void swarm_driver_destroy(swarm_driver_t d) { delete d; }

int swarm_driver_on_record(swarm_driver_t d, const swarm_engine_record* r) {
    if (!d || !r) return fail("driver: null argument");
    return d->on_record(*r);
}

int swarm_driver_run(swarm_driver_t d, uint64_t n_microbatches, uint64_t* completed) {
    if (!d) return fail("driver: null handle");
    const uint64_t target = d->completed + n_microbatches, start = d->completed;
    swarm_engine_record recs[64];
    while (d->completed < target) {
        size_t n = 0;
        if (swarm_engine_next(d->engine, recs, 1, &n) != SWARM_OK)
            return fail(std::string("driver: ") + swarm_engine_last_error());
        if (n == 0) break;  // the engine reached duration_seconds
        TRY(d->on_record(recs[0]));
    }
    if (completed) *completed = d->completed - start;
    return SWARM_OK;
}

int swarm_driver_fork(swarm_driver_t d, swarm_stream_t stream) {
    if (!d) return fail("driver: null handle");
    cudaStream_t cur = static_cast<cudaStream_t>(stream);
    CU(cudaEventRecord(d->ev_tmp, cur));
    for (Peer& p : d->peers)
        for (cudaStream_t s : p.lanes)
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
    for (Peer& p : d->peers)
        for (cudaStream_t s : p.lanes)
            if (s != cur) {
                CU(cudaEventRecord(d->ev_tmp, s));
                CU(cudaStreamWaitEvent(cur, d->ev_tmp, 0));
            }
    return SWARM_OK;
}

int swarm_driver_flush_wgrad(swarm_driver_t d) {
    if (!d) return fail("driver: null handle");
    for (Peer& p : d->peers)
        if (p.pend >= 0) TRY(d->flush(p));
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
    return it == d->local.end() ? nullptr : d->peers[it->second].st;
}

swarm_stream_t swarm_driver_peer_stream(swarm_driver_t d, int peer) {
    if (!d) return nullptr;
    auto it = d->local.find(peer);
    if (it == d->local.end()) return nullptr;
    Peer& p = d->peers[it->second];
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
    for (Peer& p : d->peers)  // the profile stream starts after every lane
        for (cudaStream_t s : p.lanes) {
            CU(cudaEventRecord(d->ev_tmp, s));
            CU(cudaStreamWaitEvent(d->prof_stream, d->ev_tmp, 0));
        }
    // queue the profiled kernels behind a GPU spin so host launch gaps fall outside their events
    if (spin_ns) TRY(swarm_gpu_spin(spin_ns, d->prof_stream));
    for (Peer& p : d->peers) {
        swarm_stage_profile(p.st, 1);
        swarm_stage_profile_weight(p.st, 1.0);
    }
    d->prof = true;
    return SWARM_OK;
}

int swarm_driver_profile_end(swarm_driver_t d, double* gemm_ms, double* gemm_flops, uint64_t* gemm_launches,
                             double* cat_ms, uint64_t* cat_launches) {
    if (!d || !d->prof) return fail("driver: profiling is off");
    d->prof = false;
    for (Peer& p : d->peers) {  // every lane continues after the profiled region
        swarm_stage_profile(p.st, 0);
        CU(cudaEventRecord(d->ev_tmp, d->prof_stream));
        for (cudaStream_t s : p.lanes) CU(cudaStreamWaitEvent(s, d->ev_tmp, 0));
    }
    double ms = 0, fl = 0;
    uint64_t n = 0;
    double cm[SWARM_PROF_CATEGORIES] = {};
    uint64_t cn[SWARM_PROF_CATEGORIES] = {};
    for (Peer& p : d->peers) {
        double a = 0, b = 0;
        uint64_t c = 0;
        TRY(swarm_stage_profile_read(p.st, &a, &b, &c));
        ms += a;
        fl += b;
        n += c;
        double pm[SWARM_PROF_CATEGORIES];
        uint64_t pn[SWARM_PROF_CATEGORIES];
        swarm_stage_profile_breakdown(p.st, pm, pn);
        for (int k = 0; k < SWARM_PROF_CATEGORIES; ++k) cm[k] += pm[k], cn[k] += pn[k];
    }
    if (gemm_ms) *gemm_ms = ms;
    if (gemm_flops) *gemm_flops = fl;
    if (gemm_launches) *gemm_launches = n;
    for (int k = 0; k < SWARM_PROF_CATEGORIES; ++k) {
        if (cat_ms) cat_ms[k] = cm[k];
        if (cat_launches) cat_launches[k] = cn[k];
    }
    return SWARM_OK;
}

int swarm_driver_peer_of_rank(swarm_driver_t d, int peer) {
    return d ? d->rank_of_peer(peer) : -1;
}

}  // extern "C"
