// NCCL transport behind the C-ABI: the stage-to-stage hop of a compressed wire
// message (the reference's dispatch_current moves a trainer to the next peer's
// queue, P/src/sim.cpp:405-436; the time model is cost_model.cpp:55-59) and the
// intra-stage gradient all-reduce (the AllReduceTick stall, sim.cpp:245-250,
// :352).  Raw NCCL, resolved at run time with dlopen so the library has no
// link-time NCCL dependency and shares the process's NCCL when torch already
// loaded one (libnccl.so.2; SWARM_NCCL_LIB overrides the path).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "swarm_b200.h"

struct swarm_comm {
    ncclComm_t c = nullptr;
    int nranks = 0, rank = 0;
};

namespace {

thread_local std::string g_err;

struct Nccl {
    bool ok = false;
    std::string why;
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) init_rank = nullptr;
    decltype(&ncclCommSplit) split = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclCommAbort) abort = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    decltype(&ncclGetVersion) version = nullptr;
    decltype(&ncclCommCount) count = nullptr;
    decltype(&ncclCommUserRank) user_rank = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL (torch's) if loaded
        const char* env = getenv("SWARM_NCCL_LIB");
        if (!h && env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2",
                           RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            n.why = std::string("NCCL not found: ") + dlerror();
            return;
        }
        bool all = true;
        auto sym = [&](auto& fp, const char* name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            if (!fp) all = false;
        };
        sym(n.get_unique_id, "ncclGetUniqueId");
        sym(n.init_rank, "ncclCommInitRank");
        sym(n.split, "ncclCommSplit");
        sym(n.destroy, "ncclCommDestroy");
        sym(n.abort, "ncclCommAbort");
        sym(n.send, "ncclSend");
        sym(n.recv, "ncclRecv");
        sym(n.all_reduce, "ncclAllReduce");
        sym(n.group_start, "ncclGroupStart");
        sym(n.group_end, "ncclGroupEnd");
        sym(n.error_string, "ncclGetErrorString");
        sym(n.version, "ncclGetVersion");
        sym(n.count, "ncclCommCount");
        sym(n.user_rank, "ncclCommUserRank");
        n.ok = all;
        if (!all) n.why = "NCCL library lacks a required symbol";
    });
    return n;
}

int fail(const std::string& m, int rc = SWARM_E_INVALID) {
    g_err = m;
    return rc;
}

int nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return SWARM_OK;
    return fail(std::string(what) + ": " + nccl().error_string(r), SWARM_E_CUDA);
}

#define NEED_NCCL()                                                              \
    do {                                                                         \
        if (!nccl().ok) return fail("NCCL unavailable: " + nccl().why, SWARM_E_UNSUPPORTED); \
    } while (0)

}  // namespace

extern "C" {

const char* swarm_comm_last_error(void) { return g_err.c_str(); }

int swarm_comm_nccl_version(void) {
    int v = 0;
    if (nccl().ok) nccl().version(&v);
    return v;
}

int swarm_comm_unique_id(void* id) {
    NEED_NCCL();
    if (!id) return fail("comm: null id buffer");
    return nccl_check(nccl().get_unique_id(static_cast<ncclUniqueId*>(id)), "ncclGetUniqueId");
}

int swarm_comm_create(const void* id, int nranks, int rank, swarm_comm_t* out) {
    NEED_NCCL();
    if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail("comm_create: bad arguments");
    ncclUniqueId u;
    memcpy(&u, id, sizeof(u));
    auto* c = new swarm_comm;
    const int rc = nccl_check(nccl().init_rank(&c->c, nranks, u, rank), "ncclCommInitRank");
    if (rc != SWARM_OK) {
        delete c;
        return rc;
    }
    c->nranks = nranks;
    c->rank = rank;
    *out = c;
    return SWARM_OK;
}

int swarm_comm_split_ex(swarm_comm_t parent, int color, int key, int max_ctas, swarm_comm_t* out) {
    NEED_NCCL();
    if (!parent || !out) return fail("comm_split: null argument");
    *out = nullptr;
    ncclComm_t nc = nullptr;
    {
        ncclConfig_t config = NCCL_CONFIG_INITIALIZER;
        if (max_ctas > 0) config.maxCTAs = max_ctas;
        const int rc = nccl_check(nccl().split(parent->c, color < 0 ? NCCL_SPLIT_NOCOLOR : color, key, &nc,
                                               max_ctas > 0 ? &config : nullptr),
                                  "ncclCommSplit");
        if (rc != SWARM_OK) return rc;
    }
    if (!nc) return SWARM_OK;  // this rank is in no group
    auto* c = new swarm_comm;
    c->c = nc;
    // the new communicator's size / rank: ranks of one color ordered by key
    int n = 0, r = 0;
    nccl().count(nc, &n);
    nccl().user_rank(nc, &r);
    c->nranks = n;
    c->rank = r;
    *out = c;
    return SWARM_OK;
}

int swarm_comm_split(swarm_comm_t parent, int color, int key, swarm_comm_t* out) {
    return swarm_comm_split_ex(parent, color, key, 0, out);
}

void swarm_comm_destroy(swarm_comm_t c) {
    if (!c) return;
    if (nccl().ok && c->c) nccl().destroy(c->c);
    delete c;
}

int swarm_comm_size(swarm_comm_t c, int* nranks, int* rank) {
    if (!c) return fail("comm: null handle");
    if (nranks) *nranks = c->nranks;
    if (rank) *rank = c->rank;
    return SWARM_OK;
}

int swarm_send_compressed(swarm_comm_t c, const void* msg, size_t bytes, int peer, swarm_stream_t stream) {
    NEED_NCCL();
    if (!c || !msg || peer < 0 || peer >= c->nranks || peer == c->rank) return fail("send_compressed: bad arguments");
    return nccl_check(nccl().send(msg, bytes, ncclUint8, peer, c->c, static_cast<cudaStream_t>(stream)), "ncclSend");
}

int swarm_recv_compressed(swarm_comm_t c, void* msg, size_t bytes, int peer, swarm_stream_t stream) {
    NEED_NCCL();
    if (!c || !msg || peer < 0 || peer >= c->nranks || peer == c->rank) return fail("recv_compressed: bad arguments");
    return nccl_check(nccl().recv(msg, bytes, ncclUint8, peer, c->c, static_cast<cudaStream_t>(stream)), "ncclRecv");
}

int swarm_allreduce_sum(swarm_comm_t c, void* buf, size_t count, int dtype, swarm_stream_t stream) {
    NEED_NCCL();
    if (!c || !buf) return fail("allreduce: bad arguments");
    ncclDataType_t t = ncclFloat32;
    if (dtype == SWARM_DTYPE_BF16) t = ncclBfloat16;
    else if (dtype != SWARM_DTYPE_F32) return fail("allreduce: dtype must be f32 or bf16");
    return nccl_check(nccl().all_reduce(buf, buf, count, t, ncclSum, c->c, static_cast<cudaStream_t>(stream)),
                      "ncclAllReduce");
}

int swarm_stage_allreduce(swarm_stage_t st, swarm_comm_t stage_comm, swarm_stream_t stream) {
    if (!st) return fail("stage_allreduce: null stage");
    if (!stage_comm || stage_comm->nranks <= 1) return SWARM_OK;  // a stage with one peer has nothing to average
    return swarm_allreduce_sum(stage_comm, swarm_stage_grads(st), swarm_stage_num_params(st), SWARM_DTYPE_F32, stream);
}

int swarm_comm_group_start(void) {
    NEED_NCCL();
    return nccl_check(nccl().group_start(), "ncclGroupStart");
}

int swarm_comm_group_end(void) {
    NEED_NCCL();
    return nccl_check(nccl().group_end(), "ncclGroupEnd");
}

}  // extern "C"
