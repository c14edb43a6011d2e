// C++ test binary: the tiny SWARM pipeline (BASELINE configs[0] shapes) driven
// entirely through the C-ABI (include/swarm_b200.h) with no Python: the host
// driver walks the engine's records, runs the visits, moves the wire messages
// (NCCL across ranks) and all-reduces.  It writes the token pool, the visit log,
// every local stage's gradient arena and the loss to --out, which
// tests/test_driver_cpp_gpu.py compares with the Python orchestrator
// (PyEngineExecutor) and with a sequential replay.
//
//   driver_test --out FILE [--stages S] [--tpp K] [--microbatches N] [--lanes L]
//               [--world W --rank R --id FILE]   (one process per GPU)
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "swarm_b200.h"

static int die(const char* what, const char* msg) {
    fprintf(stderr, "driver_test: %s: %s\n", what, msg);
    return 1;
}

int main(int argc, char** argv) {
    int S = 2, tpp = 2, N = 9, lanes = 1, world = 1, rank = 0, ticks = 0;
    std::string out, idfile;
    for (int i = 1; i + 1 < argc; i += 2) {
        const std::string k = argv[i];
        const char* v = argv[i + 1];
        if (k == "--stages") S = atoi(v);
        else if (k == "--tpp") tpp = atoi(v);
        else if (k == "--microbatches") N = atoi(v);
        else if (k == "--lanes") lanes = atoi(v);
        else if (k == "--world") world = atoi(v);
        else if (k == "--rank") rank = atoi(v);
        else if (k == "--id") idfile = v;
        else if (k == "--out") out = v;
        else if (k == "--ticks") ticks = atoi(v);
        else return die("args", ("unknown flag " + k).c_str());
    }
    if (out.empty()) return die("args", "--out is required");
    int ndev = 0;
    cudaGetDeviceCount(&ndev);
    if (ndev < 1) return die("cuda", "no device");
    cudaSetDevice(world > 1 ? rank % ndev : 0);
    swarm_comm_t comm = nullptr;
    if (world > 1) {  // rank 0 publishes the NCCL unique id through a file
        unsigned char id[128];
        if (rank == 0) {
            if (swarm_comm_unique_id(id) != SWARM_OK) return die("unique_id", swarm_comm_last_error());
            const std::string tmp = idfile + ".tmp";
            FILE* f = fopen(tmp.c_str(), "wb");
            fwrite(id, 1, 128, f);
            fclose(f);
            rename(tmp.c_str(), idfile.c_str());
        } else {
            FILE* f = nullptr;
            for (int i = 0; i < 6000 && !(f = fopen(idfile.c_str(), "rb")); ++i)
                std::this_thread::sleep_for(std::chrono::milliseconds(10));
            if (!f || fread(id, 1, 128, f) != 128) return die("unique_id", "no id file");
            fclose(f);
        }
        if (swarm_comm_create(id, world, rank, &comm) != SWARM_OK) return die("comm_create", swarm_comm_last_error());
    }
    swarm_driver_config c{};
    swarm_stage_config& m = c.model;  // BASELINE configs[0] shapes: d 256, 4 heads, seq 128, batch 8
    m.d_model = 256;
    m.n_heads = 4;
    m.d_ffn = 1024;
    m.seq_len = 128;
    m.micro_batch = 8;
    m.n_layers = 2;
    m.vocab = 512;
    m.causal = 1;
    m.wire = SWARM_WIRE_INT8;
    m.block_size = 4096;
    m.lr = 1e-3f;
    m.beta1 = 0.9f;
    m.beta2 = 0.95f;
    m.eps = 1e-8f;
    m.init_std = 0.02f;
    c.n_stages = S;
    c.world = world;
    c.rank = rank;
    c.forward_seconds = 1.0;
    c.backward_multiplier = 2.0;
    c.allreduce_period = ticks ? 10.0 : 0.0;
    c.allreduce_stall = ticks ? 0.1 : 0.0;
    c.duration_seconds = 1e9;
    c.trainers_per_peer = tpp;
    c.seed = 11;
    c.lanes = lanes;
    c.pair_wgrad = 1;
    c.use_graphs = 1;
    c.stream_per_peer = 1;
    c.n_pool = 4;
    c.comm = comm;
    swarm_driver_t d = nullptr;
    if (swarm_driver_create(&c, &d) != SWARM_OK) return die("driver_create", swarm_driver_last_error());
    uint64_t done = 0;
    if (swarm_driver_run(d, N, &done) != SWARM_OK) return die("driver_run", swarm_driver_last_error());
    if (swarm_driver_flush_wgrad(d) != SWARM_OK || swarm_driver_finish(d, nullptr) != SWARM_OK)
        return die("driver_finish", swarm_driver_last_error());
    if (cudaDeviceSynchronize() != cudaSuccess) return die("cuda", cudaGetErrorString(cudaGetLastError()));
    swarm_driver_counters k{};
    swarm_driver_stats(d, &k);
    int32_t *ptok = nullptr, *ptgt = nullptr;
    int npool = 0, ntok = 0;
    swarm_driver_pool(d, &ptok, &ptgt, &npool, &ntok);
    std::vector<int32_t> htok(size_t(npool) * ntok), htgt(htok.size());
    cudaMemcpy(htok.data(), ptok, htok.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(htgt.data(), ptgt, htgt.size() * 4, cudaMemcpyDeviceToHost);
    float loss = 0.f;
    cudaMemcpy(&loss, swarm_driver_loss_sum(d), 4, cudaMemcpyDeviceToHost);
    FILE* f = fopen(out.c_str(), "wb");
    if (!f) return die("out", "cannot open");
    const int64_t hdr[6] = {S, static_cast<int64_t>(k.n_trainers), npool, ntok, static_cast<int64_t>(done),
                            static_cast<int64_t>(k.visit_log_size)};
    fwrite(hdr, 8, 6, f);
    fwrite(htok.data(), 4, htok.size(), f);
    fwrite(htgt.data(), 4, htgt.size(), f);
    fwrite(&loss, 4, 1, f);
    for (size_t i = 0; i < k.visit_log_size; ++i) {
        uint32_t t = 0, s = 0;
        uint64_t mb = 0;
        int b = 0;
        int64_t p = 0;
        swarm_driver_visit_log(d, i, &t, &mb, &s, &b, &p);
        const int64_t rec[5] = {t, static_cast<int64_t>(mb), s, b, p};
        fwrite(rec, 8, 5, f);
    }
    const int n_peers = world >= S ? world : S;
    for (int pid = 0; pid < n_peers; ++pid) {
        swarm_stage_t st = swarm_driver_stage(d, pid);
        if (!st) continue;
        const int64_t np = static_cast<int64_t>(swarm_stage_num_params(st));
        std::vector<float> g(np), pm(np);
        cudaMemcpy(g.data(), swarm_stage_grads(st), np * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(pm.data(), swarm_stage_params(st), np * 4, cudaMemcpyDeviceToHost);
        const int64_t ph[2] = {pid, np};
        fwrite(ph, 8, 2, f);
        fwrite(g.data(), 4, np, f);
        fwrite(pm.data(), 4, np, f);
    }
    fclose(f);
    printf("driver_test rank %d: %llu microbatches, %llu visits, %llu records, %llu graph captures, %llu optimizer steps\n",
           rank, (unsigned long long)done, (unsigned long long)k.visits, (unsigned long long)k.records,
           (unsigned long long)k.captures, (unsigned long long)k.optimizer_steps);
    swarm_driver_destroy(d);
    if (comm) swarm_comm_destroy(comm);
    return 0;
}
