// po_main.cpp — pairwise optimisation (engine.hpp:377-411) driven from C++
// through include/mdg.h alone: no Python, no PyTorch.  One process per GPU:
// the batch of pairs is sharded round-robin (pair i on rank i mod world, the
// reference's cli.cpp:231 loop split), and only the per-pair results are
// gathered — over NCCL (all-gather of a fixed-size result record) or through
// files for ranks sharing a device.  Config 5 of BASELINE.json.
//
//   po_main [h w l] [--iters N] [--lr X] [--seed S] [--pairs P] [--synth]
//           [--large] [--diffeomorphic] [--sgd] [--eager] [--quiet]
//           [--rank R --world W --device D] [--gather nccl|file] [--rendezvous DIR]
//
// rank / world / device default to RANK / WORLD_SIZE / LOCAL_RANK from the
// environment (torchrun-style launchers), else 0 / 1 / 0.
// --synth: pair p is make_synth_pair(dims, seed p + 1, max_disp 2.0)
// (synth.cpp:92-192, native) and reports Dice (metrics.cpp:124-167); without
// it every pair is the U(0,1) volumes of Rng(11) (bench.py's PO workload).
// Per pair: init_model(cfg, seed) on the host (the reference Rng stream),
// N updates (loss read back and checked finite each iteration, as the
// reference loop does) and the final evaluation forward.
#include <cuda_runtime.h>
#include <nccl.h>
#include <unistd.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "mdg.h"

#define CK(x)                                                                    \
    do {                                                                         \
        cudaError_t e_ = (x);                                                    \
        if (e_ != cudaSuccess) {                                                 \
            std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));        \
            std::exit(1);                                                        \
        }                                                                        \
    } while (0)
#define MK(x)                                                                    \
    do {                                                                         \
        if ((x) != MDG_OK) {                                                     \
            std::fprintf(stderr, "%s: %s\n", #x, mdg_last_error());              \
            std::exit(1);                                                        \
        }                                                                        \
    } while (0)
#define NK(x)                                                                    \
    do {                                                                         \
        ncclResult_t r_ = (x);                                                   \
        if (r_ != ncclSuccess) {                                                 \
            std::fprintf(stderr, "%s: %s\n", #x, ncclGetErrorString(r_));        \
            std::exit(1);                                                        \
        }                                                                        \
    } while (0)

namespace {
// the per-pair result gathered from every rank (fixed size for the all-gather)
struct PairResult {
    double pair = -1, rank = -1, loss0 = 0, loss_final = 0, dice0 = 0, dice_final = 0,
           iter_ms = 0, wall_s = 0;
};

int env_int(const char *k, int dflt) {
    const char *v = std::getenv(k);
    return v ? std::atoi(v) : dflt;
}

// file rendezvous for the NCCL unique id (rank 0 writes, the others poll)
ncclUniqueId nccl_id(const std::string &dir, int rank) {
    ncclUniqueId id;
    const std::string path = dir + "/po_main_nccl.id";
    if (rank == 0) {
        NK(ncclGetUniqueId(&id));
        const std::string tmp = path + ".tmp";
        std::ofstream(tmp, std::ios::binary).write(id.internal, sizeof(id.internal));
        std::rename(tmp.c_str(), path.c_str());
    } else {
        for (;;) {
            std::ifstream f(path, std::ios::binary);
            if (f && f.read(id.internal, sizeof(id.internal))) break;
            std::this_thread::sleep_for(std::chrono::milliseconds(20));
        }
    }
    return id;
}
}  // namespace

int main(int argc, char **argv) {
    int dims[3] = {160, 192, 224}, nd = 0, iters = 50, pairs = 1, quiet = 0, eager = 0;
    int synth = 0, large = 0, diffeo = 0, sgd = 0;
    int rank = env_int("RANK", 0), world = env_int("WORLD_SIZE", 1), device = env_int("LOCAL_RANK", 0);
    std::string gather = "", rdv = ".";
    double lr = 1e-4;
    unsigned long long seed = 42;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        if (a == "--iters" && i + 1 < argc) iters = std::atoi(argv[++i]);
        else if (a == "--lr" && i + 1 < argc) lr = std::atof(argv[++i]);
        else if (a == "--seed" && i + 1 < argc) seed = std::strtoull(argv[++i], nullptr, 10);
        else if (a == "--pairs" && i + 1 < argc) pairs = std::atoi(argv[++i]);
        else if (a == "--rank" && i + 1 < argc) rank = std::atoi(argv[++i]);
        else if (a == "--world" && i + 1 < argc) world = std::atoi(argv[++i]);
        else if (a == "--device" && i + 1 < argc) device = std::atoi(argv[++i]);
        else if (a == "--gather" && i + 1 < argc) gather = argv[++i];
        else if (a == "--rendezvous" && i + 1 < argc) rdv = argv[++i];
        else if (a == "--quiet") quiet = 1;
        else if (a == "--eager") eager = 1;
        else if (a == "--synth") synth = 1;
        else if (a == "--large") large = 1;
        else if (a == "--diffeomorphic") diffeo = 1;
        else if (a == "--sgd") sgd = 1;
        else if (nd < 3) dims[nd++] = std::atoi(a.c_str());
        else {
            std::fprintf(stderr,
                         "usage: %s [h w l] [--iters N] [--lr X] [--seed S] [--pairs P] [--synth]"
                         " [--large] [--diffeomorphic] [--sgd] [--eager] [--quiet] [--rank R "
                         "--world W --device D] [--gather nccl|file] [--rendezvous DIR]\n",
                         argv[0]);
            return 2;
        }
    }
    if (gather.empty()) gather = world > 1 ? "nccl" : "none";
    CK(cudaSetDevice(device));
    if (!mdg_device_ok()) {
        std::fprintf(stderr, "po_main: libmdg needs an sm_100a device\n");
        return 1;
    }
    const mdg_dims3 d{dims[0], dims[1], dims[2]};
    const int64_t n = (int64_t)d.h * d.w * d.l;
    // ModelConfig: small or large preset (engine.hpp:38-52), optional SS
    mdg_model_config cfg;
    MK(mdg_model_config_small_preset(&cfg));
    if (large) {
        cfg.base_channels = 32;
        cfg.head_dim = 12;
        const int hl[5] = {32, 16, 8, 4, 1};
        std::memcpy(cfg.heads_per_level, hl, sizeof hl);
    }
    cfg.diffeomorphic = diffeo;
    int nt = 0;
    mdg_config_param_count(&cfg, &nt, nullptr);
    std::vector<int64_t> sizes(nt);
    const int64_t total = mdg_config_param_count(&cfg, nullptr, sizes.data());
    std::vector<std::vector<float>> host(nt);
    std::vector<float *> hp(nt), dp(nt);
    for (int i = 0; i < nt; ++i) {
        host[i].resize(sizes[i]);
        hp[i] = host[i].data();
        CK(cudaMalloc(&dp[i], sizes[i] * sizeof(float)));
    }
    std::vector<float> hf(n), hm(n);
    std::vector<int> lf, lm;
    if (!synth) {  // bench.py's PO pair: U(0,1) volumes of Rng(11)
        mdg_rng *r = mdg_rng_new(11);
        mdg_rng_fill_uniform(r, hf.data(), n, 0.0, 1.0);
        mdg_rng_fill_uniform(r, hm.data(), n, 0.0, 1.0);
        mdg_rng_free(r);
    } else {
        lf.resize(n);
        lm.resize(n);
    }
    float *fixed, *moving, *terms_d, *phi_d;
    int *lf_d = nullptr, *lm_d = nullptr, *lw_d = nullptr;
    CK(cudaMalloc(&fixed, n * sizeof(float)));
    CK(cudaMalloc(&moving, n * sizeof(float)));
    CK(cudaMalloc(&terms_d, 3 * sizeof(float)));
    CK(cudaMalloc(&phi_d, 3 * n * sizeof(float)));
    if (synth) {
        CK(cudaMalloc(&lf_d, n * sizeof(int)));
        CK(cudaMalloc(&lm_d, n * sizeof(int)));
        CK(cudaMalloc(&lw_d, n * sizeof(int)));
    }
    float *terms_h;
    CK(cudaMallocHost(&terms_h, 3 * sizeof(float)));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    auto dice_of = [&](const float *phi) {
        MK(mdg_warp_labels(lm_d, d, phi, lw_d, st));
        double dsc = 0.0;
        MK(mdg_mean_dice(lf_d, lw_d, n, 64, &dsc, st));
        return dsc;
    };

    std::vector<PairResult> mine;
    double sum_iter_ms = 0.0;
    int timed_iters = 0;
    const auto t_all = std::chrono::steady_clock::now();
    for (int p = rank; p < pairs; p += world) {
        const auto t_pair = std::chrono::steady_clock::now();
        PairResult res;
        res.pair = p;
        res.rank = rank;
        if (synth)
            MK(mdg_synth_pair(d, (uint64_t)p + 1, 2.0f, hf.data(), hm.data(), lf.data(), lm.data(),
                              nullptr));
        CK(cudaMemcpyAsync(fixed, hf.data(), n * sizeof(float), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(moving, hm.data(), n * sizeof(float), cudaMemcpyHostToDevice, st));
        if (synth) {
            CK(cudaMemcpyAsync(lf_d, lf.data(), n * sizeof(int), cudaMemcpyHostToDevice, st));
            CK(cudaMemcpyAsync(lm_d, lm.data(), n * sizeof(int), cudaMemcpyHostToDevice, st));
        }
        MK(mdg_model_init_cfg(&cfg, seed, hp.data()));
        for (int i = 0; i < nt; ++i)
            CK(cudaMemcpyAsync(dp[i], hp[i], sizes[i] * sizeof(float), cudaMemcpyHostToDevice, st));
        mdg_model *m = nullptr;
        MK(mdg_model_create_cfg(&cfg, d, dp.data(), 1.0f, 9, 0, sgd ? MDG_OPT_SGD : MDG_OPT_ADAM,
                                &m));
        std::vector<float> trace;
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        double pair_ms = 0.0;
        int pair_timed = 0;
        for (int it = 0; it <= iters; ++it) {
            const bool last = it == iters;
            CK(cudaEventRecord(e0, st));
            if (last) {
                MK(mdg_model_loss_step(m, fixed, moving, 0, terms_d, phi_d, st));
            } else if (eager) {
                MK(mdg_model_loss_step(m, fixed, moving, 1, terms_d, phi_d, st));
                MK(mdg_model_adam_step(m, lr, st));
            } else {
                MK(mdg_model_po_step(m, fixed, moving, lr, terms_d, st));  // CUDA graph
            }
            CK(cudaEventRecord(e1, st));
            CK(cudaMemcpyAsync(terms_h, terms_d, 3 * sizeof(float), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (!std::isfinite(terms_h[0])) {
                std::fprintf(stderr, "optimization: non-finite loss (%g)\n", terms_h[0]);
                return 1;
            }
            trace.push_back(terms_h[0]);
            float ms = 0.0f;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (!last && it >= 2) {  // the first updates warm the allocator / capture
                pair_ms += ms;
                ++pair_timed;
            }
            // the field of this step's forward (before its update)
            if (synth && it == 0) res.dice0 = dice_of(mdg_model_phi(m));
        }
        if (synth) res.dice_final = dice_of(phi_d);
        res.loss0 = trace.front();
        res.loss_final = trace.back();
        res.iter_ms = pair_timed ? pair_ms / pair_timed : 0.0;
        res.wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_pair).count();
        sum_iter_ms += pair_ms;
        timed_iters += pair_timed;
        if (!quiet)
            std::printf("rank %d pair %d: loss %.6f -> %.6f over %d updates%s\n", rank, p,
                        trace.front(), trace.back(), iters,
                        synth ? (", Dice " + std::to_string(res.dice0) + " -> " +
                                 std::to_string(res.dice_final)).c_str()
                              : "");
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        mdg_model_destroy(m);
        mine.push_back(res);
    }
    CK(cudaStreamSynchronize(st));
    const double wall =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_all).count();

    // gather every rank's results (fixed-size records, padded per rank)
    const int per_rank = (pairs + world - 1) / world;
    std::vector<PairResult> all((size_t)per_rank * world);
    std::vector<double> walls(world, 0.0);
    if (gather == "nccl") {  // (also at world 1 when asked: the same code path)
        ncclComm_t comm;
        NK(ncclCommInitRank(&comm, world, nccl_id(rdv, rank), rank));
        const size_t rec = sizeof(PairResult) / sizeof(double);
        std::vector<PairResult> pad(per_rank);
        for (size_t i = 0; i < mine.size(); ++i) pad[i] = mine[i];
        double *sbuf, *rbuf, *wb;
        CK(cudaMalloc(&sbuf, per_rank * rec * sizeof(double)));
        CK(cudaMalloc(&rbuf, (size_t)per_rank * world * rec * sizeof(double)));
        CK(cudaMalloc(&wb, world * sizeof(double)));
        CK(cudaMemcpy(sbuf, pad.data(), per_rank * rec * sizeof(double), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(wb + rank, &wall, sizeof(double), cudaMemcpyHostToDevice));
        NK(ncclGroupStart());
        NK(ncclAllGather(sbuf, rbuf, per_rank * rec, ncclDouble, comm, st));
        NK(ncclAllGather(wb + rank, wb, 1, ncclDouble, comm, st));
        NK(ncclGroupEnd());
        CK(cudaStreamSynchronize(st));
        CK(cudaMemcpy(all.data(), rbuf, all.size() * sizeof(PairResult), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(walls.data(), wb, world * sizeof(double), cudaMemcpyDeviceToHost));
        ncclCommDestroy(comm);
        cudaFree(sbuf);
        cudaFree(rbuf);
        cudaFree(wb);
    } else if (world > 1) {  // files: ranks that share a device (no collective)
        {
            std::ofstream f(rdv + "/po_main_rank" + std::to_string(rank) + ".bin.tmp",
                            std::ios::binary);
            f.write(reinterpret_cast<const char *>(&wall), sizeof wall);
            std::vector<PairResult> pad(per_rank);
            for (size_t i = 0; i < mine.size(); ++i) pad[i] = mine[i];
            f.write(reinterpret_cast<const char *>(pad.data()), pad.size() * sizeof(PairResult));
        }
        std::rename((rdv + "/po_main_rank" + std::to_string(rank) + ".bin.tmp").c_str(),
                    (rdv + "/po_main_rank" + std::to_string(rank) + ".bin").c_str());
        for (int r = 0; r < world; ++r)
            for (;;) {
                std::ifstream f(rdv + "/po_main_rank" + std::to_string(r) + ".bin",
                                std::ios::binary);
                if (f && f.read(reinterpret_cast<char *>(&walls[r]), sizeof(double)) &&
                    f.read(reinterpret_cast<char *>(all.data() + (size_t)r * per_rank),
                           per_rank * sizeof(PairResult)))
                    break;
                std::this_thread::sleep_for(std::chrono::milliseconds(20));
            }
    } else {
        for (size_t i = 0; i < mine.size(); ++i) all[i] = mine[i];
        walls[0] = wall;
    }
    if (rank == 0) {
        double slowest = 0.0;
        for (double w : walls) slowest = std::max(slowest, w);
        std::ostringstream js;
        js << "{\"dims\": [" << d.h << ", " << d.w << ", " << d.l << "], \"params\": " << total
           << ", \"config\": \"" << (large ? "large" : "small") << (diffeo ? "+ss" : "")
           << "\", \"optimizer\": \"" << (sgd ? "sgd" : "adam") << "\", \"iters\": " << iters
           << ", \"pairs\": " << pairs << ", \"world\": " << world << ", \"gather\": \""
           << gather << "\", \"iter_ms_rank0\": " << (timed_iters ? sum_iter_ms / timed_iters : 0.0)
           << ", \"pairs_per_sec_wall\": " << (slowest > 0 ? pairs / slowest : 0.0)
           << ", \"launches_rank0\": " << mdg_launch_count() << ", \"results\": [";
        bool first = true;
        for (const PairResult &r : all) {
            if (r.pair < 0) continue;
            js << (first ? "" : ", ") << "{\"pair\": " << (int)r.pair << ", \"rank\": "
               << (int)r.rank << ", \"loss0\": " << r.loss0 << ", \"loss_final\": "
               << r.loss_final;
            if (synth) js << ", \"dice0\": " << r.dice0 << ", \"dice_final\": " << r.dice_final;
            js << ", \"iter_ms\": " << r.iter_ms << "}";
            first = false;
        }
        js << "]}";
        std::printf("%s\n", js.str().c_str());
    }
    for (int i = 0; i < nt; ++i) cudaFree(dp[i]);
    cudaFree(fixed);
    cudaFree(moving);
    cudaFree(terms_d);
    cudaFree(phi_d);
    if (synth) {
        cudaFree(lf_d);
        cudaFree(lm_d);
        cudaFree(lw_d);
    }
    cudaFreeHost(terms_h);
    cudaStreamDestroy(st);
    return 0;
}
