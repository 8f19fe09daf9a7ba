// po_main.cpp — pairwise optimisation (engine.hpp:377-411) of the small-preset
// model driven from C++ through include/mdg.h alone: no Python, no PyTorch.
//
//   po_main [h w l] [--iters N] [--lr X] [--seed S] [--pairs P] [--quiet] [--eager]
//
// Per pair: init_model(seed) on the host (the reference Rng stream), upload,
// then N updates of run_loss_step + Adam and a final evaluation forward; the
// loss is read back every iteration and checked finite like the reference's
// loop.  The synthetic pair is U(0,1) volumes from Rng(11) (bench.py's
// run_po).  Prints the loss trace ends and ms/iteration, pairs/sec.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
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

int main(int argc, char **argv) {
    int dims[3] = {160, 192, 224}, nd = 0, iters = 50, pairs = 1, quiet = 0, eager = 0;
    double lr = 1e-4;
    unsigned long long seed = 42;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        if (a == "--iters" && i + 1 < argc) iters = std::atoi(argv[++i]);
        else if (a == "--lr" && i + 1 < argc) lr = std::atof(argv[++i]);
        else if (a == "--seed" && i + 1 < argc) seed = std::strtoull(argv[++i], nullptr, 10);
        else if (a == "--pairs" && i + 1 < argc) pairs = std::atoi(argv[++i]);
        else if (a == "--quiet") quiet = 1;
        else if (a == "--eager") eager = 1;
        else if (nd < 3) dims[nd++] = std::atoi(a.c_str());
        else {
            std::fprintf(stderr, "usage: %s [h w l] [--iters N] [--lr X] [--seed S] [--pairs P]\n",
                         argv[0]);
            return 2;
        }
    }
    if (!mdg_device_ok()) {
        std::fprintf(stderr, "po_main: libmdg needs an sm_100a device\n");
        return 1;
    }
    const mdg_dims3 d{dims[0], dims[1], dims[2]};
    const int64_t n = (int64_t)d.h * d.w * d.l;

    int nt = 0;
    mdg_model_param_count(&nt, nullptr);
    std::vector<int64_t> sizes(nt);
    const int64_t total = mdg_model_param_count(nullptr, sizes.data());
    std::vector<std::vector<float>> host(nt);
    std::vector<float *> hp(nt), dp(nt);
    for (int i = 0; i < nt; ++i) {
        host[i].resize(sizes[i]);
        hp[i] = host[i].data();
        CK(cudaMalloc(&dp[i], sizes[i] * sizeof(float)));
    }

    // the synthetic pair
    std::vector<float> hf(n), hm(n);
    mdg_rng *r = mdg_rng_new(11);
    mdg_rng_fill_uniform(r, hf.data(), n, 0.0, 1.0);
    mdg_rng_fill_uniform(r, hm.data(), n, 0.0, 1.0);
    mdg_rng_free(r);
    float *fixed, *moving, *terms_d;
    CK(cudaMalloc(&fixed, n * sizeof(float)));
    CK(cudaMalloc(&moving, n * sizeof(float)));
    CK(cudaMalloc(&terms_d, 3 * sizeof(float)));
    CK(cudaMemcpy(fixed, hf.data(), n * sizeof(float), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(moving, hm.data(), n * sizeof(float), cudaMemcpyHostToDevice));
    float *terms_h;
    CK(cudaMallocHost(&terms_h, 3 * sizeof(float)));
    cudaStream_t st;
    CK(cudaStreamCreate(&st));

    double sum_iter_ms = 0.0;
    int timed_iters = 0;
    const auto t_all = std::chrono::steady_clock::now();
    for (int p = 0; p < pairs; ++p) {
        MK(mdg_model_init(seed, hp.data()));
        for (int i = 0; i < nt; ++i)
            CK(cudaMemcpyAsync(dp[i], hp[i], sizes[i] * sizeof(float), cudaMemcpyHostToDevice, st));
        mdg_model *m = nullptr;
        MK(mdg_model_create(d, dp.data(), 1.0f, 9, 0, &m));
        std::vector<float> trace;
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        for (int it = 0; it <= iters; ++it) {
            const bool last = it == iters;
            CK(cudaEventRecord(e0, st));
            if (last) {
                MK(mdg_model_loss_step(m, fixed, moving, 0, terms_d, nullptr, st));
            } else if (eager) {
                MK(mdg_model_loss_step(m, fixed, moving, 1, terms_d, nullptr, st));
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
            if (!last && it >= 2) {  // the first updates warm the allocator
                sum_iter_ms += ms;
                ++timed_iters;
            }
        }
        if (!quiet)
            std::printf("pair %d: loss %.6f -> %.6f over %d updates\n", p, trace.front(),
                        trace.back(), iters);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        mdg_model_destroy(m);
    }
    CK(cudaStreamSynchronize(st));
    const double wall =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_all).count();
    std::printf("{\"dims\": [%d, %d, %d], \"params\": %lld, \"iters\": %d, \"pairs\": %d, "
                "\"iter_ms\": %.3f, \"pairs_per_sec_wall\": %.4f, \"launches\": %lld}\n",
                d.h, d.w, d.l, (long long)total, iters, pairs,
                timed_iters ? sum_iter_ms / timed_iters : 0.0, pairs / wall,
                (long long)mdg_launch_count());
    for (int i = 0; i < nt; ++i) cudaFree(dp[i]);
    cudaFree(fixed);
    cudaFree(moving);
    cudaFree(terms_d);
    cudaFreeHost(terms_h);
    cudaStreamDestroy(st);
    return 0;
}
