// test_engine_b200.cpp — the reference's own engine tests (tests/test_engine.cpp)
// restated without doctest and run against the UNMODIFIED reference headers
// with their float kernels bound to libmdg (-DMDREG_B200, -include
// mdreg_b200.hpp).  build_pipeline / forward / run_loss_step /
// pairwise_optimize below are the reference's code; every na_fused, subfields,
// warp, upsample and conv3 kernel they reach runs on the GPU.
//
// Prints one JSON line: per-case pass/fail, the loss traces and the number of
// libmdg kernel launches (tests/test_integration.py checks it).
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "mdreg/engine.hpp"
#include "mdreg/synth.hpp"

using namespace mdreg;

namespace {
int g_fail = 0;
std::string g_cases;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            ++g_fail;                                                            \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                        \
    } while (0)

template <class F>
void run_case(const char *name, F &&f) {
    const int before = g_fail;
    try {
        f();
    } catch (const std::exception &e) {
        ++g_fail;
        std::fprintf(stderr, "case '%s' threw: %s\n", name, e.what());
    }
    if (!g_cases.empty()) g_cases += ",";
    g_cases += std::string("\"") + name + "\":" + (g_fail == before ? "true" : "false");
}

Volume random_volume(Dims3 d, std::uint64_t seed) {  // tests/test_util.hpp:24-29
    Rng rng(seed);
    Volume v(d);
    for (auto &x : v.data) x = static_cast<float>(rng.uniform(0.0, 1.0));
    return v;
}

std::string trace_json(const std::vector<double> &t) {
    std::string s = "[";
    char buf[64];
    for (std::size_t i = 0; i < t.size(); ++i) {
        std::snprintf(buf, sizeof buf, "%s%.9g", i ? "," : "", t[i]);
        s += buf;
    }
    return s + "]";
}
}  // namespace

int main() {
    std::string traces;
    // test_engine.cpp:70-83
    run_case("residual_shape_chain_32", [] {
        ModelParams<float> params = init_model<float>(ModelConfig::small_preset(), 1);
        const SynthConfig scfg{{32, 32, 32}, 2, 1.5f};
        const SynthPair sp = make_synth_pair(scfg);
        const RegistrationResult res = forward(sp.fixed, sp.moving, params);
        CHECK(res.residuals.size() == 5);
        const int expect[5] = {2, 4, 8, 16, 32};
        for (int k = 0; k < 5 && k < (int)res.residuals.size(); ++k)
            CHECK(res.residuals[k].dims == (Dims3{expect[k], expect[k], expect[k]}));
        CHECK(res.phi.dims == (Dims3{32, 32, 32}));
        CHECK(res.warped.dims == (Dims3{32, 32, 32}));
    });
    // test_engine.cpp:84-92
    run_case("fresh_model_near_identity", [] {
        ModelParams<float> params = init_model<float>(ModelConfig::small_preset(), 3);
        const Volume img = random_volume({16, 16, 16}, 5);
        const RegistrationResult res = forward(img, img, params);
        float worst = 0.0f;
        for (float v : res.phi.data) worst = std::max(worst, std::abs(v));
        CHECK(worst <= 1e-2f);
    });
    // test_engine.cpp:94-102
    run_case("fresh_diffeomorphic_fold_free", [] {
        ModelConfig cfg = ModelConfig::small_preset();
        cfg.diffeomorphic = true;
        ModelParams<float> params = init_model<float>(cfg, 7);
        const SynthConfig scfg{{16, 16, 16}, 4, 1.0f};
        const SynthPair sp = make_synth_pair(scfg);
        const RegistrationResult res = forward(sp.fixed, sp.moving, params);
        CHECK(res.folding == 0.0);
    });
    // test_engine.cpp:104-109
    run_case("rejects_mismatched_pairs", [] {
        ModelParams<float> params = init_model<float>(ModelConfig::small_preset(), 9);
        const Volume a = random_volume({16, 16, 16}, 1);
        const Volume b = random_volume({16, 16, 20}, 2);
        bool threw = false;
        try {
            (void)forward(a, b, params);
        } catch (const invalid_input &) {
            threw = true;
        }
        CHECK(threw);
    });
    // the libmdg error path surfaces as the reference's numeric_error
    run_case("nonfinite_logit_is_numeric_error", [] {
        const Dims3 d{3, 2, 2};
        std::vector<float> Q(12 * 4, 0.1f), K(12 * 4, 0.2f), B(2 * 27, 0.0f), W(2 * 12 * 27);
        Q[7 * 4 + 3] = INFINITY;
        bool threw = false;
        try {
            kern::na_fused_fwd<float>(Q.data(), K.data(), B.data(), d, 2, 2, 3, W.data());
        } catch (const numeric_error &e) {
            threw = std::string(e.what()).find("non-finite") != std::string::npos;
        }
        CHECK(threw);
    });
    // test_engine.cpp:139-151
    run_case("po_identical_pair_stays_near_identity", [&] {
        ModelParams<float> params = init_model<float>(ModelConfig::small_preset(), 17);
        const SynthConfig scfg{{16, 16, 16}, 10, 0.0f};
        const SynthPair sp = make_synth_pair(scfg);
        OptimConfig opt;
        opt.po_iters = 50;
        opt.lambda = 0.5;
        opt.ncc_window = 9;
        const PoResult res = pairwise_optimize(sp.moving, sp.moving, params, opt);
        float worst = 0.0f;
        for (float v : res.reg.phi.data) worst = std::max(worst, std::abs(v));
        CHECK(worst <= 0.1f);
    });
    // test_engine.cpp:154-192
    run_case("po_recovers_known_translation", [&] {
        const SynthConfig scfg{{24, 24, 24}, 12, 0.0f};
        SynthPair sp = make_synth_pair(scfg);
        const Dims3 d = sp.moving.dims;
        DisplacementField gt(d);
        const std::int64_t n = voxel_count(d);
        for (std::int64_t i = 0; i < n; ++i) gt.data[i] = 2.0f;
        const Volume fixed = warp(sp.moving, gt);
        const LabelVolume labels_fixed = warp_labels(sp.labels_moving, gt);
        ModelParams<float> params = init_model<float>(ModelConfig::small_preset(), 19);
        OptimConfig opt;
        opt.po_iters = 50;
        opt.lr_init = 1e-4;
        opt.lambda = 0.5;
        opt.ncc_window = 9;
        const PoResult res =
            pairwise_optimize(fixed, sp.moving, params, opt, &labels_fixed, &sp.labels_moving);
        double epe = 0.0;
        std::int64_t cnt = 0;
        for (std::int64_t p = 0; p < n; ++p) {
            if (labels_fixed.data[p] == 0) continue;
            double e2 = 0.0;
            for (int comp = 0; comp < 3; ++comp) {
                const double diff = res.reg.phi.data[comp * n + p] - gt.data[comp * n + p];
                e2 += diff * diff;
            }
            epe += std::sqrt(e2);
            ++cnt;
        }
        CHECK(cnt > 0);
        CHECK(epe / static_cast<double>(cnt) <= 0.5);
        CHECK(res.loss_trace.back() < res.loss_trace.front());
        CHECK(res.dice_trace.back() > res.dice_trace.front());
        traces += "\"translation_loss\":" + trace_json(res.loss_trace) +
                  ",\"translation_dice\":" + trace_json(res.dice_trace) + ",";
        char buf[64];
        std::snprintf(buf, sizeof buf, "\"translation_epe\":%.6g,", epe / (double)cnt);
        traces += buf;
    });
    // test_engine.cpp:194-213
    run_case("fixed_seeds_bitwise_identical_traces", [&] {
        const SynthConfig scfg{{16, 16, 16}, 14, 1.0f};
        const SynthPair sp = make_synth_pair(scfg);
        OptimConfig opt;
        opt.po_iters = 5;
        opt.lambda = 0.5;
        opt.ncc_window = 9;
        std::vector<double> first;
        for (int run = 0; run < 2; ++run) {
            ModelParams<float> params = init_model<float>(ModelConfig::small_preset(), 21);
            const PoResult res = pairwise_optimize(sp.fixed, sp.moving, params, opt);
            if (run == 0) {
                first = res.loss_trace;
            } else {
                CHECK(res.loss_trace.size() == first.size());
                for (std::size_t i = 0; i < first.size() && i < res.loss_trace.size(); ++i)
                    CHECK(res.loss_trace[i] == first[i]);
            }
        }
        traces += "\"repeat_loss\":" + trace_json(first) + ",";
    });
    std::printf("{%s\"cases\":{%s},\"failures\":%d,\"mdg_launches\":%lld,\"build\":\"%s\"}\n",
                traces.c_str(), g_cases.c_str(), g_fail, (long long)mdg_launch_count(),
                mdg_build_info());
    return g_fail == 0 ? 0 : 1;
}
