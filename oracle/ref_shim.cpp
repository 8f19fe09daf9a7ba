// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" face over the UNMODIFIED reference headers under
// /root/reference/proj/include (compiled where they lie by oracle/Makefile into
// oracle/_ref/libmdreg_ref.so).  It is used to (a) pin the C restatement in
// oracle/mdo.c bit-for-bit, (b) generate the golden fixtures in tests/golden/,
// and (c) serve as bench.py's `--impl reference` CPU arm.  No reference source
// is copied: every body below only forwards to mdreg:: symbols.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "mdreg/attention.hpp"
#include "mdreg/bench.hpp"
#include "mdreg/metrics.hpp"
#include "mdreg/field_ops.hpp"
#include "mdreg/reghead.hpp"
#include "mdreg/sampling.hpp"
#include "mdreg/synth.hpp"

using namespace mdreg;

namespace {
thread_local std::string g_err;
Dims3 D(int h, int w, int l) { return Dims3{h, w, l}; }
}  // namespace

extern "C" {

const char *mdr_last_error() { return g_err.c_str(); }

void mdr_window_offset(int o, int nb, int off[3]) {
    auto a = window_offset(o, nb);
    off[0] = a[0];
    off[1] = a[1];
    off[2] = a[2];
}

// attention.hpp:83 (kern::na_fused_fwd); returns 1 on numeric_error
int mdr_na_fwd(const float *Q, const float *K, const float *B, int h, int w, int l, int S,
               int hd, int nb, float *W) {
    try {
        kern::na_fused_fwd<float>(Q, K, B, D(h, w, l), S, hd, nb, W);
    } catch (const numeric_error &e) {
        g_err = e.what();
        return 1;
    }
    return 0;
}

int mdr_na_naive_fwd(const float *Q, const float *K, const float *B, int h, int w, int l,
                     int S, int hd, int nb, float *W) {
    try {
        kern::na_naive_fwd<float>(Q, K, B, D(h, w, l), S, hd, nb, W);
    } catch (const numeric_error &e) {
        g_err = e.what();
        return 1;
    }
    return 0;
}

void mdr_na_bwd(const float *Q, const float *K, const float *W, int h, int w, int l, int S,
                int hd, int nb, const float *gW, float *gQ, float *gK, float *gB) {
    kern::na_fused_bwd<float>(Q, K, W, D(h, w, l), S, hd, nb, gW, gQ, gK, gB);
}

void mdr_subfields_fwd(const float *W, int h, int w, int l, int S, int nb, float *out) {
    kern::subfields_fwd<float>(W, D(h, w, l), S, nb, out);
}

void mdr_subfields_bwd(int h, int w, int l, int S, int nb, const float *gout, float *gW) {
    kern::subfields_bwd<float>(D(h, w, l), S, nb, gout, gW);
}

void mdr_resolve_axis(float x, int dim, int *i0, int *i1, float *f, int *live) {
    auto a = kern::resolve_axis<float>(x, dim);
    *i0 = a.i0;
    *i1 = a.i1;
    *f = a.f;
    *live = a.live ? 1 : 0;
}

void mdr_warp_fwd(const float *in, int C, int h, int w, int l, const float *field, float *out) {
    kern::warp_fwd<float>(in, C, D(h, w, l), field, out);
}

void mdr_warp_bwd(const float *in, int C, int h, int w, int l, const float *field,
                  const float *gout, float *gin, float *gfield) {
    kern::warp_bwd<float>(in, C, D(h, w, l), field, gout, gin, gfield);
}

void mdr_upsample2_fwd(const float *in, int C, int h, int w, int l, int th, int tw, int tl,
                       float scale, float *out) {
    kern::upsample2_fwd<float>(in, C, D(h, w, l), D(th, tw, tl), scale, out);
}

void mdr_upsample2_bwd(int C, int h, int w, int l, int th, int tw, int tl, float scale,
                       const float *gout, float *gin) {
    kern::upsample2_bwd<float>(C, D(h, w, l), D(th, tw, tl), scale, gout, gin);
}

int mdr_upsample_target_ok(int h, int w, int l, int th, int tw, int tl) {
    try {
        check_upsample_target(D(h, w, l), D(th, tw, tl));
    } catch (const invalid_input &) {
        return 0;
    }
    return 1;
}

void mdr_conv3_fwd(const float *in, int ic, int h, int w, int l, const float *k,
                   const float *bias, int oc, float *out) {
    kern::conv3_fwd<float>(in, ic, D(h, w, l), k, bias, oc, out);
}

void mdr_conv3_bwd(const float *in, int ic, int h, int w, int l, const float *k, int oc,
                   const float *gout, float *gin, float *gk, float *gbias) {
    kern::conv3_bwd<float>(in, ic, D(h, w, l), k, oc, gout, gin, gk, gbias);
}

// field_ops.hpp:42 (plain compose)
void mdr_compose_fwd(const float *prev, const float *res, int h, int w, int l, float *out) {
    DisplacementField a(D(h, w, l)), b(D(h, w, l));
    const std::size_t n3 = a.data.size();
    std::memcpy(a.data.data(), prev, n3 * sizeof(float));
    std::memcpy(b.data.data(), res, n3 * sizeof(float));
    DisplacementField c = compose(a, b);
    std::memcpy(out, c.data.data(), n3 * sizeof(float));
}

// ops.hpp:295 (tape compose) forward + backward with a caller-supplied output
// gradient; accumulates into gprev / gres like the tape would.
void mdr_compose_bwd(const float *prev, const float *res, int h, int w, int l,
                     const float *gout, float *gprev, float *gres) {
    const Dims3 d = D(h, w, l);
    const std::size_t n3 = 3 * static_cast<std::size_t>(voxel_count(d));
    Tape<float> t;
    Tensor<float> tp({3, h, w, l}), tr({3, h, w, l}), tg({3, h, w, l});
    std::memcpy(tp.data.data(), prev, n3 * sizeof(float));
    std::memcpy(tr.data.data(), res, n3 * sizeof(float));
    std::memcpy(tg.data.data(), gout, n3 * sizeof(float));
    Var vp = t.input(tp), vr = t.input(tr);
    Var c = op_compose(t, vp, vr);
    // loss = sum(c * gout) has d loss / d c = gout exactly
    Var loss = op_sum_all(t, op_mul(t, c, t.input(tg)));
    t.backward(loss);
    for (std::size_t i = 0; i < n3; ++i) {
        if (gprev) gprev[i] += t.grad(vp)[static_cast<std::int64_t>(i)];
        if (gres) gres[i] += t.grad(vr)[static_cast<std::int64_t>(i)];
    }
}

void mdr_scaling_squaring(const float *vel, int h, int w, int l, int steps, float *out) {
    DisplacementField v(D(h, w, l));
    std::memcpy(v.data.data(), vel, v.data.size() * sizeof(float));
    DisplacementField p = scaling_squaring(v, steps);
    std::memcpy(out, p.data.data(), p.data.size() * sizeof(float));
}

// synth.cpp:75 — smooth random velocity (the warp benchmark's field)
void mdr_make_smooth_velocity(int h, int w, int l, std::uint64_t seed, float magnitude,
                              float sigma, float *out) {
    DisplacementField v = make_smooth_velocity(D(h, w, l), seed, magnitude, sigma);
    std::memcpy(out, v.data.data(), v.data.size() * sizeof(float));
}

// bench.cpp:23 — the reference's own fused-vs-naive attention benchmark
double mdr_attention_bench_fused_ms(int h, int w, int l, int S, int hd, int reps,
                                    std::uint64_t seed) {
    BenchReport r = run_attention_bench(D(h, w, l), S, hd, reps, seed);
    return r.fused.time_ms;
}

// synth.cpp make_synth_pair: images, label volumes and the ground-truth field
void mdr_make_synth_pair(int h, int w, int l, std::uint64_t seed, float max_disp, float *fixed,
                         float *moving, int *labels_fixed, int *labels_moving, float *gt) {
    SynthConfig cfg;
    cfg.dims = D(h, w, l);
    cfg.seed = seed;
    cfg.max_disp = max_disp;
    SynthPair sp = make_synth_pair(cfg);
    const size_t n = sp.fixed.data.size();
    std::memcpy(fixed, sp.fixed.data.data(), n * sizeof(float));
    std::memcpy(moving, sp.moving.data.data(), n * sizeof(float));
    std::memcpy(labels_fixed, sp.labels_fixed.data.data(), n * sizeof(int));
    std::memcpy(labels_moving, sp.labels_moving.data.data(), n * sizeof(int));
    std::memcpy(gt, sp.gt_field.data.data(), 3 * n * sizeof(float));
}

// metrics.cpp:145-164 warp_labels (nearest neighbour)
void mdr_warp_labels(const int *labels, int h, int w, int l, const float *phi, int *out) {
    LabelVolume lv(D(h, w, l));
    std::memcpy(lv.data.data(), labels, lv.data.size() * sizeof(int));
    DisplacementField f(D(h, w, l));
    std::memcpy(f.data.data(), phi, f.data.size() * sizeof(float));
    LabelVolume o = warp_labels(lv, f);
    std::memcpy(out, o.data.data(), o.data.size() * sizeof(int));
}

// metrics.cpp:123-129 mean_dice
double mdr_mean_dice(const int *a, const int *b, int h, int w, int l) {
    LabelVolume la(D(h, w, l)), lb(D(h, w, l));
    std::memcpy(la.data.data(), a, la.data.size() * sizeof(int));
    std::memcpy(lb.data.data(), b, lb.data.size() * sizeof(int));
    return mean_dice(la, lb);
}

}  // extern "C"
