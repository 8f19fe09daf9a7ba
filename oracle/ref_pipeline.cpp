// ref_pipeline.cpp — TEST INFRASTRUCTURE ONLY: extern "C" access to the
// reference's decoding pyramid (engine.hpp:179-219) and Q/K projection
// (attention.hpp:351-356, ops.hpp:387-497) for pipeline-level parity.  Every
// value comes from mdreg:: operators on an mdreg::Tape; the bodies only marshal
// buffers.
//
// Packed per-level parameter block (the order of ModelParams::all_tensors,
// engine.hpp:127-131):  proj.w {K,C} | proj.b {K} | ln_g {K} | ln_b {K} |
// bias_b {S,27} | reghead.w {3,3S,3,3,3} | reghead.b {3},  K = S*hd.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "mdreg/engine.hpp"

using namespace mdreg;

namespace {
thread_local std::string g_perr;

Tensor<float> tensor_from(const float *src, std::vector<int> shape) {
    Tensor<float> t(std::move(shape));
    std::memcpy(t.data.data(), src, t.data.size() * sizeof(float));
    return t;
}

void add_into(float *dst, const Tensor<float> &g) {
    if (!dst) return;
    for (std::size_t i = 0; i < g.data.size(); ++i) dst[i] += g.data[i];
}

Dims3 D3(int h, int w, int l) { return Dims3{h, w, l}; }

int64_t level_param_count(int C, int S, int hd, int nb) {
    const int64_t K = (int64_t)S * hd, win = (int64_t)nb * nb * nb;
    return K * C + 3 * K + S * win + 3 * 3 * S * 27 + 3;
}
}  // namespace

extern "C" {

int mdr_pipeline_available() { return 1; }
const char *mdr_pipeline_error() { return g_perr.c_str(); }

int64_t mdr_level_param_count(int C, int S, int hd, int nb) {
    return level_param_count(C, S, hd, nb);
}

// op_project_qk (attention.hpp:351-356) forward, then the tape backward of
// loss = sum(Q*gQ) + sum(K*gK).  Q/K position-major {n, K}.  Grads accumulate;
// any grad pointer may be NULL; gQ == NULL skips the backward entirely.
int mdr_project_qk(const float *f, const float *m, int C, int h, int w, int l,
                   const float *weight, const float *bias, const float *ln_g,
                   const float *ln_b, int K, float *Q, float *Kout, const float *gQ,
                   const float *gK, float *gf, float *gm, float *gweight, float *gbias,
                   float *gln_g, float *gln_b) {
    try {
        const int n = h * w * l;
        Tape<float> t;
        Var fv = t.input(tensor_from(f, {C, h, w, l}));
        Var mv = t.input(tensor_from(m, {C, h, w, l}));
        ProjectionVars pv{t.input(tensor_from(weight, {K, C})), t.input(tensor_from(bias, {K})),
                          t.input(tensor_from(ln_g, {K})), t.input(tensor_from(ln_b, {K}))};
        auto [q, k] = op_project_qk(t, fv, mv, pv);
        std::memcpy(Q, t.value(q).data.data(), (size_t)n * K * sizeof(float));
        std::memcpy(Kout, t.value(k).data.data(), (size_t)n * K * sizeof(float));
        if (!gQ) return 0;
        Var lq = op_sum_all(t, op_mul(t, q, t.input(tensor_from(gQ, {n, K}))));
        Var lk = op_sum_all(t, op_mul(t, k, t.input(tensor_from(gK, {n, K}))));
        t.backward(op_add(t, lq, lk));
        add_into(gf, t.grad(fv));
        add_into(gm, t.grad(mv));
        add_into(gweight, t.grad(pv.weight));
        add_into(gbias, t.grad(pv.bias));
        add_into(gln_g, t.grad(pv.ln_gamma));
        add_into(gln_b, t.grad(pv.ln_beta));
    } catch (const std::exception &e) {
        g_perr = e.what();
        return 1;
    }
    return 0;
}

// The decoding half of build_pipeline (engine.hpp:189-216) on given encoder
// features, coarse -> fine (f_feats[k] {C_k, dims_k}).  Forward writes phi
// {3, n_fine} and (optionally) each level's residual; if gphi is non-NULL the
// tape backward of loss = sum(phi * gphi) accumulates into the packed level
// parameter grads and the feature grads (each nullable).
int mdr_decoder(int levels, const int *dims, const int *channels, const int *heads, int hd,
                int nb, int diffeomorphic, int ss_steps, const float *const *f_feats,
                const float *const *m_feats, const float *const *params, const float *gphi,
                float *phi_out, float *const *res_out, float *const *gparams,
                float *const *gf, float *const *gm) {
    try {
        Tape<float> t;
        std::vector<Var> fv, mv;
        struct LV {
            Var w, b, g, be, bias, rw, rb;
        };
        std::vector<LV> lv;
        for (int k = 0; k < levels; ++k) {
            const int h = dims[3 * k], w = dims[3 * k + 1], l = dims[3 * k + 2];
            const int C = channels[k], S = heads[k], K = S * hd, win = nb * nb * nb;
            fv.push_back(t.input(tensor_from(f_feats[k], {C, h, w, l})));
            mv.push_back(t.input(tensor_from(m_feats[k], {C, h, w, l})));
            const float *p = params[k];
            LV v;
            v.w = t.input(tensor_from(p, {K, C})), p += (int64_t)K * C;
            v.b = t.input(tensor_from(p, {K})), p += K;
            v.g = t.input(tensor_from(p, {K})), p += K;
            v.be = t.input(tensor_from(p, {K})), p += K;
            v.bias = t.input(tensor_from(p, {S, win})), p += (int64_t)S * win;
            v.rw = t.input(tensor_from(p, {3, 3 * S, 3, 3, 3})), p += 3 * 3 * S * 27;
            v.rb = t.input(tensor_from(p, {3}));
            lv.push_back(v);
        }
        // engine.hpp:191-216, level loop, with the encoder outputs supplied
        Var phi;
        std::vector<Var> res_v;
        for (int k = 0; k < levels; ++k) {
            const Dims3 d{dims[3 * k], dims[3 * k + 1], dims[3 * k + 2]};
            Var phi_up, m_in = mv[k];
            if (k > 0) {
                phi_up = op_upsample_field_2x(t, phi, d);
                m_in = op_warp(t, mv[k], phi_up);
            }
            ProjectionVars pv{lv[k].w, lv[k].b, lv[k].g, lv[k].be};
            auto [q, key] = op_project_qk(t, fv[k], m_in, pv);
            AttentionConfig acfg;
            acfg.heads = heads[k];
            acfg.head_dim = hd;
            acfg.neighborhood = nb;
            Var weights = op_na_fused(t, q, key, lv[k].bias, d, acfg);
            Var stack = op_subfields(t, weights, d, acfg);
            Var res = op_reghead_fuse(t, stack, lv[k].rw, lv[k].rb);
            if (diffeomorphic) res = op_scaling_squaring(t, res, ss_steps);
            phi = (k == 0) ? res : op_compose(t, phi_up, res);
            res_v.push_back(res);
        }
        const Tensor<float> &pv = t.value(phi);
        std::memcpy(phi_out, pv.data.data(), pv.data.size() * sizeof(float));
        if (res_out)
            for (int k = 0; k < levels; ++k)
                if (res_out[k]) {
                    const Tensor<float> &rv = t.value(res_v[k]);
                    std::memcpy(res_out[k], rv.data.data(), rv.data.size() * sizeof(float));
                }
        if (!gphi) return 0;
        Var loss = op_sum_all(t, op_mul(t, phi, t.input(tensor_from(gphi, pv.shape))));
        t.backward(loss);
        for (int k = 0; k < levels; ++k) {
            if (gf && gf[k]) add_into(gf[k], t.grad(fv[k]));
            if (gm && gm[k]) add_into(gm[k], t.grad(mv[k]));
            if (gparams && gparams[k]) {
                float *g = gparams[k];
                for (Var v : {lv[k].w, lv[k].b, lv[k].g, lv[k].be, lv[k].bias, lv[k].rw,
                              lv[k].rb}) {
                    const Tensor<float> &gt = t.grad(v);
                    add_into(g, gt);
                    g += gt.data.size();
                }
            }
        }
    } catch (const std::exception &e) {
        g_perr = e.what();
        return 1;
    }
    return 0;
}

// op_total_loss (objective.hpp:71-78) = op_ncc_loss(fixed, warp(moving, phi))
// + lambda * op_grad_reg(phi), forward and the tape backward with seed 1.
// Single-channel volumes {h,w,l}; phi {3,h,w,l}.  Writes the loss terms
// (total, ncc, reg) and accumulates gphi / gmoving (nullable).
int mdr_total_loss(const float *fixed, const float *moving, const float *phi, int h, int w,
                   int l, int window, float lambda, float *terms, float *warped, float *gphi,
                   float *gmoving) {
    try {
        Tape<float> t;
        Var f = t.input(tensor_from(fixed, {1, h, w, l}));
        Var m = t.input(tensor_from(moving, {1, h, w, l}));
        Var ph = t.input(tensor_from(phi, {3, h, w, l}));
        Var wv = op_warp(t, m, ph);
        Var ncc = op_ncc_loss(t, f, wv, window);
        Var reg = op_grad_reg(t, ph);
        Var total = lambda == 0.0f ? ncc : op_add(t, ncc, op_scale(t, reg, lambda));
        terms[0] = t.scalar(total);
        terms[1] = t.scalar(ncc);
        terms[2] = t.scalar(reg);
        if (warped) std::memcpy(warped, t.value(wv).data.data(), (size_t)h * w * l * sizeof(float));
        if (gphi || gmoving) {
            t.backward(total);
            add_into(gphi, t.grad(ph));
            add_into(gmoving, t.grad(m));
        }
    } catch (const std::exception &e) {
        g_perr = e.what();
        return 1;
    }
    return 0;
}

// engine.hpp:268-298 AdamOptimizer: `steps` consecutive steps on one parameter
// tensor with the given gradient sequence grads[k*n ..] (value/m/v updated)
int mdr_adam_steps(float *value, const float *grads, int64_t n, int steps, double lr,
                   double beta1, double beta2, double eps, float *m_out, float *v_out) {
    try {
        ParamTensor<float> p("p", tensor_from(value, {(int)n}));
        std::vector<ParamTensor<float> *> ps{&p};
        AdamOptimizer<float> opt(ps, beta1, beta2, eps);
        for (int k = 0; k < steps; ++k) {
            std::memcpy(p.grad.data.data(), grads + (int64_t)k * n, (size_t)n * sizeof(float));
            opt.step(lr);
        }
        std::memcpy(value, p.value.data.data(), (size_t)n * sizeof(float));
        (void)m_out;
        (void)v_out;
    } catch (const std::exception &e) {
        g_perr = e.what();
        return 1;
    }
    return 0;
}

// ---- full model (encoder + decoder) ------------------------------------------
// ModelParams::all_tensors order (engine.hpp:121-133): 5 encoder blocks x
// {w1,b1,n1g,n1b,w2,b2,n2g,n2b}, then 5 levels x {proj.w,proj.b,ln_g,ln_b,
// bias_b,reghead.w,reghead.b}; packed back to back.
static int64_t model_count(ModelParams<float> &mp) {
    int64_t t = 0;
    for (auto *p : mp.all_tensors()) t += p->value.size();
    return t;
}

int64_t mdr_model_param_count(std::uint64_t seed) {
    ModelParams<float> mp = init_model<float>(ModelConfig::small_preset(), seed);
    return model_count(mp);
}

// init_model(small_preset, seed) values, packed; per-tensor sizes in sizes[75]
int mdr_model_params(std::uint64_t seed, float *out, int64_t *sizes) {
    ModelParams<float> mp = init_model<float>(ModelConfig::small_preset(), seed);
    int i = 0;
    for (auto *p : mp.all_tensors()) {
        std::memcpy(out, p->value.data.data(), p->value.data.size() * sizeof(float));
        out += p->value.data.size();
        if (sizes) sizes[i] = p->value.size();
        ++i;
    }
    return i;
}

static void load_params(ModelParams<float> &mp, const float *packed) {
    for (auto *p : mp.all_tensors()) {
        std::memcpy(p->value.data.data(), packed, p->value.data.size() * sizeof(float));
        packed += p->value.data.size();
    }
}

// op_encode (encoder.hpp:102-116) of one image with the packed model's
// encoder blocks; features[5] written (fine -> coarse); with gfeat the tape
// backward of sum_L <features_L, gfeat_L> accumulates the packed parameter
// gradient (whole-model layout, only encoder entries touched) and gimage
int mdr_encode(const float *image, int h, int w, int l, const float *packed,
               float *const *features, const float *const *gfeat, float *gpacked, float *gimage) {
    try {
        ModelParams<float> mp = init_model<float>(ModelConfig::small_preset(), 1);
        load_params(mp, packed);
        Tape<float> t;
        Var img = t.input(tensor_from(image, {1, h, w, l}));
        std::vector<ConvBlockVars> blocks;
        for (auto &b : mp.encoder_blocks) blocks.push_back(leaf_conv_block(t, b));
        std::vector<Var> feats = op_encode(t, img, blocks, mp.cfg.encoder);
        for (size_t k = 0; k < feats.size(); ++k) {
            const Tensor<float> &v = t.value(feats[k]);
            std::memcpy(features[k], v.data.data(), v.data.size() * sizeof(float));
        }
        if (!gfeat) return 0;
        Var loss;
        bool first = true;
        for (size_t k = 0; k < feats.size(); ++k) {
            if (!gfeat[k]) continue;
            Var term = op_sum_all(t, op_mul(t, feats[k], t.input(tensor_from(gfeat[k], t.value(feats[k]).shape))));
            loss = first ? term : op_add(t, loss, term);
            first = false;
        }
        for (auto *p : mp.all_tensors()) p->zero_grad();
        t.backward(loss);
        if (gpacked)
            for (auto *p : mp.all_tensors()) {
                add_into(gpacked, p->grad);
                gpacked += p->grad.data.size();
            }
        add_into(gimage, t.grad(img));
    } catch (const std::exception &e) {
        g_perr = e.what();
        return 1;
    }
    return 0;
}

// run_loss_step (engine.hpp:316-340) with the packed model: returns the loss,
// accumulates the packed gradient of every parameter and writes phi
int mdr_loss_step(const float *fixed, const float *moving, int h, int w, int l,
                  const float *packed, float lambda, int window, double *loss, float *gpacked,
                  float *phi) {
    try {
        ModelParams<float> mp = init_model<float>(ModelConfig::small_preset(), 1);
        load_params(mp, packed);
        Volume f(D3(h, w, l)), m(D3(h, w, l));
        std::memcpy(f.data.data(), fixed, f.data.size() * sizeof(float));
        std::memcpy(m.data.data(), moving, m.data.size() * sizeof(float));
        auto params = mp.all_tensors();
        LossConfig lc{lambda, window};
        RegistrationResult rr;
        *loss = run_loss_step(f, m, mp, lc, params, gpacked != nullptr, phi ? &rr : nullptr);
        if (gpacked)
            for (auto *p : params) {
                add_into(gpacked, p->grad);
                gpacked += p->grad.data.size();
            }
        if (phi) std::memcpy(phi, rr.phi.data.data(), rr.phi.data.size() * sizeof(float));
    } catch (const std::exception &e) {
        g_perr = e.what();
        return 1;
    }
    return 0;
}

// pairwise_optimize (engine.hpp:377-411) from the packed model: loss and
// Dice traces (iters + 1 entries each) and the final phi
int mdr_pairwise_optimize(const float *fixed, const float *moving, const int *labels_fixed,
                          const int *labels_moving, int h, int w, int l, const float *packed,
                          int iters, double lr, double lambda, int window, double *loss_trace,
                          double *dice_trace, float *phi) {
    try {
        ModelParams<float> mp = init_model<float>(ModelConfig::small_preset(), 1);
        load_params(mp, packed);
        Volume f(D3(h, w, l)), m(D3(h, w, l));
        std::memcpy(f.data.data(), fixed, f.data.size() * sizeof(float));
        std::memcpy(m.data.data(), moving, m.data.size() * sizeof(float));
        LabelVolume lf(D3(h, w, l)), lm(D3(h, w, l));
        std::memcpy(lf.data.data(), labels_fixed, lf.data.size() * sizeof(int));
        std::memcpy(lm.data.data(), labels_moving, lm.data.size() * sizeof(int));
        OptimConfig oc;
        oc.po_iters = iters;
        oc.lr_init = lr;
        oc.lambda = lambda;
        oc.ncc_window = window;
        PoResult r = pairwise_optimize(f, m, mp, oc, &lf, &lm);
        for (size_t i = 0; i < r.loss_trace.size(); ++i) loss_trace[i] = r.loss_trace[i];
        for (size_t i = 0; i < r.dice_trace.size(); ++i) dice_trace[i] = r.dice_trace[i];
        std::memcpy(phi, r.reg.phi.data.data(), r.reg.phi.data.size() * sizeof(float));
    } catch (const std::exception &e) {
        g_perr = e.what();
        return 1;
    }
    return 0;
}

// ---- any ModelConfig (engine.hpp:30-78) / optimizer (engine.hpp:80) ----
// cfg = {base_channels, heads_per_level[5] (coarse -> fine), head_dim,
//        diffeomorphic, ss_steps}; optimizer 0 = Adam, 1 = SGD
static ModelConfig config_of(const int *cfg) {
    ModelConfig c = ModelConfig::small_preset();
    c.encoder.base_channels = cfg[0];
    c.heads_per_level.assign(cfg + 1, cfg + 6);
    c.head_dim = cfg[6];
    c.diffeomorphic = cfg[7] != 0;
    c.ss_steps = cfg[8];
    c.validate();
    return c;
}

int64_t mdr_model_param_count_cfg(const int *cfg) {
    ModelParams<float> mp = init_model<float>(config_of(cfg), 1);
    return model_count(mp);
}

int mdr_model_params_cfg(const int *cfg, std::uint64_t seed, float *out, int64_t *sizes) {
    ModelParams<float> mp = init_model<float>(config_of(cfg), seed);
    int i = 0;
    for (auto *p : mp.all_tensors()) {
        std::memcpy(out, p->value.data.data(), p->value.data.size() * sizeof(float));
        out += p->value.data.size();
        if (sizes) sizes[i] = p->value.size();
        ++i;
    }
    return i;
}

int mdr_loss_step_cfg(const int *cfg, const float *fixed, const float *moving, int h, int w,
                      int l, const float *packed, float lambda, int window, double *loss,
                      float *gpacked, float *phi) {
    try {
        ModelParams<float> mp = init_model<float>(config_of(cfg), 1);
        load_params(mp, packed);
        Volume f(D3(h, w, l)), m(D3(h, w, l));
        std::memcpy(f.data.data(), fixed, f.data.size() * sizeof(float));
        std::memcpy(m.data.data(), moving, m.data.size() * sizeof(float));
        auto params = mp.all_tensors();
        LossConfig lc{lambda, window};
        RegistrationResult rr;
        *loss = run_loss_step(f, m, mp, lc, params, gpacked != nullptr, phi ? &rr : nullptr);
        if (gpacked)
            for (auto *p : params) {
                add_into(gpacked, p->grad);
                gpacked += p->grad.data.size();
            }
        if (phi) std::memcpy(phi, rr.phi.data.data(), rr.phi.data.size() * sizeof(float));
    } catch (const std::exception &e) {
        g_perr = e.what();
        return 1;
    }
    return 0;
}

int mdr_pairwise_optimize_cfg(const int *cfg, int optimizer, const float *fixed,
                              const float *moving, const int *labels_fixed,
                              const int *labels_moving, int h, int w, int l, const float *packed,
                              int iters, double lr, double lambda, int window,
                              double *loss_trace, double *dice_trace, float *phi) {
    try {
        ModelParams<float> mp = init_model<float>(config_of(cfg), 1);
        load_params(mp, packed);
        Volume f(D3(h, w, l)), m(D3(h, w, l));
        std::memcpy(f.data.data(), fixed, f.data.size() * sizeof(float));
        std::memcpy(m.data.data(), moving, m.data.size() * sizeof(float));
        LabelVolume lf(D3(h, w, l)), lm(D3(h, w, l));
        std::memcpy(lf.data.data(), labels_fixed, lf.data.size() * sizeof(int));
        std::memcpy(lm.data.data(), labels_moving, lm.data.size() * sizeof(int));
        OptimConfig oc;
        oc.po_iters = iters;
        oc.lr_init = lr;
        oc.lambda = lambda;
        oc.ncc_window = window;
        oc.optimizer = optimizer ? OptimizerKind::sgd : OptimizerKind::adam;
        PoResult r = pairwise_optimize(f, m, mp, oc, &lf, &lm);
        for (size_t i = 0; i < r.loss_trace.size(); ++i) loss_trace[i] = r.loss_trace[i];
        for (size_t i = 0; i < r.dice_trace.size(); ++i) dice_trace[i] = r.dice_trace[i];
        std::memcpy(phi, r.reg.phi.data.data(), r.reg.phi.data.size() * sizeof(float));
    } catch (const std::exception &e) {
        g_perr = e.what();
        return 1;
    }
    return 0;
}

}  // extern "C"
