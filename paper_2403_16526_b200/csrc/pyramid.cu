// pyramid.cu — the decoding pyramid driver (build_pipeline, engine.hpp:179-219)
// as native host code over the libmdg entry points.
//
// The reference builds a tape per call and allocates every intermediate as a
// fresh tensor.  Here the pyramid object owns one device arena sized at create
// time for the saved activations of every level (phi_up, m_in, planar Q/K, LSE,
// sub-flows, residuals, scaling-squaring states) and the backward scratch, so a
// PO iteration does no allocation and no host synchronisation beyond the
// optional numeric checks.  Q/K are produced directly in the planar layout the
// fused ModeT kernels read (no transposes), W is never materialised, and the
// backward replays the levels fine -> coarse in the reference tape's order.
#include <string>
#include <vector>

#include "mdg_common.cuh"

namespace mdg {

// smallest index of a check whose tensor held a non-finite value
__global__ void nonfinite_seq_k(const float *__restrict__ x, int64_t n, unsigned seq,
                                unsigned *__restrict__ flag) {
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(x[i]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicMin(flag, seq);
}

}  // namespace mdg

using namespace mdg;

#define MDG_TRY(expr)                              \
    do {                                           \
        mdg_status _s = (expr);                    \
        if (_s != MDG_OK) return _s;               \
    } while (0)

struct mdg_pyramid {
    mdg_pyramid_config cfg{};
    struct Level {
        mdg_dims3 d;
        int64_t n;
        int C, S, K;
        float *phi_up, *m_in, *Q, *Kt, *LSE, *SF, *vel, *res, *phi, *ss_saved;
    };
    std::vector<Level> lv;
    // backward scratch, sized for the finest level
    float *g_phi_a = nullptr, *g_phi_b = nullptr, *g_res = nullptr, *g_vel = nullptr,
          *g_sf = nullptr, *g_q = nullptr, *g_k = nullptr, *g_min = nullptr,
          *g_phi_up = nullptr, *g_bias = nullptr;
    unsigned *flag = nullptr;
    void *arena = nullptr;
    int64_t bytes = 0;
    bool have_forward = false;
    std::vector<const float *> f_saved, m_saved;
    std::vector<mdg_level_params> p_saved;
    std::vector<std::string> check_names;
};

namespace {

struct Carve {
    char *base;
    int64_t off = 0;
    float *take(int64_t floats) {
        float *p = reinterpret_cast<float *>(base ? base + off : nullptr);
        off += ((floats * (int64_t)sizeof(float) + 255) / 256) * 256;
        return p;
    }
};

mdg_status validate(const mdg_pyramid_config &c) {
    MDG_REQUIRE(c.levels >= 1 && c.levels <= MDG_MAX_LEVELS,
                "pyramid: levels must be in [1, " + std::to_string(MDG_MAX_LEVELS) + "]");
    // ModelConfig::validate (engine.hpp:64-78)
    for (int k = 0; k < c.levels; ++k) {
        MDG_REQUIRE(c.heads[k] >= 1, "model: head counts must be >= 1");
        MDG_REQUIRE(k == 0 || c.heads[k] <= c.heads[k - 1],
                    "model: head counts must be non-increasing coarse to fine");
        MDG_REQUIRE(c.channels[k] >= 1, "pyramid: feature channels must be >= 1");
        MDG_REQUIRE(dims_ok(c.dims[k]) && nvox(c.dims[k]) > 0,
                    "pyramid: invalid level dims " + dims_str(c.dims[k]));
        if (k > 0) {
            const mdg_dims3 a = c.dims[k - 1], b = c.dims[k];
            // check_upsample_target (sampling.hpp:266-271)
            auto ok = [](int s, int t) { return t >= 2 * s - 1 && t <= 2 * s + 1; };
            MDG_REQUIRE(ok(a.h, b.h) && ok(a.w, b.w) && ok(a.l, b.l),
                        "upsample: target " + dims_str(b) + " is not a doubling of " +
                            dims_str(a));
        }
    }
    MDG_REQUIRE(c.head_dim >= 1, "model: head_dim must be >= 1");
    MDG_REQUIRE(c.neighborhood >= 3 && c.neighborhood % 2 == 1,
                "model: neighborhood must be odd and >= 3");
    MDG_REQUIRE(c.neighborhood == 3, "pyramid: the fused ModeT tier needs neighborhood 3");
    MDG_REQUIRE(c.ss_steps >= 1, "model: ss_steps must be >= 1");
    return MDG_OK;
}

void layout(mdg_pyramid *p, Carve &cv) {
    const mdg_pyramid_config &c = p->cfg;
    p->lv.resize(c.levels);
    int64_t nmax = 0, cmax = 0, kmax = 0, smax = 0;
    for (int k = 0; k < c.levels; ++k) {
        auto &L = p->lv[k];
        L.d = c.dims[k];
        L.n = nvox(L.d);
        L.C = c.channels[k];
        L.S = c.heads[k];
        L.K = L.S * c.head_dim;
        const int64_t n = L.n;
        L.phi_up = k > 0 ? cv.take(3 * n) : nullptr;
        L.m_in = k > 0 ? cv.take((int64_t)L.C * n) : nullptr;
        L.Q = cv.take((int64_t)L.K * n);
        L.Kt = cv.take((int64_t)L.K * n);
        L.LSE = cv.take((int64_t)L.S * n);
        L.SF = cv.take(3 * (int64_t)L.S * n);
        L.vel = c.diffeomorphic ? cv.take(3 * n) : nullptr;
        L.ss_saved = c.diffeomorphic ? cv.take((int64_t)(c.ss_steps + 1) * 3 * n) : nullptr;
        L.res = cv.take(3 * n);
        L.phi = (k > 0 && k < c.levels - 1) ? cv.take(3 * n) : nullptr;
        nmax = std::max(nmax, n);
        cmax = std::max<int64_t>(cmax, (int64_t)L.C * n);
        kmax = std::max<int64_t>(kmax, (int64_t)L.K * n);
        smax = std::max<int64_t>(smax, (int64_t)L.S);
    }
    p->g_phi_a = cv.take(3 * nmax);
    p->g_phi_b = cv.take(3 * nmax);
    p->g_res = cv.take(3 * nmax);
    p->g_vel = c.diffeomorphic ? cv.take(3 * nmax) : nullptr;
    p->g_sf = cv.take(3 * smax * nmax);
    p->g_q = cv.take(kmax);
    p->g_k = cv.take(kmax);
    p->g_min = cv.take(cmax);
    p->g_phi_up = cv.take(3 * nmax);
    p->g_bias = cv.take(smax * 27);
    p->flag = reinterpret_cast<unsigned *>(cv.take(1));
}

mdg_status zero(float *p, int64_t floats, cudaStream_t st) {
    MDG_CUDA_TRY(cudaMemsetAsync(p, 0, (size_t)floats * sizeof(float), st));
    return MDG_OK;
}

mdg_status check_seq(mdg_pyramid *p, const float *x, int64_t n, const std::string &name,
                     cudaStream_t st) {
    if (!x || n == 0) return MDG_OK;
    const unsigned seq = (unsigned)p->check_names.size();
    p->check_names.push_back(name);
    const unsigned blocks = (unsigned)std::min<int64_t>(grid1d(n, 256), 148 * 8);
    nonfinite_seq_k<<<blocks, 256, 0, st>>>(x, n, seq, p->flag);
    MDG_LAUNCHED();
    return MDG_OK;
}

}  // namespace

extern "C" {

mdg_status mdg_pyramid_create(const mdg_pyramid_config *cfg, mdg_pyramid **out) {
    MDG_REQUIRE(cfg && out, "pyramid: null pointer");
    *out = nullptr;
    MDG_TRY(validate(*cfg));
    mdg_pyramid *p = new mdg_pyramid;
    p->cfg = *cfg;
    Carve dry{nullptr};
    layout(p, dry);
    p->bytes = dry.off;
    void *mem = nullptr;
    cudaError_t e = cudaMalloc(&mem, (size_t)p->bytes);
    if (e != cudaSuccess) {
        delete p;
        return status_from_cuda(e, "pyramid arena");
    }
    p->arena = mem;
    Carve cv{reinterpret_cast<char *>(mem)};
    layout(p, cv);
    *out = p;
    return MDG_OK;
}

void mdg_pyramid_destroy(mdg_pyramid *p) {
    if (!p) return;
    if (p->arena) cudaFree(p->arena);
    delete p;
}

int64_t mdg_pyramid_bytes(const mdg_pyramid *p) { return p ? p->bytes : 0; }

mdg_status mdg_pyramid_forward(mdg_pyramid *p, const float *const *f_feats,
                               const float *const *m_feats, const mdg_level_params *params,
                               float *phi, float *const *residuals, void *stream) {
    MDG_REQUIRE(p && f_feats && m_feats && params && phi, "pyramid: null pointer");
    const mdg_pyramid_config &c = p->cfg;
    cudaStream_t st = S_(stream);
    p->have_forward = false;
    p->f_saved.assign(f_feats, f_feats + c.levels);
    p->m_saved.assign(m_feats, m_feats + c.levels);
    p->p_saved.assign(params, params + c.levels);
    for (int k = 0; k < c.levels; ++k) {
        auto &L = p->lv[k];
        const mdg_level_params &P = params[k];
        MDG_REQUIRE(f_feats[k] && m_feats[k], "pyramid: null feature map");
        MDG_REQUIRE(P.proj_w && P.proj_b && P.ln_g && P.ln_b && P.rel_bias && P.rh_w && P.rh_b,
                    "pyramid: null level parameter");
        const float *m_in = m_feats[k];
        if (k > 0) {
            const auto &Lp = p->lv[k - 1];
            const float *phi_prev = (k - 1 == 0) ? Lp.res : Lp.phi;
            MDG_TRY(mdg_upsample2_fwd(phi_prev, 3, Lp.d, L.d, 2.0f, L.phi_up, st));
            MDG_TRY(mdg_warp_fwd(m_feats[k], L.C, L.d, L.phi_up, L.m_in, st));
            m_in = L.m_in;
        }
        MDG_TRY(mdg_project_qk_fwd(f_feats[k], m_in, L.C, L.n, P.proj_w, P.proj_b, P.ln_g,
                                   P.ln_b, L.K, MDG_QK_PLANAR, L.Q, L.Kt, st));
        MDG_TRY(mdg_modet_fwd(L.Q, L.Kt, P.rel_bias, L.d, L.S, c.head_dim, c.neighborhood,
                              MDG_QK_PLANAR, L.SF, L.LSE, nullptr, st));
        if (c.check_finite) MDG_TRY(mdg_check_numeric(L.d, st));
        float *rh_out = c.diffeomorphic ? L.vel : L.res;
        // RegHead conv on the encoder's FMA-contracted kernels (TMA slab /
        // implicit GEMM): the fused tier's parity is tolerance-based, the
        // bit-exact reference-order kernel stays behind mdg_conv3_fwd
        MDG_TRY(enc_conv3_fwd(L.SF, 3 * L.S, L.d, P.rh_w, P.rh_b, 3, rh_out, st));
        if (c.diffeomorphic)
            MDG_TRY(mdg_scaling_squaring_fwd(L.vel, L.d, c.ss_steps, L.res, L.ss_saved, st));
        float *phi_k = (k == c.levels - 1) ? phi : (k == 0 ? L.res : L.phi);
        if (k > 0) MDG_TRY(mdg_compose_fwd(L.phi_up, L.res, L.d, phi_k, st));
        else if (c.levels == 1)
            MDG_CUDA_TRY(cudaMemcpyAsync(phi, L.res, 3 * L.n * sizeof(float),
                                         cudaMemcpyDeviceToDevice, st));
        if (residuals && residuals[k])
            MDG_CUDA_TRY(cudaMemcpyAsync(residuals[k], L.res, 3 * L.n * sizeof(float),
                                         cudaMemcpyDeviceToDevice, st));
    }
    p->have_forward = true;
    return MDG_OK;
}

mdg_status mdg_pyramid_backward(mdg_pyramid *p, const float *gphi, const mdg_level_grads *grads,
                                float *const *gf, float *const *gm, void *stream) {
    MDG_REQUIRE(p && gphi, "pyramid: null pointer");
    MDG_REQUIRE(p->have_forward, "pyramid: backward without a forward");
    const mdg_pyramid_config &c = p->cfg;
    cudaStream_t st = S_(stream);
    p->check_names.clear();
    if (c.check_finite)
        MDG_CUDA_TRY(cudaMemsetAsync(p->flag, 0xff, sizeof(unsigned), st));

    const float *g_phi = gphi;  // dloss/dphi on the current level grid
    float *g_next = p->g_phi_a;
    for (int k = c.levels - 1; k >= 0; --k) {
        auto &L = p->lv[k];
        const mdg_level_params &P = p->p_saved[k];
        const mdg_level_grads *G = grads ? &grads[k] : nullptr;
        const std::string tag = "lvl" + std::to_string(k) + ".";
        if (c.check_finite) MDG_TRY(check_seq(p, g_phi, 3 * L.n, tag + "compose", st));

        // phi = compose(phi_up, res) or res (engine.hpp:214)
        const float *g_res = g_phi;
        if (k > 0) {
            MDG_TRY(zero(p->g_res, 3 * L.n, st));
            MDG_TRY(zero(p->g_phi_up, 3 * L.n, st));
            MDG_TRY(mdg_compose_bwd(L.phi_up, L.res, L.d, g_phi, p->g_phi_up, p->g_res, st));
            g_res = p->g_res;
        }
        if (c.check_finite)
            MDG_TRY(check_seq(p, g_res, 3 * L.n,
                              tag + (c.diffeomorphic ? "scaling_squaring" : "reghead"), st));
        const float *g_rh = g_res;
        if (c.diffeomorphic) {
            MDG_TRY(zero(p->g_vel, 3 * L.n, st));
            MDG_TRY(mdg_scaling_squaring_bwd(L.ss_saved, L.d, c.ss_steps, g_res, p->g_vel, st));
            g_rh = p->g_vel;
        }
        // RegHead (reghead.hpp:42-47)
        MDG_TRY(enc_conv3_bwd(L.SF, 3 * L.S, L.d, P.rh_w, 3, g_rh, p->g_sf,
                              G ? G->rh_w : nullptr, G ? G->rh_b : nullptr, st,
                              /*gin_acc=*/false));
        if (c.check_finite)
            MDG_TRY(check_seq(p, p->g_sf, 3 * (int64_t)L.S * L.n, tag + "subfields", st));
        // ModeT (fused na_fused + subfields backward); gQ/gK overwritten
        float *gB = (G && G->rel_bias) ? G->rel_bias : p->g_bias;
        MDG_TRY(mdg_modet_bwd(L.Q, L.Kt, P.rel_bias, L.SF, L.LSE, p->g_sf, L.d, L.S, c.head_dim,
                              c.neighborhood, MDG_QK_PLANAR, p->g_q, p->g_k, gB, 0, st));
        // projection: K came from m_in (warped moving features) for k > 0
        const float *m_in = k > 0 ? L.m_in : p->m_saved[k];
        // the warped-moving gradient of k > 0 is an internal buffer: written,
        // not accumulated (saves its memset and read)
        float *g_min = k > 0 ? p->g_min : (gm ? gm[k] : nullptr);
        MDG_TRY(project_qk_bwd_impl(p->f_saved[k], m_in, L.C, L.n, P.proj_w, P.proj_b, P.ln_g,
                                    L.K, MDG_QK_PLANAR, p->g_q, p->g_k, gf ? gf[k] : nullptr,
                                    g_min, G ? G->proj_w : nullptr, G ? G->proj_b : nullptr,
                                    G ? G->ln_g : nullptr, G ? G->ln_b : nullptr,
                                    k > 0 ? 2 : 0, st));
        if (k > 0) {
            if (c.check_finite)
                MDG_TRY(check_seq(p, p->g_min, (int64_t)L.C * L.n, tag + "warp", st));
            // m_in = warp(m, phi_up): gradients to m and to phi_up
            MDG_TRY(mdg_warp_bwd(p->m_saved[k], L.C, L.d, L.phi_up, p->g_min,
                                 gm ? gm[k] : nullptr, p->g_phi_up, st));
            if (c.check_finite)
                MDG_TRY(check_seq(p, p->g_phi_up, 3 * L.n, tag + "upsample_field_2x", st));
            // phi_up = upsample_field_2x(phi_{k-1})
            const auto &Lp = p->lv[k - 1];
            MDG_TRY(zero(g_next, 3 * Lp.n, st));
            MDG_TRY(mdg_upsample2_bwd(3, Lp.d, L.d, 2.0f, p->g_phi_up, g_next, st));
            g_phi = g_next;
            g_next = (g_next == p->g_phi_a) ? p->g_phi_b : p->g_phi_a;
        }
    }
    if (c.check_finite) {
        // parameter leaves and feature inputs (tape.hpp:116-120 checks every node)
        for (int k = c.levels - 1; k >= 0 && grads; --k) {
            const auto &L = p->lv[k];
            const mdg_level_grads &G = grads[k];
            const std::string tag = "lvl" + std::to_string(k) + ".";
            MDG_TRY(check_seq(p, G.proj_w, (int64_t)L.K * L.C, tag + "proj.w", st));
            MDG_TRY(check_seq(p, G.proj_b, L.K, tag + "proj.b", st));
            MDG_TRY(check_seq(p, G.ln_g, L.K, tag + "proj.ln_g", st));
            MDG_TRY(check_seq(p, G.ln_b, L.K, tag + "proj.ln_b", st));
            MDG_TRY(check_seq(p, G.rel_bias, (int64_t)L.S * 27, tag + "bias_b", st));
            MDG_TRY(check_seq(p, G.rh_w, 3 * 3 * (int64_t)L.S * 27, tag + "reghead.w", st));
            MDG_TRY(check_seq(p, G.rh_b, 3, tag + "reghead.b", st));
        }
        unsigned seq = ~0u;
        MDG_CUDA_TRY(cudaMemcpyAsync(&seq, p->flag, sizeof(seq), cudaMemcpyDeviceToHost, st));
        MDG_CUDA_TRY(cudaStreamSynchronize(st));
        if (seq != ~0u && seq < p->check_names.size()) {
            set_error(MDG_ENUMERIC,
                      "non-finite gradient at op '" + p->check_names[seq] + "'");
            return MDG_ENUMERIC;
        }
    }
    return MDG_OK;
}

}  // extern "C"
