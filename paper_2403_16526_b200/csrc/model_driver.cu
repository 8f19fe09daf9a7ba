// model_driver.cu — the whole registration model as one native object:
// run_loss_step (engine.hpp:316-340) and pairwise_optimize's update
// (engine.hpp:389-398) composed from the encoder, pyramid, loss and Adam entry
// points, with no framework underneath: parameters, gradients, Adam moments
// and every intermediate live in device memory owned by the object or the
// caller; one stream; the loss is the only value read back (on request).
//
// Parameters follow ModelParams::all_tensors (engine.hpp:121-133): five
// encoder blocks {w1,b1,n1g,n1b,w2,b2,n2g,n2b}, then five decoder levels,
// coarse -> fine, {proj.w,proj.b,ln_g,ln_b,bias_b,reghead.w,reghead.b}.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "mdg_common.cuh"

using namespace mdg;

namespace {
__global__ void add_k(float *__restrict__ dst, const float *__restrict__ src, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] += src[i];
}
}  // namespace

#define MD_TRY(expr)                      \
    do {                                  \
        mdg_status _s = (expr);           \
        if (_s != MDG_OK) return _s;      \
    } while (0)

struct mdg_model {
    mdg_model_config cfg{};
    int optimizer = MDG_OPT_ADAM;
    mdg_dims3 d;
    int64_t n = 0;
    float lambda = 1.0f;
    int window = 9;
    std::vector<float *> params;    // 75, caller-owned
    std::vector<int64_t> sizes;     // elements per tensor
    std::vector<float *> grads, m, v;  // owned (one arena)
    std::vector<float *> grads_mv;     // the moving-image encoder's own gradients
    float *grads_base = nullptr, *grads_mv_base = nullptr;
    int64_t grads_len = 0, enc_len = 0;  // padded floats: all grads / encoder part
    void *arena = nullptr;
    cudaStream_t s2 = nullptr;           // second stream: the moving-image encoder
    cudaEvent_t ev[4] = {};
    // Adam's step count lives on the device (graph replays); bias
    // corrections 1 - beta^t come from a host-computed table (std::pow)
    int64_t *d_t = nullptr;
    double *d_bc = nullptr;
    int64_t tmax = 0;
    // CUDA graph of one PO iteration (mdg_model_po_step) and its key
    cudaGraphExec_t gexec = nullptr;
    const float *g_fixed = nullptr, *g_moving = nullptr;
    float *g_terms = nullptr;
    double g_lr = 0.0;
    cudaStream_t g_stream = nullptr;
    int64_t g_tmax = 0;
    bool graph_off = false;
    // key of the previous call: capture only on the second consecutive call
    // with the same key (the first runs eagerly and initialises lazily
    // allocated device state, which must not happen inside a capture)
    const float *k_fixed = nullptr, *k_moving = nullptr;
    float *k_terms = nullptr;
    double k_lr = -1.0;
    cudaStream_t k_stream = nullptr;
    mdg_encoder *enc_f = nullptr, *enc_m = nullptr;
    mdg_pyramid *pyr = nullptr;
    std::vector<float *> ff, mf, gf, gm;  // features / their gradients (fine -> coarse)
    float *phi = nullptr, *gphi = nullptr, *terms = nullptr;
    int64_t t = 0;
    double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
};

namespace {
constexpr int kLevels = MDG_ENC_LEVELS;

// ModelParams::all_tensors element counts of a config (io.cpp layout_of)
std::vector<int64_t> model_sizes(const mdg_model_config &c) {
    int nt = 0;
    mdg_config_param_count(&c, &nt, nullptr);
    std::vector<int64_t> s((size_t)nt);
    mdg_config_param_count(&c, &nt, s.data());
    return s;
}

mdg_model_config small_preset() {
    mdg_model_config c{};
    mdg_model_config_small_preset(&c);
    return c;
}

mdg_status check_config(const mdg_model_config &c) {
    // ModelConfig::validate (engine.hpp:62-76)
    MDG_REQUIRE(c.base_channels >= 1, "encoder: base_channels must be >= 1");
    for (int k = 0; k < kLevels; ++k) {
        MDG_REQUIRE(c.heads_per_level[k] >= 1, "model: head counts must be >= 1");
        MDG_REQUIRE(k == 0 || c.heads_per_level[k] <= c.heads_per_level[k - 1],
                    "model: head counts must be non-increasing coarse to fine");
    }
    MDG_REQUIRE(c.head_dim >= 1, "model: head_dim must be >= 1");
    MDG_REQUIRE(c.neighborhood == 3, "model: the B200 pyramid runs neighborhood 3");
    MDG_REQUIRE(c.ss_steps >= 1, "model: ss_steps must be >= 1");
    return MDG_OK;
}
}  // namespace

extern "C" {

int64_t mdg_model_param_count(int *ntensors, int64_t *sizes) {
    const mdg_model_config c = small_preset();
    return mdg_config_param_count(&c, ntensors, sizes);
}

mdg_status mdg_model_init_cfg(const mdg_model_config *cfg, uint64_t seed,
                              float *const *params_host) {
    // init_model(cfg, seed) (engine.hpp:143-166) on host buffers, drawn from
    // the reference Rng stream in the reference order
    MDG_REQUIRE(cfg && params_host, "model: null pointer");
    if (mdg_status e = check_config(*cfg)) return e;
    const auto s = model_sizes(*cfg);
    const int base = cfg->base_channels;
    mdg_rng *r = mdg_rng_new(seed);
    int i = 0;
    for (int k = 0; k < kLevels; ++k) {
        const int c = base << k, cin = k == 0 ? 1 : base << (k - 1);
        const double b1 = std::sqrt(6.0 / (cin * 27.0)), b2 = std::sqrt(6.0 / (c * 27.0));
        mdg_rng_fill_uniform(r, params_host[i], s[i], -b1, b1);
        for (int j = 1; j < 4; ++j)
            for (int64_t e = 0; e < s[i + j]; ++e) params_host[i + j][e] = j == 2 ? 1.0f : 0.0f;
        mdg_rng_fill_uniform(r, params_host[i + 4], s[i + 4], -b2, b2);
        for (int j = 5; j < 8; ++j)
            for (int64_t e = 0; e < s[i + j]; ++e) params_host[i + j][e] = j == 6 ? 1.0f : 0.0f;
        i += 8;
    }
    for (int k = 0; k < kLevels; ++k) {
        mdg_rng_fill_normal(r, params_host[i], s[i], 0.0, 1e-5);
        for (int j = 1; j < 5; ++j)
            for (int64_t e = 0; e < s[i + j]; ++e) params_host[i + j][e] = j == 2 ? 1.0f : 0.0f;
        mdg_rng_fill_normal(r, params_host[i + 5], s[i + 5], 0.0, 1e-5);
        for (int64_t e = 0; e < s[i + 6]; ++e) params_host[i + 6][e] = 0.0f;
        i += 7;
    }
    mdg_rng_free(r);
    return MDG_OK;
}

mdg_status mdg_model_init(uint64_t seed, float *const *params_host) {
    const mdg_model_config c = small_preset();
    return mdg_model_init_cfg(&c, seed, params_host);
}

mdg_status mdg_model_create_cfg(const mdg_model_config *cfg, mdg_dims3 d, float *const *params,
                                float lambda, int ncc_window, int check_finite, int optimizer,
                                mdg_model **out) {
    MDG_REQUIRE(cfg && params && out, "model: null pointer");
    *out = nullptr;
    if (mdg_status e = check_config(*cfg)) return e;
    MDG_REQUIRE(lambda >= 0.0f, "loss: lambda must be >= 0");
    MDG_REQUIRE(ncc_window >= 3 && ncc_window % 2 == 1, "loss: ncc_window must be odd and >= 3");
    MDG_REQUIRE(optimizer == MDG_OPT_ADAM || optimizer == MDG_OPT_SGD, "model: unknown optimizer");
    mdg_model *m = new mdg_model;
    m->cfg = *cfg;
    m->optimizer = optimizer;
    m->d = d;
    m->n = nvox(d);
    m->lambda = lambda;
    m->window = ncc_window;
    m->sizes = model_sizes(*cfg);
    m->params.assign(params, params + m->sizes.size());
    auto fail = [&](mdg_status st) {
        mdg_model_destroy(m);
        return st;
    };
    const int base = cfg->base_channels;
    mdg_status st = mdg_encoder_create(d, base, kLevels, cfg->leaky_slope, &m->enc_f);
    if (st == MDG_OK) st = mdg_encoder_create(d, base, kLevels, cfg->leaky_slope, &m->enc_m);
    if (st != MDG_OK) return fail(st);
    mdg_pyramid_config pc{};
    pc.levels = kLevels;
    std::vector<mdg_dims3> dims{d};
    for (int k = 1; k < kLevels; ++k) {
        const mdg_dims3 p = dims.back();
        dims.push_back(mdg_dims3{(p.h + 1) / 2, (p.w + 1) / 2, (p.l + 1) / 2});
    }
    for (int k = 0; k < kLevels; ++k) {  // coarse -> fine
        pc.heads[k] = cfg->heads_per_level[k];
        pc.channels[k] = base << (kLevels - 1 - k);
        pc.dims[k] = dims[kLevels - 1 - k];
    }
    pc.head_dim = cfg->head_dim;
    pc.neighborhood = cfg->neighborhood;
    pc.diffeomorphic = cfg->diffeomorphic;
    pc.ss_steps = cfg->ss_steps;
    pc.check_finite = check_finite;
    if ((st = mdg_pyramid_create(&pc, &m->pyr)) != MDG_OK) return fail(st);
    // arena: grads | moving-encoder grads | Adam moments | features + their
    // grads | phi/gphi/terms.  Tensors padded to 64 floats; the padding stays
    // zero, so the gradient blocks can be cleared and summed as flat ranges.
    int64_t tot = 0, enc = 0;
    for (size_t i = 0; i < m->sizes.size(); ++i) {
        const int64_t pad = (m->sizes[i] + 63) / 64 * 64;
        tot += pad;
        if (i < 40) enc += pad;
    }
    m->grads_len = tot;
    m->enc_len = enc;
    int64_t feat = 0;
    for (int k = 0; k < kLevels; ++k) feat += (int64_t)(base << k) * nvox(dims[k]) + 64;
    const size_t bytes =
        ((size_t)3 * tot + enc + 4 * (size_t)feat + 6 * (size_t)m->n + 64) * sizeof(float);
    cudaError_t e = cudaMalloc(&m->arena, bytes);
    if (e != cudaSuccess) return fail(status_from_cuda(e, "model arena"));
    cudaMemset(m->arena, 0, bytes);
    if ((e = cudaStreamCreateWithFlags(&m->s2, cudaStreamNonBlocking)) != cudaSuccess)
        return fail(status_from_cuda(e, "model stream"));
    for (auto &ev : m->ev)
        if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
            return fail(status_from_cuda(e, "model events"));
    if ((e = cudaMalloc(&m->d_t, sizeof(int64_t))) != cudaSuccess)
        return fail(status_from_cuda(e, "model step counter"));
    cudaMemset(m->d_t, 0, sizeof(int64_t));
    float *p = static_cast<float *>(m->arena);
    m->grads_base = p;
    for (int64_t sz : m->sizes) {
        m->grads.push_back(p);
        p += (sz + 63) / 64 * 64;
    }
    m->grads_mv_base = p;
    for (int i = 0; i < 40; ++i) {
        m->grads_mv.push_back(p);
        p += (m->sizes[i] + 63) / 64 * 64;
    }
    for (auto *vec : {&m->m, &m->v})
        for (int64_t sz : m->sizes) {
            vec->push_back(p);
            p += (sz + 63) / 64 * 64;
        }
    for (auto *vec : {&m->ff, &m->mf, &m->gf, &m->gm})
        for (int k = 0; k < kLevels; ++k) {
            vec->push_back(p);
            p += (int64_t)(base << k) * nvox(dims[k]) + 64;
        }
    m->phi = p;
    p += 3 * m->n;
    m->gphi = p;
    p += 3 * m->n;
    m->terms = p;
    *out = m;
    return MDG_OK;
}

mdg_status mdg_model_create(mdg_dims3 d, float *const *params, float lambda, int ncc_window,
                            int check_finite, mdg_model **out) {
    const mdg_model_config c = small_preset();
    return mdg_model_create_cfg(&c, d, params, lambda, ncc_window, check_finite, MDG_OPT_ADAM,
                                out);
}

void mdg_model_destroy(mdg_model *m) {
    if (!m) return;
    if (m->enc_f) mdg_encoder_destroy(m->enc_f);
    if (m->enc_m) mdg_encoder_destroy(m->enc_m);
    if (m->pyr) mdg_pyramid_destroy(m->pyr);
    if (m->arena) cudaFree(m->arena);
    if (m->s2) cudaStreamDestroy(m->s2);
    if (m->gexec) cudaGraphExecDestroy(m->gexec);
    if (m->d_t) cudaFree(m->d_t);
    if (m->d_bc) cudaFree(m->d_bc);
    for (auto ev : m->ev)
        if (ev) cudaEventDestroy(ev);
    delete m;
}

float *const *mdg_model_grads(mdg_model *m) { return m ? m->grads.data() : nullptr; }
const float *mdg_model_phi(const mdg_model *m) { return m ? m->phi : nullptr; }

mdg_status mdg_model_loss_step(mdg_model *m, const float *fixed, const float *moving,
                               int backward, float *terms, float *phi, void *stream) {
    MDG_REQUIRE(m && fixed && moving, "model: null pointer");
    cudaStream_t st = S_(stream);
    std::vector<mdg_block_params> bp(kLevels);
    std::vector<mdg_block_grads> bg(kLevels);
    std::vector<mdg_level_params> lp(kLevels);
    std::vector<mdg_level_grads> lg(kLevels);
    for (int k = 0; k < kLevels; ++k) {
        float *const *P = m->params.data() + 8 * k;
        float *const *G = m->grads.data() + 8 * k;
        bp[k] = mdg_block_params{P[0], P[1], P[2], P[3], P[4], P[5], P[6], P[7]};
        bg[k] = mdg_block_grads{G[0], G[1], G[2], G[3], G[4], G[5], G[6], G[7]};
        float *const *Q = m->params.data() + 40 + 7 * k;
        float *const *H = m->grads.data() + 40 + 7 * k;
        lp[k] = mdg_level_params{Q[0], Q[1], Q[2], Q[3], Q[4], Q[5], Q[6]};
        lg[k] = mdg_level_grads{H[0], H[1], H[2], H[3], H[4], H[5], H[6]};
    }
    std::vector<mdg_block_grads> bgm(kLevels);
    for (int k = 0; k < kLevels; ++k) {
        float *const *G = m->grads_mv.data() + 8 * k;
        bgm[k] = mdg_block_grads{G[0], G[1], G[2], G[3], G[4], G[5], G[6], G[7]};
    }
    // run_loss_step: encoder x2 (concurrently: the moving image's on a second
    // stream) -> pyramid (coarse -> fine) -> loss
    MDG_CUDA_TRY(cudaEventRecord(m->ev[0], st));
    MDG_CUDA_TRY(cudaStreamWaitEvent(m->s2, m->ev[0], 0));
    MD_TRY(mdg_encoder_forward(m->enc_m, moving, bp.data(), m->mf.data(), m->s2));
    MD_TRY(mdg_encoder_forward(m->enc_f, fixed, bp.data(), m->ff.data(), st));
    MDG_CUDA_TRY(cudaEventRecord(m->ev[1], m->s2));
    MDG_CUDA_TRY(cudaStreamWaitEvent(st, m->ev[1], 0));
    std::vector<const float *> fc(kLevels), mc(kLevels);
    for (int k = 0; k < kLevels; ++k) {
        fc[k] = m->ff[kLevels - 1 - k];
        mc[k] = m->mf[kLevels - 1 - k];
    }
    MD_TRY(mdg_pyramid_forward(m->pyr, fc.data(), mc.data(), lp.data(), m->phi, nullptr, st));
    MD_TRY(mdg_total_loss_fwd(fixed, moving, m->phi, m->d, m->window, m->lambda, m->terms,
                              nullptr, st));
    if (terms)
        MDG_CUDA_TRY(cudaMemcpyAsync(terms, m->terms, 3 * sizeof(float), cudaMemcpyDeviceToDevice, st));
    if (phi)
        MDG_CUDA_TRY(cudaMemcpyAsync(phi, m->phi, 3 * m->n * sizeof(float), cudaMemcpyDeviceToDevice, st));
    if (!backward) return MDG_OK;
    // zero_grads + tape backward (engine.hpp:332-334)
    MDG_CUDA_TRY(cudaMemsetAsync(m->grads_base, 0,
                                 (size_t)(m->grads_len + m->enc_len) * sizeof(float), st));
    MDG_CUDA_TRY(cudaMemsetAsync(m->gphi, 0, 3 * m->n * sizeof(float), st));
    MD_TRY(mdg_total_loss_bwd(fixed, moving, m->phi, m->d, m->window, m->lambda, 1.0f, m->gphi,
                              nullptr, st));
    std::vector<float *> gfc(kLevels), gmc(kLevels);
    for (int k = 0; k < kLevels; ++k) {
        gfc[k] = m->gf[kLevels - 1 - k];
        gmc[k] = m->gm[kLevels - 1 - k];
    }
    // feature gradients accumulate: clear them first
    {
        mdg_dims3 dk = m->d;
        for (int k = 0; k < kLevels; ++k) {
            const size_t bytes = (size_t)(m->cfg.base_channels << k) * nvox(dk) * sizeof(float);
            MDG_CUDA_TRY(cudaMemsetAsync(m->gf[k], 0, bytes, st));
            MDG_CUDA_TRY(cudaMemsetAsync(m->gm[k], 0, bytes, st));
            dk = mdg_dims3{(dk.h + 1) / 2, (dk.w + 1) / 2, (dk.l + 1) / 2};
        }
    }
    MD_TRY(mdg_pyramid_backward(m->pyr, m->gphi, lg.data(), gfc.data(), gmc.data(), st));
    // both encoders' backward concurrently; the moving one into its own
    // gradient block, summed into the shared weights' gradients after the join
    MDG_CUDA_TRY(cudaEventRecord(m->ev[2], st));
    MDG_CUDA_TRY(cudaStreamWaitEvent(m->s2, m->ev[2], 0));
    std::vector<const float *> gfe(m->gf.begin(), m->gf.end()), gme(m->gm.begin(), m->gm.end());
    MD_TRY(mdg_encoder_backward(m->enc_m, gme.data(), bgm.data(), nullptr, m->s2));
    MD_TRY(mdg_encoder_backward(m->enc_f, gfe.data(), bg.data(), nullptr, st));
    MDG_CUDA_TRY(cudaEventRecord(m->ev[3], m->s2));
    MDG_CUDA_TRY(cudaStreamWaitEvent(st, m->ev[3], 0));
    add_k<<<(unsigned)std::min<int64_t>((m->enc_len + 255) / 256, 148 * 4), 256, 0, st>>>(
        m->grads_base, m->grads_mv_base, m->enc_len);
    MDG_LAUNCHED();
    return MDG_OK;
}

// grow the bias-correction table to cover step t (AdamOptimizer::step,
// engine.hpp:281-282: bc = 1 - beta^t in double with std::pow)
static mdg_status ensure_bc(mdg_model *m, int64_t t) {
    if (t <= m->tmax && m->d_bc) return MDG_OK;
    int64_t cap = std::max<int64_t>(1024, m->tmax);
    while (cap < t) cap *= 2;
    std::vector<double> bc(2 * (size_t)cap);
    for (int64_t i = 1; i <= cap; ++i) {
        bc[2 * (i - 1)] = 1.0 - std::pow(m->beta1, (double)i);
        bc[2 * (i - 1) + 1] = 1.0 - std::pow(m->beta2, (double)i);
    }
    double *nb = nullptr;
    MDG_CUDA_TRY(cudaMalloc(&nb, bc.size() * sizeof(double)));
    MDG_CUDA_TRY(cudaMemcpy(nb, bc.data(), bc.size() * sizeof(double), cudaMemcpyHostToDevice));
    if (m->d_bc) {
        cudaDeviceSynchronize();
        cudaFree(m->d_bc);
    }
    m->d_bc = nb;
    m->tmax = cap;
    return MDG_OK;
}

static AdamList adam_list(const mdg_model *m) {
    AdamList L{};
    L.count = (int)m->params.size();
    for (int i = 0; i < L.count; ++i)
        L.t[i] = AdamTensor{m->params[i], m->grads[i], m->m[i], m->v[i], m->sizes[i]};
    return L;
}

// sgd_step (engine.hpp:306-311) over every tensor
static mdg_status sgd_all(mdg_model *m, double lr, cudaStream_t st) {
    for (size_t i = 0; i < m->params.size(); ++i)
        MD_TRY(mdg_sgd_step(m->params[i], m->grads[i], m->sizes[i], lr, st));
    return MDG_OK;
}

// the configured optimizer's update (graph-capturable: no host reads)
static mdg_status update(mdg_model *m, double lr, cudaStream_t st) {
    if (m->optimizer == MDG_OPT_SGD) return sgd_all(m, lr, st);
    return adam_multi_dev(adam_list(m), lr, m->beta1, m->beta2, m->eps, m->d_t, m->d_bc, st);
}

mdg_status mdg_model_adam_step(mdg_model *m, double lr, void *stream) {
    MDG_REQUIRE(m, "model: null pointer");
    ++m->t;
    MD_TRY(ensure_bc(m, m->t));
    return update(m, lr, S_(stream));
}

// One PO iteration (run_loss_step + AdamOptimizer::step, engine.hpp:389-398)
// replayed from a CUDA graph: the ~430 launches of both streams are captured
// once and re-launched as one graph while the inputs, outputs, lr and stream
// stay the same (the step count is device-side, so replays need no host
// writes).  A capture failure falls back to eager launches of the same work.
mdg_status mdg_model_po_step(mdg_model *m, const float *fixed, const float *moving, double lr,
                             float *terms, void *stream) {
    MDG_REQUIRE(m && fixed && moving, "model: null pointer");
    cudaStream_t st = S_(stream);
    const int64_t t = m->t + 1;
    MD_TRY(ensure_bc(m, t + 1024));  // table headroom: no re-capture for a while
    const bool same = m->gexec && fixed == m->g_fixed && moving == m->g_moving &&
                      terms == m->g_terms && lr == m->g_lr && st == m->g_stream &&
                      m->tmax == m->g_tmax;
    if (std::getenv("MDG_GRAPH_TRACE"))
        std::fprintf(stderr, "po_step t=%lld gexec=%d same=%d off=%d keys %d%d%d%d%d%d\n",
                     (long long)t, m->gexec != nullptr, same, m->graph_off, fixed == m->g_fixed,
                     moving == m->g_moving, terms == m->g_terms, lr == m->g_lr,
                     st == m->g_stream, m->tmax == m->g_tmax);
    const bool repeat = fixed == m->k_fixed && moving == m->k_moving && terms == m->k_terms &&
                        lr == m->k_lr && st == m->k_stream;
    m->k_fixed = fixed;
    m->k_moving = moving;
    m->k_terms = terms;
    m->k_lr = lr;
    m->k_stream = st;
    if (!same && repeat && !m->graph_off) {
        if (m->gexec) cudaGraphExecDestroy(m->gexec);
        m->gexec = nullptr;
        cudaGraph_t g = nullptr;
        bool ok = cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed) == cudaSuccess;
        if (ok) {
            const mdg_status s1 = mdg_model_loss_step(m, fixed, moving, 1, terms, nullptr, st);
            const mdg_status s2 = s1 == MDG_OK ? update(m, lr, st) : s1;
            const cudaError_t e = cudaStreamEndCapture(st, &g);
            const cudaError_t ei = (s2 == MDG_OK && e == cudaSuccess && g)
                                       ? cudaGraphInstantiate(&m->gexec, g, 0)
                                       : cudaErrorUnknown;
            ok = ei == cudaSuccess;
            if (std::getenv("MDG_GRAPH_TRACE"))
                std::fprintf(stderr, "capture: loss=%d adam=%d end=%s inst=%s last=%s msg=%s\n",
                             (int)s1, (int)s2, cudaGetErrorString(e), cudaGetErrorString(ei),
                             cudaGetErrorString(cudaPeekAtLastError()), mdg_last_error());
            if (g) cudaGraphDestroy(g);
        }
        if (!ok) {
            cudaGetLastError();  // clear the capture error; run eagerly from now on
            if (m->gexec) cudaGraphExecDestroy(m->gexec);
            m->gexec = nullptr;
            m->graph_off = true;
        } else {
            m->g_fixed = fixed;
            m->g_moving = moving;
            m->g_terms = terms;
            m->g_lr = lr;
            m->g_stream = st;
            m->g_tmax = m->tmax;
        }
    }
    ++m->t;
    if (m->gexec && (same || repeat)) {
        MDG_CUDA_TRY(cudaGraphLaunch(m->gexec, st));
        return MDG_OK;
    }
    MD_TRY(mdg_model_loss_step(m, fixed, moving, 1, terms, nullptr, st));
    return update(m, lr, st);
}

}  // extern "C"
