// encoder_driver.cu — op_encode (encoder.hpp:102-116) as native host code
// over the encoder kernels: a device arena per encoder object holds every
// level's saved activations (conv outputs, InstanceNorm statistics, pooled
// inputs); the backward replays the tape order of the reference (coarse level
// first; the pooling backward feeds the finer level's feature gradient).
#include <algorithm>
#include <vector>

#include "mdg_common.cuh"

using namespace mdg;

#define ENC_TRY(expr)                      \
    do {                                   \
        mdg_status _s = (expr);            \
        if (_s != MDG_OK) return _s;       \
    } while (0)

struct mdg_encoder {
    struct Level {
        mdg_dims3 d;
        int64_t n;
        int cin, c;
        float *x;          // block input (level 1: the image, not owned)
        float *a1, *z1, *a2;  // conv1 out, block mid, conv2 out (block out: features[k])
        float *st1, *st2;     // mean | inv per channel (2C each)
    };
    std::vector<Level> lv;
    float slope = 0.2f;
    float *scratch_a = nullptr, *scratch_b = nullptr;  // max C*n each
    void *arena = nullptr;
    int64_t bytes = 0;
    std::vector<mdg_block_params> p_saved;
    bool have_forward = false;
};

namespace {
struct Carve2 {
    char *base;
    int64_t off = 0;
    float *take(int64_t floats) {
        float *p = reinterpret_cast<float *>(base ? base + off : nullptr);
        off += ((floats * (int64_t)sizeof(float) + 255) / 256) * 256;
        return p;
    }
};

void enc_layout(mdg_encoder *e, Carve2 &cv, mdg_dims3 d0, int base, int levels) {
    e->lv.resize(levels);
    mdg_dims3 d = d0;
    int64_t mx = 0;
    for (int k = 0; k < levels; ++k) {
        auto &L = e->lv[k];
        if (k > 0) d = mdg_dims3{(d.h + 1) / 2, (d.w + 1) / 2, (d.l + 1) / 2};
        L.d = d;
        L.n = nvox(d);
        L.c = base << k;
        L.cin = k == 0 ? 1 : (base << (k - 1));
        L.x = k == 0 ? nullptr : cv.take((int64_t)L.cin * L.n);
        L.a1 = cv.take((int64_t)L.c * L.n);
        L.z1 = cv.take((int64_t)L.c * L.n);
        L.a2 = cv.take((int64_t)L.c * L.n);
        L.st1 = cv.take(2 * (int64_t)L.c);
        L.st2 = cv.take(2 * (int64_t)L.c);
        mx = std::max<int64_t>(mx, (int64_t)L.c * L.n);
    }
    e->scratch_a = cv.take(mx);
    e->scratch_b = cv.take(mx);
}
}  // namespace

extern "C" {

mdg_status mdg_encoder_conv3_fwd(const float *in, int ic, mdg_dims3 d, const float *w,
                                 const float *b, int oc, float *out, void *stream) {
    MDG_REQUIRE(ic >= 1 && oc >= 1, "conv3: channel counts must be >= 1");
    MDG_REQUIRE(dims_ok(d), "conv3: invalid dims " + dims_str(d));
    if (nvox(d) == 0) return MDG_OK;
    MDG_REQUIRE(in && w && out, "conv3: null pointer");
    return enc_conv3_fwd(in, ic, d, w, b, oc, out, S_(stream));
}

mdg_status mdg_encoder_conv3_bwd(const float *in, int ic, mdg_dims3 d, const float *w, int oc,
                                 const float *gout, float *gin, float *gw, float *gb,
                                 void *stream) {
    MDG_REQUIRE(ic >= 1 && oc >= 1, "conv3: channel counts must be >= 1");
    MDG_REQUIRE(dims_ok(d), "conv3: invalid dims " + dims_str(d));
    if (nvox(d) == 0) return MDG_OK;
    MDG_REQUIRE(in && w && gout, "conv3: null pointer");
    return enc_conv3_bwd(in, ic, d, w, oc, gout, gin, gw, gb, S_(stream));
}

// ---- depth-slab instance norm + leaky ReLU (ops.hpp:162-238 split at the
// two global reductions; slab_po.py all-reduces the sums in between)
mdg_status mdg_in_slab_sums(const float *x, int C, int64_t n, const float *mean, double *sums,
                            void *stream) {
    MDG_REQUIRE(C >= 1 && n >= 1 && n < (int64_t(1) << 31), "instance_norm: invalid sizes");
    MDG_REQUIRE(x && sums, "instance_norm: null pointer");
    return enc_in_slab_sums(x, C, n, mean, sums, S_(stream));
}

mdg_status mdg_in_lrelu_apply(const float *x, int C, int64_t n, const float *mean,
                              const float *inv, const float *g, const float *b, float slope,
                              float *z, void *stream) {
    MDG_REQUIRE(C >= 1 && n >= 1 && n < (int64_t(1) << 31), "instance_norm: invalid sizes");
    MDG_REQUIRE(x && mean && inv && g && b && z, "instance_norm: null pointer");
    return enc_in_lrelu_apply(x, C, n, g, b, slope, z, mean, inv, S_(stream));
}

mdg_status mdg_in_lrelu_bwd_sums(const float *x, const float *gz, int C, int64_t n,
                                 const float *mean, const float *inv, const float *g,
                                 const float *b, float slope, double *sums, void *stream) {
    MDG_REQUIRE(C >= 1 && n >= 1 && n < (int64_t(1) << 31), "instance_norm: invalid sizes");
    MDG_REQUIRE(x && gz && mean && inv && g && b && sums, "instance_norm: null pointer");
    return enc_in_slab_bwd_sums(x, gz, C, n, g, b, slope, mean, inv, sums, S_(stream));
}

mdg_status mdg_in_lrelu_bwd_apply(const float *x, const float *gz, int C, int64_t n,
                                  const float *mean, const float *inv, const float *g,
                                  const float *b, float slope, const float *sums, int64_t nstat,
                                  float *gx, void *stream) {
    MDG_REQUIRE(C >= 1 && n >= 1 && n < (int64_t(1) << 31) && nstat >= n,
                "instance_norm: invalid sizes");
    MDG_REQUIRE(x && gz && mean && inv && g && b && sums && gx, "instance_norm: null pointer");
    return enc_in_slab_bwd_apply(x, gz, C, n, g, b, slope, mean, inv, sums, nstat, gx,
                                 S_(stream));
}

mdg_status mdg_avgpool2_fwd(const float *in, int C, mdg_dims3 d, float *out, void *stream) {
    MDG_REQUIRE(C >= 1 && dims_ok(d), "avg_pool: invalid sizes");
    if (nvox(d) == 0) return MDG_OK;
    MDG_REQUIRE(in && out, "avg_pool: null pointer");
    return enc_avgpool_fwd(in, C, d, out, S_(stream));
}

mdg_status mdg_avgpool2_bwd(const float *gout, int C, mdg_dims3 d, float *gin, void *stream) {
    MDG_REQUIRE(C >= 1 && dims_ok(d), "avg_pool: invalid sizes");
    if (nvox(d) == 0) return MDG_OK;
    MDG_REQUIRE(gout && gin, "avg_pool: null pointer");
    return enc_avgpool_bwd(gout, C, d, gin, S_(stream));
}

mdg_status mdg_encoder_create(mdg_dims3 d, int base_channels, int levels, float slope,
                              mdg_encoder **out) {
    MDG_REQUIRE(out, "encoder: null pointer");
    *out = nullptr;
    MDG_REQUIRE(base_channels >= 1, "encoder: base_channels must be >= 1");
    MDG_REQUIRE(levels == 5, "encoder: levels is fixed at 5");
    MDG_REQUIRE(dims_ok(d), "encoder: invalid dims " + dims_str(d));
    MDG_REQUIRE(d.h >= 16 && d.w >= 16 && d.l >= 16,
                "encode: volume " + dims_str(d) + " too small for 5 pyramid levels (needs dims >= 16)");
    mdg_encoder *e = new mdg_encoder;
    e->slope = slope;
    Carve2 dry{nullptr};
    enc_layout(e, dry, d, base_channels, levels);
    e->bytes = dry.off;
    void *mem = nullptr;
    cudaError_t err = cudaMalloc(&mem, (size_t)e->bytes);
    if (err != cudaSuccess) {
        delete e;
        return status_from_cuda(err, "encoder arena");
    }
    e->arena = mem;
    Carve2 cv{reinterpret_cast<char *>(mem)};
    enc_layout(e, cv, d, base_channels, levels);
    *out = e;
    return MDG_OK;
}

void mdg_encoder_destroy(mdg_encoder *e) {
    if (!e) return;
    if (e->arena) cudaFree(e->arena);
    delete e;
}

mdg_status mdg_encoder_forward(mdg_encoder *e, const float *image, const mdg_block_params *params,
                               float *const *features, void *stream) {
    MDG_REQUIRE(e && image && params && features, "encoder: null pointer");
    cudaStream_t st = S_(stream);
    e->p_saved.assign(params, params + e->lv.size());
    for (size_t k = 0; k < e->lv.size(); ++k) {
        auto &L = e->lv[k];
        const mdg_block_params &P = params[k];
        MDG_REQUIRE(P.w1 && P.b1 && P.g1 && P.be1 && P.w2 && P.b2 && P.g2 && P.be2 && features[k],
                    "encoder: null parameter or feature buffer");
        const float *x = image;
        if (k > 0) {
            ENC_TRY(enc_avgpool_fwd(features[k - 1], L.cin, e->lv[k - 1].d, L.x, st));
            x = L.x;
        } else {
            L.x = const_cast<float *>(image);
        }
        bool fused = false;
        ENC_TRY(enc_conv3_fwd(x, L.cin, L.d, P.w1, P.b1, L.c, L.a1, st, L.st1, &fused));
        if (fused)
            ENC_TRY(enc_in_lrelu_apply(L.a1, L.c, L.n, P.g1, P.be1, e->slope, L.z1, L.st1,
                                       L.st1 + L.c, st));
        else
            ENC_TRY(enc_in_lrelu_fwd(L.a1, L.c, L.n, P.g1, P.be1, e->slope, L.z1, L.st1,
                                     L.st1 + L.c, st));
        ENC_TRY(enc_conv3_fwd(L.z1, L.c, L.d, P.w2, P.b2, L.c, L.a2, st, L.st2, &fused));
        if (fused)
            ENC_TRY(enc_in_lrelu_apply(L.a2, L.c, L.n, P.g2, P.be2, e->slope, features[k], L.st2,
                                       L.st2 + L.c, st));
        else
            ENC_TRY(enc_in_lrelu_fwd(L.a2, L.c, L.n, P.g2, P.be2, e->slope, features[k], L.st2,
                                     L.st2 + L.c, st));
    }
    e->have_forward = true;
    return MDG_OK;
}

mdg_status mdg_encoder_backward(mdg_encoder *e, const float *const *gfeatures,
                                const mdg_block_grads *grads, float *gimage, void *stream) {
    MDG_REQUIRE(e && gfeatures, "encoder: null pointer");
    MDG_REQUIRE(e->have_forward, "encoder: backward without a forward");
    cudaStream_t st = S_(stream);
    const int levels = (int)e->lv.size();
    const float *pool = nullptr;  // input gradient of the coarser level (pooled from this one)
    for (int k = levels - 1; k >= 0; --k) {
        auto &L = e->lv[k];
        const mdg_block_params &P = e->p_saved[k];
        const mdg_block_grads *G = grads ? &grads[k] : nullptr;
        float *ga = e->scratch_a, *gz1 = e->scratch_b;
        // block output z2 = lrelu(IN2(a2)); its gradient = gfeatures[k] + pool bwd
        ENC_TRY(enc_in_lrelu_bwd(L.a2, gfeatures[k], pool, L.d, L.c, L.n, P.g2, P.be2, e->slope,
                                 L.st2, L.st2 + L.c, ga, G ? G->g2 : nullptr,
                                 G ? G->be2 : nullptr, st));
        ENC_TRY(enc_conv3_bwd(L.z1, L.c, L.d, P.w2, L.c, ga, gz1, G ? G->w2 : nullptr,
                              G ? G->b2 : nullptr, st, /*gin_acc=*/false));
        // z1 = lrelu(IN1(a1)); ga reused
        ENC_TRY(enc_in_lrelu_bwd(L.a1, gz1, nullptr, L.d, L.c, L.n, P.g1, P.be1, e->slope, L.st1,
                                 L.st1 + L.c, ga, G ? G->g1 : nullptr, G ? G->be1 : nullptr,
                                 st));
        // conv1 input gradient: overwritten into scratch for the finer level's
        // fused pool backward, or accumulated into the image gradient
        float *gx = k > 0 ? gz1 : gimage;
        ENC_TRY(enc_conv3_bwd(L.x, L.cin, L.d, P.w1, L.c, ga, gx, G ? G->w1 : nullptr,
                              G ? G->b1 : nullptr, st, /*gin_acc=*/k == 0));
        pool = gx;
    }
    return MDG_OK;
}

}  // extern "C"
