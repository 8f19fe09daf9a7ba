// optim.cu — parameter updates on the device:
// AdamOptimizer::step and sgd_step (engine.hpp:268-311).  The reference does
// the per-element arithmetic in double and stores float; the kernels do the
// same with IEEE-rounded double operations in the reference's order (no
// contraction), so the updated parameters and moments are bit-identical.
#include <algorithm>
#include <cmath>

#include "mdg_common.cuh"

namespace mdg {

__global__ void adam_k(float *__restrict__ value, const float *__restrict__ grad,
                       float *__restrict__ m, float *__restrict__ v, int64_t n, double lr,
                       double b1, double b2, double eps, double bc1, double bc2) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double g = (double)grad[j];
        // mj = b1*m + (1-b1)*g ; vj = b2*v + (1-b2)*g*g  (engine.hpp:288-289)
        const double mj = __dadd_rn(__dmul_rn(b1, (double)m[j]), __dmul_rn(1.0 - b1, g));
        const double vj =
            __dadd_rn(__dmul_rn(b2, (double)v[j]), __dmul_rn(__dmul_rn(1.0 - b2, g), g));
        m[j] = (float)mj;
        v[j] = (float)vj;
        // update = lr * (mj / bc1) / (sqrt(vj / bc2) + eps)  (engine.hpp:292)
        const double upd = __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mj, bc1)),
                                     __dadd_rn(__dsqrt_rn(__ddiv_rn(vj, bc2)), eps));
        value[j] = (float)__dsub_rn((double)value[j], upd);
    }
}

// every tensor of a parameter list in one launch: grid row = tensor
__global__ void adam_multi_k(AdamList L, double lr, double b1, double b2, double eps, double bc1,
                             double bc2) {
    const AdamTensor &T = L.t[blockIdx.y];
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < T.n;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double g = (double)T.grad[j];
        const double mj = __dadd_rn(__dmul_rn(b1, (double)T.m[j]), __dmul_rn(1.0 - b1, g));
        const double vj =
            __dadd_rn(__dmul_rn(b2, (double)T.v[j]), __dmul_rn(__dmul_rn(1.0 - b2, g), g));
        T.m[j] = (float)mj;
        T.v[j] = (float)vj;
        const double upd = __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mj, bc1)),
                                     __dadd_rn(__dsqrt_rn(__ddiv_rn(vj, bc2)), eps));
        T.value[j] = (float)__dsub_rn((double)T.value[j], upd);
    }
}

// device-side step count (graph replays): t = ++*d_t, bias corrections from
// the host-computed table d_bc[2 (t-1) + {0, 1}] (std::pow, as above)
__global__ void adam_tick_k(int64_t *d_t) { ++*d_t; }

__global__ void adam_multi_dev_k(AdamList L, double lr, double b1, double b2, double eps,
                                 const int64_t *__restrict__ d_t, const double *__restrict__ d_bc) {
    const AdamTensor &T = L.t[blockIdx.y];
    const int64_t t = *d_t;
    const double bc1 = d_bc[2 * (t - 1)], bc2 = d_bc[2 * (t - 1) + 1];
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < T.n;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double g = (double)T.grad[j];
        const double mj = __dadd_rn(__dmul_rn(b1, (double)T.m[j]), __dmul_rn(1.0 - b1, g));
        const double vj =
            __dadd_rn(__dmul_rn(b2, (double)T.v[j]), __dmul_rn(__dmul_rn(1.0 - b2, g), g));
        T.m[j] = (float)mj;
        T.v[j] = (float)vj;
        const double upd = __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mj, bc1)),
                                     __dadd_rn(__dsqrt_rn(__ddiv_rn(vj, bc2)), eps));
        T.value[j] = (float)__dsub_rn((double)T.value[j], upd);
    }
}

mdg_status adam_multi_dev(const AdamList &L, double lr, double b1, double b2, double eps,
                          int64_t *d_t, const double *d_bc, cudaStream_t st) {
    adam_tick_k<<<1, 1, 0, st>>>(d_t);
    MDG_LAUNCHED();
    if (L.count == 0) return MDG_OK;
    int64_t mx = 0;
    for (int i = 0; i < L.count; ++i) mx = std::max(mx, L.t[i].n);
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(grid1d(mx, 256), 64));
    adam_multi_dev_k<<<dim3(gx, L.count), 256, 0, st>>>(L, lr, b1, b2, eps, d_t, d_bc);
    MDG_LAUNCHED();
    return MDG_OK;
}

mdg_status adam_multi(const AdamList &L, double lr, double b1, double b2, double eps, int64_t t,
                      cudaStream_t st) {
    if (L.count == 0) return MDG_OK;
    const double bc1 = 1.0 - std::pow(b1, (double)t);
    const double bc2 = 1.0 - std::pow(b2, (double)t);
    int64_t mx = 0;
    for (int i = 0; i < L.count; ++i) mx = std::max(mx, L.t[i].n);
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(grid1d(mx, 256), 64));
    adam_multi_k<<<dim3(gx, L.count), 256, 0, st>>>(L, lr, b1, b2, eps, bc1, bc2);
    MDG_LAUNCHED();
    return MDG_OK;
}

__global__ void sgd_k(float *__restrict__ value, const float *__restrict__ grad, int64_t n,
                      double lr) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x)
        value[j] = (float)__dsub_rn((double)value[j], __dmul_rn(lr, (double)grad[j]));
}

}  // namespace mdg

using namespace mdg;

extern "C" {

mdg_status mdg_adam_step(float *value, const float *grad, float *m, float *v, int64_t n,
                         double lr, double beta1, double beta2, double eps, int64_t t,
                         void *stream) {
    MDG_REQUIRE(n >= 0 && t >= 1, "adam: invalid size or step count");
    if (n == 0) return MDG_OK;
    MDG_REQUIRE(value && grad && m && v, "adam: null pointer");
    // bias corrections on the host exactly as engine.hpp:281-282
    const double bc1 = 1.0 - std::pow(beta1, (double)t);
    const double bc2 = 1.0 - std::pow(beta2, (double)t);
    const unsigned g = (unsigned)std::min<int64_t>(grid1d(n, 256), 148 * 8);
    adam_k<<<g, 256, 0, S_(stream)>>>(value, grad, m, v, n, lr, beta1, beta2, eps, bc1, bc2);
    MDG_LAUNCHED();
    return MDG_OK;
}

mdg_status mdg_sgd_step(float *value, const float *grad, int64_t n, double lr, void *stream) {
    MDG_REQUIRE(n >= 0, "sgd: invalid size");
    if (n == 0) return MDG_OK;
    MDG_REQUIRE(value && grad, "sgd: null pointer");
    const unsigned g = (unsigned)std::min<int64_t>(grid1d(n, 256), 148 * 8);
    sgd_k<<<g, 256, 0, S_(stream)>>>(value, grad, n, lr);
    MDG_LAUNCHED();
    return MDG_OK;
}

}  // extern "C"
