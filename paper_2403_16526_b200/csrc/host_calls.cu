// host_calls.cu — synchronous host-buffer drop-ins for the reference CPU
// functions (attention.hpp:83 / 127, sampling.hpp:123 / 139).  The caller
// passes host pointers exactly as to mdreg::kern::*; staging buffers come from
// the stream-ordered pool, copies and kernels run on a per-thread stream, and
// the call returns after the results are back in host memory.  With pinned
// host buffers (mdg_host_alloc) the copies run at full PCIe/C2C bandwidth.
#include <vector>

#include "mdg_common.cuh"

namespace mdg {
namespace {

struct HostStream {
    cudaStream_t st = nullptr;
    HostStream() { cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking); }
    ~HostStream() {
        if (st) cudaStreamDestroy(st);
    }
};

cudaStream_t host_stream() {
    thread_local HostStream hs;
    return hs.st;
}

// a set of device staging buffers freed (stream-ordered) on scope exit
struct Stage {
    cudaStream_t st;
    std::vector<void *> bufs;
    explicit Stage(cudaStream_t s) : st(s) {}
    ~Stage() {
        for (void *p : bufs) cudaFreeAsync(p, st);
    }
    // device copy of a host array (h2d when `upload`)
    cudaError_t get(float **dev, const float *host, size_t count, bool upload) {
        *dev = nullptr;
        if (!host) return cudaSuccess;
        void *p = nullptr;
        cudaError_t e = cudaMallocAsync(&p, count * sizeof(float) + 16, st);
        if (e != cudaSuccess) return e;
        bufs.push_back(p);
        *dev = static_cast<float *>(p);
        if (upload)
            return cudaMemcpyAsync(p, host, count * sizeof(float), cudaMemcpyHostToDevice, st);
        return cudaSuccess;
    }
    cudaError_t down(float *host, const float *dev, size_t count) {
        if (!host) return cudaSuccess;
        return cudaMemcpyAsync(host, dev, count * sizeof(float), cudaMemcpyDeviceToHost, st);
    }
};

}  // namespace
}  // namespace mdg

using namespace mdg;

#define MDG_STAGE_TRY(expr)                                            \
    do {                                                               \
        cudaError_t _e = (expr);                                       \
        if (_e != cudaSuccess) return status_from_cuda(_e, #expr);     \
    } while (0)

extern "C" {

mdg_status mdg_na_fused_fwd_host(const float *Q, const float *K, const float *B, mdg_dims3 d,
                                 int S, int hd, int nb, float *W) {
    MDG_REQUIRE(dims_ok(d) && S >= 1 && hd >= 1, "na_fused_fwd: invalid sizes");
    const size_t n = (size_t)nvox(d), win = (size_t)nb * nb * nb;
    if (n == 0) return MDG_OK;
    cudaStream_t st = host_stream();
    Stage sg(st);
    float *dQ, *dK, *dB, *dW;
    MDG_STAGE_TRY(sg.get(&dQ, Q, n * S * hd, true));
    MDG_STAGE_TRY(sg.get(&dK, K, n * S * hd, true));
    MDG_STAGE_TRY(sg.get(&dB, B, (size_t)S * win, true));
    MDG_STAGE_TRY(sg.get(&dW, W, (size_t)S * n * win, false));
    mdg_status r = mdg_na_fused_fwd(dQ, dK, dB, d, S, hd, nb, dW, st);
    if (r != MDG_OK) return r;
    MDG_STAGE_TRY(sg.down(W, dW, (size_t)S * n * win));
    MDG_STAGE_TRY(cudaStreamSynchronize(st));
    return MDG_OK;
}

mdg_status mdg_modet_fwd_host(const float *Q, const float *K, const float *B, mdg_dims3 d,
                              int S, int hd, int nb, int layout, float *SF, float *LSE) {
    MDG_REQUIRE(dims_ok(d) && S >= 1 && hd >= 1, "modet: invalid sizes");
    const size_t n = (size_t)nvox(d);
    if (n == 0) return MDG_OK;
    cudaStream_t st = host_stream();
    Stage sg(st);
    float *dQ, *dK, *dB, *dSF, *dL;
    MDG_STAGE_TRY(sg.get(&dQ, Q, n * S * hd, true));
    MDG_STAGE_TRY(sg.get(&dK, K, n * S * hd, true));
    MDG_STAGE_TRY(sg.get(&dB, B, (size_t)S * 27, true));
    MDG_STAGE_TRY(sg.get(&dSF, SF, 3 * n * S, false));
    MDG_STAGE_TRY(sg.get(&dL, LSE, n * S, false));
    mdg_status r = mdg_modet_fwd(dQ, dK, dB, d, S, hd, nb, layout, dSF, dL, nullptr, st);
    if (r != MDG_OK) return r;
    MDG_STAGE_TRY(sg.down(SF, dSF, 3 * n * S));
    MDG_STAGE_TRY(sg.down(LSE, dL, n * S));
    return consume_numeric_flag(st, d);
}

mdg_status mdg_modet_bwd_host(const float *Q, const float *K, const float *B, const float *SF,
                              const float *LSE, const float *gSF, mdg_dims3 d, int S, int hd,
                              int nb, int layout, float *gQ, float *gK, float *gB) {
    MDG_REQUIRE(dims_ok(d) && S >= 1 && hd >= 1, "modet: invalid sizes");
    const size_t n = (size_t)nvox(d);
    if (n == 0) return MDG_OK;
    cudaStream_t st = host_stream();
    Stage sg(st);
    float *dQ, *dK, *dB, *dSF, *dL, *dG, *dgQ, *dgK, *dgB;
    MDG_STAGE_TRY(sg.get(&dQ, Q, n * S * hd, true));
    MDG_STAGE_TRY(sg.get(&dK, K, n * S * hd, true));
    MDG_STAGE_TRY(sg.get(&dB, B, (size_t)S * 27, true));
    MDG_STAGE_TRY(sg.get(&dSF, SF, 3 * n * S, true));
    MDG_STAGE_TRY(sg.get(&dL, LSE, n * S, true));
    MDG_STAGE_TRY(sg.get(&dG, gSF, 3 * n * S, true));
    MDG_STAGE_TRY(sg.get(&dgQ, gQ, n * S * hd, true));  // accumulate targets go up too
    MDG_STAGE_TRY(sg.get(&dgK, gK, n * S * hd, true));
    MDG_STAGE_TRY(sg.get(&dgB, gB, (size_t)S * 27, true));
    mdg_status r =
        mdg_modet_bwd(dQ, dK, dB, dSF, dL, dG, d, S, hd, nb, layout, dgQ, dgK, dgB, 1, st);
    if (r != MDG_OK) return r;
    MDG_STAGE_TRY(sg.down(gQ, dgQ, n * S * hd));
    MDG_STAGE_TRY(sg.down(gK, dgK, n * S * hd));
    MDG_STAGE_TRY(sg.down(gB, dgB, (size_t)S * 27));
    MDG_STAGE_TRY(cudaStreamSynchronize(st));
    return MDG_OK;
}

mdg_status mdg_warp_fwd_host(const float *in, int C, mdg_dims3 d, const float *field,
                             float *out) {
    MDG_REQUIRE(dims_ok(d) && C >= 0, "warp: invalid sizes");
    const size_t n = (size_t)nvox(d);
    if (n == 0 || C == 0) return MDG_OK;
    cudaStream_t st = host_stream();
    Stage sg(st);
    float *di, *df, *dout;
    MDG_STAGE_TRY(sg.get(&di, in, n * C, true));
    MDG_STAGE_TRY(sg.get(&df, field, 3 * n, true));
    MDG_STAGE_TRY(sg.get(&dout, out, n * C, false));
    mdg_status r = mdg_warp_fwd(di, C, d, df, dout, st);
    if (r != MDG_OK) return r;
    MDG_STAGE_TRY(sg.down(out, dout, n * C));
    MDG_STAGE_TRY(cudaStreamSynchronize(st));
    return MDG_OK;
}

mdg_status mdg_warp_bwd_host(const float *in, int C, mdg_dims3 d, const float *field,
                             const float *gout, float *gin, float *gfield) {
    MDG_REQUIRE(dims_ok(d) && C >= 0, "warp: invalid sizes");
    const size_t n = (size_t)nvox(d);
    if (n == 0 || C == 0) return MDG_OK;
    cudaStream_t st = host_stream();
    Stage sg(st);
    float *di, *df, *dg, *dgi, *dgf;
    MDG_STAGE_TRY(sg.get(&di, in, n * C, true));
    MDG_STAGE_TRY(sg.get(&df, field, 3 * n, true));
    MDG_STAGE_TRY(sg.get(&dg, gout, n * C, true));
    MDG_STAGE_TRY(sg.get(&dgi, gin, n * C, true));
    MDG_STAGE_TRY(sg.get(&dgf, gfield, 3 * n, true));
    mdg_status r = mdg_warp_bwd(di, C, d, df, dg, dgi, dgf, st);
    if (r != MDG_OK) return r;
    MDG_STAGE_TRY(sg.down(gin, dgi, n * C));
    MDG_STAGE_TRY(sg.down(gfield, dgf, 3 * n));
    MDG_STAGE_TRY(cudaStreamSynchronize(st));
    return MDG_OK;
}

}  // extern "C"
