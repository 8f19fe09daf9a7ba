// mdg_common.cuh — shared internals of libmdg (B200 / sm_100a).
//
// Indexing follows the reference layout contract (common.hpp:56-59): voxel
// p = (z*w + y)*h + x, channel-major planes.  All kernels are fp32.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/mdg.h"

namespace mdg {

// ------------------------------------------------------------------ status
void set_error(mdg_status st, const std::string &msg);
mdg_status status_from_cuda(cudaError_t e, const char *where);
extern std::atomic<int64_t> g_launches;

#define MDG_CUDA_TRY(expr)                                                        \
    do {                                                                          \
        cudaError_t _e = (expr);                                                  \
        if (_e != cudaSuccess) return ::mdg::status_from_cuda(_e, #expr);         \
    } while (0)

// after a launch: count it and surface launch-config errors
#define MDG_LAUNCHED()                                                            \
    do {                                                                          \
        ::mdg::g_launches.fetch_add(1, std::memory_order_relaxed);                \
        cudaError_t _e = cudaPeekAtLastError();                                   \
        if (_e != cudaSuccess) return ::mdg::status_from_cuda(_e, __func__);      \
    } while (0)

#define MDG_REQUIRE(cond, msg)                                                    \
    do {                                                                          \
        if (!(cond)) {                                                            \
            ::mdg::set_error(MDG_EINVAL, (msg));                                  \
            return MDG_EINVAL;                                                    \
        }                                                                         \
    } while (0)

inline cudaStream_t S_(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t nvox(mdg_dims3 d) { return (int64_t)d.h * d.w * d.l; }
inline std::string dims_str(mdg_dims3 d) {
    return std::to_string(d.h) + "x" + std::to_string(d.w) + "x" + std::to_string(d.l);
}
inline bool dims_ok(mdg_dims3 d) {
    return d.h >= 0 && d.w >= 0 && d.l >= 0 && nvox(d) < (int64_t(1) << 31);
}

// ----------------------------------------------- device-side numeric flag
// One word per (device, stream): the smallest (head*n + p) key whose attention row
// produced a non-finite logit, or ~0ull.  Keys follow the reference's loop
// order (attention.hpp:91-96: head outer, then z, y, x) so atomicMin yields
// the position the reference would have thrown at.
unsigned long long *numeric_flag_ptr(cudaStream_t st);  // of (current device, st)
// read + reset; returns true if set, and the (x,y,z,head) decoded w.r.t. the
// dims of the call that is checking
mdg_status consume_numeric_flag(cudaStream_t st, mdg_dims3 d);

// Per-(device, stream) fixup queue for the fused ModeT forward: voxel-heads whose
// branch-free online softmax overflowed (logit spread > 2^7 in log2 units
// above the first row's max) or saw a non-finite logit are recomputed exactly
// by a follow-up kernel.  Layout: [0] = count (uint32), then kFixupCap keys.
constexpr int kFixupCap = 1 << 16;
unsigned long long *fixup_queue_ptr(cudaStream_t st);

// --------------------------------------------------- stream-ordered scratch
// cudaMallocAsync/cudaFreeAsync from the device's default mempool.  The pool's
// release threshold is raised once per device so freed scratch stays mapped:
// with the default (0) every synchronisation hands the memory back and the
// next call pays for a fresh mapping inside its stream.
void keep_pool_mapped();

struct Scratch {
    void *p = nullptr;
    cudaStream_t st = nullptr;
    Scratch() = default;
    Scratch(const Scratch &) = delete;
    Scratch &operator=(const Scratch &) = delete;
    cudaError_t alloc(size_t bytes, cudaStream_t s) {
        st = s;
        keep_pool_mapped();
        return cudaMallocAsync(&p, bytes ? bytes : 16, s);
    }
    ~Scratch() {
        if (p) cudaFreeAsync(p, st);
    }
    template <typename T>
    T *as() const { return reinterpret_cast<T *>(p); }
};

inline unsigned grid1d(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

// --------------------------------------------------------- device helpers
// sampling.hpp:29-49 resolve_axis — identical integer logic on the device.
struct Ax {
    int i0, i1;
    float f;
    bool live;
};

__device__ __forceinline__ Ax resolve_axis(float x, int dim) {
    Ax a;
    if (dim <= 1) {
        a.i0 = 0;
        a.i1 = 0;
        a.f = 0.0f;
        a.live = false;
        return a;
    }
    const float hi = (float)(dim - 1);
    const float xc = x < 0.0f ? 0.0f : (x > hi ? hi : x);
    int i0 = (int)floorf(xc);
    if (i0 > dim - 2) i0 = dim - 2;
    a.i0 = i0;
    a.i1 = i0 + 1;
    a.f = __fsub_rn(xc, (float)i0);
    a.live = x > 0.0f && x < hi;
    return a;
}

// IEEE-rounded helpers: keep the reference's evaluation order without FMA
// contraction so sampling results are bit-identical to the CPU reference.
__device__ __forceinline__ float mul_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_(float a, float b) { return __fsub_rn(a, b); }
// a*(1-f) + b*f with both products rounded (sampling.hpp:61-67)
__device__ __forceinline__ float lerp_(float a, float b, float f) {
    return add_(mul_(a, sub_(1.0f, f)), mul_(b, f));
}

// project.cu: the projection backward; bit i of gin_set makes input i's
// gradient an overwrite instead of an accumulation (internal buffers)
mdg_status project_qk_bwd_impl(const float *f, const float *m, int C, int64_t n,
                               const float *weight, const float *bias, const float *ln_g, int K,
                               int layout, const float *gQ, const float *gK, float *gf,
                               float *gm, float *gweight, float *gbias, float *gln_g,
                               float *gln_b, int gin_set, cudaStream_t stream);

// encoder.cu: conv block pieces (internal; driven by encoder_driver.cu)
// norm_stats (2*oc floats: mean | inv) + stats_done: when the conv path can
// fuse the InstanceNorm statistics into its epilogue it fills them and sets
// *stats_done (otherwise the caller runs enc_in_lrelu_fwd's own passes)
mdg_status enc_conv3_fwd(const float *in, int ic, mdg_dims3 d, const float *w, const float *b,
                         int oc, float *out, cudaStream_t st, float *norm_stats = nullptr,
                         bool *stats_done = nullptr);
mdg_status enc_in_lrelu_apply(const float *x, int C, int64_t n, const float *g, const float *b,
                              float slope, float *z, const float *mean, const float *inv,
                              cudaStream_t st);
// gin_acc: accumulate into gin (else overwrite)
mdg_status enc_conv3_bwd(const float *in, int ic, mdg_dims3 d, const float *w, int oc,
                         const float *gout, float *gin, float *gw, float *gb, cudaStream_t st,
                         bool gin_acc = true);
mdg_status enc_in_lrelu_fwd(const float *x, int C, int64_t n, const float *g, const float *b,
                            float slope, float *z, float *mean, float *inv, cudaStream_t st);
// gz: gradient of the block output (nullable); pg: the coarser level's input
// gradient whose 2x pool backward is added on the fly (nullable); fd: dims
mdg_status enc_in_lrelu_bwd(const float *x, const float *gz, const float *pg, mdg_dims3 fd,
                            int C, int64_t n, const float *g, const float *b, float slope,
                            const float *mean, const float *inv, float *gx, float *gg,
                            float *gbeta, cudaStream_t st);
mdg_status enc_in_slab_sums(const float *x, int C, int64_t n, const float *mean, double *sums,
                            cudaStream_t st);
mdg_status enc_in_slab_bwd_sums(const float *x, const float *gz, int C, int64_t n,
                                const float *g, const float *b, float slope, const float *mean,
                                const float *inv, double *sums, cudaStream_t st);
mdg_status enc_in_slab_bwd_apply(const float *x, const float *gz, int C, int64_t n,
                                 const float *g, const float *b, float slope, const float *mean,
                                 const float *inv, const float *sums, int64_t nstat, float *gx,
                                 cudaStream_t st);
// encoder_tc.cu: the 3x3x3 conv on tcgen05 for 32 / 64 output channels
bool enc_tc_conv_ok(int kin, int nout, mdg_dims3 d);
mdg_status enc_tc_conv(const float *in, int kin, mdg_dims3 d, const float *w, int nout, int flip,
                       const float *bias, bool acc, float *out, cudaStream_t st);
mdg_status enc_avgpool_fwd(const float *in, int C, mdg_dims3 d, float *out, cudaStream_t st);
mdg_status enc_avgpool_bwd(const float *gout, int C, mdg_dims3 d, float *gin, cudaStream_t st);
// optim.cu: AdamOptimizer::step over a whole parameter list in one launch
// (same per-element double arithmetic as mdg_adam_step: bit-identical)
struct AdamTensor {
    float *value;
    const float *grad;
    float *m, *v;
    int64_t n;
};
constexpr int kMaxAdamTensors = 80;
struct AdamList {
    AdamTensor t[kMaxAdamTensors];
    int count;
};
mdg_status adam_multi(const AdamList &L, double lr, double b1, double b2, double eps, int64_t t,
                      cudaStream_t st);
// the same with the step count on the device (++*d_t) and the bias
// corrections from a host-computed table: replayable in a CUDA graph
mdg_status adam_multi_dev(const AdamList &L, double lr, double b1, double b2, double eps,
                          int64_t *d_t, const double *d_bc, cudaStream_t st);

namespace enc {
// encoder_igemm.cu: implicit-GEMM conv for the deep levels
int igemm_fwd_bn(int cout);  // N tile (32 or 64): the weight padding it needs
mdg_status igemm_conv_fwd(const float *in, int cin, mdg_dims3 d, const float *wT, int opad,
                          const float *bias, int cout, bool acc_out, float *out, cudaStream_t st);
mdg_status igemm_conv_wgrad(const float *in, int cin, mdg_dims3 d, const float *gout, int cout,
                            float *gk, float *gb, cudaStream_t st);
}  // namespace enc

// sampling.cu: warp kernels over the voxel range [pb, pe) of a volume
mdg_status warp_fwd_range(const float *in, int C, mdg_dims3 d, const float *field, float *out,
                          int64_t pb, int64_t pe, cudaStream_t st);
mdg_status warp_bwd_range(const float *in, int C, mdg_dims3 d, const float *field,
                          const float *gout, float *gin, float *gfield, int64_t pb, int64_t pe,
                          cudaStream_t st);

// deterministic mode (runtime.cu): process-wide, initialised from the
// MDG_DETERMINISTIC environment variable, set by mdg_set_deterministic()
bool deterministic_mode();

// warp_gather.cu: the warp's input gradient as a deterministic gather for
// displacements up to kGinGatherReach voxels (after
// warp_bwd_k has put max |phi| into rbits[0]; rbits[1..] is its scratch)
constexpr int kGinGatherReach = 4;
int64_t gin_gather_scratch_words(mdg_dims3 d);
mdg_status warp_gin_gather(const float *field, const float *gout, int C, mdg_dims3 d, float *gin,
                           int64_t pb, int64_t pe, const unsigned *rbits, unsigned *dirty,
                           cudaStream_t st);

}  // namespace mdg
