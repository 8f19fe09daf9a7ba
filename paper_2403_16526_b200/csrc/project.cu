// project.cu — the Q/K producer of the ModeT operator on sm_100a:
// Q = LN(W·F + b), K = LN(W·M + b) with shared weights (attention.hpp:351-356,
// op_linear_proj ops.hpp:387-435, op_layer_norm ops.hpp:439-497, eps 1e-5,
// LayerNorm over all K = S*hd outputs of a voxel jointly).
//
// One thread per voxel: the K pre-norm values live in registers (K <= 64 via
// the KMAX templates, a two-pass global variant beyond), the C input channels
// stream through coalesced planar loads, and the output is written either in
// the reference's position-major {n, K} order or directly in the planar
// {K, n} order the tiled ModeT kernels consume (no transpose pass).
//
// Backward: the per-voxel LN + linear adjoint is recomputed from the input
// (nothing but F/M is saved), the input gradient is accumulated in place, and
// the parameter gradients (W {K,C}, b, gamma, beta) are full-volume sums done
// as grid-stride per-thread register accumulators -> fixed-order block
// reduction -> per-CTA partials -> fixed-order final sum: deterministic, and
// within fp32 reduction tolerance of the reference's sequential loops.
#include "mdg_common.cuh"

namespace mdg {

constexpr int kPB = 256;
constexpr int kSmemW = 8192;  // weights staged in smem up to this many floats

struct ProjArgs {
    const float *in[2];
    float *out[2];
    const float *gout[2];
    float *gin[2];
    int ninputs;
    int C, K;
    int64_t n;
    float eps;
    int planar;
};

__device__ __forceinline__ int64_t qk_index(int planar, int64_t p, int k, int64_t n, int K) {
    return planar ? (int64_t)k * n + p : p * K + k;
}

// stage W {K,C}, b, gamma, beta into shared memory (or point at global)
struct ProjParams {
    const float *W, *b, *g, *be;
};

__device__ __forceinline__ ProjParams stage_params(float *sm, const float *W, const float *b,
                                                   const float *g, const float *be, int K,
                                                   int C) {
    ProjParams pp;
    const int kc = K * C;
    if (kc + 3 * K <= kSmemW) {
        for (int i = threadIdx.x; i < kc; i += blockDim.x) sm[i] = W[i];
        for (int i = threadIdx.x; i < K; i += blockDim.x) {
            sm[kc + i] = b[i];
            sm[kc + K + i] = g ? g[i] : 1.0f;
            sm[kc + 2 * K + i] = be ? be[i] : 0.0f;
        }
        __syncthreads();
        pp.W = sm;
        pp.b = sm + kc;
        pp.g = sm + kc + K;
        pp.be = sm + kc + 2 * K;
    } else {
        pp.W = W;
        pp.b = b;
        pp.g = g;
        pp.be = be;
    }
    return pp;
}

// raw[k] = b[k] + sum_c W[k,c] in[c,p]  (channel order, as ops.hpp:403-406)
template <int KMAX>
__device__ __forceinline__ void project_raw(const float *__restrict__ in, int64_t p, int64_t n,
                                            int C, int K, const ProjParams &pp,
                                            float (&raw)[KMAX]) {
#pragma unroll
    for (int k = 0; k < KMAX; ++k) raw[k] = k < K ? pp.b[k] : 0.0f;
    for (int c = 0; c < C; ++c) {
        const float x = __ldg(in + (int64_t)c * n + p);
        const float *wc = pp.W + c;
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
            if (k < K) raw[k] = fmaf(wc[(int64_t)k * C], x, raw[k]);
    }
}

// two-pass mean / biased variance (ops.hpp:447-454); raw -> xhat in place
template <int KMAX>
__device__ __forceinline__ float ln_normalize(float (&raw)[KMAX], int K, float eps) {
    float mean = 0.0f;
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
        if (k < K) mean += raw[k];
    mean /= (float)K;
    float var = 0.0f;
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
        if (k < K) {
            const float t = raw[k] - mean;
            var = fmaf(t, t, var);
        }
    var /= (float)K;
    const float inv = 1.0f / sqrtf(var + eps);
#pragma unroll
    for (int k = 0; k < KMAX; ++k) raw[k] = (raw[k] - mean) * inv;
    return inv;
}

template <int KMAX>
__global__ void __launch_bounds__(kPB)
project_fwd_k(ProjArgs a, const float *__restrict__ W, const float *__restrict__ b,
              const float *__restrict__ g, const float *__restrict__ be) {
    extern __shared__ float sm[];
    const ProjParams pp = stage_params(sm, W, b, g, be, a.K, a.C);
    const int which = blockIdx.y;
    const int64_t p = (int64_t)blockIdx.x * kPB + threadIdx.x;
    if (p >= a.n) return;
    float raw[KMAX];
    project_raw<KMAX>(a.in[which], p, a.n, a.C, a.K, pp, raw);
    ln_normalize<KMAX>(raw, a.K, a.eps);
    float *out = a.out[which];
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
        if (k < a.K) out[qk_index(a.planar, p, k, a.n, a.K)] = fmaf(pp.g[k], raw[k], pp.be[k]);
}

// K > 64: raw values go through the output buffer (two extra passes over it)
__global__ void __launch_bounds__(kPB)
project_fwd_wide_k(ProjArgs a, const float *__restrict__ W, const float *__restrict__ b,
                   const float *__restrict__ g, const float *__restrict__ be) {
    const int which = blockIdx.y;
    const int64_t p = (int64_t)blockIdx.x * kPB + threadIdx.x;
    if (p >= a.n) return;
    const float *in = a.in[which];
    float *out = a.out[which];
    const int K = a.K, C = a.C;
    float mean = 0.0f;
    for (int k = 0; k < K; ++k) {
        float s = b[k];
        for (int c = 0; c < C; ++c) s = fmaf(__ldg(W + (int64_t)k * C + c), __ldg(in + (int64_t)c * a.n + p), s);
        out[qk_index(a.planar, p, k, a.n, K)] = s;
        mean += s;
    }
    mean /= (float)K;
    float var = 0.0f;
    for (int k = 0; k < K; ++k) {
        const float t = out[qk_index(a.planar, p, k, a.n, K)] - mean;
        var = fmaf(t, t, var);
    }
    var /= (float)K;
    const float inv = 1.0f / sqrtf(var + a.eps);
    for (int k = 0; k < K; ++k) {
        float &o = out[qk_index(a.planar, p, k, a.n, K)];
        o = fmaf(g[k], (o - mean) * inv, be[k]);
    }
}

// ------------------------------------------------------------------ backward
// Per-voxel adjoint (ops.hpp:470-493 then 418-431):
//   xh = (raw - mean) inv;  gg_k = gout_k gamma_k
//   graw_k = inv (gg_k - mean(gg) - xh_k mean(gg xh))
//   gin_c += sum_k graw_k W[k,c];  gW[k,c] += graw_k in_c;  gb += graw;
//   ggamma += gout xh;  gbeta += gout
// blockIdx.y = c-tile t of width CT: accumulates gW[:, t*CT .. t*CT+CT) in
// registers; tile 0 also writes gin and (EXTRA) the gb/ggamma/gbeta sums; when
// the extras do not fit next to the tile (KMAX > 8) they get their own y index.
template <int KMAX, int CT>
__global__ void __launch_bounds__(kPB)
project_bwd_k(ProjArgs a, const float *__restrict__ W, const float *__restrict__ b,
              const float *__restrict__ g, int ntiles, int extras_inline,
              float *__restrict__ part) {
    extern __shared__ float sm[];
    const ProjParams pp = stage_params(sm, W, b, g, nullptr, a.K, a.C);
    const int K = a.K, C = a.C;
    const int tile = blockIdx.y;
    const bool do_w = tile < ntiles;
    // inline: tile 0 carries all three extras; else y = ntiles + e carries extra e
    const bool do_extra = extras_inline ? tile == 0 : tile >= ntiles;
    const int extra_kind = tile - ntiles;
    const bool do_gin = tile == 0;
    const int c0 = tile * CT;
    constexpr int NE = KMAX <= 8 ? 3 * KMAX : 1;  // registers for the extras
    float acc[KMAX][CT];
    float ex[NE];
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
#pragma unroll
        for (int j = 0; j < CT; ++j) acc[k][j] = 0.0f;
#pragma unroll
    for (int i = 0; i < NE; ++i) ex[i] = 0.0f;

    const int64_t stride = (int64_t)gridDim.x * kPB;
    for (int which = 0; which < a.ninputs; ++which) {
        const float *in = a.in[which];
        const float *gout = a.gout[which];
        float *gin = a.gin[which];
        for (int64_t p = (int64_t)blockIdx.x * kPB + threadIdx.x; p < a.n; p += stride) {
            float v[KMAX];
            project_raw<KMAX>(in, p, a.n, C, K, pp, v);
            const float inv = ln_normalize<KMAX>(v, K, a.eps);  // v = xhat
            float go[KMAX], gr[KMAX];
            float sg = 0.0f, sgx = 0.0f;
#pragma unroll
            for (int k = 0; k < KMAX; ++k) {
                go[k] = k < K ? __ldg(gout + qk_index(a.planar, p, k, a.n, K)) : 0.0f;
                // rounded product, reused below: keeps gg - mean(gg) exactly 0
                // when all gg agree (K == 1), as in the reference
                gr[k] = __fmul_rn(go[k], k < K ? pp.g[k] : 0.0f);
                sg += gr[k];
                sgx = fmaf(gr[k], v[k], sgx);
            }
            const float mg = sg / (float)K, mgx = sgx / (float)K;
#pragma unroll
            for (int k = 0; k < KMAX; ++k)
                gr[k] = k < K ? inv * ((gr[k] - mg) - v[k] * mgx) : 0.0f;
            if (do_extra) {
                if constexpr (KMAX <= 8) {
#pragma unroll
                    for (int k = 0; k < KMAX; ++k) {
                        ex[k] += gr[k];
                        ex[KMAX + k] = fmaf(go[k], v[k], ex[KMAX + k]);
                        ex[2 * KMAX + k] += go[k];
                    }
                }
            }
            if (do_gin && gin) {
                for (int c = 0; c < C; ++c) {
                    const float *wc = pp.W + c;
                    float s = 0.0f;
#pragma unroll
                    for (int k = 0; k < KMAX; ++k)
                        if (k < K) s = fmaf(gr[k], wc[(int64_t)k * C], s);
                    gin[(int64_t)c * a.n + p] += s;
                }
            }
            if (do_w) {
#pragma unroll
                for (int j = 0; j < CT; ++j) {
                    if (c0 + j >= C) break;
                    const float x = __ldg(in + (int64_t)(c0 + j) * a.n + p);
#pragma unroll
                    for (int k = 0; k < KMAX; ++k) acc[k][j] = fmaf(gr[k], x, acc[k][j]);
                }
            }
            if constexpr (KMAX > 8) {
                // dedicated extras tile: acc[k][0] holds gb, ggamma or gbeta
                if (do_extra && !do_w) {
#pragma unroll
                    for (int k = 0; k < KMAX; ++k)
                        acc[k][0] += extra_kind == 0 ? gr[k]
                                     : extra_kind == 1 ? go[k] * v[k] : go[k];
                }
            }
        }
    }

    // fixed-order block reduction of every accumulator -> part[y][x][slot]
    // slots: tile rows [KMAX*CT] then (inline extras) [3*KMAX]
    __shared__ float red[kPB / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int NSLOT = KMAX * CT + NE;
    float *dst = part + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * NSLOT;
    auto reduce_slot = [&](float val, int slot) {
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) val += __shfl_xor_sync(0xffffffffu, val, m);
        if (lane == 0) red[wid] = val;
        __syncthreads();
        if (threadIdx.x == 0) {
            float s = 0.0f;
#pragma unroll
            for (int i = 0; i < kPB / 32; ++i) s += red[i];
            dst[slot] = s;
        }
        __syncthreads();
    };
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
#pragma unroll
        for (int j = 0; j < CT; ++j) reduce_slot(acc[k][j], k * CT + j);
#pragma unroll
    for (int i = 0; i < NE; ++i) reduce_slot(ex[i], KMAX * CT + i);
}

// sum the per-CTA partials (fixed order) and accumulate into the parameter
// gradients.  One block per output value.
template <int KMAX, int CT>
__global__ void __launch_bounds__(kPB)
project_bwd_final_k(const float *__restrict__ part, int nparts, int ntiles, int extras_inline,
                    int K, int C, float *__restrict__ gW, float *__restrict__ gb,
                    float *__restrict__ gg, float *__restrict__ gbe) {
    constexpr int NE = KMAX <= 8 ? 3 * KMAX : 1;
    constexpr int NSLOT = KMAX * CT + NE;
    const int o = blockIdx.x;  // output id: [0, K*C) weights, then 3K extras
    int y, slot;
    float *target;
    if (o < K * C) {
        const int k = o / C, c = o % C;
        y = c / CT;
        slot = k * CT + (c % CT);
        target = gW ? gW + o : nullptr;
    } else {
        const int e = (o - K * C) / K, k = (o - K * C) % K;  // e: 0 gb, 1 gamma, 2 beta
        if (extras_inline) {
            y = 0;
            slot = KMAX * CT + e * KMAX + k;
        } else {
            y = ntiles + e;
            slot = k * CT;
        }
        target = e == 0 ? (gb ? gb + k : nullptr) : e == 1 ? (gg ? gg + k : nullptr)
                                                           : (gbe ? gbe + k : nullptr);
    }
    if (!target) return;
    float v = 0.0f;
    for (int i = threadIdx.x; i < nparts; i += kPB)
        v += part[((int64_t)y * nparts + i) * NSLOT + slot];
    __shared__ float s[kPB];
    s[threadIdx.x] = v;
    __syncthreads();
    for (int m = kPB / 2; m > 0; m >>= 1) {
        if (threadIdx.x < m) s[threadIdx.x] += s[threadIdx.x + m];
        __syncthreads();
    }
    if (threadIdx.x == 0) *target += s[0];
}

inline size_t proj_smem(int K, int C) {
    const int need = K * C + 3 * K;
    return need <= kSmemW ? (size_t)need * sizeof(float) : 0;
}

template <int KMAX, int CT>
mdg_status project_bwd_launch(const ProjArgs &a, const float *W, const float *b,
                              const float *g, float *gW, float *gb, float *gg, float *gbe,
                              cudaStream_t st) {
    const int ntiles = (a.C + CT - 1) / CT;
    const bool want_extra = gb || gg || gbe;
    const int extras_inline = KMAX <= 8;
    const int ny = ntiles + ((!extras_inline && want_extra) ? 3 : 0);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t blocks_needed = (a.n + kPB - 1) / kPB;
    const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(blocks_needed, (int64_t)sms * 4 / std::max(1, ny) + 1));
    constexpr int NE = KMAX <= 8 ? 3 * KMAX : 1;
    constexpr int NSLOT = KMAX * CT + NE;
    Scratch part;
    MDG_CUDA_TRY(part.alloc((size_t)ny * gx * NSLOT * sizeof(float), st));
    const size_t smem = proj_smem(a.K, a.C);
    project_bwd_k<KMAX, CT><<<dim3(gx, ny), kPB, smem, st>>>(a, W, b, g, ntiles, extras_inline,
                                                            part.as<float>());
    MDG_LAUNCHED();
    if (gW || want_extra) {
        project_bwd_final_k<KMAX, CT><<<a.K * a.C + 3 * a.K, kPB, 0, st>>>(
            part.as<float>(), gx, ntiles, extras_inline, a.K, a.C, gW, gb, gg, gbe);
        MDG_LAUNCHED();
    }
    return MDG_OK;
}

}  // namespace mdg

using namespace mdg;

namespace {
mdg_status check_proj(int C, int64_t n, int K, int layout) {
    MDG_REQUIRE(C >= 1, "linear_proj: channel count must be >= 1");
    MDG_REQUIRE(K >= 1, "linear_proj: output width must be >= 1");
    MDG_REQUIRE(n >= 0 && n < (int64_t(1) << 31), "linear_proj: invalid voxel count");
    MDG_REQUIRE(layout == MDG_QK_POSMAJOR || layout == MDG_QK_PLANAR,
                "project_qk: unknown layout");
    return MDG_OK;
}
}  // namespace

extern "C" {

mdg_status mdg_project_qk_fwd(const float *f, const float *m, int C, int64_t n,
                              const float *weight, const float *bias, const float *ln_g,
                              const float *ln_b, int K, int layout, float *Q, float *Kout,
                              void *stream) {
    mdg_status s = check_proj(C, n, K, layout);
    if (s != MDG_OK) return s;
    if (n == 0) return MDG_OK;
    MDG_REQUIRE(f && weight && bias && ln_g && ln_b && Q, "project_qk: null pointer");
    MDG_REQUIRE(!m == !Kout, "project_qk: m and K must both be given or both be NULL");
    ProjArgs a{};
    a.in[0] = f;
    a.out[0] = Q;
    a.in[1] = m;
    a.out[1] = Kout;
    a.ninputs = m ? 2 : 1;
    a.C = C;
    a.K = K;
    a.n = n;
    a.eps = 1e-5f;
    a.planar = layout == MDG_QK_PLANAR;
    cudaStream_t st = S_(stream);
    const dim3 grid(grid1d(n, kPB), a.ninputs);
    const size_t smem = proj_smem(K, C);
    if (K <= 8) project_fwd_k<8><<<grid, kPB, smem, st>>>(a, weight, bias, ln_g, ln_b);
    else if (K <= 16) project_fwd_k<16><<<grid, kPB, smem, st>>>(a, weight, bias, ln_g, ln_b);
    else if (K <= 32) project_fwd_k<32><<<grid, kPB, smem, st>>>(a, weight, bias, ln_g, ln_b);
    else if (K <= 64) project_fwd_k<64><<<grid, kPB, smem, st>>>(a, weight, bias, ln_g, ln_b);
    else project_fwd_wide_k<<<grid, kPB, 0, st>>>(a, weight, bias, ln_g, ln_b);
    MDG_LAUNCHED();
    return MDG_OK;
}

mdg_status mdg_project_qk_bwd(const float *f, const float *m, int C, int64_t n,
                              const float *weight, const float *bias, const float *ln_g, int K,
                              int layout, const float *gQ, const float *gK, float *gf,
                              float *gm, float *gweight, float *gbias, float *gln_g,
                              float *gln_b, void *stream) {
    mdg_status s = check_proj(C, n, K, layout);
    if (s != MDG_OK) return s;
    if (n == 0) return MDG_OK;
    MDG_REQUIRE(K <= 64, "project_qk_bwd: K > 64 not supported by the B200 path");
    MDG_REQUIRE(f && weight && bias && ln_g && gQ, "project_qk_bwd: null pointer");
    MDG_REQUIRE(!m == !gK, "project_qk_bwd: m and gK must both be given or both be NULL");
    ProjArgs a{};
    a.in[0] = f;
    a.gout[0] = gQ;
    a.gin[0] = gf;
    a.in[1] = m;
    a.gout[1] = gK;
    a.gin[1] = gm;
    a.ninputs = m ? 2 : 1;
    a.C = C;
    a.K = K;
    a.n = n;
    a.eps = 1e-5f;
    a.planar = layout == MDG_QK_PLANAR;
    cudaStream_t st = S_(stream);
    if (K <= 8) return project_bwd_launch<8, 8>(a, weight, bias, ln_g, gweight, gbias, gln_g, gln_b, st);
    if (K <= 16) return project_bwd_launch<16, 4>(a, weight, bias, ln_g, gweight, gbias, gln_g, gln_b, st);
    if (K <= 32) return project_bwd_launch<32, 2>(a, weight, bias, ln_g, gweight, gbias, gln_g, gln_b, st);
    return project_bwd_launch<64, 1>(a, weight, bias, ln_g, gweight, gbias, gln_g, gln_b, st);
}

}  // extern "C"
