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

struct ProjArgs {
    const float *in[2];
    float *out[2];
    const float *gout[2];
    float *gin[2];
    float *graw[2];  // two-phase backward: pre-norm gradients {K, n} written here
    int gin_set;     // bit i: overwrite gin[i] instead of accumulating (internal callers)
    int ninputs;
    int C, K;
    int64_t n;
    float eps;
    int planar;
};

// pick one of the two inputs without dynamically indexing the parameter struct
// (a runtime index would copy ProjArgs into local memory in every thread)
template <typename T>
__device__ __forceinline__ T pick(int which, T a0, T a1) {
    return which ? a1 : a0;
}

__device__ __forceinline__ int64_t qk_index(int planar, int64_t p, int k, int64_t n, int K) {
    return planar ? (int64_t)k * n + p : p * K + k;
}

// Shared-memory parameter block, rows padded to KP = KMAX rounded up to 4 and
// zero-filled beyond K, so the per-channel inner loops need no guards:
//   Wt[C][KP] (W transposed: one channel's K weights contiguous) | b | g | be
template <int KMAX>
struct Pad {
    static constexpr int KP = (KMAX + 3) & ~3;
};

inline size_t proj_smem_bytes(int KMAX_, int C) {
    const int KP = (KMAX_ + 3) & ~3;
    return (size_t)(C + 3) * KP * sizeof(float);
}

template <int KMAX>
__device__ __forceinline__ void stage_params(float *sm, const float *W, const float *b,
                                             const float *g, const float *be, int K, int C) {
    constexpr int KP = Pad<KMAX>::KP;
    for (int i = threadIdx.x; i < C * KP; i += blockDim.x) {
        const int c = i / KP, k = i % KP;
        sm[i] = k < K ? W[(int64_t)k * C + c] : 0.0f;
    }
    float *tail = sm + C * KP;
    for (int k = threadIdx.x; k < KP; k += blockDim.x) {
        tail[k] = k < K ? b[k] : 0.0f;
        tail[KP + k] = (k < K && g) ? g[k] : 0.0f;
        tail[2 * KP + k] = (k < K && be) ? be[k] : 0.0f;
    }
    __syncthreads();
}

// raw[k] = b[k] + sum_c W[k,c] in[c,p]  (channel order, as ops.hpp:403-406);
// rows k >= K come out exactly 0
template <int KMAX>
__device__ __forceinline__ void project_raw(const float *__restrict__ in, int64_t n, int C,
                                            const float *sm, float (&raw)[KMAX]) {
    constexpr int KP = Pad<KMAX>::KP;
    const float *sb = sm + C * KP;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) raw[k] = sb[k];
    // channels in batches of 8: the 8 independent loads are in flight together
    // (a plain runtime-C loop serialises one global-load latency per channel)
    int c = 0;
    for (; c + 8 <= C; c += 8) {
        float x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = __ldg(in + (int64_t)(c + j) * n);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float *wc = sm + (c + j) * KP;
#pragma unroll
            for (int k = 0; k < KMAX; ++k) raw[k] = fmaf(wc[k], x[j], raw[k]);
        }
    }
    for (; c < C; ++c) {
        const float x = __ldg(in + (int64_t)c * n);
        const float *wc = sm + c * KP;
#pragma unroll
        for (int k = 0; k < KMAX; ++k) raw[k] = fmaf(wc[k], x, raw[k]);
    }
}

// two-pass mean / biased variance (ops.hpp:447-454); raw -> xhat in place
// (rows >= K set to 0); returns inv = 1/sqrt(var + eps)
template <int KMAX>
__device__ __forceinline__ float ln_normalize(float (&raw)[KMAX], int K, float eps) {
    float mean = 0.0f;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) mean += raw[k];  // padded rows are 0
    mean /= (float)K;
    float var = 0.0f;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
        const float t = k < K ? raw[k] - mean : 0.0f;
        var = fmaf(t, t, var);
    }
    var /= (float)K;
    const float inv = 1.0f / sqrtf(var + eps);
#pragma unroll
    for (int k = 0; k < KMAX; ++k) raw[k] = k < K ? (raw[k] - mean) * inv : 0.0f;
    return inv;
}

// EXACT: K == KMAX known at compile time (the fine levels' K = 6)
template <int KMAX, bool EXACT>
__global__ void __launch_bounds__(kPB)
project_fwd_k(ProjArgs a, const float *__restrict__ W, const float *__restrict__ b,
              const float *__restrict__ g, const float *__restrict__ be) {
    extern __shared__ __align__(16) float sm[];
    constexpr int KP = Pad<KMAX>::KP;
    const int K = EXACT ? KMAX : a.K, C = a.C;
    const int64_t n = a.n;
    stage_params<KMAX>(sm, W, b, g, be, K, C);
    const int which = blockIdx.y;
    const int64_t p = (int64_t)blockIdx.x * kPB + threadIdx.x;
    if (p >= n) return;
    float v[KMAX];
    project_raw<KMAX>(pick(which, a.in[0], a.in[1]) + p, n, C, sm, v);
    ln_normalize<KMAX>(v, K, a.eps);
    float *out = pick(which, a.out[0], a.out[1]);
    const float *sg = sm + (C + 1) * KP, *sbe = sm + (C + 2) * KP;
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
        if (k < K) out[qk_index(a.planar, p, k, n, K)] = fmaf(sg[k], v[k], sbe[k]);
}

// K > 64: raw values go through the output buffer (two extra passes over it)
__global__ void __launch_bounds__(kPB)
project_fwd_wide_k(ProjArgs a, const float *__restrict__ W, const float *__restrict__ b,
                   const float *__restrict__ g, const float *__restrict__ be) {
    const int which = blockIdx.y;
    const int64_t p = (int64_t)blockIdx.x * kPB + threadIdx.x;
    if (p >= a.n) return;
    const float *in = pick(which, a.in[0], a.in[1]);
    float *out = pick(which, a.out[0], a.out[1]);
    const int K = a.K, C = a.C;
    float mean = 0.0f;
    for (int k = 0; k < K; ++k) {
        float s = b[k];
        for (int c = 0; c < C; ++c)
            s = fmaf(__ldg(W + (int64_t)k * C + c), __ldg(in + (int64_t)c * a.n + p), s);
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
// registers; tile 0 also writes gin and (inline, KMAX <= 8) the gb / ggamma /
// gbeta sums; for wider K each extra gets its own y index (ntiles + e).
template <int KMAX, int CT>
struct BwdShape {
    static constexpr bool kInline = KMAX <= 8;
    static constexpr int NE = kInline ? 3 * KMAX : 1;
    static constexpr int NSLOT = KMAX * CT + NE;
};

#ifndef MDG_PROJ_BWD_MINB
#define MDG_PROJ_BWD_MINB 4  // measured: 697 vs 750 (2) vs 786 us (3) at L1 (tools/exp/proj_minb.sh)
#endif
template <int KMAX, int CT, bool EXACT>
__global__ void __launch_bounds__(kPB, KMAX <= 6 ? MDG_PROJ_BWD_MINB : 1)
project_bwd_k(ProjArgs a, const float *__restrict__ W, const float *__restrict__ b,
              const float *__restrict__ g, int ntiles, float *__restrict__ part) {
    extern __shared__ __align__(16) float sm[];
    using Sh = BwdShape<KMAX, CT>;
    constexpr int KP = Pad<KMAX>::KP;
    const int K = EXACT ? KMAX : a.K, C = a.C;
    const int64_t n = a.n;
    stage_params<KMAX>(sm, W, b, g, nullptr, K, C);
    const float *sg = sm + (C + 1) * KP;
    const int tile = blockIdx.y;
    float *const graw_out0 = a.graw[0];
    const bool do_w = tile < ntiles && !graw_out0;
    const bool do_extra = Sh::kInline ? tile == 0 : tile >= ntiles;
    const int extra_kind = tile - ntiles;
    const bool do_gin = tile == 0;
    const int c0 = tile * CT;
    float acc[KMAX][CT];
    float ex[Sh::NE];
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
#pragma unroll
        for (int j = 0; j < CT; ++j) acc[k][j] = 0.0f;
#pragma unroll
    for (int i = 0; i < Sh::NE; ++i) ex[i] = 0.0f;

    const int64_t stride = (int64_t)gridDim.x * kPB;
    for (int which = 0; which < a.ninputs; ++which) {
        const float *in = pick(which, a.in[0], a.in[1]);
        const float *gout = pick(which, a.gout[0], a.gout[1]);
        float *gin = pick(which, a.gin[0], a.gin[1]);
        for (int64_t p = (int64_t)blockIdx.x * kPB + threadIdx.x; p < n; p += stride) {
            const float *ip = in + p;
            float v[KMAX];
            project_raw<KMAX>(ip, n, C, sm, v);
            const float inv = ln_normalize<KMAX>(v, K, a.eps);  // v = xhat, 0 beyond K
            float go[KMAX], gr[KMAX];
            float sgs = 0.0f, sgx = 0.0f;
#pragma unroll
            for (int k = 0; k < KMAX; ++k) {
                go[k] = k < K ? __ldg(gout + qk_index(a.planar, p, k, n, K)) : 0.0f;
                // rounded product, reused below: keeps gg - mean(gg) exactly 0
                // when all gg agree (K == 1), as in the reference
                gr[k] = __fmul_rn(go[k], sg[k]);
                sgs += gr[k];
                sgx = fmaf(gr[k], v[k], sgx);
            }
            const float mg = sgs / (float)K, mgx = sgx / (float)K;
#pragma unroll
            for (int k = 0; k < KMAX; ++k)
                gr[k] = k < K ? inv * ((gr[k] - mg) - v[k] * mgx) : 0.0f;
            if constexpr (Sh::kInline) {
                if (do_extra) {
#pragma unroll
                    for (int k = 0; k < KMAX; ++k) {
                        ex[k] += gr[k];
                        ex[KMAX + k] = fmaf(go[k], v[k], ex[KMAX + k]);
                        ex[2 * KMAX + k] += go[k];
                    }
                }
            } else {
                if (do_extra) {
#pragma unroll
                    for (int k = 0; k < KMAX; ++k)
                        acc[k][0] += extra_kind == 0 ? gr[k]
                                     : extra_kind == 1 ? go[k] * v[k] : go[k];
                }
            }
            if (do_gin && graw_out0) {
                float *go_ = pick(which, graw_out0, a.graw[1]) + p;
#pragma unroll
                for (int k = 0; k < KMAX; ++k)
                    if (k < K) go_[(int64_t)k * n] = gr[k];
            }
            if (do_gin && gin) {
                // read-modify-write in batches of 4 with all loads first: the
                // compiler cannot prove gp[c*n] and gp[(c+1)*n] never alias,
                // so an interleaved loop would serialise load-after-store
                float *gp = gin + p;
                const bool set = (a.gin_set >> which) & 1;
                for (int c = 0; c < C; c += 4) {
                    float old[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        old[j] = (c + j < C && !set) ? gp[(int64_t)(c + j) * n] : 0.0f;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (c + j >= C) break;
                        const float *wc = sm + (c + j) * KP;
                        float s = 0.0f;
#pragma unroll
                        for (int k = 0; k < KMAX; ++k) s = fmaf(gr[k], wc[k], s);
                        gp[(int64_t)(c + j) * n] = set ? s : old[j] + s;
                    }
                }
            }
            if (do_w) {
#pragma unroll
                for (int j = 0; j < CT; ++j) {
                    if (c0 + j < C) {
                        const float x = __ldg(ip + (int64_t)(c0 + j) * n);
#pragma unroll
                        for (int k = 0; k < KMAX; ++k) acc[k][j] = fmaf(gr[k], x, acc[k][j]);
                    }
                }
            }
        }
    }

    // fixed-order block reduction of every accumulator -> part[y][x][slot]
    __shared__ float red[kPB / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float *dst = part + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * Sh::NSLOT;
    auto reduce_slot = [&](float val, int slot) {
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) val += __shfl_xor_sync(0xffffffffu, val, m);
        if (lane == 0) red[wid] = val;
        __syncthreads();
        if (threadIdx.x == 0) {
            float t = 0.0f;
#pragma unroll
            for (int i = 0; i < kPB / 32; ++i) t += red[i];
            dst[slot] = t;
        }
        __syncthreads();
    };
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
#pragma unroll
        for (int j = 0; j < CT; ++j) reduce_slot(acc[k][j], k * CT + j);
#pragma unroll
    for (int i = 0; i < Sh::NE; ++i) reduce_slot(ex[i], KMAX * CT + i);
}

// sum the per-CTA partials (fixed order) and accumulate into the parameter
// gradients.  One block per output value.
template <int KMAX, int CT>
__global__ void __launch_bounds__(kPB)
project_bwd_final_k(const float *__restrict__ part, int nparts, int ntiles, int K, int C,
                    float *__restrict__ gW, float *__restrict__ gb, float *__restrict__ gg,
                    float *__restrict__ gbe) {
    using Sh = BwdShape<KMAX, CT>;
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
        if (Sh::kInline) {
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
        v += part[((int64_t)y * nparts + i) * Sh::NSLOT + slot];
    __shared__ float s[kPB];
    s[threadIdx.x] = v;
    __syncthreads();
    for (int m = kPB / 2; m > 0; m >>= 1) {
        if (threadIdx.x < m) s[threadIdx.x] += s[threadIdx.x + m];
        __syncthreads();
    }
    if (threadIdx.x == 0) *target += s[0];
}

// Two-phase weight gradient for multi-tile levels (C > CT): instead of
// recomputing the projection once per channel tile, phase 1 writes the
// pre-norm gradients graw {K, n} and phase 2 forms gW[k, c] = sum_p graw[k,p]
// in[c,p] as a chunked outer-product reduction (shared-memory staged chunks of
// kGP voxels, kGO outputs per thread, per-CTA partials, fixed-order final sum).
constexpr int kGP = 32, kGO = 4;

__global__ void __launch_bounds__(kPB)
gram_k(const float *__restrict__ A0, const float *__restrict__ A1, const float *__restrict__ B0,
       const float *__restrict__ B1, int ninputs, int K, int C, int64_t n,
       float *__restrict__ part) {
    extern __shared__ __align__(16) float gsm[];
    float *As = gsm;            // [K][kGP]
    float *Bs = gsm + K * kGP;  // [C][kGP]
    const int KC = K * C;
    const int obase = blockIdx.y * kPB * kGO;
    float acc[kGO];
    int kk[kGO], cc[kGO];
#pragma unroll
    for (int j = 0; j < kGO; ++j) {
        acc[j] = 0.0f;
        const int o = obase + j * kPB + threadIdx.x;
        kk[j] = o < KC ? o / C : -1;
        cc[j] = o < KC ? o % C : 0;
    }
    const int64_t nchunks = (n + kGP - 1) / kGP;
    for (int which = 0; which < ninputs; ++which) {
        const float *A = which ? A1 : A0;
        const float *B = which ? B1 : B0;
        for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
            const int64_t p0 = ch * kGP;
            __syncthreads();
            for (int i = threadIdx.x; i < (K + C) * kGP; i += kPB) {
                const int r = i / kGP, q = i % kGP;
                const int64_t pp = p0 + q;
                float v = 0.0f;
                if (pp < n) v = r < K ? __ldg(A + (int64_t)r * n + pp) : __ldg(B + (int64_t)(r - K) * n + pp);
                gsm[i] = v;
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < kGO; ++j) {
                if (kk[j] < 0) continue;
                const float *ar = As + kk[j] * kGP, *br = Bs + cc[j] * kGP;
                float t = acc[j];
#pragma unroll 8
                for (int q = 0; q < kGP; ++q) t = fmaf(ar[q], br[q], t);
                acc[j] = t;
            }
        }
    }
    float *dst = part + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * (kPB * kGO);
#pragma unroll
    for (int j = 0; j < kGO; ++j) dst[j * kPB + threadIdx.x] = acc[j];
}

__global__ void __launch_bounds__(kPB)
gram_final_k(const float *__restrict__ part, int nparts, int KC, float *__restrict__ gW) {
    const int o = blockIdx.x;
    const int y = o / (kPB * kGO), lo = o % (kPB * kGO);
    float v = 0.0f;
    for (int i = threadIdx.x; i < nparts; i += kPB)
        v += part[((int64_t)y * nparts + i) * (kPB * kGO) + lo];
    __shared__ float s[kPB];
    s[threadIdx.x] = v;
    __syncthreads();
    for (int m = kPB / 2; m > 0; m >>= 1) {
        if (threadIdx.x < m) s[threadIdx.x] += s[threadIdx.x + m];
        __syncthreads();
    }
    if (threadIdx.x == 0 && o < KC) gW[o] += s[0];
}

// the weight gradient of the large two-phase level (K = 6, C = 16): each
// thread streams its own voxels (coalesced global loads) and keeps all 96
// (k, c) sums in registers; one fixed-order block reduction per block, then
// gram16_final_k adds the block partials in block order
template <int K, int C>  // K: rows of A per block tile (blockIdx.y), C: all of B
__global__ void __launch_bounds__(kPB, 1)
gram16_k(const float *__restrict__ A0, const float *__restrict__ A1, const float *__restrict__ B0,
         const float *__restrict__ B1, int ninputs, int64_t n, float *__restrict__ part) {
    A0 += (int64_t)blockIdx.y * K * n;
    if (A1) A1 += (int64_t)blockIdx.y * K * n;
    float acc[K][C];
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int c = 0; c < C; ++c) acc[k][c] = 0.0f;
    for (int which = 0; which < ninputs; ++which) {
        const float *A = which ? A1 : A0;
        const float *B = which ? B1 : B0;
        for (int64_t p = (int64_t)blockIdx.x * kPB + threadIdx.x; p < n;
             p += (int64_t)gridDim.x * kPB) {
            float a[K], b[C];
#pragma unroll
            for (int k = 0; k < K; ++k) a[k] = __ldg(A + (int64_t)k * n + p);
#pragma unroll
            for (int c = 0; c < C; ++c) b[c] = __ldg(B + (int64_t)c * n + p);
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int c = 0; c < C; ++c) acc[k][c] = fmaf(a[k], b[c], acc[k][c]);
        }
    }
    __shared__ float red[kPB / 32][K * C];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int c = 0; c < C; ++c) {
            float v = acc[k][c];
#pragma unroll
            for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
            if (lane == 0) red[wid][k * C + c] = v;
        }
    __syncthreads();
    if (threadIdx.x < K * C) {
        float v = 0.0f;
#pragma unroll
        for (int w8 = 0; w8 < kPB / 32; ++w8) v += red[w8][threadIdx.x];
        part[((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * (K * C) + threadIdx.x] = v;
    }
}

// gW[k][c] += sum over blocks (fixed order); tiles of KT rows of k
__global__ void __launch_bounds__(kPB)
gram16_final_k(const float *__restrict__ part, int nblk, int KT, int K, int C,
               float *__restrict__ gW) {
    const int o = blockIdx.x * kPB + threadIdx.x;
    if (o >= K * C) return;
    const int k = o / C, c = o % C, y = k / KT, kk = k % KT;
    float v = 0.0f;
    for (int b = 0; b < nblk; ++b) v += part[((int64_t)y * nblk + b) * (KT * C) + kk * C + c];
    gW[o] += v;
}

template <typename Kern>
cudaError_t allow_smem(Kern k, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int KMAX, bool EXACT>
mdg_status project_fwd_launch(const ProjArgs &a, const float *W, const float *b, const float *g,
                              const float *be, cudaStream_t st) {
    const size_t smem = proj_smem_bytes(KMAX, a.C);
    MDG_CUDA_TRY(allow_smem(project_fwd_k<KMAX, EXACT>, smem));
    const dim3 grid(grid1d(a.n, kPB), a.ninputs);
    project_fwd_k<KMAX, EXACT><<<grid, kPB, smem, st>>>(a, W, b, g, be);
    MDG_LAUNCHED();
    return MDG_OK;
}

template <int KMAX, int CT, bool EXACT>
mdg_status project_bwd_launch(const ProjArgs &a0, const float *W, const float *b,
                              const float *g, float *gW, float *gb, float *gg, float *gbe,
                              cudaStream_t st) {
    using Sh = BwdShape<KMAX, CT>;
    ProjArgs a = a0;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t blocks_needed = (a.n + kPB - 1) / kPB;
    const int per_sm = KMAX <= 6 ? MDG_PROJ_BWD_MINB : 1;
    // one channel tile: gW accumulates in registers next to everything else;
    // several: two-phase (graw to scratch, then the chunked reduction)
    const bool two_phase = gW && a.C > CT;
    Scratch graw;
    if (two_phase) {
        MDG_CUDA_TRY(graw.alloc((size_t)a.ninputs * a.K * a.n * sizeof(float), st));
        a.graw[0] = graw.as<float>();
        a.graw[1] = a.ninputs > 1 ? graw.as<float>() + (int64_t)a.K * a.n : nullptr;
    }
    const int ntiles = two_phase ? 1 : (a.C + CT - 1) / CT;
    const bool want_extra = gb || gg || gbe;
    const int ny = ntiles + ((!Sh::kInline && want_extra) ? 3 : 0);
    const int gx = (int)std::max<int64_t>(
        1, std::min<int64_t>(blocks_needed, ((int64_t)sms * per_sm * 2 + ny - 1) / ny));
    Scratch part;
    MDG_CUDA_TRY(part.alloc((size_t)ny * gx * Sh::NSLOT * sizeof(float), st));
    const size_t smem = proj_smem_bytes(KMAX, a.C);
    MDG_CUDA_TRY(allow_smem(project_bwd_k<KMAX, CT, EXACT>, smem));
    project_bwd_k<KMAX, CT, EXACT><<<dim3(gx, ny), kPB, smem, st>>>(a, W, b, g, ntiles,
                                                                    part.as<float>());
    MDG_LAUNCHED();
    if ((gW && !two_phase) || want_extra) {
        project_bwd_final_k<KMAX, CT><<<a.K * a.C + 3 * a.K, kPB, 0, st>>>(
            part.as<float>(), gx, ntiles, a.K, a.C, two_phase ? nullptr : gW, gb, gg, gbe);
        MDG_LAUNCHED();
    }
    if (two_phase && ((a.K == 6 && a.C == 16) || (a.K == 12 && a.C == 32))) {
        // register-tiled weight gradient for the two large two-phase levels
        const int KT = a.C == 16 ? 6 : 3, nty = a.K / KT;
        const int nblk = (int)std::max<int64_t>(
            1, std::min<int64_t>((a.n + kPB - 1) / kPB, (int64_t)sms * 2 / nty));
        Scratch gpart;
        MDG_CUDA_TRY(gpart.alloc((size_t)nty * nblk * KT * a.C * sizeof(float), st));
        if (a.C == 16)
            gram16_k<6, 16><<<dim3(nblk, nty), kPB, 0, st>>>(a.graw[0], a.graw[1], a.in[0],
                                                             a.in[1], a.ninputs, a.n,
                                                             gpart.as<float>());
        else
            gram16_k<3, 32><<<dim3(nblk, nty), kPB, 0, st>>>(a.graw[0], a.graw[1], a.in[0],
                                                             a.in[1], a.ninputs, a.n,
                                                             gpart.as<float>());
        MDG_LAUNCHED();
        gram16_final_k<<<(a.K * a.C + kPB - 1) / kPB, kPB, 0, st>>>(gpart.as<float>(), nblk, KT,
                                                                   a.K, a.C, gW);
        MDG_LAUNCHED();
    } else if (two_phase) {
        const int KC = a.K * a.C;
        const int gy = (KC + kPB * kGO - 1) / (kPB * kGO);
        const int64_t nchunks = (a.n + kGP - 1) / kGP;
        const int ggx = (int)std::max<int64_t>(1, std::min<int64_t>(nchunks, (int64_t)sms * 4 / gy + 1));
        const size_t gsmem = (size_t)(a.K + a.C) * kGP * sizeof(float);
        MDG_CUDA_TRY(allow_smem(gram_k, gsmem));
        Scratch gpart;
        MDG_CUDA_TRY(gpart.alloc((size_t)gy * ggx * kPB * kGO * sizeof(float), st));
        gram_k<<<dim3(ggx, gy), kPB, gsmem, st>>>(a.graw[0], a.graw[1], a.in[0], a.in[1],
                                                  a.ninputs, a.K, a.C, a.n, gpart.as<float>());
        MDG_LAUNCHED();
        gram_final_k<<<KC, kPB, 0, st>>>(gpart.as<float>(), ggx, KC, gW);
        MDG_LAUNCHED();
    }
    return MDG_OK;
}

// ------------------------------------------------- backward, K > 64
// The large preset's coarse levels (K = S*hd up to 32*12 = 384) keep the
// per-voxel values in global scratch instead of registers.  Simple and
// deterministic (fixed loops, no atomics); these levels hold few voxels.
// raw pre-norm values Y {K, n}
__global__ void wide_raw_k(const float *__restrict__ in, const float *__restrict__ W,
                           const float *__restrict__ b, int C, int K, int64_t n,
                           float *__restrict__ Y) {
    const int64_t i = (int64_t)blockIdx.x * kPB + threadIdx.x;
    if (i >= (int64_t)K * n) return;
    const int k = (int)(i / n);
    const int64_t p = i - (int64_t)k * n;
    float s = b[k];
    for (int c = 0; c < C; ++c) s = fmaf(__ldg(W + (int64_t)k * C + c), __ldg(in + (int64_t)c * n + p), s);
    Y[i] = s;
}
// per voxel (ops.hpp:470-493): Y <- xh, G <- graw (the pre-norm gradient)
__global__ void wide_ln_bwd_k(float *__restrict__ Y, float *__restrict__ G,
                              const float *__restrict__ gout, const float *__restrict__ gamma,
                              int K, int64_t n, int planar, float eps) {
    const int64_t p = (int64_t)blockIdx.x * kPB + threadIdx.x;
    if (p >= n) return;
    float mean = 0.0f;
    for (int k = 0; k < K; ++k) mean += Y[(int64_t)k * n + p];
    mean /= (float)K;
    float var = 0.0f;
    for (int k = 0; k < K; ++k) {
        const float t = Y[(int64_t)k * n + p] - mean;
        var = fmaf(t, t, var);
    }
    var /= (float)K;
    const float inv = 1.0f / sqrtf(var + eps);
    float sg = 0.0f, sgx = 0.0f;
    for (int k = 0; k < K; ++k) {
        const float xh = (Y[(int64_t)k * n + p] - mean) * inv;
        const float go = gout[qk_index(planar, p, k, n, K)];
        sg = fmaf(go, gamma[k], sg);
        sgx = fmaf(go * gamma[k], xh, sgx);
    }
    const float mg = sg / (float)K, mgx = sgx / (float)K;
    for (int k = 0; k < K; ++k) {
        const float xh = (Y[(int64_t)k * n + p] - mean) * inv;
        const float go = gout[qk_index(planar, p, k, n, K)];
        Y[(int64_t)k * n + p] = xh;
        G[(int64_t)k * n + p] = inv * (go * gamma[k] - mg - xh * mgx);
    }
}
// gin[c] (+)= sum_k G[k] W[k,c]
__global__ void wide_gin_k(const float *__restrict__ G, const float *__restrict__ W, int C, int K,
                           int64_t n, float *__restrict__ gin, int set) {
    const int64_t i = (int64_t)blockIdx.x * kPB + threadIdx.x;
    if (i >= (int64_t)C * n) return;
    const int c = (int)(i / n);
    const int64_t p = i - (int64_t)c * n;
    float s = 0.0f;
    for (int k = 0; k < K; ++k) s = fmaf(G[(int64_t)k * n + p], __ldg(W + (int64_t)k * C + c), s);
    gin[i] = set ? s : gin[i] + s;
}
// parameter gradients of one input (accumulated across the inputs in order):
// gW[k,c] += sum_p G[k,p] in[c,p];  gb[k] += sum G;  ggamma += sum gout xh;
// gbeta += sum gout.  One thread per (k, c) / per k, voxels in order.
__global__ void wide_param_k(const float *__restrict__ G, const float *__restrict__ X,
                             const float *__restrict__ in, const float *__restrict__ gout, int C,
                             int K, int64_t n, int planar, float *__restrict__ gW,
                             float *__restrict__ gb, float *__restrict__ gg,
                             float *__restrict__ gbe) {
    const int64_t i = (int64_t)blockIdx.x * kPB + threadIdx.x;
    if (i < (int64_t)K * C && gW) {
        const int k = (int)(i / C), c = (int)(i - (int64_t)k * C);
        float s = 0.0f;
        for (int64_t p = 0; p < n; ++p) s = fmaf(G[(int64_t)k * n + p], __ldg(in + (int64_t)c * n + p), s);
        gW[i] += s;
    }
    if (i < K) {
        const int k = (int)i;
        float sb = 0.0f, sg = 0.0f, sbe = 0.0f;
        for (int64_t p = 0; p < n; ++p) {
            const float go = gout[qk_index(planar, p, k, n, K)];
            sb += G[(int64_t)k * n + p];
            sg = fmaf(go, X[(int64_t)k * n + p], sg);
            sbe += go;
        }
        if (gb) gb[k] += sb;
        if (gg) gg[k] += sg;
        if (gbe) gbe[k] += sbe;
    }
}

static mdg_status project_bwd_wide(const ProjArgs &a, const float *W, const float *b,
                                   const float *g, float *gW, float *gb, float *gg, float *gbe,
                                   cudaStream_t st) {
    const int K = a.K, C = a.C;
    const int64_t n = a.n;
    Scratch ws;
    MDG_CUDA_TRY(ws.alloc((size_t)2 * K * n * sizeof(float), st));
    float *Y = ws.as<float>(), *G = Y + (int64_t)K * n;
    for (int i = 0; i < a.ninputs; ++i) {
        const float *in = a.in[i], *go = a.gout[i];
        float *gi = a.gin[i];
        wide_raw_k<<<grid1d((int64_t)K * n, kPB), kPB, 0, st>>>(in, W, b, C, K, n, Y);
        MDG_LAUNCHED();
        wide_ln_bwd_k<<<grid1d(n, kPB), kPB, 0, st>>>(Y, G, go, g, K, n, a.planar, a.eps);
        MDG_LAUNCHED();
        if (gi) {
            wide_gin_k<<<grid1d((int64_t)C * n, kPB), kPB, 0, st>>>(G, W, C, K, n, gi,
                                                                   (a.gin_set >> i) & 1);
            MDG_LAUNCHED();
        }
        wide_param_k<<<grid1d((int64_t)K * C, kPB), kPB, 0, st>>>(G, Y, in, go, C, K, n,
                                                                 a.planar, gW, gb, gg, gbe);
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
    MDG_REQUIRE(K > 64 || proj_smem_bytes(K, C) <= 200 * 1024,
                "project_qk: C * K too large for the shared-memory weight block");
    if (K == 6) return project_fwd_launch<6, true>(a, weight, bias, ln_g, ln_b, st);
    if (K <= 8) return project_fwd_launch<8, false>(a, weight, bias, ln_g, ln_b, st);
    if (K <= 16) return project_fwd_launch<16, false>(a, weight, bias, ln_g, ln_b, st);
    if (K <= 32) return project_fwd_launch<32, false>(a, weight, bias, ln_g, ln_b, st);
    if (K <= 64) return project_fwd_launch<64, false>(a, weight, bias, ln_g, ln_b, st);
    project_fwd_wide_k<<<dim3(grid1d(n, kPB), a.ninputs), kPB, 0, st>>>(a, weight, bias, ln_g,
                                                                         ln_b);
    MDG_LAUNCHED();
    return MDG_OK;
}

mdg_status mdg_project_qk_bwd(const float *f, const float *m, int C, int64_t n,
                              const float *weight, const float *bias, const float *ln_g, int K,
                              int layout, const float *gQ, const float *gK, float *gf,
                              float *gm, float *gweight, float *gbias, float *gln_g,
                              float *gln_b, void *stream) {
    return mdg::project_qk_bwd_impl(f, m, C, n, weight, bias, ln_g, K, layout, gQ, gK, gf, gm,
                                    gweight, gbias, gln_g, gln_b, 0, S_(stream));
}

}  // extern "C"

namespace mdg {
mdg_status project_qk_bwd_impl(const float *f, const float *m, int C, int64_t n,
                               const float *weight, const float *bias, const float *ln_g, int K,
                               int layout, const float *gQ, const float *gK, float *gf,
                               float *gm, float *gweight, float *gbias, float *gln_g,
                               float *gln_b, int gin_set, cudaStream_t stream) {
    mdg_status s = check_proj(C, n, K, layout);
    if (s != MDG_OK) return s;
    if (n == 0) return MDG_OK;
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
    a.gin_set = gin_set;
    cudaStream_t st = stream;
    if (K > 64 || proj_smem_bytes(K, C) > 200 * 1024)
        return project_bwd_wide(a, weight, bias, ln_g, gweight, gbias, gln_g, gln_b, st);
    // K == 6 (head_dim 6, one head: the fine levels) gets an exact instantiation
    if (K == 6) return project_bwd_launch<6, 8, true>(a, weight, bias, ln_g, gweight, gbias, gln_g, gln_b, st);
    if (K <= 8) return project_bwd_launch<8, 8, false>(a, weight, bias, ln_g, gweight, gbias, gln_g, gln_b, st);
    if (K <= 16) return project_bwd_launch<16, 4, false>(a, weight, bias, ln_g, gweight, gbias, gln_g, gln_b, st);
    if (K <= 32) return project_bwd_launch<32, 2, false>(a, weight, bias, ln_g, gweight, gbias, gln_g, gln_b, st);
    return project_bwd_launch<64, 1, false>(a, weight, bias, ln_g, gweight, gbias, gln_g, gln_b, st);
}

}  // namespace mdg
