// loss.cu — the registration objective on sm_100a:
//   total = NCC(fixed, warp(moving, phi)) + lambda * grad_reg(phi)
// (objective.hpp:39-78, op_boxsum ops.hpp:301-320, kern::boxsum1d ops.hpp:103-125,
// op_grad_reg ops.hpp:326-382).
//
// NCC: the five windowed statistics (sums of f, g, f^2, g^2, f*g over the
// zero-padded (2r+1)^3 box) are three separable box-sum passes over a
// 5-channel product volume; every box sum adds its taps in the reference's
// order, so the statistics are bit-identical to kern::boxsum1d.  Window counts
// are the exact integer products cx*cy*cz (what the reference's box sum of
// ones yields).  The per-voxel cc and the means are deterministic
// fixed-order reductions (fp32 tolerance vs the reference's sequential sum).
// Backward: the per-voxel adjoint of cc goes back through the box sums (a
// zero-padded box sum is self-adjoint, ops.hpp:311) into dL/dwarped, then the
// warp backward gives dL/dphi (+ dL/dmoving); grad_reg adds its stencil.
#include <algorithm>

#include "mdg_common.cuh"

namespace mdg {

constexpr int kLB = 256;
constexpr float kNccEps = 1e-5f;  // objective.hpp:34

struct LDims {
    int h, w, l;
    int n;
};

__device__ __forceinline__ void lxyz(int p, const LDims &d, int &x, int &y, int &z) {
    const int t = p / d.h;
    x = p - t * d.h;
    z = t / d.w;
    y = t - z * d.w;
}

// kern::boxsum1d along `axis` for C channel planes (blockIdx.y = channel).
// Each thread produces kStrip consecutive outputs along the summed axis from
// one register window of taps (each output still adds its own taps t0..t1 in
// order, so the sums are bit-identical to the reference); lanes run along x,
// so every tap load is coalesced.  For the x axis the strip runs along y
// instead (x stays the lane axis).
#ifndef MDG_BOX_STRIP
#define MDG_BOX_STRIP 8  // 4: +30 % box-pass time, 16: register pressure (profiles/experiments/box_strip_r02.log)
#endif
constexpr int kStrip = MDG_BOX_STRIP;
constexpr int kMaxR = 12;

// x pass, one warp per row: the row (zero-padded by R each side) is staged in
// shared memory with coalesced loads, then lane i sums the taps of outputs
// i, i+32, ... in the reference's order (bit-identical to box_axis_k<0>)
constexpr int kRowMax = 2048;  // h + 2R must fit a warp's row buffer
template <int R>
__global__ void __launch_bounds__(kLB)
box_x_rows_k(const float *__restrict__ in, LDims d, float *__restrict__ out) {
    extern __shared__ float rows_sm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int hp = d.h + 2 * R;
    float *row = rows_sm + wid * hp;
    const int c = blockIdx.y;
    const int nrows = d.w * d.l;
    const float *src = in + (int64_t)c * d.n;
    float *dst = out + (int64_t)c * d.n;
    for (int rr = blockIdx.x * (kLB / 32) + wid; rr < nrows; rr += gridDim.x * (kLB / 32)) {
        const float *s = src + (int64_t)rr * d.h;
        for (int i = lane; i < hp; i += 32) {
            const int t = i - R;
            row[i] = (t >= 0 && t < d.h) ? __ldg(s + t) : 0.0f;
        }
        __syncwarp();
        for (int x = lane; x < d.h; x += 32) {
            // taps t = x-R .. x+R clamped to the row: the zero padding must not
            // be added (0 + v == v, but the reference starts at the first
            // in-range tap), so sum only the in-range ones, in order
            const int t0 = max(0, x - R), t1 = min(d.h - 1, x + R);
            float acc = 0.0f;
#pragma unroll
            for (int q = 0; q < 2 * R + 1; ++q) {
                const int t = x - R + q;
                if (t >= t0 && t <= t1) acc = __fadd_rn(acc, row[t + R]);
            }
            dst[(int64_t)rr * d.h + x] = acc;
        }
        __syncwarp();
    }
}

template <int AX, int R>
__global__ void __launch_bounds__(kLB)
box_axis_k(const float *__restrict__ in, LDims d, float *__restrict__ out) {
    constexpr int r = R;
    const int c = blockIdx.y;
    const int len = AX == 0 ? d.h : (AX == 1 ? d.w : d.l);
    const int stride = AX == 0 ? 1 : (AX == 1 ? d.h : d.h * d.w);
    // work item = (x, strip along the pass axis or along y for AX == 0, rest)
    const int hs = AX == 0 ? d.h : d.h;
    const int ns = AX == 0 ? (d.w + kStrip - 1) / kStrip : (len + kStrip - 1) / kStrip;
    const int other = AX == 0 ? d.l : (AX == 1 ? d.l : d.w);
    const int items = hs * ns * other;
    const float *src = in + (int64_t)c * d.n;
    float *dst = out + (int64_t)c * d.n;
    for (int it = blockIdx.x * kLB + threadIdx.x; it < items; it += gridDim.x * kLB) {
        const int x = it % hs;
        const int rest = it / hs;
        const int si = rest % ns, o = rest / ns;
        if (AX == 0) {
            // one output per (x, y) of the strip, taps in order from L1
            const int z = o;
#pragma unroll
            for (int k = 0; k < kStrip; ++k) {
                const int y = si * kStrip + k;
                if (y < d.w) {
                    const float *row = src + ((int64_t)z * d.w + y) * d.h;
                    float s = 0.0f;
#pragma unroll
                    for (int q = 0; q < 2 * R + 1; ++q) {
                        const int t = x - r + q;
                        if (t >= 0 && t < d.h) s = add_(s, __ldg(row + t));
                    }
                    dst[((int64_t)z * d.w + y) * d.h + x] = s;
                }
            }
        } else {
            const int i0 = si * kStrip;
            // base of the line through (x, ., o) / (x, o, .)
            const int64_t base = AX == 1 ? (int64_t)o * d.h * d.w + x : (int64_t)o * d.h + x;
            // taps i0-r .. i0+kStrip-1+r (clamped) in registers
            float v[kStrip + 2 * R];
#pragma unroll
            for (int q = 0; q < kStrip + 2 * R; ++q) {
                const int t = i0 - r + q;
                v[q] = (t >= 0 && t < len) ? src[base + (int64_t)t * stride] : 0.0f;
            }
#pragma unroll
            for (int k = 0; k < kStrip; ++k) {
                const int i = i0 + k;
                if (i >= len) break;
                const int t0 = max(0, i - r), t1 = min(len - 1, i + r);
                float s = 0.0f;
#pragma unroll
                for (int q = 0; q < 2 * R + 1; ++q) {
                    const int t = i - r + q;
                    if (t >= t0 && t <= t1) s = add_(s, v[k + q]);
                }
                dst[base + (int64_t)i * stride] = s;
            }
        }
    }
}

// {f, g, f*f, g*g, f*g} (op_mul, objective.hpp:57-59)
__global__ void __launch_bounds__(kLB)
ncc_products_k(const float *__restrict__ f, const float *__restrict__ g, int n,
               float *__restrict__ out) {
    const int p = blockIdx.x * kLB + threadIdx.x;
    if (p >= n) return;
    const float a = f[p], b = g[p];
    out[p] = a;
    out[n + p] = b;
    out[2 * n + p] = mul_(a, a);
    out[3 * n + p] = mul_(b, b);
    out[4 * n + p] = mul_(a, b);
}

// in-bounds window count; z is bounded by the planes [zv0, zv1) that lie in
// the volume (the whole grid, or a depth slab's extended grid)
__device__ __forceinline__ float win_count(int x, int y, int z, const LDims &d, int r, int zv0,
                                           int zv1) {
    const int cx = min(x + r, d.h - 1) - max(x - r, 0) + 1;
    const int cy = min(y + r, d.w - 1) - max(y - r, 0) + 1;
    const int cz = min(z + r, zv1 - 1) - max(z - r, zv0) + 1;
    return (float)(cx * cy * cz);
}

struct NccTerms {
    float cross, vf, vg, den, cnt, sf, sg;
};
// objective.hpp:62-68, same operation order
__device__ __forceinline__ NccTerms ncc_terms(const float *S, int p, int n, float cnt) {
    NccTerms t;
    t.sf = S[p];
    t.sg = S[n + p];
    const float sff = S[2 * n + p], sgg = S[3 * n + p], sfg = S[4 * n + p];
    t.cnt = cnt;
    t.cross = sub_(sfg, __fdiv_rn(mul_(t.sf, t.sg), cnt));
    t.vf = sub_(sff, __fdiv_rn(mul_(t.sf, t.sf), cnt));
    t.vg = sub_(sgg, __fdiv_rn(mul_(t.sg, t.sg), cnt));
    t.den = add_(mul_(t.vf, t.vg), kNccEps);
    return t;
}

// per-CTA partial sums of cc over the voxels [p0, p1)
__global__ void __launch_bounds__(kLB)
ncc_cc_k(const float *__restrict__ S, LDims d, int r, int zv0, int zv1, int p0, int p1,
         float *__restrict__ part) {
    float acc = 0.0f;
    for (int p = p0 + blockIdx.x * kLB + threadIdx.x; p < p1; p += gridDim.x * kLB) {
        int x, y, z;
        lxyz(p, d, x, y, z);
        const NccTerms t = ncc_terms(S, p, d.n, win_count(x, y, z, d, r, zv0, zv1));
        acc += __fdiv_rn(mul_(t.cross, t.cross), t.den);
    }
    __shared__ float red[kLB];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int m = kLB / 2; m > 0; m >>= 1) {
        if (threadIdx.x < m) red[threadIdx.x] += red[threadIdx.x + m];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// op_grad_reg sums: for component c and axis a, sum of squared forward
// differences over the defined positions
__global__ void __launch_bounds__(kLB)
grad_reg_k(const float *__restrict__ phi, LDims d, float *__restrict__ part) {
    float acc[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) acc[i] = 0.0f;
    const int strides[3] = {1, d.h, d.h * d.w};
    for (int p = blockIdx.x * kLB + threadIdx.x; p < d.n; p += gridDim.x * kLB) {
        int x, y, z;
        lxyz(p, d, x, y, z);
        const bool ok[3] = {x < d.h - 1, y < d.w - 1, z < d.l - 1};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float *u = phi + (int64_t)c * d.n;
            const float u0 = u[p];
#pragma unroll
            for (int a = 0; a < 3; ++a)
                if (ok[a]) {
                    const float df = sub_(u[p + strides[a]], u0);
                    acc[c * 3 + a] = fmaf(df, df, acc[c * 3 + a]);
                }
        }
    }
    __shared__ float red[kLB / 32][9];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        float v = acc[i];
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
        if (lane == 0) red[wid][i] = v;
    }
    __syncthreads();
    if (threadIdx.x < 9) {
        float v = 0.0f;
        for (int w = 0; w < kLB / 32; ++w) v += red[w][threadIdx.x];
        part[(int64_t)blockIdx.x * 9 + threadIdx.x] = v;
    }
}

// final: terms[0] = total, [1] = ncc, [2] = reg (fixed-order sums)
__global__ void __launch_bounds__(kLB)
loss_final_k(const float *__restrict__ cc_part, int ncc_parts, const float *__restrict__ reg_part,
             int reg_parts, LDims d, float lambda, float *__restrict__ terms) {
    __shared__ float s[kLB];
    __shared__ float regs[9];
    float v = 0.0f;
    for (int i = threadIdx.x; i < ncc_parts; i += kLB) v += cc_part[i];
    s[threadIdx.x] = v;
    __syncthreads();
    for (int m = kLB / 2; m > 0; m >>= 1) {
        if (threadIdx.x < m) s[threadIdx.x] += s[threadIdx.x + m];
        __syncthreads();
    }
    const float cc_sum = s[0];
    if (threadIdx.x < 9) {
        float r = 0.0f;
        if (reg_part)
            for (int i = 0; i < reg_parts; ++i) r += reg_part[(int64_t)i * 9 + threadIdx.x];
        regs[threadIdx.x] = r;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // objective.hpp:69: -mean(cc);  ops.hpp:336-355: sum_c sum_a s/defined / 3
        const float ncc = -(cc_sum * (1.0f / (float)d.n));
        const int dims[3] = {d.h, d.w, d.l};
        float tot = 0.0f;
        for (int c = 0; c < 3; ++c)
            for (int a = 0; a < 3; ++a) {
                const int64_t defined = (int64_t)d.n - d.n / dims[a];
                tot += regs[c * 3 + a] / (float)defined;
            }
        const float reg = reg_part ? tot / 3.0f : 0.0f;
        terms[1] = ncc;
        terms[2] = reg;
        terms[0] = lambda == 0.0f ? ncc : ncc + reg * lambda;
    }
}

// per-voxel adjoint of cc into the three statistics that depend on g:
// G = {dL/dsg, dL/dsgg, dL/dsfg}, with dL/dcc = -seed / n; zero outside the
// voxels [p0, p1) whose cc is in the loss
__global__ void __launch_bounds__(kLB)
ncc_adjoint_k(const float *__restrict__ S, LDims d, int r, float gcc, int zv0, int zv1, int p0,
              int p1, float *__restrict__ G, const float *__restrict__ gscale = nullptr) {
    // gscale (device, nullable): dL/dcc = gcc * *gscale (the upstream gradient
    // read on the device: no host round trip inside a captured graph)
    if (gscale) gcc *= *gscale;
    const int p = blockIdx.x * kLB + threadIdx.x;
    if (p >= d.n) return;
    if (p < p0 || p >= p1) {
        G[p] = G[d.n + p] = G[2 * d.n + p] = 0.0f;
        return;
    }
    int x, y, z;
    lxyz(p, d, x, y, z);
    const NccTerms t = ncc_terms(S, p, d.n, win_count(x, y, z, d, r, zv0, zv1));
    const float inv_den = 1.0f / t.den;
    const float a = t.cross;
    // cc = a^2 / den, den = vf*vg + eps
    const float g_cross = gcc * 2.0f * a * inv_den;
    const float g_vg = -gcc * a * a * inv_den * inv_den * t.vf;
    // cross = sfg - sf*sg/cnt;  vg = sgg - sg*sg/cnt
    const float g_sg = -(g_cross * t.sf + 2.0f * g_vg * t.sg) / t.cnt;
    G[p] = g_sg;
    G[d.n + p] = g_vg;
    G[2 * d.n + p] = g_cross;
}

// dL/dwarped = box(G_sg) + 2 g box(G_sgg) + f box(G_sfg)
__global__ void __launch_bounds__(kLB)
ncc_gwarped_k(const float *__restrict__ BG, const float *__restrict__ f,
              const float *__restrict__ g, int n, float *__restrict__ gw) {
    const int p = blockIdx.x * kLB + threadIdx.x;
    if (p >= n) return;
    gw[p] = BG[p] + 2.0f * g[p] * BG[n + p] + f[p] * BG[2 * n + p];
}

// op_grad_reg backward (ops.hpp:360-378): gphi += coeff*diff at p+stride,
// -= at p; as a gather per voxel (no atomics)
__global__ void __launch_bounds__(kLB)
grad_reg_bwd_k(const float *__restrict__ phi, LDims d, float g, float *__restrict__ gphi) {
    const int p = blockIdx.x * kLB + threadIdx.x;
    if (p >= d.n) return;
    int x, y, z;
    lxyz(p, d, x, y, z);
    const int dims[3] = {d.h, d.w, d.l};
    const int pos[3] = {x, y, z};
    const int strides[3] = {1, d.h, d.h * d.w};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float *u = phi + (int64_t)c * d.n;
        float acc = 0.0f;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int64_t defined = (int64_t)d.n - d.n / dims[a];
            const float coeff = 2.0f * g / (3.0f * (float)defined);
            if (pos[a] > 0) acc += coeff * (u[p] - u[p - strides[a]]);          // as p + stride
            if (pos[a] < dims[a] - 1) acc -= coeff * (u[p + strides[a]] - u[p]);  // as p
        }
        gphi[(int64_t)c * d.n + p] += acc;
    }
}

__global__ void __launch_bounds__(kLB)
sum_parts_k(const float *__restrict__ part, int nparts, float *__restrict__ out) {
    __shared__ float s[kLB];
    float v = 0.0f;
    for (int i = threadIdx.x; i < nparts; i += kLB) v += part[i];
    s[threadIdx.x] = v;
    __syncthreads();
    for (int m = kLB / 2; m > 0; m >>= 1) {
        if (threadIdx.x < m) s[threadIdx.x] += s[threadIdx.x + m];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = s[0];
}

// three separable passes a -> b -> a -> b (both buffers owned scratch);
// the box sum ends in b
template <int R>
static void box3_r(float *a, int C, const LDims &d, float *b, cudaStream_t st) {
    const dim3 g((unsigned)std::min<int64_t>(grid1d(d.n / kStrip + d.h * d.w, kLB), 148 * 8),
                 (unsigned)C);
    if (d.h + 2 * R <= kRowMax) {
        const size_t sm = (size_t)(kLB / 32) * (d.h + 2 * R) * sizeof(float);
        if (sm > 48 * 1024)
            cudaFuncSetAttribute(box_x_rows_k<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm);
        const unsigned gx = (unsigned)std::max<int64_t>(
            1, std::min<int64_t>(((int64_t)d.w * d.l + kLB / 32 - 1) / (kLB / 32), 148 * 8));
        box_x_rows_k<R><<<dim3(gx, (unsigned)C), kLB, sm, st>>>(a, d, b);
    } else {
        box_axis_k<0, R><<<g, kLB, 0, st>>>(a, d, b);
    }
    box_axis_k<1, R><<<g, kLB, 0, st>>>(b, d, a);
    box_axis_k<2, R><<<g, kLB, 0, st>>>(a, d, b);
}

static mdg_status box3(float *a, int C, const LDims &d, int r, float *b, cudaStream_t st) {
    switch (r) {
#define MDG_BOX(RV) \
    case RV: box3_r<RV>(a, C, d, b, st); break;
        MDG_BOX(1) MDG_BOX(2) MDG_BOX(3) MDG_BOX(4) MDG_BOX(5) MDG_BOX(6) MDG_BOX(7)
        MDG_BOX(8) MDG_BOX(9) MDG_BOX(10) MDG_BOX(11) MDG_BOX(12)
#undef MDG_BOX
        default: MDG_REQUIRE(false, "ncc_loss: window > 25 is not supported");
    }
    g_launches.fetch_add(3);
    MDG_CUDA_TRY(cudaPeekAtLastError());
    return MDG_OK;
}

static mdg_status check_loss(mdg_dims3 dd, int window, float lambda) {
    MDG_REQUIRE(dims_ok(dd) && nvox(dd) > 0, "ncc_loss: invalid dims " + dims_str(dd));
    MDG_REQUIRE(window >= 3 && window % 2 == 1, "ncc_loss: window must be odd and >= 3");
    MDG_REQUIRE(window / 2 <= kMaxR, "ncc_loss: window > 25 is not supported");
    MDG_REQUIRE(lambda >= 0.0f, "loss: lambda must be >= 0");
    MDG_REQUIRE(lambda == 0.0f || (dd.h >= 2 && dd.w >= 2 && dd.l >= 2),
                "grad_reg requires dims >= 2 per axis");
    return MDG_OK;
}

}  // namespace mdg

using namespace mdg;

extern "C" {

mdg_status mdg_total_loss_fwd(const float *fixed, const float *moving, const float *phi,
                              mdg_dims3 dd, int window, float lambda, float *terms,
                              float *warped, void *stream) {
    if (mdg_status e = check_loss(dd, window, lambda)) return e;
    MDG_REQUIRE(fixed && moving && phi && terms, "total_loss: null pointer");
    cudaStream_t st = S_(stream);
    const LDims d{dd.h, dd.w, dd.l, (int)nvox(dd)};
    const int r = window / 2;
    Scratch sc;
    const int ncc_parts = (int)std::min<int64_t>(grid1d(d.n, kLB), 148 * 8);
    const int reg_parts = ncc_parts;
    MDG_CUDA_TRY(sc.alloc(((size_t)11 * d.n + ncc_parts + 9 * reg_parts + 64) * sizeof(float), st));
    float *w = warped ? warped : sc.as<float>() + (size_t)10 * d.n;
    float *prod = sc.as<float>(), *tmp = prod + (size_t)5 * d.n;
    float *cc_part = prod + (size_t)11 * d.n, *reg_part = cc_part + ncc_parts;
    // warped = warp(moving, phi) (objective.hpp:74)
    if (mdg_status e = mdg_warp_fwd(moving, 1, dd, phi, w, st)) return e;
    ncc_products_k<<<grid1d(d.n, kLB), kLB, 0, st>>>(fixed, w, d.n, prod);
    MDG_LAUNCHED();
    if (mdg_status e = box3(prod, 5, d, r, tmp, st)) return e;  // statistics in tmp
    ncc_cc_k<<<ncc_parts, kLB, 0, st>>>(tmp, d, r, 0, d.l, 0, d.n, cc_part);
    MDG_LAUNCHED();
    if (lambda != 0.0f) {
        grad_reg_k<<<reg_parts, kLB, 0, st>>>(phi, d, reg_part);
        MDG_LAUNCHED();
    }
    loss_final_k<<<1, kLB, 0, st>>>(cc_part, ncc_parts, lambda != 0.0f ? reg_part : nullptr,
                                    reg_parts, d, lambda, terms);
    MDG_LAUNCHED();
    return MDG_OK;
}

mdg_status mdg_total_loss_bwd(const float *fixed, const float *moving, const float *phi,
                              mdg_dims3 dd, int window, float lambda, float seed,
                              float *gphi, float *gmoving, void *stream) {
    if (mdg_status e = check_loss(dd, window, lambda)) return e;
    MDG_REQUIRE(fixed && moving && phi, "total_loss: null pointer");
    if (!gphi && !gmoving) return MDG_OK;
    cudaStream_t st = S_(stream);
    const LDims d{dd.h, dd.w, dd.l, (int)nvox(dd)};
    const int r = window / 2;
    Scratch sc;
    MDG_CUDA_TRY(sc.alloc((size_t)15 * d.n * sizeof(float), st));
    float *P = sc.as<float>(), *S = P + (size_t)5 * d.n, *G = P + (size_t)10 * d.n;
    float *w = P + (size_t)13 * d.n, *gw = P + (size_t)14 * d.n;
    // recompute the forward statistics (cheaper than keeping 5 volumes alive)
    if (mdg_status e = mdg_warp_fwd(moving, 1, dd, phi, w, st)) return e;
    ncc_products_k<<<grid1d(d.n, kLB), kLB, 0, st>>>(fixed, w, d.n, P);
    MDG_LAUNCHED();
    if (mdg_status e = box3(P, 5, d, r, S, st)) return e;
    // dL/dcc = seed * (-1) * (1/n)  (op_scale / op_mean_all backward)
    const float gcc = -seed * (1.0f / (float)d.n);
    ncc_adjoint_k<<<grid1d(d.n, kLB), kLB, 0, st>>>(S, d, r, gcc, 0, d.l, 0, d.n, G);
    MDG_LAUNCHED();
    if (mdg_status e = box3(G, 3, d, r, P, st)) return e;  // self-adjoint; result in P
    ncc_gwarped_k<<<grid1d(d.n, kLB), kLB, 0, st>>>(P, fixed, w, d.n, gw);
    MDG_LAUNCHED();
    if (mdg_status e = mdg_warp_bwd(moving, 1, dd, phi, gw, gmoving, gphi, st)) return e;
    if (gphi && lambda != 0.0f) {
        grad_reg_bwd_k<<<grid1d(d.n, kLB), kLB, 0, st>>>(phi, d, seed * lambda, gphi);
        MDG_LAUNCHED();
    }
    return MDG_OK;
}

// ---- NCC of one depth slab (slab_po.py): the extended grid carries r halo
// planes per side; the slab's own planes are [r, l - r)
static mdg_status check_slab_ncc(mdg_dims3 e, int window, int zv0, int zv1) {
    MDG_REQUIRE(dims_ok(e) && nvox(e) > 0, "ncc_slab: invalid dims " + dims_str(e));
    MDG_REQUIRE(window >= 3 && window % 2 == 1 && window / 2 <= kMaxR,
                "ncc_slab: window must be odd, >= 3 and <= 25");
    MDG_REQUIRE(e.l > 2 * (window / 2), "ncc_slab: no own planes inside the halos");
    MDG_REQUIRE(0 <= zv0 && zv0 <= window / 2 && e.l - window / 2 <= zv1 && zv1 <= e.l,
                "ncc_slab: the in-volume planes must cover the slab's own planes");
    return MDG_OK;
}

mdg_status mdg_ncc_slab_fwd(const float *fixed, const float *warped, mdg_dims3 e, int window,
                            int zv0, int zv1, float *cc_sum, void *stream) {
    if (mdg_status er = check_slab_ncc(e, window, zv0, zv1)) return er;
    MDG_REQUIRE(fixed && warped && cc_sum, "ncc_slab: null pointer");
    cudaStream_t st = S_(stream);
    const LDims d{e.h, e.w, e.l, (int)nvox(e)};
    const int r = window / 2, hw = e.h * e.w;
    const int parts = (int)std::min<int64_t>(grid1d(d.n, kLB), 148 * 8);
    Scratch sc;
    MDG_CUDA_TRY(sc.alloc(((size_t)10 * d.n + parts) * sizeof(float), st));
    float *prod = sc.as<float>(), *tmp = prod + (size_t)5 * d.n, *part = prod + (size_t)10 * d.n;
    ncc_products_k<<<grid1d(d.n, kLB), kLB, 0, st>>>(fixed, warped, d.n, prod);
    MDG_LAUNCHED();
    if (mdg_status er = box3(prod, 5, d, r, tmp, st)) return er;
    ncc_cc_k<<<parts, kLB, 0, st>>>(tmp, d, r, zv0, zv1, r * hw, (e.l - r) * hw, part);
    MDG_LAUNCHED();
    sum_parts_k<<<1, kLB, 0, st>>>(part, parts, cc_sum);
    MDG_LAUNCHED();
    return MDG_OK;
}

static mdg_status ncc_slab_bwd_impl(const float *fixed, const float *warped, mdg_dims3 e,
                                    int window, int zv0, int zv1, float gcc,
                                    const float *gscale, float *gwarped, void *stream) {
    if (mdg_status er = check_slab_ncc(e, window, zv0, zv1)) return er;
    MDG_REQUIRE(fixed && warped && gwarped, "ncc_slab: null pointer");
    cudaStream_t st = S_(stream);
    const LDims d{e.h, e.w, e.l, (int)nvox(e)};
    const int r = window / 2, hw = e.h * e.w;
    Scratch sc;
    MDG_CUDA_TRY(sc.alloc((size_t)13 * d.n * sizeof(float), st));
    float *P = sc.as<float>(), *S = P + (size_t)5 * d.n, *G = P + (size_t)10 * d.n;
    ncc_products_k<<<grid1d(d.n, kLB), kLB, 0, st>>>(fixed, warped, d.n, P);
    MDG_LAUNCHED();
    if (mdg_status er = box3(P, 5, d, r, S, st)) return er;
    ncc_adjoint_k<<<grid1d(d.n, kLB), kLB, 0, st>>>(S, d, r, gcc, zv0, zv1, r * hw,
                                                    (e.l - r) * hw, G, gscale);
    MDG_LAUNCHED();
    if (mdg_status er = box3(G, 3, d, r, P, st)) return er;  // self-adjoint; result in P
    ncc_gwarped_k<<<grid1d(d.n, kLB), kLB, 0, st>>>(P, fixed, warped, d.n, gwarped);
    MDG_LAUNCHED();
    return MDG_OK;
}

mdg_status mdg_ncc_slab_bwd(const float *fixed, const float *warped, mdg_dims3 e, int window,
                            int zv0, int zv1, float gcc, float *gwarped, void *stream) {
    return ncc_slab_bwd_impl(fixed, warped, e, window, zv0, zv1, gcc, nullptr, gwarped, stream);
}

mdg_status mdg_ncc_slab_bwd_dev(const float *fixed, const float *warped, mdg_dims3 e, int window,
                                int zv0, int zv1, float gcc, const float *gscale,
                                float *gwarped, void *stream) {
    MDG_REQUIRE(gscale, "ncc_slab: null gradient scale");
    return ncc_slab_bwd_impl(fixed, warped, e, window, zv0, zv1, gcc, gscale, gwarped, stream);
}

}  // extern "C"
