// modet.cu — the ModeT operator on sm_100a.
//
// Fused tier (mdg_modet_fwd / mdg_modet_bwd), nb = 3:
//   fwd: per (voxel p, head s) the 27 logits B[s,o] + <q_p, k_{p+off(o)}>
//        (out-of-bounds neighbour => logit = bias, attention.hpp:77-81) live in
//        registers; softmax and the offset-weighted sums are fused, so only
//        the sub-flow (3 floats) and the row log-sum-exp (1 float) leave the
//        SM.  W (27 floats) is never written unless asked for.
//   bwd: W is recomputed from (Q, K, B, LSE).  Using <W, gW> = gSF . SF the
//        softmax Jacobian needs no second pass over the row:
//            dl(p,o) = W(p,o) * (gSF_p . off(o) - gSF_p . SF_p)
//        dQ_p  = sum_o dl(p,o) K_{p+off(o)}            (row gather)
//        dK_q  = sum_o dl(q-off(o),o) Q_{q-off(o)}      (column gather — the
//                reference's scatter, attention.hpp:159-162, turned into a
//                gather so there are no atomics and the order is fixed)
//        dB    = sum_p dl(p,o): per-CTA partials + a fixed-order tree reduce.
//
// Reference-shaped tier (mdg_na_fused_*, mdg_subfields_*): the same maths on
// the reference's materialised W {S, n, nb^3}, any odd nb.
#include <cfloat>
#include <cmath>

#include "mdg_common.cuh"

namespace mdg {

constexpr int kBlock = 256;

template <int LAYOUT>
struct QK {
    // element (voxel p, channel c) of a Q/K tensor with SD channels
    static __device__ __forceinline__ int64_t at(int64_t p, int c, int64_t n, int SD) {
        return LAYOUT == MDG_QK_POSMAJOR ? p * SD + c : (int64_t)c * n + p;
    }
    static __device__ __forceinline__ int64_t cstride(int64_t n) {
        return LAYOUT == MDG_QK_POSMAJOR ? 1 : n;
    }
    static __device__ __forceinline__ int64_t pstride(int SD) {
        return LAYOUT == MDG_QK_POSMAJOR ? SD : 1;
    }
};

// in-bounds predicate for offset component v in {-1,0,1}
__device__ __forceinline__ bool okd(int v, bool lo, bool hi) { return v < 0 ? lo : (v > 0 ? hi : true); }

__device__ __forceinline__ void flag_nonfinite(unsigned long long *flag, int s, int64_t n,
                                               int64_t p) {
    atomicMin(flag, (unsigned long long)s * (unsigned long long)n + (unsigned long long)p);
}

// ============================================================ fused forward
template <int HD, int LAYOUT, bool WRITE_W>
__global__ void __launch_bounds__(kBlock)
modet_fwd_k(const float *__restrict__ Q, const float *__restrict__ K,
            const float *__restrict__ B, int h, int w, int l, int S, int hd_rt,
            float *__restrict__ SF, float *__restrict__ LSE, float *__restrict__ W,
            unsigned long long *__restrict__ flag) {
    constexpr int HDM = HD > 0 ? HD : 32;
    const int hd = HD > 0 ? HD : hd_rt;
    const int64_t n = (int64_t)h * w * l;
    const int64_t p = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    const int s = blockIdx.y;
    if (p >= n) return;
    const int SD = S * hd;
    const int p32_ = (int)p, t = p32_ / h;  // n < 2^31: 32-bit div/mod
    const int x = p32_ - t * h;
    const int z = t / w;
    const int y = t - z * w;
    const int64_t hw = (int64_t)h * w;
    const int64_t cs = QK<LAYOUT>::cstride(n);
    const int64_t ps = QK<LAYOUT>::pstride(SD);
    const bool xm = x > 0, xp = x < h - 1, ym = y > 0, yp = y < w - 1, zm = z > 0,
               zp = z < l - 1;

    float q[HDM];
    const float *qb = Q + QK<LAYOUT>::at(p, s * hd, n, SD);
#pragma unroll
    for (int j = 0; j < HDM; ++j)
        if (j < hd) q[j] = __ldg(qb + j * cs);
    const float *kb = K + QK<LAYOUT>::at(p, s * hd, n, SD);
    const float *bias = B + s * 27;

    float lg[27];
#pragma unroll
    for (int o = 0; o < 27; ++o) {
        const int dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
        float v = __ldg(bias + o);
        if (okd(dx, xm, xp) && okd(dy, ym, yp) && okd(dz, zm, zp)) {
            const float *kp = kb + (dx + dy * (int64_t)h + dz * hw) * ps;
            float dot = 0.0f;
#pragma unroll
            for (int j = 0; j < HDM; ++j)
                if (j < hd) dot = fmaf(q[j], __ldg(kp + j * cs), dot);
            v += dot;
        }
        lg[o] = v;
    }
    float mx = lg[0], mn = lg[0];
#pragma unroll
    for (int o = 1; o < 27; ++o) {
        mx = fmaxf(mx, lg[o]);
        mn = fminf(mn, lg[o]);
    }
    float sum = 0.0f, ax = 0.0f, ay = 0.0f, az = 0.0f;
#pragma unroll
    for (int o = 0; o < 27; ++o) {
        const int dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
        const float e = __expf(lg[o] - mx);
        lg[o] = e;
        sum += e;
        if (dx) ax += dx > 0 ? e : -e;
        if (dy) ay += dy > 0 ? e : -e;
        if (dz) az += dz > 0 ? e : -e;
    }
    const float inv = 1.0f / sum;
    if (!isfinite(sum) || mn == -INFINITY) flag_nonfinite(flag, s, n, p);
    SF[(3 * (int64_t)s + 0) * n + p] = ax * inv;
    SF[(3 * (int64_t)s + 1) * n + p] = ay * inv;
    SF[(3 * (int64_t)s + 2) * n + p] = az * inv;
    LSE[(int64_t)s * n + p] = mx + logf(sum);
    if (WRITE_W) {
        float *wr = W + ((int64_t)s * n + p) * 27;
#pragma unroll
        for (int o = 0; o < 27; ++o) wr[o] = lg[o] * inv;
    }
}

// =========================================================== fused backward
template <int HD, int LAYOUT>
__global__ void __launch_bounds__(kBlock)
modet_bwd_k(const float *__restrict__ Q, const float *__restrict__ K,
            const float *__restrict__ B, const float *__restrict__ SF,
            const float *__restrict__ LSE, const float *__restrict__ gSF, int h, int w, int l,
            int S, int hd_rt, float *__restrict__ gQ, float *__restrict__ gK,
            float *__restrict__ gBpart) {
    constexpr int HDM = HD > 0 ? HD : 32;
    const int hd = HD > 0 ? HD : hd_rt;
    const int64_t n = (int64_t)h * w * l;
    const int64_t p = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    const int s = blockIdx.y;
    const bool active = p < n;
    const int SD = S * hd;
    const int64_t hw = (int64_t)h * w;
    const int64_t cs = QK<LAYOUT>::cstride(n);
    const int64_t ps = QK<LAYOUT>::pstride(SD);
    const float *bias = B + s * 27;

    float db[27];
#pragma unroll
    for (int o = 0; o < 27; ++o) db[o] = 0.0f;

    if (active) {
        const int p32_ = (int)p, t = p32_ / h;  // n < 2^31: 32-bit div/mod
        const int x = p32_ - t * h;
        const int z = t / w;
        const int y = t - z * w;
        const bool xm = x > 0, xp = x < h - 1, ym = y > 0, yp = y < w - 1, zm = z > 0,
                   zp = z < l - 1;
        const int64_t qoff = QK<LAYOUT>::at(p, s * hd, n, SD);
        float q[HDM], k[HDM], dq[HDM], dk[HDM];
#pragma unroll
        for (int j = 0; j < HDM; ++j)
            if (j < hd) {
                q[j] = __ldg(Q + qoff + j * cs);
                k[j] = __ldg(K + qoff + j * cs);
                dq[j] = 0.0f;
                dk[j] = 0.0f;
            }
        const int64_t so = (int64_t)s * n;
        const float lse = __ldg(LSE + so + p);
        const float gx = __ldg(gSF + 3 * so + p), gy = __ldg(gSF + 3 * so + n + p),
                    gz = __ldg(gSF + 3 * so + 2 * n + p);
        const float dot = gx * __ldg(SF + 3 * so + p) + gy * __ldg(SF + 3 * so + n + p) +
                          gz * __ldg(SF + 3 * so + 2 * n + p);

#pragma unroll
        for (int o = 0; o < 27; ++o) {
            const int dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
            const float bo = __ldg(bias + o);
            const int64_t dp = dx + dy * (int64_t)h + dz * hw;
            // row part: p attends to p + off(o)
            {
                const bool in = okd(dx, xm, xp) && okd(dy, ym, yp) && okd(dz, zm, zp);
                float kv[HDM];
                float lg = bo;
                if (in) {
                    const float *kp = K + qoff + dp * ps;
                    float d0 = 0.0f;
#pragma unroll
                    for (int j = 0; j < HDM; ++j)
                        if (j < hd) {
                            kv[j] = __ldg(kp + j * cs);
                            d0 = fmaf(q[j], kv[j], d0);
                        }
                    lg += d0;
                }
                float gw = 0.0f;
                if (dx) gw += dx > 0 ? gx : -gx;
                if (dy) gw += dy > 0 ? gy : -gy;
                if (dz) gw += dz > 0 ? gz : -gz;
                const float dl = __expf(lg - lse) * (gw - dot);
                db[o] = dl;
                if (in) {
#pragma unroll
                    for (int j = 0; j < HDM; ++j)
                        if (j < hd) dq[j] = fmaf(dl, kv[j], dq[j]);
                }
            }
            // column part: p is the key of source r = p - off(o)
            {
                const bool in = okd(-dx, xm, xp) && okd(-dy, ym, yp) && okd(-dz, zm, zp);
                if (in) {
                    const int64_t r = p - dp;
                    const float *qr = Q + qoff - dp * ps;
                    float qv[HDM];
                    float d0 = 0.0f;
#pragma unroll
                    for (int j = 0; j < HDM; ++j)
                        if (j < hd) {
                            qv[j] = __ldg(qr + j * cs);
                            d0 = fmaf(qv[j], k[j], d0);
                        }
                    const float lr = __ldg(LSE + so + r);
                    const float rx = __ldg(gSF + 3 * so + r), ry = __ldg(gSF + 3 * so + n + r),
                                rz = __ldg(gSF + 3 * so + 2 * n + r);
                    const float dotr = rx * __ldg(SF + 3 * so + r) +
                                       ry * __ldg(SF + 3 * so + n + r) +
                                       rz * __ldg(SF + 3 * so + 2 * n + r);
                    float gw = 0.0f;
                    if (dx) gw += dx > 0 ? rx : -rx;
                    if (dy) gw += dy > 0 ? ry : -ry;
                    if (dz) gw += dz > 0 ? rz : -rz;
                    const float dl = __expf(bo + d0 - lr) * (gw - dotr);
#pragma unroll
                    for (int j = 0; j < HDM; ++j)
                        if (j < hd) dk[j] = fmaf(dl, qv[j], dk[j]);
                }
            }
        }
        if (gQ) {
#pragma unroll
            for (int j = 0; j < HDM; ++j)
                if (j < hd) gQ[qoff + j * cs] += dq[j];
        }
        if (gK) {
#pragma unroll
            for (int j = 0; j < HDM; ++j)
                if (j < hd) gK[qoff + j * cs] += dk[j];
        }
    }

    // dB: warp shuffle reduce, then across the CTA's warps, one partial per CTA
    __shared__ float red[kBlock / 32][27];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 0; o < 27; ++o) {
        float v = db[o];
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
        if (lane == 0) red[wid][o] = v;
    }
    __syncthreads();
    if (threadIdx.x < 27) {
        float v = 0.0f;
#pragma unroll
        for (int i = 0; i < kBlock / 32; ++i) v += red[i][threadIdx.x];
        gBpart[((int64_t)s * gridDim.x + blockIdx.x) * 27 + threadIdx.x] = v;
    }
}

// gB[s, o] += sum over CTAs of part[s, cta, o], fixed-order tree (deterministic)
__global__ void __launch_bounds__(kBlock)
reduce_parts_k(const float *__restrict__ part, int nparts, int width, float *__restrict__ out) {
    const int s = blockIdx.y, o = blockIdx.x;
    float v = 0.0f;
    for (int i = threadIdx.x; i < nparts; i += kBlock)
        v += part[((int64_t)s * nparts + i) * width + o];
    __shared__ float sm[kBlock];
    sm[threadIdx.x] = v;
    __syncthreads();
    for (int m = kBlock / 2; m > 0; m >>= 1) {
        if (threadIdx.x < m) sm[threadIdx.x] += sm[threadIdx.x + m];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[s * width + o] += sm[0];
}

// ============================================= reference-shaped tier (any nb)
// attention.hpp:83-123, W row used as the logit scratch
__global__ void __launch_bounds__(kBlock)
na_fwd_ref_k(const float *__restrict__ Q, const float *__restrict__ K,
             const float *__restrict__ B, int h, int w, int l, int S, int hd, int nb,
             float *__restrict__ W, unsigned long long *__restrict__ flag) {
    const int64_t n = (int64_t)h * w * l;
    const int64_t p = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    const int s = blockIdx.y;
    if (p >= n) return;
    const int win = nb * nb * nb, r = (nb - 1) / 2, SD = S * hd;
    const int p32_ = (int)p, t = p32_ / h;  // n < 2^31: 32-bit div/mod
    const int x = p32_ - t * h;
    const int z = t / w;
    const int y = t - z * w;
    const float *q = Q + p * SD + s * hd;
    float *wr = W + ((int64_t)s * n + p) * win;
    float mx = -INFINITY, mn = INFINITY;
    bool nan = false;
    int o = 0;
    for (int dz = -r; dz <= r; ++dz)
        for (int dy = -r; dy <= r; ++dy)
            for (int dx = -r; dx <= r; ++dx, ++o) {
                float v = B[s * win + o];
                const int xx = x + dx, yy = y + dy, zz = z + dz;
                if (xx >= 0 && xx < h && yy >= 0 && yy < w && zz >= 0 && zz < l) {
                    const float *k = K + (((int64_t)zz * w + yy) * h + xx) * SD + s * hd;
                    float dot = 0.0f;
                    for (int j = 0; j < hd; ++j) dot = fmaf(q[j], k[j], dot);
                    v += dot;
                }
                nan |= isnan(v);
                mx = fmaxf(mx, v);
                mn = fminf(mn, v);
                wr[o] = v;
            }
    if (nan || isinf(mx) || isinf(mn)) {
        flag_nonfinite(flag, s, n, p);
        return;
    }
    float sum = 0.0f;
    for (o = 0; o < win; ++o) {
        const float e = __expf(wr[o] - mx);
        wr[o] = e;
        sum += e;
    }
    const float inv = 1.0f / sum;
    for (o = 0; o < win; ++o) wr[o] *= inv;
}

// attention.hpp:127-166 split in two gathers: (1) dl rows, gQ; (2) gK.
__global__ void __launch_bounds__(kBlock)
na_bwd_ref_rows_k(const float *__restrict__ K, const float *__restrict__ W,
                  const float *__restrict__ gW, int h, int w, int l, int S, int hd, int nb,
                  float *__restrict__ dl, float *__restrict__ gQ) {
    const int64_t n = (int64_t)h * w * l;
    const int64_t p = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    const int s = blockIdx.y;
    if (p >= n) return;
    const int win = nb * nb * nb, r = (nb - 1) / 2, SD = S * hd;
    const int p32_ = (int)p, t = p32_ / h;  // n < 2^31: 32-bit div/mod
    const int x = p32_ - t * h;
    const int z = t / w;
    const int y = t - z * w;
    const int64_t row = ((int64_t)s * n + p) * win;
    float dot = 0.0f;
    for (int i = 0; i < win; ++i) dot = fmaf(W[row + i], gW[row + i], dot);
    float *gq = gQ ? gQ + p * SD + s * hd : nullptr;
    int o = 0;
    for (int dz = -r; dz <= r; ++dz)
        for (int dy = -r; dy <= r; ++dy)
            for (int dx = -r; dx <= r; ++dx, ++o) {
                const float d = W[row + o] * (gW[row + o] - dot);
                dl[row + o] = d;
                const int xx = x + dx, yy = y + dy, zz = z + dz;
                if (!gq || d == 0.0f) continue;
                if (xx < 0 || xx >= h || yy < 0 || yy >= w || zz < 0 || zz >= l) continue;
                const float *k = K + (((int64_t)zz * w + yy) * h + xx) * SD + s * hd;
                for (int j = 0; j < hd; ++j) gq[j] = fmaf(d, k[j], gq[j]);
            }
}

__global__ void __launch_bounds__(kBlock)
na_bwd_ref_cols_k(const float *__restrict__ Q, const float *__restrict__ dl, int h, int w,
                  int l, int S, int hd, int nb, float *__restrict__ gK) {
    const int64_t n = (int64_t)h * w * l;
    const int64_t p = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    const int s = blockIdx.y;
    if (p >= n) return;
    const int win = nb * nb * nb, r = (nb - 1) / 2, SD = S * hd;
    const int p32_ = (int)p, t = p32_ / h;  // n < 2^31: 32-bit div/mod
    const int x = p32_ - t * h;
    const int z = t / w;
    const int y = t - z * w;
    float *gk = gK + p * SD + s * hd;
    // the reference visits sources in ascending p, i.e. descending slot o
    int o = win - 1;
    for (int dz = r; dz >= -r; --dz)
        for (int dy = r; dy >= -r; --dy)
            for (int dx = r; dx >= -r; --dx, --o) {
                const int xx = x - dx, yy = y - dy, zz = z - dz;
                if (xx < 0 || xx >= h || yy < 0 || yy >= w || zz < 0 || zz >= l) continue;
                const int64_t src = ((int64_t)zz * w + yy) * h + xx;
                const float d = dl[((int64_t)s * n + src) * win + o];
                if (d == 0.0f) continue;
                const float *q = Q + src * SD + s * hd;
                for (int j = 0; j < hd; ++j) gk[j] = fmaf(d, q[j], gk[j]);
            }
}

// gB[s,o] += sum_p dl[s,p,o]: per-CTA partial sums over a voxel chunk
__global__ void __launch_bounds__(kBlock)
rowsum_parts_k(const float *__restrict__ dl, int64_t n, int win, int chunk,
               float *__restrict__ part) {
    const int s = blockIdx.y, c = blockIdx.x;
    const int64_t p0 = (int64_t)c * chunk;
    const int64_t p1 = min(n, p0 + chunk);
    for (int o = threadIdx.x; o < win; o += kBlock) {
        float v = 0.0f;
        for (int64_t p = p0; p < p1; ++p) v += dl[((int64_t)s * n + p) * win + o];
        part[((int64_t)s * gridDim.x + c) * win + o] = v;
    }
}

// attention.hpp:282-298.  Products with offsets in {-1,0,1} are exact, so the
// FMA form equals the reference's multiply-then-add bit for bit.
__global__ void __launch_bounds__(kBlock)
subfields_fwd_k(const float *__restrict__ W, int64_t n, int S, int nb, float *__restrict__ out) {
    const int64_t p = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    const int s = blockIdx.y;
    if (p >= n) return;
    const int win = nb * nb * nb, r = (nb - 1) / 2;
    const float *wr = W + ((int64_t)s * n + p) * win;
    float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f;
    for (int o = 0; o < win; ++o) {
        const float v = wr[o];
        a0 = fmaf(v, (float)(o % nb - r), a0);
        a1 = fmaf(v, (float)((o / nb) % nb - r), a1);
        a2 = fmaf(v, (float)(o / (nb * nb) - r), a2);
    }
    out[(3 * (int64_t)s + 0) * n + p] = a0;
    out[(3 * (int64_t)s + 1) * n + p] = a1;
    out[(3 * (int64_t)s + 2) * n + p] = a2;
}

// attention.hpp:301-316
__global__ void __launch_bounds__(kBlock)
subfields_bwd_k(int64_t n, int S, int nb, const float *__restrict__ gout, float *__restrict__ gW) {
    const int64_t p = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    const int s = blockIdx.y;
    if (p >= n) return;
    const int win = nb * nb * nb, r = (nb - 1) / 2;
    const float gx = gout[(3 * (int64_t)s + 0) * n + p];
    const float gy = gout[(3 * (int64_t)s + 1) * n + p];
    const float gz = gout[(3 * (int64_t)s + 2) * n + p];
    float *gr = gW + ((int64_t)s * n + p) * win;
    for (int o = 0; o < win; ++o) {
        const float v = __fadd_rn(__fadd_rn(__fmul_rn(gx, (float)(o % nb - r)),
                                            __fmul_rn(gy, (float)((o / nb) % nb - r))),
                                  __fmul_rn(gz, (float)(o / (nb * nb) - r)));
        gr[o] = __fadd_rn(gr[o], v);
    }
}

// attention.hpp:421-427 row-normalisation check
__global__ void __launch_bounds__(kBlock)
rows_check_k(const float *__restrict__ W, int64_t rows, int win, float tol, int *bad) {
    const int64_t r = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (r >= rows) return;
    float s = 0.0f;
    for (int o = 0; o < win; ++o) s = __fadd_rn(s, W[r * win + o]);
    if (fabs((double)s - 1.0) > (double)tol) atomicExch(bad, 1);
}

__global__ void transpose_k(const float *__restrict__ src, int64_t rows, int64_t cols,
                            int64_t tiles_c, float *__restrict__ dst) {
    // dst[c, r] = src[r, c] through a 32x33 smem tile; blockIdx.x enumerates
    // (row tile, col tile) pairs so neither extent hits the gridDim.y limit
    __shared__ float tile[32][33];
    const int64_t r0 = (int64_t)(blockIdx.x / tiles_c) * 32;
    const int64_t c0 = (int64_t)(blockIdx.x % tiles_c) * 32;
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = src[r * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) dst[c * rows + r] = tile[threadIdx.x][i];
    }
}

static mdg_status transpose(const float *src, int64_t rows, int64_t cols, float *dst,
                            cudaStream_t st) {
    const int64_t tr = (rows + 31) / 32, tc = (cols + 31) / 32;
    transpose_k<<<(unsigned)(tr * tc), dim3(32, 8), 0, st>>>(src, rows, cols, tc, dst);
    MDG_LAUNCHED();
    return MDG_OK;
}

// ----------------------------------------------------------- dispatchers
template <int LAYOUT, bool WW>
static void launch_fwd(int hd, dim3 g, cudaStream_t st, const float *Q, const float *K,
                       const float *B, mdg_dims3 d, int S, float *SF, float *LSE, float *W,
                       unsigned long long *flag) {
#define MDG_FWD(HDV) \
    modet_fwd_k<HDV, LAYOUT, WW><<<g, kBlock, 0, st>>>(Q, K, B, d.h, d.w, d.l, S, hd, SF, LSE, W, flag)
    switch (hd) {
        case 2: MDG_FWD(2); break;
        case 3: MDG_FWD(3); break;
        case 4: MDG_FWD(4); break;
        case 5: MDG_FWD(5); break;
        case 6: MDG_FWD(6); break;
        case 8: MDG_FWD(8); break;
        case 12: MDG_FWD(12); break;
        case 16: MDG_FWD(16); break;
        default: MDG_FWD(0); break;
    }
#undef MDG_FWD
}

template <int LAYOUT>
static void launch_bwd(int hd, dim3 g, cudaStream_t st, const float *Q, const float *K,
                       const float *B, const float *SF, const float *LSE, const float *gSF,
                       mdg_dims3 d, int S, float *gQ, float *gK, float *part) {
#define MDG_BWD(HDV)                                                                          \
    modet_bwd_k<HDV, LAYOUT><<<g, kBlock, 0, st>>>(Q, K, B, SF, LSE, gSF, d.h, d.w, d.l, S, hd, \
                                                   gQ, gK, part)
    switch (hd) {
        case 2: MDG_BWD(2); break;
        case 3: MDG_BWD(3); break;
        case 4: MDG_BWD(4); break;
        case 5: MDG_BWD(5); break;
        case 6: MDG_BWD(6); break;
        case 8: MDG_BWD(8); break;
        case 12: MDG_BWD(12); break;
        case 16: MDG_BWD(16); break;
        default: MDG_BWD(0); break;
    }
#undef MDG_BWD
}

static mdg_status check_attn(mdg_dims3 d, int S, int hd, int nb) {
    // attention.hpp:48-53
    MDG_REQUIRE(nb >= 3 && nb % 2 == 1, "attention: neighborhood must be odd and >= 3");
    MDG_REQUIRE(nb <= 7, "attention: neighborhood > 7 is not supported");
    MDG_REQUIRE(S >= 1 && hd >= 1, "attention: heads and head_dim must be positive");
    MDG_REQUIRE(dims_ok(d), "attention: invalid dims " + dims_str(d));
    return MDG_OK;
}

// modet_tiled.cu (planar layout, nb = 3); false => head_dim not instantiated
bool tiled_fwd(int hd, const float *Q, const float *K, const float *B, mdg_dims3 d, int S,
               float *SF, float *LSE, unsigned long long *flag, cudaStream_t st, cudaError_t *err);
bool tiled_bwd(int hd, const float *Q, const float *K, const float *B, const float *SF,
               const float *LSE, const float *gSF, mdg_dims3 d, int S, bool acc, float *gQ,
               float *gK, float *gB, cudaStream_t st, cudaError_t *err);

}  // namespace mdg

using namespace mdg;

extern "C" {

mdg_status mdg_modet_fwd(const float *Q, const float *K, const float *B, mdg_dims3 d, int S,
                         int hd, int nb, int layout, float *SF, float *LSE, float *W,
                         void *stream) {
    if (mdg_status e = check_attn(d, S, hd, nb)) return e;
    MDG_REQUIRE(nb == 3, "modet (fused tier): neighborhood must be 3; use mdg_na_fused_fwd");
    MDG_REQUIRE(hd <= 32, "modet (fused tier): head_dim must be <= 32");
    MDG_REQUIRE(layout == MDG_QK_POSMAJOR || layout == MDG_QK_PLANAR, "modet: bad Q/K layout");
    const int64_t n = nvox(d);
    if (n == 0) return MDG_OK;
    MDG_REQUIRE(Q && K && B && SF && LSE, "modet: null pointer");
    cudaStream_t st = S_(stream);
    unsigned long long *flag = numeric_flag_ptr(st);
    if (!flag) return status_from_cuda(cudaErrorMemoryAllocation, "numeric flag");
    const dim3 g(grid1d(n, kBlock), S);
    if (layout == MDG_QK_PLANAR && !W) {
        cudaError_t e = cudaSuccess;
        if (tiled_fwd(hd, Q, K, B, d, S, SF, LSE, flag, st, &e)) {
            if (e != cudaSuccess) return status_from_cuda(e, "modet_fwd_tiled");
            MDG_LAUNCHED();
            return MDG_OK;
        }
    }
    if (layout == MDG_QK_POSMAJOR) {
        if (W) launch_fwd<MDG_QK_POSMAJOR, true>(hd, g, st, Q, K, B, d, S, SF, LSE, W, flag);
        else launch_fwd<MDG_QK_POSMAJOR, false>(hd, g, st, Q, K, B, d, S, SF, LSE, W, flag);
    } else {
        if (W) launch_fwd<MDG_QK_PLANAR, true>(hd, g, st, Q, K, B, d, S, SF, LSE, W, flag);
        else launch_fwd<MDG_QK_PLANAR, false>(hd, g, st, Q, K, B, d, S, SF, LSE, W, flag);
    }
    MDG_LAUNCHED();
    return MDG_OK;
}

mdg_status mdg_modet_bwd(const float *Q, const float *K, const float *B, const float *SF,
                         const float *LSE, const float *gSF, mdg_dims3 d, int S, int hd, int nb,
                         int layout, float *gQ, float *gK, float *gB, int accumulate,
                         void *stream) {
    if (mdg_status e = check_attn(d, S, hd, nb)) return e;
    MDG_REQUIRE(nb == 3, "modet (fused tier): neighborhood must be 3; use mdg_na_fused_bwd");
    MDG_REQUIRE(hd <= 32, "modet (fused tier): head_dim must be <= 32");
    MDG_REQUIRE(layout == MDG_QK_POSMAJOR || layout == MDG_QK_PLANAR, "modet: bad Q/K layout");
    const int64_t n = nvox(d);
    if (n == 0) return MDG_OK;
    MDG_REQUIRE(Q && K && B && SF && LSE && gSF, "modet: null pointer");
    cudaStream_t st = S_(stream);
    if (layout == MDG_QK_PLANAR) {
        cudaError_t e = cudaSuccess;
        if (tiled_bwd(hd, Q, K, B, SF, LSE, gSF, d, S, accumulate != 0, gQ, gK, gB, st, &e)) {
            if (e != cudaSuccess) return status_from_cuda(e, "modet_bwd_tiled");
            return MDG_OK;
        }
    }
    if (!accumulate) {  // v1 kernels accumulate: start from zero
        if (gQ) MDG_CUDA_TRY(cudaMemsetAsync(gQ, 0, (size_t)n * S * hd * sizeof(float), st));
        if (gK) MDG_CUDA_TRY(cudaMemsetAsync(gK, 0, (size_t)n * S * hd * sizeof(float), st));
    }
    const dim3 g(grid1d(n, kBlock), S);
    Scratch part;
    MDG_CUDA_TRY(part.alloc((size_t)S * g.x * 27 * sizeof(float), st));
    if (layout == MDG_QK_POSMAJOR)
        launch_bwd<MDG_QK_POSMAJOR>(hd, g, st, Q, K, B, SF, LSE, gSF, d, S, gQ, gK, part.as<float>());
    else
        launch_bwd<MDG_QK_PLANAR>(hd, g, st, Q, K, B, SF, LSE, gSF, d, S, gQ, gK, part.as<float>());
    MDG_LAUNCHED();
    if (gB) {
        reduce_parts_k<<<dim3(27, S), kBlock, 0, st>>>(part.as<float>(), (int)g.x, 27, gB);
        MDG_LAUNCHED();
    }
    return MDG_OK;
}

mdg_status mdg_na_fused_fwd(const float *Q, const float *K, const float *B, mdg_dims3 d,
                            int S, int hd, int nb, float *W, void *stream) {
    if (mdg_status e = check_attn(d, S, hd, nb)) return e;
    const int64_t n = nvox(d);
    if (n == 0) return MDG_OK;
    MDG_REQUIRE(Q && K && B && W, "na_fused_fwd: null pointer");
    cudaStream_t st = S_(stream);
    unsigned long long *flag = numeric_flag_ptr(st);
    if (!flag) return status_from_cuda(cudaErrorMemoryAllocation, "numeric flag");
    na_fwd_ref_k<<<dim3(grid1d(n, kBlock), S), kBlock, 0, st>>>(Q, K, B, d.h, d.w, d.l, S, hd,
                                                                nb, W, flag);
    MDG_LAUNCHED();
    // the reference throws at the first bad logit (attention.hpp:110-114)
    return consume_numeric_flag(st, d);
}

mdg_status mdg_na_fused_bwd(const float *Q, const float *K, const float *W, mdg_dims3 d,
                            int S, int hd, int nb, const float *gW, float *gQ, float *gK,
                            float *gB, void *stream) {
    if (mdg_status e = check_attn(d, S, hd, nb)) return e;
    const int64_t n = nvox(d);
    if (n == 0) return MDG_OK;
    MDG_REQUIRE(Q && K && W && gW, "na_fused_bwd: null pointer");
    cudaStream_t st = S_(stream);
    const int win = nb * nb * nb;
    Scratch dl;
    MDG_CUDA_TRY(dl.alloc((size_t)S * n * win * sizeof(float), st));
    const dim3 g(grid1d(n, kBlock), S);
    na_bwd_ref_rows_k<<<g, kBlock, 0, st>>>(K, W, gW, d.h, d.w, d.l, S, hd, nb, dl.as<float>(), gQ);
    MDG_LAUNCHED();
    if (gK) {
        na_bwd_ref_cols_k<<<g, kBlock, 0, st>>>(Q, dl.as<float>(), d.h, d.w, d.l, S, hd, nb, gK);
        MDG_LAUNCHED();
    }
    if (gB) {
        const int chunk = 1024;
        const int nparts = (int)((n + chunk - 1) / chunk);
        Scratch part;
        MDG_CUDA_TRY(part.alloc((size_t)S * nparts * win * sizeof(float), st));
        rowsum_parts_k<<<dim3(nparts, S), kBlock, 0, st>>>(dl.as<float>(), n, win, chunk, part.as<float>());
        MDG_LAUNCHED();
        reduce_parts_k<<<dim3(win, S), kBlock, 0, st>>>(part.as<float>(), nparts, win, gB);
        MDG_LAUNCHED();
    }
    return MDG_OK;
}

mdg_status mdg_subfields_fwd(const float *W, mdg_dims3 d, int S, int nb, float *out,
                             void *stream) {
    if (mdg_status e = check_attn(d, S, 1, nb)) return e;
    const int64_t n = nvox(d);
    if (n == 0) return MDG_OK;
    subfields_fwd_k<<<dim3(grid1d(n, kBlock), S), kBlock, 0, S_(stream)>>>(W, n, S, nb, out);
    MDG_LAUNCHED();
    return MDG_OK;
}

mdg_status mdg_subfields_bwd(mdg_dims3 d, int S, int nb, const float *gout, float *gW,
                             void *stream) {
    if (mdg_status e = check_attn(d, S, 1, nb)) return e;
    const int64_t n = nvox(d);
    if (n == 0) return MDG_OK;
    subfields_bwd_k<<<dim3(grid1d(n, kBlock), S), kBlock, 0, S_(stream)>>>(n, S, nb, gout, gW);
    MDG_LAUNCHED();
    return MDG_OK;
}

mdg_status mdg_subfields_check_rows(const float *W, mdg_dims3 d, int S, int nb, float tol,
                                    void *stream) {
    if (mdg_status e = check_attn(d, S, 1, nb)) return e;
    const int64_t rows = (int64_t)S * nvox(d);
    if (rows == 0) return MDG_OK;
    cudaStream_t st = S_(stream);
    Scratch bad;
    MDG_CUDA_TRY(bad.alloc(sizeof(int), st));
    MDG_CUDA_TRY(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    rows_check_k<<<grid1d(rows, kBlock), kBlock, 0, st>>>(W, rows, nb * nb * nb, tol, bad.as<int>());
    MDG_LAUNCHED();
    int hbad = 0;
    MDG_CUDA_TRY(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    MDG_CUDA_TRY(cudaStreamSynchronize(st));
    MDG_REQUIRE(!hbad, "subfields: attention weights are not normalized");
    return MDG_OK;
}

mdg_status mdg_qk_posmajor_to_planar(const float *src, int64_t n, int C, float *dst,
                                     void *stream) {
    MDG_REQUIRE(n >= 0 && C >= 1, "qk layout: bad sizes");
    if (n == 0) return MDG_OK;
    return transpose(src, n, C, dst, S_(stream));
}

mdg_status mdg_qk_planar_to_posmajor(const float *src, int64_t n, int C, float *dst,
                                     void *stream) {
    MDG_REQUIRE(n >= 0 && C >= 1, "qk layout: bad sizes");
    if (n == 0) return MDG_OK;
    return transpose(src, C, n, dst, S_(stream));
}

}  // extern "C"
