// modet_tiled.cu — tiled ModeT kernels for the native planar layout.
//
// Layout: Q, K planar {S*d, n}; head s owns channel planes s*d .. s*d+d-1.
//
// Every kernel is a z-marching CTA: it owns an x-y column tile and walks a
// chunk of z.  Each step stages ONE zero-padded z-plane (tile + 1-voxel x/y
// halo) into shared memory with cp.async (zero-fill outside the volume, which
// is exactly the reference's "out-of-bounds key contributes nothing, logit =
// bias" rule, attention.hpp:77-81), double-buffered so the next plane lands
// while the current one is consumed.  A staged plane is used by the three
// voxels of a thread's column that have it in their 3x3x3 window
// (z = p-1, p, p+1: "in-flight" slots), so every staged element is read from
// shared memory once per slot instead of once per logit.
//
//   fwd  (modet_fwd_tiled_k): per voxel the 27 logits in log2 units
//        (q pre-scaled by log2 e), an online softmax processed one 3-logit
//        x-row at a time with lazy rescaling (rescale only when the running
//        max grows by > 8 in log2 units, so exponents stay <= 2^8), and the
//        offset-weighted sums; writes SF {3S,n} and LSE {S,n} (natural log).
//   bwd  row kernel (modet_bwd_row_k): p as query.  W = exp2(l - LSE*log2e)
//        recomputed, dl = W*(gSF.off(o) - gSF.SF), dQ_p += dl*K_{p+o},
//        dB_o partial per CTA.
//   bwd  column kernel (modet_bwd_col_k): q as key, gathering from the
//        staged sources r = q - off(o): dK_q += dl(r,o)*Q_r.  No atomics;
//        fixed summation order => deterministic.
#include "mdg_common.cuh"

namespace mdg {
namespace tiled {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescale = 8.0f;  // lazy-rescale threshold (log2 units)

__device__ __forceinline__ void cp_async4(float *dst, const float *src, bool pred) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src),
                 "r"(pred ? 4 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct Vol {
    int h, w, l;
    int64_t n, hw;
};

// Stage plane z of NCH channel planes (channel c at base(c)) for the tile
// with interior origin (x0, y0) into dst[c][PY][PX] (row length RL = tile+2).
// Warp-per-row, lane-per-x: coalesced 4-byte cp.async, zero-fill outside.
template <int NCH, int PY, int RL, int PX, class Base>
__device__ __forceinline__ void stage_plane(float *dst, Base base, int z, int x0, int y0,
                                            const Vol &v) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const bool zok = z >= 0 && z < v.l;
    for (int r = wid; r < NCH * PY; r += nw) {
        const int c = r / PY, ry = r - c * PY;
        const int gy = y0 - 1 + ry;
        const bool rok = zok && gy >= 0 && gy < v.w;
        const float *row = base(c);
        const int64_t roff = (int64_t)z * v.hw + (int64_t)gy * v.h;
        float *drow = dst + r * PX;
#pragma unroll
        for (int rx = lane; rx < RL; rx += 32) {
            const int gx = x0 - 1 + rx;
            const bool ok = rok && gx >= 0 && gx < v.h;
            cp_async4(drow + rx, ok ? row + roff + gx : row, ok);
        }
    }
}

// online-softmax state of one (voxel, head) row
struct Soft {
    float m, s, ax, ay, az, mn;
};

__device__ __forceinline__ void soft_init(Soft &st) {
    st.m = -INFINITY;
    st.s = st.ax = st.ay = st.az = 0.0f;
    st.mn = INFINITY;
}

// fold one x-row of three logits (dx = -1, 0, +1) at window row (dy, dz)
template <int DY, int DZ>
__device__ __forceinline__ void soft_row(Soft &st, float lm, float l0, float lp) {
    const float mr = fmaxf(fmaxf(lm, l0), lp);
    st.mn = fminf(st.mn, fminf(fminf(lm, l0), lp));
    if (mr > st.m + kRescale) {
        const float f = ex2(st.m - mr);
        st.s *= f;
        st.ax *= f;
        st.ay *= f;
        st.az *= f;
        st.m = mr;
    }
    const float em = ex2(lm - st.m), e0 = ex2(l0 - st.m), ep = ex2(lp - st.m);
    const float rs = em + e0 + ep;
    st.s += rs;
    st.ax += ep - em;
    if (DY > 0) st.ay += rs;
    if (DY < 0) st.ay -= rs;
    if (DZ > 0) st.az += rs;
    if (DZ < 0) st.az -= rs;
}

// ======================================================================= fwd
constexpr int FTX = 32, FTY = 16;                 // tile: 16 threads x 2 voxels, 16 rows
constexpr int FRL = FTX + 2, FPX = 36, FPY = FTY + 2;

template <int D>
struct FwdSlots {
    float q[3][2][D];
    Soft st[3][2];
};

template <int D, int DZ>
__device__ __forceinline__ void fwd_slot_rows(float (&q)[2][D], Soft (&st)[2], const float *P,
                                              const float *sB, int tx, int ty) {
#pragma unroll
    for (int dyi = 0; dyi < 3; ++dyi) {
        float kr[D][4];
        const float *rowp = P + (ty + dyi) * FPX + 2 * tx;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            const float2 a = *reinterpret_cast<const float2 *>(rowp + c * FPY * FPX);
            const float2 b = *reinterpret_cast<const float2 *>(rowp + c * FPY * FPX + 2);
            kr[c][0] = a.x;
            kr[c][1] = a.y;
            kr[c][2] = b.x;
            kr[c][3] = b.y;
        }
        const int ob = (DZ + 1) * 9 + dyi * 3;
        const float b0 = sB[ob], b1 = sB[ob + 1], b2 = sB[ob + 2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            float lm = b0, l0 = b1, lp = b2;
#pragma unroll
            for (int c = 0; c < D; ++c) {
                lm = fmaf(q[r][c], kr[c][r], lm);
                l0 = fmaf(q[r][c], kr[c][r + 1], l0);
                lp = fmaf(q[r][c], kr[c][r + 2], lp);
            }
            if (dyi == 0) soft_row<-1, DZ>(st[r], lm, l0, lp);
            if (dyi == 1) soft_row<0, DZ>(st[r], lm, l0, lp);
            if (dyi == 2) soft_row<1, DZ>(st[r], lm, l0, lp);
        }
    }
}

template <int D, int NEW, int MID, int OLD>
__device__ __forceinline__ void fwd_step(FwdSlots<D> &S_, int p, int zb, int ze, float *smem,
                                         const float *sB, const float *Kh, const float *Qh,
                                         const Vol &v, int x0, int y0, int tx, int ty, int x,
                                         int y, bool v0, bool v1, int s, float *SF, float *LSE,
                                         unsigned long long *flag) {
    constexpr int PLANE = D * FPY * FPX;
    const int buf = (p - zb + 1) & 1;
    cp_wait_all();
    __syncthreads();
    if (p + 1 <= ze)
        stage_plane<D, FPY, FRL, FPX>(smem + (buf ^ 1) * PLANE,
                                      [&](int c) { return Kh + (int64_t)c * v.n; }, p + 1, x0, y0,
                                      v);
    cp_commit();
    const bool has_new = p + 1 < ze, has_mid = p >= zb && p < ze, has_old = p - 1 >= zb;
    if (has_new) {
        const int64_t off = (int64_t)(p + 1) * v.hw + (int64_t)y * v.h + x;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            S_.q[NEW][0][c] = v0 ? __ldg(Qh + (int64_t)c * v.n + off) * kLog2e : 0.0f;
            S_.q[NEW][1][c] = v1 ? __ldg(Qh + (int64_t)c * v.n + off + 1) * kLog2e : 0.0f;
        }
        soft_init(S_.st[NEW][0]);
        soft_init(S_.st[NEW][1]);
    }
    const float *P = smem + buf * PLANE;
    if (has_new) fwd_slot_rows<D, -1>(S_.q[NEW], S_.st[NEW], P, sB, tx, ty);
    if (has_mid) fwd_slot_rows<D, 0>(S_.q[MID], S_.st[MID], P, sB, tx, ty);
    if (has_old) {
        fwd_slot_rows<D, 1>(S_.q[OLD], S_.st[OLD], P, sB, tx, ty);
        const int64_t off = (int64_t)(p - 1) * v.hw + (int64_t)y * v.h + x;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            if (r == 0 ? !v0 : !v1) continue;
            const Soft &t = S_.st[OLD][r];
            const float inv = 1.0f / t.s;
            float *sf = SF + 3 * (int64_t)s * v.n + off + r;
            sf[0] = t.ax * inv;
            sf[v.n] = t.ay * inv;
            sf[2 * v.n] = t.az * inv;
            LSE[(int64_t)s * v.n + off + r] = (t.m + __log2f(t.s)) * kLn2;
            if (!isfinite(t.s) || t.mn == -INFINITY)
                atomicMin(flag, (unsigned long long)s * (unsigned long long)v.n +
                                    (unsigned long long)(off + r));
        }
    }
}

template <int D>
__global__ void __launch_bounds__(256, (D <= 6 ? 2 : 1))
modet_fwd_tiled_k(const float *__restrict__ Q, const float *__restrict__ K,
                  const float *__restrict__ B, Vol v, int zc, float *__restrict__ SF,
                  float *__restrict__ LSE, unsigned long long *__restrict__ flag) {
    constexpr int PLANE = D * FPY * FPX;
    extern __shared__ __align__(16) float smem[];
    float *sB = smem + 2 * PLANE;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int x0 = blockIdx.x * FTX, y0 = blockIdx.y * FTY;
    const int nzc = (v.l + zc - 1) / zc;
    const int s = blockIdx.z / nzc;
    const int zb = (blockIdx.z - s * nzc) * zc, ze = min(zb + zc, v.l);
    const float *Kh = K + (int64_t)s * D * v.n;
    const float *Qh = Q + (int64_t)s * D * v.n;
    const int x = x0 + 2 * tx, y = y0 + ty;
    const bool v0 = y < v.w && x < v.h, v1 = y < v.w && x + 1 < v.h;
    if (threadIdx.x < 27) sB[threadIdx.x] = B[s * 27 + threadIdx.x] * kLog2e;
    stage_plane<D, FPY, FRL, FPX>(smem, [&](int c) { return Kh + (int64_t)c * v.n; }, zb - 1,
                                  x0, y0, v);
    cp_commit();
    FwdSlots<D> S_;
    for (int t = 0;; t += 3) {
        const int p = zb - 1 + t;
        if (p > ze) break;
        fwd_step<D, 0, 2, 1>(S_, p, zb, ze, smem, sB, Kh, Qh, v, x0, y0, tx, ty, x, y, v0, v1,
                             s, SF, LSE, flag);
        if (p + 1 > ze) break;
        fwd_step<D, 1, 0, 2>(S_, p + 1, zb, ze, smem, sB, Kh, Qh, v, x0, y0, tx, ty, x, y, v0,
                             v1, s, SF, LSE, flag);
        if (p + 2 > ze) break;
        fwd_step<D, 2, 1, 0>(S_, p + 2, zb, ze, smem, sB, Kh, Qh, v, x0, y0, tx, ty, x, y, v0,
                             v1, s, SF, LSE, flag);
    }
}

// ================================================================ bwd: rows
// p as query.  Tile 32 x 8, one voxel per thread, 3 in-flight z slots.
constexpr int RTX = 32, RTY = 8;
constexpr int RRL = RTX + 2, RPX = 36, RPY = RTY + 2;

template <int D>
struct RowSlots {
    float q[3][D];   // q * log2e
    float dq[3][D];
    float L[3];      // LSE * log2e
    float gx[3], gy[3], gz[3], dot[3];
};

template <int D, int DZ>
__device__ __forceinline__ void row_slot_rows(RowSlots<D> &R, int j, float (&db)[27],
                                              const float *P, const float *sB, int tx, int ty) {
#pragma unroll
    for (int dyi = 0; dyi < 3; ++dyi) {
        constexpr int dummy = 0;
        (void)dummy;
        float kr[D][3];
        const float *rowp = P + (ty + dyi) * RPX + tx;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            kr[c][0] = rowp[c * RPY * RPX];
            kr[c][1] = rowp[c * RPY * RPX + 1];
            kr[c][2] = rowp[c * RPY * RPX + 2];
        }
        const int ob = (DZ + 1) * 9 + dyi * 3;
        // coefficient gSF.off(o) - gSF.SF without the x term
        float cb = (DZ > 0 ? R.gz[j] : (DZ < 0 ? -R.gz[j] : 0.0f)) - R.dot[j];
        if (dyi == 0) cb -= R.gy[j];
        if (dyi == 2) cb += R.gy[j];
#pragma unroll
        for (int dxi = 0; dxi < 3; ++dxi) {
            float lg = sB[ob + dxi];
#pragma unroll
            for (int c = 0; c < D; ++c) lg = fmaf(R.q[j][c], kr[c][dxi], lg);
            const float W = ex2(lg - R.L[j]);
            const float cf = dxi == 0 ? cb - R.gx[j] : (dxi == 2 ? cb + R.gx[j] : cb);
            const float dl = W * cf;
            db[ob + dxi] += dl;
#pragma unroll
            for (int c = 0; c < D; ++c) R.dq[j][c] = fmaf(dl, kr[c][dxi], R.dq[j][c]);
        }
    }
}

template <int D, bool ACC, int NEW, int MID, int OLD>
__device__ __forceinline__ void row_step(RowSlots<D> &R, float (&db)[27], int p, int zb, int ze,
                                         float *smem, const float *sB, const float *Kh,
                                         const float *Qh, const float *LSEh, const float *gSFh,
                                         const float *SFh, const Vol &v, int x0, int y0, int tx,
                                         int ty, int x, int y, bool vv, float *gQh) {
    constexpr int PLANE = D * RPY * RPX;
    const int buf = (p - zb + 1) & 1;
    cp_wait_all();
    __syncthreads();
    if (p + 1 <= ze)
        stage_plane<D, RPY, RRL, RPX>(smem + (buf ^ 1) * PLANE,
                                      [&](int c) { return Kh + (int64_t)c * v.n; }, p + 1, x0, y0,
                                      v);
    cp_commit();
    const bool has_new = p + 1 < ze, has_mid = p >= zb && p < ze, has_old = p - 1 >= zb;
    if (has_new) {
        const int64_t off = (int64_t)(p + 1) * v.hw + (int64_t)y * v.h + x;
        if (vv) {
#pragma unroll
            for (int c = 0; c < D; ++c) {
                R.q[NEW][c] = __ldg(Qh + (int64_t)c * v.n + off) * kLog2e;
                R.dq[NEW][c] = 0.0f;
            }
            R.L[NEW] = __ldg(LSEh + off) * kLog2e;
            const float gx = __ldg(gSFh + off), gy = __ldg(gSFh + v.n + off),
                        gz = __ldg(gSFh + 2 * v.n + off);
            R.gx[NEW] = gx;
            R.gy[NEW] = gy;
            R.gz[NEW] = gz;
            R.dot[NEW] = gx * __ldg(SFh + off) + gy * __ldg(SFh + v.n + off) +
                         gz * __ldg(SFh + 2 * v.n + off);
        } else {
#pragma unroll
            for (int c = 0; c < D; ++c) R.q[NEW][c] = R.dq[NEW][c] = 0.0f;
            R.L[NEW] = 0.0f;
            R.gx[NEW] = R.gy[NEW] = R.gz[NEW] = R.dot[NEW] = 0.0f;  // => dl == 0
        }
    }
    const float *P = smem + buf * PLANE;
    if (has_new) row_slot_rows<D, -1>(R, NEW, db, P, sB, tx, ty);
    if (has_mid) row_slot_rows<D, 0>(R, MID, db, P, sB, tx, ty);
    if (has_old) {
        row_slot_rows<D, 1>(R, OLD, db, P, sB, tx, ty);
        if (vv && gQh) {
            const int64_t off = (int64_t)(p - 1) * v.hw + (int64_t)y * v.h + x;
#pragma unroll
            for (int c = 0; c < D; ++c) {
                float *dst = gQh + (int64_t)c * v.n + off;
                // dl was formed from log2-domain logits: d/dq = log2e-free since
                // the exponent uses q*log2e*k = (q.k)*log2e; the derivative of
                // exp(q.k) wrt q is exp(.)*k — no extra factor.
                *dst = ACC ? *dst + R.dq[OLD][c] : R.dq[OLD][c];
            }
        }
    }
}

template <int D, bool ACC>
__global__ void __launch_bounds__(256, (D <= 6 ? 2 : 1))
modet_bwd_row_k(const float *__restrict__ Q, const float *__restrict__ K,
                const float *__restrict__ B, const float *__restrict__ SF,
                const float *__restrict__ LSE, const float *__restrict__ gSF, Vol v, int zc,
                float *__restrict__ gQ, float *__restrict__ gBpart) {
    constexpr int PLANE = D * RPY * RPX;
    extern __shared__ __align__(16) float smem[];
    float *sB = smem + 2 * PLANE;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int x0 = blockIdx.x * RTX, y0 = blockIdx.y * RTY;
    const int nzc = (v.l + zc - 1) / zc;
    const int s = blockIdx.z / nzc;
    const int zb = (blockIdx.z - s * nzc) * zc, ze = min(zb + zc, v.l);
    const int64_t so = (int64_t)s * v.n;
    const float *Kh = K + so * D, *Qh = Q + so * D;
    const float *LSEh = LSE + so, *gSFh = gSF + 3 * so, *SFh = SF + 3 * so;
    float *gQh = gQ ? gQ + so * D : nullptr;
    const int x = x0 + tx, y = y0 + ty;
    const bool vv = x < v.h && y < v.w;
    if (threadIdx.x < 27) sB[threadIdx.x] = B[s * 27 + threadIdx.x] * kLog2e;
    stage_plane<D, RPY, RRL, RPX>(smem, [&](int c) { return Kh + (int64_t)c * v.n; }, zb - 1, x0,
                                  y0, v);
    cp_commit();
    RowSlots<D> R;
    float db[27];
#pragma unroll
    for (int o = 0; o < 27; ++o) db[o] = 0.0f;
    for (int t = 0;; t += 3) {
        const int p = zb - 1 + t;
        if (p > ze) break;
        row_step<D, ACC, 0, 2, 1>(R, db, p, zb, ze, smem, sB, Kh, Qh, LSEh, gSFh, SFh, v, x0, y0,
                                  tx, ty, x, y, vv, gQh);
        if (p + 1 > ze) break;
        row_step<D, ACC, 1, 0, 2>(R, db, p + 1, zb, ze, smem, sB, Kh, Qh, LSEh, gSFh, SFh, v, x0,
                                  y0, tx, ty, x, y, vv, gQh);
        if (p + 2 > ze) break;
        row_step<D, ACC, 2, 1, 0>(R, db, p + 2, zb, ze, smem, sB, Kh, Qh, LSEh, gSFh, SFh, v, x0,
                                  y0, tx, ty, x, y, vv, gQh);
    }
    // dB: warp shuffle reduce, then across warps; one partial per CTA
    cp_wait_all();
    __syncthreads();
    float *red = smem;  // reuse: [8 warps][27]
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 0; o < 27; ++o) {
        float a = db[o];
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) a += __shfl_xor_sync(0xffffffffu, a, m);
        if (lane == 0) red[wid * 27 + o] = a;
    }
    __syncthreads();
    if (threadIdx.x < 27) {
        float a = 0.0f;
#pragma unroll
        for (int i = 0; i < 8; ++i) a += red[i * 27 + threadIdx.x];
        const int cta = (blockIdx.z - s * nzc) * gridDim.x * gridDim.y + blockIdx.y * gridDim.x +
                        blockIdx.x;
        const int ncta = nzc * gridDim.x * gridDim.y;
        gBpart[((int64_t)s * ncta + cta) * 27 + threadIdx.x] = a;
    }
}

// ============================================================= bwd: columns
// q as key.  Tile 32 x 16 (16 threads x 2 voxels), 3 in-flight z slots.
// Staged source planes: Q (D channels), LSE, gSF (3), SF (3) -> after landing
// the SF x-plane is overwritten with dot = gSF.SF (one transform pass).
constexpr int CTX = 32, CTY = 16;
constexpr int CRL = CTX + 2, CPX = 36, CPY = CTY + 2;

template <int D>
struct ColSlots {
    float k[3][2][D];  // k * log2e
    float dk[3][2][D];
};

template <int D, int DZ>
__device__ __forceinline__ void col_slot_rows(float (&k)[2][D], float (&dk)[2][D], const float *P,
                                              const float *sB, int tx, int ty) {
    constexpr int CH = CPY * CPX;
    // window slot o = (dx,dy,dz) links source r = q - off(o) to key q
#pragma unroll
    for (int dyi = 0; dyi < 3; ++dyi) {
        // sources at row (ty+1) - (dyi-1) = ty + 2 - dyi, x = 2tx-1 .. 2tx+2
        const float *rowp = P + (ty + 2 - dyi) * CPX + 2 * tx;
        float qs[D][4];
#pragma unroll
        for (int c = 0; c < D; ++c) {
            const float2 a = *reinterpret_cast<const float2 *>(rowp + c * CH);
            const float2 b = *reinterpret_cast<const float2 *>(rowp + c * CH + 2);
            qs[c][0] = a.x;
            qs[c][1] = a.y;
            qs[c][2] = b.x;
            qs[c][3] = b.y;
        }
        float L[4], gx[4], cb[4];
#pragma unroll
        for (int i = 0; i < 4; i += 2) {
            const float2 l2 = *reinterpret_cast<const float2 *>(rowp + D * CH + i);
            const float2 gx2 = *reinterpret_cast<const float2 *>(rowp + (D + 1) * CH + i);
            const float2 gy2 = *reinterpret_cast<const float2 *>(rowp + (D + 2) * CH + i);
            const float2 gz2 = *reinterpret_cast<const float2 *>(rowp + (D + 3) * CH + i);
            const float2 dt2 = *reinterpret_cast<const float2 *>(rowp + (D + 4) * CH + i);
            L[i] = l2.x * kLog2e;
            L[i + 1] = l2.y * kLog2e;
            gx[i] = gx2.x;
            gx[i + 1] = gx2.y;
            // gSF.off(o) - dot without the x term, for this (dy, dz)
            float c0 = -dt2.x, c1 = -dt2.y;
            if (dyi == 0) { c0 -= gy2.x; c1 -= gy2.y; }
            if (dyi == 2) { c0 += gy2.x; c1 += gy2.y; }
            if (DZ < 0) { c0 -= gz2.x; c1 -= gz2.y; }
            if (DZ > 0) { c0 += gz2.x; c1 += gz2.y; }
            cb[i] = c0;
            cb[i + 1] = c1;
        }
        const int ob = (DZ + 1) * 9 + dyi * 3;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
#pragma unroll
            for (int dxi = 0; dxi < 3; ++dxi) {
                const int si = r + 2 - dxi;  // source x index in the strip
                float lg = sB[ob + dxi];
#pragma unroll
                for (int c = 0; c < D; ++c) lg = fmaf(qs[c][si], k[r][c], lg);
                const float W = ex2(lg - L[si]);
                const float cf = dxi == 0 ? cb[si] - gx[si] : (dxi == 2 ? cb[si] + gx[si] : cb[si]);
                const float dl = W * cf;
#pragma unroll
                for (int c = 0; c < D; ++c) dk[r][c] = fmaf(dl, qs[c][si], dk[r][c]);
            }
        }
    }
}

template <int D, bool ACC, int NEW, int MID, int OLD>
__device__ __forceinline__ void col_step(ColSlots<D> &C_, int p, int zb, int ze, float *smem,
                                         const float *sB, const float *Kh, const float *Qh,
                                         const float *LSEh, const float *gSFh, const float *SFh,
                                         const Vol &v, int x0, int y0, int tx, int ty, int x,
                                         int y, bool v0, bool v1, float *gKh) {
    constexpr int NCH = D + 7;
    constexpr int CH = CPY * CPX;
    constexpr int PLANE = NCH * CH;
    const int buf = (p - zb + 1) & 1;
    cp_wait_all();
    __syncthreads();
    // transform the landed plane: dot = gSF . SF into channel D+4
    {
        float *P = smem + buf * PLANE;
        for (int i = threadIdx.x; i < CPY * CRL; i += blockDim.x) {
            const int ry = i / CRL, rx = i - ry * CRL;
            float *e = P + ry * CPX + rx;
            e[(D + 4) * CH] = e[(D + 1) * CH] * e[(D + 4) * CH] + e[(D + 2) * CH] * e[(D + 5) * CH] +
                              e[(D + 3) * CH] * e[(D + 6) * CH];
        }
    }
    auto base = [&](int c) -> const float * {
        if (c < D) return Qh + (int64_t)c * v.n;
        if (c == D) return LSEh;
        if (c < D + 4) return gSFh + (int64_t)(c - D - 1) * v.n;
        return SFh + (int64_t)(c - D - 4) * v.n;
    };
    if (p + 1 <= ze)
        stage_plane<NCH, CPY, CRL, CPX>(smem + (buf ^ 1) * PLANE, base, p + 1, x0, y0, v);
    cp_commit();
    __syncthreads();  // transform visible
    const bool has_new = p + 1 < ze, has_mid = p >= zb && p < ze, has_old = p - 1 >= zb;
    if (has_new) {
        const int64_t off = (int64_t)(p + 1) * v.hw + (int64_t)y * v.h + x;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            C_.k[NEW][0][c] = v0 ? __ldg(Kh + (int64_t)c * v.n + off) * kLog2e : 0.0f;
            C_.k[NEW][1][c] = v1 ? __ldg(Kh + (int64_t)c * v.n + off + 1) * kLog2e : 0.0f;
            C_.dk[NEW][0][c] = C_.dk[NEW][1][c] = 0.0f;
        }
    }
    const float *P = smem + buf * PLANE;
    // key z = p+1 sees sources in plane p at dz = -1 ... wait: o = q - r, so a
    // source plane p below the key (p = z-1) is window offset dz = +1
    if (has_new) col_slot_rows<D, 1>(C_.k[NEW], C_.dk[NEW], P, sB, tx, ty);
    if (has_mid) col_slot_rows<D, 0>(C_.k[MID], C_.dk[MID], P, sB, tx, ty);
    if (has_old) {
        col_slot_rows<D, -1>(C_.k[OLD], C_.dk[OLD], P, sB, tx, ty);
        if (gKh) {
            const int64_t off = (int64_t)(p - 1) * v.hw + (int64_t)y * v.h + x;
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                if (r == 0 ? !v0 : !v1) continue;
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    float *dst = gKh + (int64_t)c * v.n + off + r;
                    *dst = ACC ? *dst + C_.dk[OLD][r][c] : C_.dk[OLD][r][c];
                }
            }
        }
    }
}

template <int D, bool ACC>
__global__ void __launch_bounds__(256, (D <= 6 ? 2 : 1))
modet_bwd_col_k(const float *__restrict__ Q, const float *__restrict__ K,
                const float *__restrict__ B, const float *__restrict__ SF,
                const float *__restrict__ LSE, const float *__restrict__ gSF, Vol v, int zc,
                float *__restrict__ gK) {
    constexpr int PLANE = (D + 7) * CPY * CPX;
    extern __shared__ __align__(16) float smem[];
    float *sB = smem + 2 * PLANE;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int x0 = blockIdx.x * CTX, y0 = blockIdx.y * CTY;
    const int nzc = (v.l + zc - 1) / zc;
    const int s = blockIdx.z / nzc;
    const int zb = (blockIdx.z - s * nzc) * zc, ze = min(zb + zc, v.l);
    const int64_t so = (int64_t)s * v.n;
    const float *Kh = K + so * D, *Qh = Q + so * D;
    const float *LSEh = LSE + so, *gSFh = gSF + 3 * so, *SFh = SF + 3 * so;
    float *gKh = gK + so * D;
    const int x = x0 + 2 * tx, y = y0 + ty;
    const bool v0 = y < v.w && x < v.h, v1 = y < v.w && x + 1 < v.h;
    if (threadIdx.x < 27) sB[threadIdx.x] = B[s * 27 + threadIdx.x] * kLog2e;
    auto base = [&](int c) -> const float * {
        if (c < D) return Qh + (int64_t)c * v.n;
        if (c == D) return LSEh;
        if (c < D + 4) return gSFh + (int64_t)(c - D - 1) * v.n;
        return SFh + (int64_t)(c - D - 4) * v.n;
    };
    stage_plane<D + 7, CPY, CRL, CPX>(smem, base, zb - 1, x0, y0, v);
    cp_commit();
    ColSlots<D> C_;
    for (int t = 0;; t += 3) {
        const int p = zb - 1 + t;
        if (p > ze) break;
        col_step<D, ACC, 0, 2, 1>(C_, p, zb, ze, smem, sB, Kh, Qh, LSEh, gSFh, SFh, v, x0, y0, tx,
                                  ty, x, y, v0, v1, gKh);
        if (p + 1 > ze) break;
        col_step<D, ACC, 1, 0, 2>(C_, p + 1, zb, ze, smem, sB, Kh, Qh, LSEh, gSFh, SFh, v, x0, y0,
                                  tx, ty, x, y, v0, v1, gKh);
        if (p + 2 > ze) break;
        col_step<D, ACC, 2, 1, 0>(C_, p + 2, zb, ze, smem, sB, Kh, Qh, LSEh, gSFh, SFh, v, x0, y0,
                                  tx, ty, x, y, v0, v1, gKh);
    }
}

// deterministic final reduction of per-CTA dB partials (fixed order tree)
__global__ void __launch_bounds__(256)
reduce_db_k(const float *__restrict__ part, int nparts, float *__restrict__ gB) {
    const int s = blockIdx.y, o = blockIdx.x;
    float a = 0.0f;
    for (int i = threadIdx.x; i < nparts; i += 256) a += part[((int64_t)s * nparts + i) * 27 + o];
    __shared__ float sm[256];
    sm[threadIdx.x] = a;
    __syncthreads();
    for (int m = 128; m > 0; m >>= 1) {
        if (threadIdx.x < m) sm[threadIdx.x] += sm[threadIdx.x + m];
        __syncthreads();
    }
    if (threadIdx.x == 0) gB[s * 27 + o] += sm[0];
}

// ------------------------------------------------------------- launchers
static int pick_zc(int tiles, int l) {
    // enough CTAs for ~4 per SM on 148 SMs, chunks of >= 8 planes
    const int want = 148 * 4;
    int nzc = (want + tiles - 1) / max(tiles, 1);
    nzc = max(1, min(nzc, (l + 7) / 8));
    return (l + nzc - 1) / nzc;
}

template <int D>
static cudaError_t fwd_launch(const float *Q, const float *K, const float *B, mdg_dims3 d, int S,
                              float *SF, float *LSE, unsigned long long *flag, cudaStream_t st) {
    const Vol v{d.h, d.w, d.l, (int64_t)d.h * d.w * d.l, (int64_t)d.h * d.w};
    const int gx = (d.h + FTX - 1) / FTX, gy = (d.w + FTY - 1) / FTY;
    const int zc = pick_zc(gx * gy * S, d.l);
    const int nzc = (d.l + zc - 1) / zc;
    const size_t sm = (2 * D * FPY * FPX + 32) * sizeof(float);
    auto k = modet_fwd_tiled_k<D>;
    if (sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<dim3(gx, gy, S * nzc), 256, sm, st>>>(Q, K, B, v, zc, SF, LSE, flag);
    return cudaPeekAtLastError();
}

template <int D>
static cudaError_t bwd_launch(const float *Q, const float *K, const float *B, const float *SF,
                              const float *LSE, const float *gSF, mdg_dims3 d, int S, bool acc,
                              float *gQ, float *gK, float *gB, cudaStream_t st) {
    const Vol v{d.h, d.w, d.l, (int64_t)d.h * d.w * d.l, (int64_t)d.h * d.w};
    cudaError_t e = cudaSuccess;
    if (gQ || gB) {
        const int gx = (d.h + RTX - 1) / RTX, gy = (d.w + RTY - 1) / RTY;
        const int zc = pick_zc(gx * gy * S, d.l);
        const int nzc = (d.l + zc - 1) / zc;
        const int ncta = gx * gy * nzc;
        float *part = nullptr;
        if ((e = cudaMallocAsync(&part, (size_t)S * ncta * 27 * sizeof(float), st))) return e;
        const size_t sm = (2 * D * RPY * RPX + 32) * sizeof(float);
        auto k = acc ? modet_bwd_row_k<D, true> : modet_bwd_row_k<D, false>;
        if (sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k<<<dim3(gx, gy, S * nzc), 256, sm, st>>>(Q, K, B, SF, LSE, gSF, v, zc, gQ, part);
        g_launches.fetch_add(1);
        if (gB) {
            reduce_db_k<<<dim3(27, S), 256, 0, st>>>(part, ncta, gB);
            g_launches.fetch_add(1);
        }
        cudaFreeAsync(part, st);
        if ((e = cudaPeekAtLastError())) return e;
    }
    if (gK) {
        const int gx = (d.h + CTX - 1) / CTX, gy = (d.w + CTY - 1) / CTY;
        const int zc = pick_zc(gx * gy * S, d.l);
        const int nzc = (d.l + zc - 1) / zc;
        const size_t sm = (2 * (D + 7) * CPY * CPX + 32) * sizeof(float);
        auto k = acc ? modet_bwd_col_k<D, true> : modet_bwd_col_k<D, false>;
        if (sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k<<<dim3(gx, gy, S * nzc), 256, sm, st>>>(Q, K, B, SF, LSE, gSF, v, zc, gK);
        g_launches.fetch_add(1);
        if ((e = cudaPeekAtLastError())) return e;
    }
    return e;
}

}  // namespace tiled

// entry points used by modet.cu (planar layout, nb = 3); false => unsupported hd
bool tiled_fwd(int hd, const float *Q, const float *K, const float *B, mdg_dims3 d, int S,
               float *SF, float *LSE, unsigned long long *flag, cudaStream_t st, cudaError_t *err) {
    using namespace tiled;
    switch (hd) {
#define MDG_T(DV) \
    case DV: *err = fwd_launch<DV>(Q, K, B, d, S, SF, LSE, flag, st); return true;
        MDG_T(1) MDG_T(2) MDG_T(3) MDG_T(4) MDG_T(5) MDG_T(6) MDG_T(8) MDG_T(12) MDG_T(16)
#undef MDG_T
        default: return false;
    }
}

bool tiled_bwd(int hd, const float *Q, const float *K, const float *B, const float *SF,
               const float *LSE, const float *gSF, mdg_dims3 d, int S, bool acc, float *gQ,
               float *gK, float *gB, cudaStream_t st, cudaError_t *err) {
    using namespace tiled;
    switch (hd) {
#define MDG_T(DV) \
    case DV: *err = bwd_launch<DV>(Q, K, B, SF, LSE, gSF, d, S, acc, gQ, gK, gB, st); return true;
        MDG_T(1) MDG_T(2) MDG_T(3) MDG_T(4) MDG_T(5) MDG_T(6) MDG_T(8) MDG_T(12) MDG_T(16)
#undef MDG_T
        default: return false;
    }
}

}  // namespace mdg
