// modet_tiled.cu — tiled ModeT kernels for the native planar layout.
//
// Layout: Q, K planar {S*d, n}; head s owns channel planes s*d .. s*d+d-1.
//
// Every kernel is a z-marching CTA of 32 x 8 threads: it owns an x-y column
// tile (one voxel column per thread) and walks a chunk of z.  Step p consumes
// one shared-memory buffer holding
//   * the HALO plane p of the arrays the thread GATHERS from (tile + 1-voxel
//     x/y halo), and
//   * the tile INTERIOR of the arrays the thread OWNS, at plane p+1 (the voxel
//     that enters the in-flight window this step),
// double-buffered.  Staging is 4-D TMA box loads (cp.async.bulk.tensor, one
// issuing thread, mbarrier completion); TMA's out-of-bounds zero fill is the
// reference's "out-of-bounds key contributes nothing, logit = bias" rule
// (attention.hpp:77-81).  The innermost TMA start coordinate must be 16-byte
// aligned, so halo boxes start at x0-4 and are 40 wide (logical halo column rx
// lives at physical column rx+3).  Volumes whose row pitch is not a multiple
// of 16 bytes (h % 4 != 0) use 4-byte cp.async into the same layout.
//
// A staged x-strip is read from shared memory ONCE per step and used by the
// three voxels of the thread's column that have plane p in their 3x3x3 window
// (z = p+1, p, p-1: the "in-flight" slots).  Slot arithmetic is unconditional
// (idle slots carry LSE = +inf / zero data), so the three slots' dependency
// chains interleave.  Channels are processed in pairs on Blackwell's packed
// FP32 pipe (FFMA2 / FADD2 / FMUL2), which doubles FP32 work per issue slot.
//
//   fwd  (modet_fwd_tiled_k): 27 logits per voxel in log2 units (q pre-scaled
//        by log2 e); branch-free online softmax one 3-logit x-row at a time —
//        the first row sets the reference max, later rows never rescale;
//        voxels whose sum overflowed or that saw a non-finite logit are queued
//        and recomputed exactly by modet_fwd_fixup_k.  Writes SF {3S,n} and
//        LSE {S,n} (natural log).  One block barrier per step (3 CTAs/SM).
//   bwd  row kernel (modet_bwd_row_k): p as query.  W = exp2(l - LSE*log2e)
//        recomputed, dl = W*(gSF.off(o) - gSF.SF) (since <W, gW> = gSF.SF),
//        dQ_p += dl*K_{p+o}, per-CTA dB partials (deterministic reduce), and
//        the per-voxel {LSE*log2e, gSF.SF} the column kernel consumes.
//   bwd  column kernel (modet_bwd_col_k): q as key, gathering from staged
//        sources r = q - off(o): dK_q += dl(r,o)*Q_r.  The reference's scatter
//        (attention.hpp:159-162) as a gather: no atomics, fixed order.
//   Both backward kernels release buffers without a block barrier: the last
//   warp to finish a step re-arms that buffer's TMA for the step two ahead.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "mdg_common.cuh"

#ifndef MDG_BWD_MINB
#define MDG_BWD_MINB 2  // resident CTAs of the row / column kernels (d <= 6)
#endif
#ifndef MDG_BWD_ROW_MINB
#define MDG_BWD_ROW_MINB MDG_BWD_MINB
#endif
#ifndef MDG_BWD_COL_MINB  // the column kernel fits 3 (79 registers, no spill):
#define MDG_BWD_COL_MINB 3  // 0.4505 vs 0.4554 ms (profiles/experiments/modet_bwd_split_minb_r02.log)
#endif
#ifndef MDG_BWD_MINB8
#define MDG_BWD_MINB8 1  // the same for d = 8..16
#endif

namespace mdg {
namespace tiled {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr int kXOff = 3;           // physical column of logical halo column 0
constexpr int kBoxX = 40;          // halo box width (starts at x0 - 4)

__host__ __device__ constexpr int up32(int v) { return (v + 31) / 32 * 32; }

// ------------------------------------------------------------ packed fp32
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 dup2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

// ------------------------------------------------------- async copy helpers
__device__ __forceinline__ unsigned su32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async4(float *dst, const float *src, bool pred) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(su32(dst)), "l"(src),
                 "r"(pred ? 4 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned phase) {
    unsigned done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(su32(b)), "r"(phase)
            : "memory");
    } while (!done);
}
// 4-D TMA box load (x, y, z, channel); OOB elements are zero-filled
__device__ __forceinline__ void tma4(float *dst, const CUtensorMap *m, int x, int y, int z, int c,
                                     uint64_t *b) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(su32(dst)),
        "l"(m), "r"(x), "r"(y), "r"(z), "r"(c), "r"(su32(b))
        : "memory");
}

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float2 ex2x2(float2 d) { return f2(ex2(d.x), ex2(d.y)); }

struct Vol {
    int h, w, l;
    int64_t n, hw;
};

// The two array sets of the operator:  set K = {K (d ch)}, set A = {Q (d ch),
// LSE (1), gSF (3), SF (3)}.  fwd gathers K / owns Q; the row kernel gathers K
// / owns A; the column kernel gathers A / owns K.
struct MapsA {
    CUtensorMap q, lse, g, sf;
};
struct Maps {
    CUtensorMap k;    // set K
    MapsA a;          // set A
    CUtensorMap aux;  // column kernel: per-source {LSE*log2e, gSF.SF} from the row kernel
};

struct Ptrs {
    const float *K, *Q, *LSE, *gSF, *SF;  // head-offset bases
    const float *AUX = nullptr;           // {2, n} of this head (column kernel)
    // column-kernel halo channel c: Q (D), aux (2), gSF (3)
    __device__ __forceinline__ const float *c_src(int c, int D, int64_t n) const {
        if (c < D) return Q + (int64_t)c * n;
        if (c < D + 2) return AUX + (int64_t)(c - D) * n;
        return gSF + (int64_t)(c - D - 2) * n;
    }
    __device__ __forceinline__ const float *a(int c, int D, int64_t n) const {
        if (c < D) return Q + (int64_t)c * n;
        if (c == D) return LSE;
        if (c < D + 4) return gSF + (int64_t)(c - D - 1) * n;
        return SF + (int64_t)(c - D - 4) * n;
    }
    __device__ __forceinline__ const float *k(int c, int64_t n) const { return K + (int64_t)c * n; }
};

// ---------------------------------------------------------------- staging
// Buffer = [halo: channel slots of HCH floats][own: channel slots of TX*TY].
template <int TX, int TY>
struct Geo {
    static constexpr int PY = TY + 2, RL = TX + 2, HCH = up32(PY * kBoxX), OCH = TX * TY;
};

// cp.async fallback, halo part: logical (ry, rx) -> physical ry*40 + rx + 3
template <int NCH, int TX, int TY, class Base>
__device__ __forceinline__ void cp_halo(float *dst, Base base, int z, int x0, int y0,
                                        const Vol &v) {
    using G = Geo<TX, TY>;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const bool zok = z >= 0 && z < v.l;
    int c = 0, ry = wid;
    for (int r = wid; r < NCH * G::PY; r += nw) {
        while (ry >= G::PY) {
            ry -= G::PY;
            ++c;
        }
        const int gy = y0 - 1 + ry;
        const bool rok = zok && gy >= 0 && gy < v.w;
        const float *row = base(c);
        const int64_t roff = (int64_t)z * v.hw + (int64_t)gy * v.h;
        float *drow = dst + c * G::HCH + ry * kBoxX + kXOff;
        for (int rx = lane; rx < G::RL; rx += 32) {
            const int gx = x0 - 1 + rx;
            const bool ok = rok && gx >= 0 && gx < v.h;
            cp_async4(drow + rx, ok ? row + roff + gx : row, ok);
        }
        ry += nw;
    }
}

// cp.async fallback, own part: (ty, tx) -> physical ty*TX + tx
template <int NCH, int TX, int TY, class Base>
__device__ __forceinline__ void cp_own(float *dst, Base base, int z, int x0, int y0,
                                       const Vol &v) {
    const bool zok = z >= 0 && z < v.l;
    for (int i = threadIdx.x; i < NCH * TX * TY; i += blockDim.x) {
        const int c = i / (TX * TY), e = i - c * (TX * TY);
        const int gy = y0 + e / TX, gx = x0 + e % TX;
        const bool ok = zok && gy < v.w && gx < v.h;
        const float *row = base(c);
        cp_async4(dst + i, ok ? row + (int64_t)z * v.hw + (int64_t)gy * v.h + gx : row, ok);
    }
}

// Strip of the 4 logical halo columns 2tx-1 .. 2tx+2 (relative to the tile:
// physical 2tx+3 .. 2tx+6) of one row, as the three overlapping pairs the two
// voxels x = 2tx, 2tx+1 need for dx = -1, 0, +1.
struct Strip {
    float2 p[3];  // {k0,k1}, {k1,k2}, {k2,k3}
};
__device__ __forceinline__ Strip strip(const float *rowp, int tx) {
    const float *e = rowp + 2 * tx + 2;
    const float k0 = e[1];
    const float2 m = *reinterpret_cast<const float2 *>(e + 2);
    const float k3 = e[4];
    Strip s;
    s.p[0] = f2(k0, m.x);
    s.p[1] = m;
    s.p[2] = f2(m.y, k3);
    return s;
}

template <int V>
using IC = std::integral_constant<int, V>;

// z-marching driver: f(p, NEW, MID, OLD) for p = zb-1 .. ze with the slot
// roles rotating every step (voxel z lives in slot (z - zb) mod 3)
template <class F>
__device__ __forceinline__ void march(int zb, int ze, F &&f) {
    for (int t = 0;; t += 3) {
        const int p = zb - 1 + t;
        if (p > ze) break;
        f(p, IC<0>(), IC<2>(), IC<1>());
        if (p + 1 > ze) break;
        f(p + 1, IC<1>(), IC<0>(), IC<2>());
        if (p + 2 > ze) break;
        f(p + 2, IC<2>(), IC<1>(), IC<0>());
    }
}

__device__ __forceinline__ void init_bars(uint64_t *bar) {
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
}

// Buffer release without a block barrier (TMA path).  Each of the 8 compute
// warps bumps the buffer's counter once it has finished reading it; the warp
// that brings it to 8 re-arms the buffer: it resets the counter and issues the
// TMA loads of the step two ahead.  No warp ever waits for another — only for
// its data (the full mbarrier) — so warps drift freely within the one step of
// slack the double buffer gives.
constexpr int kWarps = 8;
__device__ __forceinline__ bool last_out(int *cnt) {
    __syncwarp();
    bool last = false;
    if ((threadIdx.x & 31) == 0) {
        __threadfence_block();  // release this warp's reads of the buffer
        last = atomicAdd(cnt, 1) == kWarps - 1;
        if (last) {
            *cnt = 0;
            __threadfence_block();
            // generic-proxy reads ordered before the async-proxy (TMA) refill
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        }
    }
    return last;
}

// bias pairs {B*log2e, B*log2e} for the 27 window slots of head s
__device__ __forceinline__ void load_bias2(float2 *sB2, const float *B, int s) {
    if (threadIdx.x < 27) sB2[threadIdx.x] = dup2(B[s * 27 + threadIdx.x] * kLog2e);
}

// ------------------------------------------------------------ fixup queue
__device__ __forceinline__ void fixup_push(unsigned long long *q, unsigned long long key) {
    const unsigned long long i = atomicAdd(q, 1ull);
    if (i < (unsigned long long)kFixupCap) q[1 + i] = key;
}

// Exact per-voxel recomputation (attention.hpp:83-123 + 282-298 maths, true
// row max) of the queued voxel-heads; a queue overflow (pathological inputs)
// recomputes every voxel.  Non-finite logits raise the numeric flag with the
// reference's (head, z, y, x) ordering key.
template <int D>
__global__ void __launch_bounds__(256)
modet_fwd_fixup_k(const float *__restrict__ Q, const float *__restrict__ K,
                  const float *__restrict__ B, Vol v, int S, float *__restrict__ SF,
                  float *__restrict__ LSE, const unsigned long long *__restrict__ fixq,
                  unsigned long long *__restrict__ flag) {
    const unsigned long long cnt = fixq[0];
    if (cnt == 0) return;
    const bool all = cnt > (unsigned long long)kFixupCap;
    const int64_t total = all ? (int64_t)S * v.n : (int64_t)cnt;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t key = all ? i : (int64_t)fixq[1 + i];
        if (key < 0 || key >= (int64_t)S * v.n) continue;  // defensive: never this launch's
        const int s = (int)(key / v.n);
        const int64_t p = key - (int64_t)s * v.n;
        const int x = (int)(p % v.h), y = (int)((p / v.h) % v.w), z = (int)(p / v.hw);
        const float *qb = Q + (int64_t)s * D * v.n + p;
        const float *kb = K + (int64_t)s * D * v.n;
        float q[D];
#pragma unroll
        for (int c = 0; c < D; ++c) q[c] = qb[(int64_t)c * v.n];
        float lg[27];
        bool bad = false;
        float mx = -INFINITY;
#pragma unroll
        for (int o = 0; o < 27; ++o) {
            const int dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
            float a = B[s * 27 + o];
            const int xx = x + dx, yy = y + dy, zz = z + dz;
            if (xx >= 0 && xx < v.h && yy >= 0 && yy < v.w && zz >= 0 && zz < v.l) {
                const int64_t pq = ((int64_t)zz * v.w + yy) * v.h + xx;
                float dot = 0.0f;
#pragma unroll
                for (int c = 0; c < D; ++c) dot = fmaf(q[c], kb[(int64_t)c * v.n + pq], dot);
                a += dot;
            }
            bad |= !isfinite(a);
            mx = fmaxf(mx, a);
            lg[o] = a;
        }
        if (bad) {
            atomicMin(flag, (unsigned long long)key);
            continue;
        }
        float sum = 0.0f, ax = 0.0f, ay = 0.0f, az = 0.0f;
#pragma unroll
        for (int o = 0; o < 27; ++o) {
            const float e = __expf(lg[o] - mx);
            sum += e;
            ax += (o % 3 - 1) * e;
            ay += ((o / 3) % 3 - 1) * e;
            az += (o / 9 - 1) * e;
        }
        const float inv = 1.0f / sum;
        SF[(3 * (int64_t)s + 0) * v.n + p] = ax * inv;
        SF[(3 * (int64_t)s + 1) * v.n + p] = ay * inv;
        SF[(3 * (int64_t)s + 2) * v.n + p] = az * inv;
        LSE[(int64_t)s * v.n + p] = mx + logf(sum);
    }
}

// ======================================================================= fwd
constexpr int FTX = 32, FTY = 8;  // tile: one voxel per thread, a warp per x-row
using FG = Geo<FTX, FTY>;

// online-softmax state of one (voxel, head) row
struct Soft {
    float m, s, ax, ay, az;
    float mn;  // running min logit (a -inf logit is a numeric error)
};

// fold one x-row of three logits (dx = -1, 0, +1) at window row (dy, dz)
template <int DY, int DZ, bool FIRST>
__device__ __forceinline__ void soft_row(Soft &st, float lm, float l0, float lp) {
    st.mn = fminf(st.mn, fminf(fminf(lm, l0), lp));
    // The first row fixes the reference max; later rows never rescale (no
    // branch in the hot loop).  A later logit more than 128 (log2 units)
    // above it overflows the sum to inf: such voxels are queued and redone
    // exactly by modet_fwd_fixup_k.
    if (FIRST) st.m = fmaxf(fmaxf(lm, l0), lp);
    const float em = ex2(lm - st.m), e0 = ex2(l0 - st.m), ep = ex2(lp - st.m);
    const float rs = (em + e0) + ep;
    const float dx = ep - em;
    if (FIRST) {
        st.s = rs;
        st.ax = dx;
        st.ay = DY > 0 ? rs : (DY < 0 ? -rs : 0.0f);
        st.az = DZ > 0 ? rs : (DZ < 0 ? -rs : 0.0f);
    } else {
        st.s += rs;
        st.ax += dx;
        if (DY > 0) st.ay += rs;
        if (DY < 0) st.ay -= rs;
        if (DZ > 0) st.az += rs;
        if (DZ < 0) st.az -= rs;
    }
}

template <int D>
struct FwdSlots {
    static constexpr int D2 = (D + 1) / 2;
    float2 q[3][D2];  // channel pairs of q * log2e (odd D: last .y = 0)
    Soft st[3];
};

// logits of one window x-row on the packed pipe: channel pairs accumulate
// {even, odd} partial dots, combined once per logit
template <int D, int DYI, int DZ, bool FIRST>
__device__ __forceinline__ void fwd_slot(const float2 (&q)[(D + 1) / 2], Soft &st,
                                         const float2 (&kr)[(D + 1) / 2][3], const float2 *sB2) {
    constexpr int D2 = (D + 1) / 2;
    constexpr int ob = (DZ + 1) * 9 + DYI * 3;
    float2 am = f2(sB2[ob].x, 0.0f), a0 = f2(sB2[ob + 1].x, 0.0f), ap = f2(sB2[ob + 2].x, 0.0f);
#pragma unroll
    for (int c = 0; c < D2; ++c) {
        am = fma2(q[c], kr[c][0], am);
        a0 = fma2(q[c], kr[c][1], a0);
        ap = fma2(q[c], kr[c][2], ap);
    }
    soft_row<DYI - 1, DZ, FIRST>(st, am.x + am.y, a0.x + a0.y, ap.x + ap.y);
}

template <int D, bool TMA>
__device__ __forceinline__ void fwd_stage(float *buf, const Maps &m, uint64_t *bar, int p,
                                          int x0, int y0, int s, const Ptrs &P, const Vol &v,
                                          bool issuer) {
    float *own = buf + D * FG::HCH;
    if (TMA) {
        if (issuer) {
            mbar_expect_tx(bar, D * (FG::PY * kBoxX + FG::OCH) * 4);
#pragma unroll
            for (int c = 0; c < D; ++c) {
                tma4(buf + c * FG::HCH, &m.k, x0 - 4, y0 - 1, p, s * D + c, bar);
                tma4(own + c * FG::OCH, &m.a.q, x0, y0, p + 1, s * D + c, bar);
            }
        }
    } else {
        cp_halo<D, FTX, FTY>(buf, [&](int c) { return P.k(c, v.n); }, p, x0, y0, v);
        cp_own<D, FTX, FTY>(own, [&](int c) { return P.a(c, D, v.n); }, p + 1, x0, y0, v);
        cp_commit();
    }
}

template <int D, bool TMA>
#ifndef MDG_FWD_MINB
#define MDG_FWD_MINB 3
#endif
__global__ void __launch_bounds__(256, (D <= 6 ? MDG_FWD_MINB : 2))
modet_fwd_tiled_k(const __grid_constant__ Maps maps, const float *__restrict__ Q,
                  const float *__restrict__ K, const float *__restrict__ B, Vol v, int zc,
                  float *__restrict__ SF, float *__restrict__ LSE,
                  unsigned long long *__restrict__ fixq) {
    constexpr int D2 = (D + 1) / 2;
    constexpr int BUF = D * (FG::HCH + FG::OCH);
    extern __shared__ __align__(128) float smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 2 * BUF);
    float2 *sB2 = reinterpret_cast<float2 *>(smem + 2 * BUF + 8);
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int x0 = blockIdx.x * FTX, y0 = blockIdx.y * FTY;
    const int nzc = (v.l + zc - 1) / zc;
    const int s = blockIdx.z / nzc;
    const int zb = (blockIdx.z - s * nzc) * zc, ze = min(zb + zc, v.l);
    const Ptrs P{K + (int64_t)s * D * v.n, Q + (int64_t)s * D * v.n, nullptr, nullptr, nullptr};
    const int x = x0 + tx, y = y0 + ty;
    const bool vv = y < v.w && x < v.h;
    load_bias2(sB2, B, s);
    if (TMA) init_bars(bar);
    __syncthreads();
    // (the forward keeps one block barrier per step: with three resident CTAs
    // per SM the barrier wait is hidden, and it measured faster than the
    // counter-based release the backward kernels use)
    fwd_stage<D, TMA>(smem, maps, &bar[0], zb - 1, x0, y0, s, P, v, threadIdx.x == 0);
    FwdSlots<D> S_;
    march(zb, ze, [&](int p, auto NEW_, auto MID_, auto OLD_) {
        constexpr int NEW = decltype(NEW_)::value, MID = decltype(MID_)::value,
                      OLD = decltype(OLD_)::value;
        const int j = p - zb + 1, b = j & 1;
        if (TMA) mbar_wait(&bar[b], (j >> 1) & 1);
        else cp_wait_all();
        __syncthreads();
        if (p + 1 <= ze)
            fwd_stage<D, TMA>(smem + (b ^ 1) * BUF, maps, &bar[b ^ 1], p + 1, x0, y0, s, P, v,
                              threadIdx.x == 0);
        const float *buf = smem + b * BUF;
        const bool has_new = p + 1 < ze, has_old = p - 1 >= zb;
        if (has_new) {
            const float *own = buf + D * FG::HCH + ty * FTX + tx;
#pragma unroll
            for (int c = 0; c < D2; ++c) {
                const float a = own[(2 * c) * FG::OCH];
                const float bq = 2 * c + 1 < D ? own[(2 * c + 1) * FG::OCH] : 0.0f;
                S_.q[NEW][c] = mul2(f2(a, bq), dup2(kLog2e));
            }
            S_.st[NEW].mn = INFINITY;
        }
#pragma unroll
        for (int dyi = 0; dyi < 3; ++dyi) {
            // channel pairs of the 3 keys x-1, x, x+1 of window row dy = dyi-1
            float2 ks[D2][3];
#pragma unroll
            for (int c = 0; c < D2; ++c) {
                const float *e0 = buf + (2 * c) * FG::HCH + (ty + dyi) * kBoxX + kXOff + tx;
                const float *e1 = e0 + FG::HCH;
#pragma unroll
                for (int i = 0; i < 3; ++i) ks[c][i] = f2(e0[i], 2 * c + 1 < D ? e1[i] : 0.0f);
            }
            // slot z sees plane p at window offset dz = p - z; the new slot's
            // very first row initialises its softmax state
            if (dyi == 0) {
                fwd_slot<D, 0, -1, true>(S_.q[NEW], S_.st[NEW], ks, sB2);
                fwd_slot<D, 0, 0, false>(S_.q[MID], S_.st[MID], ks, sB2);
                fwd_slot<D, 0, 1, false>(S_.q[OLD], S_.st[OLD], ks, sB2);
            } else if (dyi == 1) {
                fwd_slot<D, 1, -1, false>(S_.q[NEW], S_.st[NEW], ks, sB2);
                fwd_slot<D, 1, 0, false>(S_.q[MID], S_.st[MID], ks, sB2);
                fwd_slot<D, 1, 1, false>(S_.q[OLD], S_.st[OLD], ks, sB2);
            } else {
                fwd_slot<D, 2, -1, false>(S_.q[NEW], S_.st[NEW], ks, sB2);
                fwd_slot<D, 2, 0, false>(S_.q[MID], S_.st[MID], ks, sB2);
                fwd_slot<D, 2, 1, false>(S_.q[OLD], S_.st[OLD], ks, sB2);
            }
        }
        if (has_old && vv) {
            const int64_t off = (int64_t)(p - 1) * v.hw + (int64_t)y * v.h + x;
            const Soft &t = S_.st[OLD];
            const float inv = 1.0f / t.s;
            float *sf = SF + 3 * (int64_t)s * v.n + off;
            sf[0] = t.ax * inv;
            sf[v.n] = t.ay * inv;
            sf[2 * v.n] = t.az * inv;
            LSE[(int64_t)s * v.n + off] = (t.m + __log2f(t.s)) * kLn2;
            // overflow (huge logit spread) or a non-finite logit: exact redo
            if (!isfinite(t.s) || t.mn == -INFINITY)
                fixup_push(fixq, (unsigned long long)((int64_t)s * v.n + off));
        }
    });
}

// ================================================================ bwd: rows
// p as query.  Tile 32 x 8, one voxel per thread, 3 in-flight z slots;
// channels processed in packed pairs.
constexpr int RTX = 32, RTY = 8;
using RG = Geo<RTX, RTY>;

template <int D>
struct RowSlots {
    static constexpr int D2 = (D + 1) / 2;
    float2 q[3][D2];  // channel pairs of q * log2e (odd D: last .y = 0)
    float2 dq[3][D2];
    float L[3];  // LSE * log2e
    float gx[3], gy[3], gz[3], dot[3];
};

template <int D, int DYI, int DZ>
__device__ __forceinline__ void row_slot(RowSlots<D> &R, int j, float (&db)[27],
                                         const float2 (&kr)[(D + 1) / 2][3], const float2 *sB2) {
    constexpr int D2 = (D + 1) / 2;
    constexpr int ob = (DZ + 1) * 9 + DYI * 3;
    // gSF.off(o) - gSF.SF without the x term
    float cb = -R.dot[j];
    if (DZ > 0) cb += R.gz[j];
    if (DZ < 0) cb -= R.gz[j];
    if (DYI == 0) cb -= R.gy[j];
    if (DYI == 2) cb += R.gy[j];
#pragma unroll
    for (int dxi = 0; dxi < 3; ++dxi) {
        float2 acc = f2(sB2[ob + dxi].x, 0.0f);
#pragma unroll
        for (int c = 0; c < D2; ++c) acc = fma2(R.q[j][c], kr[c][dxi], acc);
        const float W = ex2(acc.x + acc.y - R.L[j]);
        const float cf = dxi == 0 ? cb - R.gx[j] : (dxi == 2 ? cb + R.gx[j] : cb);
        const float dl = W * cf;
        db[ob + dxi] += dl;
        const float2 dl2 = dup2(dl);
#pragma unroll
        for (int c = 0; c < D2; ++c) R.dq[j][c] = fma2(dl2, kr[c][dxi], R.dq[j][c]);
    }
}

template <int D, bool TMA>
__device__ __forceinline__ void row_stage(float *buf, const Maps &m, uint64_t *bar, int p,
                                          int x0, int y0, int s, const Ptrs &P, const Vol &v,
                                          bool issuer) {
    float *own = buf + D * RG::HCH;
    if (TMA) {
        if (issuer) {
            mbar_expect_tx(bar, (D * RG::PY * kBoxX + (D + 7) * RG::OCH) * 4);
#pragma unroll
            for (int c = 0; c < D; ++c) {
                tma4(buf + c * RG::HCH, &m.k, x0 - 4, y0 - 1, p, s * D + c, bar);
                tma4(own + c * RG::OCH, &m.a.q, x0, y0, p + 1, s * D + c, bar);
            }
            tma4(own + D * RG::OCH, &m.a.lse, x0, y0, p + 1, s, bar);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                tma4(own + (D + 1 + c) * RG::OCH, &m.a.g, x0, y0, p + 1, 3 * s + c, bar);
                tma4(own + (D + 4 + c) * RG::OCH, &m.a.sf, x0, y0, p + 1, 3 * s + c, bar);
            }
        }
    } else {
        cp_halo<D, RTX, RTY>(buf, [&](int c) { return P.k(c, v.n); }, p, x0, y0, v);
        cp_own<D + 7, RTX, RTY>(own, [&](int c) { return P.a(c, D, v.n); }, p + 1, x0, y0, v);
        cp_commit();
    }
}

template <int D, bool TMA, bool ACC>
__global__ void __launch_bounds__(256, (D <= 6 ? MDG_BWD_ROW_MINB : MDG_BWD_MINB8))
modet_bwd_row_k(const __grid_constant__ Maps maps, const float *__restrict__ Q,
                const float *__restrict__ K, const float *__restrict__ B,
                const float *__restrict__ SF, const float *__restrict__ LSE,
                const float *__restrict__ gSF, Vol v, int zc, float *__restrict__ gQ,
                float *__restrict__ gBpart, float *__restrict__ aux) {
    constexpr int D2 = (D + 1) / 2;
    constexpr int BUF = D * RG::HCH + (D + 7) * RG::OCH;
    extern __shared__ __align__(128) float smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 2 * BUF);
    float2 *sB2 = reinterpret_cast<float2 *>(smem + 2 * BUF + 8);
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int x0 = blockIdx.x * RTX, y0 = blockIdx.y * RTY;
    const int nzc = (v.l + zc - 1) / zc;
    const int s = blockIdx.z / nzc;
    const int zb = (blockIdx.z - s * nzc) * zc, ze = min(zb + zc, v.l);
    const int64_t so = (int64_t)s * v.n;
    const Ptrs P{K + so * D, Q + so * D, LSE + so, gSF + 3 * so, SF + 3 * so};
    float *gQh = gQ ? gQ + so * D : nullptr;
    const int x = x0 + tx, y = y0 + ty;
    const bool vv = x < v.h && y < v.w;
    int *cnt = reinterpret_cast<int *>(smem + 2 * BUF + 8 + 64);
    load_bias2(sB2, B, s);
    if (TMA) init_bars(bar);
    if (threadIdx.x < 2) cnt[threadIdx.x] = 0;
    __syncthreads();
    row_stage<D, TMA>(smem, maps, &bar[0], zb - 1, x0, y0, s, P, v, threadIdx.x == 0);
    if (TMA) row_stage<D, TMA>(smem + BUF, maps, &bar[1], zb, x0, y0, s, P, v, threadIdx.x == 0);
    // Slots are computed unconditionally (no per-slot branches, so the three
    // slots' dependency chains interleave); a slot that holds no voxel has
    // LSE = +inf, q = g = 0, i.e. W = 0 and dl = 0 exactly: nothing reaches dB.
    RowSlots<D> R;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
#pragma unroll
        for (int c = 0; c < (D + 1) / 2; ++c) R.q[j][c] = R.dq[j][c] = f2(0.0f, 0.0f);
        R.L[j] = INFINITY;
        R.gx[j] = R.gy[j] = R.gz[j] = R.dot[j] = 0.0f;
    }
    float db[27];
#pragma unroll
    for (int o = 0; o < 27; ++o) db[o] = 0.0f;
    march(zb, ze, [&](int p, auto NEW_, auto MID_, auto OLD_) {
        constexpr int NEW = decltype(NEW_)::value, MID = decltype(MID_)::value,
                      OLD = decltype(OLD_)::value;
        const int j = p - zb + 1, b = j & 1;
        if (TMA) {
            mbar_wait(&bar[b], (j >> 1) & 1);
        } else {
            cp_wait_all();
            __syncthreads();
            if (p + 1 <= ze)
                row_stage<D, TMA>(smem + (b ^ 1) * BUF, maps, &bar[b ^ 1], p + 1, x0, y0, s, P,
                                  v, true);
        }
        const float *buf = smem + b * BUF;
        const bool has_new = p + 1 < ze, has_old = p - 1 >= zb;
        if (has_new) {
            // own data of the voxel entering the window; zero outside the
            // volume (TMA / cp.async zero fill) => dl == 0 there
            const float *own = buf + D * RG::HCH + ty * RTX + tx;
#pragma unroll
            for (int c = 0; c < D2; ++c) {
                const float a = own[(2 * c) * RG::OCH];
                const float bq = 2 * c + 1 < D ? own[(2 * c + 1) * RG::OCH] : 0.0f;
                R.q[NEW][c] = mul2(f2(a, bq), dup2(kLog2e));
                R.dq[NEW][c] = f2(0.0f, 0.0f);
            }
            // lanes outside the volume: LSE = +inf => W = 0 (no NaN into dB)
            R.L[NEW] = vv ? own[D * RG::OCH] * kLog2e : INFINITY;
            const float gx = own[(D + 1) * RG::OCH], gy = own[(D + 2) * RG::OCH],
                        gz = own[(D + 3) * RG::OCH];
            R.gx[NEW] = gx;
            R.gy[NEW] = gy;
            R.gz[NEW] = gz;
            R.dot[NEW] = gx * own[(D + 4) * RG::OCH] + gy * own[(D + 5) * RG::OCH] +
                         gz * own[(D + 6) * RG::OCH];
            // the column kernel's per-source statistics: {LSE*log2e, gSF.SF}
            if (vv && aux) {
                const int64_t off = (int64_t)(p + 1) * v.hw + (int64_t)y * v.h + x;
                aux[2 * so + off] = R.L[NEW];
                aux[2 * so + v.n + off] = R.dot[NEW];
            }
        } else {
            R.L[NEW] = INFINITY;  // past the chunk end: the slot goes idle
        }
#pragma unroll
        for (int dyi = 0; dyi < 3; ++dyi) {
            float2 kr[D2][3];
#pragma unroll
            for (int c = 0; c < D2; ++c) {
                const float *e0 = buf + (2 * c) * RG::HCH + (ty + dyi) * kBoxX + kXOff + tx;
                const float *e1 = e0 + RG::HCH;
#pragma unroll
                for (int i = 0; i < 3; ++i) kr[c][i] = f2(e0[i], 2 * c + 1 < D ? e1[i] : 0.0f);
            }
            if (dyi == 0) {
                row_slot<D, 0, -1>(R, NEW, db, kr, sB2);
                row_slot<D, 0, 0>(R, MID, db, kr, sB2);
                row_slot<D, 0, 1>(R, OLD, db, kr, sB2);
            } else if (dyi == 1) {
                row_slot<D, 1, -1>(R, NEW, db, kr, sB2);
                row_slot<D, 1, 0>(R, MID, db, kr, sB2);
                row_slot<D, 1, 1>(R, OLD, db, kr, sB2);
            } else {
                row_slot<D, 2, -1>(R, NEW, db, kr, sB2);
                row_slot<D, 2, 0>(R, MID, db, kr, sB2);
                row_slot<D, 2, 1>(R, OLD, db, kr, sB2);
            }
        }
        if (TMA && last_out(&cnt[b]) && p + 2 <= ze)
            row_stage<D, TMA>(smem + b * BUF, maps, &bar[b], p + 2, x0, y0, s, P, v, true);
        if (has_old && vv && gQh) {
            const int64_t off = (int64_t)(p - 1) * v.hw + (int64_t)y * v.h + x;
#pragma unroll
            for (int c = 0; c < D2; ++c) {
                float *d0 = gQh + (int64_t)(2 * c) * v.n + off;
                *d0 = ACC ? *d0 + R.dq[OLD][c].x : R.dq[OLD][c].x;
                if (2 * c + 1 < D) {
                    float *d1 = d0 + v.n;
                    *d1 = ACC ? *d1 + R.dq[OLD][c].y : R.dq[OLD][c].y;
                }
            }
        }
    });
    // dB: warp shuffle reduce, then across warps; one partial per CTA
    if (!TMA) cp_wait_all();
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
// q as key.  Tile 32 x 8, one key voxel per thread (consecutive lanes read
// consecutive smem columns: conflict-free), channels in packed pairs, 3
// in-flight z slots.  Staged source records (set A halo): Q (D ch), LSE,
// gSF (3), SF (3); one transform pass per plane turns LSE into LSE*log2e and
// SF_x into dot = gSF.SF.
constexpr int CTX = 32, CTY = 8;
using CG = Geo<CTX, CTY>;

template <int D>
struct ColSlots {
    static constexpr int D2 = (D + 1) / 2;
    float2 k[3][D2];  // channel pairs of k * log2e (odd D: last .y = 0)
    float2 dk[3][D2];
};

template <int D>
struct SrcStrip {
    static constexpr int D2 = (D + 1) / 2;
    float2 q[D2][3];  // channel pairs of the 3 sources x-1, x, x+1
    float L[3], gx[3], gy[3], gz[3], dt[3];
};

template <int D, int DYI, int DZ>
__device__ __forceinline__ void col_slot(ColSlots<D> &C_, int j, const SrcStrip<D> &S,
                                         const float2 *sB2) {
    constexpr int D2 = (D + 1) / 2;
    constexpr int ob = (DZ + 1) * 9 + DYI * 3;
    // window slot o = (dx,dy,dz) links source r = q - off(o) to key q: the
    // source is strip element si = 1 - dx = 2 - dxi
#pragma unroll
    for (int dxi = 0; dxi < 3; ++dxi) {
        const int si = 2 - dxi;
        float2 acc = f2(sB2[ob + dxi].x, 0.0f);
#pragma unroll
        for (int c = 0; c < D2; ++c) acc = fma2(S.q[c][si], C_.k[j][c], acc);
        // in-volume sources have l <= L; the clamp keeps W finite for the
        // zero-filled out-of-volume records (L = 0), whose cf is exactly 0
        const float W = ex2(fminf(acc.x + acc.y - S.L[si], 126.0f));
        // gSF_r.off(o) - gSF_r.SF_r
        float cf = -S.dt[si];
        if (DYI == 0) cf -= S.gy[si];
        if (DYI == 2) cf += S.gy[si];
        if (DZ < 0) cf -= S.gz[si];
        if (DZ > 0) cf += S.gz[si];
        if (dxi == 0) cf -= S.gx[si];
        if (dxi == 2) cf += S.gx[si];
        const float2 dl2 = dup2(W * cf);
#pragma unroll
        for (int c = 0; c < D2; ++c) C_.dk[j][c] = fma2(dl2, S.q[c][si], C_.dk[j][c]);
    }
}

// staged source records: Q (D ch), aux {LSE*log2e, gSF.SF} (2), gSF (3) as
// halo planes; own: K (D)
template <int D, bool TMA>
__device__ __forceinline__ void col_stage(float *buf, const Maps &m, uint64_t *bar, int p,
                                          int x0, int y0, int s, const Ptrs &P, const Vol &v,
                                          bool issuer) {
    float *own = buf + (D + 5) * CG::HCH;
    if (TMA) {
        if (issuer) {
            mbar_expect_tx(bar, ((D + 5) * CG::PY * kBoxX + D * CG::OCH) * 4);
#pragma unroll
            for (int c = 0; c < D; ++c) {
                tma4(buf + c * CG::HCH, &m.a.q, x0 - 4, y0 - 1, p, s * D + c, bar);
                tma4(own + c * CG::OCH, &m.k, x0, y0, p + 1, s * D + c, bar);
            }
#pragma unroll
            for (int c = 0; c < 2; ++c)
                tma4(buf + (D + c) * CG::HCH, &m.aux, x0 - 4, y0 - 1, p, 2 * s + c, bar);
#pragma unroll
            for (int c = 0; c < 3; ++c)
                tma4(buf + (D + 2 + c) * CG::HCH, &m.a.g, x0 - 4, y0 - 1, p, 3 * s + c, bar);
        }
    } else {
        cp_halo<D + 5, CTX, CTY>(buf, [&](int c) { return P.c_src(c, D, v.n); }, p, x0, y0, v);
        cp_own<D, CTX, CTY>(own, [&](int c) { return P.k(c, v.n); }, p + 1, x0, y0, v);
        cp_commit();
    }
}

template <int D, bool TMA, bool ACC>
__global__ void __launch_bounds__(256, (D <= 6 ? MDG_BWD_COL_MINB : MDG_BWD_MINB8))
modet_bwd_col_k(const __grid_constant__ Maps maps, const float *__restrict__ Q,
                const float *__restrict__ K, const float *__restrict__ B,
                const float *__restrict__ SF, const float *__restrict__ LSE,
                const float *__restrict__ gSF, Vol v, int zc, float *__restrict__ gK,
                const float *__restrict__ aux) {
    constexpr int D2 = (D + 1) / 2;
    constexpr int BUF = (D + 5) * CG::HCH + D * CG::OCH;
    extern __shared__ __align__(128) float smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 2 * BUF);
    float2 *sB2 = reinterpret_cast<float2 *>(smem + 2 * BUF + 8);
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int x0 = blockIdx.x * CTX, y0 = blockIdx.y * CTY;
    const int nzc = (v.l + zc - 1) / zc;
    const int s = blockIdx.z / nzc;
    const int zb = (blockIdx.z - s * nzc) * zc, ze = min(zb + zc, v.l);
    const int64_t so = (int64_t)s * v.n;
    Ptrs P{K + so * D, Q + so * D, LSE + so, gSF + 3 * so, SF + 3 * so};
    P.AUX = aux + 2 * so;
    float *gKh = gK + so * D;
    const int x = x0 + tx, y = y0 + ty;
    const bool vv = x < v.h && y < v.w;
    int *cnt = reinterpret_cast<int *>(smem + 2 * BUF + 8 + 64);
    load_bias2(sB2, B, s);
    if (TMA) init_bars(bar);
    if (threadIdx.x < 2) cnt[threadIdx.x] = 0;
    __syncthreads();
    col_stage<D, TMA>(smem, maps, &bar[0], zb - 1, x0, y0, s, P, v, threadIdx.x == 0);
    if (TMA) col_stage<D, TMA>(smem + BUF, maps, &bar[1], zb, x0, y0, s, P, v, threadIdx.x == 0);
    ColSlots<D> C_;
    march(zb, ze, [&](int p, auto NEW_, auto MID_, auto OLD_) {
        constexpr int NEW = decltype(NEW_)::value, MID = decltype(MID_)::value,
                      OLD = decltype(OLD_)::value;
        const int j = p - zb + 1, b = j & 1;
        if (TMA) {
            mbar_wait(&bar[b], (j >> 1) & 1);
        } else {
            cp_wait_all();
            __syncthreads();
            if (p + 1 <= ze)
                col_stage<D, TMA>(smem + (b ^ 1) * BUF, maps, &bar[b ^ 1], p + 1, x0, y0, s, P,
                                  v, true);
        }
        const float *buf = smem + b * BUF;
        const bool has_new = p + 1 < ze, has_old = p - 1 >= zb;
        if (has_new) {
            const float *own = buf + (D + 5) * CG::HCH + ty * CTX + tx;
#pragma unroll
            for (int c = 0; c < D2; ++c) {
                const float a = own[(2 * c) * CG::OCH];
                const float bk = 2 * c + 1 < D ? own[(2 * c + 1) * CG::OCH] : 0.0f;
                C_.k[NEW][c] = mul2(f2(a, bk), dup2(kLog2e));
                C_.dk[NEW][c] = f2(0.0f, 0.0f);
            }
        }
#pragma unroll
        for (int dyi = 0; dyi < 3; ++dyi) {
            // window row dy = dyi-1 links key row y to source row y - dy
            const float *rowp = buf + (ty + 2 - dyi) * kBoxX + kXOff + tx;
            SrcStrip<D> S;
#pragma unroll
            for (int c = 0; c < D2; ++c) {
                const float *e0 = rowp + (2 * c) * CG::HCH;
                const float *e1 = e0 + CG::HCH;
#pragma unroll
                for (int i = 0; i < 3; ++i) S.q[c][i] = f2(e0[i], 2 * c + 1 < D ? e1[i] : 0.0f);
            }
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                S.L[i] = rowp[D * CG::HCH + i];
                S.dt[i] = rowp[(D + 1) * CG::HCH + i];
                S.gx[i] = rowp[(D + 2) * CG::HCH + i];
                S.gy[i] = rowp[(D + 3) * CG::HCH + i];
                S.gz[i] = rowp[(D + 4) * CG::HCH + i];
            }
            // key z sees sources in plane p at window offset dz = z - p
            if (dyi == 0) {
                col_slot<D, 0, 1>(C_, NEW, S, sB2);
                col_slot<D, 0, 0>(C_, MID, S, sB2);
                col_slot<D, 0, -1>(C_, OLD, S, sB2);
            } else if (dyi == 1) {
                col_slot<D, 1, 1>(C_, NEW, S, sB2);
                col_slot<D, 1, 0>(C_, MID, S, sB2);
                col_slot<D, 1, -1>(C_, OLD, S, sB2);
            } else {
                col_slot<D, 2, 1>(C_, NEW, S, sB2);
                col_slot<D, 2, 0>(C_, MID, S, sB2);
                col_slot<D, 2, -1>(C_, OLD, S, sB2);
            }
        }
        if (TMA && last_out(&cnt[b]) && p + 2 <= ze)
            col_stage<D, TMA>(smem + b * BUF, maps, &bar[b], p + 2, x0, y0, s, P, v, true);
        if (has_old && vv) {
            const int64_t off = (int64_t)(p - 1) * v.hw + (int64_t)y * v.h + x;
#pragma unroll
            for (int c = 0; c < D2; ++c) {
                float *d0 = gKh + (int64_t)(2 * c) * v.n + off;
                *d0 = ACC ? *d0 + C_.dk[OLD][c].x : C_.dk[OLD][c].x;
                if (2 * c + 1 < D) {
                    float *d1 = d0 + v.n;
                    *d1 = ACC ? *d1 + C_.dk[OLD][c].y : C_.dk[OLD][c].y;
                }
            }
        }
    });
}

// ======================================================= bwd: single pass
// modet_bwd_fused_k — the whole backward (dQ, dK, dB) from ONE evaluation of
// each logit.  A CTA owns a 32x8 column tile and marches K planes p through
// its z chunk; source voxels r (the attention rows, attention.hpp:127-166)
// sit in three in-flight slots (planes p+1, p, p-1) and meet the keys of
// plane p.  For every (source, window slot) pair the thread computes
//   W  = exp2(l*log2e - LSE*log2e)         (l = B[o] + Q_r . K_q, q = r + off(o))
//   dl = W * (gSF_r . off(o) - gSF_r . SF_r)   (<W, gW> = gSF . SF)
// and uses it three times: dQ_r += dl K_q (registers, across the three steps
// the source is in flight), dB[o] += dl, and the key's contribution
// dl Q_r.  All keys a step touches lie in plane p, so the three slots'
// contributions to one key sum in registers; the x-neighbour terms move by
// warp shuffle and the y-neighbour terms through a small shared-memory
// exchange (one block barrier per step).  Keys on the tile edge also receive
// terms from sources outside the tile: three extra warps recompute those
// ring sources (the 1-voxel ring of the 34x10 source region; only the 9 of
// 27 window slots whose key falls inside the tile), so every key of the tile
// is complete inside its CTA — no atomics, no cross-CTA pass, a fixed
// summation order (deterministic).  Per voxel: 27 logits (+11 % ring work)
// instead of the two-pass kernels' 54, and no per-source side planes.
//   warps 0-7: tile rows; warp 8: source row y0-1 (keys of row y0, dy=+1);
//   warp 9: source row y0+8 (keys of row y0+7, dy=-1); warp 10: source
//   columns x0-1 (lanes 0-9) and x0+32 (lanes 16-25), rows y0-1 .. y0+8.
constexpr int kFW = 11;               // warps per CTA
constexpr int kFRows = 10;            // box rows: y0-1 .. y0+8
// floats per staged channel: the 40 x 10 box, padded so every channel starts
// on a 128-byte boundary (TMA destination alignment)
constexpr int kFBox = up32(kBoxX * kFRows);

template <int D>
struct FG1 {
    static constexpr int D2 = (D + 1) / 2;
    static constexpr int NOWN = D + 7;                 // Q (D), LSE, gSF (3), SF (3)
    static constexpr int BUF = (D + NOWN) * kFBox;     // K box of plane p + own box of p+1
    static constexpr int YX = 2 * 2 * RTY * RTX * D2;  // float2: [par][dir][pair][row][x]
    static constexpr int XX = 2 * 2 * RTY * 3 * D2;    // float2: [par][side][row][dyi][pair]
};

// one in-flight source slot
template <int D>
struct Src {
    static constexpr int D2 = (D + 1) / 2;
    float2 q[D2];   // Q_r * log2e, channel pairs
    float2 dq[D2];  // dQ_r accumulator
    float Lh;       // LSE * log2e / 2 (+inf: no source)
    float gx, gy, gz, dot;
    float mask;     // 1: counts towards dB (interior source of this chunk)
};

template <int D>
__device__ __forceinline__ void src_load(Src<D> &s, const float *own, int pos, bool valid,
                                         bool interior) {
    constexpr int D2 = (D + 1) / 2;
#pragma unroll
    for (int c = 0; c < D2; ++c) {
        const float a = own[(2 * c) * kFBox + pos];
        const float b = 2 * c + 1 < D ? own[(2 * c + 1) * kFBox + pos] : 0.0f;
        s.q[c] = mul2(f2(a, b), dup2(kLog2e));
        s.dq[c] = f2(0.0f, 0.0f);
    }
    s.Lh = valid ? own[D * kFBox + pos] * (0.5f * kLog2e) : INFINITY;
    s.gx = own[(D + 1) * kFBox + pos];
    s.gy = own[(D + 2) * kFBox + pos];
    s.gz = own[(D + 3) * kFBox + pos];
    s.dot = s.gx * own[(D + 4) * kFBox + pos] + s.gy * own[(D + 5) * kFBox + pos] +
            s.gz * own[(D + 6) * kFBox + pos];
    s.mask = interior ? 1.0f : 0.0f;
}

// dl of source slot s against key k (channel pairs).  The logit in log2
// units minus LSE*log2e is (h + sum_even) + (h + sum_odd) with
// h = (B*log2e - LSE*log2e) / 2 broadcast into both lanes of the packed
// accumulator (no pair set-up per logit); bh = B*log2e / 2.
template <int D>
__device__ __forceinline__ float dl_of(const Src<D> &s, const float2 *k, float bh, float cf) {
    constexpr int D2 = (D + 1) / 2;
    float2 acc = fma2(s.q[0], k[0], dup2(bh - s.Lh));
#pragma unroll
    for (int c = 1; c < D2; ++c) acc = fma2(s.q[c], k[c], acc);
    return ex2(acc.x + acc.y) * cf;
}

// tile row: the three slots against key row dy = DYI-1 of plane p.  Returns
// (in c3) each dx's summed key contribution (in log2e-scaled units); DQ:
// dQ and dB (interior rows only).
template <int D, int DYI, bool DQ>
__device__ __forceinline__ void fused_row(Src<D> (&S)[3], const float *kb, int kpos,
                                          const float *sB, float (&db)[27],
                                          float2 (&c3)[3][(D + 1) / 2]) {
    constexpr int D2 = (D + 1) / 2;
    float2 kr[3][D2];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int c = 0; c < D2; ++c)
            kr[i][c] = f2(kb[(2 * c) * kFBox + kpos + i],
                          2 * c + 1 < D ? kb[(2 * c + 1) * kFBox + kpos + i] : 0.0f);
    // slot 0: NEW (source plane p+1, dz = -1), 1: MID (p, 0), 2: OLD (p-1, +1)
#pragma unroll
    for (int jj = 0; jj < 3; ++jj) {
        Src<D> &s = S[jj];
        const int dz = jj - 1;
        float cb = -s.dot;
        if (dz > 0) cb += s.gz;
        if (dz < 0) cb -= s.gz;
        if (DYI == 0) cb -= s.gy;
        if (DYI == 2) cb += s.gy;
        const int ob = (dz + 1) * 9 + DYI * 3;
        const float cf[3] = {cb - s.gx, cb, cb + s.gx};
#pragma unroll
        for (int dxi = 0; dxi < 3; ++dxi) {
            const float dl = dl_of<D>(s, kr[dxi], sB[ob + dxi], cf[dxi]);
            const float2 dl2 = dup2(dl);
            if (DQ) {
                db[ob + dxi] = fmaf(dl, s.mask, db[ob + dxi]);
#pragma unroll
                for (int c = 0; c < D2; ++c) s.dq[c] = fma2(dl2, kr[dxi][c], s.dq[c]);
            }
#pragma unroll
            for (int c = 0; c < D2; ++c)
                c3[dxi][c] = jj == 0 ? mul2(dl2, s.q[c]) : fma2(dl2, s.q[c], c3[dxi][c]);
        }
    }
}

// keys of one row: lane x collects dx = 0 from itself, dx = +1 from lane x-1
// and dx = -1 from lane x+1 (in that order)
template <int D>
__device__ __forceinline__ void xcombine(float2 (&c3)[3][(D + 1) / 2], float2 *R) {
    constexpr int D2 = (D + 1) / 2;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int c = 0; c < D2; ++c) {
        float2 up, dn;
        up.x = __shfl_up_sync(0xffffffffu, c3[2][c].x, 1);
        up.y = __shfl_up_sync(0xffffffffu, c3[2][c].y, 1);
        dn.x = __shfl_down_sync(0xffffffffu, c3[0][c].x, 1);
        dn.y = __shfl_down_sync(0xffffffffu, c3[0][c].y, 1);
        if (lane == 0) up = f2(0.0f, 0.0f);
        if (lane == 31) dn = f2(0.0f, 0.0f);
        R[c] = add2(add2(c3[1][c], up), dn);
    }
}

template <int D>
__device__ __forceinline__ void fused_stage(float *buf, const Maps &m, uint64_t *bar, int p,
                                            int x0, int y0, int s) {
    float *own = buf + D * kFBox;
    mbar_expect_tx(bar, (2 * D + 7) * kBoxX * kFRows * 4);
#pragma unroll
    for (int c = 0; c < D; ++c) {
        tma4(buf + c * kFBox, &m.k, x0 - 4, y0 - 1, p, s * D + c, bar);
        tma4(own + c * kFBox, &m.a.q, x0 - 4, y0 - 1, p + 1, s * D + c, bar);
    }
    tma4(own + D * kFBox, &m.a.lse, x0 - 4, y0 - 1, p + 1, s, bar);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        tma4(own + (D + 1 + c) * kFBox, &m.a.g, x0 - 4, y0 - 1, p + 1, 3 * s + c, bar);
        tma4(own + (D + 4 + c) * kFBox, &m.a.sf, x0 - 4, y0 - 1, p + 1, 3 * s + c, bar);
    }
}

template <int D, bool ACC>
__global__ void __launch_bounds__(kFW * 32, 1)
modet_bwd_fused_k(const __grid_constant__ Maps maps, const float *__restrict__ B, Vol v, int zc,
                  float *__restrict__ gQ, float *__restrict__ gK, float *__restrict__ gBpart) {
    using G = FG1<D>;
    constexpr int D2 = G::D2;
    extern __shared__ __align__(128) float smem[];
    float2 *ybuf = reinterpret_cast<float2 *>(smem + 2 * G::BUF);
    float2 *xbuf = ybuf + G::YX;
    float *sB = reinterpret_cast<float *>(xbuf + G::XX);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sB + 32);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int x0 = blockIdx.x * RTX, y0 = blockIdx.y * RTY;
    const int nzc = (v.l + zc - 1) / zc;
    const int s = blockIdx.z / nzc;
    const int zb = (blockIdx.z - s * nzc) * zc, ze = min(zb + zc, v.l);
    const int64_t so = (int64_t)s * v.n;
    if (threadIdx.x < 27) sB[threadIdx.x] = B[s * 27 + threadIdx.x] * (0.5f * kLog2e);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        fused_stage<D>(smem, maps, &bar[0], zb - 2, x0, y0, s);
        fused_stage<D>(smem + G::BUF, maps, &bar[1], zb - 1, x0, y0, s);
    }
    // this thread's source position (box row br in 0..9, box column bc)
    int br, bc;
    bool xside_right = false, active = true;
    if (wid < 8) {
        br = wid + 1;
        bc = lane + 4;
    } else if (wid < 10) {
        br = wid == 8 ? 0 : 9;
        bc = lane + 4;
    } else {
        xside_right = lane >= 16;
        br = lane & 15;
        bc = xside_right ? 36 : 3;
        active = br < kFRows;
        if (!active) br = 0;
    }
    const int sx = x0 - 4 + bc, sy = y0 - 1 + br;
    const bool in_xy = active && sx >= 0 && sx < v.h && sy >= 0 && sy < v.w;
    const int pos = br * kBoxX + bc;
    Src<D> S[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
#pragma unroll
        for (int c = 0; c < D2; ++c) S[j].q[c] = S[j].dq[c] = f2(0.0f, 0.0f);
        S[j].Lh = INFINITY;
        S[j].gx = S[j].gy = S[j].gz = S[j].dot = S[j].mask = 0.0f;
    }
    float db[27];
#pragma unroll
    for (int o = 0; o < 27; ++o) db[o] = 0.0f;
    float *gQh = gQ ? gQ + so * D : nullptr;
    float *gKh = gK ? gK + so * D : nullptr;
    // slots: S[0] = source plane p+1 (NEW), S[1] = p (MID), S[2] = p-1 (OLD);
    // rotated by register moves at the end of each step (one copy of the
    // step body: the unrolled three-step rotation overflowed the i-cache)
    for (int p = zb - 2; p <= ze; ++p) {
        constexpr int NEW = 0, OLD = 2;
        const int j = p - (zb - 2), b = j & 1, par = j & 1;
        mbar_wait(&bar[b], (j >> 1) & 1);
        const float *buf = smem + b * G::BUF;
        {   // the source entering the window: plane p+1 (the chunk's ring planes
            // zb-1 and ze feed keys only; beyond them the slot idles)
            const int z = p + 1;
            const bool valid = in_xy && z >= 0 && z >= zb - 1 && z <= ze && z < v.l;
            src_load<D>(S[NEW], buf + D * kFBox, pos, valid,
                        valid && wid < 8 && z >= zb && z < ze);
        }
        float2 own[D2];
        if (p >= zb - 1) {
            float2 c3[3][D2];
            if (wid < 8) {
                float2 R[D2];
                // key rows dy = -1, 0, +1 (box rows wid, wid+1, wid+2)
                fused_row<D, 0, true>(S, buf, wid * kBoxX + lane + 3, sB, db, c3);
                xcombine<D>(c3, R);
                if (wid >= 1)
#pragma unroll
                    for (int c = 0; c < D2; ++c)
                        ybuf[(((par * 2 + 1) * D2 + c) * RTY + wid - 1) * RTX + lane] = R[c];
                fused_row<D, 1, true>(S, buf, (wid + 1) * kBoxX + lane + 3, sB, db, c3);
                xcombine<D>(c3, own);
                fused_row<D, 2, true>(S, buf, (wid + 2) * kBoxX + lane + 3, sB, db, c3);
                xcombine<D>(c3, R);
                if (wid <= 6)
#pragma unroll
                    for (int c = 0; c < D2; ++c)
                        ybuf[(((par * 2 + 0) * D2 + c) * RTY + wid + 1) * RTX + lane] = R[c];
            } else if (wid == 8) {  // source row y0-1 -> keys of row y0 (dy = +1)
                float2 R[D2];
                fused_row<D, 2, false>(S, buf, 1 * kBoxX + lane + 3, sB, db, c3);
                xcombine<D>(c3, R);
#pragma unroll
                for (int c = 0; c < D2; ++c)
                    ybuf[(((par * 2 + 0) * D2 + c) * RTY + 0) * RTX + lane] = R[c];
            } else if (wid == 9) {  // source row y0+8 -> keys of row y0+7 (dy = -1)
                float2 R[D2];
                fused_row<D, 0, false>(S, buf, 8 * kBoxX + lane + 3, sB, db, c3);
                xcombine<D>(c3, R);
#pragma unroll
                for (int c = 0; c < D2; ++c)
                    ybuf[(((par * 2 + 1) * D2 + c) * RTY + RTY - 1) * RTX + lane] = R[c];
            } else {  // x ring: dx = +1 (left column) / -1 (right), dy = -1, 0, +1
                const int dxi = xside_right ? 0 : 2;
                const int kc = xside_right ? 35 : 4;
#pragma unroll
                for (int dyi = 0; dyi < 3; ++dyi) {
                    const int kr_ = br + dyi - 1;  // key box row
                    float2 k[D2], acc[D2];
                    const int kp = (kr_ < 0 ? 0 : (kr_ > 9 ? 9 : kr_)) * kBoxX + kc;
#pragma unroll
                    for (int c = 0; c < D2; ++c) {
                        k[c] = f2(buf[(2 * c) * kFBox + kp],
                                  2 * c + 1 < D ? buf[(2 * c + 1) * kFBox + kp] : 0.0f);
                        acc[c] = f2(0.0f, 0.0f);
                    }
#pragma unroll
                    for (int jj = 0; jj < 3; ++jj) {
                        const Src<D> &sr = S[jj];
                        const int dz = jj - 1;
                        const float cf = -sr.dot + (dyi == 0 ? -sr.gy : (dyi == 2 ? sr.gy : 0.0f)) +
                                   (dz > 0 ? sr.gz : (dz < 0 ? -sr.gz : 0.0f)) +
                                   (xside_right ? -sr.gx : sr.gx);
                        const float dl =
                            dl_of<D>(sr, k, sB[(dz + 1) * 9 + dyi * 3 + dxi], cf);
                        const float2 dl2 = dup2(dl);
#pragma unroll
                        for (int c = 0; c < D2; ++c) acc[c] = fma2(dl2, sr.q[c], acc[c]);
                    }
                    // key row (tile-relative) = box row - 1
                    if (active && kr_ >= 1 && kr_ <= RTY)
#pragma unroll
                        for (int c = 0; c < D2; ++c)
                            xbuf[(((par * 2 + (xside_right ? 1 : 0)) * RTY + kr_ - 1) * 3 + dyi) *
                                     D2 + c] = acc[c];
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && p + 2 <= ze) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            fused_stage<D>(smem + b * G::BUF, maps, &bar[b], p + 2, x0, y0, s);
        }
        if (wid < 8) {
            const int x = x0 + lane, y = y0 + wid;
            const bool vv = x < v.h && y < v.w;
            // keys of plane p: ((from row above + own row) + from row below) + x ring
            if (p >= zb && p < ze && vv && gKh) {
                const int64_t off = (int64_t)p * v.hw + (int64_t)y * v.h + x;
#pragma unroll
                for (int c = 0; c < D2; ++c) {
                    float2 t = add2(ybuf[(((par * 2 + 0) * D2 + c) * RTY + wid) * RTX + lane],
                                    own[c]);
                    t = add2(t, ybuf[(((par * 2 + 1) * D2 + c) * RTY + wid) * RTX + lane]);
                    if (lane == 0 || lane == 31) {
                        const int sd = lane == 31 ? 1 : 0;
#pragma unroll
                        for (int dyi = 0; dyi < 3; ++dyi)
                            t = add2(t, xbuf[(((par * 2 + sd) * RTY + wid) * 3 + dyi) * D2 + c]);
                    }
                    t = mul2(t, dup2(kLn2));  // contributions carry Q * log2e
                    float *d0 = gKh + (int64_t)(2 * c) * v.n + off;
                    *d0 = ACC ? *d0 + t.x : t.x;
                    if (2 * c + 1 < D) {
                        float *d1 = d0 + v.n;
                        *d1 = ACC ? *d1 + t.y : t.y;
                    }
                }
            }
            // the source leaving the window (plane p-1) has all 27 terms of dQ
            if (p - 1 >= zb && p - 1 < ze && vv && gQh) {
                const int64_t off = (int64_t)(p - 1) * v.hw + (int64_t)y * v.h + x;
#pragma unroll
                for (int c = 0; c < D2; ++c) {
                    float *d0 = gQh + (int64_t)(2 * c) * v.n + off;
                    *d0 = ACC ? *d0 + S[OLD].dq[c].x : S[OLD].dq[c].x;
                    if (2 * c + 1 < D) {
                        float *d1 = d0 + v.n;
                        *d1 = ACC ? *d1 + S[OLD].dq[c].y : S[OLD].dq[c].y;
                    }
                }
            }
        }
        S[2] = S[1];
        S[1] = S[0];
    }
    // dB: per-CTA partial over the 8 tile warps (fixed order)
    __syncthreads();
    float *red = smem;
    if (wid < 8) {
#pragma unroll
        for (int o = 0; o < 27; ++o) {
            float a = db[o];
#pragma unroll
            for (int m = 16; m > 0; m >>= 1) a += __shfl_xor_sync(0xffffffffu, a, m);
            if (lane == 0) red[wid * 27 + o] = a;
        }
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

// ------------------------------------------- bwd: single pass, 2 CTAs / SM
// modet_bwd_fused2_k — the single-pass backward of modet_bwd_fused_k with
// the source ring folded into the 8 tile warps as uniform extra work, so the
// kernel fits two CTAs per SM (<= 128 registers, ~110 KB shared):
//   * each step the 84 ring sources' records (Q*log2e, LSE, gSF, gSF.SF) of
//     the entering plane go to a 3-plane shared ring buffer;
//   * the 236 (ring source, tile key) pairs — top / bottom rows (dy = +-1,
//     dx = -1..1) and left / right columns (dx = +-1, dy = -1..1) — are one
//     per thread: 3 logits (the three in-flight planes), their summed key
//     contribution into a per-pair slot;
//   * a key adds, in a fixed order: the row above (y exchange), its own row
//     (x shuffles), the row below, then its ring pairs.
// Interior work runs one window column (dx) at a time: K strip, three slots,
// then the x-shuffle of that column's key contribution (6 + 6 live floats
// instead of 18 + 18).  Two block barriers per step; the exchange buffers are
// double-buffered by step parity.  Deterministic (no atomics).
constexpr int kNPair = 236, kNRing = 84;

template <int D>
struct FG2 {
    static constexpr int D2 = (D + 1) / 2;
    static constexpr int BUF = (2 * D + 7) * kFBox;          // K box (p) + own box (p+1)
    static constexpr int YX = 2 * 2 * D2 * RTY * RTX;        // float2 [par][dir][pair][row][x]
    static constexpr int RC = 2 * kNPair * D2;               // float2 [par][pair][c]
    static constexpr int RR = 3 * kNRing * 12;               // float  [slot][ring][12]
    static constexpr size_t SMEM = ((size_t)2 * BUF + 2 * YX + 2 * RC + RR + 32) * 4 + 16;
};

// box position (row, column) of ring source r
__device__ __forceinline__ void ring_pos(int r, int &br, int &bc) {
    if (r < 32) {
        br = 0;
        bc = r + 4;
    } else if (r < 64) {
        br = 9;
        bc = r - 32 + 4;
    } else if (r < 74) {
        br = r - 64;
        bc = 3;
    } else {
        br = r - 74;
        bc = 36;
    }
}

// pair t -> (ring source r, key lane kx, key row ky, dx, dy)
__device__ __forceinline__ bool pair_of(int t, int &r, int &kx, int &ky, int &dx, int &dy) {
    if (t < 188) {  // top (t < 94) / bottom rows, key-major, dx = -1, 0, +1
        const bool bot = t >= 94;
        const int u = bot ? t - 94 : t;
        if (u < 2) {
            kx = 0;
            dx = u - 1;
        } else if (u < 92) {
            kx = 1 + (u - 2) / 3;
            dx = (u - 2) % 3 - 1;
        } else {
            kx = 31;
            dx = u - 92;
        }
        ky = bot ? RTY - 1 : 0;
        dy = bot ? -1 : 1;
        r = (bot ? 32 : 0) + kx - dx;
        return true;
    }
    if (t < kNPair) {  // left (t < 212) / right columns, key-major, dy = -1, 0, +1
        const bool right = t >= 212;
        const int u = right ? t - 212 : t - 188;
        ky = u / 3;
        dy = u % 3 - 1;
        kx = right ? 31 : 0;
        dx = right ? -1 : 1;
        r = (right ? 74 : 64) + (ky - dy) + 1;  // source row ky - dy, box row + 1
        return true;
    }
    return false;
}

template <int D, bool ACC>
__global__ void __launch_bounds__(256, 2)
modet_bwd_fused2_k(const __grid_constant__ Maps maps, const float *__restrict__ B, Vol v, int zc,
                   float *__restrict__ gQ, float *__restrict__ gK, float *__restrict__ gBpart) {
    using G = FG2<D>;
    constexpr int D2 = G::D2;
    extern __shared__ __align__(128) float smem[];
    float2 *ybuf = reinterpret_cast<float2 *>(smem + 2 * G::BUF);
    float2 *rcon = ybuf + G::YX;
    float *rrec = reinterpret_cast<float *>(rcon + G::RC);
    float *sB = rrec + G::RR;
    uint64_t *bar = reinterpret_cast<uint64_t *>(sB + 32);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int x0 = blockIdx.x * RTX, y0 = blockIdx.y * RTY;
    const int nzc = (v.l + zc - 1) / zc;
    const int s = blockIdx.z / nzc;
    const int zb = (blockIdx.z - s * nzc) * zc, ze = min(zb + zc, v.l);
    const int64_t so = (int64_t)s * v.n;
    if (threadIdx.x < 27) sB[threadIdx.x] = B[s * 27 + threadIdx.x] * (0.5f * kLog2e);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        fused_stage<D>(smem, maps, &bar[0], zb - 2, x0, y0, s);
        fused_stage<D>(smem + G::BUF, maps, &bar[1], zb - 1, x0, y0, s);
    }
    const int x = x0 + lane, y = y0 + wid;
    const bool in_xy = x < v.h && y < v.w;
    const int pos = (wid + 1) * kBoxX + lane + 4;  // own box position of this column
    // this thread's ring pair (t < 236) and the ring source it records (t < 84)
    int pr = 0, pkx = 0, pky = 0, pdx = 0, pdy = 0;
    const bool has_pair = pair_of(threadIdx.x, pr, pkx, pky, pdx, pdy);
    int rbr = 0, rbc = 0;
    if (threadIdx.x < kNRing) ring_pos(threadIdx.x, rbr, rbc);
    const int rsx = x0 - 4 + rbc, rsy = y0 - 1 + rbr;
    const bool rin = threadIdx.x < kNRing && rsx >= 0 && rsx < v.h && rsy >= 0 && rsy < v.w;
    Src<D> S[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
#pragma unroll
        for (int c = 0; c < D2; ++c) S[j].q[c] = S[j].dq[c] = f2(0.0f, 0.0f);
        S[j].Lh = INFINITY;
        S[j].gx = S[j].gy = S[j].gz = S[j].dot = S[j].mask = 0.0f;
    }
    float db[27];
#pragma unroll
    for (int o = 0; o < 27; ++o) db[o] = 0.0f;
    float *gQh = gQ ? gQ + so * D : nullptr;
    float *gKh = gK ? gK + so * D : nullptr;
    for (int p = zb - 2; p <= ze; ++p) {
        const int j = p - (zb - 2), b = j & 1, par = j & 1;
        mbar_wait(&bar[b], (j >> 1) & 1);
        const float *buf = smem + b * G::BUF;
        const float *own = buf + D * kFBox;
        const int z = p + 1;  // plane entering the window
        const bool zok = z >= 0 && z >= zb - 1 && z <= ze && z < v.l;
        src_load<D>(S[0], own, pos, in_xy && zok, in_xy && zok && z >= zb && z < ze);
        // ring record slot of plane q: (q - zb + 3) mod 3
        if (threadIdx.x < kNRing) {
            float *rec = rrec + ((z - zb + 3) % 3) * kNRing * 12 + threadIdx.x * 12;
            const int bp = rbr * kBoxX + rbc;
#pragma unroll
            for (int c = 0; c < D; ++c) rec[c] = own[c * kFBox + bp] * kLog2e;
            const float gx = own[(D + 1) * kFBox + bp], gy = own[(D + 2) * kFBox + bp],
                        gz = own[(D + 3) * kFBox + bp];
            rec[D] = rin && zok ? own[D * kFBox + bp] * (0.5f * kLog2e) : INFINITY;
            rec[D + 1] = gx;
            rec[D + 2] = gy;
            rec[D + 3] = gz;
            rec[D + 4] = gx * own[(D + 4) * kFBox + bp] + gy * own[(D + 5) * kFBox + bp] +
                         gz * own[(D + 6) * kFBox + bp];
        }
        const bool work = p >= zb - 1;
        float2 ownk[D2];
        if (work) {
#pragma unroll
            for (int dyi = 0; dyi < 3; ++dyi) {
                float2 R[D2];
#pragma unroll
                for (int c = 0; c < D2; ++c) R[c] = f2(0.0f, 0.0f);
                const int kpos = (wid + dyi) * kBoxX + lane + 3;
#pragma unroll
                for (int dxi = 0; dxi < 3; ++dxi) {
                    float2 kr[D2], cc[D2];
#pragma unroll
                    for (int c = 0; c < D2; ++c)
                        kr[c] = f2(buf[(2 * c) * kFBox + kpos + dxi],
                                   2 * c + 1 < D ? buf[(2 * c + 1) * kFBox + kpos + dxi] : 0.0f);
#pragma unroll
                    for (int jj = 0; jj < 3; ++jj) {
                        Src<D> &sr = S[jj];
                        const int dz = jj - 1;
                        float cf = -sr.dot;
                        if (dz > 0) cf += sr.gz;
                        if (dz < 0) cf -= sr.gz;
                        if (dyi == 0) cf -= sr.gy;
                        if (dyi == 2) cf += sr.gy;
                        if (dxi == 0) cf -= sr.gx;
                        if (dxi == 2) cf += sr.gx;
                        const int o = (dz + 1) * 9 + dyi * 3 + dxi;
                        const float dl = dl_of<D>(sr, kr, sB[o], cf);
                        const float2 dl2 = dup2(dl);
                        db[o] = fmaf(dl, sr.mask, db[o]);
#pragma unroll
                        for (int c = 0; c < D2; ++c) {
                            sr.dq[c] = fma2(dl2, kr[c], sr.dq[c]);
                            cc[c] = jj == 0 ? mul2(dl2, sr.q[c]) : fma2(dl2, sr.q[c], cc[c]);
                        }
                    }
                    // the column's key contribution: dx = -1 goes to lane-1,
                    // dx = +1 to lane+1 (fixed order: dx = -1, 0, +1)
#pragma unroll
                    for (int c = 0; c < D2; ++c) {
                        float2 t = cc[c];
                        if (dxi == 0) {
                            t.x = __shfl_down_sync(0xffffffffu, t.x, 1);
                            t.y = __shfl_down_sync(0xffffffffu, t.y, 1);
                            if (lane == 31) t = f2(0.0f, 0.0f);
                        } else if (dxi == 2) {
                            t.x = __shfl_up_sync(0xffffffffu, t.x, 1);
                            t.y = __shfl_up_sync(0xffffffffu, t.y, 1);
                            if (lane == 0) t = f2(0.0f, 0.0f);
                        }
                        R[c] = add2(R[c], t);
                    }
                }
                if (dyi == 1) {
#pragma unroll
                    for (int c = 0; c < D2; ++c) ownk[c] = R[c];
                } else if (dyi == 0 && wid >= 1) {  // keys of row wid-1, from below
#pragma unroll
                    for (int c = 0; c < D2; ++c)
                        ybuf[(((par * 2 + 1) * D2 + c) * RTY + wid - 1) * RTX + lane] = R[c];
                } else if (dyi == 2 && wid <= RTY - 2) {  // keys of row wid+1, from above
#pragma unroll
                    for (int c = 0; c < D2; ++c)
                        ybuf[(((par * 2 + 0) * D2 + c) * RTY + wid + 1) * RTX + lane] = R[c];
                }
            }
        }
        __syncthreads();  // (A) y exchange and the entering plane's ring records
        if (work && has_pair) {
            // the pair's three logits (the in-flight planes p+1, p, p-1)
            const int kp = (pky + 1) * kBoxX + pkx + 4;
            float2 k[D2];
#pragma unroll
            for (int c = 0; c < D2; ++c)
                k[c] = f2(buf[(2 * c) * kFBox + kp], 2 * c + 1 < D ? buf[(2 * c + 1) * kFBox + kp] : 0.0f);
            float2 acc[D2];
#pragma unroll
            for (int jj = 0; jj < 3; ++jj) {
                const int zz = p + 1 - jj, dz = jj - 1;
                const float *rec = rrec + ((zz - zb + 3) % 3) * kNRing * 12 + pr * 12;
                Src<D> sr;
#pragma unroll
                for (int c = 0; c < D2; ++c)
                    sr.q[c] = f2(rec[2 * c], 2 * c + 1 < D ? rec[2 * c + 1] : 0.0f);
                sr.Lh = rec[D];
                const float cf = -rec[D + 4] + (float)pdx * rec[D + 1] + (float)pdy * rec[D + 2] +
                                 (float)dz * rec[D + 3];
                const int o = (dz + 1) * 9 + (pdy + 1) * 3 + (pdx + 1);
                const float dl = dl_of<D>(sr, k, sB[o], cf);
                const float2 dl2 = dup2(dl);
#pragma unroll
                for (int c = 0; c < D2; ++c)
                    acc[c] = jj == 0 ? mul2(dl2, sr.q[c]) : fma2(dl2, sr.q[c], acc[c]);
            }
#pragma unroll
            for (int c = 0; c < D2; ++c) rcon[(par * kNPair + threadIdx.x) * D2 + c] = acc[c];
        }
        __syncthreads();  // (B) ring contributions; the stage buffer is free
        if (threadIdx.x == 0 && p + 2 <= ze) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            fused_stage<D>(smem + b * G::BUF, maps, &bar[b], p + 2, x0, y0, s);
        }
        if (in_xy && p >= zb && p < ze && gKh) {
            const int64_t off = (int64_t)p * v.hw + (int64_t)y * v.h + x;
            // ring pair ids feeding this key (key-major enumeration of pair_of)
            const int tb = lane == 0 ? 0 : (lane == 31 ? 92 : 2 + 3 * (lane - 1));
            const int tn = (lane == 0 || lane == 31) ? 2 : 3;
#pragma unroll
            for (int c = 0; c < D2; ++c) {
                float2 t = ownk[c];
                if (wid >= 1) t = add2(ybuf[(((par * 2 + 0) * D2 + c) * RTY + wid) * RTX + lane], t);
                if (wid <= RTY - 2) t = add2(t, ybuf[(((par * 2 + 1) * D2 + c) * RTY + wid) * RTX + lane]);
                if (wid == 0)
                    for (int i = 0; i < tn; ++i) t = add2(t, rcon[(par * kNPair + tb + i) * D2 + c]);
                if (wid == RTY - 1)
                    for (int i = 0; i < tn; ++i) t = add2(t, rcon[(par * kNPair + 94 + tb + i) * D2 + c]);
                if (lane == 0)
#pragma unroll
                    for (int i = 0; i < 3; ++i) t = add2(t, rcon[(par * kNPair + 188 + 3 * wid + i) * D2 + c]);
                if (lane == 31)
#pragma unroll
                    for (int i = 0; i < 3; ++i) t = add2(t, rcon[(par * kNPair + 212 + 3 * wid + i) * D2 + c]);
                t = mul2(t, dup2(kLn2));  // contributions carry Q * log2e
                float *d0 = gKh + (int64_t)(2 * c) * v.n + off;
                *d0 = ACC ? *d0 + t.x : t.x;
                if (2 * c + 1 < D) {
                    float *d1 = d0 + v.n;
                    *d1 = ACC ? *d1 + t.y : t.y;
                }
            }
        }
        if (in_xy && p - 1 >= zb && p - 1 < ze && gQh) {
            const int64_t off = (int64_t)(p - 1) * v.hw + (int64_t)y * v.h + x;
#pragma unroll
            for (int c = 0; c < D2; ++c) {
                float *d0 = gQh + (int64_t)(2 * c) * v.n + off;
                *d0 = ACC ? *d0 + S[2].dq[c].x : S[2].dq[c].x;
                if (2 * c + 1 < D) {
                    float *d1 = d0 + v.n;
                    *d1 = ACC ? *d1 + S[2].dq[c].y : S[2].dq[c].y;
                }
            }
        }
        S[2] = S[1];
        S[1] = S[0];
    }
    // dB: per-CTA partial (fixed order)
    __syncthreads();
    float *red = smem;
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
        for (int i = 0; i < RTY; ++i) a += red[i * 27 + threadIdx.x];
        const int cta = (blockIdx.z - s * nzc) * gridDim.x * gridDim.y + blockIdx.y * gridDim.x +
                        blockIdx.x;
        const int ncta = nzc * gridDim.x * gridDim.y;
        gBpart[((int64_t)s * ncta + cta) * 27 + threadIdx.x] = a;
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

// ------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// TMA usable: row pitch a multiple of 16 B, bases 16-B aligned, encoder found
static bool tma_ok(const Vol &v, std::initializer_list<const void *> ptrs) {
    if (v.h % 4 != 0 || !encoder()) return false;
    for (const void *p : ptrs)
        if (p && reinterpret_cast<uintptr_t>(p) % 16 != 0) return false;
    return true;
}

// 4-D map over planar {nch, l, w, h} with a single-channel box {bx, by, 1, 1}
static bool make_map(CUtensorMap *m, const float *base, const Vol &v, int nch, int bx, int by) {
    const cuuint64_t dims[4] = {(cuuint64_t)v.h, (cuuint64_t)v.w, (cuuint64_t)v.l, (cuuint64_t)nch};
    const cuuint64_t strides[3] = {(cuuint64_t)v.h * 4, (cuuint64_t)v.hw * 4, (cuuint64_t)v.n * 4};
    const cuuint32_t box[4] = {(cuuint32_t)bx, (cuuint32_t)by, 1, 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    return encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(base), dims,
                     strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// set-A maps with box (bx, by)
static bool make_maps_a(MapsA *m, const float *Q, const float *LSE, const float *gSF,
                        const float *SF, const Vol &v, int S, int D, int bx, int by) {
    return make_map(&m->q, Q, v, S * D, bx, by) && make_map(&m->lse, LSE, v, S, bx, by) &&
           make_map(&m->g, gSF, v, 3 * S, bx, by) && make_map(&m->sf, SF, v, 3 * S, bx, by);
}

static int pick_zc(int tiles, int l, int per_sm, int waves) {
    // about `waves` x (per_sm resident per SM on 148 SMs) CTAs, chunks of
    // >= 8 planes.  Measured at 160x192x224 (S = 1): forward best at 3,
    // backward at 5 (shorter chunks balance the last wave; 2 was 4-8 %
    // slower, 8+ pays too many chunk prologues)
    const int want = 148 * per_sm * waves;
    int nzc = (want + tiles - 1) / max(tiles, 1);
    nzc = max(1, min(nzc, (l + 7) / 8));
    return (l + nzc - 1) / nzc;
}

template <class KFn>
static void set_smem(KFn k, size_t sm) {
    if (sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
}

// shared memory: two buffers + 2 mbarriers (8 floats) + 27 bias pairs (64)
// + 2 buffer-release counters
constexpr size_t kTail = 8 + 64 + 8;

template <int D>
static cudaError_t fwd_launch(const float *Q, const float *K, const float *B, mdg_dims3 d, int S,
                              float *SF, float *LSE, unsigned long long *flag, cudaStream_t st) {
    const Vol v{d.h, d.w, d.l, (int64_t)d.h * d.w * d.l, (int64_t)d.h * d.w};
    const int gx = (d.h + FTX - 1) / FTX, gy = (d.w + FTY - 1) / FTY;
    const int zc = pick_zc(gx * gy * S, d.l, D <= 6 ? 3 : 2, 3);
    const int nzc = (d.l + zc - 1) / zc;
    const size_t sm = (2 * D * (FG::HCH + FG::OCH) + kTail) * sizeof(float);
    Maps m{};
    const bool tma = tma_ok(v, {Q, K}) && make_map(&m.k, K, v, S * D, kBoxX, FG::PY) &&
                     make_map(&m.a.q, Q, v, S * D, FTX, FTY);
    const dim3 grid(gx, gy, S * nzc);
    unsigned long long *fixq = fixup_queue_ptr(st);
    if (!fixq) return cudaErrorMemoryAllocation;
    cudaError_t e = cudaMemsetAsync(fixq, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    if (tma) {
        set_smem(modet_fwd_tiled_k<D, true>, sm);
        modet_fwd_tiled_k<D, true><<<grid, 256, sm, st>>>(m, Q, K, B, v, zc, SF, LSE, fixq);
    } else {
        set_smem(modet_fwd_tiled_k<D, false>, sm);
        modet_fwd_tiled_k<D, false><<<grid, 256, sm, st>>>(m, Q, K, B, v, zc, SF, LSE, fixq);
    }
    modet_fwd_fixup_k<D><<<148, 256, 0, st>>>(Q, K, B, v, S, SF, LSE, fixq, flag);
    g_launches.fetch_add(1);
    return cudaPeekAtLastError();
}

template <int D, bool TMA, bool ACC>
static void row_launch(dim3 g, size_t sm, cudaStream_t st, const Maps &m, const float *Q,
                       const float *K, const float *B, const float *SF, const float *LSE,
                       const float *gSF, const Vol &v, int zc, float *gQ, float *part,
                       float *aux) {
    set_smem(modet_bwd_row_k<D, TMA, ACC>, sm);
    modet_bwd_row_k<D, TMA, ACC><<<g, 256, sm, st>>>(m, Q, K, B, SF, LSE, gSF, v, zc, gQ, part,
                                                     aux);
}

template <int D, bool TMA, bool ACC>
static void col_launch(dim3 g, size_t sm, cudaStream_t st, const Maps &m, const float *Q,
                       const float *K, const float *B, const float *SF, const float *LSE,
                       const float *gSF, const Vol &v, int zc, float *gK, const float *aux) {
    set_smem(modet_bwd_col_k<D, TMA, ACC>, sm);
    modet_bwd_col_k<D, TMA, ACC><<<g, 256, sm, st>>>(m, Q, K, B, SF, LSE, gSF, v, zc, gK, aux);
}

// which backward: MDG_MODET_BWD = "two" (row + column kernels, the default:
// fastest measured), "fused1" (single pass, ring warps) or "fused2" (single
// pass, ring folded into the tile warps, 2 CTAs / SM).  At 160x192x224, S=1,
// d=6 (r02): two 0.456 ms, fused1 0.48-0.51, fused2 0.56.
static int bwd_variant() {
    static const int v = [] {
        const char *e = std::getenv("MDG_MODET_BWD");
        if (!e) return 0;
        if (!std::strcmp(e, "two")) return 0;
        if (!std::strcmp(e, "fused1")) return 1;
        if (!std::strcmp(e, "fused2")) return 2;
        return 0;
    }();
    return v;
}

template <int D, bool ACC>
static void fused_launch(dim3 g, size_t sm, cudaStream_t st, const Maps &m, const float *B,
                         const Vol &v, int zc, float *gQ, float *gK, float *part) {
    set_smem(modet_bwd_fused_k<D, ACC>, sm);
    modet_bwd_fused_k<D, ACC><<<g, kFW * 32, sm, st>>>(m, B, v, zc, gQ, gK, part);
}

// the single-pass kernel (TMA staging, head_dim <= 6: its register budget)
template <int D>
static bool bwd_fused(const float *Q, const float *K, const float *B, const float *SF,
                      const float *LSE, const float *gSF, const Vol &v, int S, bool acc,
                      float *gQ, float *gK, float *gB, cudaStream_t st, cudaError_t *err) {
    if constexpr (D > 6) {
        return false;
    } else {
        if (bwd_variant() != 1) return false;
        Maps m{};
        if (!(make_map(&m.k, K, v, S * D, kBoxX, kFRows) &&
              make_maps_a(&m.a, Q, LSE, gSF, SF, v, S, D, kBoxX, kFRows)))
            return false;
        const int gx = (v.h + RTX - 1) / RTX, gy = (v.w + RTY - 1) / RTY;
        const int zc = pick_zc(gx * gy * S, v.l, 1, 4);
        const int nzc = (v.l + zc - 1) / zc;
        const int ncta = gx * gy * nzc;
        using G = FG1<D>;
        const size_t sm = (2 * G::BUF + 2 * (G::YX + G::XX) + 32 + 8) * sizeof(float);
        float *part = nullptr;
        keep_pool_mapped();
        if ((*err = cudaMallocAsync(&part, (size_t)S * ncta * 27 * sizeof(float), st))) return true;
        const dim3 g(gx, gy, S * nzc);
        if (acc) fused_launch<D, true>(g, sm, st, m, B, v, zc, gQ, gK, part);
        else fused_launch<D, false>(g, sm, st, m, B, v, zc, gQ, gK, part);
        g_launches.fetch_add(1);
        if (gB) {
            reduce_db_k<<<dim3(27, S), 256, 0, st>>>(part, ncta, gB);
            g_launches.fetch_add(1);
        }
        cudaFreeAsync(part, st);
        *err = cudaPeekAtLastError();
        return true;
    }
}

template <int D, bool ACC>
static void fused2_launch(dim3 g, size_t sm, cudaStream_t st, const Maps &m, const float *B,
                          const Vol &v, int zc, float *gQ, float *gK, float *part) {
    set_smem(modet_bwd_fused2_k<D, ACC>, sm);
    modet_bwd_fused2_k<D, ACC><<<g, 256, sm, st>>>(m, B, v, zc, gQ, gK, part);
}

template <int D>
static bool bwd_fused2(const float *Q, const float *K, const float *B, const float *SF,
                       const float *LSE, const float *gSF, const Vol &v, int S, bool acc,
                       float *gQ, float *gK, float *gB, cudaStream_t st, cudaError_t *err) {
    if constexpr (D > 6) {
        return false;
    } else {
        Maps m{};
        if (!(make_map(&m.k, K, v, S * D, kBoxX, kFRows) &&
              make_maps_a(&m.a, Q, LSE, gSF, SF, v, S, D, kBoxX, kFRows)))
            return false;
        const int gx = (v.h + RTX - 1) / RTX, gy = (v.w + RTY - 1) / RTY;
        const int zc = pick_zc(gx * gy * S, v.l, 2, 4);
        const int nzc = (v.l + zc - 1) / zc;
        const int ncta = gx * gy * nzc;
        const size_t sm = FG2<D>::SMEM;
        float *part = nullptr;
        keep_pool_mapped();
        if ((*err = cudaMallocAsync(&part, (size_t)S * ncta * 27 * sizeof(float), st))) return true;
        const dim3 g(gx, gy, S * nzc);
        if (acc) fused2_launch<D, true>(g, sm, st, m, B, v, zc, gQ, gK, part);
        else fused2_launch<D, false>(g, sm, st, m, B, v, zc, gQ, gK, part);
        g_launches.fetch_add(1);
        if (gB) {
            reduce_db_k<<<dim3(27, S), 256, 0, st>>>(part, ncta, gB);
            g_launches.fetch_add(1);
        }
        cudaFreeAsync(part, st);
        *err = cudaPeekAtLastError();
        return true;
    }
}

template <int D>
static cudaError_t bwd_launch(const float *Q, const float *K, const float *B, const float *SF,
                              const float *LSE, const float *gSF, mdg_dims3 d, int S, bool acc,
                              float *gQ, float *gK, float *gB, cudaStream_t st) {
    const Vol v{d.h, d.w, d.l, (int64_t)d.h * d.w * d.l, (int64_t)d.h * d.w};
    const bool tma = tma_ok(v, {Q, K, SF, LSE, gSF});
    cudaError_t e = cudaSuccess;
    if (tma && bwd_variant() == 2 &&
        bwd_fused2<D>(Q, K, B, SF, LSE, gSF, v, S, acc, gQ, gK, gB, st, &e))
        return e;
    if (tma && bwd_fused<D>(Q, K, B, SF, LSE, gSF, v, S, acc, gQ, gK, gB, st, &e)) return e;
    // the row kernel always runs when dK is wanted: it writes the per-source
    // statistics {LSE*log2e, gSF.SF} the column kernel gathers
    float *aux = nullptr;
    keep_pool_mapped();
    if (gK && (e = cudaMallocAsync(&aux, (size_t)2 * S * v.n * sizeof(float), st))) return e;
    if (gQ || gB || gK) {
        const int gx = (d.h + RTX - 1) / RTX, gy = (d.w + RTY - 1) / RTY;
        const int zc = pick_zc(gx * gy * S, d.l, D <= 6 ? 2 : 1, 5);
        const int nzc = (d.l + zc - 1) / zc;
        const int ncta = gx * gy * nzc;
        float *part = nullptr;
        if ((e = cudaMallocAsync(&part, (size_t)S * ncta * 27 * sizeof(float), st))) return e;
        const size_t sm = (2 * (D * RG::HCH + (D + 7) * RG::OCH) + kTail) * sizeof(float);
        Maps m{};
        const bool t = tma && make_map(&m.k, K, v, S * D, kBoxX, RG::PY) &&
                       make_maps_a(&m.a, Q, LSE, gSF, SF, v, S, D, RTX, RTY);
        const dim3 g(gx, gy, S * nzc);
        if (t) {
            if (acc) row_launch<D, true, true>(g, sm, st, m, Q, K, B, SF, LSE, gSF, v, zc, gQ, part, aux);
            else row_launch<D, true, false>(g, sm, st, m, Q, K, B, SF, LSE, gSF, v, zc, gQ, part, aux);
        } else {
            if (acc) row_launch<D, false, true>(g, sm, st, m, Q, K, B, SF, LSE, gSF, v, zc, gQ, part, aux);
            else row_launch<D, false, false>(g, sm, st, m, Q, K, B, SF, LSE, gSF, v, zc, gQ, part, aux);
        }
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
        const int zc = pick_zc(gx * gy * S, d.l, D <= 6 ? 2 : 1, 5);
        const int nzc = (d.l + zc - 1) / zc;
        const size_t sm = (2 * ((D + 5) * CG::HCH + D * CG::OCH) + kTail) * sizeof(float);
        Maps m{};
        const bool t = tma && reinterpret_cast<uintptr_t>(aux) % 16 == 0 &&
                       make_map(&m.k, K, v, S * D, CTX, CTY) &&
                       make_map(&m.a.q, Q, v, S * D, kBoxX, CG::PY) &&
                       make_map(&m.a.g, gSF, v, 3 * S, kBoxX, CG::PY) &&
                       make_map(&m.aux, aux, v, 2 * S, kBoxX, CG::PY);
        const dim3 g(gx, gy, S * nzc);
        if (t) {
            if (acc) col_launch<D, true, true>(g, sm, st, m, Q, K, B, SF, LSE, gSF, v, zc, gK, aux);
            else col_launch<D, true, false>(g, sm, st, m, Q, K, B, SF, LSE, gSF, v, zc, gK, aux);
        } else {
            if (acc) col_launch<D, false, true>(g, sm, st, m, Q, K, B, SF, LSE, gSF, v, zc, gK, aux);
            else col_launch<D, false, false>(g, sm, st, m, Q, K, B, SF, LSE, gSF, v, zc, gK, aux);
        }
        g_launches.fetch_add(1);
        cudaFreeAsync(aux, st);
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
