// warp_gather.cu — the warp's input gradient as a deterministic GATHER.
//
// The reference scatters every source voxel's gradient into the 8 corners of
// the cell its displaced position falls in (sampling.hpp:103-118, 139-167).
// On the GPU a scatter needs float atomics, whose summation order changes from
// run to run, so two identical pairwise optimisations would drift apart
// (the reference promises bitwise-repeatable traces, test_engine.cpp:194-213).
// Here each target voxel owns its sum:
//
//   * a CTA owns a 32 x 8 column of targets and marches a z chunk;
//   * every step it BINS one plane of source voxels (the sources within the
//     displacement bound R of the tile) into per-cell lists in shared memory
//     (cell = the source's lower corner i0, integer exact as resolve_axis
//     computes it); shared-memory integer atomics only pick list slots;
//   * each target then walks the 8 cells it is a corner of, in the
//     reference's corner order, and within a cell its sources in increasing
//     voxel order (the list is sorted by source position), adding
//     ((g * wx) * wy) * wz exactly as the reference forms the term, skipping
//     g == 0 channels as the reference does.
//
// The sum order is a fixed function of the inputs: results are bit-identical
// from run to run (not bit-identical to the reference's p-ordered sum, which
// interleaves the cells; within tolerance).  R = ceil(max |phi|) comes from
// the gfield kernel (atomicMax over the field) on the device, so nothing
// synchronises with the host.  Limits and their deterministic fallbacks:
//   * a cell with more than kCap sources (strong local compression): the
//     target plane is recorded and redone by warp_gin_exact_k, a brute-force
//     window gather in the reference's own order (bit-exact);
//   * R > kRMax or a non-finite displacement: the scatter kernel with float
//     atomics runs instead (the only non-deterministic case; |phi| <= 4
//     voxels covers registration fields at every pyramid level).
#include <algorithm>

#include "mdg_common.cuh"

namespace mdg {
namespace gather {

constexpr int TX = 32, TY = 8, NT = TX * TY;
constexpr int kRMax = kGinGatherReach;
constexpr int kNP = 2 * kRMax + 3;  // cell planes in flight
constexpr int CX = TX + 1, CY = TY + 1, NCELL = CX * CY;
constexpr int kCap = 8;

__device__ __forceinline__ int ring(int c, int base) {
    const int r = (c - base) % kNP;
    return r;
}

// R from the device-side max |phi| (float bits, atomicMax'ed by the gfield
// kernel); kRMax + 1 means "out of range / non-finite"
__device__ __forceinline__ int bound_of(const unsigned *rbits) {
    const float m = __uint_as_float(*rbits);
    if (!(m <= (float)kRMax)) return kRMax + 1;  // also NaN / inf
    return (int)ceilf(m);
}

// dynamic shared memory: per cell plane slot, NCELL counters, NCELL x kCap
// position keys, and an overflow flag
constexpr size_t kSmem = (size_t)kNP * NCELL * (4 + 2 * kCap) + kNP * 4;

template <int CT>
__global__ void __launch_bounds__(NT, 3)
warp_gin_gather_k(const float *__restrict__ field, const float *__restrict__ gout, int C, int h,
                  int w, int l, int zc, int zt0, int zt1, int pb, int pe,
                  const unsigned *__restrict__ rbits, float *__restrict__ gin,
                  unsigned *__restrict__ dirty) {
    extern __shared__ __align__(16) unsigned char gsm[];
    auto cnt = reinterpret_cast<unsigned (*)[NCELL]>(gsm);
    auto keys = reinterpret_cast<unsigned short (*)[NCELL][kCap]>(gsm + (size_t)kNP * NCELL * 4);
    int *over = reinterpret_cast<int *>(gsm + (size_t)kNP * NCELL * (4 + 2 * kCap));
    const int R = bound_of(rbits);
    if (R > kRMax) return;  // warp_bwd_k's atomic scatter takes this call
    // 32-bit element offsets throughout (the host guarantees C * n < 2^31)
    const unsigned n = (unsigned)h * w * l, hw = (unsigned)h * w;
    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    // target planes [zt0, zt1): those the sources [pb, pe) can reach
    const int zb = zt0 + blockIdx.z * zc, ze = min(zb + zc, zt1);
    const int cbase = zb - 1;  // oldest cell plane this chunk needs
    for (int i = tid; i < kNP * NCELL; i += NT) (&cnt[0][0])[i] = 0;
    if (tid < kNP) over[tid] = 0;
    __syncthreads();
    const int bx0 = x0 - R - 1, by0 = y0 - R - 1;
    const int BW = TX + 2 * R + 1, BH = TY + 2 * R + 1;
    // bin source plane s: sources whose cell lies in this tile's cells
    // (x0-1 .. x0+31, y0-1 .. y0+7) and in cell planes zb-1 .. ze-1
    auto bin = [&](int s) {
        if (s < 0 || s >= l) return;
        // warp = box row (x along lanes: coalesced field loads)
        for (int ry = ty; ry < BH; ry += NT / 32) {
            const int sy = by0 + ry;
            if (sy < 0 || sy >= w) continue;
            for (int rx = tx; rx < BW; rx += 32) {
                const int sx = bx0 + rx;
                if (sx < 0 || sx >= h) continue;
                const int p = s * (int)hw + sy * h + sx;
                if (p < pb || p >= pe) continue;
                const Ax ax = resolve_axis(add_((float)sx, __ldg(field + p)), h);
                const Ax ay = resolve_axis(add_((float)sy, __ldg(field + n + p)), w);
                const Ax az = resolve_axis(add_((float)s, __ldg(field + 2 * n + p)), l);
                const int cx = ax.i0 - (x0 - 1), cy = ay.i0 - (y0 - 1), cz = az.i0;
                if (cx < 0 || cx >= CX || cy < 0 || cy >= CY || cz < zb - 1 || cz > ze - 1)
                    continue;
                const int rz = ring(cz, cbase), ci = cy * CX + cx;
                const unsigned k = atomicAdd(&cnt[rz][ci], 1u);
                if (k < kCap) {
                    // position key, increasing with p within a cell
                    keys[rz][ci][k] = (unsigned short)(((s - cz + R) << 11) | (ry << 6) | rx);
                } else {
                    over[rz] = 1;
                }
            }
        }
    };
    for (int s = zb - R - 1; s <= zb + R; ++s) bin(s);
    __syncthreads();
    const int x = x0 + tx, y = y0 + ty;
    const bool vv = x < h && y < w;
    const bool cxl = h <= 1, cyl = w <= 1, czl = l <= 1;  // collapsed axes
    // sort one cell plane's lists in place (position order; keys distinct):
    // a plane is complete once the source planes up to its index + R + 1 are
    // binned, and each list then serves up to 8 targets
    auto sort_plane = [&](int c) {
        if (c < cbase) return;
        const int r = ring(c, cbase);
        for (int ci = tid; ci < NCELL; ci += NT) {
            const int m = min((int)cnt[r][ci], kCap);
            unsigned short *kl = keys[r][ci];
            for (int a = 1; a < m; ++a) {
                const unsigned short v = kl[a];
                int b = a - 1;
                while (b >= 0 && kl[b] > v) {
                    kl[b + 1] = kl[b];
                    --b;
                }
                kl[b + 1] = v;
            }
        }
    };
    sort_plane(zb - 1);
    for (int z = zb; z < ze; ++z) {
        bin(z + R + 1);
        __syncthreads();
        sort_plane(z);
        __syncthreads();
        const bool dirt = over[ring(z - 1, cbase)] || over[ring(z, cbase)];
        if (dirt) {
            if (tid == 0) {
                const unsigned i = atomicAdd(&dirty[0], 1u);
                // (tile, z) of a plane to redo exactly
                dirty[1 + i] = ((unsigned)(blockIdx.y * gridDim.x + blockIdx.x) << 12) | (unsigned)z;
            }
        } else if (vv) {
            const unsigned t = (unsigned)z * hw + (unsigned)(y * h + x);
            float acc[CT > 0 ? CT : 16];
#pragma unroll
            for (int ch = 0; ch < (CT > 0 ? CT : 16); ++ch)
                if (CT > 0 || ch < C) acc[ch] = gin[ch * n + t];
            // the 8 cells this target is a corner of, in the reference's
            // corner order (x bit fastest, then y, then z): cell plane z - bz
            // lives in ring slot rzs[bz]; list index = own cell - (by*CX + bx)
            const int rzs[2] = {ring(czl ? 0 : z, cbase), ring(czl ? 0 : z - 1, cbase)};
            const bool okx[2] = {cxl || x <= h - 2, cxl || x >= 1};
            const bool oky[2] = {cyl || y <= w - 2, cyl || y >= 1};
            const bool okz[2] = {czl || z <= l - 2, czl || z >= 1};
            const int ci0 = (cyl ? 1 - y0 : ty + 1) * CX + (cxl ? 1 - x0 : tx + 1);
            auto cell_of = [&](int k, int &rz, int &ci) {
                const int bxb = k & 1, byb = (k >> 1) & 1, bzb = k >> 2;
                if (!(okx[bxb] && oky[byb] && okz[bzb])) return 0;
                rz = rzs[bzb];
                ci = ci0 - (cyl ? 0 : byb * CX) - (cxl ? 0 : bxb);
                return (int)cnt[rz][ci];
            };
            int total = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                int rz, ci;
                total += cell_of(k, rz, ci);
            }
            // one flat loop over the target's entries (lanes diverge only by
            // their entry counts, not per cell)
            int k = -1, j = 0, m = 0, rz = 0, ci = 0;
#pragma unroll 1
            for (int e = 0; e < total; ++e) {
                while (j >= m) {
                    ++k;
                    m = cell_of(k, rz, ci);
                    j = 0;
                }
                const unsigned key = keys[rz][ci][j++];
                const int bxb = k & 1, byb = (k >> 1) & 1, bzb = k >> 2;
                const int cxg = cxl ? 0 : x - bxb, cyg = cyl ? 0 : y - byb, czg = czl ? 0 : z - bzb;
                const int s = czg + (int)(key >> 11) - R;
                const int sy = by0 + (int)((key >> 6) & 31), sx = bx0 + (int)(key & 63);
                const unsigned p = (unsigned)s * hw + (unsigned)(sy * h + sx);
                // resolve_axis's f against the known lower corner (the cell);
                // no NaN reaches here (the bound excludes it)
                auto frac = [](float c, int dim, int i0) {
                    return __fsub_rn(fminf(fmaxf(c, 0.0f), (float)(dim - 1)), (float)i0);
                };
                const float fx = cxl ? 0.0f : frac(add_((float)sx, __ldg(field + p)), h, cxg);
                const float fy = cyl ? 0.0f : frac(add_((float)sy, __ldg(field + n + p)), w, cyg);
                const float fz = czl ? 0.0f : frac(add_((float)s, __ldg(field + 2 * n + p)), l, czg);
                const float wx = bxb ? fx : sub_(1.0f, fx);
                const float wy = byb ? fy : sub_(1.0f, fy);
                const float wz = bzb ? fz : sub_(1.0f, fz);
                const float *gp = gout + p;
#pragma unroll
                for (int ch = 0; ch < (CT > 0 ? CT : 16); ++ch) {
                    if (CT == 0 && ch >= C) break;
                    const float g = __ldg(gp + ch * n);
                    if (g != 0.0f) acc[ch] = add_(acc[ch], mul_(mul_(mul_(g, wx), wy), wz));
                }
            }
#pragma unroll
            for (int ch = 0; ch < (CT > 0 ? CT : 16); ++ch)
                if (CT > 0 || ch < C) gin[ch * n + t] = acc[ch];
        }
        __syncthreads();
        // cell plane z-1 is done: recycle its ring slot
        if (z - 1 >= cbase) {
            const int r = ring(z - 1, cbase);
            for (int i = tid; i < NCELL; i += NT) cnt[r][i] = 0;
            if (tid == 0) over[r] = 0;
        }
        // (the next step's binning writes cell planes >= z+1 only; the slot
        // just cleared is reused for plane z-1+kNP, reached after a barrier)
        __syncthreads();
    }
}

// Exact per-target gather over the whole displacement window, in the
// reference's own order (sources in increasing voxel order, a source's 8
// corners in listing order): bit-identical to the CPU scatter.  Redoes the
// target planes the binned kernel recorded as overflowing.
__global__ void __launch_bounds__(NT)
warp_gin_exact_k(const float *__restrict__ field, const float *__restrict__ gout, int C, int h,
                 int w, int l, int64_t pb, int64_t pe, int tiles_x,
                 const unsigned *__restrict__ rbits, const unsigned *__restrict__ dirty,
                 float *__restrict__ gin) {
    const int R = bound_of(rbits);
    if (R > kRMax) return;
    const unsigned nd = dirty[0];
    const int64_t n = (int64_t)h * w * l, hw = (int64_t)h * w;
    for (unsigned e = blockIdx.x; e < nd; e += gridDim.x) {
        const unsigned v = dirty[1 + e];
        const int z = (int)(v & 4095u), tile = (int)(v >> 12);
        const int x = (tile % tiles_x) * TX + (threadIdx.x & 31);
        const int y = (tile / tiles_x) * TY + (threadIdx.x >> 5);
        if (x >= h || y >= w) continue;
        const int64_t t = (int64_t)z * hw + (int64_t)y * h + x;
        float acc[16];
        for (int ch = 0; ch < C; ++ch) acc[ch] = gin[(int64_t)ch * n + t];
        for (int s = max(0, z - R - 1); s <= min(l - 1, z + R + 1); ++s)
            for (int sy = max(0, y - R - 1); sy <= min(w - 1, y + R + 1); ++sy)
                for (int sx = max(0, x - R - 1); sx <= min(h - 1, x + R + 1); ++sx) {
                    const int64_t p = (int64_t)s * hw + (int64_t)sy * h + sx;
                    if (p < pb || p >= pe) continue;
                    const Ax ax = resolve_axis(add_((float)sx, __ldg(field + p)), h);
                    const Ax ay = resolve_axis(add_((float)sy, __ldg(field + n + p)), w);
                    const Ax az = resolve_axis(add_((float)s, __ldg(field + 2 * n + p)), l);
                    if ((ax.i0 != x && ax.i1 != x) || (ay.i0 != y && ay.i1 != y) ||
                        (az.i0 != z && az.i1 != z))
                        continue;
                    const float wx[2] = {sub_(1.0f, ax.f), ax.f};
                    const float wy[2] = {sub_(1.0f, ay.f), ay.f};
                    const float wz[2] = {sub_(1.0f, az.f), az.f};
                    const int cx[2] = {ax.i0, ax.i1}, cy[2] = {ay.i0, ay.i1}, cz[2] = {az.i0, az.i1};
                    for (int ch = 0; ch < C; ++ch) {
                        const float g = __ldg(gout + (int64_t)ch * n + p);
                        if (g == 0.0f) continue;
                        for (int k = 0; k < 8; ++k) {
                            const int bx = k & 1, by = (k >> 1) & 1, bz = k >> 2;
                            if (cx[bx] == x && cy[by] == y && cz[bz] == z)
                                acc[ch] = add_(acc[ch], mul_(mul_(mul_(g, wx[bx]), wy[by]), wz[bz]));
                        }
                    }
                }
        for (int ch = 0; ch < C; ++ch) gin[(int64_t)ch * n + t] = acc[ch];
    }
}

}  // namespace gather

// host side: the three launches after the gfield kernel has filled *rbits
static int gin_gather_pick_zc(mdg_dims3 d, int planes) {
    const int tiles = ((d.h + gather::TX - 1) / gather::TX) * ((d.w + gather::TY - 1) / gather::TY);
    const int want = 148 * 3 * 4;  // ~4 waves of 3 CTAs per SM
    int nzc = (want + tiles - 1) / tiles;
    nzc = max(1, min(nzc, (planes + 11) / 12));  // chunks of >= 12 planes
    return (planes + nzc - 1) / nzc;
}

static mdg_status gin_gather_group(const float *field, const float *gout, int C, mdg_dims3 d,
                                   float *gin, int64_t pb, int64_t pe, const unsigned *rbits,
                                   unsigned *dirty, cudaStream_t st);

mdg_status warp_gin_gather(const float *field, const float *gout, int C, mdg_dims3 d, float *gin,
                           int64_t pb, int64_t pe, const unsigned *rbits, unsigned *dirty,
                           cudaStream_t st) {
    // channel groups of <= 16 (the per-target accumulators live in registers);
    // each group re-bins its cells: the dirty list is reset per group
    const int64_t n = nvox(d);
    for (int c0 = 0; c0 < C; c0 += 16) {
        if (c0 > 0) MDG_CUDA_TRY(cudaMemsetAsync(dirty, 0, sizeof(unsigned), st));
        const int cg = std::min(16, C - c0);
        if (mdg_status e = gin_gather_group(field, gout + (int64_t)c0 * n, cg, d,
                                            gin + (int64_t)c0 * n, pb, pe, rbits, dirty, st))
            return e;
    }
    return MDG_OK;
}

static mdg_status gin_gather_group(const float *field, const float *gout, int C, mdg_dims3 d,
                                   float *gin, int64_t pb, int64_t pe, const unsigned *rbits,
                                   unsigned *dirty, cudaStream_t st) {
    using namespace gather;
    const int64_t hw = (int64_t)d.h * d.w;
    const int zt0 = (int)std::max<int64_t>(0, pb / hw - kRMax - 1);
    const int zt1 = (int)std::min<int64_t>(d.l, (pe - 1) / hw + kRMax + 2);
    const int zc = gin_gather_pick_zc(d, zt1 - zt0);
    const dim3 g((d.h + TX - 1) / TX, (d.w + TY - 1) / TY, (zt1 - zt0 + zc - 1) / zc);
    MDG_REQUIRE(d.l < 4096 && (int64_t)g.x * g.y < (1 << 20) && 3 * nvox(d) < (int64_t(1) << 31),
                "warp: volume too large for the gather");
    switch (C) {
#define MDG_G(CTV)                                                                             \
    case CTV:                                                                                  \
        cudaFuncSetAttribute(warp_gin_gather_k<CTV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)kSmem);                                                      \
        warp_gin_gather_k<CTV><<<g, NT, kSmem, st>>>(field, gout, C, d.h, d.w, d.l, zc, zt0, zt1, \
                                                     (int)pb, (int)pe, rbits, gin, dirty);     \
        break;
        MDG_G(1) MDG_G(2) MDG_G(3) MDG_G(4) MDG_G(8) MDG_G(16)
#undef MDG_G
        default:
            cudaFuncSetAttribute(warp_gin_gather_k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kSmem);
            warp_gin_gather_k<0><<<g, NT, kSmem, st>>>(field, gout, C, d.h, d.w, d.l, zc, zt0, zt1,
                                                       (int)pb, (int)pe, rbits, gin, dirty);
    }
    MDG_LAUNCHED();
    warp_gin_exact_k<<<148 * 2, NT, 0, st>>>(field, gout, C, d.h, d.w, d.l, pb, pe, (int)g.x, rbits,
                                            dirty, gin);
    MDG_LAUNCHED();
    return MDG_OK;
}

// scratch words the gather path needs: [0] max|phi| bits, [1] dirty count,
// [2 ..] dirty list (one entry per tile x plane)
int64_t gin_gather_scratch_words(mdg_dims3 d) {
    return 2 + (int64_t)((d.h + gather::TX - 1) / gather::TX) *
                   ((d.w + gather::TY - 1) / gather::TY) * d.l;
}

}  // namespace mdg
