// labels.cu — label-volume evaluation on sm_100a (the Dice gate of the
// north star; metrics.cpp:100-164).
//
// warp_labels: nearest-neighbour pull x + phi(x) rounded by floor(. + 0.5f)
// and clamped, in the reference's float evaluation order — integer results,
// bit-identical.  mean_dice: exact integer counts per label (|a|, |b|,
// |a & b|) by 64-bit atomics, then the reference's double arithmetic over the
// present labels in ascending order on the host: bit-identical Dice.
#include <algorithm>
#include <vector>

#include "mdg_common.cuh"

namespace mdg {

__global__ void warp_labels_k(const int *__restrict__ labels, int h, int w, int l,
                              const float *__restrict__ phi, int *__restrict__ out) {
    const int n = h * w * l;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int t = p / h, x = p - t * h, z = t / w, y = t - z * w;
    // metrics.cpp:153-160: floor(x + phi + 0.5f), clamped
    const int xi = min(max((int)floorf(add_(add_((float)x, phi[p]), 0.5f)), 0), h - 1);
    const int yi = min(max((int)floorf(add_(add_((float)y, phi[n + p]), 0.5f)), 0), w - 1);
    const int zi = min(max((int)floorf(add_(add_((float)z, phi[2 * n + p]), 0.5f)), 0), l - 1);
    out[p] = labels[(zi * w + yi) * h + xi];
}

// counts[3*label + {0,1,2}] = {|a == label|, |b == label|, |both|};
// bad != 0 if a label falls outside [0, max_label]
__global__ void label_counts_k(const int *__restrict__ a, const int *__restrict__ b, int64_t n,
                               int max_label, unsigned long long *__restrict__ counts,
                               int *__restrict__ bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int la = a[i], lb = b[i];
        if (la < 0 || la > max_label || lb < 0 || lb > max_label) {
            *bad = 1;
            continue;
        }
        atomicAdd(&counts[3 * la], 1ull);
        atomicAdd(&counts[3 * lb + 1], 1ull);
        if (la == lb) atomicAdd(&counts[3 * la + 2], 1ull);
    }
}

}  // namespace mdg

using namespace mdg;

extern "C" {

mdg_status mdg_warp_labels(const int *labels, mdg_dims3 d, const float *phi, int *out,
                           void *stream) {
    MDG_REQUIRE(dims_ok(d), "warp_labels: invalid dims " + dims_str(d));
    const int64_t n = nvox(d);
    if (n == 0) return MDG_OK;
    MDG_REQUIRE(labels && phi && out, "warp_labels: null pointer");
    MDG_REQUIRE(labels != out, "warp_labels: output must not alias the labels");
    warp_labels_k<<<grid1d(n, 256), 256, 0, S_(stream)>>>(labels, d.h, d.w, d.l, phi, out);
    MDG_LAUNCHED();
    return MDG_OK;
}

mdg_status mdg_mean_dice(const int *a, const int *b, int64_t n, int max_label, double *dice,
                         void *stream) {
    MDG_REQUIRE(n >= 0 && max_label >= 0 && max_label < (1 << 20), "mean_dice: invalid sizes");
    MDG_REQUIRE(dice, "mean_dice: null output");
    cudaStream_t st = S_(stream);
    const size_t nc = 3 * (size_t)(max_label + 1);
    Scratch sc;
    MDG_CUDA_TRY(sc.alloc(nc * sizeof(unsigned long long) + 16, st));
    unsigned long long *counts = sc.as<unsigned long long>();
    int *bad = reinterpret_cast<int *>(counts + nc);
    MDG_CUDA_TRY(cudaMemsetAsync(counts, 0, nc * sizeof(unsigned long long) + 16, st));
    if (n > 0) {
        MDG_REQUIRE(a && b, "mean_dice: null pointer");
        const unsigned g = (unsigned)std::min<int64_t>(grid1d(n, 256), 148 * 8);
        label_counts_k<<<g, 256, 0, st>>>(a, b, n, max_label, counts, bad);
        MDG_LAUNCHED();
    }
    std::vector<unsigned long long> h(nc);
    int hbad = 0;
    MDG_CUDA_TRY(cudaMemcpyAsync(h.data(), counts, nc * sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, st));
    MDG_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    MDG_CUDA_TRY(cudaStreamSynchronize(st));
    MDG_REQUIRE(!hbad, "mean_dice: label outside [0, max_label]");
    // metrics.cpp:100-129: labels present in either volume (label 0 excluded),
    // ascending; dice = 2|a&b| / (|a|+|b|); mean in double
    double sum = 0.0;
    int present = 0;
    for (int lab = 1; lab <= max_label; ++lab) {
        const unsigned long long na = h[3 * lab], nb = h[3 * lab + 1], in = h[3 * lab + 2];
        if (na + nb == 0) continue;
        sum += 2.0 * (double)in / (double)(na + nb);
        ++present;
    }
    *dice = present ? sum / (double)present : 1.0;
    return MDG_OK;
}

}  // extern "C"
