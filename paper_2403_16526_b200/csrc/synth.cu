// synth.cu — the reference's synthetic inputs, produced natively so the
// benchmark and the PO driver consume the same bytes as the CPU reference:
//
//   mdg_synth_smooth_velocity   make_smooth_velocity  (synth.cpp:75-90)
//   mdg_synth_random_field      test::random_field    (tests/test_util.hpp:40-48)
//   mdg_synth_pair              make_synth_pair       (synth.cpp:92-192)
//
// The host parts (Rng draws, the separable Gaussian blur, the sphere phantom)
// repeat the reference's float expressions term for term, so the results are
// bit-identical (tests/test_synth.py checks them against oracle/_ref).  The
// blur runs its independent lines on a few host threads (per-line results do
// not depend on the split).  The ground-truth field's scaling-and-squaring
// and the image / label warps of make_synth_pair run on the device with the
// library's bit-exact kernels (mdg_scaling_squaring_fwd, mdg_warp_fwd,
// mdg_warp_labels).
#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

#include "mdg_common.cuh"

namespace mdg {
namespace {

// splitmix64 + Box-Muller (rng.hpp:23-67), as mdg_rng in runtime.cu
struct Rng {
    uint64_t state;
    bool has_spare = false;
    double spare = 0.0;
    explicit Rng(uint64_t s) : state(s) {}
    uint64_t next() {
        uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double normal() {
        if (has_spare) {
            has_spare = false;
            return spare;
        }
        double u1 = uniform(), u2 = uniform();
        if (u1 < 1e-300) u1 = 1e-300;
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 6.283185307179586476925286766559 * u2;
        spare = r * std::sin(a);
        has_spare = true;
        return r * std::cos(a);
    }
};

template <class F>
void parallel_lines(int count, F &&f) {
    const int nt = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (nt == 1 || count < 64) {
        f(0, count);
        return;
    }
    std::vector<std::thread> ts;
    for (int t = 0; t < nt; ++t)
        ts.emplace_back([&, t] { f((int)((int64_t)count * t / nt), (int)((int64_t)count * (t + 1) / nt)); });
    for (auto &t : ts) t.join();
}

// synth.cpp:30-58: separable Gaussian blur, border-renormalised
void gaussian_blur(float *data, mdg_dims3 d, float sigma) {
    if (sigma <= 0.0f) return;
    const int r = std::max(1, static_cast<int>(std::ceil(3.0f * sigma)));
    std::vector<float> k(static_cast<size_t>(2 * r + 1));
    for (int i = -r; i <= r; ++i)
        k[static_cast<size_t>(i + r)] = std::exp(-0.5f * (i * i) / (sigma * sigma));
    const int64_t n = (int64_t)d.h * d.w * d.l;
    std::vector<float> tmp((size_t)n);
    const int dims[3] = {d.h, d.w, d.l};
    const int64_t strides[3] = {1, d.h, (int64_t)d.h * d.w};
    float *src = data, *dst = tmp.data();
    for (int axis = 0; axis < 3; ++axis) {
        const int len = dims[axis];
        const int64_t stride = strides[axis];
        const int ou = axis == 0 ? 1 : 0;
        const int ov = axis == 2 ? 1 : 2;
        parallel_lines(dims[ov], [&](int v0, int v1) {
            for (int v = v0; v < v1; ++v)
                for (int u = 0; u < dims[ou]; ++u) {
                    const int64_t base = u * strides[ou] + v * strides[ov];
                    for (int i = 0; i < len; ++i) {
                        float s = 0.0f, wsum = 0.0f;
                        for (int t = std::max(0, i - r); t <= std::min(len - 1, i + r); ++t) {
                            const float w = k[static_cast<size_t>(t - i + r)];
                            s += w * src[base + t * stride];
                            wsum += w;
                        }
                        dst[base + i * stride] = s / wsum;
                    }
                }
        });
        std::swap(src, dst);
    }
    // three swaps: the result is in tmp
    std::copy(src, src + n, data);
}

// synth.cpp:60-71
float max_vector_norm(const float *f, int64_t n) {
    float best = 0.0f;
    for (int64_t p = 0; p < n; ++p) {
        const float x = f[p], y = f[n + p], z = f[2 * n + p];
        best = std::max(best, std::sqrt(x * x + y * y + z * z));
    }
    return best;
}

void smooth_velocity(mdg_dims3 d, uint64_t seed, float magnitude, float sigma, float *v) {
    Rng rng(seed);
    const int64_t n = (int64_t)d.h * d.w * d.l;
    for (int64_t i = 0; i < 3 * n; ++i) v[i] = static_cast<float>(rng.normal());
    for (int comp = 0; comp < 3; ++comp) gaussian_blur(v + comp * n, d, sigma);
    const float mx = max_vector_norm(v, n);
    if (mx > 0.0f)
        for (int64_t i = 0; i < 3 * n; ++i) v[i] *= magnitude / mx;
}

}  // namespace
}  // namespace mdg

using namespace mdg;

extern "C" {

mdg_status mdg_synth_smooth_velocity(mdg_dims3 d, uint64_t seed, float magnitude, float sigma,
                                     float *out) {
    MDG_REQUIRE(dims_ok(d), "synth: invalid dims " + dims_str(d));
    MDG_REQUIRE(out || nvox(d) == 0, "synth: null pointer");
    smooth_velocity(d, seed, magnitude, sigma, out);
    return MDG_OK;
}

mdg_status mdg_synth_random_field(mdg_dims3 d, uint64_t seed, float mag, float *out) {
    MDG_REQUIRE(dims_ok(d), "synth: invalid dims " + dims_str(d));
    MDG_REQUIRE(out || nvox(d) == 0, "synth: null pointer");
    Rng rng(seed);
    const int64_t m = 3 * nvox(d);
    for (int64_t i = 0; i < m; ++i) {
        const double v = rng.uniform(0.15, 1.0) * mag;
        out[i] = static_cast<float>(rng.uniform() < 0.5 ? -v : v);
    }
    return MDG_OK;
}

mdg_status mdg_synth_pair(mdg_dims3 d, uint64_t seed, float max_disp, float *fixed,
                          float *moving, int *labels_fixed, int *labels_moving, float *gt_field) {
    // SynthConfig defaults (synth.hpp:25-34)
    const float smooth_sigma = 4.0f, texture_sigma = 1.2f, translation_frac = 0.6f;
    const int num_spheres = 3, ss_steps = 7;
    MDG_REQUIRE(dims_ok(d), "synth: invalid dims " + dims_str(d));
    MDG_REQUIRE(d.h >= 8 && d.w >= 8 && d.l >= 8, "synth: dims must be >= 8 per axis");
    MDG_REQUIRE(max_disp >= 0.0f, "synth: max_disp must be >= 0");
    MDG_REQUIRE(fixed && moving && labels_fixed && labels_moving,
                "synth: null pointer");
    Rng rng(seed);
    const int64_t n = nvox(d);
    std::vector<float> texture((size_t)n);
    for (auto &v : texture) v = static_cast<float>(rng.normal());
    gaussian_blur(texture.data(), d, texture_sigma);
    float tmax = 1e-6f;
    for (float v : texture) tmax = std::max(tmax, std::abs(v));
    std::fill(labels_moving, labels_moving + n, 0);

    const int min_dim = std::min({d.h, d.w, d.l});
    struct Ball {
        float cx, cy, cz, r;
    };
    std::vector<Ball> balls;
    for (int i = 0; i < num_spheres; ++i) {
        const float r = static_cast<float>(rng.uniform(0.10, 0.15)) * min_dim;
        Ball b{};
        bool placed = false;
        for (int attempt = 0; attempt < 64 && !placed; ++attempt) {
            b.cx = static_cast<float>(rng.uniform(r + 3.0, d.h - 1 - r - 3.0));
            b.cy = static_cast<float>(rng.uniform(r + 3.0, d.w - 1 - r - 3.0));
            b.cz = static_cast<float>(rng.uniform(r + 3.0, d.l - 1 - r - 3.0));
            b.r = r;
            placed = true;
            for (const Ball &o : balls) {
                const float dx = b.cx - o.cx, dy = b.cy - o.cy, dz = b.cz - o.cz;
                if (std::sqrt(dx * dx + dy * dy + dz * dz) < b.r + o.r + 2.0f) placed = false;
            }
        }
        if (placed) balls.push_back(b);
    }
    // the phantom: texture + periodic pattern + spheres (synth.cpp:129-150)
    parallel_lines(d.l, [&](int z0, int z1) {
        for (int z = z0; z < z1; ++z)
            for (int y = 0; y < d.w; ++y)
                for (int x = 0; x < d.h; ++x) {
                    const int64_t p = ((int64_t)z * d.w + y) * d.h + x;
                    float v = 0.35f + 0.18f * texture[(size_t)p] / tmax;
                    v += 0.04f * std::cos(2.0f * 3.14159265f * x / 7.3f) *
                         std::cos(2.0f * 3.14159265f * y / 6.1f) *
                         std::cos(2.0f * 3.14159265f * z / 8.7f);
                    for (size_t bi = 0; bi < balls.size(); ++bi) {
                        const Ball &b = balls[bi];
                        const float dx = x - b.cx, dy = y - b.cy, dz = z - b.cz;
                        const float dist = std::sqrt(dx * dx + dy * dy + dz * dz);
                        if (dist <= b.r) {
                            v += 0.28f + 0.08f * static_cast<float>(bi);
                            labels_moving[p] = static_cast<int>(bi + 1);
                        } else if (dist <= b.r + 1.5f) {
                            v += (0.28f + 0.08f * static_cast<float>(bi)) * (b.r + 1.5f - dist) / 1.5f;
                        }
                    }
                    moving[p] = v;
                }
    });
    // ground truth: translation + smooth component, integrated (synth.cpp:152-183)
    const float tf = std::min(std::max(translation_frac, 0.0f), 1.0f);
    const float trans_mag = max_disp * tf;
    const float noise_mag = max_disp - trans_mag;
    float tx = static_cast<float>(rng.normal()), ty = static_cast<float>(rng.normal()),
          tz = static_cast<float>(rng.normal());
    const float tn = std::sqrt(tx * tx + ty * ty + tz * tz) + 1e-12f;
    tx *= trans_mag / tn;
    ty *= trans_mag / tn;
    tz *= trans_mag / tn;
    std::vector<float> vel((size_t)(3 * n)), gt((size_t)(3 * n));
    smooth_velocity(d, seed ^ 0x5eed5eedULL, noise_mag, smooth_sigma, vel.data());
    for (int64_t i = 0; i < n; ++i) {
        vel[(size_t)i] += tx;
        vel[(size_t)(n + i)] += ty;
        vel[(size_t)(2 * n + i)] += tz;
    }
    cudaStream_t st = nullptr;
    MDG_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct Guard {
        cudaStream_t s;
        void *bufs[5] = {};
        ~Guard() {
            for (void *b : bufs)
                if (b) cudaFreeAsync(b, s);
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    } g{st};
    MDG_CUDA_TRY(cudaMallocAsync(&g.bufs[0], 3 * n * sizeof(float), st));
    MDG_CUDA_TRY(cudaMallocAsync(&g.bufs[1], 3 * n * sizeof(float), st));
    MDG_CUDA_TRY(cudaMallocAsync(&g.bufs[2], n * sizeof(float), st));
    MDG_CUDA_TRY(cudaMallocAsync(&g.bufs[3], n * sizeof(float), st));
    MDG_CUDA_TRY(cudaMallocAsync(&g.bufs[4], 2 * n * sizeof(int), st));
    float *dv = static_cast<float *>(g.bufs[0]), *dgt = static_cast<float *>(g.bufs[1]);
    float *dmov = static_cast<float *>(g.bufs[2]), *dfix = static_cast<float *>(g.bufs[3]);
    int *dlm = static_cast<int *>(g.bufs[4]), *dlf = dlm + n;
    auto integrate = [&]() -> mdg_status {
        MDG_CUDA_TRY(cudaMemcpyAsync(dv, vel.data(), 3 * n * sizeof(float),
                                     cudaMemcpyHostToDevice, st));
        if (mdg_status e = mdg_scaling_squaring_fwd(dv, d, ss_steps, dgt, nullptr, st)) return e;
        MDG_CUDA_TRY(cudaMemcpyAsync(gt.data(), dgt, 3 * n * sizeof(float),
                                     cudaMemcpyDeviceToHost, st));
        MDG_CUDA_TRY(cudaStreamSynchronize(st));
        return MDG_OK;
    };
    if (mdg_status e = integrate()) return e;
    for (int pass = 0; pass < 3; ++pass) {
        const float mx = max_vector_norm(gt.data(), n);
        if (mx <= max_disp || mx == 0.0f) break;
        const float s = max_disp / mx;
        for (auto &v : vel) v *= s;
        if (mdg_status e = integrate()) return e;
    }
    // fixed = warp(moving, gt); labels_fixed = warp_labels(labels_moving, gt)
    MDG_CUDA_TRY(cudaMemcpyAsync(dmov, moving, n * sizeof(float), cudaMemcpyHostToDevice, st));
    MDG_CUDA_TRY(cudaMemcpyAsync(dlm, labels_moving, n * sizeof(int), cudaMemcpyHostToDevice, st));
    if (mdg_status e = mdg_warp_fwd(dmov, 1, d, dgt, dfix, st)) return e;
    if (mdg_status e = mdg_warp_labels(dlm, d, dgt, dlf, st)) return e;
    MDG_CUDA_TRY(cudaMemcpyAsync(fixed, dfix, n * sizeof(float), cudaMemcpyDeviceToHost, st));
    MDG_CUDA_TRY(cudaMemcpyAsync(labels_fixed, dlf, n * sizeof(int), cudaMemcpyDeviceToHost, st));
    MDG_CUDA_TRY(cudaStreamSynchronize(st));
    if (gt_field) std::copy(gt.begin(), gt.end(), gt_field);
    return MDG_OK;
}

}  // extern "C"
