// runtime.cu — error slots, the device numeric flag, the synthetic-input RNG,
// pinned host memory and the small exact-index entry points of libmdg.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "mdg_common.cuh"

namespace mdg {

std::atomic<int64_t> g_launches{0};

namespace {
thread_local std::string t_err;
thread_local int t_pos[4] = {-1, -1, -1, -1};

std::mutex g_flag_mu;
}  // namespace

void set_error(mdg_status st, const std::string &msg) {
    (void)st;
    t_err = msg;
}

mdg_status status_from_cuda(cudaError_t e, const char *where) {
    t_err = std::string("cuda error in ") + where + ": " + cudaGetErrorString(e);
    return MDG_ECUDA;
}

// Per-(device, stream) state: the numeric flag and the ModeT fixup queue.
// Stream-ordered use keeps one stream's calls from touching another's state,
// so concurrent streams on one device (pair-parallel host threads) are safe.
// Created once per stream and never freed (a few hundred KB), so pointers
// baked into a captured CUDA graph stay valid.  Creation may happen while the
// caller's stream is being captured: it switches this thread to relaxed
// capture mode and initialises the words on a private non-blocking stream,
// which neither joins nor breaks the capture.
namespace {
struct StreamState {
    unsigned long long *flag = nullptr, *fixq = nullptr;
};
struct StreamKey {
    int dev;
    cudaStream_t st;
    bool operator<(const StreamKey &o) const {
        return dev != o.dev ? dev < o.dev : (uintptr_t)st < (uintptr_t)o.st;
    }
};
std::map<StreamKey, StreamState> g_states;

__global__ void state_init_k(unsigned long long *flag, unsigned long long *fixq) {
    *flag = ~0ull;
    *fixq = 0ull;
}

StreamState *stream_state(cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_flag_mu);
    StreamState &s = g_states[StreamKey{dev, st}];
    if (!s.flag) {
        cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
        cudaThreadExchangeStreamCaptureMode(&mode);
        void *p = nullptr;
        cudaStream_t init = nullptr;
        bool ok = cudaMalloc(&p, (kFixupCap + 2) * sizeof(unsigned long long)) == cudaSuccess &&
                  cudaStreamCreateWithFlags(&init, cudaStreamNonBlocking) == cudaSuccess;
        if (ok) {
            auto *w = static_cast<unsigned long long *>(p);
            state_init_k<<<1, 1, 0, init>>>(w, w + 1);
            ok = cudaStreamSynchronize(init) == cudaSuccess;
            if (ok) {
                s.flag = w;
                s.fixq = w + 1;
            }
        }
        if (init) cudaStreamDestroy(init);
        if (!ok && p) cudaFree(p);
        cudaThreadExchangeStreamCaptureMode(&mode);
        if (!ok) return nullptr;
    }
    return &s;
}
}  // namespace

unsigned long long *numeric_flag_ptr(cudaStream_t st) {
    StreamState *s = stream_state(st);
    return s ? s->flag : nullptr;
}

unsigned long long *fixup_queue_ptr(cudaStream_t st) {
    StreamState *s = stream_state(st);
    return s ? s->fixq : nullptr;
}

namespace {
std::atomic<int> g_det{-1};
}
bool deterministic_mode() {
    int v = g_det.load(std::memory_order_relaxed);
    if (v < 0) {
        const char *e = std::getenv("MDG_DETERMINISTIC");
        v = (e && *e && *e != '0') ? 1 : 0;
        int expect = -1;
        g_det.compare_exchange_strong(expect, v);
        v = g_det.load();
    }
    return v == 1;
}

void keep_pool_mapped() {
    static std::mutex mu;
    static std::vector<bool> done;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    std::lock_guard<std::mutex> lk(mu);
    if ((int)done.size() <= dev) done.resize(dev + 1, false);
    if (done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done[dev] = true;
}

mdg_status consume_numeric_flag(cudaStream_t st, mdg_dims3 d) {
    unsigned long long *f = numeric_flag_ptr(st);
    if (!f) return status_from_cuda(cudaErrorMemoryAllocation, "numeric flag");
    unsigned long long key = ~0ull;
    MDG_CUDA_TRY(cudaMemcpyAsync(&key, f, sizeof(key), cudaMemcpyDeviceToHost, st));
    MDG_CUDA_TRY(cudaStreamSynchronize(st));
    if (key == ~0ull) return MDG_OK;
    MDG_CUDA_TRY(cudaMemsetAsync(f, 0xff, sizeof(key), st));
    MDG_CUDA_TRY(cudaStreamSynchronize(st));
    const int64_t n = nvox(d);
    if (n > 0) {
        const int64_t p = (int64_t)(key % (unsigned long long)n);
        t_pos[3] = (int)(key / (unsigned long long)n);
        t_pos[0] = (int)(p % d.h);
        t_pos[1] = (int)((p / d.h) % d.w);
        t_pos[2] = (int)(p / ((int64_t)d.h * d.w));
    }
    // attention.hpp:110-114 message shape
    t_err = "attention: non-finite logit at position (" + std::to_string(t_pos[0]) + "," +
            std::to_string(t_pos[1]) + "," + std::to_string(t_pos[2]) + ") head " +
            std::to_string(t_pos[3]);
    return MDG_ENUMERIC;
}

// sampling.hpp:38-49 evaluated on the device (exactness probe)
__global__ void resolve_axis_k(const float *x, int n, int dim, int *i0, int *i1, float *f,
                               int *live) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Ax a = resolve_axis(x[i], dim);
    i0[i] = a.i0;
    i1[i] = a.i1;
    f[i] = a.f;
    live[i] = a.live ? 1 : 0;
}

}  // namespace mdg

using namespace mdg;

// ------------------------------------------------------------- RNG (host)
// rng.hpp:23-67: splitmix64, uniform = top 53 bits * 2^-53, Box-Muller normal
// returning the cos branch and caching the sin branch.
struct mdg_rng {
    uint64_t state;
    bool has_spare;
    double spare;
    uint64_t next() {
        uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    double u01() { return (double)(next() >> 11) * 0x1.0p-53; }
    double normal() {
        if (has_spare) {
            has_spare = false;
            return spare;
        }
        double u1 = u01(), u2 = u01();
        if (u1 < 1e-300) u1 = 1e-300;
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 6.283185307179586476925286766559 * u2;
        spare = r * std::sin(a);
        has_spare = true;
        return r * std::cos(a);
    }
};

extern "C" {

const char *mdg_last_error(void) { return t_err.c_str(); }

void mdg_last_error_position(int *x, int *y, int *z, int *head) {
    if (x) *x = t_pos[0];
    if (y) *y = t_pos[1];
    if (z) *z = t_pos[2];
    if (head) *head = t_pos[3];
}

int mdg_device_ok(void) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return 0;
    return p.major == 10 && p.minor == 0;
}

const char *mdg_build_info(void) {
    return "libmdg: sm_100a fp32 ModeT hot path";
}

mdg_status mdg_check_numeric(mdg_dims3 d, void *stream) {
    return consume_numeric_flag(S_(stream), d);
}

int64_t mdg_launch_count(void) { return g_launches.load(); }

int mdg_set_deterministic(int on) {
    const int prev = deterministic_mode() ? 1 : 0;
    g_det.store(on ? 1 : 0);
    return prev;
}

int mdg_get_deterministic(void) { return deterministic_mode() ? 1 : 0; }

mdg_status mdg_window_offset(int o, int nb, int off[3]) {
    MDG_REQUIRE(nb >= 3 && nb % 2 == 1, "attention: neighborhood must be odd and >= 3");
    MDG_REQUIRE(o >= 0 && o < nb * nb * nb, "window_offset: slot out of range");
    const int r = (nb - 1) / 2;
    off[0] = o % nb - r;
    off[1] = (o / nb) % nb - r;
    off[2] = o / (nb * nb) - r;
    return MDG_OK;
}

mdg_status mdg_resolve_axis(const float *x, int n, int dim, int *i0, int *i1, float *f,
                            int *live, void *stream) {
    MDG_REQUIRE(n >= 0, "resolve_axis: n < 0");
    if (n == 0) return MDG_OK;
    resolve_axis_k<<<grid1d(n, 256), 256, 0, S_(stream)>>>(x, n, dim, i0, i1, f, live);
    MDG_LAUNCHED();
    return MDG_OK;
}

mdg_rng *mdg_rng_new(uint64_t seed) {
    mdg_rng *r = new mdg_rng;
    r->state = seed;
    r->has_spare = false;
    r->spare = 0.0;
    return r;
}

void mdg_rng_free(mdg_rng *r) { delete r; }

void mdg_rng_fill_uniform(mdg_rng *r, float *out, int64_t n, double lo, double hi) {
    for (int64_t i = 0; i < n; ++i) out[i] = (float)(lo + (hi - lo) * r->u01());
}

void mdg_rng_fill_normal(mdg_rng *r, float *out, int64_t n, double mean, double sd) {
    for (int64_t i = 0; i < n; ++i) out[i] = (float)(mean + sd * r->normal());
}

void *mdg_host_alloc(size_t bytes) {
    void *p = nullptr;
    if (cudaMallocHost(&p, bytes) != cudaSuccess) return nullptr;
    return p;
}

void mdg_host_free(void *p) {
    if (p) cudaFreeHost(p);
}

}  // extern "C"
