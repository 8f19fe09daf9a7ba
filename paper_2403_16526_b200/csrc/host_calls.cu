// host_calls.cu — synchronous host-buffer drop-ins for the reference CPU
// functions (attention.hpp:83 / 127, sampling.hpp:123 / 139).  The caller
// passes host pointers exactly as to mdreg::kern::*; staging buffers come from
// the stream-ordered pool, copies and kernels run on a per-thread stream, and
// the call returns after the results are back in host memory.  With pinned
// host buffers (mdg_host_alloc) the copies run at full PCIe/C2C bandwidth.
#include <algorithm>
#include <climits>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#include "mdg_common.cuh"

namespace mdg {
namespace {

struct HostStream {
    cudaStream_t st = nullptr;
    HostStream() { cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking); }
    ~HostStream() {
        if (st) cudaStreamDestroy(st);
    }
};

cudaStream_t host_stream() {
    thread_local HostStream hs;
    return hs.st;
}

// a set of device staging buffers freed (stream-ordered) on scope exit
struct Stage {
    cudaStream_t st;
    std::vector<void *> bufs;
    explicit Stage(cudaStream_t s) : st(s) {}
    ~Stage() {
        for (void *p : bufs) cudaFreeAsync(p, st);
    }
    // device copy of a host array (h2d when `upload`)
    cudaError_t get(float **dev, const float *host, size_t count, bool upload) {
        *dev = nullptr;
        if (!host) return cudaSuccess;
        void *p = nullptr;
        cudaError_t e = cudaMallocAsync(&p, count * sizeof(float) + 16, st);
        if (e != cudaSuccess) return e;
        bufs.push_back(p);
        *dev = static_cast<float *>(p);
        if (upload)
            return cudaMemcpyAsync(p, host, count * sizeof(float), cudaMemcpyHostToDevice, st);
        return cudaSuccess;
    }
    cudaError_t down(float *host, const float *dev, size_t count) {
        if (!host) return cudaSuccess;
        return cudaMemcpyAsync(host, dev, count * sizeof(float), cudaMemcpyDeviceToHost, st);
    }
};

}  // namespace
}  // namespace mdg

using namespace mdg;

#define MDG_STAGE_TRY(expr)                                            \
    do {                                                               \
        cudaError_t _e = (expr);                                       \
        if (_e != cudaSuccess) return status_from_cuda(_e, #expr);     \
    } while (0)

// ===================================================== z-chunk pipelining
// The ModeT host calls move 4-7x more bytes over PCIe than the kernels need
// time for, so they run as a three-stream pipeline over z-chunks: chunk i+1
// is uploaded (H2D engine) while chunk i computes and chunk i-1's results
// come back (D2H engine) — both copy directions busy at once.  Each chunk is
// staged as its own small volume extended by one halo plane per side; the
// halo planes are device-to-device copies from the neighbouring chunks (the
// same decomposition as the multi-GPU depth slabs, paper_2403_16526_b200/
// slab.py), so per-voxel results are bit-identical to the whole-volume call.
namespace mdg {

__global__ void fill_k(float *p, int64_t m, float v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) p[i] = v;
}

namespace {

struct PipeStreams {
    cudaStream_t up = nullptr, comp = nullptr, down = nullptr;
    PipeStreams() {
        cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&down, cudaStreamNonBlocking);
    }
    ~PipeStreams() {
        for (cudaStream_t s : {up, comp, down})
            if (s) cudaStreamDestroy(s);
    }
};
PipeStreams &pipe_streams() {
    thread_local PipeStreams ps;
    return ps;
}

// Accumulate targets (the reference's `+=` gradients) are NOT uploaded: the
// device computes each chunk's contribution into a fresh buffer, it comes
// back into pinned staging, and host threads add it into the caller's array
// (one IEEE fp32 add per element — the same operation the device would do,
// so results are bit-identical) while later chunks are still in flight.
// This removes the largest H2D stream of the backward calls.
struct PinnedStage {
    float *p = nullptr;
    size_t cap = 0;
    ~PinnedStage() {
        if (p) cudaFreeHost(p);
    }
    cudaError_t reserve(size_t floats) {
        if (floats <= cap) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMallocHost(&p, floats * sizeof(float));
        if (e == cudaSuccess) cap = floats;
        return e;
    }
};
PinnedStage &pinned_stage() {
    thread_local PinnedStage ps;
    return ps;
}

// A small persistent pool for the host-side adds.  Workers block on a
// condition variable between jobs (no spinning), so they never compete with
// the thread that is feeding the copy engines.
class AddPool {
  public:
    AddPool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        nthreads_ = (int)std::min(12u, std::max(1u, hw * 3 / 4));
        if (const char *e = std::getenv("MDG_ADD_THREADS"))  // tuning override
            nthreads_ = std::max(1, std::min(64, std::atoi(e)));
        for (int t = 1; t < nthreads_; ++t) workers_.emplace_back([this, t] { loop(t); });
    }
    ~AddPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto &w : workers_) w.join();
    }
    // dst[r*stride + i] += src[r*stride + i] for r < rows, i < m
    void add(float *dst, const float *src, int64_t m, int rows, int64_t stride) {
        dst_ = dst;
        src_ = src;
        m_ = m;
        rows_ = rows;
        stride_ = stride;
        if (m * rows < (1 << 18) || nthreads_ == 1) {
            span(0, m * rows);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(mu_);
            pending_ = nthreads_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        slice(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [this] { return pending_ == 0; });
    }

  private:
    // flat element range [a, b) of the rows x m job
    void span(int64_t a, int64_t b) {
        while (a < b) {
            const int64_t r = a / m_, i0 = a - r * m_;
            const int64_t i1 = std::min<int64_t>(m_, i0 + (b - a));
            float *d = dst_ + r * stride_;
            const float *sp = src_ + r * stride_;
            for (int64_t i = i0; i < i1; ++i) d[i] += sp[i];
            a += i1 - i0;
        }
    }
    void slice(int t) {
        const int64_t tot = m_ * rows_;
        span(tot * t / nthreads_, tot * (t + 1) / nthreads_);
    }
    void loop(int t) {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
            }
            slice(t);
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (--pending_ == 0) done_.notify_one();
            }
        }
    }
    int nthreads_ = 1;
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    uint64_t gen_ = 0;
    int pending_ = 0;
    bool stop_ = false;
    float *dst_ = nullptr;
    const float *src_ = nullptr;
    int64_t m_ = 0, stride_ = 0;
    int rows_ = 1;
};

AddPool &add_pool() {
    static AddPool pool;
    return pool;
}
// dst[r*stride + i] += src[r*stride + i]  (one fp32 add per element)
void host_add_rows(float *dst, const float *src, int64_t m, int rows, int64_t stride) {
    add_pool().add(dst, src, m, rows, stride);
}
void host_add(float *dst, const float *src, int64_t m) { host_add_rows(dst, src, m, 1, 0); }

constexpr int kPipeMinPlanes = 16;       // below this the plain call wins
constexpr int64_t kPipeMinVoxels = 1 << 20;
constexpr int kPipeChunks = 16;

bool pipeline_ok(mdg_dims3 d, int nb, int layout, bool all_ptrs) {
    return all_ptrs && nb == 3 && dims_ok(d) && d.l >= kPipeMinPlanes &&
           nvox(d) >= kPipeMinVoxels && (layout == MDG_QK_PLANAR || layout == MDG_QK_POSMAJOR);
}

// posmajor host chunk {m, C} (staged) -> interior of an extended planar
// buffer {C, m + 2hw} at offset hw, and back
__global__ void pm_to_ext_k(const float *__restrict__ src, int64_t m, int C, int64_t hw,
                            float *__restrict__ dst) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m * C) return;
    const int64_t p = i / C;
    const int c = (int)(i - p * C);
    dst[(int64_t)c * (m + 2 * hw) + hw + p] = src[i];
}
__global__ void ext_to_pm_k(const float *__restrict__ src, int64_t m, int C, int64_t hw,
                            float *__restrict__ dst) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m * C) return;
    const int64_t p = i / C;
    const int c = (int)(i - p * C);
    dst[i] = src[(int64_t)c * (m + 2 * hw) + hw + p];
}

struct Chunking {
    int nchunk;
    std::vector<int> z0, z1;
    explicit Chunking(int l) {
        nchunk = std::min(kPipeChunks, l / 4);
        for (int i = 0; i < nchunk; ++i) {
            z0.push_back((int)((int64_t)l * i / nchunk));
            z1.push_back((int)((int64_t)l * (i + 1) / nchunk));
        }
    }
    int depth(int i) const { return z1[i] - z0[i]; }
};

// One channel-major array staged chunk by chunk as extended volumes.
struct ExtArray {
    int C = 0;
    int64_t hw = 0, n = 0;
    bool posmajor = false;  // host layout {n, C}
    std::vector<float *> buf;  // per chunk {C, (D+2) hw}
    std::vector<float *> stg;  // posmajor host layout: per-chunk staging

    int64_t ext(const Chunking &ck, int i) const { return (int64_t)(ck.depth(i) + 2) * hw; }
};

// Per-thread device workspace for the pipeline: a list of blocks handed out by
// a bump cursor that is rewound at the start of every call.  Every call
// drains its streams before returning, so the next call may reuse the memory;
// after the first calls no allocation happens at all (stream-ordered pool
// allocations across three streams would keep growing the pool instead).
struct DevArena {
    struct Block {
        char *p;
        size_t size;
    };
    std::vector<Block> blocks;
    size_t bi = 0, off = 0;
    ~DevArena() {
        for (auto &b : blocks) cudaFree(b.p);
    }
    void rewind() { bi = off = 0; }
    cudaError_t take(void **out, size_t bytes) {
        bytes = (bytes + 255) / 256 * 256;
        while (bi < blocks.size() && off + bytes > blocks[bi].size) {
            ++bi;
            off = 0;
        }
        if (bi == blocks.size()) {
            Block b{nullptr, std::max(bytes, (size_t)256 << 20)};
            cudaError_t e = cudaMalloc(&b.p, b.size);
            if (e != cudaSuccess) return e;
            blocks.push_back(b);
            off = 0;
        }
        *out = blocks[bi].p + off;
        off += bytes;
        return cudaSuccess;
    }
};
DevArena &dev_arena() {
    thread_local DevArena a;
    return a;
}

struct PipeCtx {
    mdg_dims3 d;
    int64_t n, hw;
    Chunking ck;
    cudaStream_t up, comp, down;
    std::vector<cudaEvent_t> evs;
    PipeCtx(mdg_dims3 d_) : d(d_), n(nvox(d_)), hw((int64_t)d_.h * d_.w), ck(d_.l) {
        PipeStreams &ps = pipe_streams();
        up = ps.up;
        comp = ps.comp;
        down = ps.down;
        dev_arena().rewind();
        keep_pool_mapped();  // kernels' own scratch (cudaMallocAsync) stays mapped
    }
    ~PipeCtx() {
        // callers drain the streams before returning; make sure of it on the
        // error paths too before the workspace is handed to the next call
        cudaStreamSynchronize(up);
        cudaStreamSynchronize(comp);
        cudaStreamSynchronize(down);
        for (cudaEvent_t e : evs) cudaEventDestroy(e);
    }
    cudaError_t alloc(float **p, size_t floats) {
        void *q = nullptr;
        cudaError_t e = dev_arena().take(&q, floats * sizeof(float) + 16);
        if (e == cudaSuccess) *p = static_cast<float *>(q);
        return e;
    }
    cudaEvent_t event() {
        cudaEvent_t e = nullptr;
        cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        evs.push_back(e);
        return e;
    }
    cudaError_t init(ExtArray &a, int C, bool posmajor) {
        a.C = C;
        a.hw = hw;
        a.n = n;
        a.posmajor = posmajor;
        a.buf.resize(ck.nchunk);
        a.stg.assign(ck.nchunk, nullptr);
        for (int i = 0; i < ck.nchunk; ++i) {
            cudaError_t e = alloc(&a.buf[i], (size_t)C * a.ext(ck, i));
            if (e) return e;
            if (posmajor && (e = alloc(&a.stg[i], (size_t)C * ck.depth(i) * hw))) return e;
        }
        return cudaSuccess;
    }
    // H2D of chunk i's planes into the interior (on `up`)
    cudaError_t upload(ExtArray &a, const float *host, int i) {
        const int D = ck.depth(i);
        const int64_t m = (int64_t)D * hw;
        if (a.posmajor) {
            cudaError_t e = cudaMemcpyAsync(a.stg[i], host + (int64_t)ck.z0[i] * hw * a.C,
                                            (size_t)m * a.C * sizeof(float),
                                            cudaMemcpyHostToDevice, up);
            if (e) return e;
            pm_to_ext_k<<<grid1d(m * a.C, 256), 256, 0, up>>>(a.stg[i], m, a.C, hw, a.buf[i]);
            return cudaPeekAtLastError();
        }
        return cudaMemcpy2DAsync(a.buf[i] + hw, (size_t)a.ext(ck, i) * sizeof(float),
                                 host + (int64_t)ck.z0[i] * hw, (size_t)n * sizeof(float),
                                 (size_t)m * sizeof(float), a.C, cudaMemcpyHostToDevice, up);
    }
    // D2H of chunk i's interior (on `down`)
    cudaError_t download(ExtArray &a, float *host, int i) {
        const int D = ck.depth(i);
        const int64_t m = (int64_t)D * hw;
        if (a.posmajor) {
            ext_to_pm_k<<<grid1d(m * a.C, 256), 256, 0, down>>>(a.buf[i], m, a.C, hw, a.stg[i]);
            cudaError_t e = cudaPeekAtLastError();
            if (e) return e;
            return cudaMemcpyAsync(host + (int64_t)ck.z0[i] * hw * a.C, a.stg[i],
                                   (size_t)m * a.C * sizeof(float), cudaMemcpyDeviceToHost, down);
        }
        return cudaMemcpy2DAsync(host + (int64_t)ck.z0[i] * hw, (size_t)n * sizeof(float),
                                 a.buf[i] + hw, (size_t)a.ext(ck, i) * sizeof(float),
                                 (size_t)m * sizeof(float), a.C, cudaMemcpyDeviceToHost, down);
    }
    // host += staged chunk i of `a` (staging mirrors the host array's layout)
    void add_chunk(const ExtArray &a, float *host, const float *stage, int i) const {
        const int64_t m = (int64_t)ck.depth(i) * hw;
        if (a.posmajor) {
            const int64_t o = (int64_t)ck.z0[i] * hw * a.C;
            host_add(host + o, stage + o, m * a.C);
        } else {
            const int64_t o = (int64_t)ck.z0[i] * hw;
            host_add_rows(host + o, stage + o, m, a.C, n);
        }
    }
    // halo planes of chunk i from its neighbours' interiors (or `fill` at the
    // global boundary); on `comp`, after both neighbours are uploaded
    cudaError_t halos(ExtArray &a, int i, float fill, bool zero) {
        const int D = ck.depth(i);
        const size_t pl = (size_t)hw * sizeof(float), pitch = (size_t)a.ext(ck, i) * sizeof(float);
        for (int side = 0; side < 2; ++side) {
            float *dst = a.buf[i] + (side == 0 ? 0 : (int64_t)(D + 1) * hw);
            const int nb = side == 0 ? i - 1 : i + 1;
            if (zero || nb < 0 || nb >= ck.nchunk) {
                if (fill == 0.0f) {
                    cudaError_t e = cudaMemset2DAsync(dst, pitch, 0, pl, a.C, comp);
                    if (e) return e;
                } else {
                    for (int c = 0; c < a.C; ++c)
                        fill_k<<<grid1d(hw, 256), 256, 0, comp>>>(dst + c * a.ext(ck, i), hw, fill);
                }
                continue;
            }
            const int Dn = ck.depth(nb);
            const float *src = a.buf[nb] + (side == 0 ? (int64_t)Dn * hw : hw);
            cudaError_t e = cudaMemcpy2DAsync(dst, pitch, src, (size_t)a.ext(ck, nb) * sizeof(float),
                                              pl, a.C, cudaMemcpyDeviceToDevice, comp);
            if (e) return e;
        }
        return cudaPeekAtLastError();
    }
};

#define MDG_PIPE_TRY(expr)                                             \
    do {                                                               \
        cudaError_t _e = (expr);                                       \
        if (_e != cudaSuccess) return status_from_cuda(_e, #expr);     \
    } while (0)
#define MDG_PIPE_OK(expr)                                              \
    do {                                                               \
        mdg_status _s = (expr);                                        \
        if (_s != MDG_OK) return _s;                                   \
    } while (0)

mdg_status modet_fwd_host_pipelined(const float *Q, const float *K, const float *B, mdg_dims3 d,
                                    int S, int hd, int layout, float *SF, float *LSE) {
    PipeCtx P(d);
    const int N = P.ck.nchunk, C = S * hd;
    const bool pm = layout == MDG_QK_POSMAJOR;
    ExtArray q, k, sf, lse;
    MDG_PIPE_TRY(P.init(q, C, pm));
    MDG_PIPE_TRY(P.init(k, C, pm));
    MDG_PIPE_TRY(P.init(sf, 3 * S, false));
    MDG_PIPE_TRY(P.init(lse, S, false));
    float *dB = nullptr;
    MDG_PIPE_TRY(P.alloc(&dB, (size_t)S * 27));
    MDG_PIPE_TRY(cudaMemcpyAsync(dB, B, (size_t)S * 27 * sizeof(float), cudaMemcpyHostToDevice, P.up));
    std::vector<cudaEvent_t> upd(N), cmp(N);
    for (int i = 0; i < N; ++i) {
        MDG_PIPE_TRY(P.upload(q, Q, i));
        MDG_PIPE_TRY(P.upload(k, K, i));
        upd[i] = P.event();
        MDG_PIPE_TRY(cudaEventRecord(upd[i], P.up));
    }
    for (int i = 0; i < N; ++i) {
        MDG_PIPE_TRY(cudaStreamWaitEvent(P.comp, upd[std::min(i + 1, N - 1)], 0));
        MDG_PIPE_TRY(P.halos(k, i, 0.0f, false));
        MDG_PIPE_TRY(P.halos(q, i, 0.0f, true));  // halo queries: the neighbour's work
        const mdg_dims3 de{d.h, d.w, P.ck.depth(i) + 2};
        MDG_PIPE_OK(mdg_modet_fwd(q.buf[i], k.buf[i], dB, de, S, hd, 3, MDG_QK_PLANAR,
                                  sf.buf[i], lse.buf[i], nullptr, P.comp));
        cmp[i] = P.event();
        MDG_PIPE_TRY(cudaEventRecord(cmp[i], P.comp));
        MDG_PIPE_TRY(cudaStreamWaitEvent(P.down, cmp[i], 0));
        MDG_PIPE_TRY(P.download(sf, SF, i));
        MDG_PIPE_TRY(P.download(lse, LSE, i));
    }
    MDG_PIPE_TRY(cudaStreamSynchronize(P.down));
    MDG_PIPE_TRY(cudaStreamSynchronize(P.comp));
    // any non-finite logit: the caller reruns whole-volume for the exact position
    unsigned long long *f = numeric_flag_ptr(P.comp);
    if (!f) return status_from_cuda(cudaErrorMemoryAllocation, "numeric flag");
    unsigned long long key = ~0ull;
    MDG_PIPE_TRY(cudaMemcpy(&key, f, sizeof(key), cudaMemcpyDeviceToHost));
    if (key != ~0ull) {
        MDG_PIPE_TRY(cudaMemset(f, 0xff, sizeof(key)));
        return MDG_ENUMERIC;
    }
    return MDG_OK;
}

mdg_status modet_bwd_host_pipelined(const float *Q, const float *K, const float *B,
                                    const float *SF, const float *LSE, const float *gSF,
                                    mdg_dims3 d, int S, int hd, int layout, float *gQ, float *gK,
                                    float *gB, bool acc) {
    const auto te = std::chrono::steady_clock::now();
    PipeCtx P(d);
    const int N = P.ck.nchunk, C = S * hd;
    const bool pm = layout == MDG_QK_POSMAJOR;
    ExtArray q, k, sf, lse, g, gq, gk;
    MDG_PIPE_TRY(P.init(q, C, pm));
    MDG_PIPE_TRY(P.init(k, C, pm));
    MDG_PIPE_TRY(P.init(sf, 3 * S, false));
    MDG_PIPE_TRY(P.init(lse, S, false));
    MDG_PIPE_TRY(P.init(g, 3 * S, false));
    MDG_PIPE_TRY(P.init(gq, C, pm));
    MDG_PIPE_TRY(P.init(gk, C, pm));
    // accumulate: contributions land in pinned staging and host threads add
    // them into the caller's arrays; overwrite: straight into the caller's
    // arrays (no host pass)
    PinnedStage &stg = pinned_stage();
    const size_t qn = (size_t)C * P.n;
    if (acc) MDG_PIPE_TRY(stg.reserve(2 * qn));
    float *sq = acc ? stg.p : gQ, *sk = acc ? stg.p + qn : gK;
    float *dB = nullptr, *dgB = nullptr;
    MDG_PIPE_TRY(P.alloc(&dB, (size_t)S * 27));
    MDG_PIPE_TRY(P.alloc(&dgB, (size_t)S * 27));
    MDG_PIPE_TRY(cudaMemcpyAsync(dB, B, (size_t)S * 27 * sizeof(float), cudaMemcpyHostToDevice, P.up));
    if (acc)
        MDG_PIPE_TRY(cudaMemcpyAsync(dgB, gB, (size_t)S * 27 * sizeof(float),
                                     cudaMemcpyHostToDevice, P.up));
    else
        MDG_PIPE_TRY(cudaMemsetAsync(dgB, 0, (size_t)S * 27 * sizeof(float), P.up));
    std::vector<cudaEvent_t> upd(N), cmp(N), dwn(N);
    for (int i = 0; i < N; ++i) {
        MDG_PIPE_TRY(P.upload(q, Q, i));
        MDG_PIPE_TRY(P.upload(k, K, i));
        MDG_PIPE_TRY(P.upload(sf, SF, i));
        MDG_PIPE_TRY(P.upload(lse, LSE, i));
        MDG_PIPE_TRY(P.upload(g, gSF, i));
        upd[i] = P.event();
        MDG_PIPE_TRY(cudaEventRecord(upd[i], P.up));
    }
    for (int i = 0; i < N; ++i) {
        MDG_PIPE_TRY(cudaStreamWaitEvent(P.comp, upd[std::min(i + 1, N - 1)], 0));
        const mdg_dims3 de{d.h, d.w, P.ck.depth(i) + 2};
        MDG_PIPE_TRY(P.halos(q, i, 0.0f, false));
        MDG_PIPE_TRY(P.halos(k, i, 0.0f, false));
        MDG_PIPE_TRY(P.halos(sf, i, 0.0f, false));
        MDG_PIPE_TRY(P.halos(lse, i, INFINITY, false));  // phantom sources weigh 0
        // queries (dQ, dB): halo queries belong to the neighbouring chunk
        MDG_PIPE_TRY(P.halos(g, i, 0.0f, true));
        MDG_PIPE_OK(mdg_modet_bwd(q.buf[i], k.buf[i], dB, sf.buf[i], lse.buf[i], g.buf[i], de, S,
                                  hd, 3, MDG_QK_PLANAR, gq.buf[i], nullptr, dgB, 0, P.comp));
        // keys (dK): sources in the halo planes count
        MDG_PIPE_TRY(P.halos(g, i, 0.0f, false));
        MDG_PIPE_OK(mdg_modet_bwd(q.buf[i], k.buf[i], dB, sf.buf[i], lse.buf[i], g.buf[i], de, S,
                                  hd, 3, MDG_QK_PLANAR, nullptr, gk.buf[i], nullptr, 0, P.comp));
        cmp[i] = P.event();
        MDG_PIPE_TRY(cudaEventRecord(cmp[i], P.comp));
        MDG_PIPE_TRY(cudaStreamWaitEvent(P.down, cmp[i], 0));
        MDG_PIPE_TRY(P.download(gq, sq, i));
        MDG_PIPE_TRY(P.download(gk, sk, i));
        dwn[i] = P.event();
        MDG_PIPE_TRY(cudaEventRecord(dwn[i], P.down));
    }
    MDG_PIPE_TRY(cudaMemcpyAsync(gB, dgB, (size_t)S * 27 * sizeof(float), cudaMemcpyDeviceToHost, P.down));
    const bool trace = getenv("MDG_PIPE_TRACE") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    auto ms = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); };
    double t_wait = 0, t_add = 0;
    for (int i = 0; i < N; ++i) {  // host adds overlap the chunks still in flight
        const double a0 = ms();
        MDG_PIPE_TRY(cudaEventSynchronize(dwn[i]));
        const double a1 = ms();
        if (acc) {
            P.add_chunk(gq, gQ, sq, i);
            P.add_chunk(gk, gK, sk, i);
        }
        t_wait += a1 - a0;
        t_add += ms() - a1;
    }
    if (trace)
        fprintf(stderr, "modet_bwd_host pipeline: enqueue %.2f ms, adds %.2f ms, waits %.2f ms\n",
                std::chrono::duration<double, std::milli>(t0 - te).count(), t_add, t_wait);
    MDG_PIPE_TRY(cudaStreamSynchronize(P.down));
    MDG_PIPE_TRY(cudaStreamSynchronize(P.comp));
    return MDG_OK;
}

// ---------------------------------------------------------- warp pipelines
// The warp's gather (and its backward's scatter) reach is data-dependent, so
// the field is uploaded first and a device pass computes, per z-chunk, the
// exact range of z rows its samples can touch: every corner row is a clamped
// floor(z + phi_z) or that + 1 (resolve_axis), and clamping is monotone, so
// [clamp(floor(min)), clamp(floor(max) + 1)] over the chunk bounds them (any
// non-finite coordinate widens it to the whole volume).  The input then
// streams chunk by chunk and chunk i computes as soon as the rows it reaches
// have arrived; the scattered input gradient is downloaded row-chunk by
// row-chunk as soon as no later chunk can reach it.  Same kernels, same
// per-voxel arithmetic as the whole-volume call: results are identical.
__global__ void __launch_bounds__(256)
reach_k(const float *__restrict__ fz, int h, int w, int l, const int *__restrict__ z0s,
        const int *__restrict__ z1s, int *__restrict__ lo, int *__restrict__ hi) {
    const int i = blockIdx.y;
    const int hw = h * w, pb = z0s[i] * hw, pe = z1s[i] * hw;
    int a = INT_MAX, b = INT_MIN;
    for (int p = pb + blockIdx.x * 256 + threadIdx.x; p < pe; p += gridDim.x * 256) {
        const float zs = __fadd_rn((float)(p / hw), fz[p]);
        if (!isfinite(zs)) {
            a = 0;
            b = l - 1;
        } else {
            const int r = (int)floorf(fminf(fmaxf(zs, -2.0f), (float)l + 1.0f));
            a = min(a, r);
            b = max(b, r + 1);
        }
    }
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) {
        a = min(a, __shfl_xor_sync(0xffffffffu, a, m));
        b = max(b, __shfl_xor_sync(0xffffffffu, b, m));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&lo[i], a);
        atomicMax(&hi[i], b);
    }
}

struct Reach {
    std::vector<int> lo, hi;     // touched z rows per chunk (clamped)
    std::vector<int> need;       // last input chunk chunk i reads
    std::vector<int> last;       // last compute chunk that can reach row chunk j
};

// field (all chunks, on `up`) -> reach on `comp` -> host; the caller keeps
// enqueueing uploads on `up` while this waits.  `dz` = device z plane of phi.
static cudaError_t reach_enqueue(PipeCtx &P, const float *dz, int *dbuf, int *hbuf) {
    const int N = P.ck.nchunk;
    cudaError_t e = cudaMemcpyAsync(dbuf + 2 * N, P.ck.z0.data(), N * sizeof(int),
                                    cudaMemcpyHostToDevice, P.comp);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(dbuf + 3 * N, P.ck.z1.data(), N * sizeof(int), cudaMemcpyHostToDevice,
                            P.comp);
    if (e == cudaSuccess) e = cudaMemsetAsync(dbuf, 0x7f, N * sizeof(int), P.comp);
    if (e == cudaSuccess) e = cudaMemsetAsync(dbuf + N, 0x80, N * sizeof(int), P.comp);
    if (e != cudaSuccess) return e;
    reach_k<<<dim3(32, N), 256, 0, P.comp>>>(dz, P.d.h, P.d.w, P.d.l, dbuf + 2 * N, dbuf + 3 * N,
                                            dbuf, dbuf + N);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if ((e = cudaPeekAtLastError()) != cudaSuccess) return e;
    return cudaMemcpyAsync(hbuf, dbuf, 2 * N * sizeof(int), cudaMemcpyDeviceToHost, P.comp);
}

static Reach reach_decode(const PipeCtx &P, const int *hbuf) {
    const int N = P.ck.nchunk, l = P.d.l;
    Reach r;
    r.lo.resize(N);
    r.hi.resize(N);
    r.need.resize(N);
    r.last.assign(N, -1);
    auto chunk_of = [&](int z) {
        int c = 0;
        while (c + 1 < N && P.ck.z0[c + 1] <= z) ++c;
        return c;
    };
    for (int i = 0; i < N; ++i) {
        r.lo[i] = std::max(0, std::min(hbuf[i], l - 1));
        r.hi[i] = std::min(l - 1, std::max(hbuf[N + i], 0));
        if (r.hi[i] < r.lo[i]) r.hi[i] = r.lo[i];
        // inputs arrive in z order; also wait for chunk i's own rows (gout)
        r.need[i] = std::max(chunk_of(r.hi[i]), i);
        for (int j = chunk_of(r.lo[i]); j <= chunk_of(r.hi[i]); ++j) r.last[j] = std::max(r.last[j], i);
    }
    return r;
}

mdg_status warp_fwd_host_pipelined(const float *in, int C, mdg_dims3 d, const float *field,
                                   float *out) {
    PipeCtx P(d);
    const int N = P.ck.nchunk;
    const int64_t n = P.n, hw = P.hw;
    const size_t pitch = (size_t)n * sizeof(float);
    float *di, *df, *dout, *dr;
    MDG_PIPE_TRY(P.alloc(&di, (size_t)C * n));
    MDG_PIPE_TRY(P.alloc(&df, 3 * (size_t)n));
    MDG_PIPE_TRY(P.alloc(&dout, (size_t)C * n));
    MDG_PIPE_TRY(P.alloc(&dr, 4 * (size_t)N));
    PinnedStage &stg = pinned_stage();
    MDG_PIPE_TRY(stg.reserve(2 * (size_t)N));
    int *hr = reinterpret_cast<int *>(stg.p);
    MDG_PIPE_TRY(cudaMemcpyAsync(df, field, 3 * pitch, cudaMemcpyHostToDevice, P.up));
    cudaEvent_t fev = P.event();
    MDG_PIPE_TRY(cudaEventRecord(fev, P.up));
    MDG_PIPE_TRY(cudaStreamWaitEvent(P.comp, fev, 0));
    MDG_PIPE_TRY(reach_enqueue(P, df + 2 * n, reinterpret_cast<int *>(dr), hr));
    cudaEvent_t rev = P.event();
    MDG_PIPE_TRY(cudaEventRecord(rev, P.comp));
    std::vector<cudaEvent_t> upd(N);
    for (int i = 0; i < N; ++i) {
        const int64_t p0 = (int64_t)P.ck.z0[i] * hw, m = (int64_t)P.ck.depth(i) * hw;
        MDG_PIPE_TRY(cudaMemcpy2DAsync(di + p0, pitch, in + p0, pitch, m * sizeof(float), C,
                                       cudaMemcpyHostToDevice, P.up));
        upd[i] = P.event();
        MDG_PIPE_TRY(cudaEventRecord(upd[i], P.up));
    }
    MDG_PIPE_TRY(cudaEventSynchronize(rev));
    const Reach R = reach_decode(P, hr);
    for (int i = 0; i < N; ++i) {
        const int64_t p0 = (int64_t)P.ck.z0[i] * hw, m = (int64_t)P.ck.depth(i) * hw;
        MDG_PIPE_TRY(cudaStreamWaitEvent(P.comp, upd[R.need[i]], 0));
        MDG_PIPE_OK(warp_fwd_range(di, C, d, df, dout, p0, p0 + m, P.comp));
        cudaEvent_t ce = P.event();
        MDG_PIPE_TRY(cudaEventRecord(ce, P.comp));
        MDG_PIPE_TRY(cudaStreamWaitEvent(P.down, ce, 0));
        MDG_PIPE_TRY(cudaMemcpy2DAsync(out + p0, pitch, dout + p0, pitch, m * sizeof(float), C,
                                       cudaMemcpyDeviceToHost, P.down));
    }
    MDG_PIPE_TRY(cudaStreamSynchronize(P.down));
    return MDG_OK;
}

mdg_status warp_bwd_host_pipelined(const float *in, int C, mdg_dims3 d, const float *field,
                                   const float *gout, float *gin, float *gfield) {
    const auto te = std::chrono::steady_clock::now();
    auto since = [&] {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - te)
            .count();
    };
    PipeCtx P(d);
    const int N = P.ck.nchunk;
    const int64_t n = P.n, hw = P.hw;
    const size_t pitch = (size_t)n * sizeof(float);
    float *di, *df, *dg, *dgi = nullptr, *dgf = nullptr, *dr;
    MDG_PIPE_TRY(P.alloc(&di, (size_t)C * n));
    MDG_PIPE_TRY(P.alloc(&df, 3 * (size_t)n));
    MDG_PIPE_TRY(P.alloc(&dg, (size_t)C * n));
    MDG_PIPE_TRY(P.alloc(&dr, 4 * (size_t)N));
    if (gin) MDG_PIPE_TRY(P.alloc(&dgi, (size_t)C * n));
    if (gfield) MDG_PIPE_TRY(P.alloc(&dgf, 3 * (size_t)n));
    PinnedStage &stg = pinned_stage();
    MDG_PIPE_TRY(stg.reserve((size_t)(C + 3) * n + 2 * (size_t)N));
    float *si = stg.p, *sf = stg.p + (size_t)C * n;
    int *hr = reinterpret_cast<int *>(stg.p + (size_t)(C + 3) * n);
    // fresh contributions (the caller's accumulators stay on the host)
    if (dgi) MDG_PIPE_TRY(cudaMemsetAsync(dgi, 0, (size_t)C * n * sizeof(float), P.comp));
    if (dgf) MDG_PIPE_TRY(cudaMemsetAsync(dgf, 0, 3 * (size_t)n * sizeof(float), P.comp));
    MDG_PIPE_TRY(cudaMemcpyAsync(df, field, 3 * pitch, cudaMemcpyHostToDevice, P.up));
    cudaEvent_t fev = P.event();
    MDG_PIPE_TRY(cudaEventRecord(fev, P.up));
    MDG_PIPE_TRY(cudaStreamWaitEvent(P.comp, fev, 0));
    MDG_PIPE_TRY(reach_enqueue(P, df + 2 * n, reinterpret_cast<int *>(dr), hr));
    cudaEvent_t rev = P.event();
    MDG_PIPE_TRY(cudaEventRecord(rev, P.comp));
    std::vector<cudaEvent_t> upd(N), fdw(N), gdw(N, nullptr);
    for (int i = 0; i < N; ++i) {
        const int64_t p0 = (int64_t)P.ck.z0[i] * hw, m = (int64_t)P.ck.depth(i) * hw;
        MDG_PIPE_TRY(cudaMemcpy2DAsync(di + p0, pitch, in + p0, pitch, m * sizeof(float), C,
                                       cudaMemcpyHostToDevice, P.up));
        MDG_PIPE_TRY(cudaMemcpy2DAsync(dg + p0, pitch, gout + p0, pitch, m * sizeof(float), C,
                                       cudaMemcpyHostToDevice, P.up));
        upd[i] = P.event();
        MDG_PIPE_TRY(cudaEventRecord(upd[i], P.up));
    }
    const double t_enq_up = since();
    MDG_PIPE_TRY(cudaEventSynchronize(rev));
    const double t_reach = since();
    const Reach R = reach_decode(P, hr);
    std::vector<std::vector<int>> gin_after(N);  // row chunks final after compute i
    for (int j = 0; j < N; ++j) gin_after[std::max(R.last[j], 0)].push_back(j);
    for (int i = 0; i < N; ++i) {
        const int64_t p0 = (int64_t)P.ck.z0[i] * hw, m = (int64_t)P.ck.depth(i) * hw;
        MDG_PIPE_TRY(cudaStreamWaitEvent(P.comp, upd[R.need[i]], 0));
        MDG_PIPE_OK(warp_bwd_range(di, C, d, df, dg, dgi, dgf, p0, p0 + m, P.comp));
        cudaEvent_t ce = P.event();
        MDG_PIPE_TRY(cudaEventRecord(ce, P.comp));
        MDG_PIPE_TRY(cudaStreamWaitEvent(P.down, ce, 0));
        if (dgf)
            MDG_PIPE_TRY(cudaMemcpy2DAsync(sf + p0, pitch, dgf + p0, pitch, m * sizeof(float), 3,
                                           cudaMemcpyDeviceToHost, P.down));
        fdw[i] = P.event();
        MDG_PIPE_TRY(cudaEventRecord(fdw[i], P.down));
        for (int j : gin_after[i]) {
            const int64_t q0 = (int64_t)P.ck.z0[j] * hw, mq = (int64_t)P.ck.depth(j) * hw;
            if (dgi)
                MDG_PIPE_TRY(cudaMemcpy2DAsync(si + q0, pitch, dgi + q0, pitch, mq * sizeof(float),
                                               C, cudaMemcpyDeviceToHost, P.down));
            gdw[j] = P.event();
            MDG_PIPE_TRY(cudaEventRecord(gdw[j], P.down));
        }
    }
    // host adds in download order
    const double t_enq = since();
    double t_wait = 0.0, t_add = 0.0;
    for (int i = 0; i < N; ++i) {
        const int64_t p0 = (int64_t)P.ck.z0[i] * hw, m = (int64_t)P.ck.depth(i) * hw;
        double a0 = since();
        MDG_PIPE_TRY(cudaEventSynchronize(fdw[i]));
        double a1 = since();
        t_wait += a1 - a0;
        if (gfield) host_add_rows(gfield + p0, sf + p0, m, 3, n);
        t_add += since() - a1;
        for (int j : gin_after[i]) {
            const int64_t q0 = (int64_t)P.ck.z0[j] * hw, mq = (int64_t)P.ck.depth(j) * hw;
            a0 = since();
            MDG_PIPE_TRY(cudaEventSynchronize(gdw[j]));
            a1 = since();
            t_wait += a1 - a0;
            if (gin) host_add_rows(gin + q0, si + q0, mq, C, n);
            t_add += since() - a1;
        }
    }
    MDG_PIPE_TRY(cudaStreamSynchronize(P.down));
    if (getenv("MDG_PIPE_TRACE"))
        fprintf(stderr,
                "warp_bwd_host pipeline: uploads enqueued %.2f, reach known %.2f, all enqueued "
                "%.2f, waits %.2f, adds %.2f, total %.2f ms\n",
                t_enq_up, t_reach, t_enq, t_wait, t_add, since());
    return MDG_OK;
}

}  // namespace
}  // namespace mdg

extern "C" {

mdg_status mdg_na_fused_fwd_host(const float *Q, const float *K, const float *B, mdg_dims3 d,
                                 int S, int hd, int nb, float *W) {
    MDG_REQUIRE(dims_ok(d) && S >= 1 && hd >= 1, "na_fused_fwd: invalid sizes");
    const size_t n = (size_t)nvox(d), win = (size_t)nb * nb * nb;
    if (n == 0) return MDG_OK;
    cudaStream_t st = host_stream();
    Stage sg(st);
    float *dQ, *dK, *dB, *dW;
    MDG_STAGE_TRY(sg.get(&dQ, Q, n * S * hd, true));
    MDG_STAGE_TRY(sg.get(&dK, K, n * S * hd, true));
    MDG_STAGE_TRY(sg.get(&dB, B, (size_t)S * win, true));
    MDG_STAGE_TRY(sg.get(&dW, W, (size_t)S * n * win, false));
    mdg_status r = mdg_na_fused_fwd(dQ, dK, dB, d, S, hd, nb, dW, st);
    if (r != MDG_OK) return r;
    MDG_STAGE_TRY(sg.down(W, dW, (size_t)S * n * win));
    MDG_STAGE_TRY(cudaStreamSynchronize(st));
    return MDG_OK;
}

// The remaining reference kern:: entry points as host-buffer calls (the
// drop-in binding of integration/mdreg_b200.hpp): inputs up, accumulate
// targets up (the reference's +=), outputs down, synchronous.
mdg_status mdg_na_fused_bwd_host(const float *Q, const float *K, const float *W, mdg_dims3 d,
                                 int S, int hd, int nb, const float *gW, float *gQ, float *gK,
                                 float *gB) {
    MDG_REQUIRE(dims_ok(d) && S >= 1 && hd >= 1, "na_fused_bwd: invalid sizes");
    const size_t n = (size_t)nvox(d), win = (size_t)nb * nb * nb;
    if (n == 0) return MDG_OK;
    cudaStream_t st = host_stream();
    Stage sg(st);
    float *dQ, *dK, *dW, *dgW, *dgQ, *dgK, *dgB;
    MDG_STAGE_TRY(sg.get(&dQ, Q, n * S * hd, true));
    MDG_STAGE_TRY(sg.get(&dK, K, n * S * hd, true));
    MDG_STAGE_TRY(sg.get(&dW, W, (size_t)S * n * win, true));
    MDG_STAGE_TRY(sg.get(&dgW, gW, (size_t)S * n * win, true));
    MDG_STAGE_TRY(sg.get(&dgQ, gQ, n * S * hd, true));
    MDG_STAGE_TRY(sg.get(&dgK, gK, n * S * hd, true));
    MDG_STAGE_TRY(sg.get(&dgB, gB, (size_t)S * win, true));
    mdg_status r = mdg_na_fused_bwd(dQ, dK, dW, d, S, hd, nb, dgW, dgQ, dgK, dgB, st);
    if (r != MDG_OK) return r;
    MDG_STAGE_TRY(sg.down(gQ, dgQ, n * S * hd));
    MDG_STAGE_TRY(sg.down(gK, dgK, n * S * hd));
    MDG_STAGE_TRY(sg.down(gB, dgB, (size_t)S * win));
    MDG_STAGE_TRY(cudaStreamSynchronize(st));
    return MDG_OK;
}

mdg_status mdg_subfields_fwd_host(const float *W, mdg_dims3 d, int S, int nb, float *out) {
    MDG_REQUIRE(dims_ok(d) && S >= 1, "subfields: invalid sizes");
    const size_t n = (size_t)nvox(d), win = (size_t)nb * nb * nb;
    if (n == 0) return MDG_OK;
    cudaStream_t st = host_stream();
    Stage sg(st);
    float *dW, *dout;
    MDG_STAGE_TRY(sg.get(&dW, W, (size_t)S * n * win, true));
    MDG_STAGE_TRY(sg.get(&dout, out, 3 * (size_t)S * n, false));
    mdg_status r = mdg_subfields_fwd(dW, d, S, nb, dout, st);
    if (r != MDG_OK) return r;
    MDG_STAGE_TRY(sg.down(out, dout, 3 * (size_t)S * n));
    MDG_STAGE_TRY(cudaStreamSynchronize(st));
    return MDG_OK;
}

mdg_status mdg_subfields_bwd_host(mdg_dims3 d, int S, int nb, const float *gout, float *gW) {
    MDG_REQUIRE(dims_ok(d) && S >= 1, "subfields: invalid sizes");
    const size_t n = (size_t)nvox(d), win = (size_t)nb * nb * nb;
    if (n == 0) return MDG_OK;
    cudaStream_t st = host_stream();
    Stage sg(st);
    float *dg, *dgW;
    MDG_STAGE_TRY(sg.get(&dg, gout, 3 * (size_t)S * n, true));
    MDG_STAGE_TRY(sg.get(&dgW, gW, (size_t)S * n * win, true));
    mdg_status r = mdg_subfields_bwd(d, S, nb, dg, dgW, st);
    if (r != MDG_OK) return r;
    MDG_STAGE_TRY(sg.down(gW, dgW, (size_t)S * n * win));
    MDG_STAGE_TRY(cudaStreamSynchronize(st));
    return MDG_OK;
}

mdg_status mdg_upsample2_fwd_host(const float *in, int C, mdg_dims3 d, mdg_dims3 td,
                                  float scale, float *out) {
    MDG_REQUIRE(dims_ok(d) && dims_ok(td) && C >= 0, "upsample: invalid sizes");
    const size_t ni = (size_t)nvox(d), no = (size_t)nvox(td);
    if (no == 0 || C == 0) return mdg_upsample2_fwd(nullptr, C, d, td, scale, nullptr, nullptr);
    cudaStream_t st = host_stream();
    Stage sg(st);
    float *di, *dout;
    MDG_STAGE_TRY(sg.get(&di, in, ni * C, true));
    MDG_STAGE_TRY(sg.get(&dout, out, no * C, false));
    mdg_status r = mdg_upsample2_fwd(di, C, d, td, scale, dout, st);
    if (r != MDG_OK) return r;
    MDG_STAGE_TRY(sg.down(out, dout, no * C));
    MDG_STAGE_TRY(cudaStreamSynchronize(st));
    return MDG_OK;
}

mdg_status mdg_upsample2_bwd_host(int C, mdg_dims3 d, mdg_dims3 td, float scale,
                                  const float *gout, float *gin) {
    MDG_REQUIRE(dims_ok(d) && dims_ok(td) && C >= 0, "upsample: invalid sizes");
    const size_t ni = (size_t)nvox(d), no = (size_t)nvox(td);
    if (ni == 0 || C == 0 || !gin) return mdg_upsample2_bwd(C, d, td, scale, nullptr, nullptr, nullptr);
    cudaStream_t st = host_stream();
    Stage sg(st);
    float *dg, *dgi;
    MDG_STAGE_TRY(sg.get(&dg, gout, no * C, true));
    MDG_STAGE_TRY(sg.get(&dgi, gin, ni * C, true));
    mdg_status r = mdg_upsample2_bwd(C, d, td, scale, dg, dgi, st);
    if (r != MDG_OK) return r;
    MDG_STAGE_TRY(sg.down(gin, dgi, ni * C));
    MDG_STAGE_TRY(cudaStreamSynchronize(st));
    return MDG_OK;
}

mdg_status mdg_conv3_fwd_host(const float *in, int ic, mdg_dims3 d, const float *k,
                              const float *bias, int oc, float *out) {
    MDG_REQUIRE(dims_ok(d) && ic >= 1 && oc >= 1, "conv3: invalid sizes");
    const size_t n = (size_t)nvox(d);
    if (n == 0) return MDG_OK;
    cudaStream_t st = host_stream();
    Stage sg(st);
    float *di, *dk, *db, *dout;
    MDG_STAGE_TRY(sg.get(&di, in, n * ic, true));
    MDG_STAGE_TRY(sg.get(&dk, k, (size_t)oc * ic * 27, true));
    MDG_STAGE_TRY(sg.get(&db, bias, (size_t)oc, true));
    MDG_STAGE_TRY(sg.get(&dout, out, n * oc, false));
    mdg_status r = mdg_conv3_fwd(di, ic, d, dk, db, oc, dout, st);
    if (r != MDG_OK) return r;
    MDG_STAGE_TRY(sg.down(out, dout, n * oc));
    MDG_STAGE_TRY(cudaStreamSynchronize(st));
    return MDG_OK;
}

mdg_status mdg_conv3_bwd_host(const float *in, int ic, mdg_dims3 d, const float *k, int oc,
                              const float *gout, float *gin, float *gk, float *gbias) {
    MDG_REQUIRE(dims_ok(d) && ic >= 1 && oc >= 1, "conv3: invalid sizes");
    const size_t n = (size_t)nvox(d);
    if (n == 0 || (!gin && !gk && !gbias)) return MDG_OK;
    cudaStream_t st = host_stream();
    Stage sg(st);
    float *di, *dk, *dg, *dgi, *dgk, *dgb;
    MDG_STAGE_TRY(sg.get(&di, in, n * ic, true));
    MDG_STAGE_TRY(sg.get(&dk, k, (size_t)oc * ic * 27, true));
    MDG_STAGE_TRY(sg.get(&dg, gout, n * oc, true));
    MDG_STAGE_TRY(sg.get(&dgi, gin, n * ic, true));
    MDG_STAGE_TRY(sg.get(&dgk, gk, (size_t)oc * ic * 27, true));
    MDG_STAGE_TRY(sg.get(&dgb, gbias, (size_t)oc, true));
    mdg_status r = mdg_conv3_bwd(di, ic, d, dk, oc, dg, dgi, dgk, dgb, st);
    if (r != MDG_OK) return r;
    MDG_STAGE_TRY(sg.down(gin, dgi, n * ic));
    MDG_STAGE_TRY(sg.down(gk, dgk, (size_t)oc * ic * 27));
    MDG_STAGE_TRY(sg.down(gbias, dgb, (size_t)oc));
    MDG_STAGE_TRY(cudaStreamSynchronize(st));
    return MDG_OK;
}

static mdg_status modet_fwd_host_whole(const float *Q, const float *K, const float *B,
                                       mdg_dims3 d, int S, int hd, int nb, int layout, float *SF,
                                       float *LSE) {
    MDG_REQUIRE(dims_ok(d) && S >= 1 && hd >= 1, "modet: invalid sizes");
    const size_t n = (size_t)nvox(d);
    if (n == 0) return MDG_OK;
    cudaStream_t st = host_stream();
    Stage sg(st);
    float *dQ, *dK, *dB, *dSF, *dL;
    MDG_STAGE_TRY(sg.get(&dQ, Q, n * S * hd, true));
    MDG_STAGE_TRY(sg.get(&dK, K, n * S * hd, true));
    MDG_STAGE_TRY(sg.get(&dB, B, (size_t)S * 27, true));
    MDG_STAGE_TRY(sg.get(&dSF, SF, 3 * n * S, false));
    MDG_STAGE_TRY(sg.get(&dL, LSE, n * S, false));
    mdg_status r = mdg_modet_fwd(dQ, dK, dB, d, S, hd, nb, layout, dSF, dL, nullptr, st);
    if (r != MDG_OK) return r;
    MDG_STAGE_TRY(sg.down(SF, dSF, 3 * n * S));
    MDG_STAGE_TRY(sg.down(LSE, dL, n * S));
    return consume_numeric_flag(st, d);
}

static mdg_status modet_bwd_host_whole(const float *Q, const float *K, const float *B,
                                       const float *SF, const float *LSE, const float *gSF,
                                       mdg_dims3 d, int S, int hd, int nb, int layout, float *gQ,
                                       float *gK, float *gB, bool acc) {
    MDG_REQUIRE(dims_ok(d) && S >= 1 && hd >= 1, "modet: invalid sizes");
    const size_t n = (size_t)nvox(d);
    if (n == 0) return MDG_OK;
    cudaStream_t st = host_stream();
    Stage sg(st);
    float *dQ, *dK, *dB, *dSF, *dL, *dG, *dgQ, *dgK, *dgB;
    MDG_STAGE_TRY(sg.get(&dQ, Q, n * S * hd, true));
    MDG_STAGE_TRY(sg.get(&dK, K, n * S * hd, true));
    MDG_STAGE_TRY(sg.get(&dB, B, (size_t)S * 27, true));
    MDG_STAGE_TRY(sg.get(&dSF, SF, 3 * n * S, true));
    MDG_STAGE_TRY(sg.get(&dL, LSE, n * S, true));
    MDG_STAGE_TRY(sg.get(&dG, gSF, 3 * n * S, true));
    MDG_STAGE_TRY(sg.get(&dgQ, gQ, n * S * hd, acc));  // accumulate targets go up too
    MDG_STAGE_TRY(sg.get(&dgK, gK, n * S * hd, acc));
    MDG_STAGE_TRY(sg.get(&dgB, gB, (size_t)S * 27, acc));
    // the device call always adds into gB: with accumulate == 0 the caller's
    // gB is not uploaded, so start it from zero (as the pipelined path does)
    if (!acc && dgB) MDG_STAGE_TRY(cudaMemsetAsync(dgB, 0, (size_t)S * 27 * sizeof(float), st));
    mdg_status r = mdg_modet_bwd(dQ, dK, dB, dSF, dL, dG, d, S, hd, nb, layout, dgQ, dgK, dgB,
                                 acc ? 1 : 0, st);
    if (r != MDG_OK) return r;
    MDG_STAGE_TRY(sg.down(gQ, dgQ, n * S * hd));
    MDG_STAGE_TRY(sg.down(gK, dgK, n * S * hd));
    MDG_STAGE_TRY(sg.down(gB, dgB, (size_t)S * 27));
    MDG_STAGE_TRY(cudaStreamSynchronize(st));
    return MDG_OK;
}

mdg_status mdg_modet_fwd_host(const float *Q, const float *K, const float *B, mdg_dims3 d,
                              int S, int hd, int nb, int layout, float *SF, float *LSE) {
    if (pipeline_ok(d, nb, layout, Q && K && SF && LSE)) {
        mdg_status r = modet_fwd_host_pipelined(Q, K, B, d, S, hd, layout, SF, LSE);
        if (r != MDG_ENUMERIC) return r;
        // a non-finite logit: rerun whole-volume to report the reference's
        // first position exactly
    }
    return modet_fwd_host_whole(Q, K, B, d, S, hd, nb, layout, SF, LSE);
}

mdg_status mdg_modet_bwd_host(const float *Q, const float *K, const float *B, const float *SF,
                              const float *LSE, const float *gSF, mdg_dims3 d, int S, int hd,
                              int nb, int layout, float *gQ, float *gK, float *gB,
                              int accumulate) {
    if (pipeline_ok(d, nb, layout, Q && K && SF && LSE && gSF && gQ && gK && gB))
        return modet_bwd_host_pipelined(Q, K, B, SF, LSE, gSF, d, S, hd, layout, gQ, gK, gB,
                                        accumulate != 0);
    return modet_bwd_host_whole(Q, K, B, SF, LSE, gSF, d, S, hd, nb, layout, gQ, gK, gB,
                                accumulate != 0);
}

mdg_status mdg_warp_fwd_host(const float *in, int C, mdg_dims3 d, const float *field,
                             float *out) {
    MDG_REQUIRE(dims_ok(d) && C >= 0, "warp: invalid sizes");
    const size_t n = (size_t)nvox(d);
    if (n == 0 || C == 0) return MDG_OK;
    if (pipeline_ok(d, 3, MDG_QK_PLANAR, in && field && out))
        return warp_fwd_host_pipelined(in, C, d, field, out);
    cudaStream_t st = host_stream();
    Stage sg(st);
    float *di, *df, *dout;
    MDG_STAGE_TRY(sg.get(&di, in, n * C, true));
    MDG_STAGE_TRY(sg.get(&df, field, 3 * n, true));
    MDG_STAGE_TRY(sg.get(&dout, out, n * C, false));
    mdg_status r = mdg_warp_fwd(di, C, d, df, dout, st);
    if (r != MDG_OK) return r;
    MDG_STAGE_TRY(sg.down(out, dout, n * C));
    MDG_STAGE_TRY(cudaStreamSynchronize(st));
    return MDG_OK;
}

mdg_status mdg_warp_bwd_host(const float *in, int C, mdg_dims3 d, const float *field,
                             const float *gout, float *gin, float *gfield) {
    MDG_REQUIRE(dims_ok(d) && C >= 0, "warp: invalid sizes");
    const size_t n = (size_t)nvox(d);
    if (n == 0 || C == 0) return MDG_OK;
    if (pipeline_ok(d, 3, MDG_QK_PLANAR, in && field && gout && (gin || gfield)))
        return warp_bwd_host_pipelined(in, C, d, field, gout, gin, gfield);
    cudaStream_t st = host_stream();
    Stage sg(st);
    float *di, *df, *dg, *dgi, *dgf;
    MDG_STAGE_TRY(sg.get(&di, in, n * C, true));
    MDG_STAGE_TRY(sg.get(&df, field, 3 * n, true));
    MDG_STAGE_TRY(sg.get(&dg, gout, n * C, true));
    MDG_STAGE_TRY(sg.get(&dgi, gin, n * C, true));
    MDG_STAGE_TRY(sg.get(&dgf, gfield, 3 * n, true));
    mdg_status r = mdg_warp_bwd(di, C, d, df, dg, dgi, dgf, st);
    if (r != MDG_OK) return r;
    MDG_STAGE_TRY(sg.down(gin, dgi, n * C));
    MDG_STAGE_TRY(sg.down(gfield, dgf, 3 * n));
    MDG_STAGE_TRY(cudaStreamSynchronize(st));
    return MDG_OK;
}

}  // extern "C"
