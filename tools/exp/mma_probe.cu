// Throughput probe: legacy warp-level mma.sync (TF32 m16n8k8, BF16 m16n8k16)
// on sm_100a, registers only.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 mma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__global__ void probe(float *out, int iters) {
    float d[8][4] = {};
    unsigned a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
    for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(0.5f + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (KIND == 0)
                asm volatile(
                    "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, "
                    "{%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                    : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                    : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
            else
                asm volatile(
                    "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, "
                    "{%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                    : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                    : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
        }
    }
    float s = 0;
    for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float *out;
    cudaMalloc(&out, 148 * 64 * 1024 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int kind = 0; kind < 2; ++kind)
        for (int warps : {4, 8, 16}) {
            const int blocks = 148 * 4, threads = 32 * warps, iters = 2000;
            auto run = [&] {
                if (kind == 0) probe<0><<<blocks, threads>>>(out, iters);
                else probe<1><<<blocks, threads>>>(out, iters);
            };
            run();
            cudaEventRecord(e0);
            run();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double k = kind == 0 ? 8 : 16;
            const double flops = 2.0 * 16 * 8 * k * 8 * iters * (double)blocks * warps;
            printf("%s warps/blk %2d: %.1f TFLOP/s\n", kind == 0 ? "tf32 m16n8k8 " : "bf16 m16n8k16",
                   warps, flops / ms / 1e9);
        }
    return 0;
}
