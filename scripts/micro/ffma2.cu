// FFMA vs FFMA2 (fma.rn.f32x2, sm_100a) issue/throughput microbenchmark:
// same flop count, 8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r;
}
__device__ __forceinline__ void upk(unsigned long long r, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}

__global__ void k1(float* out, float m, float c, int iters) {
    float a[16];
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
    float m2 = m + threadIdx.x * 1e-9f, c2 = c;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], m2, c2);
    }
    float s = 0.f;
    for (int i = 0; i < 16; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k2(float* out, float m, float c, int iters) {
    unsigned long long a[8];
    for (int i = 0; i < 8; ++i) a[i] = pk(threadIdx.x * 1e-3f + 2 * i, threadIdx.x * 1e-3f + 2 * i + 1);
    const float mm = m + threadIdx.x * 1e-9f;
    const unsigned long long M = pk(mm, mm), Cc = pk(c, c);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(M), "l"(Cc));
    }
    float s = 0.f;
    for (int i = 0; i < 8; ++i) { float x, y; upk(a[i], x, y); s += x + y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float* d; cudaMalloc(&d, 148 * 8 * 256 * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        for (int v = 0; v < 2; ++v) {
            for (int bps : {2, 4, 8}) {
                cudaEventRecord(a);
                if (v == 0) k1<<<148 * bps, 256>>>(d, 0.999f, 1e-3f, iters);
                else k2<<<148 * bps, 256>>>(d, 0.999f, 1e-3f, iters);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                double flops = 2.0 * 16 * iters * 148.0 * bps * 256;
                if (rep) printf("%s blocks/SM=%d: %.3f ms, %.1f TFLOP/s\n", v ? "FFMA2" : "FFMA ", bps, ms, flops / ms / 1e9);
            }
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
