// Can a cluster-launched grid (B) run while a small non-cluster grid (A),
// launched first on another stream, spins waiting for B's per-item flags?
// (the persistent polish-grid question).  Bounded spins.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void kA(const unsigned* flags, int T, unsigned* claimed, int* timeouts) {
    __shared__ int s_t;
    for (;;) {
        if (threadIdx.x == 0) s_t = (int)atomicAdd(claimed, 1u);
        __syncthreads();
        const int t = s_t;
        __syncthreads();
        if (t >= T) break;
        if (threadIdx.x == 0) {
            unsigned v, spins = 0;
            for (;;) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + t) : "memory");
                if (v) break;
                if (++spins > (1u << 22)) { atomicAdd(timeouts, 1); break; }
                __nanosleep(500);
            }
        }
        __syncthreads();
    }
}

__global__ void __cluster_dims__(8, 1, 1) kB(unsigned* flags, int iters) {
    float x = threadIdx.x;
    for (int i = 0; i < iters; ++i) x = x * 0.999f + 1e-3f;
    __syncthreads();
    if (threadIdx.x == 0 && (blockIdx.x % 8) == 0) {
        __threadfence();
        atomicAdd(flags + blockIdx.x / 8, x > -1.f ? 1u : 2u);
    }
}

int main() {
    const int T = 1000;
    unsigned *flags, *claimed;
    int* timeouts;
    cudaMalloc(&flags, T * 4); cudaMalloc(&claimed, 4); cudaMalloc(&timeouts, 4);
    cudaStream_t sa, sb;
    cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking);
    cudaFuncSetAttribute(kA, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    for (int grid : {32, 64}) {
        for (int smem : {0, 36 * 1024}) {
            cudaMemset(flags, 0, T * 4); cudaMemset(claimed, 0, 4); cudaMemset(timeouts, 0, 4);
            cudaDeviceSynchronize();
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a, sa);
            kA<<<grid, 128, smem, sa>>>(flags, T, claimed, timeouts);
            kB<<<T * 8, 128, 0, sb>>>(flags, 20000);
            cudaEventRecord(b, sa);
            cudaError_t e = cudaDeviceSynchronize();
            float ms = 0; cudaEventElapsedTime(&ms, a, b);
            int to = -1; cudaMemcpy(&to, timeouts, 4, cudaMemcpyDeviceToHost);
            printf("A grid %d smem %d: %s, A done after %.3f ms, A timeouts %d\n", grid, smem, cudaGetErrorString(e), ms, to);
        }
    }
    return 0;
}
