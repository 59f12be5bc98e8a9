// diversity.cu — the solution batch and its diversity score (
// PAPER §V-C, Table III).
//   k_select_topn: the best N of a target's polished seeds, in the order of
//     R27 (fine-converged first, then the ranking cost c of R14, then slot);
//     N = 1 is exactly k_select_best's choice.  One CTA per target, bitonic
//     sort of 64-bit keys (tier | cost bits | slot) in shared memory.
//   k_mmd: per target, the maximum mean discrepancy between two point sets
//     X [N][n], Y [N2][n] in joint space: biased V-statistic of MMD^2 with a
//     Gaussian RBF k(a, b) = exp(-|a - b|^2 / (2 h^2)), h = the median of the
//     pairwise distances over X u Y (median heuristic; R36).  The
//     P = (N+N2)(N+N2-1)/2 distances are bitonic-sorted in shared memory for
//     the median; the three kernel sums accumulate in fp64 (MMD^2 is a
//     difference of O(1) means, so fp32 sums would cancel).
#include "kin.cuh"

namespace hjcd {

__device__ __forceinline__ uint32_t cost_bits_d(float x) {
    if (!(x >= 0.f)) x = CUDART_INF_F;
    return __float_as_uint(x);
}

__global__ void __launch_bounds__(256)
k_select_topn(const __grid_constant__ DevRobot rb, const __grid_constant__ DevCfg c,
              const float* __restrict__ targets, const float* __restrict__ theta,
              const float* __restrict__ ep_all, const float* __restrict__ eo_all, int N,
              float* __restrict__ q_out, float* __restrict__ pos_err, float* __restrict__ ori_err,
              int32_t* __restrict__ idx_out, int32_t* __restrict__ status) {
    __shared__ unsigned long long keys[256];
    const int t = blockIdx.x;
    const int n = rb.n, B = c.B;
    const int used = c.copies * c.K;
    for (int b = threadIdx.x; b < 256; b += blockDim.x) {
        unsigned long long key = ~0ull;
        if (b < used) {
            const float pe = ep_all[(long long)t * B + b], oe = eo_all[(long long)t * B + b];
            const float cst = c.w_p * c.w_p * pe * pe + c.w_o * c.w_o * oe * oe;   // R14
            const unsigned long long tier = (pe < c.eps_p_fine && oe < c.eps_o_fine) ? 0ull : 1ull;   // R27
            key = (tier << 63) | ((unsigned long long)cost_bits_d(cst) << 32) | (unsigned)b;
        }
        keys[b] = key;
    }
    __syncthreads();
    for (int size = 2; size <= 256; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < 128; i += blockDim.x) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const unsigned long long a = keys[lo], bb = keys[hi];
                if ((a > bb) == up) { keys[lo] = bb; keys[hi] = a; }
            }
            __syncthreads();
        }
    }
    const float* t7 = targets + 7ll * t;
    const float w = t7[3], x = t7[4], y = t7[5], z = t7[6];
    const float nq = sqrtf(w * w + x * x + y * y + z * z);
    const bool valid = fabsf(nq - 1.f) <= 1e-3f && isfinite(nq) && isfinite(t7[0]) && isfinite(t7[1]) &&
                       isfinite(t7[2]);
    for (int e = threadIdx.x; e < N * n; e += blockDim.x) {
        const int i = e / n, j = e - i * n;
        const int bi = (int)(keys[i] & 0xffffffffu);
        q_out[((long long)t * N + i) * n + j] = valid ? theta[((long long)t * B + bi) * n + j] : 0.f;
    }
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int bi = (int)(keys[i] & 0xffffffffu);
        pos_err[(long long)t * N + i] = valid ? ep_all[(long long)t * B + bi] : CUDART_INF_F;
        ori_err[(long long)t * N + i] = valid ? eo_all[(long long)t * B + bi] : CUDART_INF_F;
        if (idx_out) idx_out[(long long)t * N + i] = valid ? bi : -1;
    }
    if (status && threadIdx.x == 0) {   // of the best entry, as hjcd_solve
        const int bi = (int)(keys[0] & 0xffffffffu);
        const float pe = ep_all[(long long)t * B + bi], oe = eo_all[(long long)t * B + bi];
        int32_t st;
        if (!valid) st = HJCD_TARGET_INVALID;
        else if (pe < c.eps_p_fine && oe < c.eps_o_fine) st = HJCD_TARGET_CONVERGED;
        else if (pe < c.succ_p && oe < c.succ_o) st = HJCD_TARGET_SUCCESS;
        else st = HJCD_TARGET_NOT_CONVERGED;
        status[t] = st;
    }
}

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    return s;
}

// dynamic smem: Z [(N+N2) * n] floats, then the sort buffer [Ppad] floats
__global__ void __launch_bounds__(512)
k_mmd(const float* __restrict__ X, int N, const float* __restrict__ Y, int N2, int n, int Ppad,
      float* __restrict__ mmd2_out, float* __restrict__ bw_out) {
    extern __shared__ float sm[];
    __shared__ double red[32];
    const int t = blockIdx.x;
    const int L = N + N2;
    float* Z = sm;
    float* D = sm + L * n;
    for (int e = threadIdx.x; e < L * n; e += blockDim.x) {
        const int i = e / n, j = e - i * n;
        Z[e] = i < N ? X[((long long)t * N + i) * n + j] : Y[((long long)t * N2 + (i - N)) * n + j];
    }
    __syncthreads();
    const int P = L * (L - 1) / 2;
    // pair p -> (i, j), i < j, row-major over i
    for (int p = threadIdx.x; p < Ppad; p += blockDim.x) {
        float d = CUDART_INF_F;
        if (p < P) {
            // invert p = i*L - i(i+1)/2 + (j - i - 1)
            int i = (int)((2.0 * L - 1.0 - sqrt((2.0 * L - 1.0) * (2.0 * L - 1.0) - 8.0 * p)) * 0.5);
            while (i > 0 && i * L - i * (i + 1) / 2 > p) --i;
            while ((i + 1) * L - (i + 1) * (i + 2) / 2 <= p) ++i;
            const int j = p - (i * L - i * (i + 1) / 2) + i + 1;
            float s = 0.f;
            for (int k = 0; k < n; ++k) {
                const float df = Z[i * n + k] - Z[j * n + k];
                s = fmaf(df, df, s);
            }
            d = sqrtf(s);
        }
        D[p] = d;
    }
    __syncthreads();
    for (int size = 2; size <= Ppad; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < (Ppad >> 1); i += blockDim.x) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const float a = D[lo], b = D[hi];
                if ((a > b) == up) { D[lo] = b; D[hi] = a; }
            }
            __syncthreads();
        }
    }
    // median (numpy convention: mean of the two middle values for even P)
    const float h = (P & 1) ? D[P / 2] : 0.5f * (D[P / 2 - 1] + D[P / 2]);
    const double g = (h > 0.f) ? 1.0 / (2.0 * (double)h * (double)h) : 0.0;
    double sxx = 0.0, syy = 0.0, sxy = 0.0;
    for (int p = threadIdx.x; p < L * L; p += blockDim.x) {
        const int i = p / L, j = p - i * L;
        double s = 0.0;
        for (int k = 0; k < n; ++k) {
            const double df = (double)Z[i * n + k] - (double)Z[j * n + k];
            s += df * df;
        }
        const double kv = (h > 0.f) ? exp(-s * g) : (s == 0.0 ? 1.0 : 0.0);
        if (i < N && j < N) sxx += kv;
        else if (i >= N && j >= N) syy += kv;
        else sxy += kv;   // both (x, y) and (y, x): counted twice, halved below
    }
    sxx = block_sum(sxx, red);
    syy = block_sum(syy, red);
    sxy = block_sum(sxy, red);
    if (threadIdx.x == 0) {
        const double m2 = sxx / ((double)N * N) + syy / ((double)N2 * N2) - sxy / ((double)N * N2);
        mmd2_out[t] = (float)m2;
        if (bw_out) bw_out[t] = h;
    }
}

cudaError_t launch_select_topn(const DevRobot& rb, const DevCfg& c, const float* targets, int T, const float* theta,
                               const float* ep_all, const float* eo_all, int N, float* q_out, float* pos_err,
                               float* ori_err, int32_t* idx, int32_t* status, cudaStream_t s) {
    k_select_topn<<<T, 256, 0, s>>>(rb, c, targets, theta, ep_all, eo_all, N, q_out, pos_err, ori_err, idx, status);
    return cudaGetLastError();
}

size_t mmd_smem_bytes(int N, int N2, int n, int* Ppad) {
    const int L = N + N2;
    const int P = L * (L - 1) / 2;
    int pp = 2;
    while (pp < P) pp <<= 1;
    *Ppad = pp;
    return (size_t)(L * n + pp) * sizeof(float);
}

cudaError_t launch_mmd(const float* X, int N, const float* Y, int N2, int n, int T, float* mmd2, float* bw,
                       cudaStream_t s) {
    int Ppad;
    const size_t smem = mmd_smem_bytes(N, N2, n, &Ppad);
    // N + N2 <= 256 keeps this <= 128 KB + 32 KB (the launch checks the opt-in limit)
    cudaError_t e = cudaFuncSetAttribute(k_mmd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_mmd<<<T, 512, smem, s>>>(X, N, Y, N2, n, Ppad, mmd2, bw);
    return cudaGetLastError();
}

}  // namespace hjcd
