// select.cu — per-target selection kernels.
//   k_select_replicate: top-K of the M PO-CCD seeds by (cost, seed index) and
//     floor(B/K) replicas with Philox noise (Alg. 2 l.2-8; R14, R15).
//     One CTA per target; the M keys (order-preserving cost bits << 32 | index)
//     are bitonic-sorted in shared memory, which yields exactly the K rounds of
//     argmin-and-remove of Alg. 2 (ties -> lower index).
//   k_select_best: argmin over the B polished seeds (Alg. 2 l.9-10, R27: fine-
//     converged seeds first, then cost, then slot) with a warp-shuffle +
//     shared-memory reduction of 64-bit keys (tier | cost bits | slot).
//   k_fk: batched FK + Jacobian (Eqs. 1, 7), one thread per configuration.
//   k_pose_error64: fp64 pose error of given fp32 configurations (Eqs. 1, 4-5
//     on the fp64 chain), one thread per configuration: success decided in
//     fp64 from the returned theta, not from the solver's fp32 errors.
#include <type_traits>

#include "polish.cuh"

namespace hjcd {

__global__ void __launch_bounds__(512)
k_select_replicate(const __grid_constant__ DevRobot rb, const __grid_constant__ DevCfg c,
                   const float* __restrict__ cost, const float* __restrict__ theta, int Mpad,
                   float* __restrict__ seeds, int32_t* __restrict__ kept) {
    extern __shared__ unsigned long long keys[];
    const int t = blockIdx.x;
    const int K = c.K, B = c.B, n = rb.n;
    sort_stage1_keys(cost + (long long)t * c.M, c.M, Mpad, keys);
    if (kept)
        for (int r = threadIdx.x; r < K; r += blockDim.x) kept[(long long)t * K + r] = (int32_t)(keys[r] & 0xffffffffu);
    const uint32_t tid = (uint32_t)(c.tid_offset + t);
    const int used = c.copies * K;
    const int nb = (n + 3) / 4;   // one Philox block per 4 joints
    for (int e = threadIdx.x; e < B * nb; e += blockDim.x) {
        const int b = e / nb, blk = e - b * nb;
        float v[4] = {CUDART_NAN_F, CUDART_NAN_F, CUDART_NAN_F, CUDART_NAN_F};
        if (b < used) replica_block(rb, c, theta, keys, t, b, blk, tid, v);
        for (int q = 0; q < 4 && 4 * blk + q < n; ++q) seeds[((long long)t * B + b) * n + 4 * blk + q] = v[q];
    }
}

// T = float (hjcd_solve) or double (hjcd_solve_f64: the ranking key keeps fp32
// cost bits, the returned values are the fp64 ones)
template <class T>
__global__ void __launch_bounds__(128)
k_select_best(const __grid_constant__ DevRobot rb, const __grid_constant__ DevCfg c,
              const float* __restrict__ targets, const T* __restrict__ theta,
              const T* __restrict__ ep_all, const T* __restrict__ eo_all,
              T* __restrict__ q_out, T* __restrict__ pos_err, T* __restrict__ ori_err,
              int32_t* __restrict__ status) {
    __shared__ unsigned long long red[32];
    const int t = blockIdx.x;
    const int n = rb.n, B = c.B;
    const int used = c.copies * c.K;
    unsigned long long best = ~0ull;
    for (int b = threadIdx.x; b < used; b += blockDim.x) {
        const T pe = ep_all[(long long)t * B + b], oe = eo_all[(long long)t * B + b];
        const float cst = (float)(T(c.w_p) * T(c.w_p) * pe * pe + T(c.w_o) * T(c.w_o) * oe * oe);   // R14
        // R27: converged seeds first (bit 63), then cost, then slot
        const unsigned long long tier = (pe < T(c.eps_p_fine) && oe < T(c.eps_o_fine)) ? 0ull : 1ull;
        const unsigned long long key = (tier << 63) | ((unsigned long long)cost_bits(cst) << 32) | (unsigned)b;
        best = key < best ? key : best;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, best, off);
        best = o < best ? o : best;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) red[warp] = best;
    __syncthreads();
    if (warp == 0) {
        best = (lane < (int)(blockDim.x >> 5)) ? red[lane] : ~0ull;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const unsigned long long o = __shfl_xor_sync(0xffffffffu, best, off);
            best = o < best ? o : best;
        }
        if (lane == 0) red[0] = best;
    }
    __syncthreads();
    best = red[0];
    const int bi = (int)(best & 0xffffffffu);
    const float* t7 = targets + 7ll * t;
    const float w = t7[3], x = t7[4], y = t7[5], z = t7[6];
    const float nq = sqrtf(w * w + x * x + y * y + z * z);
    const bool valid = fabsf(nq - 1.f) <= 1e-3f && isfinite(nq) && isfinite(t7[0]) &&
                       isfinite(t7[1]) && isfinite(t7[2]);
    for (int j = threadIdx.x; j < n; j += blockDim.x)
        q_out[(long long)t * n + j] = valid ? theta[((long long)t * B + bi) * n + j] : T(0);
    if (threadIdx.x == 0) {
        const T pe = valid ? ep_all[(long long)t * B + bi] : T(CUDART_INF_F);
        const T oe = valid ? eo_all[(long long)t * B + bi] : T(CUDART_INF_F);
        pos_err[t] = pe;
        ori_err[t] = oe;
        int32_t s;
        if (!valid) s = HJCD_TARGET_INVALID;
        else if (pe < T(c.eps_p_fine) && oe < T(c.eps_o_fine)) s = HJCD_TARGET_CONVERGED;
        else if (pe < T(c.succ_p) && oe < T(c.succ_o)) s = HJCD_TARGET_SUCCESS;
        else s = HJCD_TARGET_NOT_CONVERGED;
        status[t] = s;
    }
}

// REV: the chain specialisation of the stage kernels (kin.cuh fk), so this entry
// point evaluates the same FK code path the solve does (K11 / K14); FAST: the
// SFU-sincos variant of PO-CCD (K5), else the polish stage's exact sincos
template <int NMAX, int REV, bool FAST>
__global__ void __launch_bounds__(128)
k_fk(const __grid_constant__ DevRobot rb, const float* __restrict__ q, int N, float* __restrict__ pose7,
     float* __restrict__ jac) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= N) return;
    const int n = rb.n;
    float th[NMAX];
#pragma unroll
    for (int j = 0; j < NMAX; ++j) th[j] = (j < n) ? q[(long long)s * n + j] : 0.f;
    float3 P[NMAX], Z[NMAX], pe;
    Quat qe;
    fk<NMAX, true, false, FAST, REV>(rb, th, P, Z, pe, qe);
    float* o = pose7 + 7ll * s;
    o[0] = pe.x; o[1] = pe.y; o[2] = pe.z;
    o[3] = qe.w; o[4] = qe.x; o[5] = qe.y; o[6] = qe.z;
    if (jac) {
        float* J = jac + 6ll * n * s;
#pragma unroll
        for (int j = 0; j < NMAX; ++j) {
            if (j < n) {
                float3 a, b;
                if (rb.j[j].type == HJCD_REVOLUTE) { a = cross3(Z[j], pe - P[j]); b = Z[j]; }
                else { a = Z[j]; b = f3(0.f, 0.f, 0.f); }
                J[0 * n + j] = a.x; J[1 * n + j] = a.y; J[2 * n + j] = a.z;
                J[3 * n + j] = b.x; J[4 * n + j] = b.y; J[5 * n + j] = b.z;
            }
        }
    }
}

template <int NMAX>
__global__ void __launch_bounds__(128)
k_pose_error64(const __grid_constant__ DevRobotT<double> rb, const float* __restrict__ q,
               const float* __restrict__ targets, int N, double* __restrict__ pos_err, double* __restrict__ ori_err) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= N) return;
    const int n = rb.n;
    double th[NMAX];
#pragma unroll
    for (int j = 0; j < NMAX; ++j) th[j] = (j < n) ? (double)q[(long long)s * n + j] : 0.0;
    const TargetT<double> tg = load_target<double>(targets + 7ll * s);
    const ResidT<double> r = eval_at<NMAX, false, 0>(rb, tg, th);
    pos_err[s] = tg.valid ? r.ep : CUDART_INF;
    ori_err[s] = tg.valid ? r.eo : CUDART_INF;
}

cudaError_t launch_pose_error64(const DevRobotT<double>& rb, const float* q, const float* targets, int N,
                                double* pos_err, double* ori_err, cudaStream_t s) {
    const int block = 128;
    const int grid = (N + block - 1) / block;
    if (rb.n <= 8) k_pose_error64<8><<<grid, block, 0, s>>>(rb, q, targets, N, pos_err, ori_err);
    else if (rb.n <= 16) k_pose_error64<16><<<grid, block, 0, s>>>(rb, q, targets, N, pos_err, ori_err);
    else k_pose_error64<32><<<grid, block, 0, s>>>(rb, q, targets, N, pos_err, ori_err);
    return cudaGetLastError();
}

cudaError_t launch_select_replicate(const DevRobot& rb, const DevCfg& c, const float* cost,
                                    const float* theta, int T, float* seeds, int32_t* kept,
                                    cudaStream_t s) {
    int Mpad = 2;
    while (Mpad < c.M) Mpad <<= 1;
    const size_t smem = (size_t)Mpad * sizeof(unsigned long long);
    static std::atomic<unsigned long long> attr_set{0};
    cudaError_t e = once_per_device(attr_set, [] {
        return cudaFuncSetAttribute(k_select_replicate, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    8192 * (int)sizeof(unsigned long long));
    });
    if (e != cudaSuccess) return e;
    const int block = Mpad >= 1024 ? 512 : (Mpad >= 256 ? 256 : 128);
    k_select_replicate<<<T, block, smem, s>>>(rb, c, cost, theta, Mpad, seeds, kept);
    return cudaGetLastError();
}

template <class T>
cudaError_t launch_select_best(const DevRobot& rb, const DevCfg& c, const float* targets, int T_,
                               const T* theta, const T* ep_all, const T* eo_all, T* q_out, T* pos_err,
                               T* ori_err, int32_t* status, cudaStream_t s) {
    k_select_best<T><<<T_, 128, 0, s>>>(rb, c, targets, theta, ep_all, eo_all, q_out, pos_err, ori_err, status);
    return cudaGetLastError();
}
template cudaError_t launch_select_best<float>(const DevRobot&, const DevCfg&, const float*, int, const float*,
                                               const float*, const float*, float*, float*, float*, int32_t*,
                                               cudaStream_t);
template cudaError_t launch_select_best<double>(const DevRobot&, const DevCfg&, const float*, int, const double*,
                                                const double*, const double*, double*, double*, double*, int32_t*,
                                                cudaStream_t);

cudaError_t launch_fk(const DevRobot& rb, const float* q, int N, float* pose7, float* jac, cudaStream_t s,
                      bool sfu) {
    const int block = 128;
    const int grid = (N + block - 1) / block;
    const int kind = rb.pmask ? 0 : (rb.rx ? 2 : 1);
    auto go = [&](auto nmax) {
        constexpr int NM = decltype(nmax)::value;
        if (sfu) {
            if (kind == 2) k_fk<NM, 2, true><<<grid, block, 0, s>>>(rb, q, N, pose7, jac);
            else if (kind == 1) k_fk<NM, 1, true><<<grid, block, 0, s>>>(rb, q, N, pose7, jac);
            else k_fk<NM, 0, true><<<grid, block, 0, s>>>(rb, q, N, pose7, jac);
            return;
        }
        if (kind == 2) k_fk<NM, 2, false><<<grid, block, 0, s>>>(rb, q, N, pose7, jac);
        else if (kind == 1) k_fk<NM, 1, false><<<grid, block, 0, s>>>(rb, q, N, pose7, jac);
        else k_fk<NM, 0, false><<<grid, block, 0, s>>>(rb, q, N, pose7, jac);
    };
    if (rb.n <= 8) go(std::integral_constant<int, 8>());
    else if (rb.n <= 16) go(std::integral_constant<int, 16>());
    else go(std::integral_constant<int, 32>());
    return cudaGetLastError();
}

}  // namespace hjcd
