// Initial feasible solutions, Eq. 4 (§4.3): one warp per start runs projected Adam on
//     ||A x - b||_2^2 + lambda3 sum_i (x_i - floor x_i)(ceil x_i - x_i)     over the box [l, u]
// from x0 ~ U(l, u) (splitmix64 counter, salted seed); the final x is rounded half away from zero and kept iff
// A x = b exactly (int64) — the box holds by construction (projection + integer bounds). Kept rows are written
// as int8 offsets x - l (0 <= x - l <= u - l <= 127), so the library's dedupe and lexicographic sort apply
// unchanged (subtracting l preserves lexicographic order).
// Lanes own rows of A for the residual (CSR) and coordinates for the gradient A^T r (CSC) and the Adam state.
#include <cstdio>

#include "common.cuh"
#include "kernels.h"

namespace maple {

namespace {

constexpr int kWarps = 8;
constexpr uint64_t kFeasSalt = 0x5EEDF00DCAFE0001ULL;

template <int QN>
__global__ void __launch_bounds__(kWarps * 32, 1) feasible_kernel(const FeasibleParams p) {
    extern __shared__ __align__(16) unsigned char fsm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int n = p.n, m = p.m, nnz = p.nnz;
    float* xsh = reinterpret_cast<float*>(fsm) + (size_t)wid * (n + m);
    float* rsh = xsh + n;
    // A's CSR and CSC staged once per block (every step of every warp walks them: from global memory each
    // dependent index load was an L1/L2 round trip on the step's critical path)
    int32_t* a_rp = reinterpret_cast<int32_t*>(fsm + (size_t)kWarps * (n + m) * 4);
    int32_t* a_col = a_rp + (m + 1);
    int32_t* a_val = a_col + nnz;
    int32_t* t_cp = a_val + nnz;
    int32_t* t_row = t_cp + (n + 1);
    int32_t* t_val = t_row + nnz;
    for (int i = threadIdx.x; i <= m; i += blockDim.x) a_rp[i] = p.A_rowptr[i];
    for (int i = threadIdx.x; i <= n; i += blockDim.x) t_cp[i] = p.AT_colptr[i];
    for (int i = threadIdx.x; i < nnz; i += blockDim.x) {
        a_col[i] = p.A_col[i];
        a_val[i] = p.A_val[i];
        t_row[i] = p.AT_row[i];
        t_val[i] = p.AT_val[i];
    }
    __syncthreads();
    const int64_t s = (int64_t)blockIdx.x * kWarps + wid;
    if (s >= p.k) return;
    const uint64_t seed = p.seed ^ kFeasSalt;
    float x[QN], mm[QN], vv[QN], lo[QN], hi[QN];
#pragma unroll
    for (int q = 0; q < QN; ++q) {
        const int j = lane + 32 * q;
        x[q] = mm[q] = vv[q] = 0.f;
        lo[q] = hi[q] = 0.f;
        if (j < n) {
            lo[q] = (float)p.lo[j];
            hi[q] = (float)p.hi[j];
            const double U = counter_uniform(seed, s, j, n);
            x[q] = (float)__dadd_rn((double)p.lo[j], __dmul_rn(U, (double)(p.hi[j] - p.lo[j])));
            xsh[j] = x[q];
        }
    }
    __syncwarp();
    for (int t = 0; t < p.T; ++t) {
        // residual r = A x - b (lanes over rows of A)
        for (int a = lane; a < m; a += 32) {
            float acc = -(float)p.b[a];
            for (int e = a_rp[a]; e < a_rp[a + 1]; ++e) acc = fmaf((float)a_val[e], xsh[a_col[e]], acc);
            rsh[a] = acc;
        }
        __syncwarp();
        const float4 st = p.step_tab[t];
#pragma unroll
        for (int q = 0; q < QN; ++q) {
            const int j = lane + 32 * q;
            if (j < n) {
                float acc = 0.f;  // (A^T r)_j over the nonzeros of column j
                for (int e = t_cp[j]; e < t_cp[j + 1]; ++e) acc = fmaf((float)t_val[e], rsh[t_row[e]], acc);
                const float xx = x[q];
                const float g = 2.f * acc + p.lam3 * (ceilf(xx) + floorf(xx) - 2.f * xx);
                mm[q] = p.beta1 * mm[q] + p.omb1 * g;
                vv[q] = p.beta2 * vv[q] + p.omb2 * g * g;
                const float denom = sqrtf(vv[q]) / st.y + p.eps;
                x[q] = fminf(fmaxf(xx - st.x * mm[q] / denom, lo[q]), hi[q]);   // projection onto [l, u]
            }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < QN; ++q)
            if (lane + 32 * q < n) xsh[lane + 32 * q] = x[q];
        __syncwarp();
    }
    // round half away from zero, exact check A x = b (int64)
#pragma unroll
    for (int q = 0; q < QN; ++q)
        if (lane + 32 * q < n) xsh[lane + 32 * q] = (float)round_half_away(x[q]);
    __syncwarp();
    bool ok = true;
    for (int a = lane; a < m; a += 32) {
        long long acc = -(long long)p.b[a];
        for (int e = a_rp[a]; e < a_rp[a + 1]; ++e)
            acc += (long long)a_val[e] * (long long)xsh[a_col[e]];
        ok &= acc == 0;
    }
    ok = __all_sync(0xffffffffu, ok);
    if (p.X_out) {  // debug: final continuous iterates
#pragma unroll
        for (int q = 0; q < QN; ++q)
            if (lane + 32 * q < n) p.X_out[s * n + lane + 32 * q] = x[q];
    }
    if (!ok) return;
    unsigned long long slot = 0;
    if (lane == 0) slot = atomicAdd(p.count, 1ULL);
    slot = __shfl_sync(0xffffffffu, slot, 0);
    if ((int64_t)slot >= p.cap) return;
    int8_t* dst = p.rows + (size_t)slot * p.n_pad;
    for (int i = lane; i < p.n_pad; i += 32) dst[i] = i < n ? (int8_t)((int)xsh[i] - p.lo[i]) : (int8_t)0;
}

template <int QN>
cudaError_t launch_qn(const FeasibleParams& p, cudaStream_t s) {
    const size_t smem = (size_t)kWarps * (p.n + p.m) * 4 + (size_t)(p.m + 1 + p.n + 1 + 4 * (size_t)p.nnz) * 4;
    cudaError_t e = cudaFuncSetAttribute(feasible_kernel<QN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t blocks = (p.k + kWarps - 1) / kWarps;
    feasible_kernel<QN><<<(unsigned)blocks, kWarps * 32, smem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_feasible(const FeasibleParams& p, cudaStream_t s) {
    if (p.k <= 0) return cudaSuccess;
    const int qn = (p.n + 31) / 32;
    if (qn <= 1) return launch_qn<1>(p, s);
    if (qn <= 2) return launch_qn<2>(p, s);
    if (qn <= 4) return launch_qn<4>(p, s);
    if (qn <= 8) return launch_qn<8>(p, s);
    if (qn <= 16) return launch_qn<16>(p, s);
    if (qn <= 32) return launch_qn<32>(p, s);
    return cudaErrorInvalidValue;
}

}  // namespace maple
