// SIMT descent + harvest: one warp per start (the general-shape path; the tcgen05 kernel in
// k_descent_tc.cu is the fast path for the shapes it supports).
//
// Per start, Algorithm 3 lines 4-10:
//   z0 = B+ g0, g0 ~ U(l-u, u-l) (counter RNG, fp64)
//   for t = 1..T:  grad = B^T sign(B z) + lam1 (ceil z + floor z - 2z) + lam2-term   (Eq. 3)
//                  Adam update of z (torch.optim.Adam formula, reading #9)
//                  r = round_half_away(z); if r changed: g = B r, keep iff g != 0 and |g| <= u - l
//                  (P:406-407), canonical sign (first nonzero > 0), append to the candidate buffer.
// Lanes split the n rows (forward, expansion) and the d coordinates (backward, Adam); every row's
// reduction runs in a fixed order (j ascending / i ascending), independent of placement.
#include <cstdio>

#include "common.cuh"
#include "kernels.h"

namespace maple {

namespace {

constexpr int kWarps = 8;

template <int QD>
__global__ void __launch_bounds__(kWarps * 32)
descent_simt_kernel(const DescentParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int n = p.n, d = p.d;
    // per-warp scratch: z (d f32) | s (n f32) | r (d f32) | g0 (n f64)
    const size_t per_warp = (size_t)(2 * d + n) * 4 + (size_t)n * 8;
    const size_t per_warp_al = (per_warp + 15) & ~size_t(15);
    unsigned char* base = smem_raw + per_warp_al * wid;
    double* g0sh = reinterpret_cast<double*>(base);
    float* zsh = reinterpret_cast<float*>(base + (size_t)n * 8);
    float* ssh = zsh + d;
    float* rsh = ssh + n;

    const int64_t local = (int64_t)blockIdx.x * kWarps + wid;
    if (local >= p.count) return;
    const int64_t gi = p.begin + local;

    // ---- start (Alg. 3 lines 4-5) ----
    for (int k = lane; k < n; k += 32) {
        double U = counter_uniform(p.seed, gi, k, n);
        g0sh[k] = start_coord(U, p.lo[k], p.hi[k]);
    }
    __syncwarp();
    float z[QD], m[QD], v[QD];
    int rprev[QD];
#pragma unroll
    for (int q = 0; q < QD; ++q) {
        const int j = lane + 32 * q;
        m[q] = 0.f;
        v[q] = 0.f;
        rprev[q] = 0x7fffffff;
        z[q] = 0.f;
        if (j < d) {
            double acc = 0.0;
            const double* row = p.Bp + (size_t)j * n;
            for (int k = 0; k < n; ++k) acc = fma(row[k], g0sh[k], acc);
            z[q] = (float)acc;
            zsh[j] = z[q];
            if (p.Z0_out) p.Z0_out[local * d + j] = acc;
        }
    }
    __syncwarp();

    const float b1 = p.beta1, b2 = p.beta2, omb1 = p.omb1, omb2 = p.omb2;
    for (int t = 0; t < p.T; ++t) {
        // forward: y_i = sum_j B_ij z_j, s_i = sign(y_i)
        for (int i = lane; i < n; i += 32) {
            float y = 0.f;
            for (int j = 0; j < d; ++j) y = fmaf(__ldg(p.B_dn + (size_t)j * n + i), zsh[j], y);
            ssh[i] = fsign(y);
        }
        __syncwarp();
        // backward + penalties + argmax |z|
        float gr[QD];
        float best = -1.f;
        int bestj = 0x7fffffff;
#pragma unroll
        for (int q = 0; q < QD; ++q) {
            const int j = lane + 32 * q;
            gr[q] = 0.f;
            if (j < d) {
                float acc = 0.f;
                for (int i = 0; i < n; ++i) acc = fmaf(__ldg(p.B_nd + (size_t)i * d + j), ssh[i], acc);
                const float zz = z[q];
                gr[q] = acc + p.lam1 * (ceilf(zz) + floorf(zz) - 2.f * zz);
                const float a = fabsf(zz);
                if (a > best) { best = a; bestj = j; }
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const float ob = __shfl_xor_sync(0xffffffffu, best, off);
            const int oj = __shfl_xor_sync(0xffffffffu, bestj, off);
            if (ob > best || (ob == best && oj < bestj)) { best = ob; bestj = oj; }
        }
        if (best < 1.f) {  // lam2 term active on the lowest-index argmax coordinate
#pragma unroll
            for (int q = 0; q < QD; ++q) {
                if (lane + 32 * q == bestj) {
                    const float zk = z[q];
                    gr[q] += -p.lam2 * fsign(zk) / fmaxf(zk * zk, 1e-8f);
                }
            }
        }
        // Adam (reading #9)
        const float4 st = p.step_tab[t];
#pragma unroll
        for (int q = 0; q < QD; ++q) {
            const int j = lane + 32 * q;
            if (j < d) {
                m[q] = b1 * m[q] + omb1 * gr[q];
                v[q] = b2 * v[q] + omb2 * gr[q] * gr[q];
                const float denom = sqrtf(v[q]) / st.y + p.eps;
                z[q] = z[q] - st.x * m[q] / denom;
                zsh[j] = z[q];
            }
        }
        __syncwarp();
        if (!p.harvest) continue;
        // harvest (Alg. 3 lines 9-10)
        bool changed = false;
        int r[QD];
#pragma unroll
        for (int q = 0; q < QD; ++q) {
            const int j = lane + 32 * q;
            r[q] = 0;
            if (j < d) {
                r[q] = round_half_away(z[q]);
                changed |= (r[q] != rprev[q]);
                rsh[j] = (float)r[q];
            }
        }
        if (!__any_sync(0xffffffffu, changed)) continue;
#pragma unroll
        for (int q = 0; q < QD; ++q) rprev[q] = r[q];
        __syncwarp();
        bool ok = true, nz = false;
        int first = 0x7fffffff, firstsign = 0;
        for (int i0 = 0; i0 < n; i0 += 32) {
            const int i = i0 + lane;
            int gv = 0;
            if (i < n) {
                float acc = 0.f;
                for (int j = 0; j < d; ++j) acc = fmaf(__ldg(p.B_dn + (size_t)j * n + i), rsh[j], acc);
                gv = (int)acc;
                ok &= (abs(gv) <= p.box[i]);
                nz |= (gv != 0);
                ssh[i] = (float)gv;  // reuse s as the g row buffer
            }
            const unsigned msk = __ballot_sync(0xffffffffu, gv != 0);
            if (msk && first == 0x7fffffff) {
                const int fl = __ffs(msk) - 1;
                first = i0 + fl;
                firstsign = __shfl_sync(0xffffffffu, gv, fl) > 0 ? 1 : -1;
            }
        }
        ok = __all_sync(0xffffffffu, ok);
        nz = __any_sync(0xffffffffu, nz);
        if (!(ok && nz)) continue;
        __syncwarp();
        unsigned long long slot = 0;
        if (lane == 0) slot = atomicAdd(p.cand_count, 1ULL);
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if ((int64_t)slot < p.cand_cap) {
            int8_t* dst = p.cand + (size_t)slot * p.n_pad;
            for (int i = lane; i < p.n_pad; i += 32)
                dst[i] = (i < n) ? (int8_t)(firstsign * (int)ssh[i]) : (int8_t)0;
        }
        __syncwarp();
    }
    if (p.Z_out) {
#pragma unroll
        for (int q = 0; q < QD; ++q) {
            const int j = lane + 32 * q;
            if (j < d) p.Z_out[local * d + j] = z[q];
        }
    }
}

template <int QD>
cudaError_t launch_q(const DescentParams& p, cudaStream_t s) {
    const size_t per_warp = (size_t)(2 * p.d + p.n) * 4 + (size_t)p.n * 8;
    const size_t smem = ((per_warp + 15) & ~size_t(15)) * kWarps;
    cudaError_t e = cudaFuncSetAttribute(descent_simt_kernel<QD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t blocks = (p.count + kWarps - 1) / kWarps;
    descent_simt_kernel<QD><<<(unsigned)blocks, kWarps * 32, smem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_descent_simt(const DescentParams& p, cudaStream_t s) {
    if (p.count <= 0) return cudaSuccess;
    const int qd = (p.d + 31) / 32;
    if (qd <= 1) return launch_q<1>(p, s);
    if (qd <= 2) return launch_q<2>(p, s);
    if (qd <= 4) return launch_q<4>(p, s);
    if (qd <= 8) return launch_q<8>(p, s);
    if (qd <= 16) return launch_q<16>(p, s);
    if (qd <= 32) return launch_q<32>(p, s);
    return cudaErrorInvalidValue;
}

}  // namespace maple
