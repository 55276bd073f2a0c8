// SIMT descent + harvest for general shapes: one warp per start, B in sparse form (the general-shape path;
// the tcgen05 kernel in k_descent_tc.cu is the fast path for the shapes whose state fits on chip).
//
// LLL-reduced kernel bases of the configs are sparse (C2a 4 %, C3 7.6 % nonzeros), so the two
// contractions of a step are sparse matrix-vector products, not dense GEMMs:
//   forward  y_i = sum_{j in row i} B_ij z_j      (CSR; each lane owns a load-balanced set of rows)
//   backward Γ_j = sum_{i in col j} B_ij s_i      (CSC; each lane owns a load-balanced set of columns,
//                                                  and the Adam state of those coordinates in registers)
// Per start, Algorithm 3 lines 4-10:
//   z0 = B+ g0, g0 ~ U(l-u, u-l) (counter RNG, fp64)
//   for t = 1..T:  grad = B^T sign(B z) + lam1 (ceil z + floor z - 2z) + lam2-term   (Eq. 3)
//                  Adam update of z (torch.optim.Adam formula, reading #9)
//                  r = round_half_away(z); if r changed: g = B r, keep iff g != 0 and |g| <= u - l
//                  (P:406-407), canonical sign (first nonzero > 0), append to the candidate buffer.
// Every reduction runs in a fixed order (CSR / CSC order), independent of placement.
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "kernels.h"

namespace maple {

namespace {

constexpr int kWarps = 8;

__device__ __forceinline__ float nz_val(uint32_t e) { return (float)(int)(int8_t)(e >> 16); }
__device__ __forceinline__ int nz_idx(uint32_t e) { return (int)(e & 0xFFFFu); }

// One warp per start; the start's state (z, m, v), sign vector and rounded iterate live in the warp's slice
// of shared memory, so registers stay few and 32 warps fit per SM (the contractions are latency-bound
// gathers). B entries are packed (index | int8 value << 16) and read through L1.
__global__ void __launch_bounds__(kWarps * 32)
descent_simt_kernel(const DescentParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int n = p.n, d = p.d;
    const SparseB& sb = p.sb;
    // per-warp slice: z | m | v | r (d floats each) | s (n floats; also the g row); g0 (n doubles) aliases it
    const size_t pw_f = (size_t)(4 * d + n) * 4, pw_d = (size_t)n * 8;
    const size_t per_warp = pw_f > pw_d ? pw_f : pw_d;
    const size_t per_warp_al = (per_warp + 15) & ~size_t(15);
    unsigned char* base = smem_raw + per_warp_al * wid;
    double* g0sh = reinterpret_cast<double*>(base);
    float* zsh = reinterpret_cast<float*>(base);
    float* msh = zsh + d;
    float* vsh = msh + d;
    float* rsh = vsh + d;
    float* ssh = rsh + d;

    const int64_t local = (int64_t)blockIdx.x * kWarps + wid;
    if (local >= p.count) return;
    const int64_t gi = p.begin + local;
    const int r_beg = sb.lane_rows_ptr[lane], r_end = sb.lane_rows_ptr[lane + 1];
    const int c_beg = sb.lane_cols_ptr[lane], c_end = sb.lane_cols_ptr[lane + 1];

    // ---- start (Alg. 3 lines 4-5): g0 in fp64, z0 = B+ g0 ----
    for (int k = lane; k < n; k += 32) g0sh[k] = start_coord(counter_uniform(p.seed, gi, k, n), p.lo[k], p.hi[k]);
    __syncwarp();
    float z0[32];
    const int nmine = c_end - c_beg;   // <= 32 (checked on the host)
#pragma unroll 1
    for (int q = 0; q < nmine; ++q) {
        const int j = sb.lane_cols[c_beg + q];
        double acc = 0.0;
        const double* row = p.Bp + (size_t)j * n;
        for (int k = 0; k < n; ++k) acc = fma(row[k], g0sh[k], acc);
        if (p.Z0_out) p.Z0_out[local * d + j] = acc;
        if (q < 32) z0[q] = (float)acc;
    }
    __syncwarp();
#pragma unroll 1
    for (int q = 0; q < nmine; ++q) {
        const int j = sb.lane_cols[c_beg + q];
        zsh[j] = z0[q];
        msh[j] = 0.f;
        vsh[j] = 0.f;
        rsh[j] = __int_as_float(0x7fffffff);   // "no previous round(z)": NaN never equals a rounded value
    }
    __syncwarp();

    const float b1 = p.beta1, b2 = p.beta2, omb1 = p.omb1, omb2 = p.omb2, lam1 = p.lam1, lam2 = p.lam2;
    for (int t = 0; t < p.T; ++t) {
        // forward: y_i = sum_j B_ij z_j (CSR), s_i = sign(y_i)
        for (int a = r_beg; a < r_end; ++a) {
            const int i = sb.lane_rows[a];
            float y = 0.f;
            for (int e = sb.row_ptr[i]; e < sb.row_ptr[i + 1]; ++e) {
                const uint32_t w = sb.row_pk[e];
                y = fmaf(nz_val(w), zsh[nz_idx(w)], y);
            }
            ssh[i] = fsign(y);
        }
        __syncwarp();
        // lowest-index argmax of |z| (λ2 term, Eq. 3)
        float best = -1.f;
        int bestj = 0x7fffffff;
        for (int q = c_beg; q < c_end; ++q) {
            const int j = sb.lane_cols[q];
            const float aa = fabsf(zsh[j]);
            if (aa > best || (aa == best && j < bestj)) {
                best = aa;
                bestj = j;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const float ob = __shfl_xor_sync(0xffffffffu, best, off);
            const int oj = __shfl_xor_sync(0xffffffffu, bestj, off);
            if (ob > best || (ob == best && oj < bestj)) {
                best = ob;
                bestj = oj;
            }
        }
        // backward (CSC) + penalties + Adam (reading #9) on this lane's coordinates
        const float4 st = p.step_tab[t];
        bool changed = false;
        for (int q = c_beg; q < c_end; ++q) {
            const int j = sb.lane_cols[q];
            float acc = 0.f;
            for (int e = sb.col_ptr[j]; e < sb.col_ptr[j + 1]; ++e) {
                const uint32_t w = sb.col_pk[e];
                acc = fmaf(nz_val(w), ssh[nz_idx(w)], acc);
            }
            const float zz = zsh[j];
            float gr = acc + lam1 * (ceilf(zz) + floorf(zz) - 2.f * zz);
            if (best < 1.f && j == bestj) gr += -lam2 * fsign(zz) / fmaxf(zz * zz, 1e-8f);
            const float mm = b1 * msh[j] + omb1 * gr;
            const float vv = b2 * vsh[j] + omb2 * gr * gr;
            const float zn = zz - st.x * mm / (sqrtf(vv) / st.y + p.eps);
            msh[j] = mm;
            vsh[j] = vv;
            zsh[j] = zn;
            if (p.harvest) {
                const float rn = (float)round_half_away(zn);
                changed |= rn != rsh[j];
                rsh[j] = rn;
            }
        }
        __syncwarp();
        if (!p.harvest) continue;
        // harvest (Alg. 3 lines 9-10) when round(z) changed: g = B r (CSR), box, g != 0, canonical sign
        if (!__any_sync(0xffffffffu, changed)) continue;
        bool ok = true;
        for (int a = r_beg; a < r_end; ++a) {
            const int i = sb.lane_rows[a];
            float acc = 0.f;
            for (int e = sb.row_ptr[i]; e < sb.row_ptr[i + 1]; ++e) {
                const uint32_t w = sb.row_pk[e];
                acc = fmaf(nz_val(w), rsh[nz_idx(w)], acc);
            }
            const int gv = (int)acc;
            ok &= (abs(gv) <= p.box[i]);
            ssh[i] = (float)gv;  // s is dead until the next forward: reuse it as the g row
        }
        ok = __all_sync(0xffffffffu, ok);
        if (!ok) continue;
        __syncwarp();
        int firstsign = 0;
        for (int i0 = 0; i0 < n && !firstsign; i0 += 32) {
            const int i = i0 + lane;
            const int gv = i < n ? (int)ssh[i] : 0;
            const unsigned msk = __ballot_sync(0xffffffffu, gv != 0);
            if (msk) firstsign = __shfl_sync(0xffffffffu, gv, __ffs(msk) - 1) > 0 ? 1 : -1;
        }
        if (!firstsign) continue;  // g = 0
        unsigned long long slot = 0;
        if (lane == 0) slot = atomicAdd(p.cand_count, 1ULL);
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if ((int64_t)slot < p.cand_cap) {
            int8_t* dst = p.cand + (size_t)slot * p.n_pad;
            for (int i = lane; i < p.n_pad; i += 32) dst[i] = (i < n) ? (int8_t)(firstsign * (int)ssh[i]) : (int8_t)0;
        }
        __syncwarp();
    }
    if (p.Z_out)
        for (int q = c_beg; q < c_end; ++q) {
            const int j = sb.lane_cols[q];
            p.Z_out[local * d + j] = zsh[j];
        }
}

}  // namespace

cudaError_t launch_descent_simt(const DescentParams& p, cudaStream_t s) {
    if (p.count <= 0) return cudaSuccess;
    if (p.sb.max_lane_cols > 32) return cudaErrorInvalidValue;
    const int n = p.n, d = p.d;
    const size_t per_warp = std::max<size_t>((size_t)(4 * d + n) * 4, (size_t)n * 8);
    const size_t smem = ((per_warp + 15) & ~size_t(15)) * kWarps;
    cudaError_t e = cudaFuncSetAttribute(descent_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t blocks = (p.count + kWarps - 1) / kWarps;
    descent_simt_kernel<<<(unsigned)blocks, kWarps * 32, smem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace maple
