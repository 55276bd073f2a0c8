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
#include <cstdio>

#include "common.cuh"
#include "kernels.h"

namespace maple {

namespace {

constexpr int kWarps = 8;

template <int QD>
__global__ void __launch_bounds__(kWarps * 32, 1)
descent_simt_kernel(const DescentParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int n = p.n, d = p.d;
    const SparseB& sb = p.sb;
    // optional shared-memory copy of the sparse B (all warps of the block read it)
    const int32_t* rptr = sb.row_ptr;
    const int16_t* rcol = sb.row_col;
    const float* rval = sb.row_val;
    const int32_t* cptr = sb.col_ptr;
    const int16_t* crow = sb.col_row;
    const float* cval = sb.col_val;
    unsigned char* wbase = smem_raw;
    if (sb.in_smem) {
        int32_t* s_rptr = reinterpret_cast<int32_t*>(smem_raw);
        int32_t* s_cptr = s_rptr + (n + 1);
        float* s_rval = reinterpret_cast<float*>(s_cptr + (d + 1));
        float* s_cval = s_rval + sb.nnz;
        int16_t* s_rcol = reinterpret_cast<int16_t*>(s_cval + sb.nnz);
        int16_t* s_crow = s_rcol + sb.nnz;
        for (int i = threadIdx.x; i <= n; i += blockDim.x) s_rptr[i] = sb.row_ptr[i];
        for (int i = threadIdx.x; i <= d; i += blockDim.x) s_cptr[i] = sb.col_ptr[i];
        for (int i = threadIdx.x; i < sb.nnz; i += blockDim.x) {
            s_rval[i] = sb.row_val[i];
            s_cval[i] = sb.col_val[i];
            s_rcol[i] = sb.row_col[i];
            s_crow[i] = sb.col_row[i];
        }
        rptr = s_rptr;
        cptr = s_cptr;
        rval = s_rval;
        cval = s_cval;
        rcol = s_rcol;
        crow = s_crow;
        wbase = smem_raw + sb.smem_bytes;
        __syncthreads();
    }
    // per-warp scratch: z (d f32) | s (n f32, also g) | r (d f32); g0 (n f64) aliases it in the prologue
    const size_t per_warp = ((size_t)(2 * d + n) * 4 > (size_t)n * 8 ? (size_t)(2 * d + n) * 4 : (size_t)n * 8);
    const size_t per_warp_al = (per_warp + 15) & ~size_t(15);
    unsigned char* base = wbase + per_warp_al * wid;
    double* g0sh = reinterpret_cast<double*>(base);
    float* zsh = reinterpret_cast<float*>(base);
    float* ssh = zsh + d;
    float* rsh = ssh + n;

    const int64_t local = (int64_t)blockIdx.x * kWarps + wid;
    if (local >= p.count) return;
    const int64_t gi = p.begin + local;
    // this lane's rows (forward / harvest) and coordinates (backward / Adam): load-balanced lists
    const int r_beg = sb.lane_rows_ptr[lane], r_end = sb.lane_rows_ptr[lane + 1];
    const int c_beg = sb.lane_cols_ptr[lane], c_end = sb.lane_cols_ptr[lane + 1];
    int myj[QD];
#pragma unroll
    for (int q = 0; q < QD; ++q) myj[q] = (c_beg + q < c_end) ? sb.lane_cols[c_beg + q] : -1;

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
        const int j = myj[q];
        m[q] = 0.f;
        v[q] = 0.f;
        rprev[q] = 0x7fffffff;
        z[q] = 0.f;
        if (j >= 0) {
            double acc = 0.0;
            const double* row = p.Bp + (size_t)j * n;
            for (int k = 0; k < n; ++k) acc = fma(row[k], g0sh[k], acc);
            z[q] = (float)acc;
            if (p.Z0_out) p.Z0_out[local * d + j] = acc;
        }
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < QD; ++q)
        if (myj[q] >= 0) zsh[myj[q]] = z[q];
    __syncwarp();

    const float b1 = p.beta1, b2 = p.beta2, omb1 = p.omb1, omb2 = p.omb2;
    for (int t = 0; t < p.T; ++t) {
        // forward: y_i = sum_j B_ij z_j (CSR), s_i = sign(y_i)
        for (int a = r_beg; a < r_end; ++a) {
            const int i = sb.lane_rows[a];
            float y = 0.f;
            for (int e = rptr[i]; e < rptr[i + 1]; ++e) y = fmaf(rval[e], zsh[rcol[e]], y);
            ssh[i] = fsign(y);
        }
        __syncwarp();
        // backward (CSC) + penalties + argmax |z|
        float gr[QD];
        float best = -1.f;
        int bestj = 0x7fffffff;
#pragma unroll
        for (int q = 0; q < QD; ++q) {
            const int j = myj[q];
            gr[q] = 0.f;
            if (j >= 0) {
                float acc = 0.f;
                for (int e = cptr[j]; e < cptr[j + 1]; ++e) acc = fmaf(cval[e], ssh[crow[e]], acc);
                const float zz = z[q];
                gr[q] = acc + p.lam1 * (ceilf(zz) + floorf(zz) - 2.f * zz);
                const float aa = fabsf(zz);
                if (aa > best || (aa == best && j < bestj)) {
                    best = aa;
                    bestj = j;
                }
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
        if (best < 1.f) {  // lam2 term active on the lowest-index argmax coordinate
#pragma unroll
            for (int q = 0; q < QD; ++q) {
                if (myj[q] == bestj) {
                    const float zk = z[q];
                    gr[q] += -p.lam2 * fsign(zk) / fmaxf(zk * zk, 1e-8f);
                }
            }
        }
        // Adam (reading #9)
        const float4 st = p.step_tab[t];
#pragma unroll
        for (int q = 0; q < QD; ++q) {
            const int j = myj[q];
            if (j >= 0) {
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
            const int j = myj[q];
            r[q] = 0;
            if (j >= 0) {
                r[q] = round_half_away(z[q]);
                changed |= (r[q] != rprev[q]);
                rsh[j] = (float)r[q];
            }
        }
        if (!__any_sync(0xffffffffu, changed)) continue;
#pragma unroll
        for (int q = 0; q < QD; ++q) rprev[q] = r[q];
        __syncwarp();
        bool ok = true;
        for (int a = r_beg; a < r_end; ++a) {
            const int i = sb.lane_rows[a];
            float acc = 0.f;
            for (int e = rptr[i]; e < rptr[i + 1]; ++e) acc = fmaf(rval[e], rsh[rcol[e]], acc);
            const int gv = (int)acc;
            ok &= (abs(gv) <= p.box[i]);
            ssh[i] = (float)gv;  // reuse s as the g row buffer
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
            for (int i = lane; i < p.n_pad; i += 32)
                dst[i] = (i < n) ? (int8_t)(firstsign * (int)ssh[i]) : (int8_t)0;
        }
        __syncwarp();
    }
    if (p.Z_out) {
#pragma unroll
        for (int q = 0; q < QD; ++q)
            if (myj[q] >= 0) p.Z_out[local * d + myj[q]] = z[q];
    }
}

template <int QD>
cudaError_t launch_q(const DescentParams& p, cudaStream_t s) {
    const int n = p.n, d = p.d;
    const size_t per_warp = ((size_t)(2 * d + n) * 4 > (size_t)n * 8 ? (size_t)(2 * d + n) * 4 : (size_t)n * 8);
    const size_t smem = ((per_warp + 15) & ~size_t(15)) * kWarps + (p.sb.in_smem ? p.sb.smem_bytes : 0);
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
    const int qd = p.sb.max_lane_cols;
    if (qd <= 1) return launch_q<1>(p, s);
    if (qd <= 2) return launch_q<2>(p, s);
    if (qd <= 4) return launch_q<4>(p, s);
    if (qd <= 8) return launch_q<8>(p, s);
    if (qd <= 12) return launch_q<12>(p, s);
    if (qd <= 16) return launch_q<16>(p, s);
    if (qd <= 24) return launch_q<24>(p, s);
    if (qd <= 32) return launch_q<32>(p, s);
    return cudaErrorInvalidValue;
}

}  // namespace maple
