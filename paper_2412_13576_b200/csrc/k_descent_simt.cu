// SIMT descent + harvest for general shapes: one warp per start, B in sparse form (the general-shape path;
// the tcgen05 kernel in k_descent_tc.cu is the fast path for the shapes whose state fits on chip).
//
// LLL-reduced kernel bases of the configs are sparse (C2a 4 %, C3 1.5 %, C5 0.3 % nonzeros), so the two
// contractions of a step are sparse matrix-vector products, not dense GEMMs:
//   forward  y_i = sum_{j in row i} B_ij z_j      (each lane owns a load-balanced set of rows)
//   backward Γ_j = sum_{i in col j} B_ij s_i      (each lane owns a load-balanced set of columns,
//                                                  and the Adam state (m, v) of those coordinates in registers)
// Both run from lane-major, bank-conflict-scheduled ELL words staged once per block in shared memory
// (sparse_ell.h): per slot a warp reads one 128-byte line of words and gathers one conflict-free wavefront.
// Per warp, shared memory holds z, s (reused for the harvested g row) and the ELL result queue (which also holds
// the gradient Γ); the harvest gathers round(z) straight from z. Warps stay small (about 3 KB at C3, 12 KB at C5).
// Per start, Algorithm 3 lines 4-10:
//   z0 = B+ g0, g0 ~ U(l-u, u-l) (counter RNG, fp64)
//   for t = 1..T:  grad = B^T sign(B z) + lam1 (ceil z + floor z - 2z) + lam2-term   (Eq. 3)
//                  Adam update of z (torch.optim.Adam formula, reading #9)
//                  r = round_half_away(z); if r changed: g = B r, keep iff g != 0 and |g| <= u - l
//                  (P:406-407), canonical sign (first nonzero > 0), append to the candidate buffer.
// Every reduction runs in the fixed order of its ELL schedule, independent of block / warp placement.
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "kernels.h"
#include "tc_umma.cuh"   // rcp_approx, sqrt_approx (the same Adam arithmetic as the tcgen05 kernel)

namespace maple {

namespace {

// One ELL schedule (sparse_ell.h) for this lane: wl = ell + lane, resq = res + lane; the lane's k-th completed
// piece sum goes to resq[k * 32]. Per slot: one 128-byte line of words, one conflict-free gather, one FFMA.
#ifndef MAPLE_ELL_BATCH
#define MAPLE_ELL_BATCH 8
#endif
// ROUND: gather round_half_away(x) instead of x (the harvest's g = B round(z) straight from z)
template <bool ROUND = false>
__device__ __forceinline__ void ell_run(const uint32_t* __restrict__ wl, int slots, const float* __restrict__ x,
                                        float* __restrict__ resq) {
    const char* xb = reinterpret_cast<const char*>(x);
    float acc = 0.f;
    int e = 0;
#if MAPLE_ELL_BATCH > 1
    // words and gathers of MAPLE_ELL_BATCH slots are issued before the batch's queue stores (x and the queue are
    // disjoint, which the compiler cannot prove: without this every gather waits for the previous slot's store)
    constexpr int NB = MAPLE_ELL_BATCH;
    for (; e + NB <= slots; e += NB) {
        uint32_t w[NB];
        float xv[NB];
#pragma unroll
        for (int k = 0; k < NB; ++k) w[k] = wl[(e + k) * 32];
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            xv[k] = *reinterpret_cast<const float*>(xb + (w[k] & 0xFFFCu));
            if (ROUND) xv[k] = round_half_away_f(xv[k]);
        }
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            acc = fmaf(__uint_as_float(w[k] & 0xFFFF0000u), xv[k], acc);
            if (w[k] & 1u) {
                *resq = acc;
                resq += 32;
                acc = 0.f;
            }
        }
    }
#endif
#pragma unroll 4
    for (; e < slots; ++e) {
        const uint32_t w = wl[e * 32];
        float xv = *reinterpret_cast<const float*>(xb + (w & 0xFFFCu));
        if (ROUND) xv = round_half_away_f(xv);
        acc = fmaf(__uint_as_float(w & 0xFFFF0000u), xv, acc);   // bf16 B entry; PAD words carry 0
        if (w & 1u) {
            *resq = acc;
            resq += 32;
            acc = 0.f;
        }
    }
}

// Forward outputs from the result queue: whole rows directly, split rows summed over their pieces in piece
// order (fixed; reads other lanes' queue entries, hence the warp barrier).
// store(place, row, value): whole rows at their forward place q * 32 + lane (contiguous per q, conflict-free),
// split rows at qf * 32 + f.
template <typename Store>
__device__ __forceinline__ void ell_rows(const SparseB& sb, const int* __restrict__ ownf, const int* __restrict__ fix,
                                         const int* __restrict__ fixpos, const float* __restrict__ res, int lane,
                                         Store store) {
    for (int q = 0; q < sb.qf; ++q) {
        const int o = ownf[q * 32 + lane];
        if (o >= 0) store(q * 32 + lane, o, res[q * 32 + lane]);
    }
    if (sb.nfix == 0) return;
    __syncwarp();
    for (int f = lane; f < sb.nfix; f += 32) {
        const int o = fix[3 * f], b = fix[3 * f + 1], c = fix[3 * f + 2];
        float acc = 0.f;
        for (int k = 0; k < c; ++k) acc += res[fixpos[b + k]];
        store(sb.qf * 32 + f, o, acc);
    }
}

template <int QD>
__global__ void __launch_bounds__(QD > 16 ? 512 : 1024, 1) descent_simt_kernel(const DescentParams p, int per_warp_words) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    const int n = p.n, d = p.d;
    const SparseB& sb = p.sb;
    const int Lf = sb.Lf, Lb = sb.Lb;
    // block-shared: forward ELL | backward ELL | row pieces (qf x 32) | coordinates (QD x 32) | fixups | places of s
    uint32_t* ellf = reinterpret_cast<uint32_t*>(smem_raw);
    uint32_t* ellb = ellf + Lf * 32;
    int* ownf = reinterpret_cast<int*>(ellb + Lb * 32);
    int* ownb = ownf + sb.qf * 32;
    int* fix = ownb + QD * 32;
    int* fixpos = fix + 3 * sb.nfix;
    int* poss = fixpos + sb.nfixpos;
    // (at least one row of B+ in fp64: the start computation stages B+ here before the schedules are loaded)
    const int shared_words = max((Lf + Lb + sb.qf + QD) * 32 + ((3 * sb.nfix + sb.nfixpos + n + 1) & ~1), 2 * n);

    // per warp, in owner order (sparse_ell.h / capi): z [QD*32] | s, then the g row [qf*32 + nfix] | result
    // queue; during the start computation g0 (n doubles) sits behind z (per_warp_words >= QD*32 + 2n). The
    // harvest gathers round(z) straight from z, so no rounded copy of the iterate is kept.
    const int s_words = sb.qf * 32 + sb.nfix;
    float* zsh = reinterpret_cast<float*>(smem_raw) + shared_words + (size_t)wid * per_warp_words;
    float* ssh = zsh + QD * 32;
    float* res = ssh + s_words;
    double* g0sh = reinterpret_cast<double*>(ssh);   // shared_words, per_warp_words and QD*32 are even

    const int64_t local = (int64_t)blockIdx.x * nwarps + wid;
    const bool active = local < p.count;
    const int64_t gi = p.begin + local;

    // ---- start (Alg. 3 lines 4-5): g0 in fp64 (counter RNG), z0 = B+ g0 in fp64 ----
    // The block streams B+ once through the (not yet loaded) schedule area, a few rows at a time, and every
    // warp takes the dot products of its own start with them: B+ is read from L2 once per block instead of
    // once per start (C3: 672 KB per start before). Each dot product: lanes stride k, fixed-order reduction.
    for (int k = lane; k < QD * 32; k += 32) zsh[k] = 0.f;   // unused places hold z = 0 forever
    __syncwarp();
    if (p.Z0_in) {   // starts precomputed by a DGEMM on the host side of the launch (large n d)
        if (active)
            for (int j = lane; j < d; j += 32) zsh[sb.pos_z[j]] = (float)p.Z0_in[local * d + j];
    } else {
    if (active)
        for (int k = lane; k < n; k += 32) g0sh[k] = start_coord(counter_uniform(p.seed, gi, k, n), p.lo[k], p.hi[k]);
    __syncwarp();
    {
        double* stage = reinterpret_cast<double*>(smem_raw);
        const int R = max(1, (shared_words / 2) / n);   // B+ rows per chunk (shared_words is even)
        for (int j0 = 0; j0 < d; j0 += R) {
            const int rows = min(R, d - j0);
            __syncthreads();
            for (int e = threadIdx.x; e < rows * n; e += blockDim.x) stage[e] = p.Bp[(size_t)j0 * n + e];
            __syncthreads();
            if (!active) continue;
            for (int r = 0; r < rows; ++r) {
                const double* br = stage + (size_t)r * n;
                double acc = 0.0;
                for (int k = lane; k < n; k += 32) acc = fma(br[k], g0sh[k], acc);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
                if (lane == 0) {
                    const int j = j0 + r;
                    zsh[sb.pos_z[j]] = (float)acc;
                    if (p.Z0_out) p.Z0_out[local * d + j] = acc;
                }
            }
        }
        __syncthreads();
    }
    }
    for (int k = threadIdx.x; k < Lf * 32; k += blockDim.x) ellf[k] = sb.ell_f[k];
    for (int k = threadIdx.x; k < Lb * 32; k += blockDim.x) ellb[k] = sb.ell_b[k];
    for (int k = threadIdx.x; k < sb.qf * 32; k += blockDim.x) ownf[k] = sb.own_f[k];
    for (int k = threadIdx.x; k < QD * 32; k += blockDim.x) ownb[k] = k < sb.qd * 32 ? sb.own_b[k] : -1;
    for (int k = threadIdx.x; k < 3 * sb.nfix; k += blockDim.x) fix[k] = sb.fix[k];
    for (int k = threadIdx.x; k < sb.nfixpos; k += blockDim.x) fixpos[k] = sb.fixpos[k];
    for (int k = threadIdx.x; k < n; k += blockDim.x) poss[k] = sb.pos_s[k];
    __syncthreads();
    if (!active) return;
    for (int k = QD * 32 + lane; k < per_warp_words; k += 32) zsh[k] = 0.f;   // g0 is dead: clear s, queue
    __syncwarp();
    const int* jq = ownb + lane;   // jq[q * 32]: this lane's q-th coordinate (shared table, conflict-free)
    const uint32_t* wf = ellf + lane;
    const uint32_t* wb = ellb + lane;
    float m[QD], v[QD];
#pragma unroll
    for (int q = 0; q < QD; ++q) m[q] = v[q] = 0.f;

    const float b1 = p.beta1, b2 = p.beta2, omb1 = p.omb1, omb2 = p.omb2, lam1 = p.lam1, lam2 = p.lam2, eps = p.eps;
    const float lr = p.lr;
    const int opt = p.opt;
    for (int t = 0; t < p.T; ++t) {
        // forward: s_i = sign((B z)_i)
        ell_run(wf, Lf, zsh, res + lane);
        // s = sign(Bz): whole rows sit at their queue place (owner order), so every place is converted without
        // looking up its row (places of split pieces get a value no gather reads); split rows via the fixups
        for (int q = 0; q < sb.qf; ++q) ssh[q * 32 + lane] = fsign(res[q * 32 + lane]);
        if (sb.nfix) {
            __syncwarp();
            for (int f = lane; f < sb.nfix; f += 32) {
                const int b = fix[3 * f + 1], c = fix[3 * f + 2];
                float acc = 0.f;
                for (int k = 0; k < c; ++k) acc += res[fixpos[b + k]];
                ssh[sb.qf * 32 + f] = fsign(acc);
            }
        }
        // lowest-index argmax of |z| (λ2 term, Eq. 3), over this lane's coordinates then the warp
        float best = -1.f;
        int bestj = 0x7fffffff, bestp = 0;
#pragma unroll
        for (int q = 0; q < QD; ++q) {   // unused places (j < 0) hold z = 0 and lose every tie
            const int j = jq[q * 32];
            const int jj = j >= 0 ? j : 0x7ffffffe;
            const float aa = fabsf(zsh[q * 32 + lane]);
            if (aa > best || (aa == best && jj < bestj)) {
                best = aa;
                bestj = jj;
                bestp = q * 32 + lane;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const float ob = __shfl_xor_sync(0xffffffffu, best, off);
            const int oj = __shfl_xor_sync(0xffffffffu, bestj, off);
            const int op = __shfl_xor_sync(0xffffffffu, bestp, off);
            if (ob > best || (ob == best && oj < bestj)) {
                best = ob;
                bestj = oj;
                bestp = op;
            }
        }
        // λ2 term (Eq. 3), active while max|z| < 1, on the lowest-index argmax coordinate only
        float extra = 0.f;
        if (best < 1.f) {
            const float zb = zsh[bestp];
            extra = -lam2 * fsign(zb) / fmaxf(zb * zb, 1e-8f);
        }
        __syncwarp();
        // backward: Γ = B^T s; the lane's q-th piece is its q-th coordinate, left in its own queue slot
        ell_run(wb, Lb, ssh, res + lane);
        // penalties + Adam (reading #9) on this lane's coordinates.
        // Branch-free: unused places update the scratch coordinate d (Γ = 0, z = 0: it stays 0).
        const float4 st = p.step_tab[t];
        // the first iterate is always harvested (no previous round(z)); final-only mode (reading #25): the last
        const bool final_step = t == p.T - 1;
        bool changed = p.harvest_final ? final_step : (t == 0);
#pragma unroll
        for (int q = 0; q < QD; ++q) {
            const int j = jq[q * 32];
            const int pl = q * 32 + lane;
            const float zz = zsh[pl];
            // (the queue slot of an unused place may hold a forward piece sum: read 0 there)
            // λ1 d/dz (z - floor z)(ceil z - z) = ceil z + floor z - 2z = sign(z - r) - 2 (z - r), r = round(z)
            // (z - r is exact; both forms round the same real value once), r also serves the change test
            const float ro = round_half_away_f(zz);
            const float dd = zz - ro;
            const float sd = dd != 0.f ? copysignf(1.f, dd) : 0.f;
            float gr = fmaf(lam1, fmaf(-2.f, dd, sd), j >= 0 ? res[q * 32 + lane] : 0.f);
            gr += (j == bestj) ? extra : 0.f;
            float zn;
            if (opt == 0) {   // Adam (reading #9)
                m[q] = fmaf(b1, m[q], omb1 * gr);
                v[q] = fmaf(b2, v[q], omb2 * gr * gr);
                const float den = fmaf(umma::sqrt_approx(v[q]), st.z, eps);
                zn = fmaf(-st.x * m[q], umma::rcp_approx(den), zz);
            } else if (opt == 1) {   // GD (reading #24): two roundings, as z - lr * g in fp32
                zn = __fsub_rn(zz, __fmul_rn(lr, gr));
            } else {                 // sign-GD
                zn = __fsub_rn(zz, gr > 0.f ? lr : (gr < 0.f ? -lr : 0.f));
            }
            zsh[pl] = zn;
            const float rn = round_half_away_f(zn);
            changed |= rn != ro;
        }
        __syncwarp();
        if (!p.harvest || (p.harvest_final && !final_step)) continue;
        // harvest (Alg. 3 lines 9-10) when round(z) changed: g = B r, box, g != 0, canonical sign
        if (!__any_sync(0xffffffffu, changed)) continue;
        bool ok = true;
        ell_run<true>(wf, Lf, zsh, res + lane);   // g = B round(z)
        ell_rows(sb, ownf, fix, fixpos, res, lane, [&](int pl, int i, float acc) {
            const int gv = (int)acc;
            ok &= (abs(gv) <= p.box[i]);
            ssh[pl] = (float)gv;   // s is dead until the next forward: reuse it as the g row (row i at place pl)
        });
        ok = __all_sync(0xffffffffu, ok);
        if (!ok) continue;
        __syncwarp();
        int firstsign = 0;
        for (int i0 = 0; i0 < n && !firstsign; i0 += 32) {
            const int i = i0 + lane;
            const int gv = i < n ? (int)ssh[poss[i]] : 0;
            const unsigned msk = __ballot_sync(0xffffffffu, gv != 0);
            if (msk) firstsign = __shfl_sync(0xffffffffu, gv, __ffs(msk) - 1) > 0 ? 1 : -1;
        }
        if (!firstsign) continue;  // g = 0
        unsigned long long slot = 0;
        if (lane == 0) slot = atomicAdd(p.cand_count, 1ULL);
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if ((int64_t)slot < p.cand_cap) {
            int8_t* dst = p.cand + (size_t)slot * p.n_pad;
            for (int i = lane; i < p.n_pad; i += 32) dst[i] = (i < n) ? (int8_t)(firstsign * (int)ssh[poss[i]]) : (int8_t)0;
        }
        __syncwarp();
    }
    if (p.Z_out) {
#pragma unroll
        for (int q = 0; q < QD; ++q)
            if (jq[q * 32] >= 0) p.Z_out[local * d + jq[q * 32]] = zsh[q * 32 + lane];
    }
}

template <int QD>
cudaError_t launch_qd(const DescentParams& p, cudaStream_t s) {
    const SparseB& sb = p.sb;
    const int n = p.n;
    const int per_warp_words =
        (std::max(QD * 32 + sb.qf * 32 + sb.nfix + 32 * std::max(sb.qf, QD), QD * 32 + 2 * n) + 1) & ~1;
    const size_t shared_bytes =
        (size_t)std::max((sb.Lf + sb.Lb + sb.qf + QD) * 32 + ((3 * sb.nfix + sb.nfixpos + n + 1) & ~1), 2 * n) * 4;
    int dev = 0, smem_sm = 0, smem_blk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&smem_blk, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    cudaError_t e = cudaFuncGetAttributes(&fa, descent_simt_kernel<QD>);
    if (e != cudaSuccess) return e;
    const int warps_by_regs = 65536 / (32 * std::max(fa.numRegs, 1));
    // warps per block: maximise resident warps per SM (shared memory and registers); the ELL is staged once
    // per block, so among equal occupancies the smallest block wins (shorter tail)
    int best_w = 0, best_res = -1;
    for (int w = 4; w <= fa.maxThreadsPerBlock / 32; w += 4) {
        const size_t bytes = shared_bytes + (size_t)w * per_warp_words * 4;
        if (bytes > (size_t)smem_blk) break;
        const int blocks = std::min<int>({(int)(smem_sm / (bytes + 1024)), 2048 / (32 * w), warps_by_regs / w});
        const int res = blocks * w;
        if (res > best_res) {
            best_res = res;
            best_w = w;
        }
    }
    if (best_w == 0) return cudaErrorInvalidValue;   // the ELL does not fit in shared memory
    const size_t smem = shared_bytes + (size_t)best_w * per_warp_words * 4;
    e = cudaFuncSetAttribute(descent_simt_kernel<QD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t blocks = (p.count + best_w - 1) / best_w;
    descent_simt_kernel<QD><<<(unsigned)blocks, best_w * 32, smem, s>>>(p, per_warp_words);
    return cudaGetLastError();
}

__global__ void start_g0_kernel(const DescentParams p, double* __restrict__ g0) {
    const int n = p.n;
    const int64_t total = p.count * n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = e / n;
        const int k = (int)(e - s * n);
        g0[e] = start_coord(counter_uniform(p.seed, p.begin + s, k, n), p.lo[k], p.hi[k]);
    }
}

}  // namespace

cudaError_t launch_start_g0(const DescentParams& p, double* g0, cudaStream_t s) {
    if (p.count <= 0) return cudaSuccess;
    const int64_t total = p.count * p.n;
    start_g0_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 32), 256, 0, s>>>(p, g0);
    return cudaGetLastError();
}

cudaError_t launch_descent_simt(const DescentParams& p, cudaStream_t s) {
    if (p.count <= 0) return cudaSuccess;
    const int qd = p.sb.qd;
    if (qd <= 1) return launch_qd<1>(p, s);
    if (qd <= 2) return launch_qd<2>(p, s);
    if (qd <= 4) return launch_qd<4>(p, s);
    if (qd <= 8) return launch_qd<8>(p, s);
    if (qd <= 12) return launch_qd<12>(p, s);
    if (qd <= 16) return launch_qd<16>(p, s);
    if (qd <= 24) return launch_qd<24>(p, s);
    if (qd <= 32) return launch_qd<32>(p, s);
    return cudaErrorInvalidValue;
}

}  // namespace maple
