// Tensor-core (tcgen05 / TMEM) descent + harvest kernel for sm_100a — the fast path of Algorithm 3's
// inner loop, 128 starts per CTA with the whole Adam state resident on chip for all T
// steps (no HBM traffic per step).
//
// Per CTA: 128 starts = the UMMA M dimension = the 128 TMEM lanes. 256 threads: thread (warp w, lane l)
// owns start row 32 (w % 4) + l and the column half w / 4 (TMEM lane quadrant rule of tcgen05.ld).
// Per step t (Eq. 3; Adam; harvest):
//   MMA  G = Z B^T            kind::tf32, Z split into hi + lo TF32 terms (B is exact in TF32), fp32 accum
//   MMA  H = round(z_{t-1}) B^T   kind::f16 (exact: small integers, fp32 accum) — the harvest expansion
//   epi  harvest rows whose round(z) changed: g = H row, keep iff g != 0 and |g| <= u - l, canonical sign
//   epi  S = sign(G)  (sign(0) = 0) -> f16 operand in shared memory
//   MMA  Γ = S B             kind::f16 (exact) — the ℓ1 subgradient B^T sign(Bz)
//   epi  grad = Γ + λ1 (ceil z + floor z - 2z) + λ2 term on the lowest-index argmax |z_k| (||z||_inf < 1);
//        Adam (torch formula) on registers; write Z_hi, Z_lo, round(z) operands for the next step.
// One elected thread issues every tcgen05.mma; completion is signalled through tcgen05.commit -> mbarrier.
#include <cuda_fp16.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "tc_umma.cuh"

namespace maple {

namespace {

using namespace umma;

constexpr int kRows = 128;
constexpr int kThreads = 256;
constexpr uint32_t kTmemCols = 256;

__host__ __device__ constexpr uint32_t al1k(uint32_t x) { return (x + 1023u) & ~1023u; }

template <int NP, int DP>
struct Lay {
    static constexpr int NH = NP / 2, DH = DP / 2;
    static constexpr uint32_t B32 = 0;                                   // NP x DP tf32 (forward B)
    static constexpr uint32_t B16 = al1k(B32 + NP * DP * 4);             // NP x DP f16 (harvest B)
    static constexpr uint32_t BT16 = al1k(B16 + NP * DP * 2);            // DP x NP f16 (backward B)
    static constexpr uint32_t ZHI = al1k(BT16 + DP * NP * 2);            // 128 x DP tf32 (A, hi)
    static constexpr uint32_t ZLO = al1k(ZHI + kRows * DP * 4);          // 128 x DP tf32 (A, lo)
    static constexpr uint32_t R16 = al1k(ZLO + kRows * DP * 4);          // 128 x DP f16 (A, harvest)
    static constexpr uint32_t S16 = al1k(R16 + kRows * DP * 2);          // 128 x NP f16 (A, backward)
    static constexpr uint32_t GB = al1k(S16 + kRows * NP * 2);           // 128 x NP int8 harvested rows
    static constexpr uint32_t BOX = al1k(GB + kRows * NP);               // NP int32
    static constexpr uint32_t PAIR = al1k(BOX + NP * 4);                 // pair exchange
    static constexpr uint32_t PAIR_BYTES = 2 * 2 * kRows * 4 * 2 + 3 * 2 * kRows;
    static constexpr uint32_t G0_ALIAS = ZHI;                            // fp64 128 x (NP+1) staging
    static constexpr uint32_t G0_BYTES = kRows * (NP + 1) * 8;
    static constexpr bool G0_FITS = G0_BYTES <= GB - ZHI;
    static constexpr uint32_t G0 = G0_FITS ? G0_ALIAS : al1k(PAIR + PAIR_BYTES);
    static constexpr uint32_t MBAR = al1k((G0_FITS ? PAIR + PAIR_BYTES : G0 + G0_BYTES));
    static constexpr uint32_t TOTAL = MBAR + 64;
};

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

template <int NP, int DP>
__global__ void __launch_bounds__(kThreads, 1) descent_tc_kernel(const DescentParams p) {
    using L = Lay<NP, DP>;
    constexpr int NH = L::NH, DH = L::DH;
    extern __shared__ __align__(1024) unsigned char sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int quad = warp & 3, half = warp >> 2;
    const int row = quad * 32 + lane;
    const int64_t local = (int64_t)blockIdx.x * kRows + row;
    const bool active = local < p.count;
    const int64_t gi = p.begin + local;
    const int n = p.n, d = p.d;

    float* amax = reinterpret_cast<float*>(sm + L::PAIR);        // [parity][half][row]
    int* aidx = reinterpret_cast<int*>(amax + 2 * 2 * kRows);    // [parity][half][row]
    uint8_t* chg = reinterpret_cast<uint8_t*>(aidx + 2 * 2 * kRows);  // [half][row]
    uint8_t* okf = chg + 2 * kRows;
    uint8_t* nzf = okf + 2 * kRows;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + L::MBAR);
    uint32_t* tbase_sh = reinterpret_cast<uint32_t*>(mbar + 2);
    int32_t* boxs = reinterpret_cast<int32_t*>(sm + L::BOX);
    int8_t* gbuf = reinterpret_cast<int8_t*>(sm + L::GB);

    // ---- setup: TMEM, barriers, B operands (exact small integers) ----
    if (warp == 0) tmem_alloc(tbase_sh, kTmemCols);
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        fence_mbar_init();
    }
    for (int e = tid; e < NP * DP; e += kThreads) {
        const int i = e / DP, k = e % DP;
        const float v = (i < n && k < d) ? p.B_nd[(size_t)i * d + k] : 0.f;
        *reinterpret_cast<float*>(sm + L::B32 + op_offset(i, k >> 2, NP) + (k & 3) * 4) = v;
        *reinterpret_cast<__half*>(sm + L::B16 + op_offset(i, k >> 3, NP) + (k & 7) * 2) = __float2half_rn(v);
        *reinterpret_cast<__half*>(sm + L::BT16 + op_offset(k, i >> 3, DP) + (i & 7) * 2) = __float2half_rn(v);
    }
    for (int i = tid; i < NP; i += kThreads) boxs[i] = i < n ? p.box[i] : 0;
    // ---- starts (Alg. 3 lines 4-5): g0 in fp64 from the counter RNG, z0 = B+ g0 ----
    double* g0s = reinterpret_cast<double*>(sm + L::G0);
    for (int k = half * NH; k < (half + 1) * NH; ++k) {
        double g = 0.0;
        if (active && k < n) g = start_coord(counter_uniform(p.seed, gi, k, n), p.lo[k], p.hi[k]);
        g0s[row * (NP + 1) + k] = g;
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tbase = *tbase_sh;
    float z[DH], m[DH], v[DH];
#pragma unroll
    for (int q = 0; q < DH; ++q) {
        const int j = half * DH + q;
        double acc = 0.0;
        if (j < d && active) {
            const double* bp = p.Bp + (size_t)j * n;
            for (int k = 0; k < n; ++k) acc = fma(bp[k], g0s[row * (NP + 1) + k], acc);
            if (p.Z0_out) p.Z0_out[local * d + j] = acc;
        }
        z[q] = (float)acc;
        m[q] = 0.f;
        v[q] = 0.f;
    }
    __syncthreads();  // g0 staging may alias the operand area
    // operands of step 1 + argmax of |z0|
    auto write_z = [&](int parity) {
        float lmax = -1.f;
        int lidx = 0;
#pragma unroll
        for (int c = 0; c < DH / 4; ++c) {
            float4 hi, lo;
            float* h = &hi.x;
            float* o = &lo.x;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float zz = z[4 * c + e];
                h[e] = to_tf32(zz);
                o[e] = to_tf32(zz - h[e]);
                const float a = fabsf(zz);
                if (a > lmax) {
                    lmax = a;
                    lidx = half * DH + 4 * c + e;
                }
            }
            const uint32_t off = op_offset(row, half * (DH / 4) + c, kRows);
            *reinterpret_cast<float4*>(sm + L::ZHI + off) = hi;
            *reinterpret_cast<float4*>(sm + L::ZLO + off) = lo;
        }
#pragma unroll
        for (int c = 0; c < DH / 8; ++c) {
            uint4 w;
            uint32_t* wp = &w.x;
#pragma unroll
            for (int e = 0; e < 4; ++e)
                wp[e] = pack_h2((float)round_half_away(z[8 * c + 2 * e]), (float)round_half_away(z[8 * c + 2 * e + 1]));
            *reinterpret_cast<uint4*>(sm + L::R16 + op_offset(row, half * (DH / 8) + c, kRows)) = w;
        }
        amax[(parity * 2 + half) * kRows + row] = lmax;
        aidx[(parity * 2 + half) * kRows + row] = lidx;
    };
    write_z(0);

    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t tG = tbase + lane_off, tH = tbase + NP + lane_off, tGam = tbase + 2 * NP + lane_off;
    const uint32_t sZHI = smem_u32(sm + L::ZHI), sZLO = smem_u32(sm + L::ZLO), sR = smem_u32(sm + L::R16);
    const uint32_t sS = smem_u32(sm + L::S16), sB32 = smem_u32(sm + L::B32), sB16 = smem_u32(sm + L::B16);
    const uint32_t sBT = smem_u32(sm + L::BT16);
    constexpr uint32_t LBO_A = kRows * 16, LBO_N = NP * 16, LBO_D = DP * 16, SBO = 128;
    constexpr uint32_t ID_FWD = idesc(2, kRows, NP), ID_HARV = idesc(0, kRows, NP), ID_BWD = idesc(0, kRows, DP);

    uint32_t phA = 0, phB = 0;
    const int T = p.T;
    const int t_end = p.harvest ? T + 1 : T;
    for (int t = 1; t <= t_end; ++t) {
        const bool do_fwd = t <= T;
        const bool do_harv = p.harvest && t >= 2;
        fence_proxy_async();
        fence_before();
        __syncthreads();  // B1: operands written, pair info visible
        if (tid == 0) {
            fence_after();
            if (do_fwd) {
#pragma unroll
                for (int kk = 0; kk < DP / 8; ++kk)
                    mma_tf32(tbase, desc(sZHI + kk * 2 * LBO_A, LBO_A, SBO), desc(sB32 + kk * 2 * LBO_N, LBO_N, SBO),
                             ID_FWD, kk > 0);
#pragma unroll
                for (int kk = 0; kk < DP / 8; ++kk)
                    mma_tf32(tbase, desc(sZLO + kk * 2 * LBO_A, LBO_A, SBO), desc(sB32 + kk * 2 * LBO_N, LBO_N, SBO),
                             ID_FWD, 1);
            }
            if (do_harv) {
#pragma unroll
                for (int kk = 0; kk < DP / 16; ++kk)
                    mma_f16(tbase + NP, desc(sR + kk * 2 * LBO_A, LBO_A, SBO), desc(sB16 + kk * 2 * LBO_N, LBO_N, SBO),
                            ID_HARV, kk > 0);
            }
            commit(&mbar[0]);
        }
        mbar_wait(&mbar[0], phA);
        phA ^= 1;
        fence_after();
        // ---- harvest of z_{t-1}: read H only for rows whose round(z) changed ----
        bool row_chg = false;
        if (do_harv) {
            const uint8_t cf = chg[row] | chg[kRows + row];
            row_chg = active && cf == 1;
            if (__any_sync(0xffffffffu, row_chg)) {
                uint32_t r[NH];
#pragma unroll
                for (int c = 0; c < NH / 8; ++c) ld8(tH + half * NH + 8 * c, &r[8 * c]);
#pragma unroll
                for (int c = 0; c < NH / 8; ++c) wait8(&r[8 * c]);
                bool ok = true, nz = false;
#pragma unroll
                for (int c = 0; c < NH / 4; ++c) {
                    uint32_t w = 0;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int i = half * NH + 4 * c + e;
                        const int g = (int)__uint_as_float(r[4 * c + e]);
                        ok &= abs(g) <= boxs[i];
                        nz |= g != 0;
                        w |= ((uint32_t)(g & 0xFF)) << (8 * e);
                    }
                    *reinterpret_cast<uint32_t*>(gbuf + row * NP + half * NH + 4 * c) = w;
                }
                okf[half * kRows + row] = ok;
                nzf[half * kRows + row] = nz;
            }
        }
        // ---- S = sign(B z) from the forward accumulator ----
        if (do_fwd) {
            uint32_t r[NH];
#pragma unroll
            for (int c = 0; c < NH / 8; ++c) ld8(tG + half * NH + 8 * c, &r[8 * c]);
#pragma unroll
            for (int c = 0; c < NH / 8; ++c) wait8(&r[8 * c]);
#pragma unroll
            for (int c = 0; c < NH / 8; ++c) {
                uint4 w;
                uint32_t* wp = &w.x;
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    wp[e] = pack_h2(fsign(__uint_as_float(r[8 * c + 2 * e])), fsign(__uint_as_float(r[8 * c + 2 * e + 1])));
                *reinterpret_cast<uint4*>(sm + L::S16 + op_offset(row, half * (NH / 8) + c, kRows)) = w;
            }
        }
        fence_proxy_async();
        fence_before();
        __syncthreads();  // B2: S written, harvest flags visible
        if (tid == 0 && do_fwd) {
            fence_after();
#pragma unroll
            for (int kk = 0; kk < NP / 16; ++kk)
                mma_f16(tbase + 2 * NP, desc(sS + kk * 2 * LBO_A, LBO_A, SBO), desc(sBT + kk * 2 * LBO_D, LBO_D, SBO),
                        ID_BWD, kk > 0);
            commit(&mbar[1]);
        }
        // ---- harvest write-out (half 0; overlaps the backward MMA) ----
        if (do_harv && half == 0) {
            const bool want = row_chg && okf[row] && okf[kRows + row] && (nzf[row] | nzf[kRows + row]);
            const unsigned mask = __ballot_sync(0xffffffffu, want);
            if (mask) {
                const int leader = __ffs(mask) - 1;
                unsigned long long base = 0;
                if (lane == leader) base = atomicAdd(p.cand_count, (unsigned long long)__popc(mask));
                base = __shfl_sync(0xffffffffu, base, leader);
                if (want) {
                    const unsigned long long slot = base + __popc(mask & ((1u << lane) - 1u));
                    const uint32_t* src = reinterpret_cast<const uint32_t*>(gbuf + row * NP);
                    int sgn = 0;
#pragma unroll
                    for (int c = 0; c < NP / 4; ++c) {
                        const uint32_t w = src[c];
                        if (!sgn && w) sgn = ((int8_t)(w >> (8 * ((__ffs(w) - 1) >> 3)))) > 0 ? 1 : -1;
                    }
                    if ((int64_t)slot < p.cand_cap) {
                        uint4* dst = reinterpret_cast<uint4*>(p.cand + (size_t)slot * p.n_pad);
                        const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
                        for (int c = 0; c < NP / 16; ++c) {
                            uint4 w = s4[c];
                            if (sgn < 0) {
                                w.x = __vneg4(w.x);
                                w.y = __vneg4(w.y);
                                w.z = __vneg4(w.z);
                                w.w = __vneg4(w.w);
                            }
                            dst[c] = w;
                        }
                    }
                }
            }
        }
        if (!do_fwd) break;
        mbar_wait(&mbar[1], phB);
        phB ^= 1;
        fence_after();
        // ---- Adam step on Γ (Eq. 3 subgradient) ----
        uint32_t r[DH];
#pragma unroll
        for (int c = 0; c < DH / 8; ++c) ld8(tGam + half * DH + 8 * c, &r[8 * c]);
#pragma unroll
        for (int c = 0; c < DH / 8; ++c) wait8(&r[8 * c]);
        const int par = (t - 1) & 1;
        const float a0 = amax[(par * 2 + 0) * kRows + row], a1 = amax[(par * 2 + 1) * kRows + row];
        const int i0 = aidx[(par * 2 + 0) * kRows + row], i1 = aidx[(par * 2 + 1) * kRows + row];
        const float zinf = a1 > a0 ? a1 : a0;
        const int kbest = a1 > a0 ? i1 : i0;
        const float2 st = p.step_tab[t - 1];
        const float b1 = p.beta1, b2 = p.beta2, omb1 = p.omb1, omb2 = p.omb2;
        bool ch = (t == 1), big = false;
#pragma unroll
        for (int q = 0; q < DH; ++q) {
            const int j = half * DH + q;
            const float zz = z[q];
            float g = __uint_as_float(r[q]) + p.lam1 * (ceilf(zz) + floorf(zz) - 2.f * zz);
            if (zinf < 1.f && j == kbest) g += -p.lam2 * fsign(zz) / fmaxf(zz * zz, 1e-8f);
            m[q] = b1 * m[q] + omb1 * g;
            v[q] = b2 * v[q] + omb2 * g * g;
            const float denom = sqrtf(v[q]) / st.y + p.eps;
            const float zn = zz - st.x * m[q] / denom;
            const int rn = round_half_away(zn);
            ch |= rn != round_half_away(zz);
            big |= abs(rn) > 2048;
            z[q] = zn;
        }
        // bit 0: round(z) changed; bit 1: some |round(z_j)| > 2048 (not exact in the f16 harvest operand).
        // The host only selects this kernel when max_j sum_i |B+_ji| (u_i - l_i) < 2048, so such an
        // iterate cannot map to a g inside the box and skipping it is exact.
        chg[half * kRows + row] = (uint8_t)((ch ? 1 : 0) | (big ? 2 : 0));
        write_z(t & 1);
    }
    if (p.Z_out && active) {
#pragma unroll
        for (int q = 0; q < DH; ++q) {
            const int j = half * DH + q;
            if (j < d) p.Z_out[local * d + j] = z[q];
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 0) {
        fence_after();
        tmem_dealloc(tbase, kTmemCols);
    }
}

template <int NP, int DP>
cudaError_t launch_np_dp(const DescentParams& p, cudaStream_t s) {
    using L = Lay<NP, DP>;
    // at least 80 KB so that at most two CTAs (2 x 256 TMEM columns) share an SM
    const uint32_t smem = L::TOTAL < 80 * 1024 ? 80 * 1024 : L::TOTAL;
    cudaError_t e = cudaFuncSetAttribute(descent_tc_kernel<NP, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const int64_t blocks = (p.count + kRows - 1) / kRows;
    descent_tc_kernel<NP, DP><<<(unsigned)blocks, kThreads, smem, s>>>(p);
    return cudaGetLastError();
}

// ---- self-test of the UMMA descriptor / layout conventions (single tile, exact small integers) ----
__global__ void umma_selftest_kernel(const float* A1, const float* B1, float* D1, const float* A2, const float* B2,
                                     float* D2) {
    // D1 (128 x 64) = A1 (128 x 48) B1^T (B1: 64 x 48)  kind::tf32;  D2 (128 x 48) = A2 (128 x 64) B2^T  kind::f16
    extern __shared__ __align__(1024) unsigned char sm[];
    uint8_t* a1 = sm;                   // 128 x 48 fp32 = 24576
    uint8_t* b1 = sm + 24576;           // 64 x 48 fp32 = 12288
    uint8_t* a2 = sm + 36864;           // 128 x 64 f16 = 16384
    uint8_t* b2 = sm + 53248;           // 48 x 64 f16 = 6144
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + 60416);
    uint32_t* tb = reinterpret_cast<uint32_t*>(sm + 60432);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) tmem_alloc(tb, 128);
    if (tid == 0) {
        mbar_init(mbar, 1);
        fence_mbar_init();
    }
    for (int e = tid; e < 128 * 48; e += blockDim.x) {
        const int r = e / 48, k = e % 48;
        *reinterpret_cast<float*>(a1 + op_offset(r, k >> 2, 128) + (k & 3) * 4) = A1[e];
    }
    for (int e = tid; e < 64 * 48; e += blockDim.x) {
        const int r = e / 48, k = e % 48;
        *reinterpret_cast<float*>(b1 + op_offset(r, k >> 2, 64) + (k & 3) * 4) = B1[e];
    }
    for (int e = tid; e < 128 * 64; e += blockDim.x) {
        const int r = e / 64, k = e % 64;
        *reinterpret_cast<__half*>(a2 + op_offset(r, k >> 3, 128) + (k & 7) * 2) = __float2half_rn(A2[e]);
    }
    for (int e = tid; e < 48 * 64; e += blockDim.x) {
        const int r = e / 64, k = e % 64;
        *reinterpret_cast<__half*>(b2 + op_offset(r, k >> 3, 48) + (k & 7) * 2) = __float2half_rn(B2[e]);
    }
    fence_proxy_async();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tbase = *tb;
    if (tid == 0) {
        for (int kk = 0; kk < 48 / 8; ++kk)
            mma_tf32(tbase, desc(smem_u32(a1) + kk * 2 * 2048, 2048, 128), desc(smem_u32(b1) + kk * 2 * 1024, 1024, 128),
                     idesc(2, 128, 64), kk > 0);
        for (int kk = 0; kk < 64 / 16; ++kk)
            mma_f16(tbase + 64, desc(smem_u32(a2) + kk * 2 * 2048, 2048, 128), desc(smem_u32(b2) + kk * 2 * 768, 768, 128),
                    idesc(0, 128, 48), kk > 0);
        commit(mbar);
    }
    mbar_wait(mbar, 0);
    fence_after();
    const int row = (warp & 3) * 32 + lane;
    const uint32_t ta = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    for (int c = 0; c < 64 / 8; ++c) {
        uint32_t r[8];
        ld8(ta + 8 * c, r);
        wait8(r);
        for (int e = 0; e < 8; ++e) D1[row * 64 + 8 * c + e] = __uint_as_float(r[e]);
    }
    for (int c = 0; c < 48 / 8; ++c) {
        uint32_t r[8];
        ld8(ta + 64 + 8 * c, r);
        wait8(r);
        for (int e = 0; e < 8; ++e) D2[row * 48 + 8 * c + e] = __uint_as_float(r[e]);
    }
    fence_before();
    __syncthreads();
    if (warp == 0) {
        fence_after();
        tmem_dealloc(tbase, 128);
    }
}

}  // namespace

bool descent_tc_supported(int n, int d) {  // shape only; capi also requires the f16 range bound
    const int np = (std::max(n, 16) + 15) / 16 * 16;
    const int dp = (std::max(d, 16) + 15) / 16 * 16;
    return np <= 64 && dp <= 64 && dp <= np;
}

cudaError_t launch_descent_tc(const DescentParams& p, cudaStream_t s) {
    if (p.count <= 0) return cudaSuccess;
    const int np = (std::max(p.n, 16) + 15) / 16 * 16;
    const int dp = (std::max(p.d, 16) + 15) / 16 * 16;
    if (np != p.n_pad) return cudaErrorInvalidValue;
#define MAPLE_TC_CASE(NPV, DPV) \
    if (np == NPV && dp == DPV) return launch_np_dp<NPV, DPV>(p, s);
    MAPLE_TC_CASE(16, 16)
    MAPLE_TC_CASE(32, 16)
    MAPLE_TC_CASE(32, 32)
    MAPLE_TC_CASE(48, 16)
    MAPLE_TC_CASE(48, 32)
    MAPLE_TC_CASE(48, 48)
    MAPLE_TC_CASE(64, 16)
    MAPLE_TC_CASE(64, 32)
    MAPLE_TC_CASE(64, 48)
    MAPLE_TC_CASE(64, 64)
#undef MAPLE_TC_CASE
    return cudaErrorNotSupported;
}

cudaError_t umma_selftest(const float* A1, const float* B1, float* D1, const float* A2, const float* B2, float* D2,
                          cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(umma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    if (e != cudaSuccess) return e;
    umma_selftest_kernel<<<1, 128, 64 * 1024, s>>>(A1, B1, D1, A2, B2, D2);
    return cudaGetLastError();
}

}  // namespace maple
