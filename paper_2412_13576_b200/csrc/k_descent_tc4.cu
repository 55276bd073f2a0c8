// Tensor-core (tcgen05 / TMEM) descent + harvest kernel, 4 threads per start — the same computation as
// k_descent_tc.cu (Algorithm 3's inner loop; Eq. 3; Adam; harvest)
// with twice the threads per CTA.
//
// Why: the 2-thread kernel is latency-bound (about half its issue slots idle at 14 warps per SM, capped by 128
// registers per thread). Here each of the 512 threads of a CTA owns a quarter of a start's columns, so it
// needs <= 64 registers and two CTAs (the TMEM budget: 2 x 256 columns) give 32 warps per SM.
//
// Per CTA: 128 starts = the UMMA M dimension = the 128 TMEM lanes. Thread (warp w, lane l) owns start row
// 32 (w % 4) + l (TMEM lane quadrant rule of tcgen05.ld) and part w / 4 of the columns: NP / 4 columns of G, H,
// S and the candidate row, DP / 4 coordinates of z, m, v. Per step t:
//   MMA  G = Z B^T  (kind::tf32, Z = Z_hi + Z_lo)  and  H = round(z_{t-1}) B^T  (kind::f16, exact)
//   epi  each part: S = sign(G) -> bf16 operand; harvest test of its H columns (box, first nonzero)
//   MMA  Γ = S B  (kind::f16 with bf16 operands, exact) into G's TMEM columns
//   epi  (overlapping that MMA) rows whose round(z) changed and that passed all four parts' tests: one
//        atomic per quad of warps reserves the slots, each part writes its columns of the canonical int8 row
//   epi  grad = Γ + λ1 (ceil z + floor z - 2z) + λ2 term (lowest-index argmax, ||z||_inf < 1); Adam
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "tc_umma.cuh"

namespace maple {

namespace {

using namespace umma;

constexpr int kRows = 128;
constexpr int kParts = 4;
constexpr int kThreads = kRows * kParts;
constexpr uint32_t kTmemCols = 256;

__host__ __device__ constexpr uint32_t al128(uint32_t x) { return (x + 127u) & ~127u; }

template <int NP, int DP>
struct Lay4 {
    static constexpr int NQ = NP / kParts, DQ = DP / kParts;             // multiples of 4
    static constexpr uint32_t B32 = 0;                                   // NP x DP tf32 (forward B)
    static constexpr uint32_t B16 = al128(B32 + NP * DP * 4);            // NP x DP f16 (harvest B)
    static constexpr uint32_t BT16 = al128(B16 + NP * DP * 2);           // DP x NP bf16 (backward B)
    static constexpr uint32_t ZHI = al128(BT16 + DP * NP * 2);           // 128 x DP tf32 (A, hi)
    static constexpr uint32_t ZLO = al128(ZHI + kRows * DP * 4);         // 128 x DP tf32 (A, lo)
    static constexpr uint32_t R16 = al128(ZLO + kRows * DP * 4);         // 128 x DP f16 (A, harvest)
    static constexpr uint32_t S16 = al128(R16 + kRows * DP * 2);         // 128 x NP bf16 (A, backward)
    static constexpr uint32_t BOX = al128(S16 + kRows * NP * 2);         // NP f32 (u - l)
    static constexpr uint32_t PAIR = al128(BOX + NP * 4);                // amax | aidx | chg | hx | slots
    static constexpr uint32_t PAIR_BYTES = 2 * 2 * kParts * kRows * 4 + kRows * 4 + kRows * 4 + kRows * 8;
    static constexpr int KC = 16;                                        // g0 staging chunk (coordinates)
    static constexpr uint32_t G0_BYTES = kRows * (KC + 1) * 8;           // fp64 start staging
    static constexpr bool G0_FITS = G0_BYTES <= BOX - ZHI;
    static constexpr uint32_t G0 = G0_FITS ? ZHI : al128(PAIR + PAIR_BYTES);
    static constexpr uint32_t MBAR = al128(G0_FITS ? PAIR + PAIR_BYTES : G0 + G0_BYTES);
    static constexpr uint32_t TOTAL = MBAR + 64;
    // TMEM columns: G (then Γ, DP <= NP) | H | m | v
    static constexpr uint32_t CG = 0, CX = NP, CM = 2 * NP, CV = 2 * NP + DP;
    static_assert(CV + DP <= kTmemCols, "TMEM budget");
    static_assert(NQ % 4 == 0 && DQ % 4 == 0, "4-column parts");
};

template <int NP, int DP>
__global__ void __launch_bounds__(kThreads, 2) descent_tc4_kernel(const DescentParams p) {
    using L = Lay4<NP, DP>;
    constexpr int NQ = L::NQ, DQ = L::DQ;
    extern __shared__ __align__(1024) unsigned char sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int quad = warp & 3, part = warp >> 2;
    const int row = quad * 32 + lane;
    const int64_t local = (int64_t)blockIdx.x * kRows + row;
    const bool active = local < p.count;
    const int64_t gi = p.begin + local;
    const int n = p.n, d = p.d;

    float* amax = reinterpret_cast<float*>(sm + L::PAIR);                     // [parity][part][row]
    int* aidx = reinterpret_cast<int*>(amax + 2 * kParts * kRows);            // [parity][part][row]: first argmax
    uint32_t* chg = reinterpret_cast<uint32_t*>(aidx + 2 * kParts * kRows);   // [row], byte `part`: change flags
    uint32_t* hx = chg + kRows;                                               // [row], byte `part`: harvest test
    unsigned long long* slot_sh = reinterpret_cast<unsigned long long*>(hx + kRows);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + L::MBAR);
    uint32_t* tbase_sh = reinterpret_cast<uint32_t*>(mbar + 2);
    float* boxs = reinterpret_cast<float*>(sm + L::BOX);

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
        *reinterpret_cast<__nv_bfloat16*>(sm + L::BT16 + op_offset(k, i >> 3, DP) + (i & 7) * 2) = __float2bfloat16_rn(v);
    }
    for (int i = tid; i < NP; i += kThreads) boxs[i] = i < n ? (float)p.box[i] : 0.f;
    // ---- starts (Alg. 3 lines 4-5): g0 in fp64 from the counter RNG, z0 = B+ g0 (k ascending) ----
    double* g0s = reinterpret_cast<double*>(sm + L::G0);
    double zacc[DQ];
#pragma unroll
    for (int q = 0; q < DQ; ++q) zacc[q] = 0.0;
    for (int k0 = 0; k0 < n; k0 += L::KC) {
        for (int kk = part; kk < L::KC; kk += kParts) {
            const int k = k0 + kk;
            double g = 0.0;
            if (active && k < n) g = start_coord(counter_uniform(p.seed, gi, k, n), p.lo[k], p.hi[k]);
            g0s[row * (L::KC + 1) + kk] = g;
        }
        __syncthreads();
        // k outer, coordinates inner: DQ independent fp64 chains per k (the per-coordinate sum stays k-ascending)
        const int kend = min(L::KC, n - k0);
        const double* bq = p.Bp + (size_t)(part * DQ) * n + k0;
        for (int kk = 0; kk < kend; ++kk) {
            const double g = g0s[row * (L::KC + 1) + kk];
#pragma unroll
            for (int q = 0; q < DQ; ++q)
                if (part * DQ + q < d) zacc[q] = fma(bq[(size_t)q * n + kk], g, zacc[q]);
        }
        __syncthreads();
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tbase = *tbase_sh;
    const uint32_t tl = tbase + ((uint32_t)(quad * 32) << 16);
    {   // m = v = 0 in TMEM
        const uint32_t zr[4] = {0, 0, 0, 0};
#pragma unroll
        for (int c = 0; c < DQ / 4; ++c) {
            st4(tl + L::CM + part * DQ + 4 * c, zr);
            st4(tl + L::CV + part * DQ + 4 * c, zr);
        }
        st_wait();
    }
    __syncthreads();  // g0 staging may alias the operand area
    // The iterate lives in shared memory as the forward operand: Z_hi = tf32_rna(z) and the exact residual
    // Z_lo = z - Z_hi, so z = Z_hi + Z_lo exactly. Also round(z) as f16 (the harvest operand).
    {
        float lmax = -1.f;
        int lq = 0;
#pragma unroll
        for (int c = 0; c < DQ / 4; ++c) {
            const int col = part * DQ + 4 * c;
            float4 hi, lo;
            uint32_t rn[2] = {0u, 0u};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int q = 4 * c + e, j = col + e;
                const float zz = (j < d && active) ? (float)zacc[q] : 0.f;
                if (j < d && active && p.Z0_out) p.Z0_out[local * d + j] = zacc[q];
                (&hi.x)[e] = tf32_rna(zz);
                (&lo.x)[e] = zz - tf32_rna(zz);
                const float tq = truncf(zz), dq = zz - tq;
                const float rq = fabsf(dq) >= 0.5f ? tq + copysignf(1.f, dq) : tq;
                const uint32_t hb = __half_as_ushort(__float2half_rn(rq));
                rn[e >> 1] |= (e & 1) ? (hb << 16) : hb;
                if (fabsf(zz) > lmax) {
                    lmax = fabsf(zz);
                    lq = q;
                }
            }
            const uint32_t off = op_offset(row, col >> 2, kRows);
            *reinterpret_cast<float4*>(sm + L::ZHI + off) = hi;
            *reinterpret_cast<float4*>(sm + L::ZLO + off) = lo;
            *reinterpret_cast<uint2*>(sm + L::R16 + op_offset(row, col >> 3, kRows) + (col & 7) * 2) =
                make_uint2(rn[0], rn[1]);
        }
        amax[(0 * kParts + part) * kRows + row] = lmax;
        aidx[(0 * kParts + part) * kRows + row] = lq;
    }

    const uint32_t sZHI = smem_u32(sm + L::ZHI), sZLO = smem_u32(sm + L::ZLO), sR = smem_u32(sm + L::R16);
    const uint32_t sS = smem_u32(sm + L::S16), sB32 = smem_u32(sm + L::B32), sB16 = smem_u32(sm + L::B16);
    const uint32_t sBT = smem_u32(sm + L::BT16);
    constexpr uint32_t LBO_A = kRows * 16, LBO_N = NP * 16, LBO_D = DP * 16, SBO = 128;
    constexpr uint32_t ID_FWD = idesc(2, kRows, NP), ID_HARV = idesc(0, kRows, NP), ID_BWD = idesc(1, kRows, DP);
    const float lam1 = p.lam1, lam2 = p.lam2, b1 = p.beta1, b2 = p.beta2, omb1 = p.omb1, omb2 = p.omb2, eps = p.eps;
    const int T = p.T;
    const bool harvest = p.harvest != 0;
    const int64_t cap = p.cand_cap;
    const int c_lo = part * NQ;   // this thread's columns of G, H, S and the candidate row
    // 4 exact small-integer floats -> 4 int8 bytes (low byte of the 1.5 * 2^23 magic sum)
    auto pack4 = [](const uint32_t* r4) {
        uint32_t bq[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) bq[e] = __float_as_uint(__uint_as_float(r4[e]) + 12582912.f);
        return __byte_perm(__byte_perm(bq[0], bq[1], 0x0040), __byte_perm(bq[2], bq[3], 0x0040), 0x5410);
    };

    uint32_t phA = 0, phB = 0;
    const int t_end = harvest ? T + 1 : T;
    for (int t = 1; t <= t_end; ++t) {
        const bool do_fwd = t <= T;
        const bool do_harv = harvest && t >= 2;
        fence_proxy_async();
        fence_before();
        __syncthreads();  // B1: operands written, change flags and ranges visible
        if (tid == 0) {
            fence_after();
            if (do_fwd) {
#pragma unroll
                for (int kk = 0; kk < DP / 8; ++kk)
                    mma_tf32(tbase + L::CG, desc(sZHI + kk * 2 * LBO_A, LBO_A, SBO),
                             desc(sB32 + kk * 2 * LBO_N, LBO_N, SBO), ID_FWD, kk > 0);
#pragma unroll
                for (int kk = 0; kk < DP / 8; ++kk)
                    mma_tf32(tbase + L::CG, desc(sZLO + kk * 2 * LBO_A, LBO_A, SBO),
                             desc(sB32 + kk * 2 * LBO_N, LBO_N, SBO), ID_FWD, 1);
            }
            if (do_harv) {
#pragma unroll
                for (int kk = 0; kk < DP / 16; ++kk)
                    mma_f16(tbase + L::CX, desc(sR + kk * 2 * LBO_A, LBO_A, SBO),
                            desc(sB16 + kk * 2 * LBO_N, LBO_N, SBO), ID_HARV, kk > 0);
            }
            commit(&mbar[0]);
        }
        // one warp polls the mbarrier; the others wait in the CTA barrier without issuing
        if (warp == 0) mbar_wait(&mbar[0], phA);
        phA ^= 1;
        __syncthreads();
        fence_after();
        // change flags of z_{t-1}, all four parts: bit 0 round(z) changed, bit 1 max |z| > 2047.5 (see below)
        const uint32_t cw = chg[row];
        const uint32_t cf = (cw | (cw >> 8) | (cw >> 16) | (cw >> 24)) & 0xFFu;
        const bool row_chg = do_harv && active && cf == 1u;
        const bool warp_harv = __any_sync(0xffffffffu, row_chg);
        if (do_harv) {
            // ---- harvest test of g = H row (z_{t-1}), this part's columns. Code 0: outside the box; 1: in the
            // box, all zero here; 2 / 3: first nonzero here > 0 / < 0 ----
            int code = 1;
            if (warp_harv) {
                bool ok = true;
                int sgn = 0;
#pragma unroll
                for (int c0 = 0; c0 < NQ; c0 += 4) {
                    uint32_t r[4];
                    ld4(tl + L::CX + c_lo + c0, r);
                    wait4(r);
                    const float4 bx = *reinterpret_cast<const float4*>(boxs + c_lo + c0);   // broadcast
                    ok &= fabsf(__uint_as_float(r[0])) <= bx.x;
                    ok &= fabsf(__uint_as_float(r[1])) <= bx.y;
                    ok &= fabsf(__uint_as_float(r[2])) <= bx.z;
                    ok &= fabsf(__uint_as_float(r[3])) <= bx.w;
                    const uint32_t w = pack4(r);
                    if (sgn == 0 && w != 0u) sgn = ((int8_t)(w >> (8 * ((__ffs(w) - 1) >> 3)))) > 0 ? 1 : -1;
                }
                code = !ok ? 0 : (sgn == 0 ? 1 : (sgn > 0 ? 2 : 3));
            }
            reinterpret_cast<int8_t*>(hx)[row * 4 + part] = (int8_t)code;
        }
        if (do_fwd) {
            // ---- S = sign(B z), this part's columns of G -> bf16 backward operand (bf16 rounding keeps signs) ----
            const __nv_bfloat162 zero2 = __float2bfloat162_rn(0.f);
#pragma unroll
            for (int c0 = 0; c0 < NQ; c0 += 4) {
                uint32_t r[4];
                ld4(tl + L::CG + c_lo + c0, r);
                wait4(r);
                uint2 w;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1]));
                    const __nv_bfloat162 sg = __hsub2(__hgt2(h, zero2), __hlt2(h, zero2));
                    (&w.x)[e] = *reinterpret_cast<const uint32_t*>(&sg);
                }
                const int col = c_lo + c0;
                *reinterpret_cast<uint2*>(sm + L::S16 + op_offset(row, col >> 3, kRows) + (col & 7) * 2) = w;
            }
        }
        fence_proxy_async();
        fence_before();
        __syncthreads();  // B2: S and all parts' harvest tests written; G consumed (Γ reuses its columns)
        if (do_fwd && tid == 0) {
            fence_after();
#pragma unroll
            for (int kk = 0; kk < NP / 16; ++kk)
                mma_f16(tbase + L::CG, desc(sS + kk * 2 * LBO_A, LBO_A, SBO), desc(sBT + kk * 2 * LBO_D, LBO_D, SBO),
                        ID_BWD, kk > 0);
            commit(&mbar[1]);
        }
        if (do_harv && warp_harv) {
            // ---- candidate rows (overlaps the backward MMA): every part passed the box test, g != 0 ----
            const uint32_t hw = hx[row];
            bool ok = true;
            int code = 0;
#pragma unroll
            for (int pp = 0; pp < kParts; ++pp) {   // the first nonzero lies in the first part that has one
                const int c = (int)(int8_t)(hw >> (8 * pp));
                ok &= c != 0;
                if (code == 0 && c >= 2) code = c;
            }
            const bool want = row_chg && ok && code >= 2;
            const unsigned mask = __ballot_sync(0xffffffffu, want);   // identical in the quad's four warps
            if (mask) {
                if (part == 0) {   // one atomic per quad of warps; the slots reach the other parts via shared memory
                    const int leader = __ffs(mask) - 1;
                    unsigned long long base = 0;
                    if (lane == leader) base = atomicAdd(p.cand_count, (unsigned long long)__popc(mask));
                    base = __shfl_sync(0xffffffffu, base, leader);
                    slot_sh[row] = base + __popc(mask & ((1u << lane) - 1u));
                }
                bar_sync_quad(quad);   // warps quad, quad + 4, quad + 8, quad + 12
                const unsigned long long slot = slot_sh[row];
                const bool store = want && (int64_t)slot < cap;
                int8_t* dst = p.cand + (size_t)slot * p.n_pad + c_lo;   // 4-byte aligned (n_pad, NQ % 4 == 0)
#pragma unroll
                for (int c0 = 0; c0 < NQ; c0 += 4) {
                    uint32_t r[4];
                    ld4(tl + L::CX + c_lo + c0, r);   // tcgen05.ld is warp-collective: every lane loads
                    wait4(r);
                    uint32_t w = pack4(r);
                    if (code == 3) w = __vneg4(w);
                    if (store) *reinterpret_cast<uint32_t*>(dst + c0) = w;
                }
            }
        }
        if (!do_fwd) break;
        if (warp == 0) mbar_wait(&mbar[1], phB);
        phB ^= 1;
        __syncthreads();
        fence_after();
        // ---- gradient of Eq. 3 + Adam, this thread's DQ coordinates, 4 at a time ----
        const int par = (t - 1) & 1;
        float zinf = -1.f;
        int own = 0;
#pragma unroll
        for (int pp = 0; pp < kParts; ++pp) {   // ties -> the lowest part (lower coordinate indices)
            const float a = amax[(par * kParts + pp) * kRows + row];
            if (a > zinf) {
                zinf = a;
                own = pp;
            }
        }
        // λ2 term of Eq. 3 while ||z||_inf < 1, on the lowest-index argmax coordinate (found by its owner part)
        int kq = -1;
        float extra = 0.f;
        if (zinf < 1.f && part == own) {   // the owning part's recorded first argmax
            kq = aidx[(par * kParts + part) * kRows + row];
            const int j = part * DQ + kq;
            const uint32_t off = op_offset(row, j >> 2, kRows) + (j & 3) * 4;
            const float zq = *reinterpret_cast<const float*>(sm + L::ZHI + off) +
                             *reinterpret_cast<const float*>(sm + L::ZLO + off);
            if (zq != 0.f) extra = -lam2 * copysignf(1.f, zq) / fmaxf(zq * zq, 1e-8f);
        }
        const float4 st = p.step_tab[t - 1];     // (lr / (1 - b1^t), -, 1 / sqrt(1 - b2^t))
        bool ch = (t == 1);
        float lmax = 0.f;   // max |z_new| over this part and its first index (strict >: lowest index wins)
        int lq = 0;
        auto adam = [&](auto has_extra) {
#pragma unroll
            for (int c = 0; c < DQ / 4; ++c) {
                const int col = part * DQ + 4 * c;
                uint32_t rg[4], rm[4], rv[4];
                ld4(tl + L::CG + col, rg);
                ld4(tl + L::CM + col, rm);
                ld4(tl + L::CV + col, rv);
                const uint32_t roff = op_offset(row, col >> 3, kRows) + (col & 7) * 2;
                const uint2 rw = *reinterpret_cast<const uint2*>(sm + L::R16 + roff);
                const uint32_t off = op_offset(row, col >> 2, kRows);
                float4 hi = *reinterpret_cast<const float4*>(sm + L::ZHI + off);
                float4 lo = *reinterpret_cast<const float4*>(sm + L::ZLO + off);
                wait4(rg);
                wait4(rm);
                wait4(rv);
                float rn4[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int q = 4 * c + e;
                    float& hz = (&hi.x)[e];
                    float& lz = (&lo.x)[e];
                    const float zz = hz + lz;                                   // exact
                    const float2 r2 = __half22float2(*reinterpret_cast<const __half2*>(&(&rw.x)[e >> 1]));
                    const float ro = (e & 1) ? r2.y : r2.x;
                    const float dd = zz - ro;                                   // in [-1/2, 1/2], exact
                    const float sd = dd != 0.f ? copysignf(1.f, dd) : 0.f;
                    // λ1 d/dz (z - floor z)(ceil z - z) = ceil z + floor z - 2z = sign(z - r) - 2 (z - r)
                    float g = fmaf(lam1, fmaf(-2.f, dd, sd), __uint_as_float(rg[e]));
                    if constexpr (decltype(has_extra)::value) {
                        if (q == kq) g += extra;
                    }
                    const float mm = fmaf(b1, __uint_as_float(rm[e]), omb1 * g);
                    const float vv = fmaf(b2, __uint_as_float(rv[e]), omb2 * g * g);
                    rm[e] = __float_as_uint(mm);
                    rv[e] = __float_as_uint(vv);
                    const float den = fmaf(sqrt_approx(vv), st.z, eps);
                    const float zn = fmaf(-st.x * mm, rcp_approx(den), zz);
                    const float tn = truncf(zn);
                    const float dn = zn - tn;
                    // round half away from zero; + 0 turns -0 into +0 so equal values have equal f16 bits
                    rn4[e] = (fabsf(dn) >= 0.5f ? tn + copysignf(1.f, dn) : tn) + 0.f;
                    if (fabsf(zn) > lmax) {
                        lmax = fabsf(zn);
                        lq = q;
                    }
                    hz = tf32_rna(zn);
                    lz = zn - hz;
                }
                st4(tl + L::CM + col, rm);
                st4(tl + L::CV + col, rv);
                const __half2 h01 = __floats2half2_rn(rn4[0], rn4[1]);
                const __half2 h23 = __floats2half2_rn(rn4[2], rn4[3]);
                const uint2 rnew = make_uint2(*reinterpret_cast<const uint32_t*>(&h01),
                                              *reinterpret_cast<const uint32_t*>(&h23));
                ch |= (rnew.x != rw.x) | (rnew.y != rw.y);
                *reinterpret_cast<float4*>(sm + L::ZHI + off) = hi;
                *reinterpret_cast<float4*>(sm + L::ZLO + off) = lo;
                *reinterpret_cast<uint2*>(sm + L::R16 + roff) = rnew;
            }
        };
        if (__any_sync(0xffffffffu, extra != 0.f))
            adam(std::integral_constant<bool, true>());
        else
            adam(std::integral_constant<bool, false>());
        st_wait();
        amax[((t & 1) * kParts + part) * kRows + row] = lmax;
        aidx[((t & 1) * kParts + part) * kRows + row] = lq;
        // bit 0: round(z) changed; bit 1: max |z| > 2047.5, i.e. round(z) may leave the exact f16 range of the
        // harvest operand. The host selects this kernel only when every in-box g has |B+ g|_inf < 2047, so such
        // an iterate cannot map to a g inside the box and skipping it is exact.
        reinterpret_cast<uint8_t*>(chg)[row * 4 + part] = (uint8_t)((ch ? 1 : 0) | (lmax > 2047.5f ? 2 : 0));
    }
    if (p.Z_out && active) {
#pragma unroll
        for (int q = 0; q < DQ; ++q) {
            const int j = part * DQ + q;
            const uint32_t off = op_offset(row, j >> 2, kRows) + (j & 3) * 4;
            if (j < d)
                p.Z_out[local * d + j] = *reinterpret_cast<const float*>(sm + L::ZHI + off) +
                                         *reinterpret_cast<const float*>(sm + L::ZLO + off);
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
cudaError_t launch4(const DescentParams& p, cudaStream_t s) {
    using L = Lay4<NP, DP>;
    // at least 80 KB so that at most two CTAs (2 x 256 TMEM columns) share an SM
    const uint32_t smem = L::TOTAL < 80 * 1024 ? 80 * 1024 : L::TOTAL;
    cudaError_t e = cudaFuncSetAttribute(descent_tc4_kernel<NP, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const int64_t blocks = (p.count + kRows - 1) / kRows;
    descent_tc4_kernel<NP, DP><<<(unsigned)blocks, kThreads, smem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_descent_tc4(const DescentParams& p, cudaStream_t s) {
    if (p.count <= 0) return cudaSuccess;
    const int np = (std::max(p.n, 16) + 15) / 16 * 16;
    const int dp = (std::max(p.d, 16) + 15) / 16 * 16;
    if (np != p.n_pad) return cudaErrorInvalidValue;
#define MAPLE_TC4_CASE(NPV, DPV) \
    if (np == NPV && dp == DPV) return launch4<NPV, DPV>(p, s);
    MAPLE_TC4_CASE(16, 16)
    MAPLE_TC4_CASE(32, 16)
    MAPLE_TC4_CASE(32, 32)
    MAPLE_TC4_CASE(48, 16)
    MAPLE_TC4_CASE(48, 32)
    MAPLE_TC4_CASE(48, 48)
    MAPLE_TC4_CASE(64, 16)
    MAPLE_TC4_CASE(64, 32)
    MAPLE_TC4_CASE(64, 48)
    MAPLE_TC4_CASE(64, 64)
#undef MAPLE_TC4_CASE
    return cudaErrorNotSupported;
}

}  // namespace maple
