// Multi-start Graver-best augmentation (Alg. 2; MAPLE §4.3).
//
// One CTA per incumbent x (all incumbents of all instances run in parallel). Per iteration, for every
// direction g of D = S ∪ -S (lexicographically sorted) a thread computes
//     s = g^T (Q x + c),   q = g^T Q g (precomputed),   f(x + λg) - f(x) = λ s + λ² q / 2,
// so 2Δ(λ) = 2λs + λ²q is exact in fp64 for integer data (|values| < 2^53). λ runs over the integers
// 1..λmax(x, g) that keep l <= x + λg <= u (A g = 0 keeps A x = b). The CTA takes the argmin over
// (2Δ, index of g in D, λ) among strict improvements 2Δ < 0 — the paper's argmin with the tie-break of
// reading #17 — applies x += λg and ∇ += λ Q g, and stops when no improving step exists.
#include <cfloat>
#include <cstdio>

#include "common.cuh"
#include "kernels.h"

namespace maple {

namespace {

constexpr int kAugThreads = 256;
constexpr int kMaxN = 1024;

// q_e = g_e^T Q g_e for every direction of D (per instance)
__global__ void qg_kernel(AugmentParams p) {
    const int nD = 2 * p.n_dir;
    const int64_t total = (int64_t)nD * p.n_inst;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int inst = (int)(t / nD);
        const int e = (int)(t % nD);
        const int8_t* g = p.dirs + (size_t)e * p.n_pad;
        const double* Q = p.Q + (size_t)inst * p.n * p.n;
        double acc = 0.0;
        for (int i = 0; i < p.n; ++i) {
            const int gi = g[i];
            if (!gi) continue;
            double row = 0.0;
            for (int j = 0; j < p.n; ++j) {
                const int gj = g[j];
                if (gj) row += Q[(size_t)i * p.n + j] * (double)gj;
            }
            acc += (double)gi * row;
        }
        const_cast<double*>(p.qg)[(size_t)inst * nD + e] = acc;
    }
}

struct Cand {
    double key;  // 2Δ
    int e;       // index in D
    int lam;
};

__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
    if (a.key != b.key) return a.key < b.key;
    if (a.e != b.e) return a.e < b.e;
    return a.lam < b.lam;
}

__global__ void __launch_bounds__(kAugThreads)
augment_kernel(AugmentParams p) {
    __shared__ int32_t x[kMaxN];
    __shared__ double grad[kMaxN];
    __shared__ Cand wbest[kAugThreads / 32];
    __shared__ Cand best_sh;
    __shared__ double f2_sh;
    const int inc = blockIdx.x;  // incumbent index over all instances
    const int inst = inc / p.k0;
    const int n = p.n;
    const double* Q = p.Q + (size_t)inst * n * n;
    const double* c = p.c + (size_t)inst * n;
    const double* qg = p.qg + (size_t)inst * 2 * p.n_dir;
    int32_t* xg = p.X + (size_t)inc * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = xg[i];
    __syncthreads();
    // ∇ = Q x + c ; 2 f(x) = x^T Q x + 2 c^T x + 2 c0
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double acc = c[i];
        for (int j = 0; j < n; ++j) acc += Q[(size_t)i * n + j] * (double)x[j];
        grad[i] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double f2 = 2.0 * p.c0[inst];
        for (int i = 0; i < n; ++i) f2 += (double)x[i] * (grad[i] + c[i]);  // x^T(Qx + c) + c^T x
        f2_sh = f2;
    }
    __syncthreads();
    const int nD = 2 * p.n_dir;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int it = 0;
    for (; it < p.max_iter; ++it) {
        Cand mine{DBL_MAX, 0x7fffffff, 0x7fffffff};
        for (int e = threadIdx.x; e < nD; e += blockDim.x) {
            const int8_t* g = p.dirs + (size_t)e * p.n_pad;
            double s = 0.0;
            int lmax = 0x7fffffff;
            for (int i = 0; i < n; ++i) {
                const int gi = g[i];
                if (!gi) continue;
                s += (double)gi * grad[i];
                const int room = gi > 0 ? (p.hi[i] - x[i]) / gi : (x[i] - p.lo[i]) / (-gi);
                lmax = min(lmax, room);
            }
            if (lmax < 1 || lmax == 0x7fffffff) continue;
            const double q = qg[e];
            for (int lam = 1; lam <= lmax; ++lam) {
                const double dl = (double)lam;
                const double key = 2.0 * dl * s + dl * dl * q;
                if (key < 0.0) {
                    Cand cnd{key, e, lam};
                    if (better(cnd, mine)) mine = cnd;
                }
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            Cand o;
            o.key = __shfl_xor_sync(0xffffffffu, mine.key, off);
            o.e = __shfl_xor_sync(0xffffffffu, mine.e, off);
            o.lam = __shfl_xor_sync(0xffffffffu, mine.lam, off);
            if (better(o, mine)) mine = o;
        }
        if (lane == 0) wbest[wid] = mine;
        __syncthreads();
        if (threadIdx.x == 0) {
            Cand b = wbest[0];
            for (int w = 1; w < (int)(blockDim.x / 32); ++w)
                if (better(wbest[w], b)) b = wbest[w];
            best_sh = b;
        }
        __syncthreads();
        const Cand b = best_sh;
        if (b.e == 0x7fffffff) break;  // no improving step: x is Graver-optimal w.r.t. D
        const int8_t* g = p.dirs + (size_t)b.e * p.n_pad;
        // ∇ += λ Q g
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            double acc = 0.0;
            for (int j = 0; j < n; ++j) {
                const int gj = g[j];
                if (gj) acc += Q[(size_t)i * n + j] * (double)gj;
            }
            grad[i] += (double)b.lam * acc;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] += b.lam * (int)g[i];
        if (threadIdx.x == 0) f2_sh += b.key;
        __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) xg[i] = x[i];
    if (threadIdx.x == 0) {
        p.F2[inc] = f2_sh;
        p.iters[inc] = it;
    }
}

// per instance: the best final incumbent (min 2f, ties lexicographically smallest x; reading #19)
__global__ void best_kernel(AugmentParams p, int32_t* xbest, double* f2best) {
    for (int inst = blockIdx.x * blockDim.x + threadIdx.x; inst < p.n_inst; inst += gridDim.x * blockDim.x) {
        int b = 0;
        const int base = inst * p.k0;
        for (int k = 1; k < p.k0; ++k) {
            const double fk = p.F2[base + k], fb = p.F2[base + b];
            bool take = fk < fb;
            if (fk == fb) {
                const int32_t* xa = p.X + (size_t)(base + k) * p.n;
                const int32_t* xb = p.X + (size_t)(base + b) * p.n;
                for (int i = 0; i < p.n; ++i)
                    if (xa[i] != xb[i]) {
                        take = xa[i] < xb[i];
                        break;
                    }
            }
            if (take) b = k;
        }
        for (int i = 0; i < p.n; ++i) xbest[(size_t)inst * p.n + i] = p.X[(size_t)(base + b) * p.n + i];
        f2best[inst] = p.F2[base + b];
    }
}

}  // namespace

cudaError_t launch_augment_best(const AugmentParams& p, int32_t* xbest, double* f2best, cudaStream_t s) {
    if (p.n_inst <= 0 || p.k0 <= 0) return cudaSuccess;
    best_kernel<<<(p.n_inst + 127) / 128, 128, 0, s>>>(p, xbest, f2best);
    return cudaGetLastError();
}

cudaError_t launch_augment_qg(const AugmentParams& p, cudaStream_t s) {
    const int64_t total = (int64_t)2 * p.n_dir * p.n_inst;
    if (total <= 0) return cudaSuccess;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    qg_kernel<<<(unsigned)blocks, 256, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_augment(const AugmentParams& p, cudaStream_t s) {
    if (p.n > kMaxN) return cudaErrorInvalidValue;
    const int64_t blocks = (int64_t)p.n_inst * p.k0;
    if (blocks <= 0) return cudaSuccess;
    augment_kernel<<<(unsigned)blocks, kAugThreads, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace maple
