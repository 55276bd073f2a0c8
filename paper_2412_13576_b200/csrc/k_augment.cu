// Multi-start Graver-best augmentation (Alg. 2; MAPLE §4.3).
//
// One CTA per incumbent x (all incumbents of all instances run in parallel). Per iteration, for every
// direction g of D = S ∪ -S (lexicographically sorted) a thread computes
//     s = g^T (Q x + c),   q = g^T Q g (precomputed),   f(x + λg) - f(x) = λ s + λ² q / 2,
// so 2Δ(λ) = 2λs + λ²q is exact in fp64 for integer data (|values| < 2^53). λ runs over the integers
// 1..λmax(x, g) that keep l <= x + λg <= u (A g = 0 keeps A x = b). The CTA takes the argmin over
// (2Δ, index of g in D, λ) among strict improvements 2Δ < 0 — the paper's argmin with the tie-break of
// reading #17 — applies x += λg and ∇ += λ Q g, and stops when no improving step exists.
// Separable value tables (MAPLE_OBJ_TABLE; Prop. 3): f(x) = c0 + sum_j f_j(x_j) with f_j read from a
// table over [l_j, u_j], so f(x + λg) - f(x) = sum over the support of g (ascending j) of
// f_j(x_j + λ g_j) - f_j(x_j), and 2Δ of that sum is the key (no gradient state).
// Directions are kept in ELL form (nonzero columns + values, Graver elements are sparse), so the score,
// the step bound and the gradient update all cost O(nnz(g)) instead of O(n).
#include <algorithm>
#include <cfloat>
#include <cstdio>

#include "common.cuh"
#include "kernels.h"
#include "tc_pair.cuh"   // cluster rank / barrier / mapa (the split augmentation)

namespace maple {

namespace {

constexpr int kAugThreads = 1024;   // the most threads a CTA runs (large sets: memory-level parallelism)
constexpr int kMaxN = 1024;

// ELL of D, slot-major: word[a * nD + e] = column | (uint8)value << 16 | END << 24 for the a-th nonzero of row e
// (columns ascending; END marks the row's last nonzero), so a warp scanning 32 consecutive directions reads one
// coalesced 128-byte line per slot; nnz[e] = the row's nonzero count (<= width, the compact kernel's bound)
constexpr uint32_t kEnd = 1u << 24;
__device__ __forceinline__ int wcol(uint32_t w) { return (int)(w & 0xFFFFu); }
__device__ __forceinline__ int wval(uint32_t w) { return (int)(int8_t)(w >> 16); }

__global__ void ell_fill_kernel(const int8_t* __restrict__ dirs, int nD, int n, int n_pad, int width,
                                uint32_t* __restrict__ words, int32_t* __restrict__ nnz) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nD; e += gridDim.x * blockDim.x) {
        const int8_t* g = dirs + (size_t)e * n_pad;
        int c = 0, last = -1;
        for (int i = 0; i < n; ++i)
            if (g[i] && c < width) {
                if (last >= 0) words[(size_t)(c - 1) * nD + e] = (uint32_t)last | ((uint32_t)(uint8_t)g[last] << 16);
                last = i;
                ++c;
            }
        if (last >= 0) words[(size_t)(c - 1) * nD + e] = (uint32_t)last | ((uint32_t)(uint8_t)g[last] << 16) | kEnd;
        nnz[e] = c;
    }
}

// q_e = g_e^T Q g_e for every direction of D (per instance), over the nonzeros of g_e
constexpr int kQgRegs = 24;   // directions with at most this many nonzeros keep their words in registers
// D is sorted and closed under negation with D[nD-1-e] = -D[e] (signed_merge_kernel), and q(-g) = q(g) bit for bit
// (negation is exact and commutes with every product and sum below), so each thread computes e < nD/2 and writes
// both entries
__global__ void qg_kernel(AugmentParams p) {
    const int nD = 2 * p.n_dir, half = p.n_dir;
    const int64_t total = (int64_t)half * p.n_inst;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int inst = (int)(t / half);
        const int e = (int)(t % half);
        const double* Q = p.Q + (size_t)inst * p.n * p.n;
        const int k = p.nnz[e];
        double acc = 0.0;
        if (k <= kQgRegs) {   // the direction's words read once (slot-major, coalesced over e), then k^2 Q reads
            uint32_t w[kQgRegs];
#pragma unroll
            for (int a = 0; a < kQgRegs; ++a) w[a] = a < k ? p.words[(size_t)a * nD + e] : 0u;
#pragma unroll
            for (int a = 0; a < kQgRegs; ++a) {
                if (a >= k) break;
                const double* qa = Q + (size_t)wcol(w[a]) * p.n;
                double row = 0.0;
#pragma unroll
                for (int b = 0; b < kQgRegs; ++b) {
                    if (b >= k) break;
                    row += qa[wcol(w[b])] * (double)wval(w[b]);   // the same order as below: bit-identical
                }
                acc += (double)wval(w[a]) * row;
            }
        } else {
            for (int a = 0; a < k; ++a) {
                const uint32_t wa = p.words[(size_t)a * nD + e];
                double row = 0.0;
                for (int b = 0; b < k; ++b) {
                    const uint32_t wb = p.words[(size_t)b * nD + e];
                    row += Q[(size_t)wcol(wa) * p.n + wcol(wb)] * (double)wval(wb);
                }
                acc += (double)wval(wa) * row;
            }
        }
        const_cast<double*>(p.qg)[(size_t)inst * nD + e] = acc;
        const_cast<double*>(p.qg)[(size_t)inst * nD + (nD - 1 - e)] = acc;
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

// a cluster peer's Cand (shared::cluster load of the same variable in CTA `rank`)
__device__ __forceinline__ Cand ld_peer_cand(const Cand* local, uint32_t rank) {
    const uint32_t ra = pair::mapa((uint32_t)__cvta_generic_to_shared(local), rank);
    unsigned long long k;
    int e, l;
    asm volatile("ld.shared::cluster.b64 %0, [%1];" : "=l"(k) : "r"(ra) : "memory");
    asm volatile("ld.shared::cluster.b32 %0, [%1+8];" : "=r"(e) : "r"(ra) : "memory");
    asm volatile("ld.shared::cluster.b32 %0, [%1+12];" : "=r"(l) : "r"(ra) : "memory");
    return Cand{__longlong_as_double((long long)k), e, l};
}

__global__ void __launch_bounds__(kAugThreads, 1)
augment_kernel(AugmentParams p, int staged, int split) {
    __shared__ int32_t x[kMaxN];
    __shared__ int32_t up[kMaxN], dn[kMaxN];   // room to the bounds: u - x, x - l
    __shared__ double grad[kMaxN];
    __shared__ Cand wbest[kAugThreads / 32];
    __shared__ Cand best_sh;
    __shared__ double f2_sh;
    __shared__ Cand split_best[2];   // this CTA's best of iteration it, in slot it & 1 (read by the cluster peers)
    extern __shared__ __align__(16) unsigned char dsm[];   // staged D (ELL) + q_g when it fits
    // split > 1: the incumbent's directions are scanned by a cluster of `split` CTAs (few incumbents would leave
    // SMs idle); each CTA keeps the full state and applies the same best step, combined through DSMEM
    const int inc = blockIdx.x / split;  // incumbent index over all instances
    const int crank = split > 1 ? (int)pair::cluster_rank() : 0;
    const int inst = inc / p.k0;
    const int n = p.n;
    const double* Q = p.Q + (size_t)inst * n * n;
    const double* c = p.c + (size_t)inst * n;
    const double* qg = p.qg + (size_t)inst * 2 * p.n_dir;
    const double* tab = p.tab + (size_t)inst * p.tab_len;
    int32_t* xg = p.X + (size_t)inc * n;
    if (staged) {
        const int nD2 = 2 * p.n_dir, nz = p.nzmax;
        double* s_qg = reinterpret_cast<double*>(dsm);
        int32_t* s_nnz = reinterpret_cast<int32_t*>(s_qg + nD2);
        uint32_t* s_w = reinterpret_cast<uint32_t*>(s_nnz + nD2);
        for (int e = threadIdx.x; e < nD2; e += blockDim.x) {
            s_qg[e] = qg[e];
            s_nnz[e] = p.nnz[e];
        }
        for (int e = threadIdx.x; e < nD2 * nz; e += blockDim.x) s_w[e] = p.words[e];
        qg = s_qg;
        p.nnz = s_nnz;
        p.words = s_w;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        x[i] = xg[i];
        up[i] = p.hi[i] - x[i];
        dn[i] = x[i] - p.lo[i];
    }
    __syncthreads();
    // ∇ = Q x + c ; 2 f(x) = x^T Q x + 2 c^T x + 2 c0   (tables: 2 f(x) = 2 (c0 + sum_j f_j(x_j)))
    for (int i = threadIdx.x; i < n && !p.table; i += blockDim.x) {
        double acc = c[i];
        for (int j = 0; j < n; ++j) acc += Q[(size_t)i * n + j] * (double)x[j];
        grad[i] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0 && p.table) {
        double f = p.c0[inst];
        for (int i = 0; i < n; ++i) f += tab[p.tab_off[i] + dn[i]];
        f2_sh = 2.0 * f;
    } else if (threadIdx.x == 0) {
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
        for (int e = threadIdx.x + crank * blockDim.x; e < nD; e += split * blockDim.x) {
            // step bound first, leaving at the first blocked coordinate (in a box most directions are blocked at
            // an incumbent: a binary box blocks every g with a coordinate pushing past 0 or 1), then the score
            const uint32_t* we = p.words + e;
            int lmax = 0x7fffffff;
            for (int a = 0;; ++a) {
                const uint32_t w = we[(size_t)a * nD];
                const int i = wcol(w), gi = wval(w);
                const int room = gi == 1 ? up[i] : gi == -1 ? dn[i] : gi > 0 ? up[i] / gi : dn[i] / (-gi);
                lmax = min(lmax, room);
                if (lmax < 1 || (w & kEnd)) break;
            }
            if (lmax < 1) continue;
            if (p.table) {
                for (int lam = 1; lam <= lmax; ++lam) {
                    double dlt = 0.0;
                    for (int a = 0;; ++a) {
                        const uint32_t w = we[(size_t)a * nD];
                        const int i = wcol(w);
                        const double* ti = tab + p.tab_off[i] + dn[i];
                        dlt += ti[lam * wval(w)] - ti[0];
                        if (w & kEnd) break;
                    }
                    const double key = 2.0 * dlt;
                    if (key < 0.0) {
                        Cand cnd{key, e, lam};
                        if (better(cnd, mine)) mine = cnd;
                    }
                }
                continue;
            }
            double s = 0.0;
            for (int a = 0;; ++a) {
                const uint32_t w = we[(size_t)a * nD];
                s += (double)wval(w) * grad[wcol(w)];
                if (w & kEnd) break;
            }
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
            if (split > 1) split_best[it & 1] = b;
        }
        if (split > 1) {   // combine the cluster's bests (better() is a strict total order: every CTA gets the same)
            pair::cluster_sync();
            if (threadIdx.x == 0) {
                Cand b = best_sh;
                for (int r = 0; r < split; ++r)
                    if (r != crank) {
                        const Cand o = ld_peer_cand(&split_best[it & 1], (uint32_t)r);
                        if (better(o, b)) b = o;
                    }
                best_sh = b;
            }
        }
        __syncthreads();
        const Cand b = best_sh;
        if (b.e == 0x7fffffff) break;  // no improving step: x is Graver-optimal w.r.t. D
        const int k = p.nnz[b.e];
        const uint32_t* wb = p.words + b.e;
        // ∇ += λ Q g (Q symmetric: column i of Q = row i, read coalesced)
        for (int i = threadIdx.x; i < n && !p.table; i += blockDim.x) {
            double acc = 0.0;
            for (int a = 0; a < k; ++a) {
                const uint32_t w = wb[(size_t)a * nD];
                acc += Q[(size_t)wcol(w) * n + i] * (double)wval(w);
            }
            grad[i] += (double)b.lam * acc;
        }
        __syncthreads();
        for (int a = threadIdx.x; a < k; a += blockDim.x) {
            const uint32_t w = wb[(size_t)a * nD];
            const int i = wcol(w), dx = b.lam * wval(w);
            x[i] += dx;
            up[i] -= dx;
            dn[i] += dx;
        }
        if (threadIdx.x == 0) f2_sh += b.key;
        __syncthreads();
    }
    if (split > 1) pair::cluster_sync();   // the peers' last reads of split_best are done before any CTA exits
    if (crank != 0) return;
    for (int i = threadIdx.x; i < n; i += blockDim.x) xg[i] = x[i];
    if (threadIdx.x == 0) {
        p.F2[inc] = f2_sh;
        p.iters[inc] = it;
    }
}

__device__ __forceinline__ bool inc_better(const double* F2, const int32_t* X, int n, int a, int b) {
    if (b < 0) return a >= 0;
    if (a < 0) return false;
    const double fa = F2[a], fb = F2[b];
    if (fa != fb) return fa < fb;
    const int32_t* xa = X + (size_t)a * n;
    const int32_t* xb = X + (size_t)b * n;
    for (int i = 0; i < n; ++i)
        if (xa[i] != xb[i]) return xa[i] < xb[i];
    return a < b;
}

// per instance (one block): the best final incumbent (min 2f, ties lexicographically smallest x; reading #19).
// The instance's incumbents are staged in shared memory when they fit (dynamic smem = k0 * (n*4 + 8) bytes).
__global__ void best_kernel(AugmentParams p, int32_t* xbest, double* f2best, int staged) {
    extern __shared__ __align__(16) unsigned char bsm[];
    __shared__ int cand[128];
    const int inst = blockIdx.x;
    const int base = inst * p.k0;
    const double* F2 = p.F2 + base;
    const int32_t* X = p.X + (size_t)base * p.n;
    if (staged) {
        double* sF = reinterpret_cast<double*>(bsm);
        int32_t* sX = reinterpret_cast<int32_t*>(sF + p.k0);
        for (int k = threadIdx.x; k < p.k0; k += blockDim.x) sF[k] = F2[k];
        for (int e = threadIdx.x; e < p.k0 * p.n; e += blockDim.x) sX[e] = X[e];
        __syncthreads();
        F2 = sF;
        X = sX;
    }
    int b = -1;
    for (int k = threadIdx.x; k < p.k0; k += blockDim.x)
        if (inc_better(F2, X, p.n, k, b)) b = k;
    cand[threadIdx.x] = b;
    __syncthreads();
    for (int w = 64; w > 0; w >>= 1) {
        if (threadIdx.x < w && inc_better(F2, X, p.n, cand[threadIdx.x + w], cand[threadIdx.x]))
            cand[threadIdx.x] = cand[threadIdx.x + w];
        __syncthreads();
    }
    const int bb = cand[0];
    for (int i = threadIdx.x; i < p.n; i += blockDim.x) xbest[(size_t)inst * p.n + i] = X[(size_t)bb * p.n + i];
    if (threadIdx.x == 0) f2best[inst] = F2[bb];
}

}  // namespace

cudaError_t launch_augment_ell(const int8_t* dirs, int nD, int n, int n_pad, int width, int32_t* nnz, uint32_t* words,
                               cudaStream_t s) {
    if (nD <= 0) return cudaSuccess;
    const unsigned blocks = (unsigned)std::min(148 * 8, (nD + 255) / 256);
    ell_fill_kernel<<<blocks, 256, 0, s>>>(dirs, nD, n, n_pad, width, words, nnz);
    return cudaGetLastError();
}

cudaError_t launch_augment_best(const AugmentParams& p, int32_t* xbest, double* f2best, cudaStream_t s) {
    if (p.n_inst <= 0 || p.k0 <= 0) return cudaSuccess;
    const size_t smem = (size_t)p.k0 * ((size_t)p.n * 4 + 8);
    const int staged = smem <= 160 * 1024;
    if (staged) {
        cudaError_t e = cudaFuncSetAttribute(best_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    best_kernel<<<p.n_inst, 128, staged ? smem : 0, s>>>(p, xbest, f2best, staged);
    return cudaGetLastError();
}

cudaError_t launch_augment_qg(const AugmentParams& p, cudaStream_t s) {
    if (p.table) return cudaSuccess;   // tables: no quadratic form
    const int64_t total = (int64_t)p.n_dir * p.n_inst;   // one thread per (instance, direction pair g, -g)
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
    const size_t nD2 = (size_t)2 * p.n_dir;
    const size_t smem = nD2 * 8 + nD2 * 4 + nD2 * p.nzmax * 4 + 16;
    const int staged = smem <= 96 * 1024;
    if (staged) {   // dynamic + ~12 KB static may pass the 48 KB default even when the dynamic part does not
        cudaError_t e = cudaFuncSetAttribute(augment_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int threads = nD2 > 16384 ? kAugThreads : 256;
    // few incumbents with a large D (C3: ~100 incumbents, |D| = 1.6 M): a cluster of `split` CTAs of 256 threads per
    // incumbent (four fit an SM), as many as one wave holds, so that every SM scans and each thread scans fewer
    // directions; otherwise one CTA per incumbent
    int split = 1;
    if (threads == kAugThreads && blocks < 148) split = (int)std::min<int64_t>(8, (4 * 148) / blocks);
    if (split <= 1) {
        augment_kernel<<<(unsigned)blocks, threads, staged ? smem : 0, s>>>(p, staged, 1);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(blocks * split));
    cfg.blockDim = dim3(kAugThreads / 4);
    cfg.dynamicSmemBytes = staged ? smem : 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)split;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, augment_kernel, p, staged, split);
}

}  // namespace maple
