// North-star post-processing kernels: dedupe (+ sign twins), exact check, ⊑-minimal filter, compaction
// and lexicographic sort. Rows are canonical int8 vectors (first nonzero > 0) with stride n_pad.
// Every kernel takes its row count from device memory (the producer's counter), so the whole pipeline is
// enqueued without host round trips; grids are sized from host upper bounds and loop grid-stride.
//
//  dedupe   open-addressing hash set over the whole row (64-bit key, full-row compare on a key hit):
//           set semantics of Alg. 3's "𝒢 ∪ {·}"; sign twins were collapsed by canonicalisation.
//           A plain load precedes the CAS so hot duplicate rows do not serialise on one atomic address.
//  check    (C1)-(C3) of §4: A g = 0 in exact int64 (A as CSR in shared memory), g != 0,
//           l - u <= g <= u - l; fused with the filter's encoding (thermometer code + L1 norm).
//  filter   (C4) / Def. 1-2: g is dropped iff some other row h has h ⊑ g or h ⊑ -g.
//           Rows are encoded as thermometer bitsets P = [g_i >= k], N = [g_i <= -k] (k = 1..u_i-l_i), so
//           h ⊑ g  <=>  P_h ⊆ P_g and N_h ⊆ N_g,   h ⊑ -g  <=>  P_h ⊆ N_g and N_h ⊆ P_g.
//           Only rows with strictly smaller L1 norm can dominate, so rows are bucketed by L1 (counting
//           sort) and each g scans the lower buckets tile by tile with block-wide early exit.
//  sort     bottom-up merge sort of row indices on big-endian biased keys (lexicographic int8 order).
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "kernels.h"

namespace maple {

namespace {

__device__ __forceinline__ int64_t dev_count(const unsigned long long* c, int64_t cap) {
    const int64_t k = (int64_t)*c;
    return k < cap ? k : cap;
}

__device__ __forceinline__ uint64_t row_hash(const int4* w, int nw) {
    uint64_t h = 0x243F6A8885A308D3ULL;
    for (int i = 0; i < nw; ++i) {
        const int4 v = w[i];
        const uint64_t a = ((uint64_t)(uint32_t)v.y << 32) | (uint32_t)v.x;
        const uint64_t b = ((uint64_t)(uint32_t)v.w << 32) | (uint32_t)v.z;
        h = mix64(h ^ a);
        h = mix64(h ^ b);
    }
    return h;
}

__device__ __forceinline__ bool rows_equal(const int4* a, const int4* b, int nw) {
    for (int i = 0; i < nw; ++i) {
        const int4 x = a[i], y = b[i];
        if (x.x != y.x || x.y != y.y || x.z != y.z || x.w != y.w) return false;
    }
    return true;
}

// Slot word: (32-bit hash, never 0) << 32 | ref. ref with bit 31 set = pool index of a finished row; bit 31
// clear = index of the inserting row in THIS launch's input (rows written by earlier kernels, so a thread that
// hits the key compares against them without waiting for any write of this launch: no fence, no publication
// spin). The winner of a slot takes a pool index (warp-aggregated) and records the slot; finish_dedupe_kernel
// then copies the new rows into the pool and rewrites their slots to pool references.
__global__ void dedupe_kernel(const int8_t* __restrict__ rows, const unsigned long long* dcount, int64_t cap,
                              int row_stride, int n_pad, HashSet hs) {
    const int nw = n_pad / 16;
    const int64_t count = dev_count(dcount, cap);
    if (blockIdx.x == 0 && threadIdx.x == 0 && hs.max_count) atomicMax(hs.max_count, *dcount);
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < count;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int4* src = reinterpret_cast<const int4*>(rows + (size_t)r * row_stride);
        const uint64_t h = row_hash(src, nw);
        const unsigned long long tag = ((h >> 32) | 1ULL) << 32;
        uint64_t pos = mix64(h ^ 0x9E3779B97F4A7C15ULL) & hs.mask;
        for (uint64_t probe = 0; probe <= hs.mask; ++probe) {
            unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(&hs.keys[pos]);
            if (cur == 0ULL) {
                cur = atomicCAS(&hs.keys[pos], 0ULL, tag | (unsigned long long)r);
                if (cur == 0ULL) {  // we own the slot: a new unique row
                    // opportunistic warp aggregation of the pool-index allocation
                    const unsigned am = __activemask();
                    const int lane = threadIdx.x & 31;
                    const int leader = __ffs(am) - 1;
                    unsigned long long base = 0;
                    if (lane == leader) base = atomicAdd(hs.pool_count, (unsigned long long)__popc(am));
                    base = __shfl_sync(am, base, leader);
                    const unsigned long long idx = base + __popc(am & ((1u << lane) - 1u));
                    if ((int64_t)idx >= hs.pool_cap)
                        atomicExch(hs.overflow, 1);   // the caller grows the pool and redoes the extraction
                    else
                        hs.newslot[idx] = (int64_t)pos;
                    break;
                }
            }
            if ((cur & 0xFFFFFFFF00000000ULL) == tag) {  // same hash: compare the full rows
                const uint32_t ref = (uint32_t)cur;
                const int4* other = (ref & 0x80000000u)
                                        ? reinterpret_cast<const int4*>(hs.pool + (size_t)(ref & 0x7FFFFFFFu) * n_pad)
                                        : reinterpret_cast<const int4*>(rows + (size_t)ref * row_stride);
                if (rows_equal(src, other, nw)) break;  // duplicate
            }
            pos = (pos + 1) & hs.mask;
        }
    }
}

// copy the rows inserted by the last dedupe launch into the pool and turn their slots into pool references
__global__ void finish_dedupe_kernel(const int8_t* __restrict__ rows, int row_stride, int n_pad, HashSet hs) {
    const int nw = n_pad / 16;
    const int64_t count = min((int64_t)*hs.pool_count, hs.pool_cap);
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < count; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t pos = hs.newslot[p];
        if (pos < 0) continue;
        const unsigned long long cur = hs.keys[pos];
        const uint32_t ref = (uint32_t)cur;
        const int4* src = reinterpret_cast<const int4*>(rows + (size_t)ref * row_stride);
        int4* dst = reinterpret_cast<int4*>(hs.pool + (size_t)p * n_pad);
        for (int i = 0; i < nw; ++i) dst[i] = src[i];
        hs.keys[pos] = (cur & 0xFFFFFFFF00000000ULL) | 0x80000000ULL | (unsigned long long)p;
        hs.newslot[p] = -1;
    }
}

// (C1)-(C3) + filter encoding, one thread per row. The block stages its rows in shared memory (coalesced
// 16-byte loads, padded stride n_pad + 4); A (CSR), u - l and the thermometer offsets sit in shared memory.
constexpr int kCheckThreads = 128;
__global__ void __launch_bounds__(kCheckThreads) check_codes_kernel(const int8_t* __restrict__ rows,
                                                                   const unsigned long long* dcount, int64_t cap,
                                                                   CheckParams cp, FilterWork fw, uint8_t* flags,
                                                                   unsigned long long* n_bad, int encode) {
    extern __shared__ __align__(16) int32_t sh[];
    int32_t* srp = sh;
    int32_t* scol = srp + cp.m + 1;
    int32_t* sval = scol + cp.nnz;
    int32_t* sbox = sval + cp.nnz;
    int32_t* soff = sbox + cp.n;
    int32_t* swc0 = soff + cp.n;
    int32_t* swc1 = swc0 + fw.Wh;
    // row stride n_pad + 4 bytes: an odd number of 4-byte words, so the 32 threads' reads of the same byte
    // column of their rows fall in 32 different banks (n_pad + 16 put them in two)
    const int stride = cp.n_pad + 4;
    int8_t* srow = reinterpret_cast<int8_t*>(sh + (((cp.m + 1 + 2 * cp.nnz + 2 * cp.n + 2 * fw.Wh) + 3) & ~3));
    for (int i = threadIdx.x; i <= cp.m; i += blockDim.x) srp[i] = cp.A_rowptr[i];
    for (int i = threadIdx.x; i < cp.nnz; i += blockDim.x) {
        scol[i] = cp.A_col[i];
        sval[i] = cp.A_val[i];
    }
    for (int i = threadIdx.x; i < cp.n; i += blockDim.x) {
        sbox[i] = cp.box[i];
        soff[i] = fw.off[i];
    }
    for (int w = threadIdx.x; w < fw.Wh; w += blockDim.x) {
        swc0[w] = fw.word_c0[w];
        swc1[w] = fw.word_c1[w];
    }
    const int nw = cp.n_pad / 16;
    const int64_t count = dev_count(dcount, cap);
    const int W2 = 2 * fw.Wh;
    unsigned long long bad = 0;
    for (int64_t r0 = (int64_t)blockIdx.x * kCheckThreads; r0 < count; r0 += (int64_t)gridDim.x * kCheckThreads) {
        __syncthreads();
        const int64_t nr = min((int64_t)kCheckThreads, count - r0);
        const int4* src = reinterpret_cast<const int4*>(rows + (size_t)r0 * cp.n_pad);
        for (int e = threadIdx.x; e < nr * nw; e += kCheckThreads)
        {
            const int4 v = src[e];
            uint32_t* dst = reinterpret_cast<uint32_t*>(srow + (e / nw) * stride + (e % nw) * 16);
            dst[0] = (uint32_t)v.x;
            dst[1] = (uint32_t)v.y;
            dst[2] = (uint32_t)v.z;
            dst[3] = (uint32_t)v.w;
        }
        __syncthreads();
        if (threadIdx.x >= nr) continue;
        const int8_t* g = srow + threadIdx.x * stride;
        bool ok = true, nz = false;
        int l1 = 0;
        if (fw.binary) {  // every u_i - l_i == 1: |g_i| <= 1, bytewise on 16-byte words
            const uint32_t* gw = reinterpret_cast<const uint32_t*>(g);
            for (int w = 0; w < cp.n_pad / 4; ++w) {
                const uint32_t a = __vabsss4(gw[w]);
                ok &= (a & 0xFEFEFEFEu) == 0u;
                nz |= a != 0u;
                l1 += (int)__vsadu4(a, 0u);
            }
        } else {
            for (int i = 0; i < cp.n; ++i) {
                const int v = g[i];
                nz |= (v != 0);
                ok &= (abs(v) <= sbox[i]);
                l1 += abs(v);
            }
        }
        for (int a = 0; a < cp.m && ok; ++a) {
            long long acc = 0;
            for (int e = srp[a]; e < srp[a + 1]; ++e) acc += (long long)sval[e] * (long long)g[scol[e]];
            ok &= (acc == 0);
        }
        ok &= nz;
        const int64_t r = r0 + threadIdx.x;
        flags[r] = ok ? 1 : 0;
        bad += ok ? 0 : 1;
        if (encode) {
            fw.l1[r] = ok ? l1 : -1;
            // thermometer code: coordinate i owns bits [off_i, off_i + u_i - l_i) of each half
            uint32_t* code = fw.codes + (size_t)r * W2;
            uint32_t f0 = 0u, f1 = 0u, f2 = 0u, f3 = 0u;   // 64-bit folds of P and N (bit i mod 64), the filter's prefilter
            if (fw.binary && ok) {  // bit i of P = [g_i > 0], of N = [g_i < 0] (off_i = i)
                const uint32_t* gw = reinterpret_cast<const uint32_t*>(g);
                for (int w = 0; w < fw.Wh; ++w) {
                    uint32_t pw = 0, nw_ = 0;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int wi = 8 * w + q;
                        const uint32_t x = wi < cp.n_pad / 4 ? gw[wi] : 0u;
                        const uint32_t pos = __vcmpgts4(x, 0u) & 0x01010101u;    // byte > 0
                        const uint32_t neg = (x >> 7) & 0x01010101u;              // byte < 0
                        // gather bit 8k of each byte into bit k: (x * 0x01020408) >> 24 (no carries)
                        pw |= (((pos * 0x01020408u) >> 24) & 0xFu) << (4 * q);
                        nw_ |= (((neg * 0x01020408u) >> 24) & 0xFu) << (4 * q);
                    }
                    code[w] = pw;
                    code[fw.Wh + w] = nw_;
                    if (w & 1) {
                        f1 |= pw;
                        f3 |= nw_;
                    } else {
                        f0 |= pw;
                        f2 |= nw_;
                    }
                }
            } else
            for (int hf = 0; hf < 2; ++hf) {
                for (int w = 0; w < fw.Wh; ++w) {
                    uint32_t word = 0;
                    for (int i = swc0[w]; i <= swc1[w]; ++i) {
                        const int v = hf ? -(int)g[i] : (int)g[i];   // bits [off_i, off_i + v) of this half
                        if (v <= 0) continue;
                        const int b0 = soff[i] - 32 * w, b1 = b0 + v;
                        const int a = max(b0, 0), e = min(b1, 32);
                        if (a < e) word |= (e - a == 32) ? 0xFFFFFFFFu : (((1u << (e - a)) - 1u) << a);
                    }
                    code[hf * fw.Wh + w] = word;
                    if (hf) {
                        if (w & 1) f3 |= word; else f2 |= word;
                    } else {
                        if (w & 1) f1 |= word; else f0 |= word;
                    }
                }
            }
            fw.sig[r] = make_uint4(f0, f1, f2, f3);
        }
    }
    if (bad) atomicAdd(n_bad, bad);
}

// L1 histogram with block-local (shared-memory) aggregation: one global atomic per bin per block
__global__ void hist_kernel(const int32_t* l1, const unsigned long long* dcount, int64_t cap, int32_t* hist, int nb) {
    extern __shared__ int32_t sh_hist[];
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sh_hist[i] = 0;
    __syncthreads();
    const int64_t count = dev_count(dcount, cap);
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < count; r += (int64_t)gridDim.x * blockDim.x)
        if (l1[r] >= 0) atomicAdd(&sh_hist[l1[r]], 1);
    __syncthreads();
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
        if (sh_hist[i]) atomicAdd(&hist[i], sh_hist[i]);
}

// exclusive scan of hist[0..nb) -> start[0..nb], single thread (nb <= 1025)
__global__ void scan_kernel(const int32_t* hist, int nb, int32_t* start, int32_t* cursor) {
    if (threadIdx.x == 0) {
        int32_t acc = 0;
        for (int i = 0; i < nb; ++i) {
            start[i] = acc;
            cursor[i] = acc;
            acc += hist[i];
        }
        start[nb] = acc;
    }
}

// bucket scatter: each block counts its rows per bin, reserves one contiguous range per bin with a single
// global atomic, then places its rows (the order inside a bucket is irrelevant to the filter's result)
__global__ void scatter_kernel(const int32_t* l1, const unsigned long long* dcount, int64_t cap, int32_t* cursor,
                               int32_t* order, int nb) {
    extern __shared__ int32_t sh[];
    int32_t* cnt = sh;
    int32_t* base = sh + nb;
    const int64_t count = dev_count(dcount, cap);
    const int64_t chunk = (int64_t)blockDim.x * 8;
    for (int64_t c0 = (int64_t)blockIdx.x * chunk; c0 < count; c0 += (int64_t)gridDim.x * chunk) {
        for (int i = threadIdx.x; i < nb; i += blockDim.x) cnt[i] = 0;
        __syncthreads();
        int lv[8], slot[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int64_t r = c0 + k * blockDim.x + threadIdx.x;
            lv[k] = r < count ? l1[r] : -1;
            slot[k] = lv[k] >= 0 ? atomicAdd(&cnt[lv[k]], 1) : 0;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < nb; i += blockDim.x) base[i] = cnt[i] ? atomicAdd(&cursor[i], cnt[i]) : 0;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int64_t r = c0 + k * blockDim.x + threadIdx.x;
            if (lv[k] >= 0) order[base[lv[k]] + slot[k]] = (int32_t)r;
        }
        __syncthreads();
    }
}

constexpr int kFilterThreads = 256;
constexpr int kTile = 512;

// Dominance test. Rows are visited in L1 order (order[], level_start[]); a block takes 256 consecutive
// positions and streams the candidate dominators (all rows of strictly smaller L1) through shared memory
// tile by tile as (64-bit folds of P and N, row) — the fold test is a necessary condition for h ⊑ g and for h ⊑ -g;
// the exact test on the full codes runs only for pairs that pass it. Each thread stops at its first
// dominator; the block stops when all its rows are decided.
template <int WH>
__global__ void __launch_bounds__(kFilterThreads)
dominance_kernel(FilterWork fw) {
    __shared__ uint4 tile_sig[kTile];
    __shared__ int32_t tile_row[kTile];
    __shared__ int32_t smax;
    const int Wh = fw.Wh;
    const int W2 = 2 * Wh;
    const int32_t n_valid = fw.level_start[fw.Lmax + 1];
    const int32_t nblk = (n_valid + kFilterThreads - 1) / kFilterThreads;
    for (int32_t pb = blockIdx.x; pb < nblk; pb += gridDim.x) {
        const int32_t pos = pb * kFilterThreads + threadIdx.x;
        int32_t row = pos < n_valid ? fw.order[pos] : -1, limit = 0;
        // rows outside [g_begin, g_end) (a shard of the global pass; g_end = 0: all rows) are only dominators here
        const bool active0 = row >= 0 && (fw.g_end == 0 || (row >= fw.g_begin && row < fw.g_end));
        uint32_t P[WH], N[WH];
        uint32_t fp0 = 0, fp1 = 0, fn0 = 0, fn1 = 0;
        if (active0) {
            limit = fw.level_start[fw.l1[row]];  // rows with strictly smaller L1
#pragma unroll
            for (int w = 0; w < WH; ++w) {
                P[w] = w < Wh ? fw.codes[(size_t)row * W2 + w] : 0u;
                N[w] = w < Wh ? fw.codes[(size_t)row * W2 + Wh + w] : 0u;
                if (w & 1) {
                    fp1 |= P[w];
                    fn1 |= N[w];
                } else {
                    fp0 |= P[w];
                    fn0 |= N[w];
                }
            }
        }
        bool done = !active0 || limit == 0;
        int32_t wit = -1;
        __syncthreads();
        if (threadIdx.x == 0) smax = 0;
        __syncthreads();
        const int32_t scan = min(limit, fw.scan_cap);   // the rows this thread scans here (a prefix of its dominators)
        if (active0) atomicMax(&smax, scan);
        __syncthreads();
        const int32_t maxlim = smax;
        for (int32_t t0 = 0; t0 < maxlim; t0 += kTile) {
            if (!__syncthreads_or(!done)) break;
            for (int i = threadIdx.x; i < kTile; i += kFilterThreads) {
                const int32_t q = t0 + i;
                const int32_t hr = q < maxlim ? fw.order[q] : -1;
                tile_row[i] = hr;
                tile_sig[i] = hr >= 0 ? fw.sig[hr] : make_uint4(~0u, ~0u, ~0u, ~0u);
            }
            __syncthreads();
            if (!done) {
                const int lim = min(kTile, scan - t0);
                for (int i = 0; i < lim; ++i) {
                    const uint4 hs = tile_sig[i];
                    const uint32_t pv = (hs.x & ~fp0) | (hs.y & ~fp1) | (hs.z & ~fn0) | (hs.w & ~fn1);
                    const uint32_t nv = (hs.x & ~fn0) | (hs.y & ~fn1) | (hs.z & ~fp0) | (hs.w & ~fp1);
                    if (pv != 0u && nv != 0u) continue;
                    const int32_t hr = tile_row[i];
                    const uint32_t* hc = fw.codes + (size_t)hr * W2;
                    uint32_t pos_v = 0, neg_v = 0;
#pragma unroll
                    for (int w = 0; w < WH; ++w) {
                        if (w < Wh) {
                            const uint32_t hp = hc[w], hn = hc[Wh + w];
                            pos_v |= (hp & ~P[w]) | (hn & ~N[w]);
                            neg_v |= (hp & ~N[w]) | (hn & ~P[w]);
                        }
                    }
                    if (pos_v == 0u || neg_v == 0u) {
                        done = true;
                        wit = hr;
                        break;
                    }
                }
                if (t0 + kTile >= scan) done = true;
            }
            __syncthreads();
        }
        const bool undec = active0 && wit < 0 && scan < limit;
        if (active0) {   // 2: not dominated by the scanned prefix, which is not all of its candidates (undecided)
            fw.keep[row] = (wit >= 0) ? 0 : (undec ? 2 : 1);
            fw.witness[row] = wit;
        }
        const int nu = __syncthreads_count(undec);
        if (threadIdx.x == 0 && nu) atomicAdd(fw.n_undec, nu);
    }
}

// level-synchronous pass (algo 3, below): (the G lists' total is gl_start[(Lmax + 1) n] once scanned; beyond gl_cap the indexed pass runs instead)
__device__ __forceinline__ bool gl_overflow(const FilterWork& fw) {
    return (int64_t)fw.gl_start[(size_t)(fw.Lmax + 1) * fw.n] > fw.gl_cap;
}

// ---- indexed filter (large pools) ----
// h ⊑ ±g requires supp(h) ⊆ supp(g). Every valid row h is filed under one key coordinate κ(h) ∈ supp(h) — its
// rarest coordinate over the pool (ties: lowest index) — and, inside that list, by its L1 norm: bin
// κ(h)·(Lmax+1) + L1(h). A row g then only meets the rows filed under its own support coordinates with a
// strictly smaller L1: for c ∈ supp(g) the contiguous range [bin(c, 0), bin(c, L1(g))). Each such pair is
// tested by the 64-bit folds first and then exactly on the codes, as in the tiled kernel; the keep bit is the
// same (it is defined pairwise), only the recorded witness may differ.
constexpr int kIdxMaxN = 1024;

// thread per row (16-byte loads of its bytes); every kernel of the index returns at once when the tiled prefix
// scan left no row undecided
__global__ void coord_freq_kernel(FilterWork fw, const unsigned long long* dcount, int64_t cap) {
    if (*fw.n_undec == 0) return;
    __shared__ int32_t sf[kIdxMaxN];
    for (int i = threadIdx.x; i < fw.n; i += blockDim.x) sf[i] = 0;
    __syncthreads();
    const int64_t count = dev_count(dcount, cap);
    const int nw = fw.n_pad / 16;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < count; r += (int64_t)gridDim.x * blockDim.x) {
        if (fw.l1[r] < 0) continue;
        const int4* g = reinterpret_cast<const int4*>(fw.rows + (size_t)r * fw.n_pad);
        for (int w = 0; w < nw; ++w) {
            const int4 v = g[w];
            const uint32_t q[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
#pragma unroll
            for (int b = 0; b < 16; ++b)
                if ((q[b >> 2] >> (8 * (b & 3))) & 0xFFu) atomicAdd(&sf[16 * w + b], 1);   // padding bytes are 0
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < fw.n; i += blockDim.x)
        if (sf[i]) atomicAdd(&fw.freq[i], sf[i]);
}

__global__ void key_bin_kernel(FilterWork fw, const unsigned long long* dcount, int64_t cap) {
    if (*fw.n_undec == 0) return;
    __shared__ int32_t sf[kIdxMaxN];
    for (int i = threadIdx.x; i < fw.n; i += blockDim.x) sf[i] = fw.freq[i];
    __syncthreads();
    const int64_t count = dev_count(dcount, cap);
    const int nw = fw.n_pad / 16;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < count; r += (int64_t)gridDim.x * blockDim.x) {
        const int l1 = fw.l1[r];
        if (l1 < 0) continue;
        const int4* g = reinterpret_cast<const int4*>(fw.rows + (size_t)r * fw.n_pad);
        // lowest (freq, index) over the support: freq (< 2^31) and index packed into one 64-bit key
        unsigned long long best = ~0ULL;
        for (int w = 0; w < nw; ++w) {
            const int4 v = g[w];
            const uint32_t q[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
#pragma unroll
            for (int b = 0; b < 16; ++b)
                if ((q[b >> 2] >> (8 * (b & 3))) & 0xFFu) {
                    const int i = 16 * w + b;
                    best = min(best, ((unsigned long long)(uint32_t)sf[i] << 32) | (uint32_t)i);
                }
        }
        const int bin = (int)(best & 0xFFFFFFFFu) * (fw.Lmax + 1) + l1;
        fw.key_bin[r] = bin;
        atomicAdd(&fw.bin_hist[bin], 1);
    }
}

// exclusive scan of bin_hist[0, nb) into bin_start[0, nb] and bin_cursor[0, nb): one block, chunk per thread
__global__ void __launch_bounds__(1024) bin_scan_kernel(FilterWork fw, int nb) {
    if (*fw.n_undec == 0) return;
    __shared__ int32_t part[1024];
    const int t = threadIdx.x;
    const int chunk = (nb + 1023) / 1024;
    const int b0 = min(nb, t * chunk), b1 = min(nb, b0 + chunk);
    int32_t acc = 0;
    for (int b = b0; b < b1; ++b) acc += fw.bin_hist[b];
    part[t] = acc;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {   // Hillis-Steele inclusive scan of the partial sums
        const int32_t v = t >= off ? part[t - off] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    int32_t run = part[t] - acc;
    for (int b = b0; b < b1; ++b) {
        fw.bin_start[b] = run;
        fw.bin_cursor[b] = run;
        run += fw.bin_hist[b];
    }
    if (t == 1023) fw.bin_start[nb] = part[1023];
}

__global__ void bin_scatter_kernel(FilterWork fw, const unsigned long long* dcount, int64_t cap) {
    if (*fw.n_undec == 0 || (fw.idx_fallback && !gl_overflow(fw))) return;
    const int64_t count = dev_count(dcount, cap);
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < count; r += (int64_t)gridDim.x * blockDim.x) {
        if (fw.l1[r] < 0) continue;
        const int32_t pos = atomicAdd(&fw.bin_cursor[fw.key_bin[r]], 1);
        fw.list_row[pos] = (int32_t)r;
        fw.list_sig[pos] = fw.sig[r];
    }
}

#ifndef MAPLE_IDX_UNROLL
#define MAPLE_IDX_UNROLL 4
#endif
// warp per row g: scan the lists of g's support coordinates (lanes stride each range), stop at the first
// dominator found by any lane
constexpr int kIdxThreads = 256;
template <int WH>
__global__ void __launch_bounds__(kIdxThreads) dominance_idx_kernel(FilterWork fw, const unsigned long long* dcount,
                                                                   int64_t cap) {
    if (*fw.n_undec == 0 || (fw.idx_fallback && !gl_overflow(fw))) return;
    __shared__ uint32_t gcode[kIdxThreads / 32][2 * WH];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int Wh = fw.Wh, W2 = 2 * Wh;
    const int64_t count = dev_count(dcount, cap);
    const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    uint32_t* P = gcode[wib];
    uint32_t* N = P + WH;
    for (int64_t r = warp0; r < count; r += nwarps) {
        if (fw.keep[r] != 2) continue;   // decided by the tiled prefix scan (or invalid)
        const int l1 = fw.l1[r];
        __syncwarp();
        for (int w = lane; w < Wh; w += 32) {
            P[w] = fw.codes[(size_t)r * W2 + w];
            N[w] = fw.codes[(size_t)r * W2 + Wh + w];
        }
        const uint4 gs = fw.sig[r];
        __syncwarp();
        const int8_t* g = fw.rows + (size_t)r * fw.n_pad;
        int32_t wit = -1;
        for (int i0 = 0; i0 < fw.n && wit < 0; i0 += 32) {
            const int i = i0 + lane;
            unsigned nzm = __ballot_sync(0xffffffffu, i < fw.n && g[i] != 0);
            while (nzm && wit < 0) {
                const int c = i0 + __ffs(nzm) - 1;
                nzm &= nzm - 1;
                const int bin0 = c * (fw.Lmax + 1);
                const int32_t lo = fw.bin_start[bin0], hi = fw.bin_start[bin0 + l1];
                // MAPLE_IDX_UNROLL chunks of 32 list entries per pass: their signature loads are issued together
                // (the loop is L2-latency bound), then the chunks are tested in order, so the witness is the
                // first dominator in list order exactly as with one chunk per pass
                constexpr int U = MAPLE_IDX_UNROLL;
                bool done = false;
                for (int32_t p0 = lo; p0 < hi && !done; p0 += 32 * U) {
                    uint4 hs[U];
#pragma unroll
                    for (int k = 0; k < U; ++k) {
                        const int32_t p = p0 + 32 * k + lane;
                        hs[k] = p < hi ? fw.list_sig[p] : make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
                    }
#pragma unroll
                    for (int k = 0; k < U; ++k) {
                        const int32_t p = p0 + 32 * k + lane;
                        bool found = false;
                        const uint32_t pv = (hs[k].x & ~gs.x) | (hs[k].y & ~gs.y) | (hs[k].z & ~gs.z) | (hs[k].w & ~gs.w);
                        const uint32_t nv = (hs[k].x & ~gs.z) | (hs[k].y & ~gs.w) | (hs[k].z & ~gs.x) | (hs[k].w & ~gs.y);
                        if (p < hi && (pv == 0u || nv == 0u)) {
                            const uint32_t* hc = fw.codes + (size_t)fw.list_row[p] * W2;
                            uint32_t pos_v = 0, neg_v = 0;
                            for (int w = 0; w < Wh; ++w) {
                                const uint32_t hp = hc[w], hn = hc[Wh + w];
                                pos_v |= (hp & ~P[w]) | (hn & ~N[w]);
                                neg_v |= (hp & ~N[w]) | (hn & ~P[w]);
                            }
                            found = pos_v == 0u || neg_v == 0u;
                        }
                        const unsigned fm = __ballot_sync(0xffffffffu, found);
                        if (fm) {
                            wit = fw.list_row[p0 + 32 * k + __ffs(fm) - 1];
                            done = true;
                            break;
                        }
                    }
                }
            }
        }
        if (lane == 0) {
            fw.keep[r] = wit < 0 ? 1 : 0;
            fw.witness[r] = wit;
        }
    }
}

// ---- level-synchronous filter over ⊑-minimal rows (algo 3) ----
// If some row h ⊑ ±g, then some ⊑-minimal row m ⊑ h ⊑ ±g (⊑ is a partial order on the finite pool), and
// L1(m) < L1(g). So g is dominated iff a MINIMAL row of smaller L1 dominates it, and g need only meet those.
// Levels L = 1, 2, ... (L1 norms) are decided in order: the rows of level L that the tiled prefix left undecided
// are tested against the minimal rows of levels < L filed under their support coordinates (key coordinate
// κ(h) ∈ supp(h) ⊆ supp(g), as in the indexed filter); then level L's minimal rows are appended to their key
// coordinate's list. The pairs are blocked coordinate-major: a work item is (c, 256 rows g of level L with
// c ∈ supp(g), a segment of c's list), the list tiles staged in shared memory and shared by the 256 rows.
// The keep bit is defined pairwise, so it equals the other algorithms' (only the witness may differ).
constexpr int kLvThreads = 256, kLvTile = 512, kLvSeg = 512;

// G lists: every undecided row g (keep == 2) is filed under bin L1(g) n + c for each c ∈ supp(g);
// pass 0 counts (gl_cursor as histogram), pass 1 scatters (gl_cursor as cursor)
__global__ void glist_kernel(FilterWork fw, const unsigned long long* dcount, int64_t cap, int pass) {
    if (*fw.n_undec == 0) return;
    if (pass == 1 && gl_overflow(fw)) return;
    const int64_t count = dev_count(dcount, cap);
    const int nw = fw.n_pad / 16, n = fw.n;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < count; r += (int64_t)gridDim.x * blockDim.x) {
        if (fw.keep[r] != 2) continue;
        const int base = fw.l1[r] * n;
        const int4* g = reinterpret_cast<const int4*>(fw.rows + (size_t)r * fw.n_pad);
        for (int w = 0; w < nw; ++w) {
            const int4 v = g[w];
            const uint32_t q[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
#pragma unroll
            for (int b = 0; b < 16; ++b)
                if ((q[b >> 2] >> (8 * (b & 3))) & 0xFFu) {
                    int32_t* slot = &fw.gl_cursor[base + 16 * w + b];
                    if (pass == 0) atomicAdd(slot, 1);
                    else fw.gl_rows[atomicAdd(slot, 1)] = (int32_t)r;
                }
        }
    }
}

// exclusive scan of hist[0, nb) into start[0, nb] and cursor[0, nb): one block of 1024 threads
__global__ void __launch_bounds__(1024) scan_bins_kernel(const int32_t* n_undec, int32_t* hist, int nb, int32_t* start,
                                                         int32_t* cursor) {
    if (*n_undec == 0) return;
    __shared__ int32_t part[1024];
    const int t = threadIdx.x;
    const int chunk = (nb + 1023) / 1024;
    const int b0 = min(nb, t * chunk), b1 = min(nb, b0 + chunk);
    int32_t acc = 0;
    for (int b = b0; b < b1; ++b) acc += hist[b];
    part[t] = acc;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const int32_t v = t >= off ? part[t - off] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    int32_t run = part[t] - acc;
    for (int b = b0; b < b1; ++b) {   // (cursor may alias hist)
        const int32_t h = hist[b];
        start[b] = run;
        cursor[b] = run;
        run += h;
    }
    if (t == 1023) start[nb] = part[1023];
}

// Bit-sliced pair test. A warp owns 32 rows g (lane j: g_j) and keeps, for every fold bit b, the 32-bit masks
// {j : b ∈ fold(P_gj)} and {j : b ∈ fold(N_gj)} in shared memory. A lane takes one list row h and intersects the
// masks of h's fold bits: h ⊑ g_j needs fold(P_h) ⊆ fold(P_gj) and fold(N_h) ⊆ fold(N_gj) (bit j survives the ANDs
// over P_h's bits of the P masks and over N_h's bits of the N masks), h ⊑ -g_j the same with P and N of g exchanged.
// So one lane tests h against 32 rows at once and stops as soon as no row survives (usually after a few bits); the
// surviving (h, g_j) pairs get the exact test on the full codes.
__device__ void level_tile(const FilterWork& fw, int L, int32_t* work) {
    constexpr int NWARP = kLvThreads / 32;
    __shared__ int32_t pre[kIdxMaxN + 1];
    __shared__ uint4 tsig[kLvTile];
    __shared__ int32_t trow[kLvTile];
    __shared__ uint2 mk[NWARP][64];        // per warp, fold bit b: (P mask, N mask) over its 32 rows
    __shared__ int32_t grow[NWARP][32];    // the warp's rows g
    __shared__ uint32_t dead[NWARP];       // rows of the warp found dominated in this item
    const int n = fw.n, Wh = fw.Wh, W2 = 2 * Wh, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int32_t* gs = fw.gl_start + (size_t)L * n;
    const int lb = fw.Lmax + 1;
    // work items per coordinate: ceil(|G_{L,c}| / 256) x ceil(|H_c| / kLvSeg); block-wide exclusive scan over c
    {
        constexpr int PER = (kIdxMaxN + kLvThreads - 1) / kLvThreads;
        int32_t v[PER], acc = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int c = tid * PER + k;
            int32_t it = 0;
            if (c < n) {
                const int32_t ng = gs[c + 1] - gs[c], nh = fw.h_fill[c];
                it = ((ng + kLvThreads - 1) / kLvThreads) * ((nh + kLvSeg - 1) / kLvSeg);
            }
            v[k] = acc;
            acc += it;
        }
        __shared__ int32_t wsum[NWARP];
        int32_t x = acc;   // inclusive warp scan of the per-thread totals
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[wid] = x;
        __syncthreads();
        if (tid == 0) {
            int32_t run = 0;
            for (int w = 0; w < NWARP; ++w) {
                const int32_t t2 = wsum[w];
                wsum[w] = run;
                run += t2;
            }
        }
        __syncthreads();
        const int32_t excl = x - acc + wsum[wid];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int c = tid * PER + k;
            if (c <= n) pre[c] = excl + v[k];
        }
        if (tid == kLvThreads - 1 && (tid + 1) * PER <= n) pre[n] = excl + acc;
        __syncthreads();
    }
    const int32_t total = pre[n];
    volatile uint8_t* vkeep = fw.keep;
    // items are taken dynamically (one atomic per item per block): their cost varies with how soon rows die
    __shared__ int32_t s_item;
    if (tid == 0) s_item = atomicAdd(work, 1);
    __syncthreads();
    for (int32_t item = s_item; item < total;) {
        int lo = 0, hi = n;   // the coordinate c with pre[c] <= item < pre[c + 1]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (pre[mid] <= item) lo = mid;
            else hi = mid;
        }
        const int c = lo;
        const int32_t nh = fw.h_fill[c];
        const int32_t nseg = (nh + kLvSeg - 1) / kLvSeg;
        const int32_t local = item - pre[c], gi = local / nseg, si = local % nseg;
        const int32_t e = gs[c] + gi * kLvThreads + tid;
        int32_t g = -1;
        if (e < gs[c + 1]) g = fw.gl_rows[e];
        const bool mine = g >= 0 && vkeep[g] == 2;
        uint32_t alive = __ballot_sync(0xffffffffu, mine);
        const uint4 sg = mine ? fw.sig[g] : make_uint4(0u, 0u, 0u, 0u);
        grow[wid][lane] = g;
        if (lane == 0) dead[wid] = 0u;
        // transpose the 32 rows' folds into per-bit masks: lane b writes bits b and b + 32
#pragma unroll 4
        for (int b = 0; b < 32; ++b) {
            const uint32_t p0 = __ballot_sync(0xffffffffu, (sg.x >> b) & 1u), p1 = __ballot_sync(0xffffffffu, (sg.y >> b) & 1u);
            const uint32_t n0 = __ballot_sync(0xffffffffu, (sg.z >> b) & 1u), n1 = __ballot_sync(0xffffffffu, (sg.w >> b) & 1u);
            if (lane == b) {
                mk[wid][b] = make_uint2(p0, n0);
                mk[wid][b + 32] = make_uint2(p1, n1);
            }
        }
        __syncwarp();
        const int32_t h0 = fw.bin_start[c * lb] + si * kLvSeg;
        const int32_t h1 = min(fw.bin_start[c * lb] + nh, h0 + kLvSeg);
        for (int32_t t0 = h0; t0 < h1; t0 += kLvTile) {
            if (!__syncthreads_or(alive != 0u)) break;
            const int lim = min(kLvTile, h1 - t0);
            for (int i = tid; i < lim; i += kLvThreads) {
                tsig[i] = fw.list_sig[t0 + i];
                trow[i] = fw.list_row[t0 + i];
            }
            __syncthreads();
            // rows another item (or another warp's exact test) has decided meanwhile
            alive &= __ballot_sync(0xffffffffu, g >= 0 && vkeep[g] == 2) & ~dead[wid];
            for (int i0 = 0; i0 < lim && alive; i0 += 32) {
                const int i = i0 + lane;
                uint32_t pos = 0u, neg = 0u;
                if (i < lim) {
                    const uint4 hs = tsig[i];
                    pos = alive;
                    neg = alive;
                    uint64_t fp = ((uint64_t)hs.y << 32) | hs.x, fn = ((uint64_t)hs.w << 32) | hs.z;
                    while (fp && (pos | neg)) {
                        const int b = __ffsll((long long)fp) - 1;
                        fp &= fp - 1;
                        const uint2 m = mk[wid][b];
                        pos &= m.x;
                        neg &= m.y;
                    }
                    while (fn && (pos | neg)) {
                        const int b = __ffsll((long long)fn) - 1;
                        fn &= fn - 1;
                        const uint2 m = mk[wid][b];
                        pos &= m.y;
                        neg &= m.x;
                    }
                }
                uint32_t cand = pos | neg;
                if (cand) {   // exact test on the codes for the surviving (h, g_j)
                    const int32_t hr = trow[i];
                    const uint32_t* hc = fw.codes + (size_t)hr * W2;
                    while (cand) {
                        const int j = __ffs(cand) - 1;
                        cand &= cand - 1;
                        const int32_t gj = grow[wid][j];
                        const uint32_t* gc = fw.codes + (size_t)gj * W2;
                        uint32_t pos_v = 0, neg_v = 0;
                        for (int w = 0; w < Wh; ++w) {
                            const uint32_t hp = hc[w], hn = hc[Wh + w], gp = gc[w], gn = gc[Wh + w];
                            pos_v |= (hp & ~gp) | (hn & ~gn);
                            neg_v |= (hp & ~gn) | (hn & ~gp);
                        }
                        if (pos_v == 0u || neg_v == 0u) {
                            fw.witness[gj] = hr;
                            vkeep[gj] = 0;
                            atomicOr(&dead[wid], 1u << j);
                        }
                    }
                }
                __syncwarp();
                alive &= ~dead[wid];
            }
        }
        __syncthreads();   // the tile buffers and masks are reused by the next item
        if (tid == 0) s_item = atomicAdd(work, 1);
        __syncthreads();
        item = s_item;
    }
}

// level L decided: its remaining undecided rows are minimal; every minimal row of level L joins its key
// coordinate's list (the lists hold the minimal rows of the levels below the one being tested)
__device__ void level_append(const FilterWork& fw, int L) {
    const int32_t lo = fw.level_start[L], hi = fw.level_start[L + 1];
    const int lb = fw.Lmax + 1;
    for (int32_t q = lo + blockIdx.x * blockDim.x + threadIdx.x; q < hi; q += gridDim.x * blockDim.x) {
        const int32_t r = fw.order[q];
        uint8_t k = fw.keep[r];
        if (k == 2) {
            k = 1;
            fw.keep[r] = 1;
        }
        if (k == 1) {
            const int c = fw.key_bin[r] / lb;
            const int32_t p = fw.bin_start[c * lb] + atomicAdd(&fw.h_fill[c], 1);
            fw.list_row[p] = r;
            fw.list_sig[p] = fw.sig[r];
        }
    }
}

// grid-wide barrier for the co-resident (cooperatively launched) level kernel: arrival count + generation
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* vgen = gen;
        const unsigned g0 = *vgen;
        __threadfence();
        if (atomicAdd(count, 1u) == gridDim.x - 1) {
            *count = 0u;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*vgen == g0) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

// All levels in one cooperative launch: level L's tile phase (if it has undecided rows) runs between two grid
// barriers — after every lower level's appends, before its own — and appends need no barrier of their own (a
// coordinate's list order is irrelevant). Returns at once when the tiled prefix decided every row.
__global__ void __launch_bounds__(kLvThreads) level_filter_kernel(FilterWork fw, unsigned* bar) {
    if (*fw.n_undec == 0 || gl_overflow(fw)) return;
    const int n = fw.n;
    for (int L = 1; L <= fw.Lmax; ++L) {
        if (fw.level_start[L] == fw.level_start[L + 1]) continue;   // no row has L1 = L
        if (fw.gl_start[(size_t)(L + 1) * n] > fw.gl_start[(size_t)L * n]) {
            grid_barrier(bar, bar + 1);
            level_tile(fw, L, reinterpret_cast<int32_t*>(bar + 2) + L);
            grid_barrier(bar, bar + 1);
        }
        level_append(fw, L);
    }
}

__global__ void keep_valid_kernel(const uint8_t* valid, const unsigned long long* dcount, int64_t cap, uint8_t* keep,
                                  int32_t* witness) {
    const int64_t count = dev_count(dcount, cap);
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < count; r += (int64_t)gridDim.x * blockDim.x) {
        keep[r] = valid[r];
        witness[r] = -1;
    }
}

__global__ void clear_keep_kernel(const unsigned long long* dcount, int64_t cap, uint8_t* keep) {
    const int64_t count = dev_count(dcount, cap);
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < count; r += (int64_t)gridDim.x * blockDim.x)
        keep[r] = 0;
}

// Gather the selected rows; *nz_max gets the largest nonzero count among them (the ELL width of the set, known
// to the host at the extraction's one synchronisation, so augmentation needs none).
__global__ void compact_kernel(const int8_t* __restrict__ rows, const uint8_t* sel, const unsigned long long* dcount,
                               int64_t cap, int n_pad, int8_t* out, unsigned long long* n_out,
                               unsigned long long* nz_max) {
    const int nw = n_pad / 16;
    const int64_t count = dev_count(dcount, cap);
    int my_nz = 0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < count; r += (int64_t)gridDim.x * blockDim.x) {
        if (!sel[r]) continue;
        const unsigned long long o = atomicAdd(n_out, 1ULL);
        const int4* s = reinterpret_cast<const int4*>(rows + (size_t)r * n_pad);
        int4* dd = reinterpret_cast<int4*>(out + (size_t)o * n_pad);
        int nz = 0;
        for (int i = 0; i < nw; ++i) {
            const int4 v = s[i];
            dd[i] = v;
            nz += (__popc(__vcmpne4((uint32_t)v.x, 0u)) + __popc(__vcmpne4((uint32_t)v.y, 0u)) +
                   __popc(__vcmpne4((uint32_t)v.z, 0u)) + __popc(__vcmpne4((uint32_t)v.w, 0u))) >> 3;
        }
        my_nz = max(my_nz, nz);
    }
    my_nz = __reduce_max_sync(0xffffffffu, my_nz);
    if ((threadIdx.x & 31) == 0 && my_nz) atomicMax(nz_max, (unsigned long long)my_nz);
}

__global__ void sortkey_kernel(const int8_t* __restrict__ rows, int64_t k, int n_pad, uint32_t* keys, int32_t* idx) {
    const int nk = n_pad / 4;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < k * nk; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / nk;
        const int w = (int)(t % nk);
        const uint8_t* g = reinterpret_cast<const uint8_t*>(rows + (size_t)r * n_pad + 4 * w);
        keys[t] = ((uint32_t)(g[0] ^ 0x80) << 24) | ((uint32_t)(g[1] ^ 0x80) << 16) |
                  ((uint32_t)(g[2] ^ 0x80) << 8) | (uint32_t)(g[3] ^ 0x80);
        if (w == 0) idx[r] = (int32_t)r;
    }
}

__device__ __forceinline__ int key_cmp(const uint32_t* a, const uint32_t* b, int nk) {
    for (int i = 0; i < nk; ++i) {
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    }
    return 0;
}

// one merge pass: runs of width w -> 2w
__global__ void merge_pass_kernel(const uint32_t* keys, int nk, const int32_t* in, int32_t* out, int64_t k, int64_t w) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < k; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t pair = p / (2 * w);
        const int64_t ls = pair * 2 * w;
        const int64_t rs = min(ls + w, k);
        const int64_t re = min(ls + 2 * w, k);
        const int32_t e = in[p];
        const uint32_t* ke = keys + (size_t)e * nk;
        int64_t lo, hi, off;
        if (p < rs) {  // left element: count right elements < e
            lo = rs;
            hi = re;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (key_cmp(keys + (size_t)in[mid] * nk, ke, nk) < 0) lo = mid + 1; else hi = mid;
            }
            off = (p - ls) + (lo - rs);
        } else {  // right element: count left elements <= e
            lo = ls;
            hi = rs;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (key_cmp(keys + (size_t)in[mid] * nk, ke, nk) <= 0) lo = mid + 1; else hi = mid;
            }
            off = (p - rs) + (lo - ls);
        }
        out[ls + off] = e;
    }
}

// Whole sort in one CTA for small k: keys and indices in shared memory, bottom-up merge passes separated
// by __syncthreads, then the gather of the sorted rows.
__global__ void __launch_bounds__(1024) small_sort_kernel(const int8_t* __restrict__ rows, int k, int n_pad,
                                                          int8_t* out) {
    extern __shared__ __align__(16) uint32_t ss[];
    const int nk = n_pad / 4;
    uint32_t* keys = ss;
    int32_t* ia = reinterpret_cast<int32_t*>(keys + (size_t)k * nk);
    int32_t* ib = ia + k;
    for (int t = threadIdx.x; t < k * nk; t += blockDim.x) {
        const int r = t / nk, w = t % nk;
        const uint8_t* g = reinterpret_cast<const uint8_t*>(rows + (size_t)r * n_pad + 4 * w);
        keys[t] = ((uint32_t)(g[0] ^ 0x80) << 24) | ((uint32_t)(g[1] ^ 0x80) << 16) | ((uint32_t)(g[2] ^ 0x80) << 8) |
                  (uint32_t)(g[3] ^ 0x80);
    }
    for (int r = threadIdx.x; r < k; r += blockDim.x) ia[r] = r;
    __syncthreads();
    for (int w = 1; w < k; w <<= 1) {
        for (int p = threadIdx.x; p < k; p += blockDim.x) {
            const int pair = p / (2 * w);
            const int ls = pair * 2 * w, rs = min(ls + w, k), re = min(ls + 2 * w, k);
            const int e = ia[p];
            const uint32_t* ke = keys + (size_t)e * nk;
            int lo, hi, off;
            if (p < rs) {
                lo = rs;
                hi = re;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (key_cmp(keys + (size_t)ia[mid] * nk, ke, nk) < 0) lo = mid + 1; else hi = mid;
                }
                off = (p - ls) + (lo - rs);
            } else {
                lo = ls;
                hi = rs;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (key_cmp(keys + (size_t)ia[mid] * nk, ke, nk) <= 0) lo = mid + 1; else hi = mid;
                }
                off = (p - rs) + (lo - ls);
            }
            ib[ls + off] = e;
        }
        __syncthreads();
        int32_t* t = ia;
        ia = ib;
        ib = t;
    }
    const int nw = n_pad / 16;
    for (int t = threadIdx.x; t < k * nw; t += blockDim.x) {
        const int r = t / nw, w = t % nw;
        reinterpret_cast<int4*>(out + (size_t)r * n_pad)[w] = reinterpret_cast<const int4*>(rows + (size_t)ia[r] * n_pad)[w];
    }
}

__global__ void gather_kernel(const int8_t* __restrict__ rows, const int32_t* idx, int64_t k, int n_pad, int8_t* out) {
    const int nw = n_pad / 16;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < k * nw; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / nw;
        const int w = (int)(t % nw);
        reinterpret_cast<int4*>(out + (size_t)r * n_pad)[w] =
            reinterpret_cast<const int4*>(rows + (size_t)idx[r] * n_pad)[w];
    }
}

// lexicographic compare of row a with (neg ? -b : b), int8 entries, first n coordinates
__device__ __forceinline__ int lex_cmp_signed(const int8_t* a, const int8_t* b, bool neg, int n) {
    for (int k = 0; k < n; ++k) {
        const int x = a[k], y = neg ? -(int)b[k] : (int)b[k];
        if (x != y) return x < y ? -1 : 1;
    }
    return 0;
}

// D = S ∪ -S in lexicographic order, from S sorted ascending: negation reverses the order, so -S ascending is
// N[j] = -S[k-1-j], and no row of S equals a row of -S (canonical rows have a positive first nonzero). Row i of S
// goes to i plus its rank in N (binary search): a merge, no sort. D is closed under negation and negation reverses
// the order, so D[2k-1-e] = -D[e]: the same thread writes -S[i] at 2k-1-(i + rank) (half the searches).
__global__ void signed_merge_kernel(const int8_t* __restrict__ S, int64_t k, int n, int n_pad, int8_t* out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        const int8_t* self = S + (size_t)i * n_pad;
        // rank: number of rows of N smaller than S[i]
        int64_t lo = 0, hi = k;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            const int c = -lex_cmp_signed(self, S + (size_t)(k - 1 - mid) * n_pad, true, n);   // N[mid] vs self
            if (c < 0) lo = mid + 1;
            else hi = mid;
        }
        const int64_t pos = i + lo;
        // rows are n_pad bytes, n_pad a multiple of 16: 16-byte copies, bytewise negation (mod 256, as int8_t(-v))
        const uint4* src = reinterpret_cast<const uint4*>(self);
        uint4* dp = reinterpret_cast<uint4*>(out + (size_t)pos * n_pad);
        uint4* dn = reinterpret_cast<uint4*>(out + (size_t)(2 * k - 1 - pos) * n_pad);
        for (int q = 0; q < n_pad / 16; ++q) {
            const uint4 v = src[q];
            dp[q] = v;
            dn[q] = make_uint4(__vneg4(v.x), __vneg4(v.y), __vneg4(v.z), __vneg4(v.w));
        }
    }
}

inline unsigned grid_for(int64_t work, int threads = 256, int64_t max_blocks = 148 * 16) {
    int64_t b = (work + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > max_blocks) b = max_blocks;
    return (unsigned)b;
}

}  // namespace

cudaError_t launch_dedupe(const int8_t* rows, const unsigned long long* dcount, int64_t cap, int row_stride,
                          int n_pad, const HashSet& hs, cudaStream_t s) {
    if (cap <= 0) return cudaSuccess;
    dedupe_kernel<<<grid_for(cap, 256, 148 * 8), 256, 0, s>>>(rows, dcount, cap, row_stride, n_pad, hs);
    finish_dedupe_kernel<<<grid_for(hs.pool_cap, 256, 148 * 4), 256, 0, s>>>(rows, row_stride, n_pad, hs);
    return cudaGetLastError();
}

cudaError_t launch_check_codes(const int8_t* rows, const unsigned long long* dcount, int64_t cap, const CheckParams& cp,
                               FilterWork& fw, int encode, uint8_t* flags, unsigned long long* n_bad, cudaStream_t s) {
    if (cap <= 0) return cudaSuccess;
    const size_t smem = (size_t)(((cp.m + 1 + 2 * cp.nnz + 2 * cp.n + 2 * fw.Wh) + 3) & ~3) * 4 +
                        (size_t)kCheckThreads * (cp.n_pad + 4);
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(check_codes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    check_codes_kernel<<<grid_for(cap, kCheckThreads, 148 * 8), kCheckThreads, smem, s>>>(rows, dcount, cap, cp, fw,
                                                                                          flags, n_bad, encode);
    return cudaGetLastError();
}

static cudaError_t launch_filter_tiled(const unsigned long long* dcount, int64_t cap, FilterWork& fw, cudaStream_t s,
                                       int* launches) {
    cudaError_t e;
    const int nb = fw.Lmax + 1;
    if ((e = cudaMemsetAsync(fw.hist, 0, sizeof(int32_t) * (fw.Lmax + 2), s)) != cudaSuccess) return e;
    hist_kernel<<<grid_for(cap, 256, 148 * 4), 256, nb * 4, s>>>(fw.l1, dcount, cap, fw.hist, nb);
    scan_kernel<<<1, 32, 0, s>>>(fw.hist, nb, fw.level_start, fw.cursor);
    scatter_kernel<<<grid_for((cap + 7) / 8, 256, 148 * 4), 256, 2 * nb * 4, s>>>(fw.l1, dcount, cap, fw.cursor,
                                                                                  fw.order, nb);
    clear_keep_kernel<<<grid_for(cap), 256, 0, s>>>(dcount, cap, fw.keep);
    *launches += 4;
    const unsigned blocks = grid_for(cap, kFilterThreads, 148 * 4);
#define MAPLE_DOM(WHV)                                                                                       \
    if (fw.Wh <= WHV) {                                                                                      \
        dominance_kernel<WHV><<<blocks, kFilterThreads, 0, s>>>(fw);                                         \
    } else
    MAPLE_DOM(1) MAPLE_DOM(2) MAPLE_DOM(4) MAPLE_DOM(8) MAPLE_DOM(16) MAPLE_DOM(32) return cudaErrorInvalidValue;
#undef MAPLE_DOM
    *launches += 1;
    return cudaGetLastError();
}


cudaError_t launch_filter(const unsigned long long* dcount, int64_t cap, const uint8_t* valid, FilterWork& fw,
                          int filter_minimal, cudaStream_t s, int* launches) {
    if (cap <= 0) return cudaSuccess;
    if (!filter_minimal) {
        keep_valid_kernel<<<grid_for(cap), 256, 0, s>>>(valid, dcount, cap, fw.keep, fw.witness);
        *launches += 1;
        return cudaGetLastError();
    }
    cudaError_t e;
    const int algo = fw.algo;
    fw.scan_cap = algo >= 2 ? 2 * kTile : 0x7fffffff;
    if ((e = cudaMemsetAsync(fw.n_undec, 0, sizeof(int32_t), s)) != cudaSuccess) return e;
    if ((e = launch_filter_tiled(dcount, cap, fw, s, launches)) != cudaSuccess) return e;
    if (algo == 3) {   // rows the prefix did not decide: level by level against the minimal rows below
        if (fw.n > kIdxMaxN) return cudaErrorInvalidValue;
        const int lb = fw.Lmax + 1;
        const int nbins = fw.n * lb;
        if ((e = cudaMemsetAsync(fw.freq, 0, sizeof(int32_t) * fw.n, s)) != cudaSuccess) return e;
        if ((e = cudaMemsetAsync(fw.bin_hist, 0, sizeof(int32_t) * nbins, s)) != cudaSuccess) return e;
        if ((e = cudaMemsetAsync(fw.gl_cursor, 0, sizeof(int32_t) * nbins, s)) != cudaSuccess) return e;
        if ((e = cudaMemsetAsync(fw.h_fill, 0, sizeof(int32_t) * fw.n, s)) != cudaSuccess) return e;
        coord_freq_kernel<<<grid_for(cap, 256, 148 * 4), 256, 0, s>>>(fw, dcount, cap);
        key_bin_kernel<<<grid_for(cap, 256, 148 * 8), 256, 0, s>>>(fw, dcount, cap);
        bin_scan_kernel<<<1, 1024, 0, s>>>(fw, nbins);   // bin_start: each key coordinate's list capacity
        glist_kernel<<<grid_for(cap, 256, 148 * 8), 256, 0, s>>>(fw, dcount, cap, 0);
        scan_bins_kernel<<<1, 1024, 0, s>>>(fw.n_undec, fw.gl_cursor, nbins, fw.gl_start, fw.gl_cursor);
        glist_kernel<<<grid_for(cap, 256, 148 * 8), 256, 0, s>>>(fw, dcount, cap, 1);
        *launches += 6;
        int per_sm = 0, dev = 0, nsm = 148;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, level_filter_kernel, kLvThreads, 0)) != cudaSuccess)
            return e;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const int grid = std::max(1, per_sm) * nsm;
        // after the fill counters: 2 grid-barrier words, then one work counter per level
        unsigned* bar = reinterpret_cast<unsigned*>(fw.h_fill + fw.n);
        if ((e = cudaMemsetAsync(bar, 0, (2 + fw.Lmax + 2) * sizeof(unsigned), s)) != cudaSuccess) return e;
        void* args[] = {&fw, &bar};
        if ((e = cudaLaunchCooperativeKernel((void*)level_filter_kernel, grid, kLvThreads, args, 0, s)) != cudaSuccess)
            return e;
        *launches += 1;
        // the indexed pass instead, when the G lists did not fit (its kernels return at once otherwise)
        fw.idx_fallback = 1;
        bin_scatter_kernel<<<grid_for(cap), 256, 0, s>>>(fw, dcount, cap);
        const unsigned iblocks = grid_for((cap + 7) / 8, kIdxThreads, 148 * 8);
#define MAPLE_IDX3(WHV)                                                                 \
        if (fw.Wh <= WHV) {                                                             \
            dominance_idx_kernel<WHV><<<iblocks, kIdxThreads, 0, s>>>(fw, dcount, cap); \
        } else
        MAPLE_IDX3(2) MAPLE_IDX3(8) MAPLE_IDX3(32) return cudaErrorInvalidValue;
#undef MAPLE_IDX3
        *launches += 2;
        return cudaGetLastError();
    }
    if (algo == 2) {   // rows the prefix did not decide: indexed by key coordinate and L1
        if (fw.n > kIdxMaxN) return cudaErrorInvalidValue;
        const int nbins = fw.n * (fw.Lmax + 1);
        if ((e = cudaMemsetAsync(fw.freq, 0, sizeof(int32_t) * fw.n, s)) != cudaSuccess) return e;
        if ((e = cudaMemsetAsync(fw.bin_hist, 0, sizeof(int32_t) * nbins, s)) != cudaSuccess) return e;
        coord_freq_kernel<<<grid_for(cap, 256, 148 * 4), 256, 0, s>>>(fw, dcount, cap);
        key_bin_kernel<<<grid_for(cap, 256, 148 * 8), 256, 0, s>>>(fw, dcount, cap);
        bin_scan_kernel<<<1, 1024, 0, s>>>(fw, nbins);
        bin_scatter_kernel<<<grid_for(cap), 256, 0, s>>>(fw, dcount, cap);
        *launches += 4;
        const unsigned blocks = grid_for((cap + 7) / 8, kIdxThreads, 148 * 8);
#define MAPLE_IDX(WHV)                                                                 \
        if (fw.Wh <= WHV) {                                                            \
            dominance_idx_kernel<WHV><<<blocks, kIdxThreads, 0, s>>>(fw, dcount, cap); \
        } else
        MAPLE_IDX(2) MAPLE_IDX(8) MAPLE_IDX(32) return cudaErrorInvalidValue;
#undef MAPLE_IDX
        *launches += 1;
        return cudaGetLastError();
    }
    return cudaSuccess;
}

cudaError_t launch_signed_merge(const int8_t* S, int64_t k, int n, int n_pad, int8_t* out, cudaStream_t s) {
    if (k <= 0) return cudaSuccess;
    signed_merge_kernel<<<grid_for(k), 256, 0, s>>>(S, k, n, n_pad, out);
    return cudaGetLastError();
}

cudaError_t launch_compact(const int8_t* rows, const uint8_t* sel, const unsigned long long* dcount, int64_t cap,
                           int n_pad, int8_t* out, unsigned long long* n_out, unsigned long long* nz_max, cudaStream_t s) {
    if (cap <= 0) return cudaSuccess;
    compact_kernel<<<grid_for(cap), 256, 0, s>>>(rows, sel, dcount, cap, n_pad, out, n_out, nz_max);
    return cudaGetLastError();
}

cudaError_t launch_lex_sort(const int8_t* rows, int64_t k, int n, int n_pad, uint32_t* keys, int32_t* idx0,
                            int32_t* idx1, int8_t* out, cudaStream_t s, int* launches) {
    (void)n;
    if (k <= 0) return cudaSuccess;
    const int nk = n_pad / 4;
    const size_t ssm = (size_t)k * nk * 4 + (size_t)k * 8;
    if (k <= 8192 && ssm <= 160 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(small_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
        if (e != cudaSuccess) return e;
        small_sort_kernel<<<1, 1024, ssm, s>>>(rows, (int)k, n_pad, out);
        *launches += 1;
        return cudaGetLastError();
    }
    sortkey_kernel<<<grid_for(k * nk), 256, 0, s>>>(rows, k, n_pad, keys, idx0);
    *launches += 1;
    int32_t* a = idx0;
    int32_t* b = idx1;
    for (int64_t w = 1; w < k; w <<= 1) {
        merge_pass_kernel<<<grid_for(k), 256, 0, s>>>(keys, nk, a, b, k, w);
        *launches += 1;
        int32_t* t = a;
        a = b;
        b = t;
    }
    gather_kernel<<<grid_for(k * (n_pad / 16)), 256, 0, s>>>(rows, a, k, n_pad, out);
    *launches += 1;
    return cudaGetLastError();
}

}  // namespace maple
