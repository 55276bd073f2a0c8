// C ABI of the MAPLE hot path (include/maple.h): context, extraction pipeline, merge, augmentation.
// Host code here only orchestrates: every step of the path runs in the kernels of k_*.cu; the host
// does the once-per-A exact lattice work of maple_create (lattice.cpp) and argument validation.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/maple.h"
#include "kernels.h"
#include "sparse_ell.h"
#include "lattice.h"

using namespace maple;

namespace {

// Device workspace: stream-ordered allocations from the device's default memory pool (kept cached with a
// maximal release threshold), so repeated contexts / calls do not pay cudaMalloc.
thread_local cudaStream_t g_alloc_stream = 0;

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t want) {
        if (want <= bytes) return cudaSuccess;
        if (p) cudaFreeAsync(p, g_alloc_stream);
        p = nullptr;
        bytes = 0;
        size_t b = std::max<size_t>(want, 256);
        cudaError_t e = cudaMallocAsync(&p, b, g_alloc_stream);
        if (e == cudaSuccess) bytes = b;
        return e;
    }
    void release() {
        if (p) cudaFreeAsync(p, g_alloc_stream);
        p = nullptr;
        bytes = 0;
    }
    template <class T>
    T* as() const { return reinterpret_cast<T*>(p); }
};

// Pinned host staging for per-call uploads: a copy from pageable memory first synchronises the stream, a copy
// from pinned memory is asynchronous. Bump-allocated per call; every call that uses it synchronises on the
// context stream before returning, so the next call may reuse it.
struct HostStage {
    unsigned char* p = nullptr;
    size_t bytes = 0, used = 0;
    cudaError_t reserve(size_t want) {
        used = 0;
        if (want <= bytes) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
        const size_t b = std::max<size_t>(want, 4096);
        cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&p), b);
        if (e == cudaSuccess) bytes = b;
        return e;
    }
    template <class T>
    T* take(size_t count) {   // 16-byte aligned slice; reserve() sized the total
        used = (used + 15) & ~size_t(15);
        T* r = reinterpret_cast<T*>(p + used);
        used += count * sizeof(T);
        return r;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = used = 0;
    }
};

inline int round_up(int v, int a) { return (v + a - 1) / a * a; }
inline uint64_t next_pow2(uint64_t v) {
    uint64_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

}  // namespace

struct maple_ctx {
    int device = 0;
    cudaStream_t stream = 0;
    int m = 0, n = 0, d = 0, n_pad = 16;
    std::vector<int32_t> A, l, u, box;
    std::vector<int64_t> B;       // n x d
    std::vector<double> Bp;       // d x n
    // device constants
    DevBuf A_rowptr, A_col, A_val, dl, du, dbox, B_nd, B_dn, B8, dBp, th_off, th_c0, th_c1;
    HostStage stage_aug, stage_tab;   // pinned upload staging (augmentation inputs, Adam step table)
    int tab_T = -1;                   // the step table on the device was built for (tab_T, tab_lr, betas)
    double tab_lr = 0, tab_b1 = 0, tab_b2 = 0;
    DevBuf ell_f, ell_own_f, ell_fix, ell_fixpos, ell_b, ell_owned, ell_pos_s, ell_pos_z;   // SIMT schedules of B (sparse_ell.h)
    int ell_conflicts = 0;
    DevBuf AT_ptr, AT_row, AT_val, fb, frows, fX;
    SparseB sb{};
    int nnz = 0, Lh = 0, Wh = 0;
    double rbound = 0;
    int binary = 0;               // every u_i - l_i == 1            // max_j sum_i |B+_ji| (u_i - l_i): bound on |round(z)| of any in-box g
    // params (Eq. 3 / Adam)
    double lam1 = 0.85, lam2 = 1.0, beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
    int filter_minimal = 1;
    int descent_kernel = 0;
    bool sb_ready = false;        // SIMT schedules built (build_sparse)
    DevBuf B16p, BT8p, B8p;       // CTA-pair kernel operands: B (f16 and int8, tcp_np x tcp_dp), B^T (int8, tcp_dp x tcp_np)
    int tcp_np = 0, tcp_dp = 0;   // padded shape of the CTA-pair kernel (0: the shape has none)
    bool tcp_ready = false;       // B16p / BT8p built (build_tcp)
    bool tcp_range_fail = false;  // an extraction saw an iterate beyond the f16 operand range: use SIMT from now on
    DevBuf trace;                 // debug timeline of the CTA-pair kernel (maple_debug_trace)
    bool trace_on = false;
    int filter_algo = 0;          // 0 auto (kAutoFilter), 1 tiled, 2 indexed, 3 level-synchronous
    int optimizer = 0;            // reading #24: 0 Adam, 1 GD, 2 sign-GD
    int harvest_final = 0;        // reading #25: 1 = harvest the final iterate only
    // workspace
    DevBuf ffreq, fkey, fbh, fbs, fbc, flrow, flsig;   // indexed filter (k_post.cu)
    DevBuf fgc, fgs, fgr, fhf;                         // level-synchronous filter: G lists, list fill counters
    DevBuf g0buf, z0buf;          // SIMT starts by DGEMM: g0 (chunk x n) and z0 = B+ g0 (chunk x d), fp64
    cublasHandle_t cublas = nullptr;
    DevBuf step_tab, cand, keys, idx, pool, counters, flags, codes, sig, l1, hist, level_start, cursor, order, keep,
        witness, tmp_rows, sortkeys, sidx0, sidx1, zout, z0out;
    DevBuf aQ, ac, ac0, aqg, aX, aF2, aIt, axb, af2b, atab, atoff;
    int64_t cand_cap = 0, pool_cap = 0, want_cand = 0, want_pool = 0;
    bool timings_pending = false;
    uint64_t table_slots = 0;
    std::string err;
    float t_extract[6] = {0, 0, 0, 0, 0, 0};
    float t_augment[3] = {0, 0, 0};
    int64_t launches = 0;
    int debug_keep = 0;
    std::vector<int8_t> dbg_cand;
    int64_t dbg_count = 0;
    cudaEvent_t ev[12] = {};  // 0-5: extraction phases, 8-10: augmentation
};

struct maple_dirset {
    maple_ctx* ctx = nullptr;
    int n = 0, n_pad = 16;
    int64_t size = 0, pool_size = 0, n_bad = 0;
    int8_t* rows = nullptr;       // size x n_pad, canonical, lex sorted
    int8_t* D = nullptr;          // 2*size x n_pad: rows ∪ -rows, lex sorted (lazily built)
    int32_t* D_nnz = nullptr;     // ELL of D (lazily built)
    uint32_t* D_words = nullptr;
    int D_nzmax = 1;   // ELL width of D: bound on the rows' nonzero counts, known when the set is finished
    cudaEvent_t ready = nullptr;  // recorded after the last device write to this set
};

// counters layout in ctx->counters: [0] cand_count, [1] pool_count, [2] n_bad, [3] n_keep, [4] overflow(int)
enum { C_CAND = 0, C_POOL = 1, C_BAD = 2, C_KEEP = 3, C_OVF = 4, C_MAXC = 5, C_NZMAX = 6, C_RANGE = 7, C_N = 8 };

#define FAIL(code, msg)              \
    do {                             \
        if (ctx) ctx->err = (msg);   \
        return (code);               \
    } while (0)

#define CU(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess) {                                                                   \
            if (ctx) ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);                \
            cudaGetLastError();                                                                    \
            return e_ == cudaErrorMemoryAllocation ? MAPLE_ERR_OOM : MAPLE_ERR_CUDA;               \
        }                                                                                          \
    } while (0)

namespace {

// maple_create's uploads go through this thread's pinned staging buffer as asynchronous copies (a pageable
// cudaMemcpy blocks per call); maple_create resets it on entry and synchronises the device before returning,
// so the buffer is free again for the thread's next create.
thread_local HostStage t_upload_stage;

template <class T>
cudaError_t upload(DevBuf& b, const std::vector<T>& v) {
    cudaError_t e = b.ensure(std::max<size_t>(1, v.size()) * sizeof(T));
    if (e != cudaSuccess) return e;
    if (v.empty()) return cudaSuccess;
    const size_t nb = v.size() * sizeof(T);
    HostStage& st = t_upload_stage;
    size_t off = (st.used + 15) & ~size_t(15);
    if (off + nb > st.bytes) {   // grow: the copies still reading the old buffer must finish first
        if ((e = cudaStreamSynchronize(g_alloc_stream)) != cudaSuccess) return e;
        if ((e = st.reserve(std::max(2 * st.bytes, nb + 4096))) != cudaSuccess) return e;
        off = 0;
    }
    std::memcpy(st.p + off, v.data(), nb);
    st.used = off + nb;
    return cudaMemcpyAsync(b.p, st.p + off, nb, cudaMemcpyHostToDevice, g_alloc_stream);
}

unsigned long long* counters(maple_ctx* c) { return c->counters.as<unsigned long long>(); }

int read_counters(maple_ctx* ctx, unsigned long long* h) {
    CU(cudaMemcpyAsync(h, ctx->counters.p, sizeof(unsigned long long) * C_N, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return MAPLE_OK;
}

constexpr int kGlEntriesPerRow = 32;   // G-list capacity per pool row (the level pass's support entries) ...
constexpr size_t kGlMaxEntries = size_t(64) << 20;   // ... up to 256 MB (beyond: the indexed pass, same keep set)
constexpr int kAutoFilter = 3;   // auto choice of the ⊑ filter's pair enumeration (n <= 1024)

// the ⊑ filter's pair enumeration: 1 tiled, 2 tiled prefix + key-coordinate index, 3 tiled prefix + level-synchronous
// minimal-row index (n <= 1024 for 2 and 3)
int resolved_filter_algo(const maple_ctx* ctx) {
    if (ctx->filter_algo == 1 || ctx->n > 1024) return 1;
    return ctx->filter_algo == 0 ? kAutoFilter : ctx->filter_algo;
}

// Size the candidate buffer, the hash set (pool + table) and the per-row work buffers, then reset the set.
int prepare_set(maple_ctx* ctx, int64_t cand_cap, int64_t pool_cap, int filter_minimal) {
    const int np = ctx->n_pad;
    // the hash set references rows by 31-bit indices (k_post.cu dedupe_kernel)
    if (cand_cap >= (int64_t(1) << 31) || pool_cap >= (int64_t(1) << 31)) return MAPLE_ERR_CAPACITY;
    if (cand_cap > ctx->cand_cap) {
        ctx->cand.release();
        CU(ctx->cand.ensure((size_t)cand_cap * np));
        ctx->cand_cap = cand_cap;
    }
    if (pool_cap > ctx->pool_cap) {
        const uint64_t slots = next_pow2((uint64_t)pool_cap * 2);
        ctx->pool.release();
        ctx->keys.release();
        ctx->idx.release();
        CU(ctx->pool.ensure((size_t)pool_cap * np));
        CU(ctx->keys.ensure(slots * 8));
        CU(ctx->idx.ensure((size_t)pool_cap * 8));   // the hash set's newslot array (int64 per pool row)
        ctx->table_slots = slots;
        ctx->pool_cap = pool_cap;
        const int64_t K = pool_cap;
        CU(ctx->flags.ensure(K));
        CU(ctx->keep.ensure(K));
        CU(ctx->witness.ensure(K * 4));
        CU(ctx->order.ensure(K * 4));
        CU(ctx->l1.ensure(K * 4));
        CU(ctx->sig.ensure((size_t)K * 16));
        CU(ctx->fkey.ensure((size_t)K * 4));
        CU(ctx->flrow.ensure((size_t)K * 4));
        CU(ctx->flsig.ensure((size_t)K * 16));
        CU(ctx->tmp_rows.ensure((size_t)K * np));
    }
    // thermometer codes only when the ⊑ filter runs (the unfiltered mode accepts Wh > 32, where these would be
    // K x 2 Wh words); the check kernel writes them only with encode = filter_minimal (ensure() only grows)
    if (filter_minimal) CU(ctx->codes.ensure((size_t)ctx->pool_cap * 2 * std::max(ctx->Wh, 1) * 4));
    CU(ctx->hist.ensure((size_t)(ctx->Lh + 2) * 4));
    CU(ctx->level_start.ensure((size_t)(ctx->Lh + 2) * 4));
    CU(ctx->cursor.ensure((size_t)(ctx->Lh + 2) * 4));
    {
        const size_t nbins = (size_t)ctx->n * (ctx->Lh + 1);
        CU(ctx->ffreq.ensure((size_t)ctx->n * 4));
        CU(ctx->fbh.ensure(nbins * 4));
        CU(ctx->fbs.ensure((nbins + 1) * 4));
        CU(ctx->fbc.ensure(nbins * 4 + 4));   // + the undecided-row counter
        if (filter_minimal && resolved_filter_algo(ctx) == 3) {
            CU(ctx->fgc.ensure(nbins * 4));
            CU(ctx->fgs.ensure((nbins + 1) * 4));
            CU(ctx->fgr.ensure(std::min<size_t>((size_t)ctx->pool_cap * std::min(ctx->n, kGlEntriesPerRow), kGlMaxEntries) * 4));
            CU(ctx->fhf.ensure((size_t)ctx->n * 4 + 8 + (size_t)(ctx->Lh + 2) * 4));   // + barrier words, work counters
        }
    }
    CU(cudaMemsetAsync(ctx->keys.p, 0, ctx->table_slots * 8, ctx->stream));
    CU(cudaMemsetAsync(ctx->idx.p, 0xFF, (size_t)ctx->pool_cap * 8, ctx->stream));
    CU(cudaMemsetAsync(ctx->counters.p, 0, sizeof(unsigned long long) * C_N, ctx->stream));
    return MAPLE_OK;
}

HashSet hashset(maple_ctx* ctx) {
    return HashSet{ctx->keys.as<unsigned long long>(), ctx->idx.as<int64_t>(), ctx->table_slots - 1,
                   ctx->pool.as<int8_t>(), ctx->pool_cap, counters(ctx) + C_POOL,
                   reinterpret_cast<int*>(counters(ctx) + C_OVF), counters(ctx) + C_MAXC};
}

FilterWork make_filter_work(maple_ctx* ctx, int algo) {
    const int np = ctx->n_pad;
    FilterWork fw{ctx->n, np, ctx->Lh, std::max(ctx->Wh, 1), ctx->binary, ctx->th_off.as<int32_t>(), ctx->th_c0.as<int32_t>(),
                  ctx->th_c1.as<int32_t>(), ctx->codes.as<uint32_t>(), ctx->l1.as<int32_t>(), ctx->hist.as<int32_t>(),
                  ctx->level_start.as<int32_t>(), ctx->cursor.as<int32_t>(), ctx->order.as<int32_t>(),
                  ctx->keep.as<uint8_t>(), ctx->witness.as<int32_t>(), ctx->Lh, ctx->sig.as<uint4>(),
                  algo, 0, ctx->pool.as<int8_t>(), ctx->ffreq.as<int32_t>(),
                  ctx->fkey.as<int32_t>(), ctx->fbh.as<int32_t>(), ctx->fbs.as<int32_t>(), ctx->fbc.as<int32_t>(),
                  ctx->flrow.as<int32_t>(), ctx->flsig.as<uint4>(),
                  ctx->fbc.as<int32_t>() + (size_t)ctx->n * (ctx->Lh + 1), ctx->fgc.as<int32_t>(),
                  ctx->fgs.as<int32_t>(), ctx->fgr.as<int32_t>(), ctx->fhf.as<int32_t>(),
                  (int64_t)(ctx->fgr.bytes / 4), 0, 0, 0};
    // test hook: MAPLE_GL_CAP caps the G-list capacity so the level pass's fallback (the indexed pass) is exercised
    if (const char* cap = getenv("MAPLE_GL_CAP")) fw.gl_cap = std::min<int64_t>(fw.gl_cap, atoll(cap));
    return fw;
}

// the compacted rows in ctx->tmp_rows (count h[C_KEEP]) -> a new lexicographically sorted dirset
int sorted_set_from_compacted(maple_ctx* ctx, const unsigned long long* h, maple_dirset** out) {
    cudaStream_t s = ctx->stream;
    const int np = ctx->n_pad;
    int nl = 0;
    const int64_t M = (int64_t)h[C_KEEP];
    maple_dirset* ds = new maple_dirset();
    ds->ctx = ctx;
    ds->n = ctx->n;
    ds->n_pad = np;
    ds->size = M;
    ds->pool_size = (int64_t)h[C_POOL] - (int64_t)h[C_BAD];
    ds->n_bad = (int64_t)h[C_BAD];
    ds->D_nzmax = std::max(1, (int)h[C_NZMAX]);   // the most nonzeros of a row of the set (compact kernel)
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&ds->rows), std::max<int64_t>(M, 1) * np, s);
    if (e != cudaSuccess) {
        delete ds;
        CU(e);
    }
    CU(ctx->sortkeys.ensure(std::max<int64_t>(M, 1) * np));
    CU(ctx->sidx0.ensure(std::max<int64_t>(M, 1) * 4));
    CU(ctx->sidx1.ensure(std::max<int64_t>(M, 1) * 4));
    CU(launch_lex_sort(ctx->tmp_rows.as<int8_t>(), M, ctx->n, np, ctx->sortkeys.as<uint32_t>(), ctx->sidx0.as<int32_t>(),
                       ctx->sidx1.as<int32_t>(), ds->rows, s, &nl));
    ctx->launches += nl;
    CU(cudaEventRecord(ctx->ev[5], s));
    if (cudaEventCreateWithFlags(&ds->ready, cudaEventDisableTiming) == cudaSuccess) cudaEventRecord(ds->ready, s);
    *out = ds;
    return MAPLE_OK;
}

// check -> filter -> compact of the ctx pool (device count) -> ONE host sync -> lex sort into a new dirset.
// Returns MAPLE_OK, or RETRY (1) when a candidate / pool buffer overflowed (the caller grows and redoes).
constexpr int RETRY = 1;
int finish_set(maple_ctx* ctx, int filter_minimal, maple_dirset** out) {
    cudaStream_t s = ctx->stream;
    const int np = ctx->n_pad;
    const int64_t K = ctx->pool_cap;
    CU(cudaEventRecord(ctx->ev[2], s));
    CheckParams cp{ctx->m, ctx->n, np, ctx->A_rowptr.as<int32_t>(), ctx->A_col.as<int32_t>(), ctx->A_val.as<int32_t>(),
                   ctx->nnz, ctx->dbox.as<int32_t>()};
    if (filter_minimal && ctx->Wh > 32) FAIL(MAPLE_ERR_RANGE, "⊑ filter supports sum(u-l) <= 1024");
    FilterWork fw = make_filter_work(ctx, resolved_filter_algo(ctx));
    const unsigned long long* dpool = counters(ctx) + C_POOL;
    CU(launch_check_codes(ctx->pool.as<int8_t>(), dpool, K, cp, fw, filter_minimal, ctx->flags.as<uint8_t>(),
                          counters(ctx) + C_BAD, s));
    ctx->launches++;
    CU(cudaEventRecord(ctx->ev[3], s));
    int nl = 0;
    CU(launch_filter(dpool, K, ctx->flags.as<uint8_t>(), fw, filter_minimal, s, &nl));
    ctx->launches += nl;
    CU(launch_compact(ctx->pool.as<int8_t>(), ctx->keep.as<uint8_t>(), dpool, K, np, ctx->tmp_rows.as<int8_t>(),
                      counters(ctx) + C_KEEP, counters(ctx) + C_NZMAX, s));
    ctx->launches++;
    CU(cudaEventRecord(ctx->ev[4], s));
    unsigned long long h[C_N];
    int rc = read_counters(ctx, h);
    if (rc) return rc;
    if (h[C_RANGE]) {   // the CTA-pair kernel's f16 operands overflowed (|z| > 60000): redo this extraction on SIMT
        ctx->tcp_range_fail = true;
        return RETRY;
    }
    if (h[C_OVF] || (int64_t)h[C_MAXC] > ctx->cand_cap) {
        ctx->want_cand = std::max<int64_t>(ctx->cand_cap, (int64_t)h[C_MAXC] + ((int64_t)h[C_MAXC] >> 2) + 1024);
        ctx->want_pool = h[C_OVF] ? 2 * ctx->pool_cap : ctx->pool_cap;
        return RETRY;
    }
    int rc2 = sorted_set_from_compacted(ctx, h, out);
    if (rc2) return rc2;
    ctx->timings_pending = true;
    return MAPLE_OK;
}

__global__ void canonical_copy_kernel(const int8_t* __restrict__ rows, int64_t k, int stride, int n, int n_pad,
                                      int8_t* out) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < k; r += (int64_t)gridDim.x * blockDim.x) {
        const int8_t* g = rows + (size_t)r * stride;
        int sgn = 0;
        for (int i = 0; i < n && !sgn; ++i) sgn = g[i] > 0 ? 1 : (g[i] < 0 ? -1 : 0);
        if (!sgn) sgn = 1;
        int8_t* o = out + (size_t)r * n_pad;
        for (int i = 0; i < n_pad; ++i) o[i] = i < n ? (int8_t)(sgn * g[i]) : (int8_t)0;
    }
}

int insert_rows_and_finish(maple_ctx* ctx, const int8_t* drows, int64_t k, int stride, int filter_minimal,
                           maple_dirset** out) {
    cudaStream_t s = ctx->stream;
    for (int attempt = 0; attempt < 8; ++attempt) {
        int rc = prepare_set(ctx, std::max<int64_t>(k, 1), std::max<int64_t>({k, ctx->want_pool, 1}), filter_minimal);
        if (rc) return rc;
        CU(cudaEventRecord(ctx->ev[0], s));
        const unsigned long long kk = (unsigned long long)k;
        CU(cudaMemcpyAsync(counters(ctx) + C_CAND, &kk, sizeof(kk), cudaMemcpyHostToDevice, s));
        if (k > 0) {
            unsigned blocks = (unsigned)std::min<int64_t>((k + 255) / 256, 148 * 16);
            canonical_copy_kernel<<<blocks, 256, 0, s>>>(drows, k, stride, ctx->n, ctx->n_pad, ctx->cand.as<int8_t>());
            CU(cudaGetLastError());
            ctx->launches++;
        }
        CU(cudaEventRecord(ctx->ev[1], s));
        CU(launch_dedupe(ctx->cand.as<int8_t>(), counters(ctx) + C_CAND, ctx->cand_cap, ctx->n_pad, ctx->n_pad,
                         hashset(ctx), s));
        ctx->launches++;
        rc = finish_set(ctx, filter_minimal, out);
        if (rc != RETRY) return rc;
    }
    FAIL(MAPLE_ERR_CAPACITY, "device set capacity retries exhausted");
}

int build_step_table(maple_ctx* ctx, int T, double lr) {
    // per step t: (lr / (1 - beta1^t), sqrt(1 - beta2^t), 1 / sqrt(1 - beta2^t)) computed in fp64 (torch scalars);
    // rebuilt only when (T, lr, betas) change. The pinned upload is stream-ordered: the extraction's one
    // synchronisation follows it, so the staging buffer is free again when the next call rebuilds.
    if (T == ctx->tab_T && lr == ctx->tab_lr && ctx->beta1 == ctx->tab_b1 && ctx->beta2 == ctx->tab_b2) return MAPLE_OK;
    CU(ctx->stage_tab.reserve(sizeof(float4) * T));
    float4* tab = ctx->stage_tab.take<float4>(T);
    for (int t = 1; t <= T; ++t) {
        const double bc1 = 1.0 - std::pow(ctx->beta1, t);
        const double bc2s = std::sqrt(1.0 - std::pow(ctx->beta2, t));
        tab[t - 1] = make_float4((float)(lr / bc1), (float)bc2s, (float)(1.0 / bc2s), 0.f);
    }
    CU(ctx->step_tab.ensure(sizeof(float4) * T));
    CU(cudaMemcpyAsync(ctx->step_tab.p, tab, sizeof(float4) * T, cudaMemcpyHostToDevice, ctx->stream));
    ctx->tab_T = T;
    ctx->tab_lr = lr;
    ctx->tab_b1 = ctx->beta1;
    ctx->tab_b2 = ctx->beta2;
    return MAPLE_OK;
}

DescentParams descent_params(maple_ctx* ctx, int T, uint64_t seed, int64_t n_total, int64_t begin, int64_t count) {
    DescentParams p{};
    p.n = ctx->n;
    p.d = ctx->d;
    p.n_pad = ctx->n_pad;
    p.T = T;
    p.lam1 = (float)ctx->lam1;
    p.lam2 = (float)ctx->lam2;
    p.beta1 = (float)ctx->beta1;
    p.beta2 = (float)ctx->beta2;
    p.eps = (float)ctx->eps;
    p.omb1 = (float)(1.0 - ctx->beta1);
    p.omb2 = (float)(1.0 - ctx->beta2);
    p.step_tab = ctx->step_tab.as<float4>();
    p.seed = seed;
    p.n_total = n_total;
    p.begin = begin;
    p.count = count;
    p.B_nd = ctx->B_nd.as<float>();
    p.B_dn = ctx->B_dn.as<float>();
    p.B8_nd = ctx->B8.as<int8_t>();
    p.sb = ctx->sb;
    p.Bp = ctx->dBp.as<double>();
    p.lo = ctx->dl.as<int32_t>();
    p.hi = ctx->du.as<int32_t>();
    p.box = ctx->dbox.as<int32_t>();
    p.opt = ctx->optimizer;
    p.harvest_final = ctx->harvest_final;
    p.lr = (float)ctx->tab_lr;   // the step table was just built for this call's step size
    p.tcp_np = ctx->tcp_np;
    p.tcp_dp = ctx->tcp_dp;
    p.B16p = ctx->B16p.as<uint16_t>();
    p.BT8p = ctx->BT8p.as<int8_t>();
    p.B8p = ctx->B8p.as<int8_t>();
    p.range_flag = reinterpret_cast<int*>(counters(ctx) + C_RANGE);
    p.trace = ctx->trace_on ? ctx->trace.as<unsigned long long>() : nullptr;
    return p;
}

// Sparse B for the SIMT descent: lane-major, bank-scheduled ELL words (sparse_ell.h), uploaded on the
// context's allocation stream.
int build_sparse(maple_ctx* ctx) {
    const int n = ctx->n, d = ctx->d;
    {
        std::vector<std::vector<std::pair<int, int>>> rows(n), cols(d);
        int nnz = 0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < d; ++j) {
                const int v = (int)ctx->B[(size_t)i * d + j];
                if (!v) continue;
                rows[i].emplace_back(j, v);
                cols[j].emplace_back(i, v);
                ++nnz;
            }
        // forward lists longer than a quarter of a lane's share are split (the rows of a kernel basis are
        // uneven: C3's longest has 91 nonzeros against 38 per lane); columns stay whole (Adam ownership)
        if (std::max(n, d) > kEllMaxIndex) return MAPLE_ERR_RANGE;
        const int chunk = std::max(4, ((nnz + 31) / 32 + 3) / 4);
        // Storage in owner order: coordinate j of z (and of r = round(z)) lives at its backward place q*32 + L
        // (lane L owns it for Adam), row i of s = sign(Bz) (and of the harvested g) at its forward place; split
        // rows after the qf*32 places. Adam and the forward stores then touch contiguous, conflict-free words,
        // and a gather's bank is the owner lane of what it gathers. The lane assignment depends only on the
        // list lengths, so a first pass fixes the places and the second schedules the remapped gathers.
        const EllSchedule F0 = build_ell(rows, d, chunk);
        const EllSchedule B0 = build_ell(cols, n, 0);
        const int qf0 = std::max(F0.max_pieces, 1), qd0 = std::max(B0.max_pieces, 1);
        std::vector<int> pz(d, -1), ps(n, -1);
        for (size_t k = 0; k < B0.owned.size(); ++k)
            if (B0.owned[k] >= 0) pz[B0.owned[k]] = (int)k;
        for (size_t k = 0; k < F0.owned.size(); ++k)
            if (F0.owned[k] >= 0) ps[F0.owned[k]] = (int)k;
        for (size_t f3 = 0; f3 < F0.fixup.size(); f3 += 3) ps[F0.fixup[f3]] = qf0 * 32 + (int)(f3 / 3);
        auto remap = [](std::vector<std::vector<std::pair<int, int>>> L, const std::vector<int>& pos) {
            for (auto& l : L)
                for (auto& e : l) e.first = pos[e.first];
            return L;
        };
        const EllSchedule F = build_ell(remap(rows, pz), qd0 * 32, chunk);
        const EllSchedule Bk = build_ell(remap(cols, ps), qf0 * 32 + (int)F0.fixup.size() / 3, 0);
        if (F.owned != F0.owned || Bk.owned != B0.owned || F.fixup != F0.fixup) return MAPLE_ERR_RANGE;   // (cannot happen: the lane assignment depends on list lengths only)
        for (int i = 0; i < n; ++i)
            if (ps[i] < 0) return MAPLE_ERR_RANGE;   // (cannot happen: the lane assignment depends on list lengths only)
        for (int j = 0; j < d; ++j)
            if (pz[j] < 0) return MAPLE_ERR_RANGE;   // (cannot happen: the lane assignment depends on list lengths only)
        CU(upload(ctx->ell_pos_s, std::vector<int32_t>(ps.begin(), ps.end())));
        CU(upload(ctx->ell_pos_z, std::vector<int32_t>(pz.begin(), pz.end())));
        std::vector<int32_t> fix = F.fixup, fixpos = F.fixpos;
        if (fix.empty()) fix.push_back(0);
        if (fixpos.empty()) fixpos.push_back(0);
        CU(upload(ctx->ell_f, F.words));
        CU(upload(ctx->ell_own_f, F.owned));
        CU(upload(ctx->ell_fix, fix));
        CU(upload(ctx->ell_fixpos, fixpos));
        CU(upload(ctx->ell_b, Bk.words));
        CU(upload(ctx->ell_owned, Bk.owned));
        SparseB& sb = ctx->sb;
        sb.nnz = nnz;
        sb.Lf = F.slots;
        sb.qf = F.max_pieces;
        sb.nfix = (int)F.fixup.size() / 3;
        sb.nfixpos = (int)F.fixpos.size();
        sb.Lb = Bk.slots;
        sb.qd = Bk.max_pieces;
        sb.ell_f = ctx->ell_f.as<uint32_t>();
        sb.own_f = ctx->ell_own_f.as<int32_t>();
        sb.fix = ctx->ell_fix.as<int32_t>();
        sb.fixpos = ctx->ell_fixpos.as<int32_t>();
        sb.ell_b = ctx->ell_b.as<uint32_t>();
        sb.own_b = ctx->ell_owned.as<int32_t>();
        sb.pos_s = ctx->ell_pos_s.as<int32_t>();
        sb.pos_z = ctx->ell_pos_z.as<int32_t>();
        ctx->ell_conflicts = F.conflicts + Bk.conflicts;
    }
    // the staged copies must land before the staging buffer is reused (a lazy build runs inside an extraction)
    CU(cudaStreamSynchronize(g_alloc_stream));
    t_upload_stage.used = 0;
    ctx->sb_ready = true;
    return MAPLE_OK;
}

constexpr int kAutoTc = 2;   // auto choice for tensor-core shapes

// Padded operand copies for the CTA-pair kernel (k_descent_tcp.cu): B as IEEE half (exact small integers),
// tcp_np x tcp_dp, and B^T as int8, tcp_dp x tcp_np, zero padded; uploaded on the context's stream.
int build_tcp(maple_ctx* ctx) {
    const int n = ctx->n, d = ctx->d, np = ctx->tcp_np, dp = ctx->tcp_dp;
    std::vector<uint16_t> b16((size_t)np * dp, 0);
    std::vector<int8_t> bt8((size_t)dp * np, 0), b8((size_t)np * dp, 0);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < d; ++j) {
            const int v = (int)ctx->B[(size_t)i * d + j];
            b16[(size_t)i * dp + j] = __half_as_ushort(__float2half_rn((float)v));
            bt8[(size_t)j * np + i] = (int8_t)v;
            b8[(size_t)i * dp + j] = (int8_t)v;
        }
    CU(upload(ctx->B16p, b16));
    CU(upload(ctx->BT8p, bt8));
    CU(upload(ctx->B8p, b8));
    CU(cudaStreamSynchronize(g_alloc_stream));
    t_upload_stage.used = 0;
    ctx->tcp_ready = true;
    return MAPLE_OK;
}

// the CTA-pair kernel runs Adam with every-step harvest (the default variant) on the shapes it was instantiated for
bool tcp_ok(const maple_ctx* ctx) {
    // the harvest operand is round(z) as int8: exact for every in-box g when |B+ g|_inf <= rbound < 127
    return ctx->tcp_np > 0 && ctx->optimizer == 0 && ctx->harvest_final == 0 && !ctx->tcp_range_fail &&
           ctx->rbound < 127.0;
}

// the descent kernel an extraction launches: 1 SIMT, 2 tcgen05 (small shapes), 4 CTA-pair tcgen05 (large shapes)
int which_descent(const maple_ctx* ctx) {
    const bool tc_ok = descent_tc_supported(ctx->n, ctx->d) && ctx->rbound < 2047.0;
    if (ctx->descent_kernel == 4) return tcp_ok(ctx) ? 4 : 1;   // documented in maple.h: SIMT where tcp cannot run
    if (ctx->descent_kernel != 0) return ctx->descent_kernel;
    if (tc_ok) return kAutoTc;
    return tcp_ok(ctx) ? 4 : 1;
}

// build the schedules / operand copies of the kernel the next launch uses (once per context)
int ensure_descent_operands(maple_ctx* ctx) {
    const int w = which_descent(ctx);
    if (w == 1 && !ctx->sb_ready) return build_sparse(ctx);
    if (w == 4 && !ctx->tcp_ready) return build_tcp(ctx);
    return MAPLE_OK;
}

// The SIMT kernel computes z0 = B+ g0 per warp (fp64, a fixed-order reduction) — cheap for small n d, but at C5
// (n d = 900,000 fp64 FMAs per start) it is a quarter of the kernel. Above this size the starts of a launch are one
// cuBLAS DGEMM Z0 = G0 B+^T (a plain library GEMM on the fp64 tensor cores) in chunks, and the kernel reads them.
constexpr int64_t kGemmStartsMinND = 200000;
constexpr int64_t kGemmStartsChunk = 65536;

// cuBLAS is opened on first use (dlopen), so processes that never take this path (every shape but C5's) do not
// pay its module registration when they create their first context
struct CublasApi {
    bool tried = false, ok = false;
    cublasStatus_t (*create)(cublasHandle_t*) = nullptr;
    cublasStatus_t (*destroy)(cublasHandle_t) = nullptr;
    cublasStatus_t (*set_stream)(cublasHandle_t, cudaStream_t) = nullptr;
    cublasStatus_t (*dgemm)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int, const double*,
                            const double*, int, const double*, int, const double*, double*, int) = nullptr;
};
CublasApi& cublas_api() {
    static CublasApi api;
    if (!api.tried) {
        api.tried = true;
        void* h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("/usr/local/cuda/lib64/libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.create = reinterpret_cast<decltype(api.create)>(dlsym(h, "cublasCreate_v2"));
            api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(h, "cublasDestroy_v2"));
            api.set_stream = reinterpret_cast<decltype(api.set_stream)>(dlsym(h, "cublasSetStream_v2"));
            api.dgemm = reinterpret_cast<decltype(api.dgemm)>(dlsym(h, "cublasDgemm_v2"));
            api.ok = api.create && api.destroy && api.set_stream && api.dgemm;
        }
    }
    return api;
}

cudaError_t simt_with_gemm_starts(maple_ctx* ctx, const DescentParams& p) {
    cudaStream_t s = ctx->stream;
    CublasApi& cb = cublas_api();
    if (!cb.ok) return launch_descent_simt(p, s);   // no cuBLAS: the kernel computes its starts itself
    if (!ctx->cublas) {
        if (cb.create(&ctx->cublas) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
    }
    if (cb.set_stream(ctx->cublas, s) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
    const int n = ctx->n, d = ctx->d;
    const int64_t ch = std::min<int64_t>(p.count, kGemmStartsChunk);
    cudaError_t e;
    if ((e = ctx->g0buf.ensure((size_t)ch * n * 8)) != cudaSuccess) return e;
    if (!p.Z0_out && (e = ctx->z0buf.ensure((size_t)ch * d * 8)) != cudaSuccess) return e;
    const double one = 1.0, zero = 0.0;
    for (int64_t off = 0; off < p.count; off += ch) {
        DescentParams q = p;
        q.begin = p.begin + off;
        q.count = std::min(ch, p.count - off);
        if (p.Z_out) q.Z_out = p.Z_out + off * d;
        double* z0 = p.Z0_out ? p.Z0_out + off * d : ctx->z0buf.as<double>();
        if ((e = launch_start_g0(q, ctx->g0buf.as<double>(), s)) != cudaSuccess) return e;
        // column-major: Z0^T (d x cnt) = (B+ as n x d col-major)^T (G0^T: n x cnt col-major)
        if (cb.dgemm(ctx->cublas, CUBLAS_OP_T, CUBLAS_OP_N, d, (int)q.count, n, &one, p.Bp, n,
                     ctx->g0buf.as<double>(), n, &zero, z0, d) != CUBLAS_STATUS_SUCCESS)
            return cudaErrorUnknown;
        q.Z0_in = z0;
        q.Z0_out = nullptr;
        if ((e = launch_descent_simt(q, s)) != cudaSuccess) return e;
        ctx->launches += 2;
    }
    return cudaSuccess;
}

cudaError_t run_descent(maple_ctx* ctx, const DescentParams& p) {
    ctx->launches++;
    switch (which_descent(ctx)) {
        case 2: return launch_descent_tc(p, ctx->stream);
        case 4: return launch_descent_tcp(p, ctx->stream);
        default:
            if ((int64_t)ctx->n * ctx->d >= kGemmStartsMinND) return simt_with_gemm_starts(ctx, p);
            return launch_descent_simt(p, ctx->stream);
    }
}

int check_extract_args(maple_ctx* ctx, int64_t n_starts, int64_t begin, int64_t end, int32_t steps, double lr) {
    if (!ctx) return MAPLE_ERR_BAD_ARG;
    if (n_starts < 1) FAIL(MAPLE_ERR_BAD_ARG, "n_starts must be >= 1");
    if (steps < 1) FAIL(MAPLE_ERR_BAD_ARG, "steps must be >= 1");
    if (!(lr > 0.0) || !std::isfinite(lr)) FAIL(MAPLE_ERR_BAD_ARG, "step_size must be > 0");
    if (begin < 0 || end > n_starts || begin > end) FAIL(MAPLE_ERR_BAD_ARG, "bad start range");
    if (ctx->descent_kernel == 2 &&
        !(descent_tc_supported(ctx->n, ctx->d) && ctx->rbound < 2047.0))
        FAIL(MAPLE_ERR_RANGE, "tcgen05 descent kernel does not support this (n, d)");
    if (ctx->descent_kernel == 4 && ctx->tcp_np == 0)
        FAIL(MAPLE_ERR_RANGE, "CTA-pair tcgen05 descent kernel does not support this (n, d)");
    return MAPLE_OK;
}

}  // namespace

extern "C" {

int maple_create(const int32_t* A, int32_t m, int32_t n, const int32_t* l, const int32_t* u, int device,
                 maple_ctx** out) {
    maple_ctx* ctx = nullptr;
    if (!A || !l || !u || !out || m < 1 || n < 1) return MAPLE_ERR_BAD_ARG;
    *out = nullptr;
    for (int i = 0; i < n; ++i)
        if (l[i] > u[i]) return MAPLE_ERR_BAD_BOUNDS;
    if (m >= n) return MAPLE_ERR_FULL_RANK;
    if (n > MAPLE_MAX_N) return MAPLE_ERR_RANGE;
    for (int i = 0; i < n; ++i)
        if ((int64_t)u[i] - l[i] > 127) return MAPLE_ERR_RANGE;
    std::unique_ptr<maple_ctx> hold(new maple_ctx());
    ctx = hold.get();
    ctx->m = m;
    ctx->n = n;
    ctx->d = n - m;
    ctx->n_pad = round_up(std::max(n, 16), 16);
    ctx->A.assign(A, A + (size_t)m * n);
    ctx->l.assign(l, l + n);
    ctx->u.assign(u, u + n);
    ctx->box.resize(n);
    for (int i = 0; i < n; ++i) ctx->box[i] = u[i] - l[i];
    std::string err;
    int rc = host_kernel_basis(A, m, n, ctx->B, err);
    if (rc == 0) rc = host_lll(ctx->B, n, ctx->d, err);
    if (rc == 0) rc = host_pinv(ctx->B, n, ctx->d, ctx->Bp, err);
    if (rc) return rc;
    const int d = ctx->d;
    // exact re-verification of Thm. 1's A B = 0 and the int8 device range
    for (int r = 0; r < m; ++r)
        for (int j = 0; j < d; ++j) {
            __int128 s = 0;
            for (int i = 0; i < n; ++i) s += (__int128)A[(size_t)r * n + i] * ctx->B[(size_t)i * d + j];
            if (s != 0) return MAPLE_ERR_OVERFLOW;
        }
    for (int64_t v : ctx->B)
        if (v > 127 || v < -127) return MAPLE_ERR_RANGE;
    for (int j = 0; j < d; ++j) {
        double s = 0;
        for (int i = 0; i < n; ++i) s += std::fabs(ctx->Bp[(size_t)j * n + i]) * ctx->box[i];
        ctx->rbound = std::max(ctx->rbound, s);
    }
    if (cudaSetDevice(device) != cudaSuccess) return MAPLE_ERR_CUDA;
    ctx->device = device;
    g_alloc_stream = 0;
    if (t_upload_stage.used) {   // a previous create of this thread that failed early may still be copying
        cudaStreamSynchronize(0);
        t_upload_stage.used = 0;
    }
    {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    for (auto& e : ctx->ev)
        if (cudaEventCreate(&e) != cudaSuccess) return MAPLE_ERR_CUDA;
    // CSR of A
    std::vector<int32_t> rp(m + 1, 0), col, val;
    for (int r = 0; r < m; ++r) {
        for (int i = 0; i < n; ++i)
            if (A[(size_t)r * n + i]) {
                col.push_back(i);
                val.push_back(A[(size_t)r * n + i]);
            }
        rp[r + 1] = (int32_t)col.size();
    }
    ctx->nnz = (int)col.size();
    std::vector<int32_t> atp(n + 1, 0), atr, atv;  // CSC of A
    for (int i = 0; i < n; ++i) {
        for (int r = 0; r < m; ++r)
            if (A[(size_t)r * n + i]) {
                atr.push_back(r);
                atv.push_back(A[(size_t)r * n + i]);
            }
        atp[i + 1] = (int32_t)atr.size();
    }
    std::vector<float> bnd((size_t)n * d), bdn((size_t)d * n);
    std::vector<int8_t> b8((size_t)n * d);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < d; ++j) {
            const int64_t v = ctx->B[(size_t)i * d + j];
            bnd[(size_t)i * d + j] = (float)v;
            bdn[(size_t)j * n + i] = (float)v;
            b8[(size_t)i * d + j] = (int8_t)v;
        }
    // thermometer code map (filter): coordinate i owns bits [off_i, off_i + u_i - l_i) of each half
    std::vector<int32_t> toff(n);
    int lh = 0;
    for (int i = 0; i < n; ++i) {
        toff[i] = lh;
        lh += ctx->box[i];
    }
    ctx->Lh = lh;
    ctx->Wh = (ctx->Lh + 31) / 32;
    ctx->binary = 1;
    for (int i = 0; i < n; ++i) ctx->binary &= (ctx->box[i] == 1);
    std::vector<int32_t> wc0(std::max(ctx->Wh, 1), 0), wc1(std::max(ctx->Wh, 1), -1);
    for (int w = 0; w < ctx->Wh; ++w) {
        int c0 = -1, c1 = -1;
        for (int i = 0; i < n; ++i) {
            const int b0 = toff[i], b1 = toff[i] + ctx->box[i];
            if (b1 > 32 * w && b0 < 32 * (w + 1) && b1 > b0) {
                if (c0 < 0) c0 = i;
                c1 = i;
            }
        }
        wc0[w] = c0 < 0 ? 0 : c0;
        wc1[w] = c1;
    }
    CU(upload(ctx->A_rowptr, rp));
    CU(upload(ctx->A_col, col));
    CU(upload(ctx->A_val, val));
    CU(upload(ctx->AT_ptr, atp));
    CU(upload(ctx->AT_row, atr));
    CU(upload(ctx->AT_val, atv));
    CU(upload(ctx->dl, ctx->l));
    CU(upload(ctx->du, ctx->u));
    CU(upload(ctx->dbox, ctx->box));
    CU(upload(ctx->B_nd, bnd));
    CU(upload(ctx->B_dn, bdn));
    CU(upload(ctx->B8, b8));
    CU(upload(ctx->dBp, ctx->Bp));
    // the SIMT schedules are built now only when the SIMT kernel is the automatic choice; a tcgen05-shaped
    // context builds them on its first SIMT launch (maple_set_descent_kernel(1))
    tcp_shape(ctx->n, ctx->d, &ctx->tcp_np, &ctx->tcp_dp);
    {
        const int rc = ensure_descent_operands(ctx);
        if (rc) return rc;
    }
    CU(upload(ctx->th_off, toff));
    CU(upload(ctx->th_c0, wc0));
    CU(upload(ctx->th_c1, wc1));
    CU(ctx->counters.ensure(sizeof(unsigned long long) * C_N));
    CU(cudaMemset(ctx->counters.p, 0, sizeof(unsigned long long) * C_N));
    CU(cudaDeviceSynchronize());
    *out = hold.release();
    return MAPLE_OK;
}

int maple_kernel_basis(const int32_t* A, int32_t m, int32_t n, int32_t* B_out, double* Bp_out) {
    if (!A || !B_out || m < 1 || n < 1) return MAPLE_ERR_BAD_ARG;
    if (m >= n) return MAPLE_ERR_FULL_RANK;
    std::vector<int64_t> B;
    std::vector<double> Bp;
    std::string err;
    const int d = n - m;
    int rc = host_kernel_basis(A, m, n, B, err);
    if (rc == 0) rc = host_lll(B, n, d, err);
    if (rc == 0 && Bp_out) rc = host_pinv(B, n, d, Bp, err);
    if (rc) return rc;
    for (size_t i = 0; i < B.size(); ++i) {
        if (B[i] > INT32_MAX || B[i] < INT32_MIN) return MAPLE_ERR_OVERFLOW;
        B_out[i] = (int32_t)B[i];
    }
    if (Bp_out) std::memcpy(Bp_out, Bp.data(), Bp.size() * sizeof(double));
    return MAPLE_OK;
}

void maple_destroy(maple_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    g_alloc_stream = ctx->stream;
    DevBuf* bufs[] = {&ctx->trace, &ctx->B16p, &ctx->BT8p, &ctx->B8p, &ctx->A_rowptr, &ctx->A_col, &ctx->A_val, &ctx->dl, &ctx->du, &ctx->dbox, &ctx->B_nd,
                      &ctx->B_dn, &ctx->B8, &ctx->dBp, &ctx->th_off, &ctx->th_c0, &ctx->th_c1,
                      &ctx->ell_f, &ctx->ell_own_f, &ctx->ell_fix, &ctx->ell_fixpos, &ctx->ell_b, &ctx->ell_owned, &ctx->ell_pos_s, &ctx->ell_pos_z, &ctx->AT_ptr, &ctx->AT_row,
                      &ctx->AT_val, &ctx->fb, &ctx->frows, &ctx->fX, &ctx->step_tab, &ctx->cand,
                      &ctx->keys, &ctx->idx, &ctx->pool, &ctx->counters, &ctx->flags, &ctx->codes, &ctx->sig, &ctx->ffreq, &ctx->fkey, &ctx->fbh, &ctx->fbs, &ctx->fbc, &ctx->flrow, &ctx->flsig, &ctx->l1,
                      &ctx->fgc, &ctx->fgs, &ctx->fgr, &ctx->fhf, &ctx->g0buf, &ctx->z0buf,
                      &ctx->hist, &ctx->level_start, &ctx->cursor, &ctx->order, &ctx->keep, &ctx->witness,
                      &ctx->tmp_rows, &ctx->sortkeys, &ctx->sidx0, &ctx->sidx1, &ctx->zout, &ctx->z0out,
                      &ctx->aQ, &ctx->ac, &ctx->ac0, &ctx->aqg, &ctx->aX, &ctx->aF2, &ctx->aIt, &ctx->axb,
                      &ctx->af2b, &ctx->atab, &ctx->atoff};
    for (DevBuf* b : bufs) b->release();
    cudaStreamSynchronize(ctx->stream);
    ctx->stage_aug.release();
    ctx->stage_tab.release();
    if (ctx->cublas) cublas_api().destroy(ctx->cublas);
    for (auto& e : ctx->ev)
        if (e) cudaEventDestroy(e);
    delete ctx;
    g_alloc_stream = 0;   // the caller may destroy that stream next; later DevBuf users start from the legacy stream
}

int maple_set_stream(maple_ctx* ctx, void* stream) {
    if (!ctx) return MAPLE_ERR_BAD_ARG;
    cudaStreamSynchronize(ctx->stream);  // workspace allocated on the old stream is now safe to reuse
    ctx->stream = reinterpret_cast<cudaStream_t>(stream);
    return MAPLE_OK;
}

int maple_set_extract_params(maple_ctx* ctx, double lambda1, double lambda2, double beta1, double beta2, double eps,
                             int32_t filter_minimal) {
    if (!ctx) return MAPLE_ERR_BAD_ARG;
    if (!(lambda1 >= 0) || !(lambda2 >= 0) || !(beta1 >= 0 && beta1 < 1) || !(beta2 >= 0 && beta2 < 1) || !(eps > 0))
        FAIL(MAPLE_ERR_BAD_ARG, "bad extraction parameters");
    ctx->lam1 = lambda1;
    ctx->lam2 = lambda2;
    ctx->beta1 = beta1;
    ctx->beta2 = beta2;
    ctx->eps = eps;
    ctx->filter_minimal = filter_minimal ? 1 : 0;
    return MAPLE_OK;
}

int maple_selftest_umma(int device, const float* A1, const float* B1, float* D1, const float* A2, const float* B2,
                        float* D2) {
    maple_ctx* ctx = nullptr;
    if (!A1 || !B1 || !D1 || !A2 || !B2 || !D2) return MAPLE_ERR_BAD_ARG;
    CU(cudaSetDevice(device));
    g_alloc_stream = 0;
    const size_t sz[6] = {128 * 48, 64 * 48, 128 * 64, 128 * 64, 48 * 64, 128 * 48};
    DevBuf b[6];
    for (int i = 0; i < 6; ++i) CU(b[i].ensure(sz[i] * 4));
    CU(cudaMemcpy(b[0].p, A1, sz[0] * 4, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(b[1].p, B1, sz[1] * 4, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(b[3].p, A2, sz[3] * 4, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(b[4].p, B2, sz[4] * 4, cudaMemcpyHostToDevice));
    CU(umma_selftest(b[0].as<float>(), b[1].as<float>(), b[2].as<float>(), b[3].as<float>(), b[4].as<float>(),
                     b[5].as<float>(), 0));
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(D1, b[2].p, sz[2] * 4, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(D2, b[5].p, sz[5] * 4, cudaMemcpyDeviceToHost));
    for (auto& x : b) x.release();
    return MAPLE_OK;
}

int maple_selftest_pair(int device, const uint16_t* Ah, const uint16_t* Bh, const int8_t* A8, const int8_t* B8,
                        float* raw1, int32_t* raw2) {
    maple_ctx* ctx = nullptr;
    if (!Ah || !Bh || !A8 || !B8 || !raw1 || !raw2) return MAPLE_ERR_BAD_ARG;
    CU(cudaSetDevice(device));
    g_alloc_stream = 0;
    const size_t sz[6] = {128 * 32 * 2, 160 * 32 * 2, 128 * 64, 128 * 64, 2 * 128 * 80 * 4, 2 * 128 * 64 * 4};
    DevBuf b[6];
    for (int i = 0; i < 6; ++i) CU(b[i].ensure(sz[i]));
    CU(cudaMemcpy(b[0].p, Ah, sz[0], cudaMemcpyHostToDevice));
    CU(cudaMemcpy(b[1].p, Bh, sz[1], cudaMemcpyHostToDevice));
    CU(cudaMemcpy(b[2].p, A8, sz[2], cudaMemcpyHostToDevice));
    CU(cudaMemcpy(b[3].p, B8, sz[3], cudaMemcpyHostToDevice));
    CU(cudaMemset(b[4].p, 0xFF, sz[4]));
    CU(cudaMemset(b[5].p, 0xFF, sz[5]));
    CU(pair_selftest(b[0].p, b[1].p, b[2].p, b[3].p, b[4].as<float>(), b[5].as<int32_t>(), 0));
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(raw1, b[4].p, sz[4], cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(raw2, b[5].p, sz[5], cudaMemcpyDeviceToHost));
    for (auto& x : b) x.release();
    return MAPLE_OK;
}

int maple_set_descent_kernel(maple_ctx* ctx, int32_t which) {
    if (!ctx || which < 0 || which > 4 || which == 3) return MAPLE_ERR_BAD_ARG;
    ctx->descent_kernel = which;
    return MAPLE_OK;
}

int maple_set_descent_variant(maple_ctx* ctx, int32_t optimizer, int32_t harvest_final) {
    if (!ctx || optimizer < 0 || optimizer > 2 || harvest_final < 0 || harvest_final > 1) return MAPLE_ERR_BAD_ARG;
    ctx->optimizer = optimizer;
    ctx->harvest_final = harvest_final;
    return MAPLE_OK;
}

int maple_set_filter_algorithm(maple_ctx* ctx, int32_t which) {
    if (!ctx || which < 0 || which > 3) return MAPLE_ERR_BAD_ARG;
    ctx->filter_algo = which;
    return MAPLE_OK;
}

int maple_descent_kernel(const maple_ctx* ctx) {
    if (!ctx) return MAPLE_ERR_BAD_ARG;
    return which_descent(ctx);
}

int maple_debug_trace(maple_ctx* ctx, int32_t enable, uint64_t* host_out) {
    if (!ctx) return MAPLE_ERR_BAD_ARG;
    g_alloc_stream = ctx->stream;
    if (enable) {
        CU(ctx->trace.ensure(2 * 16 * 16 * 8));
        CU(cudaMemsetAsync(ctx->trace.p, 0, 2 * 16 * 16 * 8, ctx->stream));
    }
    ctx->trace_on = enable != 0;
    if (host_out && ctx->trace.p) {
        CU(cudaMemcpyAsync(host_out, ctx->trace.p, 2 * 16 * 16 * 8, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
    }
    return MAPLE_OK;
}

int maple_set_debug(maple_ctx* ctx, int32_t keep_candidates) {
    if (!ctx) return MAPLE_ERR_BAD_ARG;
    ctx->debug_keep = keep_candidates ? 1 : 0;
    return MAPLE_OK;
}

int maple_get_basis(const maple_ctx* ctx, int32_t* B_out) {
    if (!ctx || !B_out) return MAPLE_ERR_BAD_ARG;
    for (size_t i = 0; i < ctx->B.size(); ++i) B_out[i] = (int32_t)ctx->B[i];
    return MAPLE_OK;
}

int maple_get_pinv(const maple_ctx* ctx, double* Bp_out) {
    if (!ctx || !Bp_out) return MAPLE_ERR_BAD_ARG;
    std::memcpy(Bp_out, ctx->Bp.data(), ctx->Bp.size() * sizeof(double));
    return MAPLE_OK;
}

int32_t maple_dim_n(const maple_ctx* ctx) { return ctx ? ctx->n : -1; }
int32_t maple_dim_d(const maple_ctx* ctx) { return ctx ? ctx->d : -1; }
const char* maple_last_error(const maple_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }
int64_t maple_kernel_launches(const maple_ctx* ctx) { return ctx ? ctx->launches : -1; }

int maple_last_timings(const maple_ctx* ctx_c, float* e6, float* a3) {
    maple_ctx* ctx = const_cast<maple_ctx*>(ctx_c);
    if (!ctx) return MAPLE_ERR_BAD_ARG;
    if (ctx->timings_pending) {
        // events: 0 start, 1 descent done, 2 dedupe done, 3 check done, 4 filter + compact done, 5 sorted
        CU(cudaEventSynchronize(ctx->ev[5]));
        float t[5];
        cudaEventElapsedTime(&t[0], ctx->ev[0], ctx->ev[1]);
        cudaEventElapsedTime(&t[1], ctx->ev[1], ctx->ev[2]);
        cudaEventElapsedTime(&t[2], ctx->ev[2], ctx->ev[3]);
        cudaEventElapsedTime(&t[3], ctx->ev[3], ctx->ev[4]);
        cudaEventElapsedTime(&t[4], ctx->ev[4], ctx->ev[5]);
        for (int i = 0; i < 5; ++i) ctx->t_extract[i] = t[i];
        cudaEventElapsedTime(&ctx->t_extract[5], ctx->ev[0], ctx->ev[5]);
        ctx->timings_pending = false;
    }
    if (e6) std::memcpy(e6, ctx->t_extract, sizeof(ctx->t_extract));
    if (a3) std::memcpy(a3, ctx->t_augment, sizeof(ctx->t_augment));
    return MAPLE_OK;
}

int maple_extract_range(maple_ctx* ctx, int64_t n_starts, int64_t begin, int64_t end, int32_t steps,
                        double step_size, uint64_t seed, maple_dirset** out) {
    if (ctx) g_alloc_stream = ctx->stream;
    int rc = check_extract_args(ctx, n_starts, begin, end, steps, step_size);
    if (rc) return rc;
    if (!out) FAIL(MAPLE_ERR_BAD_ARG, "out is null");
    if (ctx->filter_minimal && ctx->Wh > 32) FAIL(MAPLE_ERR_RANGE, "⊑ filter supports sum(u-l) <= 1024");
    CU(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    rc = build_step_table(ctx, steps, step_size);
    if (rc) return rc;
    const int np = ctx->n_pad;
    const int64_t total = end - begin;
    const int64_t chunk_max = 1 << 18;
    const int64_t nchunks = std::max<int64_t>(1, (total + chunk_max - 1) / chunk_max);
    const int64_t per_chunk = std::min(total, chunk_max);
    // initial capacities (grown on overflow): ~32 candidate rows per start per chunk; the unique pool can
    // never exceed the candidates of one chunk times the number of chunks
    if (ctx->want_cand < per_chunk * 32) ctx->want_cand = std::max<int64_t>(per_chunk * 32, 4096);
    for (int attempt = 0; attempt < 8; ++attempt) {
        const int64_t pool_want = std::max<int64_t>(ctx->want_pool, std::max(ctx->want_cand, ctx->cand_cap) *
                                                                         std::min<int64_t>(nchunks, 4));
        rc = prepare_set(ctx, std::max(ctx->want_cand, ctx->cand_cap), pool_want, ctx->filter_minimal);
        if (rc) return rc;
        ctx->dbg_cand.clear();
        ctx->dbg_count = 0;
        CU(cudaEventRecord(ctx->ev[0], s));
        for (int64_t c0 = begin; c0 < end; c0 += chunk_max) {
            const int64_t cnt = std::min(chunk_max, end - c0);
            CU(cudaMemsetAsync(counters(ctx) + C_CAND, 0, 8, s));
            rc = ensure_descent_operands(ctx);
            if (rc) return rc;
            DescentParams p = descent_params(ctx, steps, seed, n_starts, c0, cnt);
            p.harvest = 1;
            p.cand = ctx->cand.as<int8_t>();
            p.cand_cap = ctx->cand_cap;
            p.cand_count = counters(ctx) + C_CAND;
            CU(run_descent(ctx, p));
            if (c0 + chunk_max >= end) CU(cudaEventRecord(ctx->ev[1], s));
            if (ctx->debug_keep) {
                unsigned long long h[C_N];
                rc = read_counters(ctx, h);
                if (rc) return rc;
                const int64_t nc = std::min<int64_t>((int64_t)h[C_CAND], ctx->cand_cap);
                const size_t off = ctx->dbg_cand.size();
                ctx->dbg_cand.resize(off + (size_t)nc * np);
                if (nc) CU(cudaMemcpy(ctx->dbg_cand.data() + off, ctx->cand.p, (size_t)nc * np, cudaMemcpyDeviceToHost));
                ctx->dbg_count += nc;
            }
            CU(launch_dedupe(ctx->cand.as<int8_t>(), counters(ctx) + C_CAND, ctx->cand_cap, np, np, hashset(ctx), s));
            ctx->launches++;
        }
        rc = finish_set(ctx, ctx->filter_minimal, out);
        if (rc != RETRY) return rc;
    }
    FAIL(MAPLE_ERR_CAPACITY, "device set capacity retries exhausted");
}

int maple_extract(maple_ctx* ctx, int64_t n_starts, int32_t steps, double step_size, uint64_t seed,
                  maple_dirset** out) {
    return maple_extract_range(ctx, n_starts, 0, n_starts, steps, step_size, seed, out);
}

int maple_dirset_merge(maple_ctx* ctx, const int8_t* rows, int64_t k, int32_t stride, maple_dirset** out) {
    if (ctx) g_alloc_stream = ctx->stream;
    if (!ctx || !out || k < 0 || (k > 0 && !rows) || stride < ctx->n) return MAPLE_ERR_BAD_ARG;
    if (ctx->filter_minimal && ctx->Wh > 32) FAIL(MAPLE_ERR_RANGE, "⊑ filter supports sum(u-l) <= 1024");
    CU(cudaSetDevice(ctx->device));
    return insert_rows_and_finish(ctx, rows, k, stride, ctx->filter_minimal, out);
}

int maple_set_filter_minimal(maple_ctx* ctx, int32_t on) {
    if (!ctx || on < 0 || on > 1) return MAPLE_ERR_BAD_ARG;
    ctx->filter_minimal = on;
    return MAPLE_OK;
}

namespace {
// the rows of `pool` (a set of this context: unique, canonical, exact) as the context's hash-set pool, count M
int load_pool(maple_ctx* ctx, const maple_dirset* pool, int filter_minimal) {
    const int64_t M = pool->size;
    int rc = prepare_set(ctx, 1, std::max<int64_t>(M, 1), filter_minimal);
    if (rc) return rc;
    const unsigned long long mm = (unsigned long long)M;
    CU(cudaMemcpyAsync(counters(ctx) + C_POOL, &mm, sizeof(mm), cudaMemcpyHostToDevice, ctx->stream));
    if (M > 0) CU(cudaMemcpyAsync(ctx->pool.p, pool->rows, (size_t)M * ctx->n_pad, cudaMemcpyDeviceToDevice, ctx->stream));
    return MAPLE_OK;
}
}  // namespace

int maple_dirset_keep_range(maple_ctx* ctx, const maple_dirset* pool, int64_t begin, int64_t end, uint8_t* keep_dev) {
    if (ctx) g_alloc_stream = ctx->stream;
    if (!ctx || !pool || pool->ctx != ctx || begin < 0 || end < begin || end > pool->size || (end > begin && !keep_dev))
        return MAPLE_ERR_BAD_ARG;
    if (ctx->Wh > 32) FAIL(MAPLE_ERR_RANGE, "⊑ filter supports sum(u-l) <= 1024");
    if (end == begin) return MAPLE_OK;
    CU(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    int rc = load_pool(ctx, pool, 1);
    if (rc) return rc;
    const int np = ctx->n_pad;
    const int64_t K = ctx->pool_cap;
    // pairwise against every pool row of smaller L1 (not only the minimal ones: those are decided on other shards)
    FilterWork fw = make_filter_work(ctx, ctx->n > 1024 ? 1 : 2);
    fw.g_begin = begin;
    fw.g_end = end;
    CheckParams cp{ctx->m, ctx->n, np, ctx->A_rowptr.as<int32_t>(), ctx->A_col.as<int32_t>(), ctx->A_val.as<int32_t>(),
                   ctx->nnz, ctx->dbox.as<int32_t>()};
    const unsigned long long* dpool = counters(ctx) + C_POOL;
    CU(launch_check_codes(ctx->pool.as<int8_t>(), dpool, K, cp, fw, 1, ctx->flags.as<uint8_t>(), counters(ctx) + C_BAD, s));
    int nl = 0;
    CU(launch_filter(dpool, K, ctx->flags.as<uint8_t>(), fw, 1, s, &nl));
    ctx->launches += 1 + nl;
    CU(cudaMemcpyAsync(keep_dev, ctx->keep.as<uint8_t>() + begin, (size_t)(end - begin), cudaMemcpyDeviceToDevice, s));
    CU(cudaStreamSynchronize(s));
    return MAPLE_OK;
}

int maple_dirset_select(maple_ctx* ctx, const maple_dirset* pool, const uint8_t* keep_dev, maple_dirset** out) {
    if (ctx) g_alloc_stream = ctx->stream;
    if (!ctx || !pool || pool->ctx != ctx || !out || (pool->size > 0 && !keep_dev)) return MAPLE_ERR_BAD_ARG;
    CU(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    int rc = load_pool(ctx, pool, 0);
    if (rc) return rc;
    const unsigned long long* dpool = counters(ctx) + C_POOL;
    CU(launch_compact(ctx->pool.as<int8_t>(), keep_dev, dpool, ctx->pool_cap, ctx->n_pad, ctx->tmp_rows.as<int8_t>(),
                      counters(ctx) + C_KEEP, counters(ctx) + C_NZMAX, s));
    ctx->launches++;
    unsigned long long h[C_N];
    rc = read_counters(ctx, h);
    if (rc) return rc;
    h[C_POOL] = (unsigned long long)pool->pool_size;   // the selected set reports the pool it came from
    h[C_BAD] = 0;
    rc = sorted_set_from_compacted(ctx, h, out);
    if (rc) return rc;
    CU(cudaStreamSynchronize(s));
    return MAPLE_OK;
}

int maple_dirset_from_host(maple_ctx* ctx, const int32_t* rows, int64_t k, int32_t filter_minimal,
                           maple_dirset** out) {
    if (ctx) g_alloc_stream = ctx->stream;
    if (!ctx || !out || k < 0 || (k > 0 && !rows)) return MAPLE_ERR_BAD_ARG;
    if (filter_minimal && ctx->Wh > 32) FAIL(MAPLE_ERR_RANGE, "⊑ filter supports sum(u-l) <= 1024");
    CU(cudaSetDevice(ctx->device));
    const int np = ctx->n_pad;
    std::vector<int8_t> h((size_t)std::max<int64_t>(k, 1) * np, 0);
    for (int64_t r = 0; r < k; ++r)
        for (int i = 0; i < ctx->n; ++i) {
            const int32_t v = rows[(size_t)r * ctx->n + i];
            if (v > 127 || v < -127) FAIL(MAPLE_ERR_RANGE, "row entry outside int8");
            h[(size_t)r * np + i] = (int8_t)v;
        }
    DevBuf tmp;   // stream-ordered on ctx->stream (g_alloc_stream), like the upload and the kernels that read it
    CU(tmp.ensure(h.size()));
    CU(cudaMemcpyAsync(tmp.p, h.data(), h.size(), cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));   // h is pageable and local
    int rc = insert_rows_and_finish(ctx, tmp.as<int8_t>(), k, np, filter_minimal ? 1 : 0, out);
    tmp.release();
    return rc;
}

int64_t maple_dirset_size(const maple_dirset* ds) { return ds ? ds->size : -1; }
int64_t maple_dirset_pool_size(const maple_dirset* ds) { return ds ? ds->pool_size : -1; }
int32_t maple_dirset_stride(const maple_dirset* ds) { return ds ? ds->n_pad : -1; }
const int8_t* maple_dirset_device_rows(const maple_dirset* ds) { return ds ? ds->rows : nullptr; }

int maple_dirset_copy(const maple_dirset* ds, int32_t* host_rows) {
    if (!ds || (!host_rows && ds->size > 0)) return MAPLE_ERR_BAD_ARG;
    if (ds->size == 0) return MAPLE_OK;
    maple_ctx* ctx = ds->ctx;
    std::vector<int8_t> h((size_t)ds->size * ds->n_pad);
    CU(cudaMemcpyAsync(h.data(), ds->rows, h.size(), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    for (int64_t r = 0; r < ds->size; ++r)
        for (int i = 0; i < ds->n; ++i) host_rows[(size_t)r * ds->n + i] = h[(size_t)r * ds->n_pad + i];
    return MAPLE_OK;
}

int maple_dirset_copy_i8(const maple_dirset* ds, int8_t* host_rows) {
    if (!ds || (!host_rows && ds->size > 0)) return MAPLE_ERR_BAD_ARG;
    if (ds->size == 0) return MAPLE_OK;
    maple_ctx* ctx = ds->ctx;
    CU(cudaMemcpy2DAsync(host_rows, (size_t)ds->n, ds->rows, (size_t)ds->n_pad, (size_t)ds->n, (size_t)ds->size,
                         cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return MAPLE_OK;
}

int maple_dirset_copy_raw(const maple_dirset* ds, int8_t* host_rows) {
    if (!ds || (!host_rows && ds->size > 0)) return MAPLE_ERR_BAD_ARG;
    if (ds->size == 0) return MAPLE_OK;
    maple_ctx* ctx = ds->ctx;
    CU(cudaMemcpyAsync(host_rows, ds->rows, (size_t)ds->size * ds->n_pad, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return MAPLE_OK;
}

int maple_dirset_copy_device(const maple_dirset* ds, int8_t* dst) {
    if (!ds || (!dst && ds->size > 0)) return MAPLE_ERR_BAD_ARG;
    if (ds->size == 0) return MAPLE_OK;
    maple_ctx* ctx = ds->ctx;
    CU(cudaMemcpyAsync(dst, ds->rows, (size_t)ds->size * ds->n_pad, cudaMemcpyDeviceToDevice, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return MAPLE_OK;
}

void maple_dirset_free(maple_dirset* ds) {
    if (!ds) return;
    // wait for the producing work (the set's own event; augmentation, which builds D, synchronises its stream
    // before returning), then frees back to the pool on the per-thread stream: idle, so the blocks are
    // reusable at once by the next stream-ordered allocation on any stream, and no legacy-stream barrier
    // against the context's stream is inserted
    if (ds->ready) {
        cudaEventSynchronize(ds->ready);
        cudaEventDestroy(ds->ready);
    }
    if (ds->rows) cudaFreeAsync(ds->rows, cudaStreamPerThread);
    if (ds->D) cudaFreeAsync(ds->D, cudaStreamPerThread);
    if (ds->D_nnz) cudaFreeAsync(ds->D_nnz, cudaStreamPerThread);
    if (ds->D_words) cudaFreeAsync(ds->D_words, cudaStreamPerThread);
    delete ds;
}

int64_t maple_debug_candidates(maple_ctx* ctx, int32_t* host_rows, int64_t cap) {
    if (!ctx) return MAPLE_ERR_BAD_ARG;
    if (host_rows) {
        const int64_t k = std::min(cap, ctx->dbg_count);
        for (int64_t r = 0; r < k; ++r)
            for (int i = 0; i < ctx->n; ++i)
                host_rows[(size_t)r * ctx->n + i] = ctx->dbg_cand[(size_t)r * ctx->n_pad + i];
    }
    return ctx->dbg_count;
}

int maple_debug_descent(maple_ctx* ctx, int64_t n_starts, int64_t begin, int64_t end, int32_t steps,
                        double step_size, uint64_t seed, float* Z_out, double* Z0_out) {
    if (ctx) g_alloc_stream = ctx->stream;
    int rc = check_extract_args(ctx, n_starts, begin, end, steps, step_size);
    if (rc) return rc;
    if (!Z_out) FAIL(MAPLE_ERR_BAD_ARG, "Z_out is null");
    CU(cudaSetDevice(ctx->device));
    rc = build_step_table(ctx, steps, step_size);
    if (rc) return rc;
    const int64_t cnt = end - begin;
    if (cnt == 0) return MAPLE_OK;
    CU(ctx->zout.ensure((size_t)cnt * ctx->d * sizeof(float)));
    CU(ctx->z0out.ensure((size_t)cnt * ctx->d * sizeof(double)));
    rc = ensure_descent_operands(ctx);
    if (rc) return rc;
    DescentParams p = descent_params(ctx, steps, seed, n_starts, begin, cnt);
    p.harvest = 0;
    p.Z_out = ctx->zout.as<float>();
    p.Z0_out = ctx->z0out.as<double>();
    CU(run_descent(ctx, p));
    CU(cudaMemcpyAsync(Z_out, ctx->zout.p, (size_t)cnt * ctx->d * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
    if (Z0_out)
        CU(cudaMemcpyAsync(Z0_out, ctx->z0out.p, (size_t)cnt * ctx->d * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return MAPLE_OK;
}

static int augment_impl(maple_ctx* ctx, const maple_dirset* ds, int32_t n_inst, const maple_objective* f,
                        const int32_t* b, const int32_t* x0, int32_t k0, int32_t* x_best, double* f_best,
                        int32_t* iters) {
    if (ctx) g_alloc_stream = ctx->stream;
    const int n = ctx->n, m = ctx->m, np = ctx->n_pad;
    cudaStream_t s = ctx->stream;
    // exact feasibility of every incumbent
    for (int t = 0; t < n_inst; ++t)
        for (int k = 0; k < k0; ++k) {
            const int32_t* x = x0 + ((size_t)t * k0 + k) * n;
            for (int i = 0; i < n; ++i)
                if (x[i] < ctx->l[i] || x[i] > ctx->u[i]) FAIL(MAPLE_ERR_INFEASIBLE, "x0 outside [l, u]");
            for (int r = 0; r < m; ++r) {
                int64_t acc = 0;
                for (int i = 0; i < n; ++i) acc += (int64_t)ctx->A[(size_t)r * n + i] * x[i];
                if (acc != b[(size_t)t * m + r]) FAIL(MAPLE_ERR_INFEASIBLE, "x0 violates A x = b");
            }
        }
    const bool table = n_inst > 0 && f[0].kind == MAPLE_OBJ_TABLE;
    for (int t = 0; t < n_inst; ++t) {
        if (!f[t].Q || (f[t].kind != MAPLE_OBJ_QUADRATIC && f[t].kind != MAPLE_OBJ_SEPARABLE &&
                        f[t].kind != MAPLE_OBJ_TABLE))
            FAIL(MAPLE_ERR_BAD_ARG, "bad objective");
        if ((f[t].kind == MAPLE_OBJ_TABLE) != table) FAIL(MAPLE_ERR_BAD_ARG, "mixed objective kinds in one batch");
        if (!table && !f[t].c) FAIL(MAPLE_ERR_BAD_ARG, "bad objective");
    }
    // separable value tables (MAPLE_OBJ_TABLE): coordinate j's table starts at sum_{i<j} (u_i - l_i + 1)
    std::vector<int32_t> toff(n);
    int64_t tab_len = 0;
    for (int i = 0; i < n && table; ++i) {
        toff[i] = (int32_t)tab_len;
        tab_len += (int64_t)ctx->u[i] - ctx->l[i] + 1;
        if (tab_len > (int64_t(1) << 27)) FAIL(MAPLE_ERR_BAD_ARG, "value table longer than 2^27 entries");
    }
    CU(cudaEventRecord(ctx->ev[8], s));
    maple_dirset* dsm = const_cast<maple_dirset*>(ds);
    const int64_t K = ds->size;
    if (!dsm->D && K > 0) {
        // D = S ∪ -S in lexicographic order (the tie-break order of Alg. 2, reading #17) by a merge of the sorted
        // set with its reversed negation, then its ELL form; stream-ordered, no host synchronisation
        CU(cudaMallocAsync(reinterpret_cast<void**>(&dsm->D), (size_t)2 * K * np, s));
        CU(launch_signed_merge(ds->rows, K, n, np, dsm->D, s));
        ctx->launches++;
        const int w = dsm->D_nzmax;
        CU(cudaMallocAsync(reinterpret_cast<void**>(&dsm->D_nnz), (size_t)2 * K * sizeof(int32_t), s));
        CU(cudaMallocAsync(reinterpret_cast<void**>(&dsm->D_words), (size_t)2 * K * w * sizeof(uint32_t), s));
        CU(launch_augment_ell(dsm->D, (int)(2 * K), n, np, w, dsm->D_nnz, dsm->D_words, s));
        ctx->launches++;
    }
    // objective data (dense Q per instance), staged in pinned memory
    const int64_t ninc = (int64_t)n_inst * k0;
    const size_t nQ = table ? (size_t)n_inst * tab_len : (size_t)n_inst * n * n, nc = (size_t)n_inst * n;
    CU(ctx->stage_aug.reserve(nQ * 8 + nc * 8 + (size_t)n_inst * 8 + (size_t)ninc * n * 4 + (size_t)n * 4 + 128));
    double* Q = ctx->stage_aug.take<double>(nQ);
    double* c = ctx->stage_aug.take<double>(nc);
    double* c0 = ctx->stage_aug.take<double>(n_inst);
    int32_t* X0 = ctx->stage_aug.take<int32_t>((size_t)ninc * n);
    if (!table) std::memset(Q, 0, nQ * 8);
    std::memcpy(X0, x0, (size_t)ninc * n * 4);
    for (int t = 0; t < n_inst; ++t) {
        if (table) {   // the tables as given; c unused
            std::memcpy(Q + (size_t)t * tab_len, f[t].Q, sizeof(double) * tab_len);
            c0[t] = f[t].c0;
            continue;
        }
        double* Qt = Q + (size_t)t * n * n;
        if (f[t].kind == MAPLE_OBJ_QUADRATIC) {
            // the kernels use grad = Q x + c, which is the gradient of 1/2 x^T Q x only for symmetric Q:
            // use the symmetric part (same objective values, exact in fp64 for integer data)
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j)
                    Qt[(size_t)i * n + j] = 0.5 * (f[t].Q[(size_t)i * n + j] + f[t].Q[(size_t)j * n + i]);
        } else
            for (int i = 0; i < n; ++i) Qt[(size_t)i * n + i] = f[t].Q[i];
        std::memcpy(c + (size_t)t * n, f[t].c, sizeof(double) * n);
        c0[t] = f[t].c0;
    }
    CU(ctx->aQ.ensure(nQ * 8));
    CU(ctx->ac.ensure(nc * 8));
    CU(ctx->ac0.ensure((size_t)n_inst * 8));
    CU(ctx->aqg.ensure((size_t)std::max<int64_t>(2 * K, 1) * n_inst * 8));
    CU(ctx->aX.ensure((size_t)ninc * n * 4));
    CU(ctx->aF2.ensure((size_t)ninc * 8));
    CU(ctx->aIt.ensure((size_t)ninc * 4));
    CU(ctx->axb.ensure((size_t)n_inst * n * 4));
    CU(ctx->af2b.ensure((size_t)n_inst * 8));
    CU(cudaMemcpyAsync(ctx->aQ.p, Q, nQ * 8, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(ctx->ac.p, c, nc * 8, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(ctx->ac0.p, c0, (size_t)n_inst * 8, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(ctx->aX.p, X0, (size_t)ninc * n * 4, cudaMemcpyHostToDevice, s));
    if (table) {
        int32_t* toff_h = ctx->stage_aug.take<int32_t>(n);
        std::memcpy(toff_h, toff.data(), (size_t)n * 4);
        CU(ctx->atoff.ensure((size_t)n * 4));
        CU(cudaMemcpyAsync(ctx->atoff.p, toff_h, (size_t)n * 4, cudaMemcpyHostToDevice, s));
    }
    AugmentParams p{};
    p.n = n;
    p.m = m;
    p.n_pad = np;
    p.n_dir = (int)K;
    p.dirs = dsm->D;
    p.nnz = dsm->D_nnz;
    p.words = dsm->D_words;
    p.nzmax = dsm->D_nzmax;
    p.Q = ctx->aQ.as<double>();
    p.c = ctx->ac.as<double>();
    p.c0 = ctx->ac0.as<double>();
    p.qg = ctx->aqg.as<double>();
    p.lo = ctx->dl.as<int32_t>();
    p.hi = ctx->du.as<int32_t>();
    p.X = ctx->aX.as<int32_t>();
    p.k0 = k0;
    p.n_inst = n_inst;
    p.F2 = ctx->aF2.as<double>();
    p.iters = ctx->aIt.as<int32_t>();
    p.max_iter = 1 << 20;
    p.table = table ? 1 : 0;
    p.tab = ctx->aQ.as<double>();   // TABLE: the staged value tables
    p.tab_off = ctx->atoff.as<int32_t>();
    p.tab_len = tab_len;
    CU(launch_augment_qg(p, s));
    if (!table) ctx->launches++;
    CU(cudaEventRecord(ctx->ev[9], s));
    CU(launch_augment(p, s));
    CU(launch_augment_best(p, ctx->axb.as<int32_t>(), ctx->af2b.as<double>(), s));
    ctx->launches += 2;
    CU(cudaEventRecord(ctx->ev[10], s));
    std::vector<double> f2(n_inst);
    CU(cudaMemcpyAsync(x_best, ctx->axb.p, (size_t)n_inst * n * 4, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(f2.data(), ctx->af2b.p, (size_t)n_inst * 8, cudaMemcpyDeviceToHost, s));
    if (iters) CU(cudaMemcpyAsync(iters, ctx->aIt.p, (size_t)ninc * 4, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    for (int t = 0; t < n_inst; ++t) f_best[t] = f2[t] / 2.0;
    float t;
    cudaEventElapsedTime(&t, ctx->ev[8], ctx->ev[9]);
    ctx->t_augment[0] = t;
    cudaEventElapsedTime(&t, ctx->ev[9], ctx->ev[10]);
    ctx->t_augment[1] = t;
    cudaEventElapsedTime(&t, ctx->ev[8], ctx->ev[10]);
    ctx->t_augment[2] = t;
    return MAPLE_OK;
}

int maple_feasible_starts(maple_ctx* ctx, const int32_t* b, int32_t k, int32_t steps, double step_size,
                          double lambda3, uint64_t seed, int32_t* x_out, int32_t cap, int32_t* count, float* X_debug) {
    if (ctx) g_alloc_stream = ctx->stream;
    if (!ctx || !b || !count || k < 1 || steps < 1 || !(step_size > 0) || !(lambda3 >= 0) || cap < 0 ||
        (cap > 0 && !x_out))
        return MAPLE_ERR_BAD_ARG;
    CU(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const int n = ctx->n, m = ctx->m, np = ctx->n_pad;
    int rc = build_step_table(ctx, steps, step_size);
    if (rc) return rc;
    CU(ctx->fb.ensure((size_t)m * 4));
    CU(cudaMemcpyAsync(ctx->fb.p, b, (size_t)m * 4, cudaMemcpyHostToDevice, s));
    CU(ctx->frows.ensure((size_t)k * np));
    if (X_debug) CU(ctx->fX.ensure((size_t)k * n * 4));
    rc = prepare_set(ctx, std::max<int64_t>(ctx->cand_cap, k), std::max<int64_t>(ctx->pool_cap, k), 0);
    if (rc) return rc;
    FeasibleParams p{};
    p.n = n;
    p.m = m;
    p.n_pad = np;
    p.T = steps;
    p.k = k;
    p.lam3 = (float)lambda3;
    p.beta1 = (float)ctx->beta1;
    p.beta2 = (float)ctx->beta2;
    p.eps = (float)ctx->eps;
    p.omb1 = (float)(1.0 - ctx->beta1);
    p.omb2 = (float)(1.0 - ctx->beta2);
    p.step_tab = ctx->step_tab.as<float4>();
    p.seed = seed;
    p.nnz = ctx->nnz;
    p.A_rowptr = ctx->A_rowptr.as<int32_t>();
    p.A_col = ctx->A_col.as<int32_t>();
    p.A_val = ctx->A_val.as<int32_t>();
    p.AT_colptr = ctx->AT_ptr.as<int32_t>();
    p.AT_row = ctx->AT_row.as<int32_t>();
    p.AT_val = ctx->AT_val.as<int32_t>();
    p.b = ctx->fb.as<int32_t>();
    p.lo = ctx->dl.as<int32_t>();
    p.hi = ctx->du.as<int32_t>();
    p.rows = ctx->frows.as<int8_t>();
    p.cap = k;
    p.count = counters(ctx) + C_CAND;
    p.X_out = X_debug ? ctx->fX.as<float>() : nullptr;
    CU(launch_feasible(p, s));
    ctx->launches++;
    CU(launch_dedupe(ctx->frows.as<int8_t>(), counters(ctx) + C_CAND, k, np, np, hashset(ctx), s));
    ctx->launches++;
    unsigned long long h[C_N];
    rc = read_counters(ctx, h);
    if (rc) return rc;
    const int64_t U = (int64_t)h[C_POOL];
    CU(ctx->tmp_rows.ensure((size_t)std::max<int64_t>(U, 1) * np));
    CU(ctx->sortkeys.ensure((size_t)std::max<int64_t>(U, 1) * np));
    CU(ctx->sidx0.ensure((size_t)std::max<int64_t>(U, 1) * 4));
    CU(ctx->sidx1.ensure((size_t)std::max<int64_t>(U, 1) * 4));
    int nl = 0;
    CU(launch_lex_sort(ctx->pool.as<int8_t>(), U, n, np, ctx->sortkeys.as<uint32_t>(), ctx->sidx0.as<int32_t>(),
                       ctx->sidx1.as<int32_t>(), ctx->tmp_rows.as<int8_t>(), s, &nl));
    ctx->launches += nl;
    std::vector<int8_t> hrows((size_t)std::max<int64_t>(U, 1) * np);
    if (U) CU(cudaMemcpyAsync(hrows.data(), ctx->tmp_rows.p, (size_t)U * np, cudaMemcpyDeviceToHost, s));
    if (X_debug) CU(cudaMemcpyAsync(X_debug, ctx->fX.p, (size_t)k * n * 4, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    const int64_t w = std::min<int64_t>(U, cap);
    for (int64_t r = 0; r < w; ++r)
        for (int i = 0; i < n; ++i) x_out[(size_t)r * n + i] = ctx->l[i] + (int32_t)hrows[(size_t)r * np + i];
    *count = (int32_t)U;
    return MAPLE_OK;
}

int maple_augment(maple_ctx* ctx, const maple_dirset* ds, const maple_objective* f, const int32_t* b,
                  const int32_t* x0, int32_t k0, int32_t* x_best, double* f_best, int32_t* status, int32_t* iters) {
    if (!ctx || !ds || !f || !b || !x_best || !f_best || !status || k0 < 0 || (k0 > 0 && !x0))
        return MAPLE_ERR_BAD_ARG;
    if (ds->n != ctx->n) FAIL(MAPLE_ERR_BAD_ARG, "direction set belongs to another n");
    CU(cudaSetDevice(ctx->device));
    if (k0 == 0) {
        *status = MAPLE_STATUS_NO_FEASIBLE;
        return MAPLE_OK;
    }
    *status = MAPLE_STATUS_OK;
    return augment_impl(ctx, ds, 1, f, b, x0, k0, x_best, f_best, iters);
}

int maple_augment_many(maple_ctx* ctx, const maple_dirset* ds, int32_t n_inst, const maple_objective* f,
                       const int32_t* b, const int32_t* x0, int32_t k0, int32_t* x_best, double* f_best) {
    if (!ctx || !ds || !f || !b || !x0 || !x_best || !f_best || n_inst < 1 || k0 < 1) return MAPLE_ERR_BAD_ARG;
    if (ds->n != ctx->n) FAIL(MAPLE_ERR_BAD_ARG, "direction set belongs to another n");
    CU(cudaSetDevice(ctx->device));
    return augment_impl(ctx, ds, n_inst, f, b, x0, k0, x_best, f_best, nullptr);
}

}  // extern "C"
