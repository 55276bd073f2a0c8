/*
 * maple.h — C ABI of the B200-native MAPLE hot path (arXiv 2412.13576, "GPU-based Graver Basis
 * Extraction for Nonlinear Integer Optimization").
 *
 * Problem (model (1)):  min f(x)  s.t.  A x = b,  l <= x <= u,  x in Z^n,
 * with A in Z^{m x n} of full row rank m < n. A, l, u are shared by every call on a context; f and b vary
 * per augmentation call (the paper's "flexibility").
 *
 * Conventions (all entry points):
 *  - Return value: 0 (MAPLE_OK) or a negative MAPLE_ERR_* code; no C++ exception crosses the ABI.
 *    maple_last_error(ctx) then holds a one-line human-readable reason.
 *  - Pointers documented "host" are ordinary host memory; "device" are CUDA device pointers on the
 *    context's device. Every input is copied (the caller may free it on return) unless stated.
 *  - Matrices are dense row-major int32 / float64 unless stated. Sizes are element counts.
 *  - Work is enqueued on the context's stream (maple_set_stream; default: the legacy default stream) and
 *    every call that returns host data synchronises that stream before returning.
 *  - A context is not thread-safe; distinct contexts are independent. One context = one device.
 *  - Determinism: for a fixed (A, l, u, parameters, seed) every result is bit-identical across runs and
 *    across any partition of the starts into ranges (maple_extract_range), i.e. across 1..8 GPUs.
 */
#ifndef MAPLE_H
#define MAPLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---------------------------------------------------------------------------- */
#define MAPLE_OK                   0
#define MAPLE_ERR_BAD_ARG         -1   /* null pointer, bad size, lambda < 0, N < 1, T < 1, lr <= 0 ... */
#define MAPLE_ERR_BAD_BOUNDS      -2   /* some l_i > u_i (SPEC S:243 BadBounds) */
#define MAPLE_ERR_RANK_DEFICIENT  -3   /* rank(A) < m */
#define MAPLE_ERR_FULL_RANK       -4   /* m >= n: Ker_Z(A) = {0} */
#define MAPLE_ERR_OVERFLOW        -5   /* exact host integer arithmetic (checked __int128) overflowed */
#define MAPLE_ERR_RANGE           -6   /* a value does not fit the device encoding (|B_ij| > 127,
                                          max(u-l) > 127, n > MAPLE_MAX_N, ...) */
#define MAPLE_ERR_CUDA            -7   /* a CUDA runtime call or kernel failed */
#define MAPLE_ERR_OOM             -8   /* device allocation failed */
#define MAPLE_ERR_CAPACITY        -9   /* a device set outgrew its hard cap */
#define MAPLE_ERR_INFEASIBLE     -10   /* an x0 row violates A x = b or l <= x <= u */
#define MAPLE_ERR_COMM           -11   /* reserved for the multi-GPU merge (collectives run in the caller) */

/* augmentation status (not an error) */
#define MAPLE_STATUS_OK            0
#define MAPLE_STATUS_NO_FEASIBLE   1   /* k0 == 0: no incumbent to augment */

/* objective kinds for maple_objective.kind */
#define MAPLE_OBJ_QUADRATIC        0   /* f(x) = 1/2 x^T Q x + c^T x + c0, Q dense n x n */
#define MAPLE_OBJ_SEPARABLE        1   /* same with Q diagonal: Q points to the n diagonal entries */
/* Separable f(x) = c0 + sum_j f_j(x_j) with ANY real f_j (Prop. 3: G(A) is a test set when every
 * f_j is convex), given by its values on the integer box: Q points to sum_j (u_j - l_j + 1) doubles, the
 * table of coordinate j starting at offset sum_{i<j} (u_i - l_i + 1), entry k = f_j(l_j + k); c is ignored
 * (may be NULL). Scores are f(x + lambda g) - f(x) = sum over the support of g, ascending j, of
 * f_j(x_j + lambda g_j) - f_j(x_j) in fp64 (exact for integer tables below 2^53). The box must hold at most
 * 2^27 table entries. Cannot be mixed with the quadratic kinds in one maple_augment_many batch (BAD_ARG). */
#define MAPLE_OBJ_TABLE            2

#define MAPLE_MAX_N             1024   /* device row encoding limit on n */

typedef struct maple_ctx maple_ctx;
typedef struct maple_dirset maple_dirset;

typedef struct maple_objective {
    int32_t kind;          /* MAPLE_OBJ_QUADRATIC, MAPLE_OBJ_SEPARABLE or MAPLE_OBJ_TABLE */
    const double* Q;       /* host; n*n row-major (QUADRATIC, symmetrised), n (SEPARABLE) or the value table
                              (TABLE, sum_j (u_j - l_j + 1) entries) */
    const double* c;       /* host; n (ignored for TABLE) */
    double c0;
} maple_objective;

/* ---- context ------------------------------------------------------------------------------------
 * maple_create — Alg. 3 lines 2-3 and the Remark on B^{-1}, run once per A:
 *   HNF  A C = (H | 0) with C unimodular (Prop. 1) in checked __int128 arithmetic;
 *   B = C[:, m:] (Thm. 1: Ker_Z(A) = L(B));  B <- LLL(B) with the paper's Siegel condition
 *   ||B*_{k-1}||^2 <= 2 ||B*_k||^2 (Def. P:136-144, Alg. 1);  B+ = (B^T B)^{-1} B^T in fp64;
 *   A B = 0 re-verified exactly; then A, B (int8 + fp32 copies), B+ and the box M = [l-u, u-l]
 *    are uploaded to `device`.
 * A: host int32 m*n row-major.  l, u: host int32 n.  device: CUDA ordinal.  out: receives the context,
 * owned by the library until maple_destroy.
 * Errors: BAD_ARG, BAD_BOUNDS, RANK_DEFICIENT, FULL_RANK, OVERFLOW, RANGE, CUDA, OOM.              */
int maple_create(const int32_t* A, int32_t m, int32_t n, const int32_t* l, const int32_t* u, int device,
                 maple_ctx** out);
void maple_destroy(maple_ctx* ctx);

/* Host-only part of maple_create (no device needed): the reduced kernel basis B (host int32 n x d
 * row-major, d = n - m) and, if Bp_out != NULL, B+ (host fp64 d x n) exactly as maple_create computes
 * them. Errors as maple_create minus CUDA/OOM. */
int maple_kernel_basis(const int32_t* A, int32_t m, int32_t n, int32_t* B_out, double* Bp_out);

/* Enqueue all further work on `stream` (a cudaStream_t, e.g. torch.cuda.current_stream().cuda_stream). */
int maple_set_stream(maple_ctx* ctx, void* stream);

/* Eq. 3 weights and Adam moments (reading #9): defaults lambda1 = 0.85, lambda2 = 1,
 * beta1 = 0.9, beta2 = 0.999, eps = 1e-8. filter_minimal = 1 (north star: keep only ⊑-minimal rows,
 * condition C4 P:283) or 0 (the paper's unfiltered pool). Errors: BAD_ARG (negative lambda,
 * beta outside [0,1), eps <= 0). */
int maple_set_extract_params(maple_ctx* ctx, double lambda1, double lambda2, double beta1, double beta2,
                             double eps, int32_t filter_minimal);

/* Copy the context's reduced kernel basis B (n x d, d = n - m, row-major) to host int32 `B_out`
 * (n*d elements). B is not unique; this is the one every extraction on ctx uses. */
int maple_get_basis(const maple_ctx* ctx, int32_t* B_out);
/* Copy B+ (d x n, row-major fp64) to host. */
int maple_get_pinv(const maple_ctx* ctx, double* Bp_out);
int32_t maple_dim_n(const maple_ctx* ctx);
int32_t maple_dim_d(const maple_ctx* ctx);
const char* maple_last_error(const maple_ctx* ctx);

/* ---- extraction ---------------------------------------------------------------------------------
 * maple_extract — Algorithm 3 plus the north-star post-processing, all on the device:
 *   starts i = 0..n_starts-1: g0 ~ U(l-u, u-l) from a splitmix64 counter keyed by (seed, i, j), z0 = B+ g0
 *   (P:386); `steps` Adam steps (lr = step_size) on Eq. 3; after every step the
 *   rounded iterate g = B round(z) (half away from zero) is harvested if g != 0 and g in M;
 *   then the exact check A g = 0 (C1-C3), dedupe with sign twins collapsed (first nonzero > 0),
 *   the ⊑-minimality filter (Def. 1-2; unless filter_minimal = 0) and a lexicographic sort.
 * out: receives a direction set owned by the library until maple_dirset_free.
 * Errors: BAD_ARG (n_starts < 1, steps < 1, step_size <= 0), CAPACITY, CUDA, OOM.                    */
int maple_extract(maple_ctx* ctx, int64_t n_starts, int32_t steps, double step_size, uint64_t seed,
                  maple_dirset** out);

/* Same computation restricted to global start indices [begin, end) of an n_starts-start run (the RNG is
 * keyed by the global index, so the union over any partition equals maple_extract's candidate set).
 * Used for multi-GPU sharding: each rank extracts its range, the caller all-gathers the rows
 * (torch.distributed / NCCL), then maple_dirset_merge runs the global dedupe + filter + sort. */
int maple_extract_range(maple_ctx* ctx, int64_t n_starts, int64_t begin, int64_t end, int32_t steps,
                        double step_size, uint64_t seed, maple_dirset** out);

/* Global pass over caller rows: `rows` is a DEVICE int8 buffer of k rows with row stride `stride`
 * (>= n) bytes; rows are checked, deduped (with sign twins), filtered and sorted exactly like the tail
 * of maple_extract. The buffer is only read during the call. */
int maple_dirset_merge(maple_ctx* ctx, const int8_t* rows, int64_t k, int32_t stride, maple_dirset** out);

/* Row-sharded global ⊑ pass (Def. 1-2). With the filter off
 * (maple_set_filter_minimal(ctx, 0)) maple_dirset_merge gives the deduped, sorted union `pool` of all ranks'
 * local sets — identical on every rank. Each rank then decides the rows [begin, end) of `pool`:
 * maple_dirset_keep_range writes keep_dev[i] = 1 iff row begin + i is ⊑-minimal in the whole pool (no other pool
 * row h has h ⊑ ±g), else 0 (end - begin bytes, DEVICE buffer of the caller; synchronised). After an all-gather of
 * the keep bytes, maple_dirset_select keeps the rows with keep_dev[i] != 0 (pool->size DEVICE bytes) and returns
 * them as a new sorted set — equal to maple_dirset_merge with the filter on. `pool` must belong to ctx.
 * Errors: BAD_ARG (null, foreign set, range outside [0, size]), RANGE (sum(u-l) > 1024), CUDA, OOM. Host only. */
int maple_set_filter_minimal(maple_ctx* ctx, int32_t on);
int maple_dirset_keep_range(maple_ctx* ctx, const maple_dirset* pool, int64_t begin, int64_t end, uint8_t* keep_dev);
int maple_dirset_select(maple_ctx* ctx, const maple_dirset* pool, const uint8_t* keep_dev, maple_dirset** out);

/* Direction-set accessors: canonical rows (first nonzero > 0), lexicographically sorted, size x n. */
int64_t maple_dirset_size(const maple_dirset* ds);
int64_t maple_dirset_pool_size(const maple_dirset* ds);   /* unique checked rows before the ⊑ filter */
int maple_dirset_copy(const maple_dirset* ds, int32_t* host_rows);            /* size*n int32, host */
/* Same rows as int8 (every entry lies in [-(u-l), u-l] with u-l <= 127): one strided device-to-host copy of
 * size*n bytes into caller-owned host memory (pageable or pinned), synchronised on the context stream. */
int maple_dirset_copy_i8(const maple_dirset* ds, int8_t* host_rows);
/* One contiguous device-to-host copy of the size x stride int8 rows as stored (stride = maple_dirset_stride >= n,
 * bytes n..stride-1 of a row are 0) into host_rows (size x stride bytes; pinned memory makes it one DMA at link
 * speed). Enqueued on the context stream and synchronised. */
int maple_dirset_copy_raw(const maple_dirset* ds, int8_t* host_rows);
const int8_t* maple_dirset_device_rows(const maple_dirset* ds);   /* borrowed; stride maple_dirset_stride */
/* Device-to-device copy of the size x stride int8 rows into caller memory `dst` (e.g. a torch tensor that
 * feeds the NCCL all-gather); enqueued on the context stream and synchronised. */
int maple_dirset_copy_device(const maple_dirset* ds, int8_t* dst);
int32_t maple_dirset_stride(const maple_dirset* ds);
void maple_dirset_free(maple_dirset* ds);

/* Import host rows (k x n int32) as a direction set after the same check/dedupe/filter/sort. */
int maple_dirset_from_host(maple_ctx* ctx, const int32_t* rows, int64_t k, int32_t filter_minimal,
                           maple_dirset** out);

/* ---- initial feasible solutions (NEXT #1) -------------------------------------------------------
 * maple_feasible_starts — Eq. 4 (§4.3): projected Adam (the extraction's Adam settings) from k
 * starts x0 ~ U(l, u) (splitmix64 counter, seed salted) on ||A x - b||^2 + lambda3 sum_i (x_i - floor x_i)
 * (ceil x_i - x_i) over [l, u] (lambda3 = 0.1 in the paper); each final x rounded half away from zero
 * is kept iff A x = b exactly; duplicates collapse; rows come out lexicographically sorted.
 * b: host int32 m (right-hand side, varies per call). x_out: host int32 cap x n (out). *count receives the
 * number of distinct feasible points found (rows beyond cap are dropped). X_debug (optional, host fp32 k x n):
 * the final continuous iterates. "No feasible point found" is count = 0, not an error.
 * Errors: BAD_ARG, CUDA, OOM.                                                                        */
int maple_feasible_starts(maple_ctx* ctx, const int32_t* b, int32_t k, int32_t steps, double step_size,
                          double lambda3, uint64_t seed, int32_t* x_out, int32_t cap, int32_t* count,
                          float* X_debug);

/* ---- augmentation -------------------------------------------------------------------------------
 * maple_augment — Graver-best augmentation (Alg. 2) from each of the k0 incumbents x0 (host,
 * k0 x n int32) in parallel, with test set D = ds ∪ -ds; each iteration takes the argmin of
 * f(x + lambda g) over g in D, integer lambda in [1, lambda_max(x, g)] with x + lambda g in [l, u] and
 * f(x + lambda g) < f(x) (ties: lexicographically smallest g, then smaller lambda), until no improving step
 * exists; returns the best final incumbent (ties: lexicographically smallest x) — MAPLE's multi-start
 * (§4.3). f is evaluated exactly via 2 f in fp64 (exact for integer data below 2^53).
 * f: objective (host arrays). b: host int32 m. x_best: host int32 n (out). f_best: host (out).
 * status: MAPLE_STATUS_*. iters (optional, host int32 k0, may be NULL): augmentation steps per incumbent.
 * Errors: BAD_ARG, INFEASIBLE (some x0 violates A x = b or the box), CUDA, OOM.                     */
int maple_augment(maple_ctx* ctx, const maple_dirset* ds, const maple_objective* f, const int32_t* b,
                  const int32_t* x0, int32_t k0, int32_t* x_best, double* f_best, int32_t* status,
                  int32_t* iters);

/* Batched shared-A augmentation (configs[3]): n_inst instances, instance t uses objective f[t],
 * right-hand side b[t*m..], incumbents x0[t*k0*n..]; outputs x_best[t*n..], f_best[t]. */
int maple_augment_many(maple_ctx* ctx, const maple_dirset* ds, int32_t n_inst, const maple_objective* f,
                       const int32_t* b, const int32_t* x0, int32_t k0, int32_t* x_best, double* f_best);

/* ---- instrumentation / parity hooks (used by tests and bench.py) -------------------------------
 * maple_debug_descent: run only the descent of starts [begin, end) (no harvest side effects) and copy
 * the final iterates (end-begin) x d fp32 to host `Z_out` (and, if Z0_out != NULL, the starts z0 in fp64).
 * maple_debug_candidates: after the last maple_extract / maple_extract_range on ctx, copy the harvested
 * candidate multiset (the rows handed to dedupe; in-box, nonzero, canonical) to host int32 rows; returns
 * the row count (call with host_rows = NULL, cap = 0 to query). Enabled by maple_set_debug(ctx, 1).
 * maple_last_timings: device milliseconds of the last extraction's phases
 * [descent, dedupe, check, filter, sort, total] and of the last augmentation [precompute, iterate, total]. */
int maple_debug_descent(maple_ctx* ctx, int64_t n_starts, int64_t begin, int64_t end, int32_t steps,
                        double step_size, uint64_t seed, float* Z_out, double* Z0_out);
int maple_set_debug(maple_ctx* ctx, int32_t keep_candidates);
/* Debug timeline of the CTA-pair descent kernel: enable != 0 arms it for the next launches (cleared); host_out (if not
 * NULL) receives 2 x 16 x 16 uint64 %globaltimer stamps [cta][step][slot] of the first pair's steps 0..15. */
int maple_debug_trace(maple_ctx* ctx, int32_t enable, uint64_t* host_out);
int64_t maple_debug_candidates(maple_ctx* ctx, int32_t* host_rows, int64_t cap);
int maple_last_timings(const maple_ctx* ctx, float* extract_ms6, float* augment_ms3);
/* Number of CUDA kernel launches the library issued since the context was created. */
int64_t maple_kernel_launches(const maple_ctx* ctx);
/* tcgen05 self-test on `device` (host buffers): D1 (128x64) = A1 (128x48) B1^T (B1 64x48) with kind::tf32 and
 * D2 (128x48) = A2 (128x64) B2^T (B2 48x64) with kind::f16, through the same shared-memory layout and
 * descriptors as the descent kernel; the caller compares with an exact host product. */
int maple_selftest_umma(int device, const float* A1, const float* B1, float* D1, const float* A2, const float* B2,
                        float* D2);
/* CTA-pair tcgen05 self-test on `device` (host buffers) for the large-shape descent kernel: a cluster of two CTAs,
 * each holding 64 rows of A; D1 = Ah Bh^T with kind::f16 (Ah 128x32, Bh 160x32, IEEE half bit patterns, fp32 D)
 * and D2 = A8 B8^T with kind::i8 (A8 128x64, B8 128x64, s32 D), B operands loaded by 3-D TMA boxes into the
 * canonical SWIZZLE_NONE layout, N split across the pair. raw1 (2 x 128 x 80 fp32) and raw2 (2 x 128 x 64 int32)
 * receive each CTA's TMEM lanes x columns as read back with tcgen05.ld 32x32b; the caller checks the layout
 * (row m of CTA r at lane m + 64 (n >= N/2), column n mod N/2) against an exact host product. */
int maple_selftest_pair(int device, const uint16_t* Ah, const uint16_t* Bh, const int8_t* A8, const int8_t* B8,
                        float* raw1, int32_t* raw2);
/* Select the descent kernel: 0 = auto (tcgen05 when the shape fits, else the CTA-pair tcgen05 kernel when its shape
 * fits, else SIMT), 1 = SIMT, 2 = tcgen05 (n, d <= 64; 2 threads per start), 4 = CTA-pair tcgen05 (large shapes, e.g. n = 300, d = 280: z in TMEM, B streamed by
 * TMA; Adam with every-step harvest only — a variant or an iterate beyond its f16 operand range runs SIMT). */
int maple_set_descent_kernel(maple_ctx* ctx, int32_t which);
/* The descent kernel the next extraction on `ctx` launches: 1 = SIMT (sparse B, warp per start), 2 = tcgen05,
 * 4 = CTA-pair tcgen05;
 * negative error code for a null context. Host only. */
int maple_descent_kernel(const maple_ctx* ctx);
/* Descent variants (DESIGN readings #24-#25). Alg. 3 line 8 updates z with "first-order
 * methods such as Adam": optimizer 0 = Adam (default, torch.optim.Adam formula), 1 = plain gradient descent
 * z <- z - step_size * g, 2 = sign gradient descent z <- z - step_size * sign(g) (sign(0) = 0), g the Eq. 3
 * subgradient. harvest_final = 1 applies Alg. 3 lines 9-10 to the final iterate z_T only (0: after
 * every step, the paper's loop). The CTA-pair kernel implements the default only: a variant extraction on a context
 * whose kernel would be 4 runs SIMT. Returns BAD_ARG for a null context or out-of-range values. Host only. */
int maple_set_descent_variant(maple_ctx* ctx, int32_t optimizer, int32_t harvest_final);
/* Select the ⊑-minimality filter's pair enumeration (Def. 1-2; the kept set is the same for all):
 * 0 = auto (level-synchronous when n <= 1024, else tiled), 1 = tiled (every row against all rows of smaller L1
 * norm), 2 = indexed (every row against the rows filed under one of its support coordinates with smaller L1 norm),
 * 3 = level-synchronous (L1 levels in increasing order, every row against the ⊑-minimal rows of smaller L1 filed
 * under its support coordinates — sufficient because ⊑ is a partial order — tested 32 rows at a time with
 * bit-sliced fold masks; one cooperative launch). 2 and 3 need n <= 1024 (else tiled).
 * Returns BAD_ARG for a null context or another value. Host only. */
int maple_set_filter_algorithm(maple_ctx* ctx, int32_t which);

#ifdef __cplusplus
}
#endif
#endif /* MAPLE_H */
