// Launch wrappers of the MAPLE device kernels (host-callable; implemented in k_*.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace maple {

// Sparse B for the SIMT path: CSR (rows i, for B z and B r), CSC (columns j, for B^T s) and load-balanced
// per-lane row / column lists (snake order by nonzero count). Column lists bound the per-lane Adam state.
struct SparseB {   // lane-major ELL schedules of B (sparse_ell.h), built once per context
    int nnz;                      // nonzeros of B
    int Lf, qf, nfix, nfixpos;    // forward (rows of B): slots, pieces per lane, split rows, their pieces
    int Lb, qd;                   // backward (columns of B): slots, coordinates per lane (whole columns)
    const uint32_t* ell_f;        // Lf * 32 words, gather z / r (places qd * 32, owner order)
    const int32_t* own_f;         // qf * 32: row of each piece, -1 for pieces of split rows / unused
    const int32_t* fix;           // nfix triples (row, first, count) into fixpos
    const int32_t* fixpos;        // queue positions q * 32 + lane of the split rows' pieces
    const uint32_t* ell_b;        // Lb * 32 words, gather s (places qf * 32 + nfix)
    const int32_t* own_b;         // qd * 32: coordinate owned by lane L in place q, or -1
    const int32_t* pos_s;         // n: place of row i in s (forward place q * 32 + L; split rows qf * 32 + f)
    const int32_t* pos_z;         // d: place of coordinate j in z (its backward place q * 32 + L)
    // z and r live in owner order: coordinate own_b[k] at place k (qd * 32 places); the forward words gather
    // places, not coordinates
};

struct DescentParams {
    int n, d, n_pad, T;
    float lam1, lam2, beta1, beta2, eps;
    float omb1, omb2;             // (1 - beta1), (1 - beta2) rounded from fp64 (torch.optim.Adam scalars)
    const float4* step_tab;       // per step t=1..T: (lr/(1-beta1^t), sqrt(1-beta2^t), 1/sqrt(1-beta2^t), 0)
    uint64_t seed;
    int64_t n_total;              // RNG key space (global start count)
    int64_t begin, count;         // global starts [begin, begin + count)
    const float* B_nd;            // B, n x d row-major (fp32, exact small integers)
    const float* B_dn;            // B^T, d x n row-major
    const int8_t* B8_nd;          // B as int8, n x d
    SparseB sb;                   // sparse B (SIMT path)
    const double* Bp;             // B+, d x n row-major
    const int32_t* lo;            // l (n)
    const int32_t* hi;            // u (n)
    const int32_t* box;           // u - l (n)
    int harvest;                  // 0: descent only (debug)
    int opt;                      // line 8's update (reading #24): 0 Adam, 1 GD (z - lr g), 2 sign-GD (z - lr sign g)
    int harvest_final;            // 1: harvest the final iterate only (reading #25)
    float lr;                     // step size (GD / sign-GD)
    int8_t* cand;                 // candidate rows, stride n_pad
    int64_t cand_cap;
    unsigned long long* cand_count;
    float* Z_out;                 // optional: final iterates (count x d)
    double* Z0_out;               // optional: starts (count x d)
    const double* Z0_in;          // optional (SIMT): the starts z0 = B+ g0 precomputed by a DGEMM (count x d, fp64)
    // CTA-pair tcgen05 kernel (k_descent_tcp.cu): padded operand copies of B and the range flag
    int tcp_np, tcp_dp;           // padded n (multiple of 64) and d (multiple of 96 / 32, see tcp_shape)
    const uint16_t* B16p;         // B as IEEE half, tcp_np x tcp_dp row-major (zero padded)
    const int8_t* BT8p;           // B^T as int8, tcp_dp x tcp_np row-major (zero padded)
    const int8_t* B8p;            // B as int8, tcp_np x tcp_dp row-major (zero padded; the harvest operand)
    int* range_flag;              // set to 1 if an iterate left the f16 range of the operands (|z| > 60000)
    unsigned long long* trace;    // optional (debug): per-step %globaltimer stamps of the first pair (tcp kernel)
};

// SIMT descent + harvest (one warp per start). Returns a cudaError_t.
cudaError_t launch_descent_simt(const DescentParams& p, cudaStream_t s);
// g0 (count x n, fp64) of global starts [begin, begin + count): the same counter RNG and box map as the kernels
cudaError_t launch_start_g0(const DescentParams& p, double* g0, cudaStream_t s);
// tcgen05 descent + harvest (128 starts per CTA, state resident on chip). Returns cudaErrorNotSupported
// when the shape does not fit the kernel's tile limits.
cudaError_t launch_descent_tc(const DescentParams& p, cudaStream_t s);
bool descent_tc_supported(int n, int d);
// single-tile tcgen05 self-test (device pointers): D1 = A1 B1^T (tf32, 128x48 * 48x64), D2 = A2 B2^T (f16, 128x64 * 64x48)
cudaError_t umma_selftest(const float* A1, const float* B1, float* D1, const float* A2, const float* B2, float* D2,
                          cudaStream_t s);

// CTA-pair tcgen05 descent + harvest (64 starts per CTA, 128 per pair; state on chip: z in TMEM, Adam m / v in
// registers). tcp_shape: the padded (np, dp) a shape runs at, false when no instantiation fits.
bool tcp_shape(int n, int d, int* np, int* dp);
cudaError_t launch_descent_tcp(const DescentParams& p, cudaStream_t s);
// CTA-pair (cta_group::2) self-test (k_descent_tcp.cu): device pointers; see maple_selftest_pair
cudaError_t pair_selftest(const void* Ah, const void* Bh, const void* A8, const void* B8, float* raw1, int32_t* raw2,
                          cudaStream_t s);

struct HashSet {
    unsigned long long* keys;     // 0 = empty; else (32-bit hash | 1) << 32 | ref (k_post.cu dedupe_kernel)
    int64_t* newslot;             // per pool index: table slot of a row inserted by the running launch, else -1
    uint64_t mask;                // slots - 1
    int8_t* pool;                 // unique rows, stride n_pad
    int64_t pool_cap;
    unsigned long long* pool_count;
    int* overflow;
    unsigned long long* max_count;  // running max of the input counts (detects candidate-buffer overflow)
};

// Insert min(*dcount, cap) rows (stride row_stride) into the set; new unique rows are appended to the pool
// (two launches: the insert and the copy of the new rows). Row indices must be < 2^31.
cudaError_t launch_dedupe(const int8_t* rows, const unsigned long long* dcount, int64_t cap, int row_stride,
                          int n_pad, const HashSet& hs, cudaStream_t s);

struct CheckParams {
    int m, n, n_pad;
    const int32_t* A_rowptr;      // CSR of A
    const int32_t* A_col;
    const int32_t* A_val;
    int nnz;
    const int32_t* box;           // u - l
};
struct FilterWork {
    int n, n_pad;
    int Lh, Wh;                   // thermometer bits per half, 32-bit words per half
    int binary;                   // all u_i - l_i == 1: bit i of a half <-> coordinate i (fast path)
    const int32_t* off;           // n: first thermometer bit of coordinate i (prefix sum of u - l)
    const int32_t* word_c0;       // Wh: first coordinate with a bit in word w
    const int32_t* word_c1;       // Wh: last coordinate with a bit in word w
    uint32_t* codes;              // count x 2Wh
    int32_t* l1;                  // count
    int32_t* hist;                // Lmax + 2
    int32_t* level_start;         // Lmax + 2
    int32_t* cursor;              // Lmax + 2
    int32_t* order;               // count
    uint8_t* keep;                // count
    int32_t* witness;             // count
    int Lmax;
    uint4* sig;                   // count: 64-bit folds (bit i mod 64) of the two code halves (the filter's prefilter)
    int algo;                     // 1: tiled scan of all lower-L1 rows; 2: tiled prefix, then indexed by key coordinate;
                                  // 3: tiled prefix, then level-synchronous over minimal rows (coordinate-major tiles)
    int scan_cap;                 // tiled scan: rows of smaller L1 scanned per row (set by launch_filter)
    const int8_t* rows;           // the rows themselves (stride n_pad): supports, for the indexed filter
    int32_t* freq;                // n: rows having coordinate i in their support
    int32_t* key_bin;             // count: key coordinate * (Lmax + 1) + L1
    int32_t* bin_hist;            // n * (Lmax + 1)
    int32_t* bin_start;           // n * (Lmax + 1) + 1
    int32_t* bin_cursor;          // n * (Lmax + 1)
    int32_t* list_row;            // count: rows in bin order
    uint4* list_sig;              // count: their folds, in bin order
    int32_t* n_undec;             // rows the tiled prefix left undecided (the index is built only if > 0)
    // level-synchronous filter (algo 3)
    int32_t* gl_cursor;           // (Lmax + 1) n: histogram, then cursor of the G lists (undecided rows by (L1, c))
    int32_t* gl_start;            // (Lmax + 1) n + 1
    int32_t* gl_rows;             // sum of |supp| over the undecided rows (capacity count x n)
    int32_t* h_fill;              // n: minimal rows appended so far to each key coordinate's list
    int64_t gl_cap;               // capacity of gl_rows; the level pass falls back to the indexed pass beyond it
    int idx_fallback;             // 1: the indexed-pass kernels run only when the G lists overflowed (algo 3)
    int64_t g_begin, g_end;       // decide keep only for rows [g_begin, g_end) (a shard of the global pass); g_end = 0: all
};
// flags[r] = 1 iff A g = 0 (exact int64), g != 0 and |g| <= u - l (conditions C1-C3), for the first
// min(*dcount, cap) rows; with encode != 0 also the filter's thermometer codes and L1 norms.
cudaError_t launch_check_codes(const int8_t* rows, const unsigned long long* dcount, int64_t cap, const CheckParams& cp,
                               FilterWork& fw, int encode, uint8_t* flags, unsigned long long* n_bad, cudaStream_t s);
// keep[r] (and witness[r]) for the ⊑ filter, or keep = valid when filter_minimal == 0
cudaError_t launch_filter(const unsigned long long* dcount, int64_t cap, const uint8_t* valid, FilterWork& fw,
                          int filter_minimal, cudaStream_t s, int* launches);
// Gather rows with sel[r] != 0 into out (stride n_pad) in an arbitrary order; count to *n_out (device), the
// largest nonzero count among them to *nz_max (atomic max).
cudaError_t launch_compact(const int8_t* rows, const uint8_t* sel, const unsigned long long* dcount, int64_t cap,
                           int n_pad, int8_t* out, unsigned long long* n_out, unsigned long long* nz_max, cudaStream_t s);
// Lexicographic sort of k rows (stride n_pad, n bytes compared as signed int8). keys/idx scratch:
// keys: k * n_pad/4 uint32, idx0/idx1: k int32. Result written to out rows.
cudaError_t launch_lex_sort(const int8_t* rows, int64_t k, int n, int n_pad, uint32_t* keys, int32_t* idx0,
                            int32_t* idx1, int8_t* out, cudaStream_t s, int* launches);

// ---- Eq. 4 feasible starts ----
struct FeasibleParams {
    int n, m, n_pad, T;
    int64_t k;                    // number of starts
    float lam3, beta1, beta2, eps, omb1, omb2;
    const float4* step_tab;
    uint64_t seed;
    int nnz;                      // nonzeros of A (the CSR / CSC arrays below are staged in shared memory)
    const int32_t* A_rowptr;      // CSR of A
    const int32_t* A_col;
    const int32_t* A_val;
    const int32_t* AT_colptr;     // CSC of A (rows of A^T)
    const int32_t* AT_row;
    const int32_t* AT_val;
    const int32_t* b;             // m
    const int32_t* lo;            // l
    const int32_t* hi;            // u
    int8_t* rows;                 // kept x - l, stride n_pad
    int64_t cap;
    unsigned long long* count;
    float* X_out;                 // optional debug: final iterates (k x n)
};
cudaError_t launch_feasible(const FeasibleParams& p, cudaStream_t s);

// ---- augmentation ----
struct AugmentParams {
    int n, m, n_pad;
    int n_dir;                    // canonical directions K; D = ±, sorted lexicographically: 2K entries
    const int8_t* dirs;           // D, 2K x n_pad (lex sorted, both signs)
    const int32_t* nnz;           // ELL of D: nonzeros per row (2K)
    const uint32_t* words;        // nzmax x 2K, slot-major: column | (uint8)value << 16 | END << 24 (columns ascending)
    int nzmax;
    const double* Q;              // n x n (per instance: Q + inst * n * n)
    const double* c;              // n (per instance)
    const double* c0;             // per instance
    const double* qg;             // per instance: g^T Q g for every D entry (2K)
    int table;                    // 1: separable value tables (MAPLE_OBJ_TABLE) instead of Q, c
    const double* tab;            // per instance: tab + inst * tab_len; entry tab_off[j] + (x_j - l_j) = f_j(x_j)
    const int32_t* tab_off;       // n offsets (shared: l, u are the context's)
    int64_t tab_len;
    const int32_t* lo;
    const int32_t* hi;
    int32_t* X;                   // incumbents, (n_inst * k0) x n, updated in place
    int k0, n_inst;
    double* F2;                   // per incumbent: final 2 f(x)
    int32_t* iters;               // per incumbent
    int max_iter;
};
cudaError_t launch_augment_qg(const AugmentParams& p, cudaStream_t s);
cudaError_t launch_augment(const AugmentParams& p, cudaStream_t s);
// slot-major ELL words of the 2K rows of D (width x nD, width >= every row's nonzero count) and nnz
cudaError_t launch_augment_ell(const int8_t* dirs, int nD, int n, int n_pad, int width, int32_t* nnz, uint32_t* words,
                               cudaStream_t s);
cudaError_t launch_augment_best(const AugmentParams& p, int32_t* xbest, double* f2best, cudaStream_t s);
// D = S ∪ -S in lexicographic order from a lexicographically sorted canonical S (a merge; 2k rows into out)
cudaError_t launch_signed_merge(const int8_t* S, int64_t k, int n, int n_pad, int8_t* out, cudaStream_t s);

}  // namespace maple
