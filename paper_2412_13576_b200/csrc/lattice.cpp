// Host exact lattice step of maple_create — Alg. 3 lines 2-3, run once per A.
//
//   HNF (Prop. 1): column operations A C = (H | 0), C unimodular, in checked __int128.
//   B = C[:, m:]            (Thm. 1 setup: Ker_Z(A) = L(B)).
//   LLL (Alg. 1) with the paper's Siegel test ||B*_{k-1}||^2 > 2 ||B*_k||^2 (Def. P:136-144):
//     integer basis updates are exact; the Gram-Schmidt data are recomputed from exact inner products at
//     every visit of k (Schnorr-Euchner style). Fast path: basis in doubles while |entries| < 2^20 (exact
//     integers and inner products), fp64 Gram-Schmidt; otherwise checked __int128 + long double.
//   B+ = (B^T B)^{-1} B^T (Remark P:321-324): exact Gram matrix, fp64 Cholesky solve.
// Independent of oracle/lattice.py (which uses Python big integers and a different LLL bookkeeping).
#include <algorithm>
#include <immintrin.h>
#include <cmath>
#include <cstdint>
#include <string>
#include <thread>
#include <vector>

#include "lattice.h"

namespace maple {
namespace {

typedef __int128 i128;

struct Overflow {};

inline i128 mul_chk(i128 a, i128 b) {
    i128 r;
    if (__builtin_mul_overflow(a, b, &r)) throw Overflow();
    return r;
}
inline i128 add_chk(i128 a, i128 b) {
    i128 r;
    if (__builtin_add_overflow(a, b, &r)) throw Overflow();
    return r;
}
inline i128 sub_chk(i128 a, i128 b) {
    i128 r;
    if (__builtin_sub_overflow(a, b, &r)) throw Overflow();
    return r;
}
// floor division for i128
inline i128 fdiv(i128 a, i128 b) {
    i128 q = a / b, r = a % b;
    if (r != 0 && ((r < 0) != (b < 0))) --q;
    return q;
}
inline i128 iabs(i128 a) { return a < 0 ? -a : a; }

}  // namespace

int host_kernel_basis(const int32_t* A, int m, int n, std::vector<int64_t>& B, std::string& err) {
    // Column-major working copies: M (m x n) and C (n x n), column j contiguous, so a column operation streams
    // two contiguous columns; C starts as the identity and stays sparse, and zero entries of the source column
    // are skipped (no checked multiply), which keeps the operation count near the nonzeros touched.
    std::vector<i128> M(size_t(m) * n), C(size_t(n) * n, 0);
    for (int r = 0; r < m; ++r)
        for (int j = 0; j < n; ++j) M[size_t(j) * m + r] = A[size_t(r) * n + j];
    for (int i = 0; i < n; ++i) C[size_t(i) * n + i] = 1;
    auto mcol = [&](int j) { return &M[size_t(j) * m]; };
    auto ccol = [&](int j) { return &C[size_t(j) * n]; };
    auto axpy = [&](int j, int p, i128 q) {  // col_j -= q col_p
        if (q == 0) return;
        i128 *mj = mcol(j), *cj = ccol(j);
        const i128 *mp = mcol(p), *cp = ccol(p);
        for (int r = 0; r < m; ++r)
            if (mp[r] != 0) mj[r] = sub_chk(mj[r], mul_chk(q, mp[r]));
        for (int r = 0; r < n; ++r)
            if (cp[r] != 0) cj[r] = sub_chk(cj[r], mul_chk(q, cp[r]));
    };
    auto cswap = [&](int a, int b) {
        if (a == b) return;
        std::swap_ranges(mcol(a), mcol(a) + m, mcol(b));
        std::swap_ranges(ccol(a), ccol(a) + n, ccol(b));
    };
    auto Mrc = [&](int r, int j) -> i128& { return M[size_t(j) * m + r]; };
    try {
        for (int i = 0; i < m; ++i) {
            for (;;) {
                int p = -1, cnt = 0;
                for (int j = i; j < n; ++j)
                    if (Mrc(i, j) != 0) {
                        ++cnt;
                        if (p < 0 || iabs(Mrc(i, j)) < iabs(Mrc(i, p))) p = j;
                    }
                if (cnt == 0) {
                    err = "rank(A) < m: row " + std::to_string(i) + " has no pivot";
                    return -3;
                }
                if (cnt == 1) {
                    cswap(i, p);
                    break;
                }
                for (int j = i; j < n; ++j)
                    if (j != p && Mrc(i, j) != 0) axpy(j, p, fdiv(Mrc(i, j), Mrc(i, p)));
            }
            if (Mrc(i, i) < 0) {
                for (int r = 0; r < m; ++r) mcol(i)[r] = -mcol(i)[r];
                for (int r = 0; r < n; ++r) ccol(i)[r] = -ccol(i)[r];
            }
            for (int j = 0; j < i; ++j)
                if (Mrc(i, j) != 0) axpy(j, i, fdiv(Mrc(i, j), Mrc(i, i)));
        }
    } catch (Overflow&) {
        err = "integer overflow in HNF (checked __int128)";
        return -5;
    }
    const int d = n - m;
    B.assign(size_t(n) * d, 0);
    for (int j0 = 0; j0 < d; j0 += 16)   // blocked transpose: 16 contiguous columns of C -> 16 adjacent entries of B
        for (int r = 0; r < n; ++r)
            for (int j = j0; j < std::min(d, j0 + 16); ++j) {
                const i128 v = C[size_t(m + j) * n + r];
                if (v > INT64_MAX || v < INT64_MIN) {
                    err = "kernel basis entry exceeds int64";
                    return -5;
                }
                B[size_t(r) * d + j] = (int64_t)v;
            }
    return 0;
}

namespace {

// 4 independent accumulators (ILP / vectorisation); the sum of exact integer products is exact in double
// while every partial sum stays below 2^53 (guaranteed by the caller's entry bound)
inline double dot4_scalar(const double* a, const double* b, int len) {
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    int r = 0;
    for (; r + 4 <= len; r += 4) {
        s0 += a[r] * b[r];
        s1 += a[r + 1] * b[r + 1];
        s2 += a[r + 2] * b[r + 2];
        s3 += a[r + 3] * b[r + 3];
    }
    for (; r < len; ++r) s0 += a[r] * b[r];
    return (s0 + s1) + (s2 + s3);
}

// the same dot product with 4 x 4 AVX2 FMA lanes, chosen at run time when the host CPU has AVX2 + FMA (the
// library is built for baseline x86-64); a different summation order than the scalar version — equally valid
// for the fp64 Gram-Schmidt data and Cholesky factors (exact integer sums stay exact either way)
__attribute__((target("avx2,fma"))) double dot4_avx2(const double* a, const double* b, int len) {
    __m256d s0 = _mm256_setzero_pd(), s1 = _mm256_setzero_pd(), s2 = _mm256_setzero_pd(), s3 = _mm256_setzero_pd();
    int r = 0;
    for (; r + 16 <= len; r += 16) {
        s0 = _mm256_fmadd_pd(_mm256_loadu_pd(a + r), _mm256_loadu_pd(b + r), s0);
        s1 = _mm256_fmadd_pd(_mm256_loadu_pd(a + r + 4), _mm256_loadu_pd(b + r + 4), s1);
        s2 = _mm256_fmadd_pd(_mm256_loadu_pd(a + r + 8), _mm256_loadu_pd(b + r + 8), s2);
        s3 = _mm256_fmadd_pd(_mm256_loadu_pd(a + r + 12), _mm256_loadu_pd(b + r + 12), s3);
    }
    for (; r + 4 <= len; r += 4) s0 = _mm256_fmadd_pd(_mm256_loadu_pd(a + r), _mm256_loadu_pd(b + r), s0);
    const __m256d t = _mm256_add_pd(_mm256_add_pd(s0, s1), _mm256_add_pd(s2, s3));
    alignas(32) double v[4];
    _mm256_store_pd(v, t);
    double acc = (v[0] + v[1]) + (v[2] + v[3]);
    for (; r < len; ++r) acc += a[r] * b[r];
    return acc;
}

const bool kHaveAvx2 = __builtin_cpu_supports("avx2") && __builtin_cpu_supports("fma");

inline double dot4(const double* a, const double* b, int len) {
    return kHaveAvx2 ? dot4_avx2(a, b, len) : dot4_scalar(a, b, len);
}

// LLL fast path: the same algorithm as the exact path below (size reduction against j = k-1..0, Siegel test,
// Schnorr-Euchner recomputation of row k), with the basis held in doubles. Valid while every entry stays below
// 2^20 in magnitude: then every inner product is an exact integer (n * 2^40 < 2^53 for n <= 8192) and every
// basis update is exact. Returns 0 on success, 1 if the bound would be exceeded (the caller then runs the exact
// path from the original input), -3 on dependent columns.
int lll_fast(std::vector<int64_t>& Bnd, int n, int d, std::string& err) {
    constexpr double kMax = 1048576.0;   // 2^20
    if (n > 8192) return 1;
    std::vector<double> b((size_t)d * n);   // column k contiguous
    for (int r = 0; r < n; ++r)
        for (int k = 0; k < d; ++k) {
            const int64_t v = Bnd[(size_t)r * d + k];
            if (v >= (int64_t)kMax || v <= -(int64_t)kMax) return 1;
            b[(size_t)k * n + r] = (double)v;
        }
    std::vector<double> mu((size_t)d * d, 0.0), rr((size_t)d * d, 0.0), Bs(d, 0.0);
    auto col = [&](int k) { return &b[(size_t)k * n]; };
    // nonzero rows of every column (kernel bases are sparse: C5 has ~4 nonzeros per column of 1000) and, per row,
    // the columns nonzero there: the Gram row <b_k, b_j> (j < k) then costs the actual column overlaps only
    std::vector<std::vector<int>> nz(d), rc(n);
    auto unlink = [&](int k) {
        for (int r : nz[k]) {
            auto& v = rc[r];
            for (size_t t = 0; t < v.size(); ++t)
                if (v[t] == k) {
                    v[t] = v.back();
                    v.pop_back();
                    break;
                }
        }
    };
    auto link = [&](int k) {
        nz[k].clear();
        const double* c = col(k);
        for (int r = 0; r < n; ++r)
            if (c[r] != 0.0) {
                nz[k].push_back(r);
                rc[r].push_back(k);
            }
    };
    auto refresh = [&](int k) {
        unlink(k);
        link(k);
    };
    for (int k = 0; k < d; ++k) link(k);
    auto sdot = [&](int a, int c) {   // exact: integer products and partial sums below 2^53
        const std::vector<int>& s = nz[a].size() <= nz[c].size() ? nz[a] : nz[c];
        const double *x = col(a), *y = col(c);
        double acc = 0.0;
        for (int r : s) acc += x[r] * y[r];
        return acc;
    };
    // row k of the Gram-Schmidt data: r_kj = <b_k, b_j> - sum_{l<j} mu_jl r_kl, as a dense unit-triangular
    // recurrence over the contiguous rows of mu (vectorised dot products), starting at the first j whose Gram
    // entry is nonzero (r_kj = 0 before it)
    std::vector<double> gk(d, 0.0);
    std::vector<int> touched;
    auto gso_row = [&](int k) {
        double* rk = &rr[(size_t)k * d];
        double* mk = &mu[(size_t)k * d];
        touched.clear();
        const double* xk = col(k);
        int f = k;
        for (int r : nz[k])
            for (int j : rc[r])
                if (j < k) {
                    if (gk[j] == 0.0) touched.push_back(j);
                    gk[j] += xk[r] * col(j)[r];   // exact integers
                    f = std::min(f, j);
                }
        for (int j = 0; j < f; ++j) rk[j] = mk[j] = 0.0;
        for (int j = f; j < k; ++j) {
            const double s = gk[j] - dot4(&mu[(size_t)j * d + f], rk + f, j - f);
            rk[j] = s;
            mk[j] = s / Bs[j];
        }
        for (int j : touched) gk[j] = 0.0;
        Bs[k] = sdot(k, k) - dot4(mk + f, rk + f, k - f);
    };
    gso_row(0);
    if (Bs[0] <= 0) {
        err = "dependent kernel columns";
        return -3;
    }
    int k = 1;
    long iters = 0;
    while (k < d) {
        if (++iters > 200000000L) return 1;
        for (int pass = 0; pass < 64; ++pass) {
            gso_row(k);
            bool changed = false;
            for (int j = k - 1; j >= 0; --j) {
                const double mkj = mu[(size_t)k * d + j];
                const double q = std::nearbyint(mkj);
                if (std::fabs(mkj) > 0.5 + 1e-12 && q != 0) {
                    if (std::fabs(q) >= kMax) return 1;
                    double* bk = col(k);
                    const double* bj = col(j);
                    double mx = 0;
                    for (int r : nz[j]) {
                        bk[r] -= q * bj[r];   // exact: |q|, |b| < 2^20 -> |q b| < 2^40
                        mx = std::fmax(mx, std::fabs(bk[r]));
                    }
                    if (mx >= kMax) return 1;
                    for (int l = 0; l < j; ++l) mu[(size_t)k * d + l] -= q * mu[(size_t)j * d + l];
                    mu[(size_t)k * d + j] -= q;
                    changed = true;
                }
            }
            if (changed) refresh(k);
            if (!changed) break;
        }
        if (Bs[k] <= 0) {
            err = "dependent kernel columns";
            return -3;
        }
        if (Bs[k - 1] > 2.0 * Bs[k] * (1.0 + 1e-12)) {  // Siegel test (Alg. 1 line 5)
            unlink(k);
            unlink(k - 1);
            std::swap_ranges(col(k), col(k) + n, col(k - 1));
            link(k);
            link(k - 1);
            gso_row(k - 1);
            k = (k - 1 > 1) ? k - 1 : 1;
            if (k == 1) gso_row(0);
        } else {
            ++k;
        }
    }
    for (int r = 0; r < n; ++r)
        for (int kk = 0; kk < d; ++kk) Bnd[(size_t)r * d + kk] = (int64_t)b[(size_t)kk * n + r];
    return 0;
}

}  // namespace

int host_lll(std::vector<int64_t>& Bnd, int n, int d, std::string& err) {
    if (d <= 1) return 0;
    {
        std::vector<int64_t> trial = Bnd;
        const int rc = lll_fast(trial, n, d, err);
        if (rc <= 0) {
            if (rc == 0) Bnd.swap(trial);
            return rc;
        }
    }
    // exact path (entries beyond the fast path's bound)
    // columns b_k as contiguous vectors
    std::vector<std::vector<i128>> b(d, std::vector<i128>(n));
    for (int r = 0; r < n; ++r)
        for (int k = 0; k < d; ++k) b[k][r] = Bnd[size_t(r) * d + k];
    typedef long double ld;
    std::vector<std::vector<ld>> mu(d, std::vector<ld>(d, 0)), rr(d, std::vector<ld>(d, 0));
    std::vector<ld> Bs(d, 0);
    auto dot = [&](int a, int c) {
        i128 s = 0;
        for (int r = 0; r < n; ++r) s = add_chk(s, mul_chk(b[a][r], b[c][r]));
        return (ld)s;
    };
    auto gso_row = [&](int k) {
        for (int j = 0; j < k; ++j) {
            ld s = dot(k, j);
            for (int l = 0; l < j; ++l) s -= mu[j][l] * rr[k][l];
            rr[k][j] = s;
            mu[k][j] = s / Bs[j];
        }
        ld s = dot(k, k);
        for (int j = 0; j < k; ++j) s -= mu[k][j] * rr[k][j];
        Bs[k] = s;
    };
    try {
        gso_row(0);
        if (Bs[0] <= 0) {
            err = "dependent kernel columns";
            return -3;
        }
        int k = 1;
        long iters = 0;
        while (k < d) {
            if (++iters > 200000000L) {
                err = "LLL did not terminate";
                return -5;
            }
            // size-reduce b_k against j = k-1 .. 0 (reading #5), repeating until |mu_kj| <= 1/2
            for (int pass = 0; pass < 64; ++pass) {
                gso_row(k);
                bool changed = false;
                for (int j = k - 1; j >= 0; --j) {
                    ld q = std::nearbyint(mu[k][j]);
                    if (std::fabs(mu[k][j]) > 0.5L + 1e-12L && q != 0) {
                        i128 qi = (i128)(long long)q;
                        for (int r = 0; r < n; ++r) b[k][r] = sub_chk(b[k][r], mul_chk(qi, b[j][r]));
                        for (int l = 0; l < j; ++l) mu[k][l] -= q * mu[j][l];
                        mu[k][j] -= q;
                        changed = true;
                    }
                }
                if (!changed) break;
            }
            if (Bs[k] <= 0) {
                err = "dependent kernel columns";
                return -3;
            }
            if (Bs[k - 1] > 2.0L * Bs[k] * (1.0L + 1e-12L)) {  // Siegel test (Alg. 1 line 5)
                std::swap(b[k], b[k - 1]);
                gso_row(k - 1);
                k = (k - 1 > 1) ? k - 1 : 1;
                if (k == 1) gso_row(0);
            } else {
                ++k;
            }
        }
    } catch (Overflow&) {
        err = "integer overflow in LLL (checked __int128)";
        return -5;
    }
    for (int r = 0; r < n; ++r)
        for (int k = 0; k < d; ++k) {
            i128 v = b[k][r];
            if (v > INT64_MAX || v < INT64_MIN) {
                err = "LLL basis entry exceeds int64";
                return -5;
            }
            Bnd[size_t(r) * d + k] = (int64_t)v;
        }
    return 0;
}

namespace {

// f(i) for i in [0, count) on up to hardware_concurrency threads (interleaved indices: the triangular loops below
// have uneven rows); each i is computed by exactly one thread in the same arithmetic order as serially
template <class F>
void parallel_for(int count, F f) {
    const int nt = std::max(1, std::min<int>((int)std::thread::hardware_concurrency(), std::min(32, count / 16)));
    if (nt <= 1) {
        for (int i = 0; i < count; ++i) f(i);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            for (int i = t; i < count; i += nt) f(i);
        });
    for (auto& x : th) x.join();
}

// B+ fast path (|entries| < 2^20, n <= 8192): G = B^T B exactly in int64 from the rows' outer products (the
// rows of a reduced kernel basis are sparse), fp64 Cholesky G = L L^T, G^{-1} = L^{-T} L^{-1}, then each column
// of B+ = G^{-1} (row c of B) touches only the row's nonzeros. Returns 1 when out of range (exact path instead).
int pinv_fast(const std::vector<int64_t>& B, int n, int d, std::vector<double>& Bp, std::string& err) {
    if (n > 8192) return 1;
    std::vector<std::vector<std::pair<int, int64_t>>> rows(n);
    for (int r = 0; r < n; ++r)
        for (int j = 0; j < d; ++j) {
            const int64_t v = B[(size_t)r * d + j];
            if (v >= (1 << 20) || v <= -(1 << 20)) return 1;
            if (v) rows[r].emplace_back(j, v);
        }
    std::vector<int64_t> Gi((size_t)d * d, 0);   // |G_ij| <= n 2^40 < 2^53: exact, and exact as a double
    for (const auto& rw : rows)
        for (const auto& a : rw)
            for (const auto& b : rw)
                if (b.first <= a.first) Gi[(size_t)a.first * d + b.first] += a.second * b.second;
    std::vector<double> L((size_t)d * d, 0.0);   // lower triangle, row-major
    for (int j = 0; j < d; ++j) {
        double* Lj = &L[(size_t)j * d];
        const double s = (double)Gi[(size_t)j * d + j] - dot4(Lj, Lj, j);
        if (!(s > 0)) {
            err = "B^T B is not positive definite";
            return -3;
        }
        Lj[j] = std::sqrt(s);
        const double inv = 1.0 / Lj[j];
        for (int i = j + 1; i < d; ++i) {
            double* Li = &L[(size_t)i * d];
            Li[j] = ((double)Gi[(size_t)i * d + j] - dot4(Li, Lj, j)) * inv;
        }
    }
    // X = L^{-1} (lower triangular), stored transposed (Xt[j][i] = X[i][j]) so both loops below read rows; the
    // columns of X are independent triangular solves (one per thread at a time)
    std::vector<double> Xt((size_t)d * d, 0.0);
    parallel_for(d, [&](int j) {   // column j of X: L x = e_j, x_i = 0 for i < j, written in place into Xt row j
        double* col = &Xt[(size_t)j * d];
        col[j] = 1.0 / L[(size_t)j * d + j];
        for (int i = j + 1; i < d; ++i) {
            const double* Li = &L[(size_t)i * d];
            col[i] = -dot4(Li + j, &col[j], i - j) / Li[i];
        }
    });
    // G^{-1} = X^T X: (G^{-1})_{ab} = sum_{i >= max(a,b)} X_ia X_ib = dot of Xt rows a and b from max(a, b)
    std::vector<double> Ginv((size_t)d * d);
    parallel_for(d, [&](int a) {   // each thread writes only its own rows (lower triangle): no false sharing
        for (int b = 0; b <= a; ++b) Ginv[(size_t)a * d + b] = dot4(&Xt[(size_t)a * d + a], &Xt[(size_t)b * d + a], d - a);
    });
    for (int a = 0; a < d; ++a)
        for (int b = 0; b < a; ++b) Ginv[(size_t)b * d + a] = Ginv[(size_t)a * d + b];
    // column c of B+ = sum over row c's nonzeros (j, v) of v * column j of G^{-1}: accumulated contiguously as
    // row c of B+^T (one thread per c), then transposed in 32 x 32 blocks
    std::vector<double> BpT((size_t)n * d, 0.0);
    parallel_for(n, [&](int c) {
        double* out = &BpT[(size_t)c * d];
        for (const auto& e : rows[c]) {
            const double v = (double)e.second;
            const double* g = &Ginv[(size_t)e.first * d];   // column e.first of the symmetric G^{-1}
            for (int i = 0; i < d; ++i) out[i] += v * g[i];
        }
    });
    Bp.assign((size_t)d * n, 0.0);
    for (int c0 = 0; c0 < n; c0 += 32)
        for (int i0 = 0; i0 < d; i0 += 32)
            for (int i = i0; i < std::min(d, i0 + 32); ++i)
                for (int c = c0; c < std::min(n, c0 + 32); ++c) Bp[(size_t)i * n + c] = BpT[(size_t)c * d + i];
    return 0;
}

}  // namespace

int host_pinv(const std::vector<int64_t>& B, int n, int d, std::vector<double>& Bp, std::string& err) {
    {
        const int rc = pinv_fast(B, n, d, Bp, err);
        if (rc <= 0) return rc;
    }
    // exact-Gram path: G = B^T B in __int128, then Cholesky G = L L^T in long double, Bp = G^{-1} B^T.
    typedef long double ld;
    std::vector<ld> G(size_t(d) * d);
    for (int i = 0; i < d; ++i)
        for (int j = 0; j <= i; ++j) {
            i128 s = 0;
            for (int r = 0; r < n; ++r) s += (i128)B[size_t(r) * d + i] * B[size_t(r) * d + j];
            G[size_t(i) * d + j] = G[size_t(j) * d + i] = (ld)s;
        }
    std::vector<ld> L(size_t(d) * d, 0);
    for (int j = 0; j < d; ++j) {
        ld s = G[size_t(j) * d + j];
        for (int k = 0; k < j; ++k) s -= L[size_t(j) * d + k] * L[size_t(j) * d + k];
        if (s <= 0) {
            err = "B^T B is not positive definite";
            return -3;
        }
        L[size_t(j) * d + j] = std::sqrt(s);
        for (int i = j + 1; i < d; ++i) {
            ld t = G[size_t(i) * d + j];
            for (int k = 0; k < j; ++k) t -= L[size_t(i) * d + k] * L[size_t(j) * d + k];
            L[size_t(i) * d + j] = t / L[size_t(j) * d + j];
        }
    }
    Bp.assign(size_t(d) * n, 0.0);
    std::vector<ld> y(d);
    for (int c = 0; c < n; ++c) {  // solve G x = B^T e_c = row c of B
        for (int i = 0; i < d; ++i) {
            ld t = (ld)B[size_t(c) * d + i];
            for (int k = 0; k < i; ++k) t -= L[size_t(i) * d + k] * y[k];
            y[i] = t / L[size_t(i) * d + i];
        }
        for (int i = d - 1; i >= 0; --i) {
            ld t = y[i];
            for (int k = i + 1; k < d; ++k) t -= L[size_t(k) * d + i] * y[k];
            y[i] = t / L[size_t(i) * d + i];
        }
        for (int i = 0; i < d; ++i) Bp[size_t(i) * n + c] = (double)y[i];
    }
    return 0;
}

}  // namespace maple
