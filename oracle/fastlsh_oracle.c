/*
 * fastlsh_oracle.c — TEST INFRASTRUCTURE ONLY. Plain, slow, obviously-correct CPU reference.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library. It shares no code, header, table or generator with the CUDA path in
 * paper_2309_15479_b200/ (and neither includes the other).
 *
 * What it computes, in IEEE double (f32 inputs are exact in double):
 *
 *   Sampling operator S (§3.1): S(v) = (v[idx_0], ..., v[idx_{m-1}]), a multiset of
 *   m i.i.d. indices — duplicates are kept and counted.
 *
 *   FastLSH hash, Eq. 5 (§3.1):
 *       h(v) = floor( (a . S(v) + b) / w )
 *   with the dot product summed left to right over j = 0..m-1 (each product a_j * x_j of two f32
 *   values is exact in double), then + b, then / w, then floor toward -inf.
 *
 *   E2LSH, Eq. 1 (§2.2) is the same routine with m = n and the identity plan
 *   idx_j = j, so identity-FastLSH and E2LSH agree bit for bit (Eq. 5 reduces to Eq. 1).
 *
 *   scale = ||a|| * ||S(v)|| (multiset norm; duplicates counted) — the north_star tolerance unit.
 *
 * Parity pins: see tests/test_oracle_pins.py (paper worked example, hand-computed dyadic case,
 * identity == E2LSH, collision statistics vs the p-stable closed form, exact moments, brute force).
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

/* out[j] = v[idx[j]] — the sampling operator S(v) of PAPER.md:150. */
void oracle_apply_sampling(const double* v, int32_t n, const int32_t* idx, int32_t m, double* out) {
    (void)n;
    for (int32_t j = 0; j < m; ++j) out[j] = v[idx[j]];
}

/*
 * For every row r < N and hash i < k:
 *   p[r*k+i]     = sum_j a[i*m+j] * X[r*n + idx[i*m+j]]        (left to right)
 *   scale[r*k+i] = sqrt(sum_j a^2) * sqrt(sum_j X[..]^2)
 *   code[r*k+i]  = floor((p + b[i]) / w)  as int64; INT64_MIN if the quotient is not finite or
 *                  does not fit in int64.
 * Any of p/scale/code may be NULL. Rows are independent; `nthreads` > 1 splits them with OpenMP
 * (the per-row arithmetic and its order do not change).
 */
void oracle_hash(const float* X, int64_t N, int32_t n, const int32_t* idx, const float* a,
                 const float* b, double w, int32_t k, int32_t m, double* p, double* scale,
                 int64_t* code, int32_t nthreads) {
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int64_t r = 0; r < N; ++r) {
        const float* v = X + r * (int64_t)n;
        for (int32_t i = 0; i < k; ++i) {
            const int32_t* S = idx + (int64_t)i * m;
            const float* ai = a + (int64_t)i * m;
            double dot = 0.0, aa = 0.0, xx = 0.0;
            for (int32_t j = 0; j < m; ++j) {
                double x = (double)v[S[j]];
                double c = (double)ai[j];
                dot += c * x;
                aa += c * c;
                xx += x * x;
            }
            int64_t o = (int64_t)r * k + i;
            if (p) p[o] = dot;
            if (scale) scale[o] = sqrt(aa) * sqrt(xx);
            if (code) {
                double q = floor((dot + (double)b[i]) / w);
                code[o] = (isfinite(q) && q >= -9.2233720368547758e18 && q < 9.2233720368547758e18)
                              ? (int64_t)q : INT64_MIN;
            }
        }
    }
    (void)nthreads;
}

/* E2LSH of Eq. 1 with a dense coefficient matrix A[k][n] (row i = a_i): the identity plan. */
void oracle_e2lsh(const float* X, int64_t N, int32_t n, const float* A, const float* b, double w,
                  int32_t k, double* p, double* scale, int64_t* code, int32_t nthreads) {
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int64_t r = 0; r < N; ++r) {
        const float* v = X + r * (int64_t)n;
        for (int32_t i = 0; i < k; ++i) {
            const float* ai = A + (int64_t)i * n;
            double dot = 0.0, aa = 0.0, xx = 0.0;
            for (int32_t j = 0; j < n; ++j) {
                double x = (double)v[j];
                double c = (double)ai[j];
                dot += c * x;
                aa += c * c;
                xx += x * x;
            }
            int64_t o = (int64_t)r * k + i;
            if (p) p[o] = dot;
            if (scale) scale[o] = sqrt(aa) * sqrt(xx);
            if (code) {
                double q = floor((dot + (double)b[i]) / w);
                code[o] = (isfinite(q) && q >= -9.2233720368547758e18 && q < 9.2233720368547758e18)
                              ? (int64_t)q : INT64_MIN;
            }
        }
    }
    (void)nthreads;
}

int oracle_has_openmp(void) {
#ifdef _OPENMP
    return 1;
#else
    return 0;
#endif
}
