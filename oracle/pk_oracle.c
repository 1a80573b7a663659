/*
 * pk_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference interpreter's semantics
 * (parakern.interp.run_program, /root/reference/pkg/src/parakern/interp.py:215-225)
 * for the seven program families the executor binds to CUDA kernels.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library; the product path never does.
 *
 * What is restated, per interp.py:
 *   - bindings evaluated once with C99 truncating division      (interp.py:43-50, 68-69)
 *   - meta_for nests executed as a sequential lexicographic loop  (interp.py:158-174)
 *   - serial context loops (Jacobi t, matmul k) around the nest    (interp.py:148-152)
 *   - integer arithmetic: exact (int64 here; inputs are kept small enough
 *     that no intermediate exceeds int32 -- SURVEY App. C.5)
 *   - floating point: Python float == IEEE binary64, evaluated in program
 *     order (ascending reduction index), compiled with -ffp-contract=off so
 *     no FMA contraction changes the rounding
 * Programs: jacobi.mfk / transpose.mfk / addition.mfk are the reference's
 * shipped examples (pkg/src/parakern/data/); reverse / matvec / matmul /
 * jacobi2d are the SURVEY Appendix A programs shipped in
 * paper_1801_04348_b200/data/programs/.
 *
 * Independent outputs are spread over OpenMP threads; each output's own
 * reduction order is the interpreter's, so results do not depend on the
 * thread count.
 *
 * Return codes match include/pk.h: 0 ok, 3 = division by zero (the
 * interpreter raises ZeroDivisionError while evaluating a binding).
 */
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define PKO_OK 0
#define PKO_E_PARAM 1
#define PKO_E_DIV0 3

typedef int64_t i64;

/* C99 truncating division (interp.py:43-46). */
static i64 c_div(i64 a, i64 b) { return a / b; }
/* C99 remainder (interp.py:49-50). */
static i64 c_mod(i64 a, i64 b) { return a % b; }

static i64 max0(i64 v) { return v > 0 ? v : 0; }

int pko_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void pko_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ---------------------------------------------------------------------------
 * reverse.mfk:  dim = N/(s*B);  c[N-1-p] = a[p],
 * p = i*s*B + k*B + j  for i<dim, j<B, k<s.  The covered p form [0, dim*s*B).
 * ------------------------------------------------------------------------- */
int pko_reverse_i32(i64 N, i64 s, i64 B, const int32_t *a, int32_t *c) {
    if (s * B == 0) return PKO_E_DIV0;
    i64 dim = c_div(N, s * B);
    i64 P = max0(dim) * s * B;
    if (s < 0 || B < 0) P = 0; /* empty meta_for ranges */
    #pragma omp parallel for schedule(static)
    for (i64 p = 0; p < P; p++) c[N - 1 - p] = a[p];
    return PKO_OK;
}

/* ---------------------------------------------------------------------------
 * transpose.mfk (pkg/src/parakern/data/transpose.mfk:13-20):
 *   dim0 = N/B0, dim1 = N/(s*B1);  c[i*N + j] = a[j][i]
 *   i = v0*B0 + u0 < dim0*B0,  j = (v1*s + k)*B1 + u1 < dim1*s*B1.
 * Word permutation: 32-bit patterns move unchanged (int or float bits).
 * ------------------------------------------------------------------------- */
int pko_transpose_u32(i64 N, i64 s, i64 B0, i64 B1, const uint32_t *a, uint32_t *c) {
    if (B0 == 0 || s * B1 == 0) return PKO_E_DIV0;
    i64 I = max0(c_div(N, B0)) * B0;
    i64 J = max0(c_div(N, s * B1)) * s * B1;
    if (B0 < 0 || B1 < 0 || s < 0) { I = 0; J = 0; }
    #pragma omp parallel for schedule(static)
    for (i64 i = 0; i < I; i++)
        for (i64 j = 0; j < J; j++) c[i * N + j] = a[j * N + i];
    return PKO_OK;
}

/* ---------------------------------------------------------------------------
 * jacobi.mfk (pkg/src/parakern/data/jacobi.mfk:9-25), a[2N]:
 *   dim = (N-2)/(s*B);  for t<T: for p<dim*s*B:
 *     t even: a[p+1]   = (a[N+p] + a[N+p+1] + a[N+p+2]) / 3
 *     t odd:  a[N+p+1] = (a[p]   + a[p+1]   + a[p+2])   / 3
 * One schedule instance per t (interp.py:148-152); within it the source
 * half is never written, so the sweep order does not matter.
 * ------------------------------------------------------------------------- */
int pko_jacobi1d_i32(i64 T, i64 N, i64 s, i64 B, int32_t *a) {
    if (s * B == 0) return PKO_E_DIV0;
    i64 dim = c_div(N - 2, s * B);
    i64 P = max0(dim) * s * B;
    if (s < 0 || B < 0) P = 0;
    for (i64 t = 0; t < T; t++) {
        int32_t *dst = (c_mod(t, 2) == 0) ? a : a + N;
        const int32_t *src = (c_mod(t, 2) == 0) ? a + N : a;
        #pragma omp parallel for schedule(static)
        for (i64 p = 0; p < P; p++) {
            i64 sum = (i64)src[p] + (i64)src[p + 1] + (i64)src[p + 2];
            dst[p + 1] = (int32_t)c_div(sum, 3);
        }
    }
    return PKO_OK;
}

/* ---------------------------------------------------------------------------
 * jacobi2d.mfk, a[2N][N] row-major:
 *   dim0 = (N-2)/B0, dim1 = (N-2)/(s*B1)
 *   i = v0*B0+u0+1 in [1, dim0*B0],  j = (v1*s+k)*B1+u1+1 in [1, dim1*s*B1]
 *   t even: a[N+i][j] = (a[i-1][j] + a[i+1][j] + a[i][j-1] + a[i][j+1] + a[i][j]) / 5
 *   t odd:  a[i][j]   = (a[N+i-1][j] + ... + a[N+i][j]) / 5
 * ------------------------------------------------------------------------- */
int pko_jacobi2d_i32(i64 T, i64 N, i64 s, i64 B0, i64 B1, int32_t *a) {
    if (B0 == 0 || s * B1 == 0) return PKO_E_DIV0;
    i64 I = max0(c_div(N - 2, B0)) * B0;
    i64 J = max0(c_div(N - 2, s * B1)) * s * B1;
    if (B0 < 0 || B1 < 0 || s < 0) { I = 0; J = 0; }
    for (i64 t = 0; t < T; t++) {
        int32_t *dst = (c_mod(t, 2) == 0) ? a + N * N : a;
        const int32_t *src = (c_mod(t, 2) == 0) ? a : a + N * N;
        #pragma omp parallel for schedule(static)
        for (i64 i = 1; i <= I; i++) {
            for (i64 j = 1; j <= J; j++) {
                i64 sum = (i64)src[(i - 1) * N + j] + (i64)src[(i + 1) * N + j] +
                          (i64)src[i * N + j - 1] + (i64)src[i * N + j + 1] +
                          (i64)src[i * N + j];
                dst[i * N + j] = (int32_t)c_div(sum, 5);
            }
        }
    }
    return PKO_OK;
}

/* ---------------------------------------------------------------------------
 * matvec.mfk:  dim = N/(s*B)
 *   r = i*s*B + k*B + j < dim*s*B;  for q<N: y[r] = y[r] + a[r][q]*x[q]
 * Ascending q per row (the interpreter's order).
 * ------------------------------------------------------------------------- */
int pko_matvec_i32(i64 N, i64 s, i64 B, const int32_t *a, const int32_t *x, int32_t *y) {
    if (s * B == 0) return PKO_E_DIV0;
    i64 R = max0(c_div(N, s * B)) * s * B;
    if (s < 0 || B < 0) R = 0;
    #pragma omp parallel for schedule(static)
    for (i64 r = 0; r < R; r++) {
        i64 acc = y[r];
        for (i64 q = 0; q < N; q++) acc = acc + (i64)a[r * N + q] * (i64)x[q];
        y[r] = (int32_t)acc;
    }
    return PKO_OK;
}

/* Same program over Python floats: binary64 with the interpreter's order,
 * y = (((y + a0*x0) + a1*x1) + ...).  Inputs are the f32 values widened. */
int pko_matvec_f64(i64 N, i64 s, i64 B, const float *a, const float *x, double *y) {
    if (s * B == 0) return PKO_E_DIV0;
    i64 R = max0(c_div(N, s * B)) * s * B;
    if (s < 0 || B < 0) R = 0;
    #pragma omp parallel for schedule(static)
    for (i64 r = 0; r < R; r++) {
        double acc = y[r];
        for (i64 q = 0; q < N; q++) {
            double prod = (double)a[r * N + q] * (double)x[q];
            acc = acc + prod;
        }
        y[r] = acc;
    }
    return PKO_OK;
}

/* ---------------------------------------------------------------------------
 * matmul.mfk (paper Fig. 3):
 *   dim0 = n/B0, dim1 = n/(ub1*s), kdim = n/B0
 *   for k<kdim (serial context loop), for every (p, q) of the nest, for z<B0:
 *     c[p][q] = c[p][q] + a[p][B0*k+z] * b[B0*k+z][q]
 *   p < dim0*B0, q < dim1*ub1*s; the reduction index kk = B0*k+z runs
 *   ascending over [0, kdim*B0) for every output.
 * ------------------------------------------------------------------------- */
int pko_matmul_f64_rows(i64 n, i64 B0, i64 ub1, i64 s, i64 r0, i64 r1, const float *a, const float *b,
                        double *c);

static void matmul_extents(i64 n, i64 B0, i64 ub1, i64 s, i64 *M, i64 *Nc, i64 *K) {
    i64 dim0 = c_div(n, B0), dim1 = c_div(n, ub1 * s), kdim = c_div(n, B0);
    *M = max0(dim0) * B0;
    *Nc = max0(dim1) * ub1 * s;
    *K = max0(kdim) * B0;
    if (B0 < 0 || ub1 < 0 || s < 0) { *M = 0; *Nc = 0; *K = 0; }
}

int pko_matmul_i32(i64 n, i64 B0, i64 ub1, i64 s, const int32_t *a, const int32_t *b, int32_t *c) {
    if (B0 == 0 || ub1 * s == 0) return PKO_E_DIV0;
    i64 M, Nc, K;
    matmul_extents(n, B0, ub1, s, &M, &Nc, &K);
    #pragma omp parallel for schedule(static)
    for (i64 p = 0; p < M; p++) {
        for (i64 q = 0; q < Nc; q++) {
            i64 acc = c[p * n + q];
            for (i64 kk = 0; kk < K; kk++) acc = acc + (i64)a[p * n + kk] * (i64)b[kk * n + q];
            c[p * n + q] = (int32_t)acc;
        }
    }
    return PKO_OK;
}

int pko_matmul_f64(i64 n, i64 B0, i64 ub1, i64 s, const float *a, const float *b, double *c) {
    return pko_matmul_f64_rows(n, B0, ub1, s, 0, n, a, b, c);
}

/* The rows [r0, r1) of the same program (a bounded sample of one run: the
 * rows are independent, every output keeps its ascending-kk sequence). */
int pko_matmul_f64_rows(i64 n, i64 B0, i64 ub1, i64 s, i64 r0, i64 r1, const float *a, const float *b, double *c) {
    if (B0 == 0 || ub1 * s == 0) return PKO_E_DIV0;
    i64 M, Nc, K;
    matmul_extents(n, B0, ub1, s, &M, &Nc, &K);
    if (r0 < 0) r0 = 0;
    if (r1 > M) r1 = M;
    #pragma omp parallel for schedule(static)
    for (i64 p = r0; p < r1; p++) {
        double *crow = c + p * n;
        /* ascending kk per output; the q loop is innermost only for cache
         * locality -- every c[p][q] still sees kk = 0, 1, 2, ... in order */
        for (i64 kk = 0; kk < K; kk++) {
            double av = (double)a[p * n + kk];
            const float *brow = b + kk * n;
            for (i64 q = 0; q < Nc; q++) {
                double prod = av * (double)brow[q];
                crow[q] = crow[q] + prod;
            }
        }
    }
    return PKO_OK;
}

/* ---------------------------------------------------------------------------
 * addition.mfk (pkg/src/parakern/data/addition.mfk:11-23), flat a,b,c[N*N]:
 *   dim0 = N/B0, dim1 = N/(2*B1);  i < dim0*B0, j < dim1*B1
 *   if (i < N && j < N/2) { c[iN+j] = a+b;  c[iN+j+N/2] = a+b (twin) }
 * ------------------------------------------------------------------------- */
int pko_addition_i32(i64 N, i64 B0, i64 B1, const int32_t *a, const int32_t *b, int32_t *c) {
    if (B0 == 0 || 2 * B1 == 0) return PKO_E_DIV0;
    i64 I = max0(c_div(N, B0)) * B0;
    i64 J = max0(c_div(N, 2 * B1)) * B1;
    if (B0 < 0 || B1 < 0) { I = 0; J = 0; }
    i64 half = c_div(N, 2);
    #pragma omp parallel for schedule(static)
    for (i64 i = 0; i < I; i++) {
        if (i >= N) continue;
        for (i64 j = 0; j < J; j++) {
            if (!(j < half)) continue;
            c[i * N + j] = (int32_t)((i64)a[i * N + j] + (i64)b[i * N + j]);
            c[i * N + j + half] = (int32_t)((i64)a[i * N + j + half] + (i64)b[i * N + j + half]);
        }
    }
    return PKO_OK;
}
