/* oracle/direct.c -- fp64 CPU oracle for the radial-SVD alignment landscape.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this file's library.  It shares no code, header, table or
 * constant with the CUDA path (paper_2202_07235_b200/csrc) and is never called by it.
 *
 * Plain, slow, obviously correct direct summation, complex128 interleaved (re, im):
 *
 *  O1  full-rank landscape, the discretization of the paper's inner product
 *        X(gamma) = <A, R_gamma B> = iint A(k,psi)^dagger B(k, psi - gamma) k dk dpsi
 *      (§2.2) with the radial quadrature sum_r w_r and the
 *      trapezoidal psi rule with dpsi = 2 pi / Q:
 *        X[k] = sum_{r<R} w_r dpsi sum_{j<Q} conj(a[r][j]) b[r][(j-k) mod Q],  gamma_k = 2 pi k / Q.
 *      Rotation by +gamma is the angular shift psi -> psi - gamma, so the
 *      template sample at angle psi_j - gamma_k is b[r][(j-k) mod Q].
 *
 *  O2  rank-H landscape: principal image rings (§3.2) built in psi-space,
 *        at[h][j] = sum_r U[r][h] eta_r a[r][j],  eta_r = sqrt(w_r)       (reading G2)
 *      then the same direct angular correlation over the H principal rings,
 *        X[k] = dpsi sum_{h<H} sum_{j<Q} conj(at[h][j]) bt[h][(j-k) mod Q].
 *      No FFT and no eigen-solver is used here; U is an input.
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC oracle/direct.c -o oracle/liboracle.so -lm
 * (no -ffast-math).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static const double ORACLE_TWO_PI = 6.283185307179586476925286766559;

/* O1 for one pair.  a, b: [R][Q] complex (2*R*Q doubles).  X: [Q] complex out. */
void oracle_landscape_full(int R, int Q, const double *w, const double *a, const double *b,
                           double *X)
{
    const double dpsi = ORACLE_TWO_PI / (double)Q;
    for (int k = 0; k < Q; ++k) {
        double xr = 0.0, xi = 0.0;
        for (int r = 0; r < R; ++r) {
            const double *ar = a + 2 * (size_t)r * Q;
            const double *br = b + 2 * (size_t)r * Q;
            double sr = 0.0, si = 0.0;
            for (int j = 0; j < Q; ++j) {
                int jj = j - k;
                if (jj < 0) jj += Q;
                const double are = ar[2 * j], aim = ar[2 * j + 1];
                const double bre = br[2 * jj], bim = br[2 * jj + 1];
                /* conj(a) * b */
                sr += are * bre + aim * bim;
                si += are * bim - aim * bre;
            }
            xr += w[r] * dpsi * sr;
            xi += w[r] * dpsi * si;
        }
        X[2 * k] = xr;
        X[2 * k + 1] = xi;
    }
}

/* O1 over a list of pairs: A [NA][R][Q], B [NB][R][Q]; pair p = (ia[p], ib[p]); X [P][Q]. */
void oracle_landscape_full_pairs(int R, int Q, const double *w, const double *A,
                                 const double *B, int64_t P, const int64_t *ia,
                                 const int64_t *ib, double *X, int nthreads)
{
    const size_t row = 2 * (size_t)R * Q;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int64_t p = 0; p < P; ++p)
        oracle_landscape_full(R, Q, w, A + row * ia[p], B + row * ib[p], X + 2 * (size_t)Q * p);
}

/* Principal rings in psi-space: at[h][j] = sum_r U[r*H + h] sqrt(w_r) a[r][j].
 * U is [R][H] row-major (column h = principal vector u_h).  a: [R][Q]; at: [H][Q]. */
void oracle_principal_rings(int R, int Q, int H, const double *w, const double *U,
                            const double *a, double *at)
{
    for (int h = 0; h < H; ++h) {
        for (int j = 0; j < Q; ++j) {
            double sr = 0.0, si = 0.0;
            for (int r = 0; r < R; ++r) {
                const double c = U[(size_t)r * H + h] * sqrt(w[r]);
                sr += c * a[2 * ((size_t)r * Q + j)];
                si += c * a[2 * ((size_t)r * Q + j) + 1];
            }
            at[2 * ((size_t)h * Q + j)] = sr;
            at[2 * ((size_t)h * Q + j) + 1] = si;
        }
    }
}

/* Direct angular correlation of principal rings: X[k] = dpsi sum_h sum_j conj(at) bt(j-k). */
void oracle_correlate_rings(int H, int Q, const double *at, const double *bt, double *X)
{
    const double dpsi = ORACLE_TWO_PI / (double)Q;
    for (int k = 0; k < Q; ++k) {
        double xr = 0.0, xi = 0.0;
        for (int h = 0; h < H; ++h) {
            const double *ah = at + 2 * (size_t)h * Q;
            const double *bh = bt + 2 * (size_t)h * Q;
            for (int j = 0; j < Q; ++j) {
                int jj = j - k;
                if (jj < 0) jj += Q;
                xr += ah[2 * j] * bh[2 * jj] + ah[2 * j + 1] * bh[2 * jj + 1];
                xi += ah[2 * j] * bh[2 * jj + 1] - ah[2 * j + 1] * bh[2 * jj];
            }
        }
        X[2 * k] = dpsi * xr;
        X[2 * k + 1] = dpsi * xi;
    }
}

/* O2 over a list of pairs.  Principal rings are formed per row on the fly (slow, simple). */
void oracle_landscape_rank_pairs(int R, int Q, int H, const double *w, const double *U,
                                 const double *A, const double *B, int64_t P,
                                 const int64_t *ia, const int64_t *ib, double *X, int nthreads)
{
    const size_t row = 2 * (size_t)R * Q;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
    {
        double *at = (double *)malloc(sizeof(double) * 2 * (size_t)H * Q);
        double *bt = (double *)malloc(sizeof(double) * 2 * (size_t)H * Q);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t p = 0; p < P; ++p) {
            oracle_principal_rings(R, Q, H, w, U, A + row * ia[p], at);
            oracle_principal_rings(R, Q, H, w, U, B + row * ib[p], bt);
            oracle_correlate_rings(H, Q, at, bt, X + 2 * (size_t)Q * p);
        }
        free(at);
        free(bt);
    }
}

/* O2 on precomputed principal rings (AT [NA][H][Q], BT [NB][H][Q]) over a pair list. */
void oracle_correlate_pairs(int H, int Q, const double *AT, const double *BT, int64_t P,
                            const int64_t *ia, const int64_t *ib, double *X, int nthreads)
{
    const size_t row = 2 * (size_t)H * Q;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int64_t p = 0; p < P; ++p)
        oracle_correlate_rings(H, Q, AT + row * ia[p], BT + row * ib[p], X + 2 * (size_t)Q * p);
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
