// rsvd_eigen.cpp -- host fp64 symmetric eigen-solver for the R x R kernel matrix C (row a0).
//
// The paper takes "the singular-value-decomposition" of the symmetric PSD kernel C to get the
// principal vectors u_1..u_H; for a symmetric matrix that is its eigen-decomposition
// (reading G7).  R <= 256, so a host solver costs ~ms.
//
// Algorithm: Householder reduction to tridiagonal form with accumulated orthogonal factor, then
// implicit symmetric QR steps with Wilkinson shifts and deflation (the textbook symmetric QR
// algorithm), all in fp64 with a fixed operation order, so the result is deterministic.  Output:
// eigenvalues descending (stable order), eigenvectors normalised with the sign rule "largest-|.|
// entry positive" (first such entry on ties).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/rsvd.h"

namespace rsvd {
rsvd_status fail(rsvd_status st, const std::string &msg);
}

namespace {

// A (n x n, row-major, symmetric) -> tridiagonal (d, e) with A = Z T Z^T.
void householder_tridiag(int n, std::vector<double> &A, std::vector<double> &Z,
                         std::vector<double> &d, std::vector<double> &e) {
    Z.assign((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) Z[(size_t)i * n + i] = 1.0;
    std::vector<double> v(n), p(n), q(n);
    for (int k = 0; k + 2 < n; ++k) {
        const int m = n - k - 1;                 // length of x = A[k+1..n-1][k]
        double alpha = 0.0;
        for (int i = 0; i < m; ++i) alpha += A[(size_t)(k + 1 + i) * n + k] * A[(size_t)(k + 1 + i) * n + k];
        alpha = std::sqrt(alpha);
        if (alpha == 0.0) continue;
        const double x0 = A[(size_t)(k + 1) * n + k];
        if (x0 > 0) alpha = -alpha;              // v = x - alpha e1, alpha = -sign(x0) ||x||
        for (int i = 0; i < m; ++i) v[i] = A[(size_t)(k + 1 + i) * n + k];
        v[0] -= alpha;
        double vv = 0.0;
        for (int i = 0; i < m; ++i) vv += v[i] * v[i];
        if (vv == 0.0) continue;
        const double beta = 2.0 / vv;
        // trailing block B = A[k+1.., k+1..]:  B <- H B H = B - v q^T - q v^T
        for (int i = 0; i < m; ++i) {
            double s = 0.0;
            const double *row = &A[(size_t)(k + 1 + i) * n + (k + 1)];
            for (int j = 0; j < m; ++j) s += row[j] * v[j];
            p[i] = beta * s;
        }
        double vp = 0.0;
        for (int i = 0; i < m; ++i) vp += v[i] * p[i];
        const double K = 0.5 * beta * vp;
        for (int i = 0; i < m; ++i) q[i] = p[i] - K * v[i];
        for (int i = 0; i < m; ++i) {
            double *row = &A[(size_t)(k + 1 + i) * n + (k + 1)];
            for (int j = 0; j < m; ++j) row[j] -= v[i] * q[j] + q[i] * v[j];
        }
        A[(size_t)(k + 1) * n + k] = alpha;
        A[(size_t)k * n + (k + 1)] = alpha;
        for (int i = 1; i < m; ++i) {
            A[(size_t)(k + 1 + i) * n + k] = 0.0;
            A[(size_t)k * n + (k + 1 + i)] = 0.0;
        }
        // Z <- Z H on columns k+1..n-1
        for (int r = 0; r < n; ++r) {
            double *zr = &Z[(size_t)r * n + (k + 1)];
            double s = 0.0;
            for (int j = 0; j < m; ++j) s += zr[j] * v[j];
            s *= beta;
            for (int j = 0; j < m; ++j) zr[j] -= s * v[j];
        }
    }
    d.resize(n);
    e.assign(n > 1 ? n - 1 : 0, 0.0);
    for (int i = 0; i < n; ++i) d[i] = A[(size_t)i * n + i];
    for (int i = 0; i + 1 < n; ++i) e[i] = A[(size_t)(i + 1) * n + i];
}

// Implicit symmetric QR on the tridiagonal (d, e), accumulating rotations into the columns of Z,
// held transposed (Zt[col][row]) so that each rotation updates two contiguous vectors.
bool tridiag_qr(int n, std::vector<double> &d, std::vector<double> &e, std::vector<double> &Zt) {
    if (n <= 1) return true;
    const double eps = 2.220446049250313e-16;
    double anorm = 0.0;
    for (int i = 0; i < n; ++i) anorm = std::fmax(anorm, std::fabs(d[i]) + (i < n - 1 ? std::fabs(e[i]) : 0.0) + (i > 0 ? std::fabs(e[i - 1]) : 0.0));
    const double floor_abs = anorm * 1e-30;
    int iter = 0;
    const int max_iter = 60 * n;
    int hi = n - 1;
    while (hi > 0) {
        // deflate negligible off-diagonals
        for (int i = 0; i < hi; ++i)
            if (std::fabs(e[i]) <= eps * (std::fabs(d[i]) + std::fabs(d[i + 1])) || std::fabs(e[i]) <= floor_abs)
                e[i] = 0.0;
        while (hi > 0 && e[hi - 1] == 0.0) --hi;
        if (hi == 0) break;
        int lo = hi - 1;
        while (lo > 0 && e[lo - 1] != 0.0) --lo;
        if (++iter > max_iter) return false;
        // Wilkinson shift from the trailing 2x2 of the unreduced block [lo, hi]
        const double delta = 0.5 * (d[hi - 1] - d[hi]);
        const double b2 = e[hi - 1] * e[hi - 1];
        const double den = delta + (delta >= 0 ? 1.0 : -1.0) * std::hypot(delta, e[hi - 1]);
        const double mu = (den != 0.0) ? d[hi] - b2 / den : d[hi] - std::fabs(e[hi - 1]);
        double x = d[lo] - mu, z = e[lo];
        double bulge = 0.0;
        for (int k = lo; k < hi; ++k) {
            if (k > lo) { x = e[k - 1]; z = bulge; }
            const double r = std::hypot(x, z);
            double c = 1.0, s = 0.0;
            if (r != 0.0) { c = x / r; s = -z / r; }
            if (k > lo) e[k - 1] = r;
            const double ak = d[k], ak1 = d[k + 1], bk = e[k];
            d[k] = c * c * ak - 2.0 * c * s * bk + s * s * ak1;
            d[k + 1] = s * s * ak + 2.0 * c * s * bk + c * c * ak1;
            e[k] = c * s * (ak - ak1) + (c * c - s * s) * bk;
            if (k + 1 < hi) {
                bulge = -s * e[k + 1];
                e[k + 1] = c * e[k + 1];
            }
            double *__restrict__ zk = &Zt[(size_t)k * n];
            double *__restrict__ zk1 = &Zt[(size_t)(k + 1) * n];
            for (int row = 0; row < n; ++row) {
                const double a = zk[row], b = zk1[row];
                zk[row] = c * a - s * b;
                zk1[row] = s * a + c * b;
            }
        }
    }
    return true;
}

}  // namespace

extern "C" rsvd_status rsvd_eigen_basis(const double *C, int32_t R, int32_t H, double *U, double *lambda) {
    using rsvd::fail;
    if (R <= 0 || R > 256) return fail(RSVD_ERR_UNSUPPORTED, "R must be in [1, 256]");
    if (H < 1 || H > R) return fail(RSVD_ERR_UNSUPPORTED, "H must satisfy 1 <= H <= R");
    if (!C || !U) return fail(RSVD_ERR_ARG, "NULL pointer");
    const int n = R;
    std::vector<double> A((size_t)n * n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const double a = C[(size_t)i * n + j], b = C[(size_t)j * n + i];
            if (!std::isfinite(a)) return fail(RSVD_ERR_NUMERIC, "kernel matrix has non-finite entries");
            A[(size_t)i * n + j] = 0.5 * (a + b);
        }
    std::vector<double> Z, d, e;
    householder_tridiag(n, A, Z, d, e);
    std::vector<double> Zt((size_t)n * n);
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) Zt[(size_t)c * n + r] = Z[(size_t)r * n + c];
    if (!tridiag_qr(n, d, e, Zt)) return fail(RSVD_ERR_NUMERIC, "eigen-solver did not converge");
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    // stable descending sort (insertion sort: n <= 256, deterministic)
    for (int i = 1; i < n; ++i) {
        const int v = order[i];
        int j = i - 1;
        while (j >= 0 && d[order[j]] < d[v]) { order[j + 1] = order[j]; --j; }
        order[j + 1] = v;
    }
    for (int h = 0; h < H; ++h) {
        const int col = order[h];
        double nrm = 0.0;
        int imax = 0;
        double amax = -1.0;
        for (int r = 0; r < n; ++r) {
            const double z = Zt[(size_t)col * n + r];
            nrm += z * z;
            if (std::fabs(z) > amax) { amax = std::fabs(z); imax = r; }
        }
        nrm = std::sqrt(nrm);
        const double sgn = (Zt[(size_t)col * n + imax] < 0) ? -1.0 : 1.0;
        for (int r = 0; r < n; ++r) U[(size_t)r * H + h] = sgn * Zt[(size_t)col * n + r] / nrm;
    }
    if (lambda)
        for (int i = 0; i < n; ++i) lambda[i] = d[order[i]];
    return RSVD_OK;
}

// Row f3 (per-CTF-group bases): targets of CTF group g are the templates multiplied
// ring by ring by a radial CTF c_g(k_r), so that group's kernel is D C D with D = diag(c_g) (C the
// kernel of the raw templates: every term of C is bilinear in one ring r and one ring r').  U is the
// basis of D C D (for the group's images); U_tmpl = D U compresses the RAW templates into the
// group's CTF-corrected targets (the projection sum_r U[r,h] sqrt(w_r) c_g(k_r) b[r,j]).
extern "C" rsvd_status rsvd_eigen_basis_ctf(const double *C, int32_t R, const double *ctf, int32_t H, double *U,
                                            double *U_tmpl, double *lambda) {
    using rsvd::fail;
    if (R <= 0 || R > 256) return fail(RSVD_ERR_UNSUPPORTED, "R must be in [1, 256]");
    if (!C || !ctf || !U) return fail(RSVD_ERR_ARG, "NULL pointer");
    std::vector<double> Cg((size_t)R * R);
    for (int r = 0; r < R; ++r) {
        if (!std::isfinite(ctf[r])) return fail(RSVD_ERR_ARG, "CTF values must be finite");
        for (int c = 0; c < R; ++c) Cg[(size_t)r * R + c] = ctf[r] * C[(size_t)r * R + c] * ctf[c];
    }
    const rsvd_status st = rsvd_eigen_basis(Cg.data(), R, H, U, lambda);
    if (st != RSVD_OK) return st;
    if (U_tmpl)
        for (int r = 0; r < R; ++r)
            for (int h = 0; h < H; ++h) U_tmpl[(size_t)r * H + h] = ctf[r] * U[(size_t)r * H + h];
    return RSVD_OK;
}
