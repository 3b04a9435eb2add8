// rsvd_eigen.cpp -- host fp64 symmetric eigen-solver for the R x R kernel matrix C (row a0).
//
// The paper takes "the singular-value-decomposition" of the symmetric PSD kernel C to get the
// principal vectors u_1..u_H; for a symmetric matrix that is its eigen-decomposition
// (reading G7).  R <= 256, so a host solver costs ~ms.
//
// Algorithm: Householder reduction to tridiagonal form with accumulated orthogonal factor, then
// implicit symmetric QR steps with Wilkinson shifts and deflation (the textbook symmetric QR
// algorithm), all in fp64 with a fixed operation order, so the result is deterministic.  For
// H <= R/2 the QR steps run without accumulating vectors and the H leading eigenvectors come from
// inverse iteration on the tridiagonal form (each pair checked by its residual, else the full QR
// path), which drops the O(R^3) rotation updates and the accumulation of the Householder factor.  Output:
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

// A (n x n, row-major, symmetric; only the lower triangle is read after the first step) -> tridiagonal
// (d, e) with A = Z T Z^T, Z = H_0 H_1 ... H_{n-3},
// H_k = I - beta_k v_k v_k^T acting on indices k+1..n-1.  The reflectors are kept in refl (row k:
// v_k at offsets k+1.., beta_k in betas[k], 0 = identity); accumulate_z forms Z from them.
void householder_tridiag(int n, std::vector<double> &A, std::vector<double> &d, std::vector<double> &e,
                         std::vector<double> &refl, std::vector<double> &betas) {
    refl.assign((size_t)n * n, 0.0);
    betas.assign(n, 0.0);
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
        // trailing block B = A[k+1.., k+1..] (only its lower triangle is kept up to date):
        // p = beta B v by the symmetric matvec over row prefixes (a dot and an axpy, both contiguous),
        // then B <- H B H = B - v q^T - q v^T on the lower triangle
        for (int i = 0; i < m; ++i) p[i] = 0.0;
        for (int i = 0; i < m; ++i) {
            const double *row = &A[(size_t)(k + 1 + i) * n + (k + 1)];
            const double vi = v[i];
            // the dot over the row prefix in four interleaved partial sums (fixed order; four
            // independent add chains instead of one), the axpy into p alongside
            double s4[4] = {0.0, 0.0, 0.0, 0.0};
            int j = 0;
            for (; j + 4 <= i; j += 4) {
                for (int u = 0; u < 4; ++u) {
                    s4[u] += row[j + u] * v[j + u];
                    p[j + u] += row[j + u] * vi;
                }
            }
            for (; j < i; ++j) {
                s4[0] += row[j] * v[j];
                p[j] += row[j] * vi;
            }
            p[i] += row[i] * vi + ((s4[0] + s4[1]) + (s4[2] + s4[3]));
        }
        for (int i = 0; i < m; ++i) p[i] *= beta;
        double vp = 0.0;
        for (int i = 0; i < m; ++i) vp += v[i] * p[i];
        const double K = 0.5 * beta * vp;
        for (int i = 0; i < m; ++i) q[i] = p[i] - K * v[i];
        for (int i = 0; i < m; ++i) {
            double *row = &A[(size_t)(k + 1 + i) * n + (k + 1)];
            const double vi = v[i], qi = q[i];
            for (int j = 0; j <= i; ++j) row[j] -= vi * q[j] + qi * v[j];
        }
        A[(size_t)(k + 1) * n + k] = alpha;
        A[(size_t)k * n + (k + 1)] = alpha;
        for (int i = 1; i < m; ++i) {
            A[(size_t)(k + 1 + i) * n + k] = 0.0;
            A[(size_t)k * n + (k + 1 + i)] = 0.0;
        }
        betas[k] = beta;
        for (int j = 0; j < m; ++j) refl[(size_t)k * n + k + 1 + j] = v[j];
    }
    d.resize(n);
    e.assign(n > 1 ? n - 1 : 0, 0.0);
    for (int i = 0; i < n; ++i) d[i] = A[(size_t)i * n + i];
    for (int i = 0; i + 1 < n; ++i) e[i] = A[(size_t)(i + 1) * n + i];
}

// Z = H_0 H_1 ... H_{n-3} (Z <- Z H_k on columns k+1..n-1, k ascending)
void accumulate_z(int n, const std::vector<double> &refl, const std::vector<double> &betas, std::vector<double> &Z) {
    Z.assign((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) Z[(size_t)i * n + i] = 1.0;
    for (int k = 0; k + 2 < n; ++k) {
        if (betas[k] == 0.0) continue;
        const int m = n - k - 1;
        const double *vk = &refl[(size_t)k * n + k + 1];
        for (int r = 0; r < n; ++r) {
            double *zr = &Z[(size_t)r * n + (k + 1)];
            double s = 0.0;
            for (int j = 0; j < m; ++j) s += zr[j] * vk[j];
            s *= betas[k];
            for (int j = 0; j < m; ++j) zr[j] -= s * vk[j];
        }
    }
}

// Implicit symmetric QR on the tridiagonal (d, e), accumulating rotations into the columns of Z,
// held transposed (Zt[col][row]) so that each rotation updates two contiguous vectors.
bool tridiag_qr(int n, std::vector<double> &d, std::vector<double> &e, std::vector<double> *Zt) {
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
            if (!Zt) continue;                   // eigenvalues only
            double *__restrict__ zk = &(*Zt)[(size_t)k * n];
            double *__restrict__ zk1 = &(*Zt)[(size_t)(k + 1) * n];
            for (int row = 0; row < n; ++row) {
                const double a = zk[row], b = zk1[row];
                zk[row] = c * a - s * b;
                zk1[row] = s * a + c * b;
            }
        }
    }
    return true;
}


// Top-H eigenvectors of the tridiagonal T = (d, e) by inverse iteration (tridiagonal LU with partial
// pivoting, fixed start vector, 3 steps) with modified Gram-Schmidt against the vectors already found
// (which keeps clusters -- e.g. the numerical null space of a low-rank kernel -- orthonormal), then
// back-transformed with the Householder reflectors.  Every pair is checked a posteriori:
// ||T y - lambda y|| <= 64 n eps ||T||, else false and the caller runs the QR algorithm with
// accumulated vectors.
bool top_vectors_inverse_iteration(int n, const std::vector<double> &d, const std::vector<double> &e,
                                   const std::vector<double> &lam_sorted, int H, const std::vector<double> &refl,
                                   const std::vector<double> &betas, std::vector<double> &V /* [H][n] */) {
    const double eps = 2.220446049250313e-16;
    double tnorm = 0.0;
    for (int i = 0; i < n; ++i) tnorm = std::fmax(tnorm, std::fabs(d[i]) + (i < n - 1 ? std::fabs(e[i]) : 0.0) + (i > 0 ? std::fabs(e[i - 1]) : 0.0));
    std::vector<double> Y((size_t)H * n);
    std::vector<double> a(n), b(n), c(n), c2(n), x(n);
    std::vector<char> swp(n);
    for (int h = 0; h < H; ++h) {
        const double sigma = lam_sorted[h];
        // LU of T - sigma I with partial pivoting: rows hold (a_i, b_i, c2_i) = (diag, super, super^2)
        for (int i = 0; i < n; ++i) { a[i] = d[i] - sigma; b[i] = i + 1 < n ? e[i] : 0.0; c2[i] = 0.0; }
        for (int i = 0; i + 1 < n; ++i) {
            const double sub = e[i];
            if (std::fabs(sub) > std::fabs(a[i])) {          // swap rows i and i+1
                swp[i] = 1;
                const double na = sub, nb = a[i + 1], nc = i + 2 < n ? e[i + 1] : 0.0;
                const double m = a[i] / sub;
                const double oa1 = b[i], oc = c2[i];
                a[i] = na; b[i] = nb; c2[i] = nc;
                c[i] = m;
                a[i + 1] = oa1 - m * nb;
                b[i + 1] = oc - m * nc;
            } else {
                swp[i] = 0;
                const double m = a[i] != 0.0 ? sub / a[i] : 0.0;
                c[i] = m;
                a[i + 1] -= m * b[i];
            }
        }
        for (int i = 0; i < n; ++i)
            if (std::fabs(a[i]) < eps * tnorm) a[i] = (a[i] < 0 ? -1.0 : 1.0) * eps * tnorm;
        for (int i = 0; i < n; ++i) x[i] = 1.0 + 1e-3 * (double)((i * 7 + h * 3) % 11);
        for (int it = 0; it < 3; ++it) {
            for (int i = 0; i + 1 < n; ++i) {                 // forward: apply L^{-1} P
                if (swp[i]) { const double t = x[i]; x[i] = x[i + 1]; x[i + 1] = t; }
                x[i + 1] -= c[i] * x[i];
            }
            for (int i = n - 1; i >= 0; --i) {                // back: U^{-1}
                double v = x[i];
                if (i + 1 < n) v -= b[i] * x[i + 1];
                if (i + 2 < n) v -= c2[i] * x[i + 2];
                x[i] = v / a[i];
            }
            for (int g = 0; g < h; ++g) {                     // modified Gram-Schmidt
                const double *y = &Y[(size_t)g * n];
                double dot = 0.0;
                for (int i = 0; i < n; ++i) dot += y[i] * x[i];
                for (int i = 0; i < n; ++i) x[i] -= dot * y[i];
            }
            double nrm = 0.0;
            for (int i = 0; i < n; ++i) nrm += x[i] * x[i];
            nrm = std::sqrt(nrm);
            if (!(nrm > 0.0) || !std::isfinite(nrm)) return false;
            for (int i = 0; i < n; ++i) x[i] /= nrm;
        }
        double r2 = 0.0;                                      // a-posteriori residual on T
        for (int i = 0; i < n; ++i) {
            double t = d[i] * x[i] - sigma * x[i];
            if (i > 0) t += e[i - 1] * x[i - 1];
            if (i + 1 < n) t += e[i] * x[i + 1];
            r2 += t * t;
        }
        if (!(std::sqrt(r2) <= 64.0 * n * eps * tnorm)) return false;
        std::copy(x.begin(), x.end(), Y.begin() + (size_t)h * n);
    }
    // back-transform: v_h = Z y_h = H_0 (H_1 (... (H_{n-3} y_h)))
    V = Y;
    for (int h = 0; h < H; ++h) {
        double *v = &V[(size_t)h * n];
        for (int k = n - 3; k >= 0; --k) {
            if (betas[k] == 0.0) continue;
            const double *vk = &refl[(size_t)k * n];
            double s4[4] = {0.0, 0.0, 0.0, 0.0};                // four interleaved partial sums
            int j = k + 1;
            for (; j + 4 <= n; j += 4)
                for (int u = 0; u < 4; ++u) s4[u] += vk[j + u] * v[j + u];
            for (; j < n; ++j) s4[0] += vk[j] * v[j];
            const double s = ((s4[0] + s4[1]) + (s4[2] + s4[3])) * betas[k];
            for (int j = k + 1; j < n; ++j) v[j] -= s * vk[j];
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
    std::vector<double> Z, d, e, refl, betas;
    const bool fast = 2 * H <= n;
    householder_tridiag(n, A, d, e, refl, betas);
    auto emit = [&](const double *vec, int h) {      // normalise + sign rule into column h of U
        double nrm = 0.0, amax = -1.0;
        int imax = 0;
        for (int r = 0; r < n; ++r) {
            nrm += vec[r] * vec[r];
            if (std::fabs(vec[r]) > amax) { amax = std::fabs(vec[r]); imax = r; }
        }
        nrm = std::sqrt(nrm);
        const double sgn = (vec[imax] < 0) ? -1.0 : 1.0;
        for (int r = 0; r < n; ++r) U[(size_t)r * H + h] = sgn * vec[r] / nrm;
    };
    if (fast) {
        // top-H fast path: eigenvalues by QR without vectors (the same d/e arithmetic as below, so
        // bitwise the same eigenvalues), vectors by inverse iteration when they are well separated
        std::vector<double> d2 = d, e2 = e;
        if (!tridiag_qr(n, d2, e2, nullptr)) return fail(RSVD_ERR_NUMERIC, "eigen-solver did not converge");
        std::vector<double> ls = d2;
        for (int i = 1; i < n; ++i) {                 // stable descending insertion sort
            const double v = ls[i];
            int j = i - 1;
            while (j >= 0 && ls[j] < v) { ls[j + 1] = ls[j]; --j; }
            ls[j + 1] = v;
        }
        std::vector<double> V;
        if (top_vectors_inverse_iteration(n, d, e, ls, H, refl, betas, V)) {
            for (int h = 0; h < H; ++h) emit(&V[(size_t)h * n], h);
            if (lambda)
                for (int i = 0; i < n; ++i) lambda[i] = ls[i];
            return RSVD_OK;
        }
    }
    accumulate_z(n, refl, betas, Z);
    std::vector<double> Zt((size_t)n * n);
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) Zt[(size_t)c * n + r] = Z[(size_t)r * n + c];
    if (!tridiag_qr(n, d, e, &Zt)) return fail(RSVD_ERR_NUMERIC, "eigen-solver did not converge");
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    // stable descending sort (insertion sort: n <= 256, deterministic)
    for (int i = 1; i < n; ++i) {
        const int v = order[i];
        int j = i - 1;
        while (j >= 0 && d[order[j]] < d[v]) { order[j + 1] = order[j]; --j; }
        order[j + 1] = v;
    }
    for (int h = 0; h < H; ++h) emit(&Zt[(size_t)order[h] * n], h);
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
