/* rsvd_vol.h -- C ABI of librsvd, row f4: aligning many volumes to one target with the radial- and
 * degree-SVD (arXiv 2202.07235 §5).  Same library, status codes, stream and
 * error conventions as rsvd.h (which this header includes).
 *
 * Data (all device memory, caller-owned, row-major, little-endian):
 *   coefficients   complex64 [n][R][(L+1)^2]: the spherical-harmonic coefficients A_l^m(k_r) of each
 *                  volume's shells, packed lm = l*l + l + m, -l <= m <= l.
 *   w              fp64 [R]: radial quadrature weights for k^2 dk.
 *   U              fp64 [R][HC] radial principal vectors, V fp64 [L+1][HD] degree principal vectors
 *                  (columns; from rsvd_vol_kernels + rsvd_eigen_basis).
 *   shells         complex64 [n][HC][(L+1)^2]: [u_h^T A]_l^m = sum_r U[r][h] sqrt(w_r) A_l^m(k_r)
 *                  (PAPER.md:921-927 with eta_r = sqrt(w_r)).
 *   Y              complex64 [n][HD][M][M], M = 2L+1: Steps 1 + 1b of Eq. volume_innerproduct_pm
 *                  (PAPER.md:1017-1020), Y_j(m1, m2) at [i][j][m2 + L][m1 + L] (m1 fastest).
 *   T              fp32 [nb][HD][M][M]: [v_j^T d]_{m1 m2}(beta_b) = sum_l V[l][j] d^l_{m1 m2}(beta_b)
 *                   at [b][j][m2 + L][m1 + L] (m1 fastest).
 *   X              fp32 [n][nb][P][P]: Re X(tau) at tau = (gamma_g, beta_b, alpha_a),
 *                  alpha_a = 2 pi a / P, gamma_g = 2 pi g / P, element ((i*nb + b)*P + a)*P + g
 *                  (Step 3; the P-point grid is DESIGN.md reading V1).
 *   best_key       uint64 [n]: per volume max over (b, a, g) of X packed as in rsvd.h (value order in
 *                  the high word, ~flat index in the low word, flat = (b*P + a)*P + g: the smallest
 *                  flat index wins ties); decode with rsvd_winners_unpack(keys, n, P*P, ...) which
 *                  returns t = b and k = a*P + g.  Reset to 0 (rsvd_winners_reset) before the first call.
 * Limits: 1 <= L <= 63 (M <= 127), P a power of two in [32, 128] with P >= M, 1 <= HC <= 32,
 * 1 <= HD <= 32, HD <= L + 1, HC <= R <= 256.  Violations return RSVD_ERR_ARG before any launch.
 */
#ifndef RSVD_VOL_H
#define RSVD_VOL_H

#include "rsvd.h"

#ifdef __cplusplus
extern "C" {
#endif

/* (L+1)^2 coefficients per shell; -1 if L < 0. */
int64_t rsvd_vol_ncoef(int32_t L);

/* Radial and degree kernels of the target(s) (DESIGN.md readings
 * V2/V3), averaged over nB targets, fp64 on the device:
 *   C[r][s] = (1/nB) sum_t sum_{l>=1, m} sqrt(w_r w_s) Re conj(B_t,l^m(k_r)) B_t,l^m(k_s)     [R][R]
 *   D[l][l'] = (1/nB) sum_t sum_r w_r sum_m Re conj(B_t,l^m(k_r)) B_t,l'^m(k_r), l, l' >= 1     [L+1][L+1]
 * (row and column 0 of D are 0).  Either output may be NULL.  Deterministic (fixed summation order). */
rsvd_status rsvd_vol_kernels(const void *B, int64_t nB, int32_t R, int32_t L, const double *w, double *C, double *D,
                             rsvd_stream_t stream);

/* Principal shells of n volumes or targets (fp32 accumulation of U sqrt(w) rounded to
 * fp32).  Items 6/7 of the operation count. */
rsvd_status rsvd_vol_compress(const void *A, int64_t n, int32_t R, int32_t L, const double *w, const double *U,
                              int32_t HC, void *shells, rsvd_stream_t stream);

/* Degree-compressed Wigner-d table T for the nb angles beta[] (fp64 device array): d^l_{m1 m2}(beta) from
 * the closed-form seed at l = max(|m1|, |m2|) and the three-term recurrence in l, accumulated against V in
 * fp64 and rounded to fp32.  A per-target precomputation (item 5). */
rsvd_status rsvd_vol_wigner_table(const double *beta, int32_t nb, int32_t L, const double *V, int32_t HD, float *T,
                                  rsvd_stream_t stream);

/* Steps 1 + 1b for n volumes against one target (items 8/9):
 * Y_j(m1,m2) = sum_{l >= max(|m1|,|m2|)} V[l][j] sum_h conj(sA[l,m1][h]) sB[l,m2][h]; fp32. */
rsvd_status rsvd_vol_degrees(const void *shellsA, int64_t n, const void *shellB, int32_t L, int32_t HC,
                             const double *V, int32_t HD, void *Y, rsvd_stream_t stream);

/* Steps 2 + 3 (+ argmax), items 10/11: per (volume, beta) F = sum_j T[b][.][.][j] Y[i][.][.][j]
 * placed on the P x P order grid (m mod P), 2-D forward DFT sum e^{-i m1 alpha_a} e^{-i m2 gamma_g}, Re; fp32.
 * X (landscape) and/or best_key (argmax, max-merged into the existing keys) may be NULL, not both. */
rsvd_status rsvd_vol_align(const void *Y, int64_t n, const float *T, int32_t nb, int32_t L, int32_t HD, int32_t P,
                           float *X, uint64_t *best_key, rsvd_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* RSVD_VOL_H */
