/* rsvd.h -- C ABI of the B200 radial-SVD rotational-alignment library (librsvd.so).
 *
 * Method: A. Rangan, "Radial-recombination for rigid rotational alignment of images and volumes"
 * (arXiv 2202.07235).  Citations "PAPER.md:L" refer to lines of that paper's LaTeX source.
 *
 * The library computes, for every (image m, template t) pair of polar-Fourier images sampled on a
 * shared grid of R rings (radial nodes k_r, weights w_r) x Q equispaced angles psi_j = 2 pi j / Q,
 * the rank-H landscape of inner products over the rotation angles gamma_k = 2 pi k / Q,
 *
 *   Re X(gamma_k) = Re[ 2 pi sum_q e^{-2 pi i q k / Q} sum_{h<H} conj(A_q[m,h]) B_q[t,h] ]
 *                                                       (Eq. image_innerproduct_pm)
 *
 * with A_q[m,h] = sum_r U[r,h] sqrt(w_r) ahat_m[r,q] and ahat = (1/Q) DFT over psi (PAPER.md:240-244,
 * principal image rings PAPER.md:580-585; readings G1/G2), and its per-pair or per-image
 * maximum over gamma (the maximum-likelihood alignment).  At H = R and any
 * orthogonal U this equals sum_r w_r dpsi sum_j Re(conj(a[r,j]) b[r,(j-k) mod Q]).
 *
 * Conventions (all entry points):
 *  - Device pointers are CUDA device memory owned by the caller; host pointers are marked (host).
 *  - Complex data is interleaved float32 (re, im) = 8-byte elements; complex buffers must be 16-byte
 *    aligned.  Rings are [n][R][Q] row-major, angle fastest.
 *  - Every call returns rsvd_status; no C++ exception crosses the ABI.  Arguments are validated
 *    before any launch; on a non-OK return no work was enqueued and rsvd_last_error() (thread-local)
 *    holds a message.  Launch failures return RSVD_ERR_CUDA; asynchronous device faults surface on
 *    a later call or stream synchronisation.
 *  - All device work is enqueued on `stream` (NULL = legacy default stream).  Only
 *    rsvd_build_basis synchronises (it returns host outputs).  Calls are reentrant across streams.
 *  - The align path allocates no memory: the caller passes a workspace.  rsvd_build_basis allocates
 *    scratch with cudaMallocAsync on `stream` and frees it before returning.
 *  - Supported sizes: Q a power of two in [32, 1024]; 1 <= H <= R <= 256.  Sizes of 0 rows/templates
 *    are valid empty problems (no work, RSVD_OK).  Negative sizes, NULL or misaligned pointers and
 *    non-finite or non-positive weights are RSVD_ERR_ARG; unsupported Q/R/H are RSVD_ERR_UNSUPPORTED.
 */
#ifndef RSVD_H
#define RSVD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *rsvd_stream_t; /* == cudaStream_t */

typedef enum {
    RSVD_OK = 0,
    RSVD_ERR_ARG = 1,          /* bad size, NULL / misaligned pointer, non-finite weight   */
    RSVD_ERR_UNSUPPORTED = 2,  /* Q not a power of two in [32,1024], R > 256, H > R, ...  */
    RSVD_ERR_CUDA = 3,         /* a CUDA runtime call or launch failed                     */
    RSVD_ERR_NUMERIC = 4       /* non-finite kernel matrix or eigen-solver non-convergence */
} rsvd_status;

typedef enum { RSVD_SIDE_IMAGE = 0, RSVD_SIDE_TEMPLATE = 1 } rsvd_side;
typedef enum { RSVD_PER_PAIR = 0, RSVD_PER_IMAGE = 1 } rsvd_reduce;

/* Thread-local message describing the last non-OK status returned on this thread. */
const char *rsvd_last_error(void);
/* ABI version of this header (bumped when a signature or the block layout changes): 6 (5 adds the
 * f4 volume entry points of rsvd_vol.h, 6 rsvd_kernel_translated_sh). */
int32_t rsvd_abi_version(void);

/* ------------------------------------------------------------------ sizes */
/* Bytes of one compressed block buffer holding `rows` images (side IMAGE) or templates (side
 * TEMPLATE) at (Q, H).  The layout is opaque (it depends on the contraction path, see
 * rsvd_path_for); read it back only through rsvd_blocks_unpack. */
int64_t rsvd_block_bytes(int64_t rows, int32_t Q, int32_t H, rsvd_side side);
/* Contraction path used for (Q, H): 1 = FP32 SIMT, 2 = tcgen05 tensor cores on CTA pairs with an
 * fp16 hi/lo split of both (power-of-two row-scaled) operands, 3 MMAs per product, fp32
 * accumulation (~fp32 accuracy, same 1e-5 gate as the SIMT path).  Default (AUTO): tensor cores whenever a row's H x Q coefficient
 * block fits in shared memory (H * Q <= 24576), else SIMT.  rsvd_set_path(0 auto | 1 simt | 2 tc)
 * overrides it process-wide (also env RSVD_PATH=auto|simt|tc); blocks must be produced and consumed
 * under the same path. */
int32_t rsvd_path_for(int32_t Q, int32_t H);
void rsvd_set_path(int32_t path);
/* Templates per fixed chunk of the kernel-matrix partial sums (rsvd_kernel_partials). */
int64_t rsvd_kernel_chunk(void);
/* Bytes of the partial-sum buffer for T templates with R rings: ceil(T/chunk) * R * R doubles. */
int64_t rsvd_kernel_partials_bytes(int64_t T, int32_t R);
/* Recommended align workspace bytes for an M x T problem (chunk of the per-pair spectra, sized to
 * stay resident in L2).  Any size >= rsvd_align_min_workspace_bytes(Q) works. */
int64_t rsvd_align_workspace_bytes(int64_t M, int64_t T, int32_t Q, int32_t H);
int64_t rsvd_align_min_workspace_bytes(int32_t Q);

/* ------------------------------------------------------------------ row a0: basis (precompute)
 * Kernel matrix (Eq. Image_simple_kern PAPER.md:661-665 averaged over targets, Eq.
 * image_cost_and_kern :704-708, constants dropped, real part; G6):
 *   C[r][r'] = (1/(T Q)) sqrt(w_r w_r') sum_t Re sum_j W_t[r,j] conj(W_t[r',j]),
 *   W_t[r,j] = b_t[r,j] - (1/Q) sum_j' b_t[r,j']     (angular mean removed == q = 0 excluded)
 * and its eigen-decomposition C = V diag(lambda) V^T, lambda descending (the paper's "SVD of C",
 * :667).  U = first H columns of V.  Sign rule: the largest-|.| entry of each column is positive.
 *
 * rsvd_kernel_partials: device, deterministic.  For each fixed chunk c of rsvd_kernel_chunk()
 *   consecutive templates (the last may be short) writes the un-normalised, unweighted partial
 *   P_c[r][r'] = sum_{t in c} Re( sum_j b_t[r,j] conj(b_t[r',j]) - (1/Q) S_t[r] conj(S_t[r']) ),
 *   S_t[r] = sum_j b_t[r,j], in fp64 to partials [ceil(T/chunk)][R][R] (device).  P_c is symmetric and
 *   only its lower triangle (entries r >= r') is written; the upper-triangle entries of the buffer are
 *   left as the caller allocated them (rsvd_kernel_reduce reads the lower triangle only).  A rank holding
 *   templates [t0, t0+T) with t0 % chunk == 0 produces exactly the global chunks t0/chunk... so that
 *   the concatenation over ranks is independent of the sharding.
 * rsvd_kernel_reduce: device.  Sums partials[0..nchunks) in a fixed tree over the chunk index (chunk c into
 *   partial sum c mod 8 in ascending c, then the 8 partial sums in order; fixed order => bitwise
 *   identical for any sharding) and writes C (device fp64 [R][R], exactly symmetric) using the
 *   device weights w[R] and the global template count T_total.
 * rsvd_eigen_basis: host only.  Householder tridiagonalisation + implicit QL/QR with Wilkinson
 *   shifts, fp64, deterministic; for H <= R/2 the H leading vectors come from inverse iteration on the
 *   tridiagonal form (residual-checked, else the full QR path).  U (host [R][H] row-major), lambda
 *   (host [R], may be NULL).
 * rsvd_build_basis: single-device convenience = partials + reduce + D2H + eigen.  Synchronises. */
rsvd_status rsvd_kernel_partials(const void *templates, int64_t T, int32_t R, int32_t Q,
                                 double *partials, rsvd_stream_t stream);
rsvd_status rsvd_kernel_reduce(const double *partials, int64_t nchunks, int32_t R, int64_t T_total,
                               int32_t Q, const double *w, double *C, rsvd_stream_t stream);
rsvd_status rsvd_eigen_basis(const double *C, int32_t R, int32_t H, double *U, double *lambda);

/* rsvd_eigen_basis_device: the same eigenbasis computed on the device (one CTA, C in shared memory), so
 *   a step needs no host round trip between the kernel matrix and Step 1 (DESIGN.md
 *   reading G7).  C: device fp64 [R][R] (symmetrised as (C + C^T)/2); U: device fp64 [R][H] row-major;
 *   lambda (may be NULL): device fp64 [R], descending; info: device int32, set to 0 on success or 1 when
 *   an eigenvector fails the a-posteriori residual test ||T y - lambda y|| <= 64 R eps ||T|| (U is then
 *   unusable; run rsvd_eigen_basis on the same C).  Householder tridiagonalisation, bisection on the
 *   Sturm count for every eigenvalue, inverse iteration with Gram-Schmidt for the top H vectors,
 *   back-transform; fixed reduction orders (bitwise reproducible).  Eigenvalues agree with
 *   rsvd_eigen_basis to O(eps ||C||), vectors with the same sign rule.  R <= 128, H * R <= 8192, else
 *   RSVD_ERR_UNSUPPORTED.  Asynchronous on `stream`. */
rsvd_status rsvd_eigen_basis_device(const double *C, int32_t R, int32_t H, double *U, double *lambda,
                                    int32_t *info, rsvd_stream_t stream);
/* Row f3 (per-CTF-group bases; PAPER.md:715-724 builds one kernel and basis per CTF): host only.
 * For targets = templates multiplied ring by ring by a radial CTF ctf[r] = c_g(k_r), the group's
 * kernel is diag(ctf) C diag(ctf) with C the raw templates' kernel (rsvd_kernel_reduce output
 * copied to the host), so one kernel-partials pass serves every group.  U (host [R][H]): the group
 * basis, used to compress the group's images; U_tmpl (host [R][H], may be NULL) = diag(ctf) U:
 * compressing the RAW templates with it yields the group's CTF-corrected targets.  Same
 * eigen-solver, ordering, sign rule and errors as rsvd_eigen_basis; non-finite ctf is RSVD_ERR_ARG. */
rsvd_status rsvd_eigen_basis_ctf(const double *C, int32_t R, const double *ctf, int32_t H, double *U,
                                 double *U_tmpl, double *lambda);
rsvd_status rsvd_build_basis(const void *templates, int64_t T, int32_t R, int32_t Q,
                             const double *w_host, int32_t H, double *U_host, double *lambda_host,
                             rsvd_stream_t stream);

/* ------------------------------------------------------------------ row a1: compress (Step 1)
 * For each row (image if side == RSVD_SIDE_IMAGE, template otherwise) computes the H principal
 * image rings' Fourier-Bessel coefficients
 *   A_q[n,h] = (1/Q) sum_j e^{-2 pi i q j/Q} sum_r U[r,h] sqrt(w_r) a_n[r,j]   (q = 0..Q-1)
 * (PAPER.md:580-585 with eta_r = sqrt(w_r), reading G2; projection in psi-space then the length-Q
 * DFT -- the two linear maps commute) and stores them, fp32, in the opaque block layout of `side`.
 *   rings:  device [n][R][Q] complex64;  w: device fp64 [R];  U: device fp64 [R][H] row-major
 *   blocks: device, rsvd_block_bytes(n, Q, H) bytes, 16-byte aligned; fully overwritten.
 * rsvd_blocks_unpack (test/debug): reads blocks back as canonical coefficients
 *   coeffs: device [n][Q][H] complex64, coeffs[n][q][h] = A_q[n,h]. */
rsvd_status rsvd_compress(const void *rings, int64_t n, int32_t R, int32_t Q, const double *w,
                          const double *U, int32_t H, rsvd_side side, void *blocks,
                          rsvd_stream_t stream);
rsvd_status rsvd_blocks_unpack(const void *blocks, int64_t n, int32_t Q, int32_t H, rsvd_side side,
                               void *coeffs, rsvd_stream_t stream);

/* ------------------------------------------------------------------ row f2: translations (NEXT)
 * Translations inside the method (PAPER.md:37-39 defers them; configs "Translations"): compresses S
 * translated copies of each base row without materialising them.  Output row b*S + s is the row
 * rsvd_compress would produce from
 *   a_s[r][j] = a_b[r][j] exp(-i k_r (dx_s cos psi_j + dy_s sin psi_j))
 * (the Fourier shift theorem with the transform convention of PAPER.md:80; reading G15):
 *   rings: device [n_base][R][Q] complex64;  k: device fp64 [R] radial wavenumbers k_r;
 *   shifts: device fp64 [S][2] (dx_s, dy_s) in the units of 1/k;  w, U as for rsvd_compress;
 *   blocks: device, rsvd_block_bytes(n_base * S, Q, H, side) bytes.  Each base ring is read once
 *   from HBM (its S copies are built in registers); the ramp is evaluated in fp32 (|k d| <= ~2 rad
 *   on the configs: phase error ~1e-7).  S >= 1; NULL k / shifts with n_base > 0 are RSVD_ERR_ARG. */
/* rsvd_build_basis_translated: as rsvd_build_basis, for the translation-averaged objective of
 * Eq. eq_Image_single_cost_with_translations with a discrete distribution of S
 * equally weighted shifts: C is averaged over the T x S translated templates (each angularly
 * centred), C = (1/(T S Q)) sqrt(w w') sum_{t,s} Re sum_j W_ts W_ts^H (the exact finite-sum kernel;
 * the paper's closed form for a Gaussian shift distribution, :1152-1166, is rsvd_kernel_translated_sh,
 * which needs the volume's spherical-harmonic coefficients instead of templates).  Host inputs: w, k
 * [R] fp64 (weights, radial wavenumbers), shifts [S][2] fp64 (dx, dy).  The ramps are built in fp64
 * on the device.  Synchronises; allocates scratch (S*R*Q complex fp64 + partials). */
rsvd_status rsvd_build_basis_translated(const void *templates, int64_t T, int32_t R, int32_t Q,
                                        const double *w_host, const double *k_host,
                                        const double *shifts_host, int32_t S, int32_t H,
                                        double *U_host, double *lambda_host, rsvd_stream_t stream);
/* rsvd_kernel_translated_sh: the closed-form kernel of Eq. template_cost_with_translations
 * -- targets = projections of one volume at uniformly distributed views, shifted
 * by an isotropic Gaussian translation of standard deviation sigma (per axis) -- from the volume's
 * spherical-harmonic coefficients:
 *   C[r][r'] = sqrt(w_r w_r') Re[ (sum_{l,m} conj(B_l^m(k_r)) B_l^m(k_r')) E+(k_r, k_r')
 *                                 - conj(B_0^0(k_r)) B_0^0(k_r') E-(k_r) E-(k_r') ],
 *   E+ = exp(-sigma^2 (k_r - k_r')^2 / 2) (= the printed product form),
 *   E- = exp(-k^2 sigma^2 / 2) (= the printed Bessel form, I_{-1/2} - I_{1/2} in closed form),
 * up to the paper's constant factor (the same C the paper's Rayleigh quotient uses; DESIGN.md reading
 * T1: the printed mean term keeps l = 0 only, an approximation of the view average).  Feed C to
 * rsvd_eigen_basis for U.  Bsh: device complex128 [R][(L+1)^2], index l*l + l + m, 16-B aligned;
 * k, w: device fp64 [R] (radial nodes of the image grid and their weights); C: device fp64 [R][R].
 * sigma >= 0 (0: no translations).  Asynchronous on `stream`; deterministic (fixed reduction order). */
rsvd_status rsvd_kernel_translated_sh(const void *Bsh, int32_t R, int32_t L, const double *k, const double *w,
                                      double sigma, double *C, rsvd_stream_t stream);
rsvd_status rsvd_compress_translated(const void *rings, int64_t n_base, int32_t R, int32_t Q,
                                     const double *w, const double *k, const double *U, int32_t H,
                                     const double *shifts, int32_t S, rsvd_side side, void *blocks,
                                     rsvd_stream_t stream);

/* ------------------------------------------------------------------ numeric precision of the TC path
 * rsvd_set_precision(0) (default, also RSVD_PRECISION unset): the fp32-grade path -- every product on
 *   the tensor cores is the error-compensated fp16 hi/lo split (3 MMAs) and the spectrum between Steps
 *   2 and 3 is fp32; landscapes within 1e-5 max|X| of the fp64 oracle (north_star's FP32 gate).
 * rsvd_set_precision(1) (or RSVD_PRECISION=fast): the single-pass tensor-core path north_star allows
 *   for "any TF32/BF16 tensor-core path" -- one fp16 MMA per product (hi x hi, row-scaled fp16
 *   operands) and an fp16 spectrum (accumulators x 2^-20), half the spectrum bytes; landscapes within
 *   2e-3 max|X|.  Applies to rsvd_align_argmax / _landscape / _grouped on the TC layout at Q_out == Q
 *   (Q <= 512); other calls keep the fp32-grade path.  Process-global, like rsvd_set_path.
 * rsvd_precision: the current setting. */
void rsvd_set_precision(int32_t precision);
int32_t rsvd_precision(void);

/* Step 1 kernel choice on the TC layout (row a1).  mode 1 (default, also
 * RSVD_COMPRESS_MMA unset): the tensor-core projection (compress_mma_kernel: tcgen05 kind::tf32 with a
 * three-term split, ~fp32 accuracy) where the shape fits (2Q >= 256, H <= 32, 4 | H when H > 8,
 * R <= 256, un-translated rows) and measurement says it is faster (H > 16, or H = 16 at Q <= 256);
 * mode 2: that kernel wherever the shape fits; mode 0: always the FFMA2 projection (compress_tc_kernel).
 * Both write the same operand layout to the same accuracy gate.  Process-global; no error return.
 * rsvd_compress_mma_mode: the current mode. */
void rsvd_set_compress_mma(int32_t mode);
int32_t rsvd_compress_mma_mode(void);

/* ------------------------------------------------------------------ rows a2-a4: align
 * Step 2: S_q[m,t] = sum_h conj(A_q[m,h]) B_q[t,h] for all q;
 * Step 3: X_k = 2 pi sum_q e^{-2 pi i q k/Q} S_q, k = 0..Q-1 (forward sign, G3);
 * Step 4: the score is Re X_k (G5).
 * img_blocks from rsvd_compress(side=IMAGE, n=M), tmpl_blocks from rsvd_compress(side=TEMPLATE, n=T).
 * work: device scratch of work_bytes >= rsvd_align_min_workspace_bytes(Q), 16-byte aligned.
 *
 * rsvd_align_argmax, mode RSVD_PER_PAIR: best_val[m*T + t] = max_k Re X_k, best_k[m*T + t] = the
 *   smallest maximising k (SPEC.md tie rule, G9).  best_key unused (may be NULL).
 * mode RSVD_PER_IMAGE: for each image m, atomically max-accumulates into best_key[m] the packed key
 *   (ord(max Re X) << 32) | (0xFFFFFFFF - ((t_offset + t) * Q + k)), ord = order-preserving map of
 *   float bits, so the maximum key is the largest value with the lexicographically smallest (t, k).
 *   Requires (t_offset + T) * Q < 2^32.  best_key must be initialised by rsvd_winners_reset (it
 *   accumulates over calls, e.g. template batches or shards).  best_val/best_k unused (may be NULL).
 * rsvd_align_landscape: X[m*ld_m + t*ld_t + k] = Re X_k (float32), k contiguous; ld_t >= Q,
 *   ld_m >= T*ld_t not required (caller strides); X 16-byte aligned when ld_t, ld_m are multiples of 4. */
rsvd_status rsvd_align_argmax(const void *img_blocks, int64_t M, const void *tmpl_blocks, int64_t T,
                              int64_t t_offset, int32_t Q, int32_t H, rsvd_reduce mode, void *work,
                              int64_t work_bytes, float *best_val, int32_t *best_k,
                              uint64_t *best_key, rsvd_stream_t stream);
rsvd_status rsvd_align_landscape(const void *img_blocks, int64_t M, const void *tmpl_blocks,
                                 int64_t T, int32_t Q, int32_t H, void *work, int64_t work_bytes,
                                 float *X, int64_t ld_m, int64_t ld_t, rsvd_stream_t stream);

/* ------------------------------------------------------------------ row f3: CTF-grouped align
 * The paper builds "the objective-function and kernel for each CTF separately" over the
 * micrograph groups of its example (:715) and repeats precompute steps 1-3 per CTF (:781).  One call
 * aligns G independent groups g: the group's images (compressed with its basis U_g from
 * rsvd_eigen_basis_ctf) against its CTF-corrected targets (the raw templates compressed with
 * diag(c_g) U_g), with exactly the semantics, outputs and errors of rsvd_align_argmax per group
 * (PER_PAIR: best_val/best_k [M_g][T_g]; PER_IMAGE: best_key [M_g], t_offset per group).  Every group
 * descriptor is validated before any work is enqueued; the groups run back to back on `stream` and
 * share `work`.  groups: HOST array of G descriptors (device pointers inside). */
typedef struct {
    const void *img_blocks;   /* rsvd_compress(side=IMAGE, n=M) with the group's U_g */
    int64_t M;
    const void *tmpl_blocks;  /* rsvd_compress(side=TEMPLATE, n=T) with diag(c_g) U_g */
    int64_t T;
    int64_t t_offset;         /* PER_IMAGE: global index of the group's first template */
    float *best_val;          /* PER_PAIR outputs (device) */
    int32_t *best_k;
    uint64_t *best_key;       /* PER_IMAGE outputs (device, rsvd_winners_reset first) */
} rsvd_align_group;
rsvd_status rsvd_align_argmax_grouped(const rsvd_align_group *groups, int32_t G, int32_t Q, int32_t H,
                                      rsvd_reduce mode, void *work, int64_t work_bytes, rsvd_stream_t stream);

/* ------------------------------------------------------------------ row f1: finer gamma (NEXT)
 * "If a finer resolution in gamma is required then the array [of Fourier coefficients] can be
 * zero-padded prior to the FFT".  Same as rsvd_align_argmax / rsvd_align_landscape
 * but on the grid gamma_k = 2 pi k / Q_out, Q_out = Q * 2^p <= 1024 (Q_out == Q is the plain call):
 *   Re X(gamma) = pi [ U_0 + 2 Re sum_{n=1}^{Q/2-1} e^{-i n gamma} U_n + U_{Q/2} cos(Q gamma / 2) ],
 * U_n = S_n + conj(S_{Q-n}), i.e. the trigonometric interpolant with the Nyquist bin split
 * symmetrically between +-Q/2 (reading G4); it equals the plain landscape at every
 * gamma_{k 2^p}.  Indices k / packed keys / strides refer to the Q_out grid ((t_offset+T)*Q_out < 2^32
 * for PER_IMAGE; ld_t >= Q_out).  work >= rsvd_align_min_workspace_bytes(Q_out).
 * best_gamma (PER_PAIR only, device [M][T] float, may be NULL): 3-point parabolic refinement of the
 *   first argmax k (SPEC.md argmax_refine): gamma = 2 pi (k + d) / Q_out, d = (y_{k-1} - y_{k+1}) /
 *   (2 (y_{k-1} - 2 y_k + y_{k+1})) clamped to [-1/2, 1/2] (0 if the samples are not a strict peak),
 *   neighbours cyclic, gamma in [0, 2 pi).  Non-PER_PAIR with best_gamma != NULL is RSVD_ERR_ARG. */
rsvd_status rsvd_align_argmax_fine(const void *img_blocks, int64_t M, const void *tmpl_blocks,
                                   int64_t T, int64_t t_offset, int32_t Q, int32_t H, int32_t Q_out,
                                   rsvd_reduce mode, void *work, int64_t work_bytes, float *best_val,
                                   int32_t *best_k, uint64_t *best_key, float *best_gamma,
                                   rsvd_stream_t stream);
rsvd_status rsvd_align_landscape_fine(const void *img_blocks, int64_t M, const void *tmpl_blocks,
                                      int64_t T, int32_t Q, int32_t H, int32_t Q_out, void *work,
                                      int64_t work_bytes, float *X, int64_t ld_m, int64_t ld_t,
                                      rsvd_stream_t stream);

/* ------------------------------------------------------------------ per-image winners
 * rsvd_winners_reset: keys[0..M) = 0 (below every real key).
 * rsvd_winners_unpack: (val, t, k) from packed keys; val/t/k device [M].
 * rsvd_combine_winners: keys [G][M] (e.g. after an all-gather of every rank's keys over NVLink);
 *   out = max over G per image (== the lexicographic (value, -t, -k) maximum), written as packed
 *   keys to out_keys (may be NULL) and unpacked to val/t/k (each may be NULL). */
rsvd_status rsvd_winners_reset(uint64_t *keys, int64_t M, rsvd_stream_t stream);
rsvd_status rsvd_winners_unpack(const uint64_t *keys, int64_t M, int32_t Q, float *val, int32_t *t,
                                int32_t *k, rsvd_stream_t stream);
rsvd_status rsvd_combine_winners(const uint64_t *keys, int32_t G, int64_t M, int32_t Q,
                                 uint64_t *out_keys, float *val, int32_t *t, int32_t *k,
                                 rsvd_stream_t stream);

/* ------------------------------------------------------------------ instrumentation
 * rsvd_launch_count: monotonic count of kernels this library has launched in the process.
 * rsvd_timing_enable(1): from now on every contraction / FFT-reduce / compress / kernel-partials
 *   launch is bracketed by CUDA events recorded on its own stream (process-global, thread-safe).
 * rsvd_timing_read: synchronises on the recorded events, returns per-kind total milliseconds and
 *   launch counts (kinds: 0 contraction, 1 fft_reduce, 2 compress, 3 kernel partials, 4 fused align) for the
 *   spans recorded since the previous read, and recycles the events.
 * rsvd_probe_fp32: the measured FP32 peak of the current device (roofline denominator Pi_fp32 of
 *   SURVEY.md 8(d)): one launch of register-only dependency chains on every SM (4 x 256 threads per
 *   SM, 8 chains per thread, `iters` x 32 instructions per chain), timed with CUDA events on `stream`
 *   after a short warm-up launch; synchronises.  kind 0 = FFMA, 1 = FFMA2 (packed fp32x2, sm_100),
 *   2 = FADD2, 3 = DFMA (fp64: the kernel-partials peak, 16 chains per thread), 4 / 5 = fp64 tensor-core
 *   mma.sync m8n8k4 / m16n8k4 (8 accumulator fragments per warp).  *tflops = flops / elapsed (FFMA 2,
 *   FFMA2 4, FADD2 2, DFMA 2 flops per lane and instruction; DMMA 2 M N K per warp instruction).
 *   Not part of the method; allocates a 1 KB scratch buffer. */
int64_t rsvd_launch_count(void);
void rsvd_timing_enable(int32_t on);
rsvd_status rsvd_timing_read(double *ms, int64_t *count, int32_t nkinds);
rsvd_status rsvd_probe_fp32(int32_t kind, int32_t iters, double *tflops, rsvd_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* RSVD_H */
