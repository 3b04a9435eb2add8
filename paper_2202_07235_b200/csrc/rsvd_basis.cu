// rsvd_basis.cu -- row a0: the template kernel matrix C and its eigenbasis (precompute).
//
// C[r][r'] = (1/(T Q)) sqrt(w_r w_r') sum_t Re sum_j W_t[r,j] conj(W_t[r',j]),  W_t = b_t minus its
// angular mean.  This is Eq. Image_simple_kern (q = 0 excluded) averaged over the
// targets as in Eq. image_cost_and_kern, written in psi-space by Parseval
// (sum_{q != 0} conj(xhat_q) yhat_q = (1/Q) sum_j conj(x_j - xbar)(y_j - ybar), xhat = DFT/Q).
// Constants (2 pi)^3 / (4 sigma_hat^2) are dropped (they do not move eigenvectors; reading G6).
//
// Determinism: the per-chunk partials depend only on the chunk's templates and are summed in chunk
// order, so C (and U) are bitwise identical for any sharding of the templates over GPUs.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "rsvd_common.cuh"

namespace rsvd {

#ifndef RSVD_KCHUNK
#define RSVD_KCHUNK 8       // 8: twice the CTAs of 16 for small template shards (G = 8: partials 2.3 -> 1.6 ms)
#endif
constexpr int KCHUNK = RSVD_KCHUNK;   // templates per partial (rsvd_kernel_chunk)
constexpr int BT = 64;         // output tile (rows) of C per CTA
#ifndef RSVD_KP_JB
#define RSVD_KP_JB 16
#endif
#ifndef RSVD_KP_MINB
#define RSVD_KP_MINB 4      // 4 CTAs (16 warps) per SM: 16-sample slabs, 128 registers without spills; measured
                            // 11.4 -> 10.8 ms (3 CTAs), 9.39 -> 9.20 ms (4 CTAs, latency-bound: profiles/r02b_partials_fp64.txt)
#endif
constexpr int JB = RSVD_KP_JB;   // angular samples per smem slab
constexpr int NTHR = 128;
constexpr int KA = 8, KBB = 4; // per-thread register tile: rows ty + 8a (a < 8) x columns tx + 16b (b < 4)

// grid: (ntile, ntile, nchunks), only tiles with ti >= tj.  Thread (ty, tx) owns rows
// r_a = ti*64 + ty + 8a (a < 8) and r'_b = tj*64 + tx + 16b (b < 4): 64 DFMA per 12 shared loads (the
// eight row loads are warp broadcasts), so the fp64 pipe, not shared memory, sets the pace.  Samples are widened to fp64 once,
// when staged in shared memory, so the inner loop is pure DFMA (products of fp32 values are exact in
// fp64; accumulation order is fixed).
// ramp (row f2, may be NULL): [S][R][Q] fp64 complex factors exp(-i k_r (dx_s cos psi_j + dy_s sin psi_j));
// every template then contributes its S translated copies (the discrete translation average of
// Eq. eq_Image_single_cost_with_translations).
__device__ __forceinline__ void kp_cp_async16(void *smem, const void *gmem, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gmem), "r"(valid ? 16 : 0) : "memory");
}
// MMA = true: the Gram on the fp64 tensor cores (mma.sync m8n8k4 .f64; measured 37.1 TF/s on B200 vs
// 34.1 for DFMA, tools/gpu_dmma_probe.sh) -- the product X X^T of the slab's fp64 rows with K = 2 JB reals
// (re, im interleaved, so sum_k X[r][k] X[r'][k] = Re(x_r conj x_r')).  Warp w owns the 32 x 32 block
// (rows 32 (w / 2), columns 32 (w % 2)) of the 64 x 64 tile as 4 x 4 m8n8 accumulators; per k-step of 4
// it loads 4 A and 4 B fragments (8 LDS.64, conflict-free with the 2 JB + 4 double row stride) for 16
// MMAs (4096 FMAs), where the SIMT tile issues 12 loads per 32 DFMAs per thread.
template <bool MMA> struct KpLayout { static constexpr int SJ = MMA ? JB + 2 : JB + 1; };   // double2 per staged row
template <bool MMA>
__global__ void __launch_bounds__(NTHR, RSVD_KP_MINB) kernel_partials_kernel(const float2 *__restrict__ tmpl,
                                                               int64_t T, int R, int Q,
                                                               double *__restrict__ partials,
                                                               const double2 *__restrict__ ramp, int S) {
    const int ti = blockIdx.x, tj = blockIdx.y;
    if (ti < tj) return;
    const int64_t c = blockIdx.z;
    const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;     // ty < 8, tx < 16
    constexpr int SJ = KpLayout<MMA>::SJ;
    extern __shared__ __align__(16) double2 kp_smem[];
    double2 (*xi)[SJ] = reinterpret_cast<double2 (*)[SJ]>(kp_smem);
    // diagonal tiles (ti == tj) multiply the slab by itself: stage it once and alias xj to xi
    const bool diag = ti == tj;
    double2 (*xj)[SJ] = diag ? xi : reinterpret_cast<double2 (*)[SJ]>(kp_smem + BT * SJ);
    __shared__ double si[BT][2], sj[BT][2];       // per-template row sums (re, im)

    // SIMT: acc[a][b] = entry (ty + 8a, tx + 16b).  MMA: acc[a][b][e] = entry
    // (wr + 8a + lane / 4, wc + 8b + 2 (lane % 4) + e) of the m8n8 accumulator fragments.
    constexpr int NA = MMA ? 4 : KA, NB = MMA ? 4 : KBB, NE = MMA ? 2 : 1;
    const int lane = tid & 31, wr = (tid >> 6) * 32, wc = ((tid >> 5) & 1) * 32;
    double acc[NA][NB][NE];
#pragma unroll
    for (int a = 0; a < NA; ++a)
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int e = 0; e < NE; ++e) acc[a][b][e] = 0.0;
    auto row_of = [&](int a) { return MMA ? wr + 8 * a + (lane >> 2) : ty + 8 * a; };
    auto col_of = [&](int b, int e) { return MMA ? wc + 8 * b + 2 * (lane & 3) + e : tx + 16 * b; };

    const int64_t t_begin = c * KCHUNK;
    const int64_t t_end = min(T, t_begin + KCHUNK);
    // slabs k = (translated template ts, samples j0 .. j0 + JB) in order; the raw fp32 samples of slab
    // k + 1 stream into shared memory (cp.async, zero-filled outside the grid) while slab k is
    // multiplied, so the global-load latency hides behind the DFMA loop
    const int nslab_t = (Q + JB - 1) / JB;
    const int64_t ts0 = t_begin * S, nslab = (t_end * S - ts0) * nslab_t;
    float2 *rawi = reinterpret_cast<float2 *>(kp_smem + 2 * BT * SJ);      // [BT][JB]
    float2 *rawj = rawi + BT * JB;
    // cp.async mapping: thread -> 16-B chunk jc of rows rr0 + RSTEP i (no divisions in the slab loop)
    constexpr int CPR = JB / 2, RSTEP = NTHR / CPR, NPASS = BT / RSTEP;
    static_assert(NTHR % CPR == 0 && BT % RSTEP == 0, "cp.async mapping");
    const int jc = tid % CPR, rr0 = tid / CPR;
    auto issue = [&](int64_t t, int j0) {
        const float2 *bt = tmpl + t * (int64_t)R * Q;
        const int j = j0 + 2 * jc;
#pragma unroll
        for (int i = 0; i < NPASS; ++i) {                 // 16-B chunks of 2 samples
            const int rr = rr0 + RSTEP * i;
            const int r1 = ti * BT + rr, r2 = tj * BT + rr;
            const bool v1 = r1 < R && j < Q, v2 = r2 < R && j < Q;
            kp_cp_async16(rawi + rr * JB + 2 * jc, v1 ? bt + r1 * Q + j : bt, v1);
            if (!diag) kp_cp_async16(rawj + rr * JB + 2 * jc, v2 ? bt + r2 * Q + j : bt, v2);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    // widening mapping: thread -> sample jw of rows rw0 + WSTEP i
    constexpr int WSTEP = NTHR / JB;
    static_assert(NTHR % JB == 0 && BT % WSTEP == 0, "widening mapping");
    const int jw = tid % JB, rw0 = tid / JB;
    // slab coordinates carried without divisions: template t_c, translated copy s_c, slab sl
    int64_t t_c = t_begin;
    int s_c = 0, sl = 0;
    if (nslab > 0) issue(t_c, 0);
    for (int64_t k = 0; k < nslab; ++k) {
        int64_t t_n = t_c;
        int s_n = s_c, sl_n = sl + 1;
        if (sl_n == nslab_t) { sl_n = 0; if (++s_n == S) { s_n = 0; ++t_n; } }
        const int j0 = sl * JB;
        const double2 *rp = ramp ? ramp + (int64_t)s_c * R * Q : nullptr;
        if (sl == 0 && tid < BT) { si[tid][0] = si[tid][1] = 0.0; sj[tid][0] = sj[tid][1] = 0.0; }
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();                                   // slab k landed; slab k - 1 fully consumed
        // widen to fp64 (products of fp32 values are then exact)
#pragma unroll
        for (int i = 0; i < BT / WSTEP; ++i) {
            const int rr = rw0 + WSTEP * i;
            const float2 u = rawi[rr * JB + jw];
            double2 du = make_double2((double)u.x, (double)u.y);
            if (rp) {                                  // translated copy: exact fp64 complex product
                const int r1 = ti * BT + rr, j = j0 + jw;
                const double2 a = (r1 < R && j < Q) ? rp[(int64_t)r1 * Q + j] : make_double2(1.0, 0.0);
                du = make_double2(du.x * a.x - du.y * a.y, du.x * a.y + du.y * a.x);
            }
            xi[rr][jw] = du;
            if (!diag) {
                const float2 v = rawj[rr * JB + jw];
                double2 dv = make_double2((double)v.x, (double)v.y);
                if (rp) {
                    const int r2 = tj * BT + rr, j = j0 + jw;
                    const double2 b = (r2 < R && j < Q) ? rp[(int64_t)r2 * Q + j] : make_double2(1.0, 0.0);
                    dv = make_double2(dv.x * b.x - dv.y * b.y, dv.x * b.y + dv.y * b.x);
                }
                xj[rr][jw] = dv;
            }
        }
        __syncthreads();                                   // fp64 slab ready, raw buffer free
        if (k + 1 < nslab) issue(t_n, sl_n * JB);
        // row sums (fp64, fixed order): threads 0-63 the rows of xi, 64-127 those of xj; row rr starts
        // at sample rr mod JB, so the 8 threads of a 128-bit wavefront hit distinct banks
        {
            static_assert((JB & (JB - 1)) == 0 && NTHR == 2 * BT, "row-sum mapping");
            const int rr = tid & (BT - 1);
            const double2 *xr = tid < BT ? &xi[rr][0] : &xj[rr][0];
            double sr[4] = {0, 0, 0, 0}, sim[4] = {0, 0, 0, 0};      // 4 independent chains, fixed order
#pragma unroll
            for (int s2 = 0; s2 < JB; ++s2) {
                const double2 v = xr[(rr + s2) & (JB - 1)];
                sr[s2 & 3] += v.x; sim[s2 & 3] += v.y;
            }
            double (*sd)[2] = tid < BT ? si : sj;
            sd[rr][0] += (sr[0] + sr[1]) + (sr[2] + sr[3]);
            sd[rr][1] += (sim[0] + sim[1]) + (sim[2] + sim[3]);
        }
        // Gram: Re(x_r conj(x_r')) = xr xr' + xi xi'.  On a diagonal tile only r >= r' is ever read
        // (kernel_reduce_kernel takes the lower triangle), so register entries (a, b) whose rows all lie
        // above their columns for every thread (ty + 8a < 16b, i.e. a < 2b) are skipped: 12 of 32.
        auto gram = [&](auto diag_c) {
            constexpr bool DIAG = decltype(diag_c)::value;
            if constexpr (MMA) {
                // diagonal tile: the warp block above the diagonal (wr < wc) and the m8n8 blocks a < b of
                // the two diagonal warp blocks are never read
                if (DIAG && wr < wc) return;
                const double *xa = reinterpret_cast<const double *>(&xi[wr + (lane >> 2)][0]) + (lane & 3);
                const double *xb = reinterpret_cast<const double *>(&xj[wc + (lane >> 2)][0]) + (lane & 3);
#pragma unroll
                for (int k0 = 0; k0 < 2 * JB; k0 += 4) {
                    double af[4], bf[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) af[a] = xa[a * 8 * 2 * SJ + k0];
#pragma unroll
                    for (int b = 0; b < 4; ++b) bf[b] = xb[b * 8 * 2 * SJ + k0];
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b)
                            if (!DIAG || wr != wc || a >= b)
                                asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                                             : "+d"(acc[a][b][0]), "+d"(acc[a][b][NE - 1])
                                             : "d"(af[a]), "d"(bf[b]));
                }
            } else {
#pragma unroll 4
            for (int jj = 0; jj < JB; ++jj) {
                double2 av[KA], bv[KBB];
#pragma unroll
                for (int a = 0; a < KA; ++a) av[a] = xi[ty + 8 * a][jj];
#pragma unroll
                for (int b = 0; b < KBB; ++b) bv[b] = xj[tx + 16 * b][jj];
#pragma unroll
                for (int a = 0; a < KA; ++a)
#pragma unroll
                    for (int b = 0; b < KBB; ++b)
                        if (!DIAG || a >= 2 * b)
                            acc[a][b][0] = fma(av[a].x, bv[b].x, fma(av[a].y, bv[b].y, acc[a][b][0]));
            }
            }
        };
        if (ti == tj) gram(std::true_type{});
        else gram(std::false_type{});
        if (sl == nslab_t - 1) {
            __syncthreads();                               // every row sum of this template is complete
            // remove the angular mean: - (1/Q) Re(S_r conj(S_r'))
            const double invQ = 1.0 / (double)Q;
#pragma unroll
            for (int a = 0; a < NA; ++a)
#pragma unroll
                for (int b = 0; b < NB; ++b)
#pragma unroll
                    for (int e = 0; e < NE; ++e) {
                        const int ra = row_of(a), cb = col_of(b, e);
                        const double re = si[ra][0] * sj[cb][0] + si[ra][1] * sj[cb][1];
                        acc[a][b][e] -= re * invQ;
                    }
            __syncthreads();       // every thread has read si/sj before the next template zeroes them
        }
        t_c = t_n;
        s_c = s_n;
        sl = sl_n;
    }
    double *out = partials + c * (int64_t)R * R;
#pragma unroll
    for (int a = 0; a < NA; ++a)
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                const int r1 = ti * BT + row_of(a), r2 = tj * BT + col_of(b, e);
                if (r1 < R && r2 < R && r1 >= r2) out[(int64_t)r1 * R + r2] = acc[a][b][e];   // lower triangle only
            }
}
template <bool MMA>
constexpr size_t kp_smem_bytes() {
    return 2 * (size_t)BT * KpLayout<MMA>::SJ * sizeof(double2) + 2 * (size_t)BT * JB * sizeof(float2);
}
static std::atomic<uint64_t> g_partials_attr[2];   // per-device max-smem attribute of kernel_partials_kernel<MMA>

// Gram kernel choice: the fp64 tensor-core form (default) or the DFMA tile (RSVD_KP_SIMT=1, A/B only)
static bool kp_use_mma() {
    static const bool simt = [] { const char *e = std::getenv("RSVD_KP_SIMT"); return e && e[0] == '1'; }();
    return !simt;
}
static rsvd_status launch_partials(dim3 grid, cudaStream_t s, const float2 *tmpl, int64_t T, int R, int Q,
                                   double *partials, const double2 *ramp, int S) {
    const bool mma = kp_use_mma();
    const void *fn = mma ? (const void *)kernel_partials_kernel<true> : (const void *)kernel_partials_kernel<false>;
    const size_t smem = mma ? kp_smem_bytes<true>() : kp_smem_bytes<false>();
    const cudaError_t e = smem_attr_once(fn, (int)smem, g_partials_attr[mma ? 1 : 0]);
    if (e != cudaSuccess) return cuda_check(e, "kernel_partials attribute");
    if (mma) kernel_partials_kernel<true><<<grid, NTHR, smem, s>>>(tmpl, T, R, Q, partials, ramp, S);
    else kernel_partials_kernel<false><<<grid, NTHR, smem, s>>>(tmpl, T, R, Q, partials, ramp, S);
    count_launches(1);
    return cuda_check(cudaGetLastError(), "kernel_partials launch");
}

// C[r][r'] = sqrt(w_r w_r') / (T Q) * sum_c P_c[max(r,r')][min(r,r')] (lower triangle is the
// computed one; reading it for both halves makes C exactly symmetric).  The chunk sum is a fixed
// two-level tree (chunk c into partial sum c mod 8 in ascending c, then the 8 partial sums in order),
// so C is bitwise the same for any sharding of the chunks over ranks.
constexpr int KR_WARPS = 8;    // chunk-parallel reduce: warp w sums chunks w, w + 8, ... of 32 entries
__global__ void __launch_bounds__(KR_WARPS * 32) kernel_reduce_kernel(const double *__restrict__ partials, int64_t nchunks,
                                                                       int R, double scale, const double *__restrict__ w,
                                                                       double *__restrict__ C) {
    __shared__ double part[KR_WARPS][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t idx = (int64_t)blockIdx.x * 32 + lane;
    const bool ok = idx < (int64_t)R * R;
    const int r = ok ? (int)(idx / R) : 0, s = ok ? (int)(idx % R) : 0;
    const int hi = r > s ? r : s, lo = r > s ? s : r;
    // tiles with ti < tj were skipped: the element (hi, lo) always lies in a computed tile
    double acc = 0.0;
    if (ok)
        for (int64_t c = warp; c < nchunks; c += KR_WARPS) acc += partials[c * (int64_t)R * R + (int64_t)hi * R + lo];
    part[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && ok) {
        double t = part[0][lane];                           // fixed order over the warps: deterministic
#pragma unroll
        for (int i = 1; i < KR_WARPS; ++i) t += part[i][lane];
        C[idx] = t * scale * sqrt(w[r]) * sqrt(w[s]);
    }
}

// ramp[s][r][j] = exp(-i k_r (dx_s cos psi_j + dy_s sin psi_j)), fp64 (row f2; reading G15)
__global__ void ramp_kernel(const double *__restrict__ k, const double *__restrict__ shifts, int S, int R, int Q,
                            double2 *__restrict__ ramp) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)S * R * Q) return;
    const int j = (int)(idx % Q), r = (int)((idx / Q) % R), s = (int)(idx / ((int64_t)R * Q));
    double sn, cs;
    sincospi(2.0 * j / (double)Q, &sn, &cs);
    const double ph = -k[r] * (shifts[2 * s] * cs + shifts[2 * s + 1] * sn);
    double ps, pc;
    sincos(ph, &ps, &pc);
    ramp[idx] = make_double2(pc, ps);
}

// ------------------------------------------------------------------ row f2: closed-form translation kernel
// Eq. template_cost_with_translations: from the target volume's spherical-harmonic
// coefficients B_l^m(k_r), one warp per entry (r, r' <= r), fixed lane-strided order over the
// (L+1)^2 coefficients and a fixed shuffle tree (deterministic):
//   C[r][r'] = sqrt(w_r w_r') Re[ S(r, r') E+(k_r, k_r') - conj(B_0^0(k_r)) B_0^0(k_r') E-(k_r) E-(k_r') ],
//   S(r, r') = sum_{l,m} conj(B_l^m(k_r)) B_l^m(k_r'),
// with the printed E+ = exp(-s^2 (k^2 + k'^2)/2) exp(k k' s^2) evaluated as exp(-s^2 (k - k')^2 / 2)
// and the printed Bessel-form E- as its closed form exp(-k^2 s^2 / 2) (I_{-1/2}(x) - I_{1/2}(x) =
// sqrt(2/(pi x)) e^{-x}; pinned by tests/test_oracle_pins.py::test_T1_E_minus_is_a_gaussian).
__global__ void kernel_translated_sh_kernel(const double2 *__restrict__ Bsh, int R, int nlm,
                                            const double *__restrict__ k, const double *__restrict__ w,
                                            double sigma, double *__restrict__ C) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= (int64_t)R * R) return;
    const int r = (int)(warp / R), c = (int)(warp % R);
    if (c > r) return;
    const double2 *a = Bsh + (int64_t)r * nlm, *b = Bsh + (int64_t)c * nlm;
    double re = 0.0;
    for (int i = lane; i < nlm; i += 32) re += a[i].x * b[i].x + a[i].y * b[i].y;      // Re conj(a) b
    for (int off = 16; off >= 1; off >>= 1) re += __shfl_xor_sync(0xffffffffu, re, off);
    if (lane == 0) {
        const double kr = k[r], kc = k[c], s2 = sigma * sigma;
        const double ep = exp(-0.5 * s2 * (kr - kc) * (kr - kc));
        const double em = exp(-0.5 * s2 * kr * kr) * exp(-0.5 * s2 * kc * kc);
        const double b0 = a[0].x * b[0].x + a[0].y * b[0].y;
        const double v = sqrt(w[r]) * sqrt(w[c]) * (re * ep - b0 * em);
        C[(int64_t)r * R + c] = v;
        C[(int64_t)c * R + r] = v;
    }
}

}  // namespace rsvd

using namespace rsvd;

extern "C" int64_t rsvd_kernel_chunk(void) { return KCHUNK; }

extern "C" int64_t rsvd_kernel_partials_bytes(int64_t T, int32_t R) {
    if (T < 0 || R <= 0) return -1;
    return (T + KCHUNK - 1) / KCHUNK * (int64_t)R * R * (int64_t)sizeof(double);
}

static rsvd_status check_grid(int32_t R, int32_t Q) {
    if (R <= 0) return fail(RSVD_ERR_ARG, "R must be positive");
    if (R > 256) return fail(RSVD_ERR_UNSUPPORTED, "R > 256 is not supported");
    if (Q <= 0) return fail(RSVD_ERR_ARG, "Q must be positive");
    if (!is_pow2(Q) || Q < 32 || Q > 1024)
        return fail(RSVD_ERR_UNSUPPORTED, "Q must be a power of two in [32, 1024]");
    return RSVD_OK;
}

extern "C" rsvd_status rsvd_kernel_partials(const void *templates, int64_t T, int32_t R, int32_t Q,
                                            double *partials, rsvd_stream_t stream) {
    rsvd_status st = check_grid(R, Q);
    if (st != RSVD_OK) return st;
    if (T < 0) return fail(RSVD_ERR_ARG, "T must be >= 0");
    if (T == 0) return RSVD_OK;
    if (!templates || !partials) return fail(RSVD_ERR_ARG, "NULL pointer");
    if (!aligned16(templates) || (reinterpret_cast<uintptr_t>(partials) & 7u))
        return fail(RSVD_ERR_ARG, "misaligned pointer");
    const int nt = (R + BT - 1) / BT;
    const int64_t nchunks = (T + KCHUNK - 1) / KCHUNK;
    if (nchunks > 65535) return fail(RSVD_ERR_UNSUPPORTED, "too many template chunks in one call");
    dim3 grid(nt, nt, (unsigned)nchunks);
    const bool timed = timing_enabled();
    cudaEvent_t ev0 = timed ? timing_event((cudaStream_t)stream) : nullptr;
    const rsvd_status st2 = launch_partials(grid, (cudaStream_t)stream, reinterpret_cast<const float2 *>(templates), T, R,
                                            Q, partials, nullptr, 1);
    if (st2 != RSVD_OK) return st2;
    if (timed) timing_span(ev0, timing_event((cudaStream_t)stream), TK_BASIS);
    return RSVD_OK;
}

extern "C" rsvd_status rsvd_kernel_reduce(const double *partials, int64_t nchunks, int32_t R,
                                          int64_t T_total, int32_t Q, const double *w, double *C,
                                          rsvd_stream_t stream) {
    rsvd_status st = check_grid(R, Q);
    if (st != RSVD_OK) return st;
    if (nchunks <= 0 || T_total <= 0) return fail(RSVD_ERR_ARG, "need at least one template chunk");
    if (!partials || !w || !C) return fail(RSVD_ERR_ARG, "NULL pointer");
    const double scale = 1.0 / ((double)T_total * (double)Q);
    const int64_t n = (int64_t)R * R;
    kernel_reduce_kernel<<<(unsigned)((n + 31) / 32), KR_WARPS * 32, 0, (cudaStream_t)stream>>>(
        partials, nchunks, R, scale, w, C);
    count_launches(1);
    return cuda_check(cudaGetLastError(), "kernel_reduce launch");
}

extern "C" rsvd_status rsvd_kernel_translated_sh(const void *Bsh, int32_t R, int32_t L, const double *k,
                                                 const double *w, double sigma, double *C, rsvd_stream_t stream) {
    if (R < 1 || R > 256) return fail(RSVD_ERR_UNSUPPORTED, "R must be in [1, 256]");
    if (L < 0 || L > 1023) return fail(RSVD_ERR_UNSUPPORTED, "L must be in [0, 1023]");
    if (!(sigma >= 0.0) || !std::isfinite(sigma)) return fail(RSVD_ERR_ARG, "sigma must be finite and >= 0");
    if (!Bsh || !k || !w || !C) return fail(RSVD_ERR_ARG, "NULL pointer");
    if (!aligned16(Bsh)) return fail(RSVD_ERR_ARG, "misaligned pointer");
    const int nlm = (L + 1) * (L + 1);
    const int64_t threads = (int64_t)R * R * 32;
    kernel_translated_sh_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const double2 *>(Bsh), R, nlm, k, w, sigma, C);
    count_launches(1);
    return cuda_check(cudaGetLastError(), "kernel_translated_sh launch");
}

extern "C" rsvd_status rsvd_build_basis_translated(const void *templates, int64_t T, int32_t R, int32_t Q,
                                                   const double *w_host, const double *k_host,
                                                   const double *shifts_host, int32_t S, int32_t H, double *U_host,
                                                   double *lambda_host, rsvd_stream_t stream) {
    rsvd_status st = check_grid(R, Q);
    if (st != RSVD_OK) return st;
    if (T <= 0) return fail(RSVD_ERR_ARG, "T must be >= 1 to build a basis");
    if (S < 1) return fail(RSVD_ERR_ARG, "S must be >= 1");
    if (H < 1 || H > R) return fail(RSVD_ERR_UNSUPPORTED, "H must satisfy 1 <= H <= R");
    if (!templates || !w_host || !k_host || !shifts_host || !U_host) return fail(RSVD_ERR_ARG, "NULL pointer");
    if (!aligned16(templates)) return fail(RSVD_ERR_ARG, "misaligned pointer");
    for (int r = 0; r < R; ++r)
        if (!std::isfinite(w_host[r]) || !(w_host[r] > 0.0) || !std::isfinite(k_host[r]))
            return fail(RSVD_ERR_ARG, "weights must be finite and > 0, wavenumbers finite");
    for (int i = 0; i < 2 * S; ++i)
        if (!std::isfinite(shifts_host[i])) return fail(RSVD_ERR_ARG, "shifts must be finite");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nchunks = (T + KCHUNK - 1) / KCHUNK;
    if (nchunks > 65535) return fail(RSVD_ERR_UNSUPPORTED, "too many template chunks in one call");
    const size_t pbytes = (size_t)nchunks * R * R * sizeof(double);
    const size_t rbytes = (size_t)S * R * Q * sizeof(double2);
    const size_t wbytes = (size_t)R * sizeof(double), cbytes = (size_t)R * R * sizeof(double);
    const size_t kbytes = (size_t)R * sizeof(double), sbytes = (size_t)2 * S * sizeof(double);
    void *scratch = nullptr;
    cudaError_t e = cudaMallocAsync(&scratch, rbytes + pbytes + wbytes + cbytes + kbytes + sbytes, s);
    if (e != cudaSuccess) return cuda_check(e, "cudaMallocAsync(basis scratch)");
    double2 *ramp = (double2 *)scratch;
    double *partials = (double *)((char *)scratch + rbytes);
    double *w_dev = partials + (size_t)nchunks * R * R;
    double *C_dev = w_dev + R;
    double *k_dev = C_dev + (size_t)R * R;
    double *s_dev = k_dev + R;
    std::vector<double> C((size_t)R * R);
    st = RSVD_OK;
    if ((e = cudaMemcpyAsync(w_dev, w_host, wbytes, cudaMemcpyHostToDevice, s)) != cudaSuccess) st = cuda_check(e, "copy w");
    if (st == RSVD_OK && (e = cudaMemcpyAsync(k_dev, k_host, kbytes, cudaMemcpyHostToDevice, s)) != cudaSuccess)
        st = cuda_check(e, "copy k");
    if (st == RSVD_OK && (e = cudaMemcpyAsync(s_dev, shifts_host, sbytes, cudaMemcpyHostToDevice, s)) != cudaSuccess)
        st = cuda_check(e, "copy shifts");
    if (st == RSVD_OK) {
        const int64_t n = (int64_t)S * R * Q;
        ramp_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(k_dev, s_dev, S, R, Q, ramp);
        count_launches(1);
        st = cuda_check(cudaGetLastError(), "ramp launch");
    }
    if (st == RSVD_OK) {
        const int nt = (R + BT - 1) / BT;
        dim3 grid(nt, nt, (unsigned)nchunks);
        st = launch_partials(grid, s, reinterpret_cast<const float2 *>(templates), T, R, Q, partials, ramp, S);
    }
    if (st == RSVD_OK) st = rsvd_kernel_reduce(partials, nchunks, R, T * (int64_t)S, Q, w_dev, C_dev, stream);
    if (st == RSVD_OK && (e = cudaMemcpyAsync(C.data(), C_dev, cbytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        st = cuda_check(e, "copy C");
    cudaFreeAsync(scratch, s);
    if (st != RSVD_OK) return st;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_check(e, "basis sync");
    return rsvd_eigen_basis(C.data(), R, H, U_host, lambda_host);
}

extern "C" rsvd_status rsvd_build_basis(const void *templates, int64_t T, int32_t R, int32_t Q,
                                        const double *w_host, int32_t H, double *U_host,
                                        double *lambda_host, rsvd_stream_t stream) {
    rsvd_status st = check_grid(R, Q);
    if (st != RSVD_OK) return st;
    if (T <= 0) return fail(RSVD_ERR_ARG, "T must be >= 1 to build a basis");
    if (H < 1 || H > R) return fail(RSVD_ERR_UNSUPPORTED, "H must satisfy 1 <= H <= R");
    if (!templates || !w_host || !U_host) return fail(RSVD_ERR_ARG, "NULL pointer");
    for (int r = 0; r < R; ++r)
        if (!std::isfinite(w_host[r]) || !(w_host[r] > 0.0))
            return fail(RSVD_ERR_ARG, "weights must be finite and > 0");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nchunks = (T + KCHUNK - 1) / KCHUNK;
    const size_t pbytes = (size_t)nchunks * R * R * sizeof(double);
    void *scratch = nullptr;
    const size_t wbytes = (size_t)R * sizeof(double), cbytes = (size_t)R * R * sizeof(double);
    cudaError_t e = cudaMallocAsync(&scratch, pbytes + wbytes + cbytes, s);
    if (e != cudaSuccess) return cuda_check(e, "cudaMallocAsync(basis scratch)");
    double *partials = (double *)scratch;
    double *w_dev = partials + (size_t)nchunks * R * R;
    double *C_dev = w_dev + R;
    std::vector<double> C((size_t)R * R);
    st = RSVD_OK;
    if ((e = cudaMemcpyAsync(w_dev, w_host, wbytes, cudaMemcpyHostToDevice, s)) != cudaSuccess)
        st = cuda_check(e, "copy w");
    if (st == RSVD_OK) st = rsvd_kernel_partials(templates, T, R, Q, partials, stream);
    if (st == RSVD_OK) st = rsvd_kernel_reduce(partials, nchunks, R, T, Q, w_dev, C_dev, stream);
    if (st == RSVD_OK && (e = cudaMemcpyAsync(C.data(), C_dev, cbytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        st = cuda_check(e, "copy C");
    cudaFreeAsync(scratch, s);
    if (st != RSVD_OK) return st;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_check(e, "basis sync");
    return rsvd_eigen_basis(C.data(), R, H, U_host, lambda_host);
}
