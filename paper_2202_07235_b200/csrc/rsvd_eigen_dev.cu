// rsvd_eigen_dev.cu -- row a0 on the device: the eigenbasis U_H of the R x R kernel matrix C without a
// host round trip ("the singular-value-decomposition" of the symmetric PSD kernel = its
// eigen-decomposition, reading G7).  Same textbook algorithm family as the host solver
// (rsvd_eigen.cpp), organised for one CTA of 512 threads with C resident in shared memory (R <= 128):
//
//   1. Householder tridiagonalisation T = Z^T C Z (full symmetric trailing block in shared memory;
//      per step: block reductions for ||x|| and v.p, the matvec p = beta B v with 4 threads per
//      column, the rank-2 update B -= v q^T + q v^T column-parallel; reflector k kept in row k);
//   2. every eigenvalue of T by bisection on the Sturm count (4 threads per eigenvalue, each evaluating
//      one of 4 interior points of the bracket, so a round shrinks it 5-fold) -- absolute accuracy
//      O(eps ||T||), the descending order is the index order;
//   3. the top-H eigenvectors of T by inverse iteration (thread per vector: tridiagonal LU of T - lambda I
//      with partial pivoting, 3 solves from the host solver's start vectors), each solve followed by
//      a block-parallel Gram-Schmidt (two classical passes) against the vectors before it, so clusters
//      stay orthonormal;
//   4. back-transform y -> Z y with the reflectors (warp per vector), normalisation and the sign rule
//      "largest-|.| entry positive, first on ties".
//
// Every reduction has a fixed order, so U is bitwise reproducible run to run.  *info = 0 on success; 1 when
// an inverse-iteration pair fails the a-posteriori residual test ||T y - lambda y|| <= 64 n eps ||T||
// (U is then not usable: callers run the host solver on the same C).
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>

#include "rsvd_common.cuh"

namespace rsvd {

constexpr int EV_THREADS = 512;
constexpr int EV_WARPS = EV_THREADS / 32;
constexpr int EV_MAXN = 128;
constexpr int EV_MAXY = 8192;          // H * n doubles of eigenvector workspace (64 KB)
#ifndef RSVD_EV_STOP
#define RSVD_EV_STOP 0                 // diagnostic builds only: return after phase 1 / 2 / 3
#endif

// block sum with one barrier: consecutive calls alternate between two partial buffers (red[2][EV_WARPS]),
// so a buffer is rewritten only after every thread has passed the barrier of the call in between
__device__ __forceinline__ double ev_block_sum(double x, double *red, int &rb) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *buf = red + rb * EV_WARPS;
    rb ^= 1;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
    if (lane == 0) buf[warp] = x;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < EV_WARPS; ++w) t += buf[w];      // same order in every thread
    return t;
}

// 1 / q to ~1 ulp: the hardware reciprocal seed (rcp.approx.ftz.f64) and two Newton steps -- half the
// latency of the IEEE division sequence on the Sturm recurrence's critical path (|q| >= pivmin is normal)
__device__ __forceinline__ double ev_rcp(double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    double e = fma(-q, r, 1.0);
    r = fma(r, e, r);
    e = fma(-q, r, 1.0);
    return fma(r, e, r);
}

// number of eigenvalues of T = (d, e) below sigma (Sturm sequence; e2 = e^2, pivmin guards zero pivots)
__device__ __forceinline__ int ev_sturm(int n, const double *d, const double *e2, double sigma, double pivmin) {
    int cnt = 0;
    double q = d[0] - sigma;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
    for (int i = 1; i < n; ++i) {
        q = (d[i] - sigma) - e2[i - 1] * ev_rcp(q);
        if (fabs(q) < pivmin) q = -pivmin;
        cnt += q < 0.0;
    }
    return cnt;
}

__global__ void __launch_bounds__(EV_THREADS, 1) eigen_basis_kernel(const double *__restrict__ C, int n, int H,
                                                                     double *__restrict__ U, double *__restrict__ lambda,
                                                                     int *__restrict__ info) {
    extern __shared__ __align__(16) double ev_smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int LDA = n + 4;                       // padded: the matvec's 4 rows x 4 columns per half-warp hit distinct banks
    double *A = ev_smem;                         // [n][LDA]; row k < n - 2 becomes reflector k
    double *d = A + n * LDA, *e = d + EV_MAXN, *e2 = e + EV_MAXN, *beta = e2 + EV_MAXN;
    double *v = beta + EV_MAXN, *p = v + EV_MAXN, *lam = p + EV_MAXN, *red = lam + EV_MAXN;   // red: [EV_WARPS]
    double *Y = red + 2 * EV_WARPS;              // [H][n] eigenvectors of T, then of C
    __shared__ int bad;
    if (tid == 0) bad = 0;
    int rb = 0;                                  // ev_block_sum buffer toggle (uniform)
    const double eps = 2.220446049250313e-16;

    for (int idx = tid; idx < n * n; idx += EV_THREADS) {
        const int i = idx / n, j = idx - (idx / n) * n;
        A[i * LDA + j] = 0.5 * (C[(size_t)i * n + j] + C[(size_t)j * n + i]);
    }
    __syncthreads();

    // ---- 1. Householder tridiagonalisation
    const int col = tid & 127, rg = tid >> 7;    // update mapping: column j = col, rows rg, rg + 4, ...
    const int pc = tid >> 2, pr = tid & 3;       // matvec mapping: column pc, rows pr, pr + 4, ...
    for (int k = 0; k + 2 < n; ++k) {
        const int m = n - k - 1, b0 = k + 1;
        const double xi = tid < m ? A[k * LDA + b0 + tid] : 0.0;
        const double a2 = ev_block_sum(xi * xi, red, rb);
        const double x0 = A[k * LDA + b0];
        double alpha = sqrt(a2);
        if (alpha == 0.0) {                      // uniform: nothing to annihilate
            if (tid == 0) { d[k] = A[k * LDA + k]; e[k] = 0.0; beta[k] = 0.0; }
            __syncthreads();
            continue;
        }
        if (x0 > 0) alpha = -alpha;              // v = x - alpha e1, alpha = -sign(x0) ||x||
        const double bk = 2.0 / (2.0 * a2 - 2.0 * x0 * alpha);     // 2 / ||v||^2
        if (tid < m) v[tid] = tid == 0 ? xi - alpha : xi;
        __syncthreads();
        double pp = 0.0;
        if (pc < m)
            for (int j = pr; j < m; j += 4) pp += A[(b0 + j) * LDA + b0 + pc] * v[j];
        pp += __shfl_xor_sync(0xffffffffu, pp, 1);
        pp += __shfl_xor_sync(0xffffffffu, pp, 2);
        if (pr == 0 && pc < m) p[pc] = bk * pp;
        __syncthreads();
        const double vp = ev_block_sum(tid < m ? v[tid] * p[tid] : 0.0, red, rb);
        const double K = 0.5 * bk * vp;
        if (tid < m) p[tid] -= K * v[tid];       // q = p - K v, in place
        __syncthreads();
        if (col < m) {
            const double qj = p[col], vj = v[col];
            for (int i = rg; i < m; i += 4) A[(b0 + i) * LDA + b0 + col] -= v[i] * qj + p[i] * vj;
        }
        if (tid < m) A[k * LDA + b0 + tid] = v[tid];                 // reflector k in row k
        if (tid == 0) { d[k] = A[k * LDA + k]; e[k] = alpha; beta[k] = bk; }
        __syncthreads();
    }
    if (tid == 0) {
        if (n >= 2) {
            d[n - 2] = A[(n - 2) * LDA + n - 2];
            e[n - 2] = A[(n - 1) * LDA + n - 2];
            beta[n - 2] = 0.0;
        }
        d[n - 1] = A[(n - 1) * LDA + n - 1];
        beta[n - 1] = 0.0;
    }
    __syncthreads();
    if (tid < n - 1) e2[tid] = e[tid] * e[tid];
    __syncthreads();

    if (RSVD_EV_STOP == 1) return;
    // ---- 2. all eigenvalues by bisection (lam[t] = t-th largest)
    double tnorm = 0.0, glo = 0.0, ghi = 0.0;
    for (int i = 0; i < n; ++i) {
        const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < n ? fabs(e[i]) : 0.0);
        tnorm = fmax(tnorm, fabs(d[i]) + r);
        glo = i == 0 ? d[i] - r : fmin(glo, d[i] - r);
        ghi = i == 0 ? d[i] + r : fmax(ghi, d[i] + r);
    }
    const double pivmin = fmax(tnorm * 1e-300, 1e-300);
    {
        const int t = tid >> 2, sub = tid & 3;           // eigenvalue t (descending), probe point sub
        const int a = n - 1 - t;                         // ascending index
        double lo = glo - 2.0 * eps * tnorm - pivmin, hi = ghi + 2.0 * eps * tnorm + pivmin;
        const unsigned gm = 0xfu << (lane & ~3);
        for (int it = 0; it < 200; ++it) {
            // stop at relative width 2 eps or absolute width eps ||T|| / 4 (uniform over the 4 lanes)
            if (!(hi - lo > 2.0 * eps * fmax(fabs(lo), fabs(hi)) && hi - lo > 0.25 * eps * tnorm + pivmin)) break;
            const double x = lo + (hi - lo) * (double)(sub + 1) / 5.0;
            const int c = t < n ? ev_sturm(n, d, e2, x, pivmin) : 0;
            // bracket: the largest probe with count <= a is the new lo, the smallest with count > a the new hi
            const unsigned ok = __ballot_sync(gm, c <= a) >> (lane & ~3) & 0xfu;
            const double x0p = __shfl_sync(gm, x, (lane & ~3) + 0), x1p = __shfl_sync(gm, x, (lane & ~3) + 1);
            const double x2p = __shfl_sync(gm, x, (lane & ~3) + 2), x3p = __shfl_sync(gm, x, (lane & ~3) + 3);
            const double xs[4] = {x0p, x1p, x2p, x3p};
            // the largest probe with count <= a is the new lo, the next probe (count > a) the new hi; this
            // keeps a valid bracket even if rounding made the counts non-monotone
            const int last = ok ? 31 - __clz((int)ok) : -1;
            const double nlo = last >= 0 ? xs[last] : lo;
            const double nhi = last < 3 ? xs[last + 1] : hi;
            lo = nlo;
            hi = nhi;
        }
        if (sub == 0 && t < n) lam[t] = 0.5 * (lo + hi);
    }
    __syncthreads();
    if (tid < n && lambda) lambda[tid] = lam[tid];

    if (RSVD_EV_STOP == 2) return;
    // ---- 3. top-H eigenvectors of T by inverse iteration + block Gram-Schmidt after every solve
    // thread h keeps its LU factors in local memory (4 KB per thread: the driver reserves local memory for
    // every resident thread, ~1.3 GB on 148 SMs, retained by the context); Y[h] holds the iterate
    double la[EV_MAXN], lb[EV_MAXN], lc2[EV_MAXN], lm[EV_MAXN];
    unsigned swp[EV_MAXN / 32];
    if (tid < H) {
        const int h = tid;
        const double sigma = lam[h];
        for (int i = 0; i < n; ++i) { la[i] = d[i] - sigma; lb[i] = i + 1 < n ? e[i] : 0.0; lc2[i] = 0.0; }
        for (int w = 0; w < EV_MAXN / 32; ++w) swp[w] = 0u;
        for (int i = 0; i + 1 < n; ++i) {
            const double sb = e[i];
            if (fabs(sb) > fabs(la[i])) {        // swap rows i and i + 1
                swp[i >> 5] |= 1u << (i & 31);
                const double na = sb, nb = la[i + 1], nc = i + 2 < n ? e[i + 1] : 0.0;
                const double mm = la[i] / sb;
                const double oa1 = lb[i], oc = lc2[i];
                la[i] = na; lb[i] = nb; lc2[i] = nc;
                lm[i] = mm;
                la[i + 1] = oa1 - mm * nb;
                lb[i + 1] = oc - mm * nc;
            } else {
                const double mm = la[i] != 0.0 ? sb / la[i] : 0.0;
                lm[i] = mm;
                la[i + 1] -= mm * lb[i];
            }
        }
        for (int i = 0; i < n; ++i) {
            if (fabs(la[i]) < eps * tnorm) la[i] = (la[i] < 0 ? -1.0 : 1.0) * eps * tnorm;
            la[i] = 1.0 / la[i];                 // the back solve multiplies by the reciprocal pivots
        }
        for (int i = 0; i < n; ++i) Y[h * n + i] = 1.0 + 1e-3 * (double)((i * 7 + h * 3) % 11);
    }
    for (int it = 0; it < 3; ++it) {
        if (tid < H) {
            double *x = Y + tid * n;
            for (int i = 0; i + 1 < n; ++i) {
                if (swp[i >> 5] >> (i & 31) & 1u) { const double t = x[i]; x[i] = x[i + 1]; x[i + 1] = t; }
                x[i + 1] -= lm[i] * x[i];
            }
            for (int i = n - 1; i >= 0; --i) {
                double s = x[i];
                if (i + 1 < n) s -= lb[i] * x[i + 1];
                if (i + 2 < n) s -= lc2[i] * x[i + 2];
                x[i] = s * la[i];
            }
        }
        __syncthreads();
        // Gram-Schmidt in vector order: y_h -= sum_{g < h} (y_g . y_h) y_g twice, then normalise
        for (int h = 0; h < H; ++h) {
            double *yh = Y + h * n;
            for (int pass = 0; pass < 2 && h > 0; ++pass) {
                // warp w computes the dots with g = w, w + 16, ... (lane-strided, fixed shuffle tree)
                for (int g = warp; g < h; g += EV_WARPS) {
                    const double *yg = Y + g * n;
                    double s = 0.0;
                    for (int i = lane; i < n; i += 32) s += yg[i] * yh[i];
#pragma unroll
                    for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
                    if (lane == 0) p[g] = s;
                }
                __syncthreads();
                if (tid < n) {
                    double acc = yh[tid];
                    for (int g = 0; g < h; ++g) acc -= p[g] * Y[g * n + tid];
                    yh[tid] = acc;
                }
                __syncthreads();
            }
            const double nr = ev_block_sum(tid < n ? yh[tid] * yh[tid] : 0.0, red, rb);
            const double inv = 1.0 / sqrt(nr);
            if (tid < n) yh[tid] *= inv;
            __syncthreads();
        }
    }
    // a-posteriori residual on T
    if (tid < H) {
        const double *x = Y + tid * n;
        const double sigma = lam[tid];
        double r2 = 0.0;
        for (int i = 0; i < n; ++i) {
            double t = d[i] * x[i] - sigma * x[i];
            if (i > 0) t += e[i - 1] * x[i - 1];
            if (i + 1 < n) t += e[i] * x[i + 1];
            r2 += t * t;
        }
        if (!(sqrt(r2) <= 64.0 * n * eps * tnorm)) atomicExch(&bad, 1);
    }
    __syncthreads();

    if (RSVD_EV_STOP == 3) return;
    // ---- 4. back-transform (warp per vector), normalise, sign rule
    for (int h = warp; h < H; h += EV_WARPS) {
        double *y = Y + h * n;
        double yr[EV_MAXN / 32];                 // entries lane + 32 u of the vector, in registers
#pragma unroll
        for (int u = 0; u < EV_MAXN / 32; ++u) yr[u] = lane + 32 * u < n ? y[lane + 32 * u] : 0.0;
        for (int k = n - 3; k >= 0; --k) {
            const double bk = beta[k];
            if (bk == 0.0) continue;
            const double *vk = A + k * LDA;      // reflector entries at k + 1 .. n - 1
            double vr[EV_MAXN / 32];
            double s = 0.0;
#pragma unroll
            for (int u = 0; u < EV_MAXN / 32; ++u) {
                const int j = lane + 32 * u;
                vr[u] = (j > k && j < n) ? vk[j] : 0.0;
                s = fma(vr[u], yr[u], s);
            }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            s *= bk;
#pragma unroll
            for (int u = 0; u < EV_MAXN / 32; ++u) yr[u] = fma(-s, vr[u], yr[u]);
        }
        double nr = 0.0, amax = -1.0;
        int imax = n;
#pragma unroll
        for (int u = 0; u < EV_MAXN / 32; ++u) {
            const int r = lane + 32 * u;
            if (r < n) {
                nr = fma(yr[u], yr[u], nr);
                const double a = fabs(yr[u]);
                if (a > amax) { amax = a; imax = r; }
            }
        }
        double ymax = 0.0;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            nr += __shfl_xor_sync(0xffffffffu, nr, off);
            const double oa = __shfl_xor_sync(0xffffffffu, amax, off);
            const int oi = __shfl_xor_sync(0xffffffffu, imax, off);
            if (oa > amax || (oa == amax && oi < imax)) { amax = oa; imax = oi; }
        }
#pragma unroll
        for (int u = 0; u < EV_MAXN / 32; ++u)
            if (lane + 32 * u == imax) ymax = yr[u];
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) ymax += __shfl_xor_sync(0xffffffffu, ymax, off);   // one lane holds it
        const double sgn = ymax < 0 ? -1.0 : 1.0;
        const double sc = sgn / sqrt(nr);
#pragma unroll
        for (int u = 0; u < EV_MAXN / 32; ++u) {
            const int r = lane + 32 * u;
            if (r < n) U[(size_t)r * H + h] = sc * yr[u];
        }
    }
    if (tid == 0 && info) *info = bad;
}

static size_t eigen_dev_smem(int n, int H) {
    return ((size_t)n * (n + 4) + 7 * EV_MAXN + 2 * EV_WARPS + (size_t)H * n) * sizeof(double);
}
static std::atomic<uint64_t> g_eigen_dev_attr{0};

}  // namespace rsvd

using namespace rsvd;

extern "C" rsvd_status rsvd_eigen_basis_device(const double *C, int32_t R, int32_t H, double *U, double *lambda,
                                               int32_t *info, rsvd_stream_t stream) {
    if (R <= 0 || R > EV_MAXN) return fail(RSVD_ERR_UNSUPPORTED, "device eigen-solver: R must be in [1, 128]");
    if (H < 1 || H > R) return fail(RSVD_ERR_UNSUPPORTED, "H must satisfy 1 <= H <= R");
    if ((int64_t)H * R > EV_MAXY) return fail(RSVD_ERR_UNSUPPORTED, "device eigen-solver: H * R > 8192");
    if (!C || !U || !info) return fail(RSVD_ERR_ARG, "NULL pointer");
    if ((reinterpret_cast<uintptr_t>(C) | reinterpret_cast<uintptr_t>(U) | reinterpret_cast<uintptr_t>(lambda)) & 7u)
        return fail(RSVD_ERR_ARG, "misaligned pointer");
    const size_t smem = eigen_dev_smem(R, H);
    // the attribute is set once per device, so it must cover the largest supported (R, H)
    const cudaError_t e = smem_attr_once((const void *)eigen_basis_kernel, (int)eigen_dev_smem(EV_MAXN, EV_MAXY / EV_MAXN),
                                         g_eigen_dev_attr);
    if (e != cudaSuccess) return cuda_check(e, "eigen_basis attribute");
    eigen_basis_kernel<<<1, EV_THREADS, smem, (cudaStream_t)stream>>>(C, R, H, U, lambda, info);
    count_launches(1);
    return cuda_check(cudaGetLastError(), "eigen_basis launch");
}
