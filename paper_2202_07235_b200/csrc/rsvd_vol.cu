// rsvd_vol.cu -- row f4: volume alignment with the radial- and degree-SVD (§5, :783-1049).
//
// Kernels (one launch each, all on the caller's stream):
//   vol_kernel_C / vol_kernel_D  fp64 radial and degree kernels of the target(s) (:951-954, :1001-1007);
//                                one warp per output entry, lanes stride the sum, fixed shuffle tree.
//   vol_compress_kernel          principal shells sum_r U[r][h] sqrt(w_r) A[r][lm] (:921-927); thread per
//                                (volume, lm), the basis column staged in shared memory.
//   vol_wigner_kernel            [v_j^T d]_{m1 m2}(beta) (:981-984); thread per (beta, m1, m2), d^l from the
//                                closed-form seed at l0 = max(|m1|,|m2|) and the three-term recurrence in l
//                                (fp64), accumulated against V.
//   vol_degrees_kernel           Steps 1 + 1b (:1017-1020); CTA per (volume, m2), thread per m1.
//   vol_align_kernel             Steps 2 + 3 (+ argmax) (:1021-1023); CTA per (volume, beta): Step 2 and
//                                the DFT over m1 per m2 column (warp-distributed FFT of rsvd_common.cuh)
//                                into a P x M shared tile, then the DFT over m2 per alpha row, Re, landscape
//                                row stores and/or a packed-key max per volume.
// Layouts (include/rsvd_vol.h): shells [n][HC][NC], T [nb][HD][M(m2)][M(m1)], Y [n][HD][M(m2)][M(m1)] --
// the index a warp's lanes walk is always the fastest one.
#include <cuda_runtime.h>
#include <math.h>

#include "../../include/rsvd_vol.h"
#include "rsvd_common.cuh"

namespace rsvd {

__device__ __forceinline__ uint32_t vol_ord(float v) {
    const uint32_t u = __float_as_uint(v);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// ------------------------------------------------------------------ kernels C and D (fp64)
__global__ void vol_kernel_C(const float2 *__restrict__ B, int64_t nB, int R, int NC, const double *__restrict__ w,
                             double *__restrict__ C) {
    const int64_t e = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;      // (r, s) entry
    const int lane = threadIdx.x & 31;
    if (e >= (int64_t)R * R) return;
    const int r = (int)(e / R), s = (int)(e % R);
    double acc = 0.0;
    for (int64_t t = 0; t < nB; ++t) {
        const float2 *br = B + (t * R + r) * NC, *bs = B + (t * R + s) * NC;
        for (int j = 1 + lane; j < NC; j += 32) {                                        // l >= 1
            const float2 a = br[j], b = bs[j];
            acc += (double)a.x * b.x + (double)a.y * b.y;                                // Re conj(a) b
        }
    }
    acc = warp_sum_d(acc);
    if (lane == 0) C[e] = acc * sqrt(w[r] * w[s]) / (double)nB;
}

__global__ void vol_kernel_D(const float2 *__restrict__ B, int64_t nB, int R, int L, const double *__restrict__ w,
                             double *__restrict__ D) {
    const int64_t e = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;      // (l, l') entry
    const int lane = threadIdx.x & 31;
    const int L1 = L + 1, NC = L1 * L1;
    if (e >= (int64_t)L1 * L1) return;
    const int l = (int)(e / L1), lp = (int)(e % L1);
    double acc = 0.0;
    if (l >= 1 && lp >= 1) {
        const int mm = min(l, lp), nm = 2 * mm + 1;
        for (int64_t t = 0; t < nB; ++t)
            for (int i = lane; i < R * nm; i += 32) {
                const int r = i / nm, m = i % nm - mm;
                const float2 a = B[(t * R + r) * NC + l * l + l + m], b = B[(t * R + r) * NC + lp * lp + lp + m];
                acc += w[r] * ((double)a.x * b.x + (double)a.y * b.y);
            }
    }
    acc = warp_sum_d(acc);
    if (lane == 0) D[e] = acc / (double)nB;
}

// ------------------------------------------------------------------ principal shells
constexpr int VC_HB = 8;                       // principal vectors per pass
__global__ void vol_compress_kernel(const float2 *__restrict__ A, int64_t n, int R, int NC, const double *__restrict__ w,
                                    const double *__restrict__ U, int HC, float2 *__restrict__ shells) {
    extern __shared__ float us[];              // [R][HC] U sqrt(w), fp32
    for (int i = threadIdx.x; i < R * HC; i += blockDim.x) us[i] = (float)(U[i] * sqrt(w[i / HC]));
    __syncthreads();
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;                 // (volume, lm)
    if (idx >= n * NC) return;
    const int64_t v = idx / NC;
    const int j = (int)(idx % NC);
    const float2 *a = A + v * R * NC + j;
    for (int h0 = 0; h0 < HC; h0 += VC_HB) {
        float2 acc[VC_HB];
#pragma unroll
        for (int h = 0; h < VC_HB; ++h) acc[h] = make_float2(0.f, 0.f);
        for (int r = 0; r < R; ++r) {
            const float2 x = a[(int64_t)r * NC];
#pragma unroll
            for (int h = 0; h < VC_HB; ++h) {
                const float u = (h0 + h < HC) ? us[r * HC + h0 + h] : 0.f;
                acc[h].x = fmaf(u, x.x, acc[h].x);
                acc[h].y = fmaf(u, x.y, acc[h].y);
            }
        }
#pragma unroll
        for (int h = 0; h < VC_HB; ++h)
            if (h0 + h < HC) shells[(v * HC + h0 + h) * NC + j] = acc[h];          // [n][HC][NC]
    }
}

// ------------------------------------------------------------------ Wigner-d table
__device__ double ipow(double x, int e) {
    double r = 1.0;
    for (; e > 0; e >>= 1, x *= x)
        if (e & 1) r *= x;
    return r;
}
// d^{l0}_{m1 m2}(beta) at l0 = max(|m1|, |m2|) (Wigner's sum collapses to one term; DESIGN.md §6 f4)
__device__ double wigner_seed(int l0, int m1, int m2, double c, double s) {
    auto sqrt_binom = [&](int k) {
        return exp(0.5 * (lgamma(2.0 * l0 + 1.0) - lgamma(k + 1.0) - lgamma(2.0 * l0 - k + 1.0)));
    };
    if (abs(m1) == l0) {
        if (m1 == l0) return (((l0 - m2) & 1) ? -1.0 : 1.0) * sqrt_binom(l0 + m2) * ipow(c, l0 + m2) * ipow(s, l0 - m2);
        return sqrt_binom(l0 + m2) * ipow(c, l0 - m2) * ipow(s, l0 + m2);
    }
    if (m2 == l0) return sqrt_binom(l0 + m1) * ipow(c, l0 + m1) * ipow(s, l0 - m1);
    return (((l0 + m1) & 1) ? -1.0 : 1.0) * sqrt_binom(l0 + m1) * ipow(c, l0 - m1) * ipow(s, l0 + m1);
}

constexpr int VOL_HMAX = 32;
__global__ void vol_wigner_kernel(const double *__restrict__ beta, int nb, int L, const double *__restrict__ V, int HD,
                                  float *__restrict__ T) {
    extern __shared__ double vs[];             // [L+1][HD]
    for (int i = threadIdx.x; i < (L + 1) * HD; i += blockDim.x) vs[i] = V[i];
    __syncthreads();
    const int M = 2 * L + 1;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;                 // (b, m2, m1)
    if (idx >= (int64_t)nb * M * M) return;
    const int b = (int)(idx / (M * M));
    const int e = (int)(idx % (M * M));
    const int m2 = e / M - L, m1 = e % M - L;
    const double bt = beta[b];
    double sh, ch, sb, cb;
    sincos(0.5 * bt, &sh, &ch);
    sincos(bt, &sb, &cb);
    double acc[VOL_HMAX];
#pragma unroll
    for (int j = 0; j < VOL_HMAX; ++j) acc[j] = 0.0;
    const int l0 = max(abs(m1), abs(m2));
    double dprev = 0.0, d = wigner_seed(l0, m1, m2, ch, sh);
    for (int l = l0;; ++l) {
#pragma unroll
        for (int j = 0; j < VOL_HMAX; ++j)
            if (j < HD) acc[j] = fma(vs[l * HD + j], d, acc[j]);
        if (l == L) break;
        double dn;
        if (l == 0) {
            dn = cb;                                                                     // d^1_00 = cos beta
        } else {                                                                         // three-term recurrence in l
            const double num = (2.0 * l + 1.0) * ((double)l * (l + 1) * cb - (double)m1 * m2) * d -
                               (l + 1.0) * sqrt(((double)l * l - m1 * m1) * ((double)l * l - m2 * m2)) * dprev;
            dn = num / (l * sqrt(((l + 1.0) * (l + 1) - m1 * m1) * ((l + 1.0) * (l + 1) - m2 * m2)));
        }
        dprev = d;
        d = dn;
    }
    float *out = T + (int64_t)b * HD * M * M + e;                                       // [nb][HD][M(m2)][M(m1)]
#pragma unroll
    for (int j = 0; j < VOL_HMAX; ++j)
        if (j < HD) out[(int64_t)j * M * M] = (float)acc[j];
}

// ------------------------------------------------------------------ Steps 1 + 1b
// CTA per (volume, m2): the target's (l, m2) shells and V staged in shared memory; thread per m1 reads
// the volume's shells sA[v][h][(l, m1)] (consecutive m1 -> consecutive addresses) and writes
// Y[v][j][m2][m1] (coalesced).
template <int HDM>
__global__ void __launch_bounds__(128) vol_degrees_kernel(const float2 *__restrict__ sA, const float2 *__restrict__ sB,
                                                          int L, int HC, const double *__restrict__ V, int HD,
                                                          float2 *__restrict__ Y) {
    extern __shared__ float2 smem_f2[];
    const int M = 2 * L + 1, NC = (L + 1) * (L + 1);
    const int64_t v = blockIdx.y;
    const int m2 = (int)blockIdx.x - L;
    float2 *bs = smem_f2;                                   // [L+1][HC] target shells at (l, m2)
    float *vv = reinterpret_cast<float *>(bs + (L + 1) * HC); // [L+1][HD]
    for (int i = threadIdx.x; i < (L + 1) * HC; i += blockDim.x) {
        const int l = i / HC, h = i % HC;
        bs[i] = l >= abs(m2) ? sB[(int64_t)h * NC + l * l + l + m2] : make_float2(0.f, 0.f);
    }
    for (int i = threadIdx.x; i < (L + 1) * HD; i += blockDim.x) vv[i] = (float)V[i];
    __syncthreads();
    const float2 *av = sA + v * HC * NC;
    for (int m1i = threadIdx.x; m1i < M; m1i += blockDim.x) {
        const int m1 = m1i - L;
        float2 acc[HDM];
#pragma unroll
        for (int j = 0; j < HDM; ++j) acc[j] = make_float2(0.f, 0.f);
        for (int l = max(abs(m1), abs(m2)); l <= L; ++l) {
            const float2 *a = av + l * l + l + m1;
            const float2 *bl = bs + l * HC;
            float2 x = make_float2(0.f, 0.f);
            for (int h = 0; h < HC; ++h) {                                               // conj(a) b
                const float2 p = a[(int64_t)h * NC], q = bl[h];
                x.x = fmaf(p.x, q.x, fmaf(p.y, q.y, x.x));
                x.y = fmaf(p.x, q.y, fmaf(-p.y, q.x, x.y));
            }
#pragma unroll
            for (int j = 0; j < HDM; ++j)
                if (j < HD) {
                    const float vj = vv[l * HD + j];
                    acc[j].x = fmaf(vj, x.x, acc[j].x);
                    acc[j].y = fmaf(vj, x.y, acc[j].y);
                }
        }
        float2 *out = Y + (v * HD * M + (m2 + L)) * M + m1i;                            // [n][HD][M(m2)][M(m1)]
#pragma unroll
        for (int j = 0; j < HDM; ++j)
            if (j < HD) out[(int64_t)j * M * M] = acc[j];
    }
}

// ------------------------------------------------------------------ Steps 2 + 3 (+ argmax)
// CTA per (volume, beta), 2 CTAs per SM at P = 128.  Pass 1 (warp per m2 column): Step 2 for the column
// straight from global memory (lanes over m1, coalesced in the m1-fastest layouts of T and Y), DFT over
// m1 in registers, store G[a][m2] (P x M tile).  Pass 2 (warp per alpha row a): DFT over m2 (positions
// m2 mod P, zero outside [-L, L]), Re, landscape row store and packed-key max.
constexpr int VA_THREADS = 256;
template <int P>
__global__ void __launch_bounds__(VA_THREADS, 2) vol_align_kernel(const float2 *__restrict__ Y, const float *__restrict__ T,
                                                                  int nb, int L, int HD, float *__restrict__ X,
                                                                  unsigned long long *__restrict__ best_key) {
    constexpr int E = P / 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2 *tw = reinterpret_cast<float2 *>(smem_raw);     // [E][32]
    float2 *G = tw + E * 32;                               // [P][M] (M odd: conflict-free column stores)
    __shared__ unsigned long long red[VA_THREADS / 32];
    const int M = 2 * L + 1;
    const int b = blockIdx.x;
    const int64_t v = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < E * 32; i += VA_THREADS) tw[i] = twiddle_N(i % 32, i / 32, P);
    float2 stw[5];
    lane_stage_twiddles<32>(lane, stw);
    __syncthreads();
    const int b5 = (int)(__brev((unsigned)lane) >> 27);
    const int64_t MM = (int64_t)M * M;
    const float *Tb = T + (int64_t)b * HD * MM;
    const float2 *Yv = Y + v * HD * MM;
    // FFT position n = lane + 32 e <-> order m = n (n <= L) or n - P (n >= P - L), else 0
    int mi[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int n = lane + 32 * e;
        mi[e] = n <= L ? n + L : (n >= P - L ? n - P + L : -1);
    }
    for (int c = warp; c < M; c += VA_THREADS / 32) {                                   // m2 column c = m2 + L
        float2 x[E];
#pragma unroll
        for (int e = 0; e < E; ++e) x[e] = make_float2(0.f, 0.f);
        const float *tc = Tb + (int64_t)c * M;
        const float2 *yc = Yv + (int64_t)c * M;
        for (int j = 0; j < HD; ++j) {                                                   // Step 2
#pragma unroll
            for (int e = 0; e < E; ++e)
                if (mi[e] >= 0) {
                    const float t = __ldg(tc + j * MM + mi[e]);
                    const float2 y = __ldg(yc + j * MM + mi[e]);
                    x[e].x = fmaf(t, y.x, x[e].x);
                    x[e].y = fmaf(t, y.y, x[e].y);
                }
        }
        fft_dist<E, 32>(x, lane, tw, stw);                                               // over m1 -> alpha
#pragma unroll
        for (int k1 = 0; k1 < E; ++k1) G[(k1 + E * b5) * M + c] = x[brev(k1, clog2(E))];
    }
    __syncthreads();
    unsigned long long best = 0ull;
    float *Xo = X ? X + ((v * nb + b) * (int64_t)P) * P : nullptr;
    for (int r = warp; r < P; r += VA_THREADS / 32) {                                   // alpha row r
        float2 x[E];
#pragma unroll
        for (int e = 0; e < E; ++e) x[e] = mi[e] >= 0 ? G[r * M + mi[e]] : make_float2(0.f, 0.f);
        fft_dist<E, 32>(x, lane, tw, stw);                                               // over m2 -> gamma
#pragma unroll
        for (int k1 = 0; k1 < E; ++k1) {
            const int g = k1 + E * b5;
            const float val = x[brev(k1, clog2(E))].x;
            if (Xo) Xo[r * P + g] = val;
            const uint32_t flat = (uint32_t)((b * P + r) * P + g);
            const unsigned long long key = ((unsigned long long)vol_ord(val) << 32) | (0xFFFFFFFFu - flat);
            best = key > best ? key : best;
        }
    }
    if (best_key) {
#pragma unroll
        for (int off = 16; off; off >>= 1) {
            const unsigned long long o = __shfl_xor_sync(0xffffffffu, best, off);
            best = o > best ? o : best;
        }
        if (lane == 0) red[warp] = best;
        __syncthreads();
        if (tid == 0) {
            for (int i = 1; i < VA_THREADS / 32; ++i) best = red[i] > best ? red[i] : best;
            atomicMax(best_key + v, best);
        }
    }
}

template <int P>
static cudaError_t launch_vol_align(const float2 *Y, int64_t n, const float *T, int nb, int L, int HD, float *X,
                                    unsigned long long *keys, cudaStream_t s) {
    const size_t smem = ((size_t)(P / 32) * 32 + (size_t)P * (2 * L + 1)) * sizeof(float2);
    cudaError_t e = cudaFuncSetAttribute(vol_align_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    vol_align_kernel<P><<<dim3((unsigned)nb, (unsigned)n), VA_THREADS, smem, s>>>(Y, T, nb, L, HD, X, keys);
    return cudaGetLastError();
}

}  // namespace rsvd

using namespace rsvd;

static bool vol_L_ok(int32_t L) { return L >= 1 && L <= 63; }

extern "C" int64_t rsvd_vol_ncoef(int32_t L) { return L < 0 ? -1 : (int64_t)(L + 1) * (L + 1); }

extern "C" rsvd_status rsvd_vol_kernels(const void *B, int64_t nB, int32_t R, int32_t L, const double *w, double *C,
                                        double *D, rsvd_stream_t stream) {
    if (nB < 1 || R < 1 || R > 256 || !vol_L_ok(L)) return fail(RSVD_ERR_ARG, "vol_kernels: bad sizes");
    if (!B || !w || (!C && !D)) return fail(RSVD_ERR_ARG, "vol_kernels: NULL pointer");
    cudaStream_t s = (cudaStream_t)stream;
    const int NC = (L + 1) * (L + 1);
    if (C) {
        const int64_t warps = (int64_t)R * R;
        vol_kernel_C<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(reinterpret_cast<const float2 *>(B), nB, R, NC, w, C);
        count_launches(1);
    }
    if (D) {
        const int64_t warps = (int64_t)(L + 1) * (L + 1);
        vol_kernel_D<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(reinterpret_cast<const float2 *>(B), nB, R, L, w, D);
        count_launches(1);
    }
    return cuda_check(cudaGetLastError(), "vol_kernels launch");
}

extern "C" rsvd_status rsvd_vol_compress(const void *A, int64_t n, int32_t R, int32_t L, const double *w,
                                         const double *U, int32_t HC, void *shells, rsvd_stream_t stream) {
    if (n < 0 || R < 1 || R > 256 || !vol_L_ok(L) || HC < 1 || HC > VOL_HMAX || HC > R)
        return fail(RSVD_ERR_ARG, "vol_compress: bad sizes");
    if (n == 0) return RSVD_OK;
    if (!A || !w || !U || !shells) return fail(RSVD_ERR_ARG, "vol_compress: NULL pointer");
    const int NC = (L + 1) * (L + 1);
    const int64_t total = n * NC;
    vol_compress_kernel<<<(unsigned)((total + 255) / 256), 256, (size_t)R * HC * sizeof(float), (cudaStream_t)stream>>>(
        reinterpret_cast<const float2 *>(A), n, R, NC, w, U, HC, reinterpret_cast<float2 *>(shells));
    count_launches(1);
    return cuda_check(cudaGetLastError(), "vol_compress launch");
}

extern "C" rsvd_status rsvd_vol_wigner_table(const double *beta, int32_t nb, int32_t L, const double *V, int32_t HD,
                                             float *T, rsvd_stream_t stream) {
    if (nb < 0 || !vol_L_ok(L) || HD < 1 || HD > VOL_HMAX || HD > L + 1) return fail(RSVD_ERR_ARG, "vol_wigner: bad sizes");
    if (nb == 0) return RSVD_OK;
    if (!beta || !V || !T) return fail(RSVD_ERR_ARG, "vol_wigner: NULL pointer");
    const int M = 2 * L + 1;
    const int64_t total = (int64_t)nb * M * M;
    vol_wigner_kernel<<<(unsigned)((total + 127) / 128), 128, (size_t)(L + 1) * HD * sizeof(double), (cudaStream_t)stream>>>(
        beta, nb, L, V, HD, T);
    count_launches(1);
    return cuda_check(cudaGetLastError(), "vol_wigner launch");
}

extern "C" rsvd_status rsvd_vol_degrees(const void *shellsA, int64_t n, const void *shellB, int32_t L, int32_t HC,
                                        const double *V, int32_t HD, void *Y, rsvd_stream_t stream) {
    if (n < 0 || n > 65535 || !vol_L_ok(L) || HC < 1 || HC > VOL_HMAX || HD < 1 || HD > VOL_HMAX || HD > L + 1)
        return fail(RSVD_ERR_ARG, "vol_degrees: bad sizes (n <= 65535 per call)");
    if (n == 0) return RSVD_OK;
    if (!shellsA || !shellB || !V || !Y) return fail(RSVD_ERR_ARG, "vol_degrees: NULL pointer");
    const int M = 2 * L + 1;
    const size_t smem = (size_t)(L + 1) * HC * sizeof(float2) + (size_t)(L + 1) * HD * sizeof(float);
    const dim3 grid((unsigned)M, (unsigned)n);
    auto a = reinterpret_cast<const float2 *>(shellsA);
    auto b = reinterpret_cast<const float2 *>(shellB);
    auto y = reinterpret_cast<float2 *>(Y);
    cudaStream_t s = (cudaStream_t)stream;
    if (HD <= 8) vol_degrees_kernel<8><<<grid, 128, smem, s>>>(a, b, L, HC, V, HD, y);
    else if (HD <= 16) vol_degrees_kernel<16><<<grid, 128, smem, s>>>(a, b, L, HC, V, HD, y);
    else vol_degrees_kernel<32><<<grid, 128, smem, s>>>(a, b, L, HC, V, HD, y);
    count_launches(1);
    return cuda_check(cudaGetLastError(), "vol_degrees launch");
}

extern "C" rsvd_status rsvd_vol_align(const void *Y, int64_t n, const float *T, int32_t nb, int32_t L, int32_t HD,
                                      int32_t P, float *X, uint64_t *best_key, rsvd_stream_t stream) {
    if (n < 0 || n > 65535 || nb < 0 || !vol_L_ok(L) || HD < 1 || HD > VOL_HMAX || HD > L + 1)
        return fail(RSVD_ERR_ARG, "vol_align: bad sizes (n <= 65535 per call)");
    if ((P != 32 && P != 64 && P != 128) || P < 2 * L + 1) return fail(RSVD_ERR_ARG, "vol_align: P must be 32/64/128 and >= 2L+1");
    if ((int64_t)nb * P * P > 0xFFFFFFFFLL) return fail(RSVD_ERR_ARG, "vol_align: nb * P * P exceeds the key index");
    if (n == 0 || nb == 0) return RSVD_OK;
    if (!Y || !T || (!X && !best_key)) return fail(RSVD_ERR_ARG, "vol_align: NULL pointer");
    cudaStream_t s = (cudaStream_t)stream;
    auto keys = reinterpret_cast<unsigned long long *>(best_key);
    auto y = reinterpret_cast<const float2 *>(Y);
    cudaError_t e;
    switch (P) {
        case 32: e = launch_vol_align<32>(y, n, T, nb, L, HD, X, keys, s); break;
        case 64: e = launch_vol_align<64>(y, n, T, nb, L, HD, X, keys, s); break;
        default: e = launch_vol_align<128>(y, n, T, nb, L, HD, X, keys, s); break;
    }
    count_launches(1);
    return cuda_check(e, "vol_align launch");
}
