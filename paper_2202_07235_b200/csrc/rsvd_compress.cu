// rsvd_compress.cu -- row a1 (Step 1): compress rings onto the H principal image rings and take
// their Fourier-Bessel coefficients, stored in the align kernel's block layout.
//
//   A_q[n,h] = (1/Q) sum_j e^{-2 pi i q j/Q} sum_r U[r,h] sqrt(w_r) a_n[r,j]
//
// The principal image ring [u_h^T A](psi_j) = sum_r u_{h,r} A(k_r, psi_j) eta_r is PAPER.md:580-585
// (eta_r = sqrt(w_r): DESIGN.md reading G2); its Fourier-Bessel coefficients are the discrete
// transform of PAPER.md:240-244 normalised as (1/Q) DFT (reading G1).  Projecting in psi-space first
// and transforming H rings (instead of R) is the same linear map.
//
// Block layout (opaque; ABI version 1): float2 blocks[(N+1)][Kpad][rows_pad], N = Q/2,
//   image side    alpha[q][h][n] = conj(A_q[n,h]),   alpha[q][H+h][n] = A_{(Q-q) mod Q}[n,h]
//   template side  beta[q][h][n] = B_q[n,h],          beta[q][H+h][n] = conj(B_{(Q-q) mod Q}[n,h])
// for q = 0..N, zero elsewhere, so that sum_j alpha[q][j][m] beta[q][j][t] = S_q + conj(S_{Q-q})
// with S_q[m,t] = sum_h conj(A_q[m,h]) B_q[t,h] (Step 2).
#include <cuda_runtime.h>

#include <cmath>

#include "rsvd_common.cuh"

namespace rsvd {

constexpr int CP_THREADS = 256;
constexpr int CP_HC = 16;        // principal rings per pass

template <int LOGQ>
__global__ void __launch_bounds__(CP_THREADS) compress_kernel(const float2 *__restrict__ rings, int64_t n,
                                                              int R, const double *__restrict__ w,
                                                              const double *__restrict__ U, int H,
                                                              int side, int64_t rows_pad, int Kpad,
                                                              float2 *__restrict__ blocks,
                                                              const double *__restrict__ kr,
                                                              const double *__restrict__ shifts, int S) {
    constexpr int Q = 1 << LOGQ;
    constexpr int L = 32;
    constexpr int E = Q / L;
    constexpr int N = Q / 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2 *tw = reinterpret_cast<float2 *>(smem_raw);              // [E][L]
    float2 *at = tw + E * L;                                        // [CP_HC][Q]
    float *up = reinterpret_cast<float *>(at + CP_HC * Q);          // [R][CP_HC]

    const int64_t row = blockIdx.x;                  // output row = base * S + shift
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < E * L; i += CP_THREADS) tw[i] = twiddle_N(i % L, i / L, Q);
    float2 stw[clog2(L)];
    lane_stage_twiddles<L>(lane, stw);
    const float2 *ring = rings + (row / S) * (int64_t)R * Q;
    double dx = 0.0, dy = 0.0;                       // row f2: translated copy (row % S) of the base row
    if (shifts) { dx = shifts[2 * (row % S)]; dy = shifts[2 * (row % S) + 1]; }
    const double invQ = 1.0 / (double)Q;

    for (int h0 = 0; h0 < H; h0 += CP_HC) {
        const int hc = min(CP_HC, H - h0);
        __syncthreads();
        for (int i = tid; i < R * CP_HC; i += CP_THREADS) {
            const int r = i / CP_HC, hh = i % CP_HC;
            up[i] = (hh < hc) ? (float)(U[(int64_t)r * H + h0 + hh] * sqrt(w[r]) * invQ) : 0.f;
        }
        __syncthreads();
        // psi-space projection: at[hh][j] = sum_r up[r][hh] a[r][j]
        for (int j = tid; j < Q; j += CP_THREADS) {
            float2 acc[CP_HC];
#pragma unroll
            for (int hh = 0; hh < CP_HC; ++hh) acc[hh] = make_float2(0.f, 0.f);
            float uj = 0.f;
            if (shifts) {
                double sn, cs;
                sincospi(2.0 * (double)j / (double)Q, &sn, &cs);
                uj = (float)(dx * cs + dy * sn);
            }
            for (int r = 0; r < R; ++r) {
                float2 a = __ldg(ring + (int64_t)r * Q + j);
                if (shifts) {                        // a exp(-i k_r (dx cos psi_j + dy sin psi_j))
                    float sn, cs;
                    __sincosf(-(float)kr[r] * uj, &sn, &cs);   // |arg| <~ 2 rad: abs error ~4e-7
                    a = make_float2(a.x * cs - a.y * sn, a.x * sn + a.y * cs);
                }
                const float4 *u4 = reinterpret_cast<const float4 *>(up + r * CP_HC);
#pragma unroll
                for (int g = 0; g < CP_HC / 4; ++g) {
                    const float4 u = u4[g];
                    acc[4 * g + 0] = __ffma2_rn(a, make_float2(u.x, u.x), acc[4 * g + 0]);
                    acc[4 * g + 1] = __ffma2_rn(a, make_float2(u.y, u.y), acc[4 * g + 1]);
                    acc[4 * g + 2] = __ffma2_rn(a, make_float2(u.z, u.z), acc[4 * g + 2]);
                    acc[4 * g + 3] = __ffma2_rn(a, make_float2(u.w, u.w), acc[4 * g + 3]);
                }
            }
#pragma unroll
            for (int hh = 0; hh < CP_HC; ++hh) at[hh * Q + j] = acc[hh];
        }
        __syncthreads();
        // length-Q forward DFT of each principal ring (warp per ring)
        for (int hh = warp; hh < hc; hh += CP_THREADS / 32) {
            float2 v[E];
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = at[hh * Q + lane + L * e];
            fft_dist<E, L>(v, lane, tw, stw);
            const int h = h0 + hh;
            const int b = (int)(__brev((unsigned)lane) >> 27);
#pragma unroll
            for (int k1 = 0; k1 < E; ++k1) {
                const int q = k1 + E * b;
                const float2 X = v[brev(k1, clog2(E))];
                if (q <= N) {
                    const float2 val = side == RSVD_SIDE_IMAGE ? c_conj(X) : X;
                    blocks[((int64_t)q * Kpad + h) * rows_pad + row] = val;
                }
                if (q >= N || q == 0) {
                    const int qq = (Q - q) & (Q - 1);
                    const float2 val = side == RSVD_SIDE_IMAGE ? X : c_conj(X);
                    blocks[((int64_t)qq * Kpad + H + h) * rows_pad + row] = val;
                }
            }
        }
    }
}

// canonical coefficients coeffs[n][q][h] from the block layout (test / debug path)
__global__ void unpack_kernel(const float2 *__restrict__ blocks, int64_t n, int Q, int H, int side,
                              int64_t rows_pad, int Kpad, float2 *__restrict__ coeffs) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = n * (int64_t)Q * H;
    if (idx >= total) return;
    const int h = (int)(idx % H);
    const int q = (int)((idx / H) % Q);
    const int64_t row = idx / ((int64_t)H * Q);
    const int N = Q / 2;
    float2 v;
    if (q <= N) {
        v = blocks[((int64_t)q * Kpad + h) * rows_pad + row];
        if (side == RSVD_SIDE_IMAGE) v = c_conj(v);
    } else {
        v = blocks[((int64_t)(Q - q) * Kpad + H + h) * rows_pad + row];
        if (side == RSVD_SIDE_TEMPLATE) v = c_conj(v);
    }
    coeffs[idx] = v;
}

template <int LOGQ>
static cudaError_t launch_compress(const float2 *rings, int64_t n, int R, const double *w,
                                   const double *U, int H, int side, int64_t rows_pad, int Kpad,
                                   float2 *blocks, const double *kr, const double *shifts, int S, cudaStream_t s) {
    constexpr int Q = 1 << LOGQ;
    const size_t smem = (size_t)Q * sizeof(float2) + (size_t)CP_HC * Q * sizeof(float2) +
                        (size_t)R * CP_HC * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(compress_kernel<LOGQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    const bool timed = timing_enabled();
    cudaEvent_t ev0 = timed ? timing_event(s) : nullptr;
    compress_kernel<LOGQ><<<(unsigned)n, CP_THREADS, smem, s>>>(rings, n, R, w, U, H, side, rows_pad,
                                                                 Kpad, blocks, kr, shifts, S);
    e = cudaGetLastError();
    if (e == cudaSuccess) {
        count_launches(1);
        if (timed) timing_span(ev0, timing_event(s), TK_COMPRESS);
    }
    return e;
}

}  // namespace rsvd

using namespace rsvd;

extern "C" int64_t rsvd_block_bytes(int64_t rows, int32_t Q, int32_t H, rsvd_side side) {
    if (rows < 0 || Q < 2 || H < 1) return -1;
    if (resolve_path(Q, H) == PATH_TC) return tc_block_bytes(rows, Q, H, side);
    return (int64_t)(Q / 2 + 1) * kpad_of(H) * rows_pad_of(rows) * (int64_t)sizeof(float2);
}

// n = output rows (base rows * S); shifts == NULL is the plain compress (S = 1)
static rsvd_status compress_impl(const void *rings, int64_t n, int32_t R, int32_t Q, const double *w,
                                 const double *U, int32_t H, rsvd_side side, void *blocks, const double *kr,
                                 const double *shifts, int32_t S, rsvd_stream_t stream) {
    if (R <= 0) return fail(RSVD_ERR_ARG, "R must be positive");
    if (R > 256) return fail(RSVD_ERR_UNSUPPORTED, "R > 256 is not supported");
    if (Q <= 0) return fail(RSVD_ERR_ARG, "Q must be positive");
    if (!is_pow2(Q) || Q < 32 || Q > 1024) return fail(RSVD_ERR_UNSUPPORTED, "Q must be a power of two in [32, 1024]");
    if (H < 1 || H > R) return fail(RSVD_ERR_UNSUPPORTED, "H must satisfy 1 <= H <= R");
    if (side != RSVD_SIDE_IMAGE && side != RSVD_SIDE_TEMPLATE) return fail(RSVD_ERR_ARG, "bad side");
    if (n < 0) return fail(RSVD_ERR_ARG, "n must be >= 0");
    if (n == 0) return RSVD_OK;
    if (n > 0x7fffffffLL) return fail(RSVD_ERR_UNSUPPORTED, "too many rows in one call");
    if (!rings || !w || !U || !blocks) return fail(RSVD_ERR_ARG, "NULL pointer");
    if (!aligned16(rings) || !aligned16(blocks)) return fail(RSVD_ERR_ARG, "complex buffers must be 16-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    if (resolve_path(Q, H) == PATH_TC) {
        if (tc_rows_pad_side(n, side) > n) {
            cudaError_t e = cudaMemsetAsync(blocks, 0, (size_t)tc_block_bytes(n, Q, H, side), s);
            if (e != cudaSuccess) return cuda_check(e, "memset blocks");
        }
        const bool timed = timing_enabled();
        cudaEvent_t ev0 = timed ? timing_event(s) : nullptr;
        cudaError_t e = launch_compress_tc(reinterpret_cast<const float2 *>(rings), n, R, Q, w, U, H, side,
                                           reinterpret_cast<float *>(blocks), kr, shifts, S, s);
        if (e == cudaSuccess) {
            count_launches(1);
            if (timed) timing_span(ev0, timing_event(s), TK_COMPRESS);
        }
        return cuda_check(e, "compress (tc layout) launch");
    }
    const int Kpad = (int)kpad_of(H);
    const int64_t rows_pad = rows_pad_of(n);
    if (Kpad > 2 * H || rows_pad > n) {
        cudaError_t e = cudaMemsetAsync(blocks, 0, (size_t)rsvd_block_bytes(n, Q, H, side), s);
        if (e != cudaSuccess) return cuda_check(e, "memset blocks");
    }
    const float2 *rg = reinterpret_cast<const float2 *>(rings);
    float2 *bl = reinterpret_cast<float2 *>(blocks);
    cudaError_t e;
    switch (ilog2(Q)) {
        case 5: e = launch_compress<5>(rg, n, R, w, U, H, side, rows_pad, Kpad, bl, kr, shifts, S, s); break;
        case 6: e = launch_compress<6>(rg, n, R, w, U, H, side, rows_pad, Kpad, bl, kr, shifts, S, s); break;
        case 7: e = launch_compress<7>(rg, n, R, w, U, H, side, rows_pad, Kpad, bl, kr, shifts, S, s); break;
        case 8: e = launch_compress<8>(rg, n, R, w, U, H, side, rows_pad, Kpad, bl, kr, shifts, S, s); break;
        case 9: e = launch_compress<9>(rg, n, R, w, U, H, side, rows_pad, Kpad, bl, kr, shifts, S, s); break;
        default: e = launch_compress<10>(rg, n, R, w, U, H, side, rows_pad, Kpad, bl, kr, shifts, S, s); break;
    }
    return cuda_check(e, "compress launch");
}

extern "C" rsvd_status rsvd_compress(const void *rings, int64_t n, int32_t R, int32_t Q, const double *w,
                                     const double *U, int32_t H, rsvd_side side, void *blocks,
                                     rsvd_stream_t stream) {
    return compress_impl(rings, n, R, Q, w, U, H, side, blocks, nullptr, nullptr, 1, stream);
}

extern "C" rsvd_status rsvd_compress_translated(const void *rings, int64_t n_base, int32_t R, int32_t Q,
                                                const double *w, const double *k, const double *U, int32_t H,
                                                const double *shifts, int32_t S, rsvd_side side, void *blocks,
                                                rsvd_stream_t stream) {
    if (S < 1) return fail(RSVD_ERR_ARG, "S must be >= 1");
    if (n_base < 0) return fail(RSVD_ERR_ARG, "n_base must be >= 0");
    if (n_base > 0x7fffffffLL / S) return fail(RSVD_ERR_UNSUPPORTED, "too many rows in one call");
    if (n_base > 0 && (!k || !shifts)) return fail(RSVD_ERR_ARG, "NULL pointer");
    return compress_impl(rings, n_base * S, R, Q, w, U, H, side, blocks, k, shifts, S, stream);
}

extern "C" rsvd_status rsvd_blocks_unpack(const void *blocks, int64_t n, int32_t Q, int32_t H, rsvd_side side,
                                          void *coeffs, rsvd_stream_t stream) {
    if (Q <= 0 || !is_pow2(Q) || Q < 32 || Q > 1024) return fail(RSVD_ERR_UNSUPPORTED, "Q must be a power of two in [32, 1024]");
    if (H < 1) return fail(RSVD_ERR_ARG, "H must be >= 1");
    if (n < 0) return fail(RSVD_ERR_ARG, "n must be >= 0");
    if (n == 0) return RSVD_OK;
    if (!blocks || !coeffs) return fail(RSVD_ERR_ARG, "NULL pointer");
    if (resolve_path(Q, H) == PATH_TC) {
        cudaError_t e = launch_unpack_tc(reinterpret_cast<const float *>(blocks), n, Q, H, side,
                                         reinterpret_cast<float2 *>(coeffs), (cudaStream_t)stream);
        count_launches(1);
        return cuda_check(e, "unpack (tc layout) launch");
    }
    const int64_t total = n * (int64_t)Q * H;
    unpack_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const float2 *>(blocks), n, Q, H, side, rows_pad_of(n), (int)kpad_of(H),
        reinterpret_cast<float2 *>(coeffs));
    count_launches(1);
    return cuda_check(cudaGetLastError(), "unpack launch");
}
