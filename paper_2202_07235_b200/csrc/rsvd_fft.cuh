// rsvd_fft.cuh -- Steps 3-4 of the align path: length-Q landscape transform of each pair's packed
// spectrum (forward sign per DESIGN.md G3) fused with the argmax over gamma
// or the landscape store.
//
// Input: the contraction's planar workspace (re plane, then im plane, each [(n * Mc + ml) * Tc + tl]
// floats, q-major), n < N = Q/2, holding
// U_n = S_n + conj(S_{Q-n}) for n in [1, N) and (U_0, U_N) packed in slot 0.  With Y = U/2 (the
// Hermitian part of S, whose transform is Re X), the real length-Q transform is computed as one
// complex length-N FFT of Z_n = (Y_n + conj Y_{N-n}) + i W_Q^n (Y_n - conj Y_{N-n}); its output
// z_n = x_{2n} + i x_{2n+1} with Re X_k = 2 pi x_k.
//
// Schedule: persistent CTAs loop over work items (one template x TB images); the TB spectra of
// the next item are prefetched into shared memory with cp.async while the current item is
// transformed (double buffer).  Per pair (one warp): Z formation from the staged spectra,
// in-register DIF of length E = N/32 over x[l + 32 e], twiddle W_N^{l k1}, one warp transpose through
// shared memory, then length-32 sub-DFTs as fft_dist<E, 32/E> (in-register DIF + log2(32/E) shuffle
// stages).  N <= 32 uses one shuffle pass with 32/N pairs per warp.
#pragma once

#include "rsvd_common.cuh"

namespace rsvd {

enum { MODE_PAIR = 0, MODE_IMAGE = 1, MODE_LANDSCAPE = 2 };
constexpr int FR_THREADS = 256;
constexpr int FR_WARPS = FR_THREADS / 32;

__device__ __forceinline__ uint32_t ord_f32(float v) {
    const uint32_t u = __float_as_uint(v);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit_fr() { asm volatile("cp.async.commit_group;\n" ::); }
template <int NWAIT>
__device__ __forceinline__ void cp_async_wait_fr() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NWAIT)); }

template <int N>
struct FftCfg {
    static constexpr int L = N < 32 ? N : 32;      // lanes per pair in the first pass
    static constexpr int E = N / L;                // elements per lane
    static constexpr int GP = 32 / L;              // pairs per warp in flight (N < 32)
    static constexpr int G = E > 1 ? 32 / E : 1;   // lanes per length-32 sub-DFT after the transpose
    static constexpr int TB = N >= 512 ? 8 : 16;   // templates per work item
    static constexpr int P = 32 + G;               // transpose row stride (8-byte units); P = G mod 16
    static constexpr int SROW = TB + 1;            // staged spectrum row stride (odd: conflict-free columns)
    static constexpr int SBUF = N * SROW;          // float2 per stage buffer
    static constexpr int V = TB / 4;               // float4 per plane row of an item
    static constexpr int RPP = FR_THREADS / V;     // rows per staging pass
    static constexpr int PASSES = (N + RPP - 1) / RPP;
    static constexpr size_t smem_bytes() {
        return (size_t)SBUF * 8 + (E > 1 ? (size_t)FR_WARPS * E * P * 8 : 0) + (size_t)N * 8 + 16;
    }
};

struct FftOut {
    float *best_val;
    int32_t *best_k;
    unsigned long long *best_key;
    float *X;
    int64_t ld_m, ld_t, T, t_offset;
};

template <int LOGN, int MODE>
__global__ void __launch_bounds__(FR_THREADS) fft_reduce_kernel(const float *__restrict__ Upk, int64_t Mc,
                                                                int64_t Tc, int64_t m0, int64_t t0, int64_t mcv,
                                                                int64_t tcv, FftOut out) {
    constexpr int N = 1 << LOGN;
    constexpr int Q = 2 * N;
    using C = FftCfg<N>;
    constexpr int L = C::L, E = C::E, G = C::G, GP = C::GP, TB = C::TB, P = C::P, SROW = C::SROW;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2 *S = reinterpret_cast<float2 *>(smem_raw);                  // [N][SROW] staged spectra
    float2 *Xs = S + C::SBUF;                                           // [warps][E][P] transpose scratch
    float2 *pre = Xs + (E > 1 ? FR_WARPS * E * P : 0);                 // [N]      W_Q^n (E == 1 path)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // work item = (template tl, block of TB consecutive images); workspace [plane][n][t][m]
    const int64_t nmb = (mcv + TB - 1) / TB;
    const int64_t nitems = tcv * nmb;

    // Staging: 16-byte loads of the re / im plane rows of an item into registers (issued one item
    // ahead, so their latency hides behind the transform), then 8-byte stores of (re, im) pairs into
    // the odd-stride interleaved tile S[n][SROW] (conflict-free both ways).
    const int64_t plane4 = (int64_t)N * Mc * Tc / 4;
    const int64_t row4 = Mc * Tc / 4;
    const int n0 = tid / C::V, c4 = tid % C::V;
    float4 rre[C::PASSES], rim[C::PASSES];
    auto load = [&](int64_t it) {
        const int64_t tl = it / nmb, mb0 = (it % nmb) * TB;
        const float4 *g = reinterpret_cast<const float4 *>(Upk + tl * Mc + mb0) + (int64_t)n0 * row4 + c4;
#pragma unroll
        for (int j = 0; j < C::PASSES; ++j) {
            if (n0 + j * C::RPP < N) {
                rre[j] = __ldg(g + (int64_t)j * C::RPP * row4);
                rim[j] = __ldg(g + (int64_t)j * C::RPP * row4 + plane4);
            }
        }
    };
    auto store = [&]() {
#pragma unroll
        for (int j = 0; j < C::PASSES; ++j) {
            const int n = n0 + j * C::RPP;
            if (n < N) {
                float2 *d = S + n * SROW + 4 * c4;
                d[0] = make_float2(rre[j].x, rim[j].x);
                d[1] = make_float2(rre[j].y, rim[j].y);
                d[2] = make_float2(rre[j].z, rim[j].z);
                d[3] = make_float2(rre[j].w, rim[j].w);
            }
        }
    };

    int64_t item = blockIdx.x;
    if (item < nitems) { load(item); store(); }
    if (item + gridDim.x < nitems) load(item + gridDim.x);
    for (int i = tid; i < N && E == 1; i += FR_THREADS) {
        float sn, cs;
        sincospif(2.0f * (float)i / (float)Q, &sn, &cs);
        pre[i] = make_float2(cs, -sn);
    }
    __syncthreads();

    const float PI = 3.14159265358979323846f;
    // per-lane constants
    const int g1 = lane / L, l1 = lane % L;                  // E == 1 layout
    const int k1p = lane / G, s2 = lane % G;                 // E > 1 layout after the transpose
    float2 stwL[clog2(L) > 0 ? clog2(L) : 1];
    float2 stwG[clog2(G) > 0 ? clog2(G) : 1];
    lane_stage_twiddles<L>(l1, stwL);
    lane_stage_twiddles<G>(s2, stwG);
    float2 *xw = Xs + warp * E * P;
    float2 preR[E], twNR[E], tw32R[E];                   // per-lane twiddles (E > 1 path)
#pragma unroll
    for (int e = 0; e < E; ++e) {
        float sn, cs;
        sincospif(2.0f * (float)(lane + 32 * e) / (float)Q, &sn, &cs);
        preR[e] = make_float2(cs, -sn);                  // W_Q^{l + 32 e}
        twNR[e] = twiddle_N(lane, e, N);                 // W_N^{l e}
        tw32R[e] = twiddle_N(s2, e, 32);                 // W_32^{s e}
    }

    for (; item < nitems; item += gridDim.x) {
        const int64_t tl = item / nmb, mb0 = (item % nmb) * TB;
        const int64_t t = t0 + tl;

        if constexpr (E == 1) {
            const float2 one = make_float2(1.f, 0.f);
            for (int tt = warp * GP + g1; tt < TB; tt += FR_WARPS * GP) {
                const int64_t ml = mb0 + tt;
                const bool valid = ml < mcv;
                const int64_t m = m0 + ml;
                float2 z[1];
                const float2 u = S[l1 * SROW + tt];
                if (l1 == 0) {
                    z[0] = make_float2(u.x + u.y, u.x - u.y);
                } else {
                    const float2 mm = S[(N - l1) * SROW + tt];
                    const float2 sm = make_float2(u.x + mm.x, u.y - mm.y);
                    const float2 d = make_float2(u.x - mm.x, u.y + mm.y);
                    const float2 wd = c_mul(pre[l1], d);
                    z[0] = make_float2(sm.x - wd.y, sm.y + wd.x);
                }
                fft_dist<1, L>(z, l1, &one, stwL);
                const int b = (int)(__brev((unsigned)l1) >> (32 - clog2(L)));
                const float vx = PI * z[0].x, vy = PI * z[0].y;
                if constexpr (MODE == MODE_LANDSCAPE) {
                    if (valid)
                        reinterpret_cast<float2 *>(out.X + m * out.ld_m + t * out.ld_t)[b] = make_float2(vx, vy);
                } else {
                    float bv = vx;
                    int bk = 2 * b;
                    if (vy > bv) { bv = vy; bk = 2 * b + 1; }
#pragma unroll
                    for (int off = L / 2; off >= 1; off >>= 1) {
                        const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
                        const int ok = __shfl_xor_sync(0xffffffffu, bk, off);
                        if (ov > bv || (ov == bv && ok < bk)) { bv = ov; bk = ok; }
                    }
                    if constexpr (MODE == MODE_PAIR) {
                        if (valid && l1 == 0) {
                            out.best_val[m * out.T + t] = bv;
                            out.best_k[m * out.T + t] = bk;
                        }
                    } else if (valid) {
                        const uint32_t idx = (uint32_t)((out.t_offset + t) * Q + bk);
                        const unsigned long long key =
                            ((unsigned long long)ord_f32(bv) << 32) | (unsigned long long)(0xFFFFFFFFu - idx);
                        if (l1 == 0) atomicMax(out.best_key + m, key);
                    }
                }
            }
        } else {
            const int l = lane;
            // affine per-lane row pointers: u at rows l + 32e, mirror at rows N - l - 32e
            const float2 *su = S + l * SROW;
            const float2 *sm_ = S + (N - l) * SROW;
            for (int tt = warp; tt < TB; tt += FR_WARPS) {
                const int64_t ml = mb0 + tt;
                const bool valid = ml < mcv;
                const int64_t m = m0 + ml;
                float2 z[E];
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const float2 u = su[e * 32 * SROW + tt];
                    const float2 mm = sm_[tt - e * 32 * SROW];                 // row N - n (l = 0, e = 0: unused)
                    const float2 sm = make_float2(u.x + mm.x, u.y - mm.y);     // U + conj M
                    const float2 d = make_float2(u.x - mm.x, u.y + mm.y);      // U - conj M
                    const float2 wd = c_mul(preR[e], d);
                    z[e] = make_float2(sm.x - wd.y, sm.y + wd.x);              // (s + i w d), pi applied last
                }
                if (l == 0) z[0] = make_float2(S[tt].x + S[tt].y, S[tt].x - S[tt].y);   // n = 0: (U_0, U_N)
                dif_reg<E>(z);
#pragma unroll
                for (int k1 = 1; k1 < E; ++k1) {
                    const int r = brev(k1, clog2(E));
                    z[r] = c_mul(z[r], twNR[k1]);
                }
                __syncwarp();
#pragma unroll
                for (int k1 = 0; k1 < E; ++k1) xw[k1 * P + l] = z[brev(k1, clog2(E))];
                __syncwarp();
#pragma unroll
                for (int u = 0; u < E; ++u) z[u] = xw[k1p * P + s2 + G * u];
                dif_reg<E>(z);
#pragma unroll
                for (int k = 1; k < E; ++k) {
                    const int r = brev(k, clog2(E));
                    z[r] = c_mul(z[r], tw32R[k]);
                }
                dif_lanes<E, G>(z, s2, stwG);
                const int b = (int)(__brev((unsigned)s2) >> (32 - clog2(G)));
                if constexpr (MODE == MODE_LANDSCAPE) {
                    if (valid) {
                        float2 *dst = reinterpret_cast<float2 *>(out.X + m * out.ld_m + t * out.ld_t);
#pragma unroll
                        for (int k2a = 0; k2a < E; ++k2a) {
                            const float2 v = z[brev(k2a, clog2(E))];
                            dst[k1p + E * (k2a + E * b)] = make_float2(PI * v.x, PI * v.y);
                        }
                    }
                } else {
                    float bv = -INFINITY;
                    int bk = 0x7fffffff;
#pragma unroll
                    for (int k2a = 0; k2a < E; ++k2a) {          // index increases with k2a for a fixed lane
                        const float2 v = z[brev(k2a, clog2(E))];
                        const int kk = 2 * (k1p + E * (k2a + E * b));
                        if (v.x > bv) { bv = v.x; bk = kk; }
                        if (v.y > bv) { bv = v.y; bk = kk + 1; }
                    }
#pragma unroll
                    for (int off = 16; off >= 1; off >>= 1) {
                        const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
                        const int ok = __shfl_xor_sync(0xffffffffu, bk, off);
                        if (ov > bv || (ov == bv && ok < bk)) { bv = ov; bk = ok; }
                    }
                    bv *= PI;
                    if constexpr (MODE == MODE_PAIR) {
                        if (valid && l == 0) {
                            out.best_val[m * out.T + t] = bv;
                            out.best_k[m * out.T + t] = bk;
                        }
                    } else if (valid) {
                        const uint32_t idx = (uint32_t)((out.t_offset + t) * Q + bk);
                        const unsigned long long key =
                            ((unsigned long long)ord_f32(bv) << 32) | (unsigned long long)(0xFFFFFFFFu - idx);
                        if (l == 0) atomicMax(out.best_key + m, key);
                    }
                }
            }
        }
        __syncthreads();                                 // everyone is done with S
        const int64_t next = item + gridDim.x;
        if (next < nitems) {
            store();                                     // item `next` (loaded one iteration ago)
            if (next + gridDim.x < nitems) load(next + gridDim.x);
        }
        __syncthreads();
    }
}

inline int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

template <int LOGN, int MODE>
static cudaError_t launch_fft_mode(cudaStream_t s, const float *Upk, int64_t Mc, int64_t Tc, int64_t m0, int64_t t0,
                                   int64_t mcv, int64_t tcv, const FftOut &out) {
    using C = FftCfg<(1 << LOGN)>;
    const size_t smem = C::smem_bytes();
    static int occ = 0;
    if (!occ) {
        cudaError_t e = cudaFuncSetAttribute(fft_reduce_kernel<LOGN, MODE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fft_reduce_kernel<LOGN, MODE>, FR_THREADS, smem);
        if (e != cudaSuccess || occ < 1) occ = 1;
    }
    const int64_t nitems = tcv * ((mcv + C::TB - 1) / C::TB);
    const int64_t grid = std::min<int64_t>(nitems, (int64_t)num_sms() * occ);
    fft_reduce_kernel<LOGN, MODE><<<(unsigned)grid, FR_THREADS, smem, s>>>(Upk, Mc, Tc, m0, t0, mcv, tcv, out);
    return cudaGetLastError();
}

template <int LOGN>
static cudaError_t launch_fft(int mode, cudaStream_t s, const float *Upk, int64_t Mc, int64_t Tc, int64_t m0,
                              int64_t t0, int64_t mcv, int64_t tcv, const FftOut &out) {
    if (mode == MODE_PAIR) return launch_fft_mode<LOGN, MODE_PAIR>(s, Upk, Mc, Tc, m0, t0, mcv, tcv, out);
    if (mode == MODE_IMAGE) return launch_fft_mode<LOGN, MODE_IMAGE>(s, Upk, Mc, Tc, m0, t0, mcv, tcv, out);
    return launch_fft_mode<LOGN, MODE_LANDSCAPE>(s, Upk, Mc, Tc, m0, t0, mcv, tcv, out);
}

}  // namespace rsvd
