// rsvd_fft.cuh -- Steps 3-4 of the align path: length-Q landscape transform of each pair's packed
// spectrum (forward sign per DESIGN.md G3) fused with the argmax over gamma
// or the landscape store.
//
// Input: the contraction's planar workspace (re plane, then im plane, each [(n * Tc + tl) * Mc + ml]
// floats, image index fastest), n < N = Q/2, holding U_n = S_n + conj(S_{Q-n}) for n in [1, N) and
// (U_0, U_N) packed in slot 0.  With Y = U/2 (the Hermitian part of S, whose transform is Re X) the
// real length-Q transform is one complex length-N FFT of
//   Z_n = (Y_n + conj Y_{N-n}) + i W_Q^n (Y_n - conj Y_{N-n}),
// whose output z_k = x_{2k} + i x_{2k+1}, Re X_k = 2 pi x_k.  Z is formed from U (= 2Y), so the
// transform carries a factor 2 and the result is scaled by pi.
//
// Schedule (persistent CTAs; work item = one template x TB images, TB * N1 = 256 threads):
//   TMA     thread 0 streams item i+2's 2N plane rows x TB images (one 3-D tensor-map box per 256
//           rows) into a 2-deep shared ring, completion on an mbarrier -- no registers held in
//           flight, and the request is issued as soon as the ring slot is consumed;
//   stage   one thread per (row pair {n, N-n}, 4 images): Z_n and Z_{N-n} from the same two values
//           (Z_{N-n} = conj(s) + i conj(W d) when Z_n = s + i W d) into ZY[image][n];
//   pass 1  one thread per (image, n1): in-register DIF DFT of length N2 over Z[n1 + N1 n2],
//           twiddle W_N^{n1 k1}, written back in place (after a barrier) as
//           ZY[image][k1 N1 + (n1 ^ sw(k1))] -- the XOR swizzle makes the pass-2 column reads
//           conflict-free;
//   pass 2  one thread per (image, k1): in-register DIF DFT of length N1 over n1, giving
//           z[k1 + N2 k2]; landscape store, or max then first-argmax over the N2 lanes of the pair.
// Both passes are shuffle-free FFMA/FADD work with N2 (N1) independent complex values per thread.
#pragma once

#include <cuda.h>
#include <stdlib.h>

#include "rsvd_common.cuh"

namespace rsvd {

enum { MODE_PAIR = 0, MODE_IMAGE = 1, MODE_LANDSCAPE = 2 };
constexpr int FR_THREADS = 256;

__device__ __forceinline__ uint32_t ord_f32(float v) {
    const uint32_t u = __float_as_uint(v);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

template <int LOGN>
struct FftCfg {
    static constexpr int N = 1 << LOGN;
    static constexpr int Q = 2 * N;
    static constexpr int NH = N / 2;
    static constexpr int N1 = 1 << (LOGN / 2);        // pass-2 DFT length = threads per image in pass 1
    static constexpr int N2 = N / N1;                 // pass-1 DFT length = threads per image in pass 2
    static constexpr int TB = FR_THREADS / N1;        // images per work item
    static constexpr int C4 = TB / 4;                 // float4 columns per plane row of an item
    static constexpr int ST_TASKS = NH * C4;          // staging tasks: (row pair, 4 images)
    static constexpr int ST_PER = (ST_TASKS + FR_THREADS - 1) / FR_THREADS;
    static constexpr int P2_PER = TB * N2 / FR_THREADS;
    static constexpr int SZ = N + 1;                  // ZY row stride (float2): SZ = 1 mod 4
    static constexpr int SWD = N1 >= 16 ? 1 : 16 / N1;
    static constexpr int ROWS = 2 * N;                // plane rows of an item (re then im)
    static constexpr int BOXR = ROWS < 256 ? ROWS : 256;
    static constexpr int NBOX = ROWS / BOXR;
    static constexpr int UBYTES = ROWS * TB * 4;      // one ring slot
    static constexpr int NST = 2;
    static constexpr size_t smem_bytes() {
        return 1024 + (size_t)NST * UBYTES + (size_t)TB * SZ * 8 + (size_t)NH * 8 + (size_t)N2 * N1 * 8 + 64;
    }
};

struct FftOut {
    float *best_val;
    int32_t *best_k;
    unsigned long long *best_key;
    float *X;
    int64_t ld_m, ld_t, T, t_offset;
    const float *sc_m, *sc_t;      // TC path: exact power-of-two row scales of the operands (NULL = 1)
    float *best_gamma;             // PER_PAIR, optional: parabolic-refined argmax angle (radians)
};

// 3-point parabolic refinement of the first argmax bk (SPEC.md argmax_refine, reading in DESIGN.md):
// the lanes of a pair hold Re X at k = 2 (k1 + N2 k2) + {0, 1} in wj[brev(k2)] (x, y); the samples at
// bk -+ 1 (cyclic) are fetched from their owner lanes, gamma = 2 pi (bk + d) / Q with the vertex
// offset d = (y- - y+) / (2 (y- - 2 y0 + y+)) clamped to [-1/2, 1/2] (0 when not a strict maximum).
template <int N1, int N2, bool R4 = false>
__device__ __forceinline__ float parabolic_gamma(const float2 (&wj)[N1], int k1, int bk, float y0, unsigned gmask) {
    constexpr int Qn = 2 * N1 * N2;
    auto fetch = [&](int i) {
        const int c = i >> 1, kk1 = c % N2, kk2 = c / N2;
        float v = 0.f;
        if (kk1 == k1) {
#pragma unroll
            for (int k2 = 0; k2 < N1; ++k2)
                if (k2 == kk2) {
                    const float2 z = wj[R4 ? dpos4<N1>(k2) : brev(k2, clog2(N1))];
                    v = (i & 1) ? z.y : z.x;
                }
        }
#pragma unroll
        for (int off = N2 / 2; off >= 1; off >>= 1) v += __shfl_xor_sync(gmask, v, off);   // one nonzero term
        return v;
    };
    const float ym = fetch((bk - 1) & (Qn - 1)), yp = fetch((bk + 1) & (Qn - 1));
    const float den = ym - 2.f * y0 + yp;
    float d = den < 0.f ? 0.5f * (ym - yp) / den : 0.f;
    d = fminf(0.5f, fmaxf(-0.5f, d));
    float g = 6.283185307179586f * ((float)bk + d) / (float)Qn;
    if (g < 0.f) g += 6.283185307179586f;
    return g;
}

__device__ __forceinline__ uint32_t fr_smem(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void fr_mbar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "FR_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra FR_WAIT;\n\t}" ::"r"(fr_smem(b)),
        "r"(parity)
        : "memory");
}

template <int LOGN, int MODE>
__global__ void __launch_bounds__(FR_THREADS, 2) fft_reduce_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                   int64_t Mc, int64_t Tc, int64_t m0, int64_t t0,
                                                                   int64_t mcv, int64_t tcv, FftOut out) {
    using C = FftCfg<LOGN>;
    constexpr int N = C::N, Q = C::Q, NH = C::NH, N1 = C::N1, N2 = C::N2, TB = C::TB, C4 = C::C4, SZ = C::SZ;
    constexpr int SP = C::ST_PER;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // pointer arithmetic on the __shared__ array (not an integer round trip) keeps LDS/STS addressing
    unsigned char *base = smem_raw + ((1024u - (fr_smem(smem_raw) & 1023u)) & 1023u);
    float *Ur = reinterpret_cast<float *>(base);                             // [NST][ROWS][TB]
    float2 *ZY = reinterpret_cast<float2 *>(base + C::NST * C::UBYTES);      // [TB][SZ]
    float2 *Wq = ZY + TB * SZ;                                               // [NH]  W_Q^r
    float2 *Tw = Wq + NH;                                                    // [N2][N1] W_N^{n1 k1}
    uint64_t *full = reinterpret_cast<uint64_t *>(Tw + N2 * N1);             // [NST]

    const int tid = threadIdx.x;
    const int nmb = (int)((mcv + TB - 1) / TB);                  // 32-bit item arithmetic
    const int nitems = (int)tcv * nmb;
    const int grid = (int)gridDim.x;
    (void)Mc; (void)Tc;

    auto issue = [&](int it, int slot) {                         // thread 0 only
        const int tl = it / nmb, mb0 = (it - tl * nmb) * TB;
        const uint32_t bar = fr_smem(full + slot);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((uint32_t)C::UBYTES)
                     : "memory");
#pragma unroll
        for (int bx = 0; bx < C::NBOX; ++bx) {
            const uint32_t dst = fr_smem(Ur + (size_t)slot * (C::UBYTES / 4) + (size_t)bx * C::BOXR * TB);
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                ::"r"(dst), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(mb0), "r"(tl), "r"(bx * C::BOXR), "r"(bar)
                : "memory");
        }
    };

    if (tid == 0) {
        for (int sl = 0; sl < C::NST; ++sl)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(fr_smem(full + sl)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int sl = 0; sl < C::NST; ++sl)
            if ((int)blockIdx.x + sl * grid < nitems) issue((int)blockIdx.x + sl * grid, sl);
    }
    for (int i = tid; i < NH; i += FR_THREADS) {
        float sn, cs;
        sincospif(2.0f * (float)i / (float)Q, &sn, &cs);
        Wq[i] = make_float2(cs, -sn);
    }
    for (int i = tid; i < N2 * N1; i += FR_THREADS) Tw[i] = twiddle_N(i % N1, i / N1, N);
    const int p1 = tid / N1, n1 = tid % N1;
    __syncthreads();

    const float PI = 3.14159265358979323846f;
    int kk = 0;
    for (int item = blockIdx.x; item < nitems; item += grid, ++kk) {
        const int slot = kk & 1;
        const int tl = item / nmb, mb0 = (item - tl * nmb) * TB;
        const int64_t t = t0 + tl;
        const float st = out.sc_t ? __ldg(out.sc_t + t) : 1.f;
        fr_mbar_wait(full + slot, (uint32_t)(kk >> 1) & 1u);

        // ---- stage: task q = tid + 256 i -> (row pair r = q / C4, column c4 = q % C4)
        {
            const float4 *U4 = reinterpret_cast<const float4 *>(Ur + (size_t)slot * (C::UBYTES / 4));
#pragma unroll
            for (int i = 0; i < SP; ++i) {
                const int q = tid + FR_THREADS * i;
                if (SP > 1 && q >= C::ST_TASKS) break;
                if (SP == 1 && q >= C::ST_TASKS) continue;
                const int r = q / C4, c4 = q % C4;
                const int rb = r ? N - r : NH;                 // r = 0 also carries the self-mirror row N/2
                const float4 a_re = U4[r * C4 + c4], a_im = U4[(N + r) * C4 + c4];
                const float4 b_re = U4[rb * C4 + c4], b_im = U4[(N + rb) * C4 + c4];
                const float ar[4] = {a_re.x, a_re.y, a_re.z, a_re.w}, ai[4] = {a_im.x, a_im.y, a_im.z, a_im.w};
                const float br[4] = {b_re.x, b_re.y, b_re.z, b_re.w}, bi[4] = {b_im.x, b_im.y, b_im.z, b_im.w};
                float2 *z = ZY + 4 * c4 * SZ;
                const float2 wq = Wq[r];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (r == 0) {
                        z[j * SZ] = make_float2(ar[j] + ai[j], ar[j] - ai[j]);      // n = 0: (U_0, U_N)
                        z[j * SZ + NH] = make_float2(2.f * br[j], 2.f * bi[j]);     // n = N/2: 2 U_{N/2}
                    } else {
                        const float sx = ar[j] + br[j], sy = ai[j] - bi[j];         // s = U_n + conj U_{N-n}
                        const float dx = ar[j] - br[j], dy = ai[j] + bi[j];         // d = U_n - conj U_{N-n}
                        const float px = wq.x * dx - wq.y * dy, py = wq.x * dy + wq.y * dx;
                        z[j * SZ + r] = make_float2(sx - py, sy + px);              // s + i p
                        z[j * SZ + N - r] = make_float2(sx + py, px - sy);          // conj(s) + i conj(p)
                    }
                }
            }
        }
        __syncthreads();                                       // (A) ZY holds Z; ring slot consumed
        if (tid == 0 && item + 2 * grid < nitems) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(item + 2 * grid, slot);
        }
        uint32_t stale[C::P2_PER];                             // MODE_IMAGE: image keys, read ahead
        if constexpr (MODE == MODE_IMAGE) {
#pragma unroll
            for (int j = 0; j < C::P2_PER; ++j) {
                const int ml = mb0 + (tid + FR_THREADS * j) / N2;
                stale[j] = ml < mcv ? (uint32_t)(__ldcg(out.best_key + m0 + ml) >> 32) : 0u;
            }
        }

        // ---- pass 1
        float2 v[N2];
        {
            const float2 *zr = ZY + p1 * SZ + n1;
#pragma unroll
            for (int n2 = 0; n2 < N2; ++n2) v[n2] = zr[N1 * n2];
        }
        __syncthreads();                                       // (B) all Z read: rewrite in place
        dif_reg<N2>(v);
        {
            float2 *yw = ZY + p1 * SZ;
#pragma unroll
            for (int k1 = 0; k1 < N2; ++k1) {
                float2 x = v[brev(k1, clog2(N2))];
                if (k1) x = c_mul(x, Tw[k1 * N1 + n1]);
                yw[k1 * N1 + (n1 ^ ((k1 / C::SWD) % N1))] = x;
            }
        }
        __syncthreads();                                       // (C) Y complete

        // ---- pass 2
        float2 w[C::P2_PER][N1];
#pragma unroll
        for (int j = 0; j < C::P2_PER; ++j) {
            const int task = tid + FR_THREADS * j;
            const int p = task / N2, k1 = task % N2;
            const float2 *yr = ZY + p * SZ + k1 * N1;
            const int sw = (k1 / C::SWD) % N1;
#pragma unroll
            for (int i = 0; i < N1; ++i) w[j][i] = yr[i ^ sw];
        }
        __syncthreads();                                       // (D) ZY free for the next item
#pragma unroll
        for (int j = 0; j < C::P2_PER; ++j) {
            const int task = tid + FR_THREADS * j;
            const int p = task / N2, k1 = task % N2;
            dif_reg<N1>(w[j]);                                 // w[brev(k2)] = z[k1 + N2 k2]
            const int64_t ml = mb0 + p;
            const bool valid = ml < mcv;
            const int64_t m = m0 + ml;
            // PI / (s_m s_t): exact power-of-two rescale of the TC path's scaled operands
            const float mul = PI / (((valid && out.sc_m) ? __ldg(out.sc_m + m) : 1.f) * st);
            if constexpr (MODE == MODE_LANDSCAPE) {
                if (valid) {
                    float2 *dst = reinterpret_cast<float2 *>(out.X + m * out.ld_m + t * out.ld_t);
#pragma unroll
                    for (int k2 = 0; k2 < N1; ++k2) {
                        const float2 z = w[j][brev(k2, clog2(N1))];
                        dst[k1 + N2 * k2] = make_float2(mul * z.x, mul * z.y);
                    }
                }
            } else {
                const unsigned gmask = N2 >= 32 ? 0xffffffffu
                                                : (((1u << (N2 & 31)) - 1u) << ((threadIdx.x & 31) & ~(N2 - 1)));
                float mx = -INFINITY;
#pragma unroll
                for (int k2 = 0; k2 < N1; ++k2) mx = fmaxf(mx, fmaxf(w[j][k2].x, w[j][k2].y));
#pragma unroll
                for (int off = N2 / 2; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(gmask, mx, off));
                const float bv = mul * mx;
                bool go = valid;
                if constexpr (MODE == MODE_IMAGE) {
                    // filter against a possibly stale copy of the image's key: keys only grow, so a
                    // pair whose value is below it can never win (ties fall through to the key compare)
                    go = valid && ord_f32(bv) >= stale[j];
                }
                if (go) {                                      // uniform over the pair's lanes
                    int bk = 0x7fffffff;
#pragma unroll
                    for (int k2 = N1 - 1; k2 >= 0; --k2) {     // descending: the smallest index wins
                        const float2 z = w[j][brev(k2, clog2(N1))];
                        const int kx = 2 * (k1 + N2 * k2);
                        if (z.y == mx) bk = kx + 1;
                        if (z.x == mx) bk = kx;
                    }
#pragma unroll
                    for (int off = N2 / 2; off >= 1; off >>= 1) bk = min(bk, __shfl_xor_sync(gmask, bk, off));
                    float gam = 0.f;
                    if constexpr (MODE == MODE_PAIR) {
                        if (out.best_gamma) gam = parabolic_gamma<N1, N2>(w[j], k1, bk, mx, gmask);
                    }
                    if (k1 == 0) {
                        if constexpr (MODE == MODE_PAIR) {
                            out.best_val[m * out.T + t] = bv;
                            out.best_k[m * out.T + t] = bk;
                            if (out.best_gamma) out.best_gamma[m * out.T + t] = gam;
                        } else {
                            const uint32_t idx = (uint32_t)((out.t_offset + t) * Q + bk);
                            const unsigned long long key =
                                ((unsigned long long)ord_f32(bv) << 32) | (unsigned long long)(0xFFFFFFFFu - idx);
                            atomicMax(out.best_key + m, key);
                        }
                    }
                }
            }
        }
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link dependency).
typedef CUresult (*PFN_encodeTiled_fr)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                       const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline PFN_encodeTiled_fr encode_tiled_fn() {
    static PFN_encodeTiled_fr fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled_fr>(p);
    }
    return fn;
}

// 3-D view of the planar workspace: (image ml, template tl, plane row = plane * N + n), box (TB, 1, BOXR).
template <int LOGN>
static cudaError_t make_spectrum_tmap(CUtensorMap *tm, const float *Upk, int64_t Mc, int64_t Tc) {
    using C = FftCfg<LOGN>;
    PFN_encodeTiled_fr enc = encode_tiled_fn();
    if (!enc) return cudaErrorNotSupported;
    const cuuint64_t dims[3] = {(cuuint64_t)Mc, (cuuint64_t)Tc, (cuuint64_t)C::ROWS};
    const cuuint64_t strides[2] = {(cuuint64_t)Mc * 4, (cuuint64_t)Mc * Tc * 4};
    const cuuint32_t box[3] = {(cuuint32_t)C::TB, 1u, (cuuint32_t)C::BOXR};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(Upk), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int LOGN, int MODE>
static cudaError_t launch_fft_mode(cudaStream_t s, const CUtensorMap &tm, int64_t Mc, int64_t Tc, int64_t m0,
                                   int64_t t0, int64_t mcv, int64_t tcv, const FftOut &out) {
    using C = FftCfg<LOGN>;
    const size_t smem = C::smem_bytes();
    static std::atomic<uint64_t> attr{0};
    cudaError_t e = smem_attr_once((const void *)fft_reduce_kernel<LOGN, MODE>, (int)smem, attr);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fft_reduce_kernel<LOGN, MODE>, FR_THREADS, smem);
    if (e != cudaSuccess || occ < 1) occ = 1;
    const int64_t nitems = tcv * ((mcv + C::TB - 1) / C::TB);
    const int64_t grid = std::min<int64_t>(nitems, (int64_t)num_sms() * occ);
    fft_reduce_kernel<LOGN, MODE><<<(unsigned)grid, FR_THREADS, smem, s>>>(tm, Mc, Tc, m0, t0, mcv, tcv, out);
    return cudaGetLastError();
}

template <int LOGN>
static cudaError_t launch_fft(int mode, cudaStream_t s, const CUtensorMap &tm, int64_t Mc, int64_t Tc, int64_t m0,
                              int64_t t0, int64_t mcv, int64_t tcv, const FftOut &out) {
    if (mode == MODE_PAIR) return launch_fft_mode<LOGN, MODE_PAIR>(s, tm, Mc, Tc, m0, t0, mcv, tcv, out);
    if (mode == MODE_IMAGE) return launch_fft_mode<LOGN, MODE_IMAGE>(s, tm, Mc, Tc, m0, t0, mcv, tcv, out);
    return launch_fft_mode<LOGN, MODE_LANDSCAPE>(s, tm, Mc, Tc, m0, t0, mcv, tcv, out);
}

}  // namespace rsvd
