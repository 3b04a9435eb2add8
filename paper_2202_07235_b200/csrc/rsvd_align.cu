// rsvd_align.cu -- rows a2-a4: per-pair contraction over the principal rings (Step 2),
// length-Q landscape transform (Step 3, :673) and argmax / landscape emission (Step 4, :504-517).
//
// Data flow per chunk of (Mc x Tc) pairs, all on `stream`:
//   contract_kernel   U_q[m,t] = sum_j alpha[q][j][m] beta[q][j][t] = S_q + conj(S_{Q-q}), q = 0..N
//                     (N = Q/2; S_q = sum_h conj(A_q[m,h]) B_q[t,h]) -> workspace Upk[n][t][m] (q-major,
//                     coalesced stores; Upk[0] packs the two real values (U_0, U_N)).  FP32 SIMT,
//                     register tiled, cp.async double-buffered operand tiles.
//   contract_tc_kernel (rsvd_tc.cu) the same U_q on tcgen05 CTA pairs (fp16 hi/lo split, TMA-fed).
//   fft_reduce_kernel (rsvd_fft.cuh) Re X_k = 2 pi Re sum_q e^{-2 pi i qk/Q} S_q, fused with the
//                     per-pair argmax (smallest k on ties), the per-image packed-key max, or the
//                     landscape store.  The M x T x Q landscape never leaves the chip unless asked.
// The workspace chunk is sized to stay L2-resident between the two kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>

#include "rsvd_common.cuh"
#include "rsvd_fft.cuh"
#include "rsvd_fft2.cuh"
#include "rsvd_fftc.cuh"

namespace rsvd {

// ------------------------------------------------------------------ contraction (Step 2)
// Spectrum workspace layout (q-major): Upk[(n * Mc + ml) * Tc + tl], n in [0, N), ml < Mc, tl < Tc.
constexpr int CT_TILE = 64;    // m and t tile
constexpr int CT_KC = 16;      // complex K per pipeline stage
constexpr int CT_QB = 4;       // q values per CTA
constexpr int CT_THREADS = 256;

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int NWAIT>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NWAIT)); }

// grid: (Tc/64, Mc/64, ceil((N+1)/QB)).  Thread (ty, tx) owns m = ty*4 + i, t = tx + 16 j.
__global__ void __launch_bounds__(CT_THREADS, 3) contract_kernel(const float2 *__restrict__ alpha,
                                                                 const float2 *__restrict__ beta,
                                                                 int64_t Mpad, int64_t Tpad, int Kpad, int N,
                                                                 int64_t m0, int64_t t0, int64_t Mc, int64_t Tc,
                                                                 float *__restrict__ Upk, int Nout) {
    __shared__ __align__(16) float2 As[2][CT_KC][CT_TILE];
    __shared__ __align__(16) float2 Bs[2][CT_KC][CT_TILE];

    const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
    const int64_t bt = (int64_t)blockIdx.x * CT_TILE, bm = (int64_t)blockIdx.y * CT_TILE;
    const int q0 = blockIdx.z * CT_QB;
    const int nq = min(CT_QB, N + 1 - q0);
    const int nk = Kpad / CT_KC;
    const int iters = nq * nk;

    auto load_stage = [&](int it, int buf) {
        const int q = q0 + it / nk, kc = it % nk;
        const float2 *ga = alpha + ((int64_t)q * Kpad + kc * CT_KC) * Mpad + m0 + bm;
        const float2 *gb = beta + ((int64_t)q * Kpad + kc * CT_KC) * Tpad + t0 + bt;
#pragma unroll
        for (int c = tid; c < CT_KC * 32; c += CT_THREADS) {
            const int kk = c >> 5, ch = c & 31;
            cp_async16(&As[buf][kk][ch * 2], ga + (int64_t)kk * Mpad + ch * 2);
            cp_async16(&Bs[buf][kk][ch * 2], gb + (int64_t)kk * Tpad + ch * 2);
        }
        cp_async_commit();
    };

    float2 acc[4][4];
    load_stage(0, 0);
    for (int it = 0; it < iters; ++it) {
        const int buf = it & 1;
        if (it + 1 < iters) {
            load_stage(it + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const int kc = it % nk;
        if (kc == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int kk = 0; kk < CT_KC; ++kk) {
            // thread (ty, tx) owns images m = tx + 16 i and templates t = ty * 4 + j
            const float4 b01 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][ty * 4]);
            const float4 b23 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][ty * 4 + 2]);
            const float2 b[4] = {make_float2(b01.x, b01.y), make_float2(b01.z, b01.w),
                                 make_float2(b23.x, b23.y), make_float2(b23.z, b23.w)};
            float2 a[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[buf][kk][tx + 16 * i];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    acc[i][j].x = fmaf(a[i].x, b[j].x, acc[i][j].x);
                    acc[i][j].x = fmaf(-a[i].y, b[j].y, acc[i][j].x);
                    acc[i][j].y = fmaf(a[i].x, b[j].y, acc[i][j].y);
                    acc[i][j].y = fmaf(a[i].y, b[j].x, acc[i][j].y);
                }
        }
        if (kc == nk - 1) {          // q finished: planar [n][t][m] stores, 16 lanes = 64 contiguous bytes
            const int q = q0 + it / nk;
            const int n = (q == N) ? 0 : q;
            float *const re = Upk, *const im = Upk + (int64_t)Nout * Mc * Tc;   // planes of Nout rows
            const int64_t o = ((int64_t)n * Tc + bt) * Mc + bm;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int64_t p = o + (int64_t)(ty * 4 + j) * Mc + tx + 16 * i;
                    if (q == 0) re[p] = acc[i][j].x;                 // U_0 (real) -> re plane slot 0
                    else if (q == N && Nout > N) re[p + (int64_t)N * Tc * Mc] = 0.5f * acc[i][j].x;   // padded: split Nyquist
                    else if (q == N) im[p] = acc[i][j].x;            // U_N (real) -> im plane slot 0
                    else { re[p] = acc[i][j].x; im[p] = acc[i][j].y; }
                }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ driver
struct AlignArgs {
    const float2 *alpha, *beta;
    int64_t M, T, t_offset;
    int Q, H;
    int mode;
    void *work;
    int64_t work_bytes;
    float *best_val;
    int32_t *best_k;
    unsigned long long *best_key;
    float *X;
    int64_t ld_m, ld_t;
    int Qout;              // output grid (Q, or Q * 2^p zero-padded: rsvd_align_*_fine)
    float *best_gamma;     // PER_PAIR, optional: parabolic-refined angle
};

// Steps 3-4 kernel: fft2 (rsvd_fft2.cuh) for N = Q/2 <= 256; the original schedule (rsvd_fft.cuh)
// for N = 512 or when RSVD_FFT=1 / RSVD_FFT_V1=1 (kept for comparison).
static int fft_version(int LOGN) {
    static const int v = [] {
        const char *e = getenv("RSVD_FFT");
        const char *e1 = getenv("RSVD_FFT_V1");
        if (e1 && atoi(e1)) return 1;
        return e ? atoi(e) : 2;
    }();
    if (LOGN > 8) return 1;
    return v == 1 ? 1 : 2;
}

static cudaError_t make_tmap_any(int LOGN, CUtensorMap *tm, const float *Upk, int64_t Mc, int64_t Tc) {
    if (fft_version(LOGN) >= 2) {
        switch (LOGN) {
            case 4: return make_spectrum_tmap2<4>(tm, Upk, Mc, Tc);
            case 5: return make_spectrum_tmap2<5>(tm, Upk, Mc, Tc);
            case 6: return make_spectrum_tmap2<6>(tm, Upk, Mc, Tc);
            case 7: return make_spectrum_tmap2<7>(tm, Upk, Mc, Tc);
            default: return make_spectrum_tmap2<8>(tm, Upk, Mc, Tc);
        }
    }
    switch (LOGN) {
        case 4: return make_spectrum_tmap<4>(tm, Upk, Mc, Tc);
        case 5: return make_spectrum_tmap<5>(tm, Upk, Mc, Tc);
        case 6: return make_spectrum_tmap<6>(tm, Upk, Mc, Tc);
        case 7: return make_spectrum_tmap<7>(tm, Upk, Mc, Tc);
        case 8: return make_spectrum_tmap<8>(tm, Upk, Mc, Tc);
        default: return make_spectrum_tmap<9>(tm, Upk, Mc, Tc);
    }
}

static cudaError_t make_spectrum_tmap2_any(int LOGN, CUtensorMap *tm, const float *Upk, int64_t Mc, int64_t Tc, int eb) {
    switch (LOGN) {
        case 4: return make_spectrum_tmap2<4>(tm, Upk, Mc, Tc, eb);
        case 5: return make_spectrum_tmap2<5>(tm, Upk, Mc, Tc, eb);
        case 6: return make_spectrum_tmap2<6>(tm, Upk, Mc, Tc, eb);
        case 7: return make_spectrum_tmap2<7>(tm, Upk, Mc, Tc, eb);
        default: return make_spectrum_tmap2<8>(tm, Upk, Mc, Tc, eb);
    }
}

static cudaError_t launch_fft_any(int LOGN, int mode, cudaStream_t s, const CUtensorMap &tm, int64_t Mc, int64_t Tc,
                                  int64_t m0, int64_t t0, int64_t mcv, int64_t tcv, const FftOut &o, float *Upk,
                                  bool half = false) {
    static const bool discard = [] { const char *e = getenv("RSVD_NO_DISCARD"); return !(e && atoi(e)); }();
    float *dU = discard ? Upk : nullptr;
    const int v = fft_version(LOGN);
    if (v == 2) {
        switch (LOGN) {
            case 4: return launch_fft2<4>(mode, s, tm, m0, t0, mcv, tcv, o, dU, Mc, Tc, half);
            case 5: return launch_fft2<5>(mode, s, tm, m0, t0, mcv, tcv, o, dU, Mc, Tc, half);
            case 6: return launch_fft2<6>(mode, s, tm, m0, t0, mcv, tcv, o, dU, Mc, Tc, half);
            case 7: return launch_fft2<7>(mode, s, tm, m0, t0, mcv, tcv, o, dU, Mc, Tc, half);
            default: return launch_fft2<8>(mode, s, tm, m0, t0, mcv, tcv, o, dU, Mc, Tc, half);
        }
    }
    switch (LOGN) {
        case 4: return launch_fft<4>(mode, s, tm, Mc, Tc, m0, t0, mcv, tcv, o);
        case 5: return launch_fft<5>(mode, s, tm, Mc, Tc, m0, t0, mcv, tcv, o);
        case 6: return launch_fft<6>(mode, s, tm, Mc, Tc, m0, t0, mcv, tcv, o);
        case 7: return launch_fft<7>(mode, s, tm, Mc, Tc, m0, t0, mcv, tcv, o);
        case 8: return launch_fft<8>(mode, s, tm, Mc, Tc, m0, t0, mcv, tcv, o);
        default: return launch_fft<9>(mode, s, tm, Mc, Tc, m0, t0, mcv, tcv, o);
    }
}

cudaError_t launch_align_fused(const void *alpha, int64_t M, const void *beta, int64_t T, int Q, int H, int mode,
                               void *work, int64_t work_bytes, const FftOut &out, cudaStream_t s, bool *launched);

static rsvd_status run_align(const AlignArgs &a, cudaStream_t s) {
    const int N = a.Q / 2;
    const int Nout = a.Qout / 2;             // spectrum rows per plane (zero-padded when Qout > Q)
    const int Kpad = (int)kpad_of(a.H);
    const bool tc = resolve_path(a.Q, a.H) == PATH_TC;
    // fast path (<= 2e-3 gate): single fp16 MMA per product and an fp16 spectrum (half the workspace
    // bytes per pair); TC layout, fft2 transform, plain Q_out == Q grid only
    const bool fast = tc && resolve_precision() == PREC_FAST && a.Qout == a.Q && fft_version(ilog2(a.Q / 2)) == 2;
    const int eb = fast ? 2 : 4;
    // Steps 3-4 with pass 1 on the tensor cores (rsvd_fftc.cuh): TC layout, Q in {256, 512}, argmax
    // modes, plain grid; the contraction then writes the split hi/lo fp16 spectrum (fmt 2, same bytes)
    const char *fftc_e = getenv("RSVD_FFTC");
    const int fftc_env = fftc_e ? atoi(fftc_e) : 0;
    const int lognq = ilog2(a.Q / 2);
    const bool fftc = tc && !fast && fftc_env && a.Qout == a.Q && (lognq == 7 || lognq == 8) && a.mode != MODE_LANDSCAPE;
    // pair tiles: SIMT 64 x 64; TC 128 images x 256 templates (one tcgen05 CTA-pair tile)
    const int64_t TM = tc ? 128 : 64, TT = tc ? 256 : CT_TILE;
    const int64_t Mpad = tc ? tc_rows_pad_side(a.M, RSVD_SIDE_IMAGE) : rows_pad_of(a.M);
    const int64_t Tpad = tc ? tc_rows_pad_side(a.T, RSVD_SIDE_TEMPLATE) : rows_pad_of(a.T);
    // chunk: Mc x Tc pairs (multiples of the tile) with Mc * Tc * N * 8 <= work_bytes.  Chunks are
    // visited t-outer / m-inner, so a chunk's template blocks stay in L2 while image blocks stream.
    const int64_t tile_bytes = TM * TT * Nout * 2 * (int64_t)eb;
    const int64_t ntiles = a.work_bytes / tile_bytes;
    if (ntiles < 1) return fail(RSVD_ERR_ARG, "workspace smaller than rsvd_align_min_workspace_bytes(Q)");
    const int64_t tmax = Tpad / TT, mmax = Mpad / TM;
    // TC: template tiles per chunk (RSVD_TCT, experiment override; default 1 -- the chunk's image tiles
    // share one template tile whose operands stay in L2 while image operands stream)
    const char *tct_e = getenv("RSVD_TCT");
    const int64_t tct_tc = tct_e ? std::max(1, atoi(tct_e)) : 1;
    int64_t tct = std::min<int64_t>(tmax, tc ? std::min(tct_tc, ntiles) : std::max<int64_t>(1, (int64_t)std::sqrt((double)ntiles)));
    int64_t mct = std::min(mmax, std::max<int64_t>(1, ntiles / tct));
    tct = std::min(tmax, std::max(tct, ntiles / mct));      // widen t when rows run out
    const int64_t Mc = mct * TM, Tc = tct * TT;
    CUtensorMap tmA, tmB;
    cudaError_t e;
    if (tc) {
        if ((e = make_tc_operand_tmap(&tmA, a.alpha, a.M, a.Q, a.H, RSVD_SIDE_IMAGE)) != cudaSuccess)
            return cuda_check(e, "image operand tensor map");
        if ((e = make_tc_operand_tmap(&tmB, a.beta, a.T, a.Q, a.H, RSVD_SIDE_TEMPLATE)) != cudaSuccess)
            return cuda_check(e, "template operand tensor map");
    }
    float *Upk = reinterpret_cast<float *>(a.work);
    const FftOut o{a.best_val, a.best_k, a.best_key, a.X, a.ld_m, a.ld_t, a.T, a.t_offset,
                   tc ? tc_scales(a.alpha, a.M, a.Q, a.H, RSVD_SIDE_IMAGE) : nullptr,
                   tc ? tc_scales(a.beta, a.T, a.Q, a.H, RSVD_SIDE_TEMPLATE) : nullptr, a.best_gamma};
    if (tc && Nout == N && !fast && !fftc) {
        // one persistent launch: contraction and transform roles over an L2-sized spectrum ring
        // (rsvd_fused.cu); falls through to the two-kernel chunk loop where it does not apply
        cudaEvent_t ev0 = timing_enabled() ? timing_event(s) : nullptr;
        bool launched = false;
        cudaError_t ef = launch_align_fused(a.alpha, a.M, a.beta, a.T, a.Q, a.H, a.mode, a.work, a.work_bytes, o, s,
                                            &launched);
        if (ef != cudaSuccess) return cuda_check(ef, "fused align launch");
        if (launched) {
            count_launches(1);
            if (ev0) timing_span(ev0, timing_event(s), TK_FUSED);
            return RSVD_OK;
        }
    }
    if (Nout > N) {
        // rows the contraction never writes (im row 0, rows N..Nout-1 except re row N) must read as 0;
        // they are written here once per call and never discarded from L2 (no discard when padded)
        e = cudaMemsetAsync(Upk, 0, (size_t)2 * Nout * Mc * Tc * sizeof(float), s);
        if (e != cudaSuccess) return cuda_check(e, "padded workspace reset");
    }
    const int LOGN = ilog2(Nout);
    CUtensorMap tmap;
    if ((e = fftc ? make_fftc_tmap_any(LOGN, &tmap, Upk, Mc, Tc)
              : (fast ? make_spectrum_tmap2_any(LOGN, &tmap, Upk, Mc, Tc, 2) : make_tmap_any(LOGN, &tmap, Upk, Mc, Tc))) !=
        cudaSuccess)
        return cuda_check(e, "spectrum tensor map");
    const bool timed = timing_enabled();
    bool first = true;
    for (int64_t t0 = 0; t0 < Tpad; t0 += Tc) {
        const int64_t tc_ = std::min(Tc, Tpad - t0);
        const int64_t tcv = std::min(tc_, a.T - t0);
        for (int64_t m0 = 0; m0 < Mpad; m0 += Mc) {
            const int64_t mc = std::min(Mc, Mpad - m0);
            const int64_t mcv = std::min(mc, a.M - m0);
            cudaEvent_t ev0 = timed ? timing_event(s) : nullptr;
            if (tc) {
                e = launch_contract_tc(tmA, tmB, a.H, N, Nout, m0, t0, mc, tc_, Mc, Tc, Upk, num_sms(), first,
                                       fast ? 1 : (fftc ? 2 : 0), s);
                first = false;
                if (e != cudaSuccess) return cuda_check(e, "contract (tcgen05) launch");
            } else {
                dim3 g1((unsigned)(tc_ / CT_TILE), (unsigned)(mc / CT_TILE), (unsigned)((N + 1 + CT_QB - 1) / CT_QB));
                contract_kernel<<<g1, CT_THREADS, 0, s>>>(a.alpha, a.beta, Mpad, Tpad, Kpad, N, m0, t0, Mc, Tc, Upk, Nout);
                if ((e = cudaGetLastError()) != cudaSuccess) return cuda_check(e, "contract launch");
            }
            cudaEvent_t ev1 = timed ? timing_event(s) : nullptr;
            e = fftc ? launch_fftc(LOGN, a.mode, s, tmap, m0, t0, mcv, tcv, o, Mc)
                     : launch_fft_any(LOGN, a.mode, s, tmap, Mc, Tc, m0, t0, mcv, tcv, o, Nout > N ? nullptr : Upk, fast);
            if (e != cudaSuccess) return cuda_check(e, "fft_reduce launch");
            count_launches(2);
            if (timed) {
                cudaEvent_t ev2 = timing_event(s);
                timing_span(ev0, ev1, TK_CONTRACT);
                timing_span(ev1, ev2, TK_FFT);
            }
        }
    }
    return RSVD_OK;
}

static rsvd_status check_common(const void *img, int64_t M, const void *tmpl, int64_t T, int32_t Q, int32_t H,
                                void *work, int64_t work_bytes) {
    if (Q <= 0) return fail(RSVD_ERR_ARG, "Q must be positive");
    if (!is_pow2(Q) || Q < 32 || Q > 1024) return fail(RSVD_ERR_UNSUPPORTED, "Q must be a power of two in [32, 1024]");
    if (H < 1) return fail(RSVD_ERR_ARG, "H must be >= 1");
    if (H > 256) return fail(RSVD_ERR_UNSUPPORTED, "H > 256 is not supported");
    if (M < 0 || T < 0) return fail(RSVD_ERR_ARG, "M and T must be >= 0");
    if (M > 0x7fffffffLL || T > 0x7fffffffLL) return fail(RSVD_ERR_UNSUPPORTED, "M, T must be < 2^31");
    if (M == 0 || T == 0) return RSVD_OK;
    if (!img || !tmpl || !work) return fail(RSVD_ERR_ARG, "NULL pointer");
    if (!aligned16(img) || !aligned16(tmpl) || !aligned16(work)) return fail(RSVD_ERR_ARG, "buffers must be 16-byte aligned");
    if (work_bytes < rsvd_align_min_workspace_bytes(Q)) return fail(RSVD_ERR_ARG, "workspace too small");
    return RSVD_OK;
}

// ------------------------------------------------------------------ winners
__device__ __forceinline__ float unord_f32(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}

__global__ void winners_unpack_kernel(const unsigned long long *__restrict__ keys, int G, int64_t M, int Q,
                                      unsigned long long *__restrict__ out_keys, float *__restrict__ val,
                                      int32_t *__restrict__ t, int32_t *__restrict__ k) {
    const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= M) return;
    unsigned long long best = 0ull;
    for (int gi = 0; gi < G; ++gi) {
        const unsigned long long v = keys[(int64_t)gi * M + m];
        best = v > best ? v : best;
    }
    if (out_keys) out_keys[m] = best;
    const uint32_t idx = 0xFFFFFFFFu - (uint32_t)(best & 0xFFFFFFFFull);
    if (val) val[m] = best ? unord_f32((uint32_t)(best >> 32)) : -INFINITY;
    if (t) t[m] = best ? (int32_t)(idx / (uint32_t)Q) : -1;
    if (k) k[m] = best ? (int32_t)(idx % (uint32_t)Q) : -1;
}

}  // namespace rsvd

using namespace rsvd;

extern "C" int64_t rsvd_align_min_workspace_bytes(int32_t Q) {
    if (Q < 2) return -1;
    return (int64_t)128 * 256 * (Q / 2) * (int64_t)sizeof(float2);     // one 128 x 256 pair tile (either path)
}

extern "C" int64_t rsvd_align_workspace_bytes(int64_t M, int64_t T, int32_t Q, int32_t H) {
    (void)H;
    if (Q < 2 || M < 0 || T < 0) return -1;
    const int64_t full = tc_rows_pad(std::max<int64_t>(M, 1)) * tc_rows_pad(std::max<int64_t>(T, 1)) * (Q / 2) * 8;
    const int64_t target = 128ll << 20;    // chunk of the spectrum workspace (measured best on B200)
    return std::max(rsvd_align_min_workspace_bytes(Q), std::min(full, target));
}

static rsvd_status check_qout(int32_t Q, int32_t Qout, int64_t work_bytes) {
    if (Qout < Q || !is_pow2(Qout) || Qout > 1024)
        return fail(RSVD_ERR_UNSUPPORTED, "Q_out must be Q times a power of two, at most 1024");
    if (work_bytes < rsvd_align_min_workspace_bytes(Qout)) return fail(RSVD_ERR_ARG, "workspace too small for Q_out");
    return RSVD_OK;
}

extern "C" rsvd_status rsvd_align_argmax_fine(const void *img_blocks, int64_t M, const void *tmpl_blocks, int64_t T,
                                              int64_t t_offset, int32_t Q, int32_t H, int32_t Q_out,
                                              rsvd_reduce mode, void *work, int64_t work_bytes, float *best_val,
                                              int32_t *best_k, uint64_t *best_key, float *best_gamma,
                                              rsvd_stream_t stream) {
    rsvd_status st = check_common(img_blocks, M, tmpl_blocks, T, Q, H, work, work_bytes);
    if (st != RSVD_OK || M == 0 || T == 0) return st;
    if ((st = check_qout(Q, Q_out, work_bytes)) != RSVD_OK) return st;
    if (mode == RSVD_PER_PAIR) {
        if (!best_val || !best_k) return fail(RSVD_ERR_ARG, "PER_PAIR needs best_val and best_k");
    } else if (mode == RSVD_PER_IMAGE) {
        if (!best_key) return fail(RSVD_ERR_ARG, "PER_IMAGE needs best_key");
        if (best_gamma) return fail(RSVD_ERR_ARG, "best_gamma is a PER_PAIR output");
        if (t_offset < 0) return fail(RSVD_ERR_ARG, "t_offset must be >= 0");
        if ((uint64_t)(t_offset + T) * (uint64_t)Q_out >= 0xFFFFFFFFull)
            return fail(RSVD_ERR_UNSUPPORTED, "(t_offset + T) * Q_out must be < 2^32 for packed keys");
    } else {
        return fail(RSVD_ERR_ARG, "bad mode");
    }
    AlignArgs a{reinterpret_cast<const float2 *>(img_blocks), reinterpret_cast<const float2 *>(tmpl_blocks),
                M, T, t_offset, Q, H, mode == RSVD_PER_PAIR ? MODE_PAIR : MODE_IMAGE, work, work_bytes,
                best_val, best_k, reinterpret_cast<unsigned long long *>(best_key), nullptr, 0, 0, Q_out, best_gamma};
    return run_align(a, (cudaStream_t)stream);
}

extern "C" rsvd_status rsvd_align_argmax(const void *img_blocks, int64_t M, const void *tmpl_blocks, int64_t T,
                                         int64_t t_offset, int32_t Q, int32_t H, rsvd_reduce mode, void *work,
                                         int64_t work_bytes, float *best_val, int32_t *best_k, uint64_t *best_key,
                                         rsvd_stream_t stream) {
    return rsvd_align_argmax_fine(img_blocks, M, tmpl_blocks, T, t_offset, Q, H, Q, mode, work, work_bytes, best_val,
                                  best_k, best_key, nullptr, stream);
}

// Row f3: G independent (image-group, CTF-corrected template) problems in one call.  All groups are
// validated first (no partial enqueue on a bad descriptor), then run back to back on the stream.
extern "C" rsvd_status rsvd_align_argmax_grouped(const rsvd_align_group *groups, int32_t G, int32_t Q, int32_t H,
                                                 rsvd_reduce mode, void *work, int64_t work_bytes,
                                                 rsvd_stream_t stream) {
    if (G < 0) return fail(RSVD_ERR_ARG, "G must be >= 0");
    if (G == 0) return RSVD_OK;
    if (!groups) return fail(RSVD_ERR_ARG, "NULL group array");
    if (mode != RSVD_PER_PAIR && mode != RSVD_PER_IMAGE) return fail(RSVD_ERR_ARG, "bad mode");
    for (int g = 0; g < G; ++g) {
        const rsvd_align_group &d = groups[g];
        rsvd_status st = check_common(d.img_blocks, d.M, d.tmpl_blocks, d.T, Q, H, work, work_bytes);
        if (st != RSVD_OK) return fail(st, "group " + std::to_string(g) + ": " + rsvd_last_error());
        if (d.M == 0 || d.T == 0) continue;
        if (mode == RSVD_PER_PAIR && (!d.best_val || !d.best_k))
            return fail(RSVD_ERR_ARG, "group " + std::to_string(g) + ": PER_PAIR needs best_val and best_k");
        if (mode == RSVD_PER_IMAGE) {
            if (!d.best_key) return fail(RSVD_ERR_ARG, "group " + std::to_string(g) + ": PER_IMAGE needs best_key");
            if (d.t_offset < 0 || (uint64_t)(d.t_offset + d.T) * (uint64_t)Q >= 0xFFFFFFFFull)
                return fail(RSVD_ERR_UNSUPPORTED, "group " + std::to_string(g) + ": (t_offset + T) * Q must be < 2^32");
        }
    }
    for (int g = 0; g < G; ++g) {
        const rsvd_align_group &d = groups[g];
        if (d.M == 0 || d.T == 0) continue;
        AlignArgs a{reinterpret_cast<const float2 *>(d.img_blocks), reinterpret_cast<const float2 *>(d.tmpl_blocks),
                    d.M, d.T, d.t_offset, Q, H, mode == RSVD_PER_PAIR ? MODE_PAIR : MODE_IMAGE, work, work_bytes,
                    d.best_val, d.best_k, reinterpret_cast<unsigned long long *>(d.best_key), nullptr, 0, 0, Q, nullptr};
        const rsvd_status st = run_align(a, (cudaStream_t)stream);
        if (st != RSVD_OK) return st;
    }
    return RSVD_OK;
}

extern "C" rsvd_status rsvd_align_landscape_fine(const void *img_blocks, int64_t M, const void *tmpl_blocks,
                                                 int64_t T, int32_t Q, int32_t H, int32_t Q_out, void *work,
                                                 int64_t work_bytes, float *X, int64_t ld_m, int64_t ld_t,
                                                 rsvd_stream_t stream) {
    rsvd_status st = check_common(img_blocks, M, tmpl_blocks, T, Q, H, work, work_bytes);
    if (st != RSVD_OK || M == 0 || T == 0) return st;
    if ((st = check_qout(Q, Q_out, work_bytes)) != RSVD_OK) return st;
    if (!X) return fail(RSVD_ERR_ARG, "NULL landscape pointer");
    if (ld_t < Q_out || ld_m < 0) return fail(RSVD_ERR_ARG, "bad landscape strides");
    if ((ld_t & 1) || (ld_m & 1) || (reinterpret_cast<uintptr_t>(X) & 7u))
        return fail(RSVD_ERR_ARG, "landscape strides must be even and X 8-byte aligned");
    AlignArgs a{reinterpret_cast<const float2 *>(img_blocks), reinterpret_cast<const float2 *>(tmpl_blocks),
                M, T, 0, Q, H, MODE_LANDSCAPE, work, work_bytes, nullptr, nullptr, nullptr, X, ld_m, ld_t, Q_out,
                nullptr};
    return run_align(a, (cudaStream_t)stream);
}

extern "C" rsvd_status rsvd_align_landscape(const void *img_blocks, int64_t M, const void *tmpl_blocks, int64_t T,
                                            int32_t Q, int32_t H, void *work, int64_t work_bytes, float *X,
                                            int64_t ld_m, int64_t ld_t, rsvd_stream_t stream) {
    return rsvd_align_landscape_fine(img_blocks, M, tmpl_blocks, T, Q, H, Q, work, work_bytes, X, ld_m, ld_t, stream);
}

extern "C" rsvd_status rsvd_winners_reset(uint64_t *keys, int64_t M, rsvd_stream_t stream) {
    if (M < 0) return fail(RSVD_ERR_ARG, "M must be >= 0");
    if (M == 0) return RSVD_OK;
    if (!keys) return fail(RSVD_ERR_ARG, "NULL pointer");
    return cuda_check(cudaMemsetAsync(keys, 0, (size_t)M * sizeof(uint64_t), (cudaStream_t)stream), "winners reset");
}

extern "C" rsvd_status rsvd_winners_unpack(const uint64_t *keys, int64_t M, int32_t Q, float *val, int32_t *t,
                                           int32_t *k, rsvd_stream_t stream) {
    return rsvd_combine_winners(keys, 1, M, Q, nullptr, val, t, k, stream);
}

extern "C" rsvd_status rsvd_combine_winners(const uint64_t *keys, int32_t G, int64_t M, int32_t Q, uint64_t *out_keys,
                                            float *val, int32_t *t, int32_t *k, rsvd_stream_t stream) {
    if (G < 1 || M < 0 || Q < 1) return fail(RSVD_ERR_ARG, "bad sizes");
    if (M == 0) return RSVD_OK;
    if (!keys) return fail(RSVD_ERR_ARG, "NULL pointer");
    winners_unpack_kernel<<<(unsigned)((M + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const unsigned long long *>(keys), G, M, Q, reinterpret_cast<unsigned long long *>(out_keys),
        val, t, k);
    count_launches(1);
    return cuda_check(cudaGetLastError(), "combine launch");
}
