// rsvd_fft2.cuh -- Steps 3-4 of the align path (PAPER.md:673 transform, forward sign per DESIGN.md
// G3; PAPER.md:504-517 argmax), restructured for N = Q/2 <= 256: same mathematics as rsvd_fft.cuh
// (one complex length-N FFT of Z_n = (Y_n + conj Y_{N-n}) + i W_Q^n (Y_n - conj Y_{N-n}) per pair,
// z_k = x_{2k} + i x_{2k+1}, Re X_k = 2 pi x_k; Z is formed from U = 2Y, so results are scaled by pi).
//
// Four-step N = N1 x N2 (N1 = 2^floor(log2 N / 2) columns, N2 >= N1 rows), lane = image:
//   work item  one template x 32 images; a CTA holds G independent warp groups of N1/2 warps that
//              take its items in turn from a ring of G + 1 shared-memory slots (each the TMA target of
//              one item and, in place, its transpose buffer; one mbarrier each); groups synchronise
//              with named barriers only, and a slot is refilled G + 1 items ahead once read;
//   TMA        the group's 2N spectrum rows x 32 images land in its slot (3-D tensor-map boxes);
//   pass 1     warp c of a group owns the mirror column pair {c, N1 - c} (warp 0: the self-mirror
//              columns 0 and N1/2), so Z_n and Z_{N-n} are formed in registers from the two values
//              they share (no staging pass), then two in-register DIF DFTs of length N2 over n2,
//              twiddles W_N^{n1 k1}, and stores over the slot as ZY[image][k1][n1] with padded strides
//              (N1 + 1 per k1 block, odd per image: conflict-free for both passes, no index swizzle);
//   pass 2     one thread per (image, k1): in-register DIF DFT of length N1 over n1 -> z[k1 + N2 k2];
//              landscape store, or max then first argmax over the N2 lanes of the pair; the next
//              item's TMA is issued as soon as the slot has been read.
#pragma once

#include <cuda_fp16.h>

#include "rsvd_fft.cuh"

namespace rsvd {

#ifdef RSVD_TRACE
#ifdef RSVD_TRACE_TU_FUSED
RSVD_TRACE_DEFINE(fused)
#else
RSVD_TRACE_DEFINE(fft)
#endif
#endif

#ifndef RSVD_FFT2_L2PROMO
#define RSVD_FFT2_L2PROMO 3     // spectrum TMA L2 promotion: 0 none, 1 64B, 2 128B, 3 256B (CUtensorMapL2promotion)
#endif
#ifndef RSVD_FFT2_ONECOL
#define RSVD_FFT2_ONECOL 0      // 1: pass 1 with one column per warp (1024 threads, <= 64 registers); measured slower
#endif

// EB: bytes per spectrum element (4 = fp32, 2 = fp16 fast path).  ONE: pass 1 with one column per warp
// (N1 warps per group, 1024 threads per CTA) instead of one mirror column pair per warp (N1/2 warps,
// 512 threads): half the registers per thread, so twice the warps hide the FP and shared-memory latency,
// at the cost of forming each Z value pair twice (once per mirror column).
template <int LOGN, int EB = 4, bool ONE = false>
struct Fft2Cfg {
    static constexpr int N = 1 << LOGN;
    static constexpr int Q = 2 * N;
    static constexpr int N1 = 1 << (LOGN / 2);        // columns (pass-2 length)
    static constexpr int N2 = N / N1;                 // rows (pass-1 length), N2 in {N1, 2 N1}
    static constexpr int TASKS = ONE ? N1 : N1 / 2;   // warps per group
    static constexpr int GT = 32 * TASKS;             // threads per group
    static constexpr int G = (ONE ? 32 : 16) / TASKS; // groups per CTA (1024 / 512 threads)
    static constexpr int THREADS = G * GT;
    static constexpr int TB = 32;                     // images per item (lane = image)
    static constexpr int ROWS = 2 * N;                // re plane rows, then im plane rows
    static constexpr int BOXR = ROWS < 256 ? ROWS : 256;
    static constexpr int NBOX = ROWS / BOXR;
    static constexpr int UBYTES = ROWS * TB * EB;
    static constexpr int SK = N1 + 1;                 // ZY stride of one k1 block (float2)
    static constexpr int SZ = N2 * SK + 1;            // ZY stride of one image (odd)
    static constexpr int ZBYTES = TB * SZ * 8;
    static constexpr int SLOT = ((UBYTES > ZBYTES ? UBYTES : ZBYTES) + 1023) / 1024 * 1024;
    static constexpr int P2_PER = TB * N2 / GT;       // pass-2 tasks per thread
    static constexpr int NSLOT = G + 1;               // one slot in flight beyond the G being processed
    static constexpr size_t smem_bytes() { return 1024 + (size_t)NSLOT * SLOT + (size_t)N * 8 + (size_t)(N / 2) * 8 + NSLOT * 20 + 64; }
};

// Z_r and Z_{N-r} from a = U_r, b = U_{N-r} (0 < r < N/2), w = W_Q^r.
__device__ __forceinline__ void z_pair(float2 a, float2 b, float2 w, float2 &zr, float2 &zm) {
    const float2 sv = c_add(a, make_float2(b.x, -b.y));     // s = U_r + conj U_{N-r}
    const float2 dv = c_add(a, make_float2(-b.x, b.y));     // d = U_r - conj U_{N-r}
    const float2 p = c_mul(dv, w);
    zr = c_add(sv, make_float2(-p.y, p.x));                // s + i p
    zm = c_add(make_float2(sv.x, -sv.y), make_float2(p.y, p.x));   // conj(s) + i conj(p)
}

// One work item (one template x 32 images) of a warp group: pass 1 straight from the item's landed
// slot U, pass 2 and the fused output.  `release()` is called by every thread once the slot has been
// read for the last time (its warps may then let the slot be refilled).  Images m_first + p,
// p < n_valid, are real; t is the template index within the call (out.T columns, out.t_offset).
// Spectrum element types: float (the fp32-grade path) or __half (the <= 2e-3 fast path: the contraction
// stored its fp32 accumulators times FAST_SPEC_SCALE as fp16, so the result is scaled back by 1/that).
constexpr float FAST_SPEC_SCALE = 1.0f / 1048576.0f;            // 2^-20: keeps |D| (< 2^35) inside fp16 range
template <class Tin> __device__ __forceinline__ float spec_f(Tin x);
template <> __device__ __forceinline__ float spec_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float spec_f<__half>(__half x) { return __half2float(x); }
template <class Tin> constexpr float spec_unscale() { return sizeof(Tin) == 2 ? 1048576.0f : 1.0f; }

template <int LOGN, int MODE, class Release, class Tin = float, bool ONE = false>
__device__ __forceinline__ void fft2_item(float *U, int gt, int warp, int lane, int gbar_id, const float2 *Wn,
                                          const float2 *Wq, int64_t m_first, int n_valid, int64_t t, float st,
                                          const uint32_t (&stale)[Fft2Cfg<LOGN, 4, ONE>::P2_PER],
                                          const float (&smv)[Fft2Cfg<LOGN, 4, ONE>::P2_PER], const FftOut &out,
                                          Release release) {
    using C = Fft2Cfg<LOGN, 4, ONE>;
    constexpr int N = C::N, Q = C::Q, N1 = C::N1, N2 = C::N2, TB = C::TB, SZ = C::SZ, GT = C::GT;
    float2 *ZY = reinterpret_cast<float2 *>(U);                           // [TB][SZ], in place after pass-1 reads
    auto gbar = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(gbar_id), "n"(GT) : "memory"); };
    const float PI = 3.14159265358979323846f * spec_unscale<Tin>();

    // ---- pass 1: Z from the ring, DFTs of length N2 (one column per warp, or a mirror column pair)
    const Tin *Ui = reinterpret_cast<const Tin *>(U);
    auto ld = [&](int n) { return make_float2(spec_f<Tin>(Ui[n * TB + lane]), spec_f<Tin>(Ui[(N + n) * TB + lane])); };
    if constexpr (ONE) {
        float2 za[N2];
        const int c = warp;                                // column c: rows c + N1 n2
        if (c == 0) {
            const float2 u0 = ld(0);                       // (U_0, U_N) packed
            za[0] = make_float2(u0.x + u0.y, u0.x - u0.y);
            const float2 uh = ld(N / 2);
            za[N2 / 2] = make_float2(2.f * uh.x, 2.f * uh.y);
#pragma unroll
            for (int n2 = 1; n2 < N2 / 2; ++n2) z_pair(ld(N1 * n2), ld(N1 * (N2 - n2)), Wq[N1 * n2], za[n2], za[N2 - n2]);
        } else if (c == N1 / 2) {
#pragma unroll
            for (int n2 = 0; n2 < N2 / 2; ++n2) {
                const int r = N1 / 2 + N1 * n2;
                z_pair(ld(r), ld(N - r), Wq[r], za[n2], za[N2 - 1 - n2]);
            }
        } else {
            // Z_r for r = c + N1 n2: from (U_r, U_{N-r}) with W_Q^r when r < N/2 (n2 < N2/2), else as the
            // mirror output of the pair at r' = N - r < N/2 (the mirror column's warp forms the same pair)
#pragma unroll
            for (int n2 = 0; n2 < N2; ++n2) {
                const int r = c + N1 * n2;
                float2 zr, zm;
                if (n2 < N2 / 2) {
                    z_pair(ld(r), ld(N - r), Wq[r], zr, zm);
                    za[n2] = zr;
                } else {
                    z_pair(ld(N - r), ld(r), Wq[N - r], zr, zm);
                    za[n2] = zm;
                }
            }
        }
        gbar();                                            // (A) every U read: slot becomes ZY
        dif4<N2>(za);
        float2 *yw = ZY + lane * SZ + c;
        const float2 *tw = Wn + c * N2;
#pragma unroll
        for (int k1 = 0; k1 < N2; ++k1) {
            float2 x = za[dpos4<N2>(k1)];
            if (k1) x = c_mul(x, tw[k1]);
            yw[k1 * C::SK] = x;
        }
    } else {
    float2 za[N2], zb[N2];
    const int ca = warp == 0 ? 0 : warp;
    const int cb = warp == 0 ? N1 / 2 : N1 - warp;
    if (warp == 0) {
        // column 0: rows N1*n2; pairs (n2, N2 - n2); n2 = 0 -> Z_0, n2 = N2/2 -> Z_{N/2}
        {
            const float2 u0 = ld(0);                                  // (U_0, U_N) packed
            za[0] = make_float2(u0.x + u0.y, u0.x - u0.y);
            const float2 uh = ld(N / 2);
            za[N2 / 2] = make_float2(2.f * uh.x, 2.f * uh.y);
#pragma unroll
            for (int n2 = 1; n2 < N2 / 2; ++n2) z_pair(ld(N1 * n2), ld(N1 * (N2 - n2)), Wq[N1 * n2], za[n2], za[N2 - n2]);
        }
        // column N1/2: rows N1/2 + N1 n2; pairs (n2, N2 - 1 - n2)
#pragma unroll
        for (int n2 = 0; n2 < N2 / 2; ++n2) {
            const int r = N1 / 2 + N1 * n2;
            z_pair(ld(r), ld(N - r), Wq[r], zb[n2], zb[N2 - 1 - n2]);
        }
    } else {
        // columns c and N1 - c: (c, n2) <-> (N1 - c, N2 - 1 - n2)
#pragma unroll
        for (int n2 = 0; n2 < N2 / 2; ++n2) {
            const int ra = ca + N1 * n2, rb = cb + N1 * n2;
            z_pair(ld(ra), ld(N - ra), Wq[ra], za[n2], zb[N2 - 1 - n2]);
            z_pair(ld(rb), ld(N - rb), Wq[rb], zb[n2], za[N2 - 1 - n2]);
        }
    }
    gbar();                                                // (A) every U read: slot becomes ZY
    dif4<N2>(za);
    dif4<N2>(zb);
    {
        float2 *ywa = ZY + lane * SZ + ca, *ywb = ZY + lane * SZ + cb;
        const float2 *twa = Wn + ca * N2, *twb = Wn + cb * N2;
#pragma unroll
        for (int k1 = 0; k1 < N2; ++k1) {
            float2 xa = za[dpos4<N2>(k1)], xb = zb[dpos4<N2>(k1)];
            if (k1) {
                xa = c_mul(xa, twa[k1]);
                xb = c_mul(xb, twb[k1]);
            }
            ywa[k1 * C::SK] = xa;
            ywb[k1 * C::SK] = xb;
        }
    }
    }
    gbar();                                                // (B) ZY complete

    // ---- pass 2
    float2 w[C::P2_PER][N1];
#pragma unroll
    for (int j = 0; j < C::P2_PER; ++j) {
        const int task = gt + GT * j;
        const int p = task / N2, k1 = task % N2;
        const float2 *yr = ZY + p * SZ + k1 * C::SK;
#pragma unroll
        for (int i = 0; i < N1; ++i) w[j][i] = yr[i];
    }
    release();                                             // (C) this thread's reads of the slot are done
#pragma unroll
    for (int j = 0; j < C::P2_PER; ++j) dif4<N1>(w[j]);   // w[dpos4(k2)] = z[k1 + N2 k2]
    if constexpr (MODE == MODE_LANDSCAPE) {
#pragma unroll
        for (int j = 0; j < C::P2_PER; ++j) {
            const int task = gt + GT * j;
            const int p = task / N2, k1 = task % N2;
            if (p < n_valid) {
                const float mul = PI / (smv[j] * st);
                float2 *dst = reinterpret_cast<float2 *>(out.X + (m_first + p) * out.ld_m + t * out.ld_t);
#pragma unroll
                for (int k2 = 0; k2 < N1; ++k2) dst[k1 + N2 * k2] = c_scale(w[j][dpos4<N1>(k2)], mul);
            }
        }
    } else {
        // max over the pair: a balanced tree per task (short dependency chains), then the N2-lane
        // butterfly with the tasks' shuffles interleaved
        const unsigned gmask = N2 >= 32 ? 0xffffffffu
                                        : (((1u << (N2 & 31)) - 1u) << ((threadIdx.x & 31) & ~(N2 - 1)));
        float mx[C::P2_PER];
#pragma unroll
        for (int j = 0; j < C::P2_PER; ++j) {
            float r[N1];
#pragma unroll
            for (int k2 = 0; k2 < N1; ++k2) r[k2] = fmaxf(w[j][k2].x, w[j][k2].y);
#pragma unroll
            for (int h = N1 / 2; h >= 1; h >>= 1)
#pragma unroll
                for (int k2 = 0; k2 < h; ++k2) r[k2] = fmaxf(r[k2], r[k2 + h]);
            mx[j] = r[0];
        }
#pragma unroll
        for (int off = N2 / 2; off >= 1; off >>= 1)
#pragma unroll
            for (int j = 0; j < C::P2_PER; ++j) mx[j] = fmaxf(mx[j], __shfl_xor_sync(gmask, mx[j], off));
#pragma unroll
        for (int j = 0; j < C::P2_PER; ++j) {
            const int task = gt + GT * j;
            const int p = task / N2, k1 = task % N2;
            const bool valid = p < n_valid;
            const int64_t m = m_first + p;
            const float bv = (PI / (smv[j] * st)) * mx[j];
            bool go = valid;
            if constexpr (MODE == MODE_IMAGE) go = valid && ord_f32(bv) >= stale[j];
            if (go) {                                      // uniform over the pair's lanes
                int bk = 0x7fffffff;
#pragma unroll
                for (int k2 = N1 - 1; k2 >= 0; --k2) {     // descending: the smallest index wins
                    const float2 z = w[j][dpos4<N1>(k2)];
                    const int kx = 2 * (k1 + N2 * k2);
                    if (z.y == mx[j]) bk = kx + 1;
                    if (z.x == mx[j]) bk = kx;
                }
#pragma unroll
                for (int off = N2 / 2; off >= 1; off >>= 1) bk = min(bk, __shfl_xor_sync(gmask, bk, off));
                float gam = 0.f;
                if constexpr (MODE == MODE_PAIR) {
                    if (out.best_gamma) gam = parabolic_gamma<N1, N2, true>(w[j], k1, bk, mx[j], gmask);
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

// per-image side data of an item's pass-2 tasks (image scale; MODE_IMAGE: the image's current key),
// fetched before the item's data wait so its latency hides behind it
template <int LOGN, int MODE, bool ONE = false>
__device__ __forceinline__ void fft2_side(int gt, int64_t m_first, int n_valid, const FftOut &out,
                                          uint32_t (&stale)[Fft2Cfg<LOGN, 4, ONE>::P2_PER],
                                          float (&smv)[Fft2Cfg<LOGN, 4, ONE>::P2_PER]) {
    using C = Fft2Cfg<LOGN, 4, ONE>;
#pragma unroll
    for (int j = 0; j < C::P2_PER; ++j) {
        const int p = (gt + C::GT * j) / C::N2;
        const bool ok = p < n_valid;
        smv[j] = (ok && out.sc_m) ? __ldg(out.sc_m + m_first + p) : 1.f;
        stale[j] = 0u;
        if constexpr (MODE == MODE_IMAGE) stale[j] = ok ? (uint32_t)(__ldcg(out.best_key + m_first + p) >> 32) : 0u;
    }
}

// shared tables of the transform: Wn[c][k1] = W_N^{c k1}, Wq[r] = W_Q^r (r < N/2)
template <int LOGN>
__device__ __forceinline__ void fft2_tables(float2 *Wn, float2 *Wq, int tid, int nthreads) {
    using C = Fft2Cfg<LOGN>;
    for (int i = tid; i < C::N; i += nthreads) Wn[i] = twiddle_N(i / C::N2, i % C::N2, C::N);
    for (int i = tid; i < C::N / 2; i += nthreads) {
        float sn, cs;
        sincospif(2.0f * (float)i / (float)C::Q, &sn, &cs);
        Wq[i] = make_float2(cs, -sn);
    }
}

template <int LOGN, int MODE, class Tin = float>
__global__ void __launch_bounds__(Fft2Cfg<LOGN, 4, RSVD_FFT2_ONECOL>::THREADS, 1) fft2_reduce_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                               int64_t m0, int64_t t0, int64_t mcv,
                                                                               int64_t tcv, FftOut out,
                                                                               float *__restrict__ Upk, int64_t Mc,
                                                                               int64_t Tc) {
    using C = Fft2Cfg<LOGN, (int)sizeof(Tin), RSVD_FFT2_ONECOL>;
    constexpr int N = C::N, TB = C::TB, G = C::G, GT = C::GT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // pointer arithmetic on the __shared__ array (not an integer round trip) keeps LDS/STS addressing
    unsigned char *base = smem_raw + ((1024u - (fr_smem(smem_raw) & 1023u)) & 1023u);
    float2 *Wn = reinterpret_cast<float2 *>(base + C::NSLOT * C::SLOT);   // [N1][N2] W_N^{c k1}
    float2 *Wq = Wn + N;                                             // [N/2]  W_Q^r
    uint64_t *full = reinterpret_cast<uint64_t *>(Wq + N / 2);       // [NSLOT]
    // tag[s] = local index of the item whose load was last issued into slot s.  A group may reach
    // its wait for item i while slot i % NSLOT still holds (or is loading) item i - NSLOT: the parity
    // wait alone would then pass one phase early, so it first waits for the tag.
    uint64_t *empty = full + C::NSLOT;                                // [NSLOT] slot read out (TASKS warps)
    volatile int *tag = reinterpret_cast<volatile int *>(empty + C::NSLOT);   // [NSLOT]

    const int tid = threadIdx.x;
    const int g = tid / GT, gt = tid - g * GT;
    const int warp = gt >> 5, lane = tid & 31;
#ifdef RSVD_TRACE
    __shared__ unsigned long long trs[4];
    if (tid == 0) trs[0] = trace_now();
    bool tr_first = true;
#endif
    const int nmb = (int)((mcv + TB - 1) / TB);
    const int nitems = (int)tcv * nmb;
    const int grid = (int)gridDim.x;
    // local index i -> item blockIdx.x + grid * i, processed by group i % G in slot i % NSLOT
    auto item_of = [&](int i) { return (int)blockIdx.x + grid * i; };

    auto issue = [&](int i) {                                    // one thread
        const int it = item_of(i), sl = i % C::NSLOT;
        tag[sl] = i;
        const int tl = it / nmb, mb0 = (it - tl * nmb) * TB;
        const uint32_t bar = fr_smem(full + sl);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((uint32_t)C::UBYTES)
                     : "memory");
#pragma unroll
        for (int bx = 0; bx < C::NBOX; ++bx) {
            const uint32_t dst = fr_smem(base + (size_t)sl * C::SLOT + (size_t)bx * C::BOXR * TB * sizeof(Tin));
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                ::"r"(dst), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(mb0), "r"(tl), "r"(bx * C::BOXR), "r"(bar)
                : "memory");
        }
    };

    // PDL: the next chunk's contraction may be scheduled as SMs free up (it waits for us before
    // writing the workspace); our own input is the previous kernel's output, so wait for it first.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (tid == 0) {
        for (int sl = 0; sl < C::NSLOT; ++sl) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(fr_smem(full + sl)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(fr_smem(empty + sl)), "r"(C::TASKS));
            tag[sl] = -1;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fft2_tables<LOGN>(Wn, Wq, tid, C::THREADS);
    asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef RSVD_TRACE
    if (tid == 0) trs[1] = trace_now();
#endif
    if (tid == 0)
        for (int i = 0; i < C::NSLOT; ++i)
            if (item_of(i) < nitems) issue(i);
    __syncthreads();

    // item coordinates advance by G * grid items per iteration: carry instead of a division per item
    const int step = G * grid, dtl = step / nmb, dmb = step - dtl * nmb;
    int tl = item_of(g) / nmb, mbi = item_of(g) - tl * nmb;
    // this thread's discard rows r = gt, gt + GT, ... (row stride Tc * Mc floats)
    float *const dbase = (Upk && sizeof(Tin) == 4) ? Upk + (int64_t)gt * Tc * Mc : nullptr;
    const int64_t dstride = (int64_t)GT * Tc * Mc;
    for (int i = g; item_of(i) < nitems; i += G, tl += dtl, mbi += dmb) {
        if (mbi >= nmb) { mbi -= nmb; ++tl; }
        const int sl = i % C::NSLOT;
        float *U = reinterpret_cast<float *>(base + (size_t)sl * C::SLOT);    // [ROWS][TB]
        const int mb0 = mbi * TB;
        const int64_t t = t0 + tl;
        const float st = out.sc_t ? __ldg(out.sc_t + t) : 1.f;
        const int n_valid = (int)(mcv - mb0 < TB ? mcv - mb0 : TB);
        uint32_t stale[C::P2_PER];
        float smv[C::P2_PER];
        fft2_side<LOGN, MODE, RSVD_FFT2_ONECOL>(gt, m0 + mb0, n_valid, out, stale, smv);
        while (tag[sl] != i) {}
        fr_mbar_wait(full + sl, (uint32_t)(i / C::NSLOT) & 1u);
#ifdef RSVD_TRACE
        if (tr_first && tid == 0) trs[2] = trace_now();
        tr_first = false;
#endif
        // the item's 2N spectrum rows (one 128-B line each: 32 images x fp32) are now in shared memory
        // and dead in HBM terms: drop them from L2 without write-back (the next chunk's contraction
        // rewrites every line before it is read again)
        if (dbase) {
            const float *pd = dbase + (int64_t)tl * Mc + mb0;
#pragma unroll
            for (int r = gt; r < C::ROWS; r += GT, pd += dstride)
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(pd) : "memory");
        }
        // (C) one arrival per warp once its reads are done (release); only the group's issuing thread
        // waits for all TASKS warps before refilling the slot NSLOT items ahead
        auto release = [&]() {
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(fr_smem(empty + sl)) : "memory");
            if (gt == 0 && item_of(i + C::NSLOT) < nitems) {
                fr_mbar_wait(empty + sl, (uint32_t)(i / C::NSLOT) & 1u);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(i + C::NSLOT);
            }
        };
        fft2_item<LOGN, MODE, decltype(release), Tin, RSVD_FFT2_ONECOL>(U, gt, warp, lane, 1 + g, Wn, Wq, m0 + mb0,
                                                                         n_valid, t, st, stale, smv, out, release);
    }
#ifdef RSVD_TRACE
    __syncthreads();
    if (tid == 0) {
        TraceRec r;
        r.t0 = trs[0]; r.t1 = trs[1]; r.t2 = trs[2]; r.t3 = trace_now();
        r.kind_blk = (1u << 24) | blockIdx.x;
        r.key = ((unsigned)(m0 / 128) << 16) | (unsigned)(t0 / 256);
        trace_put(r);
    }
#endif
}

// 3-D view of the planar workspace with 32-image boxes (the fft2 work item).
// eb = bytes per element: 4 (fp32 spectrum) or 2 (fp16 spectrum of the fast path).
template <int LOGN>
static cudaError_t make_spectrum_tmap2(CUtensorMap *tm, const float *Upk, int64_t Mc, int64_t Tc, int eb = 4) {
    using C = Fft2Cfg<LOGN>;
    PFN_encodeTiled_fr enc = encode_tiled_fn();
    if (!enc) return cudaErrorNotSupported;
    const cuuint64_t dims[3] = {(cuuint64_t)Mc, (cuuint64_t)Tc, (cuuint64_t)C::ROWS};
    const cuuint64_t strides[2] = {(cuuint64_t)Mc * eb, (cuuint64_t)Mc * Tc * eb};
    const cuuint32_t box[3] = {(cuuint32_t)C::TB, 1u, (cuuint32_t)C::BOXR};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    const CUresult r = enc(tm, eb == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(Upk), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)RSVD_FFT2_L2PROMO,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int LOGN, int MODE, class Tin = float>
static cudaError_t launch_fft2_mode(cudaStream_t s, const CUtensorMap &tm, int64_t m0, int64_t t0, int64_t mcv,
                                    int64_t tcv, const FftOut &out, float *Upk, int64_t Mc, int64_t Tc) {
    using C = Fft2Cfg<LOGN, (int)sizeof(Tin), RSVD_FFT2_ONECOL>;
    const size_t smem = C::smem_bytes();
    static std::atomic<uint64_t> attr{0};
    const cudaError_t e = smem_attr_once((const void *)fft2_reduce_kernel<LOGN, MODE, Tin>, (int)smem, attr);
    if (e != cudaSuccess) return e;
    const int64_t nitems = tcv * ((mcv + C::TB - 1) / C::TB);
    const int64_t grid = std::min<int64_t>((nitems + C::G - 1) / C::G, (int64_t)num_sms());
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(C::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fft2_reduce_kernel<LOGN, MODE, Tin>, tm, m0, t0, mcv, tcv, out, Upk, Mc, Tc);
}

template <int LOGN, class Tin = float>
static cudaError_t launch_fft2_t(int mode, cudaStream_t s, const CUtensorMap &tm, int64_t m0, int64_t t0, int64_t mcv,
                                 int64_t tcv, const FftOut &out, float *Upk, int64_t Mc, int64_t Tc) {
    if (mode == MODE_PAIR) return launch_fft2_mode<LOGN, MODE_PAIR, Tin>(s, tm, m0, t0, mcv, tcv, out, Upk, Mc, Tc);
    if (mode == MODE_IMAGE) return launch_fft2_mode<LOGN, MODE_IMAGE, Tin>(s, tm, m0, t0, mcv, tcv, out, Upk, Mc, Tc);
    return launch_fft2_mode<LOGN, MODE_LANDSCAPE, Tin>(s, tm, m0, t0, mcv, tcv, out, Upk, Mc, Tc);
}
template <int LOGN>
static cudaError_t launch_fft2(int mode, cudaStream_t s, const CUtensorMap &tm, int64_t m0, int64_t t0, int64_t mcv,
                               int64_t tcv, const FftOut &out, float *Upk, int64_t Mc, int64_t Tc, bool half = false) {
    return half ? launch_fft2_t<LOGN, __half>(mode, s, tm, m0, t0, mcv, tcv, out, Upk, Mc, Tc)
                : launch_fft2_t<LOGN, float>(mode, s, tm, m0, t0, mcv, tcv, out, Upk, Mc, Tc);
}

}  // namespace rsvd
