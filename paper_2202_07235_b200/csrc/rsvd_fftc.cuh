// rsvd_fftc.cuh -- Steps 3-4 of the align path (PAPER.md:673 transform, forward sign per DESIGN.md
// G3; PAPER.md:504-517 argmax) with pass 1 of the four-step transform on the tcgen05 tensor cores.
//
// The mathematics is rsvd_fft2.cuh's: Z_n = (U_n + conj U_{N-n}) + i W_Q^n (U_n - conj U_{N-n}),
// z = DFT_N(Z) by the four-step split n = n1 + N1 n2, Re X_k = pi x_k with z_k = x_2k + i x_2k+1.
// Pass 1 -- Z for a mirror column pair {c, N1 - c} (warp-level in fft2), the DFT of length N2 over n2
// and the twiddle W_N^{c k1} -- is LINEAR in the 64 real inputs (Re, Im of the pair's 2 N2 spectrum
// slots, including the packed (U_0, U_N) slot), so it is one real 64 x 64 matrix B_cp per column pair,
// built once on the host in fp64 (fftc_build_matrices, a direct transcription of fft2's pass 1).
// Here:
//   spectrum   the contraction (rsvd_tc.cu, fmt 2) stores every value x = v 2^-20 as fp16 hi = fp16(x)
//              and lo = fp16((x - hi) 2^10) in planes [n][part][t][m], part = re_hi, im_hi, re_lo, im_lo
//              (4 B per value, as fp32);
//   stage A    per batch (one template x 128 images) and column pair: the pair's hi and lo planes land
//              by TMA (5-D map, SWIZZLE_128B) as two MN-major [128 images x 64 inputs] fp16 operand
//              tiles, B_cp (hi, lo; K-major, pre-swizzled) by a bulk copy; three kind::f16 MMAs per
//              K = 16 step (A_hi B_hi + A_hi B_lo + A_lo B_hi, fp32 accumulate: ~2^-22 per term) write
//              Y[k1][c] for the pair's two columns into TMEM (lane = image, 64 columns per pair);
//   stage B    16 SIMT warps read Y from TMEM (warp w: lane quadrant w % 4, k1 in [4 (w / 4), +4)),
//              run pass 2 (the DFT of length N1 over the columns, exactly fft2's) and the max / first
//              argmax over their k1; the 4 warps of a quadrant combine through shared memory.
// Warp roles: 0-15 stage B, 16 TMA producer, 17 TMEM allocator + MMA issuer.  A 4-stage ring
// (48 KB per stage: A hi/lo 32 KB + B 16 KB) feeds the MMA; TMEM holds 1 (N = 256) or 2 (N = 128)
// batches.  Per-pair and per-image modes (landscape stays on fft2, whose lanes store coalesced rows).
#pragma once

#include <cuda_fp16.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "rsvd_fft2.cuh"
#include "rsvd_tcgen05.cuh"

namespace rsvd {

template <int LOGN>
struct FftcCfg {
    static constexpr int N = 1 << LOGN;
    static constexpr int Q = 2 * N;
    static constexpr int N1 = 1 << (LOGN / 2);        // columns
    static constexpr int N2 = N / N1;                 // rows (16 for LOGN = 7, 8)
    static constexpr int NCP = N1 / 2;                // mirror column pairs
    static constexpr int BM = 128;                    // images per batch (MMA M)
    static constexpr uint32_t A_BYTES = 32768;        // [hl][mh][col][32 rows x 128 B]
    static constexpr uint32_t B_BYTES = 16384;        // B_hi, B_lo: 64 rows x 128 B each
    static constexpr uint32_t STAGE = A_BYTES;        // A ring; every B_cp stays resident
    static constexpr uint32_t BRES = (uint32_t)NCP * B_BYTES;
    static constexpr int STAGES = NCP == 8 ? 2 : 4;
    static constexpr int SUBS = 4;                    // stage-B warps per TMEM lane quadrant
    static constexpr int KPS = N2 / SUBS;             // k1 values per stage-B warp
    static constexpr int TCOLS = NCP * 64;            // TMEM columns per batch
    static constexpr int NACC = 512 / TCOLS;          // batches resident in TMEM
    static constexpr int THREADS = 18 * 32;
    static_assert(N2 == 16, "fftc: N in {128, 256}");
    static constexpr size_t smem_bytes() {
        return 1024 + (size_t)BRES + (size_t)STAGES * STAGE + 2 * SUBS * 128 * 8 + (2 * STAGES + 2 * NACC + 1) * 8 + 16;
    }
};

__host__ __device__ constexpr int fftc_ca(int cp, int N1) { return cp == 0 ? 0 : cp; }
__host__ __device__ constexpr int fftc_cb(int cp, int N1) { return cp == 0 ? N1 / 2 : N1 - cp; }

// UMMA shared-memory descriptor for an MN-major SWIZZLE_128B tile: 64-element (128 B) MN rows, 8-row
// K atoms 1024 B apart (SBO), MN blocks of 64 elements LBO bytes apart.
__device__ __forceinline__ uint64_t mn_sw128_desc(uint32_t saddr, uint32_t lbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
__device__ __forceinline__ void tc_mma_f16_1(uint32_t dtmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dtmem),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
}
// D = A B + D 2^-10 (scale-input-d): folds the 2^10-prescaled correction terms back into the result
__device__ __forceinline__ void tc_mma_f16_1_sd10(uint32_t dtmem, uint64_t da, uint64_t db, uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, 1, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p, 10;\n\t}\n" ::"r"(dtmem),
        "l"(da), "l"(db), "r"(idesc)
        : "memory");
}
__device__ __forceinline__ void tc_commit_1(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld_x4(uint32_t taddr, uint32_t (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr));
}
__device__ __forceinline__ void mbar_arrive_local(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

template <int LOGN, int MODE>
__global__ void __launch_bounds__(FftcCfg<LOGN>::THREADS, 1)
    fftc_reduce_kernel(const __grid_constant__ CUtensorMap tmS, const unsigned char *__restrict__ Bg, int64_t m0,
                       int64_t t0, int64_t mcv, int64_t tcv, FftOut out, int64_t Mc) {
    using C = FftcCfg<LOGN>;
    constexpr int N1 = C::N1, N2 = C::N2, NCP = C::NCP, Q = C::Q;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char *bres = base + C::STAGES * C::STAGE;                              // [NCP][B_BYTES]
    float2 *red = reinterpret_cast<float2 *>(bres + C::BRES);                       // [2][SUBS][128] (value, index)
    uint64_t *bfull = reinterpret_cast<uint64_t *>(red + 2 * C::SUBS * 128);
    uint64_t *full = bfull + 1;
    uint64_t *empty = full + C::STAGES;
    uint64_t *tfull = empty + C::STAGES;
    uint64_t *tempty = tfull + C::NACC;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + C::NACC);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nbm = (int)(Mc / C::BM);
    const int nitems = (int)tcv * nbm;
    const int grid = (int)gridDim.x;

    if (warp == 16 && lane == 0) {
        for (int s = 0; s < C::STAGES; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
        for (int a = 0; a < C::NACC; ++a) { mbar_init(tfull + a, 1); mbar_init(tempty + a, 16); }
        mbar_init(bfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 17) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    asm volatile("griddepcontrol.wait;" ::: "memory");

    if (warp == 16) {
        // ---------------- producer: per (batch, column pair) the A hi/lo tiles (8 TMA boxes) + B_cp
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmS)) : "memory");
            int it = 0;
            // the pass-1 matrices once per CTA (resident for the whole kernel)
            mbar_expect_tx(bfull, C::BRES);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(bres)),
                "l"(Bg), "r"(C::BRES), "r"(smem_u32(bfull))
                : "memory");
            for (int item = blockIdx.x; item < nitems; item += grid) {
                const int tl = item / nbm, mb = item - tl * nbm;
#pragma unroll 1
                for (int cp = 0; cp < NCP; ++cp, ++it) {
                    const int s = it % C::STAGES;
                    mbar_wait(empty + s, ((uint32_t)(it / C::STAGES) & 1u) ^ 1u);
                    const uint32_t fb = smem_u32(full + s);
                    mbar_expect_tx(full + s, C::STAGE);
                    const uint32_t st = smem_u32(base + (size_t)s * C::STAGE);
                    const int cols[2] = {fftc_ca(cp, N1), fftc_cb(cp, N1)};
#pragma unroll
                    for (int hl = 0; hl < 2; ++hl)
#pragma unroll
                        for (int mh = 0; mh < 2; ++mh)
#pragma unroll
                            for (int col = 0; col < 2; ++col) {
                                const uint32_t dst = st + (uint32_t)(hl * 16384 + mh * 8192 + col * 4096);
                                asm volatile(
                                    "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
                                    " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
                                    "l"(reinterpret_cast<uint64_t>(&tmS)), "r"(mb * C::BM + 64 * mh), "r"(tl),
                                    "r"(2 * hl), "r"(cols[col]), "r"(0), "r"(fb)
                                    : "memory");
                            }
                }
            }
            for (int k = 0; k < C::STAGES && k < it; ++k) {          // drain: the last commits have landed
                const int j = it - 1 - k;
                mbar_wait(empty + (j % C::STAGES), (uint32_t)(j / C::STAGES) & 1u);
            }
        }
    } else if (warp == 17) {
        // ---------------- MMA issuer: D[image][out] += A[image][in] B[out][in] (M = 128, N = 64, K = 64)
        if (lane == 0) {
            const uint32_t idesc = (1u << 4) | (1u << 15) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
            int it = 0, bi = 0;
            mbar_wait(bfull, 0);
            for (int item = blockIdx.x; item < nitems; item += grid, ++bi) {
                const int acc = bi % C::NACC;
                mbar_wait(tempty + acc, (((uint32_t)(bi / C::NACC)) & 1u) ^ 1u);
                tc_fence_after();
#pragma unroll 1
                for (int cp = 0; cp < NCP; ++cp, ++it) {
                    const int s = it % C::STAGES;
                    mbar_wait(full + s, (uint32_t)(it / C::STAGES) & 1u);
                    tc_fence_after();
                    const uint32_t st = smem_u32(base + (size_t)s * C::STAGE);
                    const uint64_t a_hi = mn_sw128_desc(st, 8192), a_lo = mn_sw128_desc(st + 16384, 8192);
                    const uint32_t sb = smem_u32(bres + (size_t)cp * C::B_BYTES);
                    const uint64_t b_hi = sw128_desc(sb), b_lo = sw128_desc(sb + 8192);
                    const uint32_t dt = tmem + (uint32_t)(acc * C::TCOLS + cp * 64);
                    // corrections first, each operand's lo part stored x 2^10 (keeps it out of the fp16
                    // subnormals, which the tensor core flushes): D = 2^10 (A_lo B_hi + A_hi B_lo); then
                    // D = A_hi B_hi + 2^-10 D (scale-input-d) and the remaining hi x hi steps
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t oa = (uint64_t)(128 * k), ob = (uint64_t)(2 * k);   // 2 KB / 32 B per K = 16
                        tc_mma_f16_1(dt, a_lo + oa, b_hi + ob, idesc, k ? 1u : 0u);
                        tc_mma_f16_1(dt, a_hi + oa, b_lo + ob, idesc, 1u);
                    }
                    tc_mma_f16_1_sd10(dt, a_hi, b_hi, idesc);
#pragma unroll
                    for (int k = 1; k < 4; ++k)
                        tc_mma_f16_1(dt, a_hi + (uint64_t)(128 * k), b_hi + (uint64_t)(2 * k), idesc, 1u);
                    tc_commit_1(empty + s);
                }
                tc_commit_1(tfull + acc);
            }
        }
    } else {
        // ---------------- stage B: pass 2 + max / first argmax from TMEM
        const int quad = warp & 3, sub = warp >> 2;
        const int row = quad * 32 + lane;                   // image within the batch
        const float PI = 3.14159265358979323846f / RSVD_SPLIT_SCALE;
        int bi = 0;
        for (int item = blockIdx.x; item < nitems; item += grid, ++bi) {
            const int tl = item / nbm, mb = item - tl * nbm;
            const int acc = bi % C::NACC;
            const int64_t t = t0 + tl;
            const int64_t ml = (int64_t)mb * C::BM + row;
            const bool valid = ml < mcv;
            const int64_t m = m0 + ml;
            const float st = out.sc_t ? __ldg(out.sc_t + t) : 1.f;
            const float smv = (valid && out.sc_m) ? __ldg(out.sc_m + m) : 1.f;
            uint32_t stale = 0u;
            if constexpr (MODE == MODE_IMAGE) {
                if (sub == 0 && valid) stale = (uint32_t)(__ldcg(out.best_key + m) >> 32);
            }
            mbar_wait(tfull + acc, ((uint32_t)(bi / C::NACC)) & 1u);
            tc_fence_after();
            const uint32_t tb = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * C::TCOLS);
            float bestv = -INFINITY;
            int bestk = 0x7fffffff;
#pragma unroll 1
            for (int kk = 0; kk < C::KPS; ++kk) {
                const int k1 = sub * C::KPS + kk;
                uint32_t r[NCP][4];
#pragma unroll
                for (int cp = 0; cp < NCP; ++cp) tmem_ld_x4(tb + (uint32_t)(cp * 64 + k1 * 4), r[cp]);
                tmem_wait_ld();
                float2 w[N1];
#pragma unroll
                for (int cp = 0; cp < NCP; ++cp) {
                    w[fftc_ca(cp, N1)] = make_float2(__uint_as_float(r[cp][0]), __uint_as_float(r[cp][1]));
                    w[fftc_cb(cp, N1)] = make_float2(__uint_as_float(r[cp][2]), __uint_as_float(r[cp][3]));
                }
                dif4<N1>(w);                                 // w[dpos4(k2)] = z[k1 + N2 k2]
#pragma unroll
                for (int k2 = 0; k2 < N1; ++k2) {            // ascending k: strict > keeps the first maximum
                    const float2 z = w[dpos4<N1>(k2)];
                    const int kx = 2 * (k1 + N2 * k2);
                    if (z.x > bestv || (z.x == bestv && kx < bestk)) { bestv = z.x; bestk = kx; }
                    if (z.y > bestv || (z.y == bestv && kx + 1 < bestk)) { bestv = z.y; bestk = kx + 1; }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_local(tempty + acc);  // this warp's TMEM reads of the batch are done
            float2 *rb = red + (size_t)(bi & 1) * C::SUBS * 128;
            rb[sub * 128 + row] = make_float2(bestv, __int_as_float(bestk));
            asm volatile("bar.sync %0, %1;" ::"r"(1 + quad), "n"(128) : "memory");
            if (sub == 0 && valid) {
                float v = rb[row].x;
                int k = __float_as_int(rb[row].y);
#pragma unroll
                for (int j = 1; j < C::SUBS; ++j) {
                    const float2 e = rb[j * 128 + row];
                    const int ke = __float_as_int(e.y);
                    if (e.x > v || (e.x == v && ke < k)) { v = e.x; k = ke; }
                }
                const float bv = (PI / (smv * st)) * v;
                if constexpr (MODE == MODE_PAIR) {
                    out.best_val[m * out.T + t] = bv;
                    out.best_k[m * out.T + t] = k;
                } else {
                    if (ord_f32(bv) >= stale) {
                        const uint32_t idx = (uint32_t)((out.t_offset + t) * Q + k);
                        const unsigned long long key =
                            ((unsigned long long)ord_f32(bv) << 32) | (unsigned long long)(0xFFFFFFFFu - idx);
                        atomicMax(out.best_key + m, key);
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 17) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// ------------------------------------------------------------------ host: pass-1 matrices
// Pass 1 of fft2 for column pair cp applied to the 64 real inputs in[] (column ca then cb; per column
// n2-major, (Re, Im) of slot n = c + N1 n2; slot 0 holds (U_0, U_N)), in fp64: the 64 outputs
// out[k1 * 4 + colsel * 2 + reim] = Re / Im of W_N^{c k1} sum_n2 W_N2^{n2 k1} Z[c + N1 n2].
template <int LOGN>
static void fftc_pass1_ref(int cp, const double *in, double *outv) {
    using C = FftcCfg<LOGN>;
    constexpr int N = C::N, Q = C::Q, N1 = C::N1, N2 = C::N2;
    const int cols[2] = {fftc_ca(cp, N1), fftc_cb(cp, N1)};
    auto slot = [&](int n, double &re, double &im) {          // slot value of n in this pair's columns
        const int c = n % N1, n2 = n / N1, sel = (c == cols[0]) ? 0 : 1;
        re = in[sel * 32 + n2 * 2];
        im = in[sel * 32 + n2 * 2 + 1];
    };
    const double PI = 3.14159265358979323846;
    for (int sel = 0; sel < 2; ++sel) {
        const int c = cols[sel];
        double zr[N2], zi[N2];
        for (int n2 = 0; n2 < N2; ++n2) {
            const int n = c + N1 * n2;
            double ar, ai, br, bi;
            if (n == 0) {                                    // (U_0, U_N): Z_0 = (U_0 + U_N) + i (U_0 - U_N)
                slot(0, ar, ai);
                zr[n2] = ar + ai;
                zi[n2] = ar - ai;
                continue;
            }
            if (n == N / 2) {                                // Z_{N/2} = 2 U_{N/2}
                slot(n, ar, ai);
                zr[n2] = 2 * ar;
                zi[n2] = 2 * ai;
                continue;
            }
            const int r = n < N / 2 ? n : N - n;             // z_pair(U_r, U_{N-r}, W_Q^r)
            slot(r, ar, ai);
            slot(N - r, br, bi);
            const double sr = ar + br, si = ai - bi, dr = ar - br, di = ai + bi;
            const double wr = cos(2 * PI * r / Q), wi = -sin(2 * PI * r / Q);
            const double pr = dr * wr - di * wi, pi = dr * wi + di * wr;
            if (n < N / 2) { zr[n2] = sr - pi; zi[n2] = si + pr; }           // Z_n = s + i p
            else { zr[n2] = sr + pi; zi[n2] = pr - si; }                      // Z_n = conj(s) + i conj(p)
        }
        for (int k1 = 0; k1 < N2; ++k1) {
            double yr = 0, yi = 0;
            for (int n2 = 0; n2 < N2; ++n2) {
                const double a = -2 * PI * (double)(n2 * k1) / N2;
                yr += zr[n2] * cos(a) - zi[n2] * sin(a);
                yi += zr[n2] * sin(a) + zi[n2] * cos(a);
            }
            const double a = -2 * PI * (double)((c * k1) % N) / N;
            outv[k1 * 4 + sel * 2] = yr * cos(a) - yi * sin(a);
            outv[k1 * 4 + sel * 2 + 1] = yr * sin(a) + yi * cos(a);
        }
    }
}

// B_cp (hi, lo) for every column pair, K-major SWIZZLE_128B images (64 rows x 128 B), NCP x 16 KB.
template <int LOGN>
static std::vector<unsigned char> fftc_build_matrices() {
    using C = FftcCfg<LOGN>;
    std::vector<unsigned char> img((size_t)C::NCP * C::B_BYTES, 0);
    std::vector<double> e(64), o(64);
    for (int cp = 0; cp < C::NCP; ++cp) {
        double Bm[64][64];
        for (int k = 0; k < 64; ++k) {
            for (int j = 0; j < 64; ++j) e[j] = (j == k) ? 1.0 : 0.0;
            fftc_pass1_ref<LOGN>(cp, e.data(), o.data());
            for (int r = 0; r < 64; ++r) Bm[r][k] = o[r];
        }
        for (int hl = 0; hl < 2; ++hl)
            for (int r = 0; r < 64; ++r)
                for (int k = 0; k < 64; ++k) {
                    const float x = (float)Bm[r][k];
                    const __half hi = __float2half_rn(x);
                    const __half v = hl == 0 ? hi : __float2half_rn((float)((Bm[r][k] - (double)__half2float(hi)) * 1024.0));
                    const size_t byte = (size_t)r * 128 + ((((size_t)k * 2) >> 4) ^ (size_t)(r & 7)) * 16 + (((size_t)k * 2) & 15);
                    std::memcpy(&img[(size_t)cp * C::B_BYTES + (size_t)hl * 8192 + byte], &v, 2);
                }
    }
    return img;
}

// pass-1 matrices on the current device (built and uploaded once per device and N)
template <int LOGN>
static const unsigned char *fftc_matrices_dev(cudaError_t *err) {
    static std::mutex mu;
    static const unsigned char *cache[64] = {};
    int dev = 0;
    *err = cudaGetDevice(&dev);
    if (*err != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> g(mu);
    if (!cache[dev & 63]) {
        const std::vector<unsigned char> img = fftc_build_matrices<LOGN>();
        void *p = nullptr;
        if ((*err = cudaMalloc(&p, img.size())) != cudaSuccess) return nullptr;
        if ((*err = cudaMemcpy(p, img.data(), img.size(), cudaMemcpyHostToDevice)) != cudaSuccess) return nullptr;
        cache[dev & 63] = static_cast<const unsigned char *>(p);
    }
    return cache[dev & 63];
}

// 5-D view of the split spectrum: (image m, template t, part, n1, n2), n = n1 + N1 n2; box (64, 1, 2, 1, N2)
template <int LOGN>
static cudaError_t make_fftc_tmap(CUtensorMap *tm, const void *Upk, int64_t Mc, int64_t Tc) {
    using C = FftcCfg<LOGN>;
    PFN_encodeTiled_fr enc = encode_tiled_fn();
    if (!enc) return cudaErrorNotSupported;
    const cuuint64_t dims[5] = {(cuuint64_t)Mc, (cuuint64_t)Tc, 4, (cuuint64_t)C::N1, (cuuint64_t)C::N2};
    const cuuint64_t strides[4] = {(cuuint64_t)Mc * 2, (cuuint64_t)Mc * Tc * 2, (cuuint64_t)Mc * Tc * 8,
                                   (cuuint64_t)Mc * Tc * 8 * C::N1};
    const cuuint32_t box[5] = {64u, 1u, 2u, 1u, (cuuint32_t)C::N2};
    const cuuint32_t estr[5] = {1u, 1u, 1u, 1u, 1u};
    const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, const_cast<void *>(Upk), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int LOGN, int MODE>
static cudaError_t launch_fftc_mode(cudaStream_t s, const CUtensorMap &tm, const unsigned char *Bg, int64_t m0,
                                    int64_t t0, int64_t mcv, int64_t tcv, const FftOut &out, int64_t Mc) {
    using C = FftcCfg<LOGN>;
    const size_t smem = C::smem_bytes();
    static std::atomic<uint64_t> attr{0};
    const cudaError_t e = smem_attr_once((const void *)fftc_reduce_kernel<LOGN, MODE>, (int)smem, attr);
    if (e != cudaSuccess) return e;
    const int64_t nitems = tcv * (Mc / C::BM);
    const int64_t grid = std::min<int64_t>(nitems, (int64_t)num_sms());
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
    return cudaLaunchKernelEx(&cfg, fftc_reduce_kernel<LOGN, MODE>, tm, Bg, m0, t0, mcv, tcv, out, Mc);
}

// Steps 3-4 on one chunk of the split spectrum (rsvd_align.cu, fmt 2); modes PAIR / IMAGE, LOGN 7 or 8.
static cudaError_t launch_fftc(int LOGN, int mode, cudaStream_t s, const CUtensorMap &tm, int64_t m0, int64_t t0,
                               int64_t mcv, int64_t tcv, const FftOut &out, int64_t Mc) {
    cudaError_t e = cudaSuccess;
    if (LOGN == 8) {
        const unsigned char *Bg = fftc_matrices_dev<8>(&e);
        if (!Bg) return e;
        return mode == MODE_PAIR ? launch_fftc_mode<8, MODE_PAIR>(s, tm, Bg, m0, t0, mcv, tcv, out, Mc)
                                 : launch_fftc_mode<8, MODE_IMAGE>(s, tm, Bg, m0, t0, mcv, tcv, out, Mc);
    }
    const unsigned char *Bg = fftc_matrices_dev<7>(&e);
    if (!Bg) return e;
    return mode == MODE_PAIR ? launch_fftc_mode<7, MODE_PAIR>(s, tm, Bg, m0, t0, mcv, tcv, out, Mc)
                             : launch_fftc_mode<7, MODE_IMAGE>(s, tm, Bg, m0, t0, mcv, tcv, out, Mc);
}
static cudaError_t make_fftc_tmap_any(int LOGN, CUtensorMap *tm, const void *Upk, int64_t Mc, int64_t Tc) {
    return LOGN == 8 ? make_fftc_tmap<8>(tm, Upk, Mc, Tc) : make_fftc_tmap<7>(tm, Upk, Mc, Tc);
}

}  // namespace rsvd
