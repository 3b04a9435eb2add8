// rsvd_tc.cu -- tensor-core path of Step 2 (the q-batched complex contraction) on
// sm_100a: tcgen05.mma kind::f16 on CTA pairs (cta_group::2, M = 256) with an fp16 hi/lo split of
// both operands (error-compensated, ~fp32 accuracy), TMA-fed from operand rows that Step 1 (compress)
// writes pre-expanded, plus the path selection.
//
// Real embedding of U_q[m,t] = sum_j alpha[q][j][m] beta[q][j][t] (alpha/beta: rsvd_compress.cu):
// two A rows per image and one B row per template (K = 4H reals, j-interleaved),
//   A_re[m] = (Re a_j, -Im a_j)_j ,  A_im[m] = (Im a_j, Re a_j)_j ,  B[t] = (Re b_j, Im b_j)_j
//   D[m][t] = A_re . B = Re U ,  D[64 + m][t] = A_im . B = Im U      (per CTA: 64 images).
// Each row is scaled by an exact power of two s (row max in [2^13, 2^14)) and split
// x s = hi + lo, hi = fp16(x s), lo = fp16(x s - hi); D = Ahi Bhi + Ahi Blo + Alo Bhi (fp32
// accumulation in TMEM) carries ~2^-22 relative error per term.  The Step-3 kernel multiplies each
// pair's result by 1 / (s_m s_t) (exact).
//
// Operand layout (opaque; written by compress_tc_kernel), per side, fp16:
//   op[q][kb][row][64],  q = 0..N (N = Q/2), kb < KB = ceil(4H/32); elements 0-31 of a row are the
//   hi parts of the k-block's 32 reals, 32-63 the lo parts (one 128-B line per row and k-block),
//   image rows: image m -> rows (m/64)*128 + m%64 (A_re) and + 64 (A_im); 2 * round_up(M,128) rows;
//   template rows: t; round_up(T,256) rows.  Then float scale[rows_pad] (s per image / template).
// A 4-D tensor map (64 x rows x KB x (N+1)) with SWIZZLE_128B loads one (q, kb) box of 128 rows x
// 128 B (16 KB, full-line TMA requests) straight into the UMMA K-major SW128 layout, where hi and lo
// are the two 32-element K halves of the same tile (descriptor start +0 / +64 B).
//
// contract_tc_kernel: one CTA pair per (128-image x 256-template tile, group of q), 6 warps per CTA:
//   warp 0    TMA producer (both CTAs: own 128 A rows + own half of the 256 B rows; completion on the
//             leader's full barrier, expect_tx posted by the leader);
//   warp 1    TMEM allocator (both) + MMA issuer (leader): per stage 3 x (1 or 2) tcgen05.mma
//             256x256x16 into one of two 256-column accumulators, commits multicast to both CTAs;
//   warps 2-5 epilogue (both): tcgen05.ld 32x32b of their lane quadrant (lanes 0-63 Re U, 64-127
//             Im U), coalesced stores to the planar spectrum workspace, remote arrive on the
//             leader's accumulator-empty barrier.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "rsvd_common.cuh"
#include "rsvd_tcgen05.cuh"

namespace rsvd {

typedef CUresult (*PFN_encodeTiled_tc)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                       const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled_tc encode_fn() {
    static PFN_encodeTiled_tc fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled_tc>(p);
    }
    return fn;
}

#ifdef RSVD_TRACE
RSVD_TRACE_DEFINE(contract)
#endif
constexpr int TC_THREADS = 6 * 32;
constexpr int TC_STAGES = 7;
constexpr int TC_PIMG = 128;                        // images per CTA pair (64 per CTA)
constexpr int TC_TT = 256;                          // templates per CTA pair (128 per CTA)
constexpr uint32_t TC_OPND_BYTES = 128u * 128u;     // 128 rows x (32 hi + 32 lo) fp16
constexpr uint32_t TC_STAGE_BYTES = 2 * TC_OPND_BYTES;    // A + B: 32 KB
constexpr size_t TC_SMEM = (size_t)TC_STAGES * TC_STAGE_BYTES + 1024 + 256;

int tc_kb(int H) { return (H + 7) / 8; }                    // 32-element k-blocks of K = 4H
static int tc_steps(int H) { return (4 * H + 15) / 16; }    // K = 16 MMA steps
int64_t tc_rows_pad_side(int64_t rows, int side) { return round_up(rows, side == RSVD_SIDE_TEMPLATE ? TC_TT : TC_PIMG); }
int64_t tc_rows_pad(int64_t rows) { return round_up(rows, 256); }
static int64_t tc_op_rows(int64_t rows, int side) {
    return side == RSVD_SIDE_TEMPLATE ? round_up(rows, TC_TT) : 2 * round_up(rows, TC_PIMG);
}
static int64_t tc_op_bytes(int64_t rows, int Q, int H, int side) {
    return (int64_t)(Q / 2 + 1) * tc_kb(H) * 2 * tc_op_rows(rows, side) * 64;
}
int64_t tc_block_bytes(int64_t rows, int Q, int H, int side) {
    return tc_op_bytes(rows, Q, H, side) + round_up(tc_rows_pad_side(rows, side) * 4, 256);
}
const float *tc_scales(const void *blocks, int64_t rows, int Q, int H, int side) {
    return reinterpret_cast<const float *>(reinterpret_cast<const char *>(blocks) + tc_op_bytes(rows, Q, H, side));
}

// ------------------------------------------------------------------ contraction kernel
#ifndef RSVD_TC_L2PROMO
#define RSVD_TC_L2PROMO 3       // operand TMA L2 promotion (CUtensorMapL2promotion; 3 = 256B)
#endif
#ifndef RSVD_WS_POLICY
#define RSVD_WS_POLICY 2      // spectrum-store L2 policy: 0 default, 1 evict_last, 2 evict_first (measured best)
#endif
// Spectrum stores carry an L2 evict_first hint: measured on Large, the contraction drops from 73.4 to
// 65.9 ms (the transform, which reads the chunk back, is unchanged at 80 ms; align 133.7 -> 132.0 ms).
__device__ __forceinline__ void st_spectrum(float *p, float v, uint64_t pol) {
#if RSVD_WS_POLICY == 0
    (void)pol;
    *p = v;
#else
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
#endif
}
// Items (tile, q-group) of one chunk, tile = (128-image tile mt_l < mtl, 256-template tile nt_l < ntl);
// cluster c processes items c, c + nclusters, ...  Upk planar: re plane [(n*Tc + tl)*Mc + ml], im
// plane at + N*Mc*Tc (floats); slot n = 0 packs (U_0, U_N).
template <int fmt>      // compile-time spectrum format: one lean epilogue per format
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1) contract_tc_kernel(
    const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int steps, int KB, int N,
    int mtl, int ntl, int mt0, int nt0, int qg, int nqg, int nitems, int64_t Mc, int64_t Tc,
    float *__restrict__ Upk, int Nout, int operands_fresh) {
    // fmt: spectrum format -- 0 fp32 planes; 1 fp16 planes (single-MMA fast path); 2 split fp16 hi/lo
    // planes for the tensor-core transform (rsvd_fftc.cuh): [n][part][t][m], part = re_hi, im_hi, re_lo,
    // im_lo, value = (hi + lo 2^-10) 2^20
    constexpr bool fast = fmt == 1;
    extern __shared__ unsigned char smem_raw[];
    unsigned char *base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint64_t *bars = reinterpret_cast<uint64_t *>(base + TC_STAGES * TC_STAGE_BYTES);
    uint64_t *full = bars, *empty = bars + TC_STAGES, *tfull = bars + 2 * TC_STAGES, *tempty = bars + 2 * TC_STAGES + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * TC_STAGES + 4);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_rank();
    const int cl = (int)(blockIdx.x >> 1), ncl = (int)(gridDim.x >> 1);
#ifdef RSVD_TRACE
    __shared__ unsigned long long trs[4];
    if (tid == 0) trs[0] = trace_now();
#endif
    // PDL: the next kernel (Step 3 on this chunk) may be scheduled as SMs free up; it waits for us.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < TC_STAGES; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
        for (int a = 0; a < 2; ++a) { mbar_init(tfull + a, 1); mbar_init(tempty + a, 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer (both CTAs)
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
            // PDL: the operand rows may have just been written by the kernel before us on the stream
            // (Step 1, compress): then the first TMA must wait for that grid.  Later chunks of one align
            // call follow the library's own Step-3 kernel, which does not write operands, so their
            // loads may overlap its tail.
            if (operands_fresh) asm volatile("griddepcontrol.wait;" ::: "memory");
            // chunks run template-tile outer / image inner: a chunk's template operands are re-read by
            // every following chunk of the same template tile, image operands by none of them
            uint64_t pol_stream, pol_keep;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
            int it = 0;
            for (int item = cl; item < nitems; item += ncl) {
                const int tile = item / nqg, qgi = item - tile * nqg;
                const int mt_l = tile / ntl, nt_l = tile - mt_l * ntl;
                const int q_begin = qgi * qg, q_end = min(N + 1, q_begin + qg);
                const int rowA = (mt0 + mt_l) * 2 * TC_PIMG + (int)rank * 128;
                const int rowB = (nt0 + nt_l) * TC_TT + (int)rank * 128;
                for (int q = q_begin; q < q_end; ++q) {
                    for (int kb = 0; kb < KB; ++kb, ++it) {
                        const int s = it % TC_STAGES;
                        mbar_wait(empty + s, ((uint32_t)(it / TC_STAGES) & 1u) ^ 1u);
                        const uint32_t fb = smem_u32(full + s);
                        if (rank == 0) mbar_expect_tx(full + s, 2 * TC_STAGE_BYTES);
                        const uint32_t fbl = rank == 0 ? fb : mapa_rank(fb, 0);
                        const uint32_t dst = smem_u32(base + s * TC_STAGE_BYTES);
                        tma_load_4d_pair(dst, &tmA, 0, rowA, kb, q, fbl, pol_stream);
                        tma_load_4d_pair(dst + TC_OPND_BYTES, &tmB, 0, rowB, kb, q, fbl, pol_keep);
                    }
                }
            }
            // drain: the last MMA commit of every stage has arrived here before the CTA may exit
            for (int k = 0; k < TC_STAGES && k < it; ++k) {
                const int j = it - 1 - k;
                mbar_wait(empty + (j % TC_STAGES), (uint32_t)(j / TC_STAGES) & 1u);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (leader CTA)
        if (rank == 0 && lane == 0) {
            const uint32_t idesc = (1u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
            int it = 0, qi = 0;
            for (int item = cl; item < nitems; item += ncl) {
                const int qgi = item % nqg;
                const int q_begin = qgi * qg, q_end = min(N + 1, q_begin + qg);
                for (int q = q_begin; q < q_end; ++q, ++qi) {
                    const int acc = qi & 1;
                    mbar_wait(tempty + acc, (((uint32_t)qi >> 1) & 1u) ^ 1u);
                    tc_fence_after();
                    const uint32_t dt = tmem + (uint32_t)(acc * 256);
                    for (int kb = 0; kb < KB; ++kb, ++it) {
                        const int s = it % TC_STAGES;
                        mbar_wait(full + s, (uint32_t)(it / TC_STAGES) & 1u);
                        tc_fence_after();
                        const uint32_t sa = smem_u32(base + s * TC_STAGE_BYTES);
                        const uint64_t a_hi = sw128_desc(sa), a_lo = a_hi + 4;          // lo: K half at +64 B
                        const uint64_t b_hi = sw128_desc(sa + TC_OPND_BYTES), b_lo = b_hi + 4;
                        const int nst = min(2, steps - 2 * kb);
                        for (int k = 0; k < nst; ++k) {
                            const uint64_t o = (uint64_t)(2 * k);          // +32 B per K=16 fp16 step
                            tc_mma_f16_pair(dt, a_hi + o, b_hi + o, idesc, (kb | k) ? 1u : 0u);
                            if (!fast) {                                   // fast path (<= 2e-3): hi x hi only
                                tc_mma_f16_pair(dt, a_hi + o, b_lo + o, idesc, 1u);
                                tc_mma_f16_pair(dt, a_lo + o, b_hi + o, idesc, 1u);
                            }
                        }
                        tc_commit_pair(empty + s);       // both CTAs' stage s free once these complete
                    }
                    tc_commit_pair(tfull + acc);          // accumulator ready in both CTAs
                }
            }
        }
    } else {
        // ---------------- epilogue (both CTAs)
        const int quad = warp & 3;                 // TMEM lane quadrant this warp may access
        const int row = quad * 32 + lane;
        const bool re_rows = row < 64;
        // planes of Nout rows; Nout > N is the zero-padded (finer-gamma) spectrum of rsvd_align_*_fine:
        // U_N / 2 goes to row N of the re plane (the split Nyquist bin, reading G4)
        float *const plane_re = Upk, *const plane_im = Upk + (int64_t)Nout * Mc * Tc;
        const bool padded = Nout > N;
        const uint32_t te0 = rank == 0 ? smem_u32(tempty) : mapa_rank(smem_u32(tempty), 0);
        // PDL: operands are read-only, so TMA + MMA above may overlap the previous kernel's tail; the
        // workspace is only written after that kernel (Step 3 of the previous chunk) has finished.
        asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef RSVD_TRACE
        if (warp == 2 && lane == 0) trs[1] = trace_now();
        bool tr_first = true;
#endif
        uint64_t pol_ws = 0;
#if RSVD_WS_POLICY == 1
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_ws));
#elif RSVD_WS_POLICY == 2
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_ws));
#endif
        int qi = 0;
        for (int item = cl; item < nitems; item += ncl) {
            const int tile = item / nqg, qgi = item - tile * nqg;
            const int mt_l = tile / ntl, nt_l = tile - mt_l * ntl;
            const int q_begin = qgi * qg, q_end = min(N + 1, q_begin + qg);
            const int64_t ml = (int64_t)mt_l * TC_PIMG + rank * 64 + (row & 63);
            for (int q = q_begin; q < q_end; ++q, ++qi) {
                const int acc = qi & 1;
                mbar_wait(tfull + acc, ((uint32_t)qi >> 1) & 1u);
                tc_fence_after();
#ifdef RSVD_TRACE
                if (tr_first && warp == 2 && lane == 0) trs[2] = trace_now();
                tr_first = false;
#endif
                // q = 0: Re U_0 -> re plane slot 0; q = N: Re U_N -> im plane slot 0; Im rows of both dropped
                const bool store = (q != 0 && q != N) || re_rows;
                const bool nyq_packed = q == N && !padded;
                float *plane = nyq_packed ? plane_im : ((q == 0 || q == N || re_rows) ? plane_re : plane_im);
                const int n = nyq_packed ? 0 : q;
                const float qs = (q == N && padded) ? 0.5f : 1.f;
                // workspace [n][t][m]: the 32 lanes hold 32 consecutive images -> each store is one 128-B line
                float *dst = plane + ((int64_t)n * Tc + (int64_t)nt_l * TC_TT) * Mc + ml;
                const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * 256);
                // 64-column batches, the next batch's TMEM loads in flight while this one is stored
                uint32_t v[2][2][32];
                tmem_ld32(tbase, v[0][0]);
                tmem_ld32(tbase + 32, v[0][1]);
                tmem_wait_ld();
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int cur = b & 1;
                    if (b < 3) {
                        tmem_ld32(tbase + (uint32_t)(64 * b + 64), v[cur ^ 1][0]);
                        tmem_ld32(tbase + (uint32_t)(64 * b + 96), v[cur ^ 1][1]);
                    }
                    if constexpr (fmt == 0) {
                        if (store) {
#pragma unroll
                        for (int h = 0; h < 2; ++h)
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                st_spectrum(dst + (int64_t)(64 * b + 32 * h + i) * Mc, qs * __uint_as_float(v[cur][h][i]), pol_ws);
                        }
                    } else if (fmt == 2 && store) {
                        // split hi/lo fp16 (same 4 B per value): hi = fp16(x), lo = fp16(x - hi), x = v 2^-20
                        const bool imv = (nyq_packed || (q != 0 && q != N && !re_rows));
                        __half *sp = reinterpret_cast<__half *>(Upk) +
                                     (((int64_t)n * 4 + (imv ? 1 : 0)) * Tc + (int64_t)nt_l * TC_TT + 64 * b) * Mc + ml;
                        const int64_t lo_off = (int64_t)2 * Tc * Mc;
#pragma unroll
                        for (int h = 0; h < 2; ++h)
#pragma unroll
                            for (int i = 0; i < 32; ++i) {
                                const float x = RSVD_SPLIT_SCALE * __uint_as_float(v[cur][h][i]);
                                const __half hi = __float2half_rn(x);
                                const __half lo = __float2half_rn((x - __half2float(hi)) * 1024.0f);
                                __half *e = sp + (int64_t)(32 * h + i) * Mc;
                                e[0] = hi;
                                e[lo_off] = lo;
                            }
                    } else if (store) {
                        // fast path: fp16 spectrum (same [n][t][m] planes, 2 B per value), accumulators
                        // scaled by FAST_SPEC_SCALE = 2^-20 into fp16 range; the transform scales back
                        __half *hdst = reinterpret_cast<__half *>(Upk) + (dst - Upk);
#pragma unroll
                        for (int h = 0; h < 2; ++h)
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                hdst[(int64_t)(64 * b + 32 * h + i) * Mc] =
                                    __float2half_rn(qs * (1.0f / 1048576.0f) * __uint_as_float(v[cur][h][i]));
                    }
                    tmem_wait_ld();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(te0 + (uint32_t)(acc * 8));
            }
        }
    }
    tc_fence_before();
    cluster_sync_relaxed();
#ifdef RSVD_TRACE
    if (tid == 0) {
        TraceRec r;
        r.t0 = trs[0]; r.t1 = trs[1]; r.t2 = trs[2]; r.t3 = trace_now();
        r.kind_blk = (0u << 24) | blockIdx.x;
        r.key = ((unsigned)mt0 << 16) | (unsigned)nt0;
        trace_put(r);
    }
#endif
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// ------------------------------------------------------------------ TC operand emission (Step 1 tail)
// Position of coefficient q in a principal ring's row of `at` after the in-place DFT: the lane that
// produced q = k1 + E b writes E consecutive coefficients, so the k1 slot is XOR-permuted by b
// within each group of E (E = Q/32) -- lanes of one store then hit distinct banks.
__device__ __forceinline__ int at_pos(int q, int E) { return (q & ~(E - 1)) | ((q ^ (q / E)) & (E - 1)); }

// From the coefficients at[h][q] (smem, [H][Q]) of one row: the exact power-of-two row scale s
// (max |Re|,|Im| of the stored values times s in [2^13, 2^14)), then the hi/lo fp16 operand rows.
// block-wide max of one float per thread (exact, order-independent)
__device__ float block_max(float mx, float *red) {
#pragma unroll
    for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
        for (int off = 16; off; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
        if (threadIdx.x == 0) red[32] = v;
    }
    __syncthreads();
    return red[32];
}
// exact power-of-two row scale that maps a bound m on the row's |coefficients| into [2^13, 2^14)
__device__ __forceinline__ float scale_for(float m) {
    if (!(m > 0.f) || !isfinite(m)) return 1.f;
    return ldexpf(1.f, 13 - ilogbf(m));
}

// the same split for a pair, packed: (hi.x, hi.y) and (lo.x, lo.y) as half2 bit patterns
__device__ __forceinline__ void split_h2(float2 v, uint32_t &hi, uint32_t &lo) {
    const __half2 h = __float22half2_rn(v);
    const float2 hf = __half22float2(h);
    const __half2 l = __float22half2_rn(make_float2(v.x - hf.x, v.y - hf.y));
    hi = *reinterpret_cast<const uint32_t *>(&h);
    lo = *reinterpret_cast<const uint32_t *>(&l);
}

// Operand rows of this CTA's quarters (4 complex k-slots = 16 B of hi and 16 B of lo): global quarter
// gq of the row's 4*KB quarters holds alpha/beta slots j = 4 gq .. 4 gq + 3 (j < H: coefficient h = j,
// H <= j < 2H: mirror h = j - H, j >= 2H: zero padding).  at holds principal rings h0 .. h0 + hg - 1.
struct QuarterSet { int a0, a1, b0, b1, c0, c1; };        // up to three ranges [x0, x1) of global quarters
__device__ void emit_tc_rows(const float2 *at, int h0, int H, int Q, int KB, int side, int64_t row,
                             int64_t op_rows, float s, QuarterSet qs, __half *__restrict__ ops,
                             int t0 = -1, int nt = 0) {
    const int N = Q / 2;
    const int E = Q / 32;
    const int na = qs.a1 - qs.a0, nb = qs.b1 - qs.b0, nc = qs.c1 - qs.c0, nq = na + nb + nc;
    const int total = (N + 1) * nq;                       // (q, owned quarter)
    if (t0 < 0) { t0 = threadIdx.x; nt = blockDim.x; }
    for (int idx = t0; idx < total; idx += nt) {
        const int lq = idx % nq;
        const int q = idx / nq;
        const int gq = lq < na ? qs.a0 + lq : (lq < na + nb ? qs.b0 + lq - na : qs.c0 + lq - na - nb);
        const int qu = gq & 3, kb = gq >> 2;
        float2 c[4];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int j = gq * 4 + jj;                    // complex index of alpha/beta
            float2 a = make_float2(0.f, 0.f);
            if (j < H) {
                a = at[(j - h0) * Q + at_pos(q, E)];
                if (side == RSVD_SIDE_IMAGE) a = c_conj(a);
            } else if (j < 2 * H) {
                a = at[(j - H - h0) * Q + at_pos((Q - q) & (Q - 1), E)];
                if (side == RSVD_SIDE_TEMPLATE) a = c_conj(a);
            }
            c[jj] = make_float2(a.x * s, a.y * s);
        }
        const int64_t sub = (int64_t)q * KB + kb;         // (q, kb): rows of 64 fp16 (hi | lo)
        if (side == RSVD_SIDE_TEMPLATE) {
            uint4 hi, lo;
            split_h2(c[0], hi.x, lo.x); split_h2(c[1], hi.y, lo.y); split_h2(c[2], hi.z, lo.z); split_h2(c[3], hi.w, lo.w);
            *reinterpret_cast<uint4 *>(ops + (sub * op_rows + row) * 64 + qu * 8) = hi;
            *reinterpret_cast<uint4 *>(ops + (sub * op_rows + row) * 64 + 32 + qu * 8) = lo;
        } else {
            const int64_t rre = (row / 64) * 128 + row % 64, rim = rre + 64;
            uint4 rh, rl, ih, il;                         // A_re = (Re a, -Im a), A_im = (Im a, Re a)
            split_h2(make_float2(c[0].x, -c[0].y), rh.x, rl.x); split_h2(make_float2(c[0].y, c[0].x), ih.x, il.x);
            split_h2(make_float2(c[1].x, -c[1].y), rh.y, rl.y); split_h2(make_float2(c[1].y, c[1].x), ih.y, il.y);
            split_h2(make_float2(c[2].x, -c[2].y), rh.z, rl.z); split_h2(make_float2(c[2].y, c[2].x), ih.z, il.z);
            split_h2(make_float2(c[3].x, -c[3].y), rh.w, rl.w); split_h2(make_float2(c[3].y, c[3].x), ih.w, il.w);
            *reinterpret_cast<uint4 *>(ops + (sub * op_rows + rre) * 64 + qu * 8) = rh;
            *reinterpret_cast<uint4 *>(ops + (sub * op_rows + rre) * 64 + 32 + qu * 8) = rl;
            *reinterpret_cast<uint4 *>(ops + (sub * op_rows + rim) * 64 + qu * 8) = ih;
            *reinterpret_cast<uint4 *>(ops + (sub * op_rows + rim) * 64 + 32 + qu * 8) = il;
        }
    }
}

// Step 1 for the TC layout: rings -> principal rings (psi-space projection with the fp64 basis rounded
// to fp32) -> length-Q DFT -> row scale -> fp16 hi/lo operand rows.  Normally one CTA per row holds
// the row's whole [H][Q] coefficient block in shared memory and projects all H rings in one pass over
// the rings.  When that block does not fit (large H x Q) and 4 | H, the row is split over
// ceil(H / CPT_HG) CTAs, one per group of CPT_HG principal rings (adjacent in the grid, so the row's
// rings come from HBM once and from L2 for the other groups).  Every CTA of a row derives the same row
// scale without communicating, from the bound |coefficient| <= sqrt(2) max|Re, Im a| * max_h
// sum_r |U'[r][h]|.  The rings stream through shared memory in slabs of whole rings with
// double-buffered bulk copies (cp.async.bulk + mbarrier), so loads run ahead of the projection FMAs.
constexpr int CPT_HG = 8;                                  // principal rings per CTA when split
template <int Q, bool SPLIT>
struct CptCfg {
    static constexpr int THREADS = (SPLIT || Q < 512) ? 256 : 512;
    static constexpr int MIN_BLOCKS = SPLIT ? (Q >= 1024 ? 2 : 3) : (Q <= 256 ? 2 : 1);
};

template <int LOGQ, int HC, bool SPLIT>
__global__ void __launch_bounds__(CptCfg<(1 << LOGQ), SPLIT>::THREADS, CptCfg<(1 << LOGQ), SPLIT>::MIN_BLOCKS)
compress_tc_kernel(
    const float2 *__restrict__ rings, int64_t n, int R, const double *__restrict__ w, const double *__restrict__ U,
    int H, int side, int KB, int64_t op_rows, int slab_rings, int ngroups, __half *__restrict__ ops,
    float *__restrict__ scales, const double *__restrict__ kr, const double *__restrict__ shifts, int S) {
    constexpr int Q = 1 << LOGQ;
    constexpr int L = 32;
    constexpr int E = Q / L;
    constexpr int CPT_THREADS = CptCfg<Q, SPLIT>::THREADS;
    constexpr int JPT = Q >= CPT_THREADS ? Q / CPT_THREADS : 1;      // angular samples per thread
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int group = (int)(blockIdx.x % ngroups);
    const int64_t row = blockIdx.x / ngroups;                         // output row = base * S + shift
    const int gh0 = ngroups > 1 ? group * CPT_HG : 0;                 // this CTA's principal rings
    const int ghc = ngroups > 1 ? min(CPT_HG, H - gh0) : H;
    const int hmax = ngroups > 1 ? CPT_HG : H;
    const int slab_f2 = slab_rings * Q;
    float2 *slab = reinterpret_cast<float2 *>(smem_raw);              // [2][slab_rings][Q]
    double *sw = reinterpret_cast<double *>(slab + 2 * slab_f2);     // [R] sqrt(w_r) (R rounded to even)
    float2 *tw = reinterpret_cast<float2 *>(sw + (R + 1) / 2 * 2);    // [E][L] (16-B aligned: up is read as float4)
    float2 *at = tw + E * L;                                          // [hmax][Q]
    float *up = reinterpret_cast<float *>(at + (size_t)hmax * Q);     // [R][HC]
    float *red = up + (size_t)R * HC;                                 // [33]
    uint64_t *bar = reinterpret_cast<uint64_t *>(red + 34);           // [2] (8-byte aligned: 34 floats)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float2 *ring = rings + (row / S) * (int64_t)R * Q;
    const int nslab = (R + slab_rings - 1) / slab_rings;
    // row f2: translated copy s of the base row, a[r][j] exp(-i k_r (dx cos psi_j + dy sin psi_j))
    // (the Fourier shift theorem with the convention of PAPER.md:80; reading G15)
    float uj[JPT];
    if (shifts) {
        const int sh = (int)(row % S);
        const double dx = shifts[2 * sh], dy = shifts[2 * sh + 1];
#pragma unroll
        for (int jj = 0; jj < JPT; ++jj) {
            double sn, cs;
            sincospi(2.0 * (double)(tid + CPT_THREADS * jj) / (double)Q, &sn, &cs);
            uj[jj] = (float)(dx * cs + dy * sn);
        }
    }
    auto issue = [&](int s, int buf) {                                // thread 0
        const int r0 = s * slab_rings, nr = min(slab_rings, R - r0);
        const uint32_t bytes = (uint32_t)nr * Q * 8u;
        const uint32_t b = smem_u32(bar + buf);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(slab + (size_t)buf * slab_f2)),
                     "l"(ring + (int64_t)r0 * Q), "r"(bytes), "r"(b)
                     : "memory");
    };
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + 1)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < E * L; i += CPT_THREADS) tw[i] = twiddle_N(i % L, i / L, Q);
    for (int r = tid; r < R; r += CPT_THREADS) sw[r] = sqrt(w[r]);
    float2 stw[clog2(L)];
    lane_stage_twiddles<L>(lane, stw);
    const double invQ = 1.0 / (double)Q;
    __syncthreads();
    // c = max_h sum_r |U[r][h]| sqrt(w_r) / Q, every h, fixed summation order (identical in every group)
    float cmax = 0.f;
    for (int h = warp; h < H; h += CPT_THREADS / 32) {
        double c = 0.0;
        for (int r = lane; r < R; r += 32) c += fabs(U[(int64_t)r * H + h]) * sw[r];
#pragma unroll
        for (int off = 16; off; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
        cmax = fmaxf(cmax, (float)(c * invQ));
    }
    float amax = 0.f;                                                 // max |Re|, |Im| of the row's samples
    int ks = 0;                                                       // slabs consumed so far (all passes)
    for (int hp = 0; hp < ghc; hp += HC) {
        const int hc = min(HC, ghc - hp);
        __syncthreads();
        for (int i = tid; i < R * HC; i += CPT_THREADS) {
            const int r = i / HC, hh = i % HC;
            up[i] = (hh < hc) ? (float)(U[(int64_t)r * H + gh0 + hp + hh] * sw[r] * invQ) : 0.f;
        }
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(0, ks & 1);
            if (nslab > 1) issue(1, (ks + 1) & 1);
        }
        __syncthreads();
        float2 acc[JPT][HC];
#pragma unroll
        for (int jj = 0; jj < JPT; ++jj)
#pragma unroll
            for (int hh = 0; hh < HC; ++hh) acc[jj][hh] = make_float2(0.f, 0.f);
        for (int s = 0; s < nslab; ++s, ++ks) {
            const int buf = ks & 1;
            asm volatile(
                "{\n\t.reg .pred p;\n"
                "CPT_WAIT:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                "@!p bra CPT_WAIT;\n\t}" ::"r"(smem_u32(bar + buf)),
                "r"((uint32_t)(ks >> 1) & 1u)
                : "memory");
            const float2 *sl = slab + (size_t)buf * slab_f2;
            const int r0 = s * slab_rings, nr = min(slab_rings, R - r0);
            if (tid < Q) {
#pragma unroll 2
                for (int rr = 0; rr < nr; ++rr) {
                    const float4 *u4 = reinterpret_cast<const float4 *>(up + (r0 + rr) * HC);
                    float2 a[JPT];
#pragma unroll
                    for (int jj = 0; jj < JPT; ++jj) {
                        a[jj] = sl[rr * Q + tid + CPT_THREADS * jj];
                        amax = fmaxf(amax, fmaxf(fabsf(a[jj].x), fabsf(a[jj].y)));
                    }
                    if (shifts) {
                        const float k = (float)kr[r0 + rr];
#pragma unroll
                        for (int jj = 0; jj < JPT; ++jj) {
                            float sn, cs;
                            __sincosf(-k * uj[jj], &sn, &cs);      // |arg| <~ 2 rad: abs error ~4e-7
                            a[jj] = make_float2(a[jj].x * cs - a[jj].y * sn, a[jj].x * sn + a[jj].y * cs);
                        }
                    }
#pragma unroll
                    for (int g = 0; g < HC / 4; ++g) {
                        const float4 u = u4[g];
#pragma unroll
                        for (int jj = 0; jj < JPT; ++jj) {
                            acc[jj][4 * g + 0] = __ffma2_rn(a[jj], make_float2(u.x, u.x), acc[jj][4 * g + 0]);
                            acc[jj][4 * g + 1] = __ffma2_rn(a[jj], make_float2(u.y, u.y), acc[jj][4 * g + 1]);
                            acc[jj][4 * g + 2] = __ffma2_rn(a[jj], make_float2(u.z, u.z), acc[jj][4 * g + 2]);
                            acc[jj][4 * g + 3] = __ffma2_rn(a[jj], make_float2(u.w, u.w), acc[jj][4 * g + 3]);
                        }
                    }
                }
            }
            __syncthreads();                                          // slab buffer free
            if (tid == 0 && s + 2 < nslab) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(s + 2, buf);
            }
        }
        if (tid < Q) {
#pragma unroll
            for (int jj = 0; jj < JPT; ++jj)
#pragma unroll
                for (int hh = 0; hh < HC; ++hh)
                    if (hh < hc) at[(hp + hh) * Q + tid + CPT_THREADS * jj] = acc[jj][hh];
        }
    }
    __syncthreads();
    // in-place length-Q forward DFT of each principal ring, natural order
    for (int h = warp; h < ghc; h += CPT_THREADS / 32) {
        float2 v[E];
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = at[h * Q + lane + L * e];
        fft_dist<E, L>(v, lane, tw, stw);
        __syncwarp();
        const int b = (int)(__brev((unsigned)lane) >> 27);
#pragma unroll
        for (int k1 = 0; k1 < E; ++k1) at[h * Q + at_pos(k1 + E * b, E)] = v[brev(k1, clog2(E))];
    }
    // |A_q[h]| <= sum_r |U'[r][h]| sum_j |a[r][j]| <= sqrt(2) amax * Q cmax (U' holds the 1/Q)
    cmax = block_max(cmax, red);                                      // block_max syncs: at[] complete
    amax = block_max(amax, red);
    const float s = scale_for(1.41421356f * (float)Q * amax * cmax * 1.0000002f);
    if (tid == 0 && group == 0) scales[row] = s;
    QuarterSet qs;
    if (ngroups > 1) {                                                // 4 | H: quarters never straddle groups
        qs = {gh0 / 4, (gh0 + ghc) / 4, (H + gh0) / 4, (H + gh0 + ghc) / 4, group == 0 ? H / 2 : 0,
              group == 0 ? 4 * KB : 0};
    } else {
        qs = {0, 4 * KB, 0, 0, 0, 0};
    }
    emit_tc_rows(at, gh0, H, Q, KB, side, row, op_rows, s, qs, ops);
}

// principal rings per projection pass (acc[JPT][HC] in registers; more passes re-stream the rings)
static int compress_hc(int H, bool split) {
    if (split) return CPT_HG;
    return H <= 8 ? 8 : (H <= 16 ? 16 : (H <= 24 ? 24 : 32));
}
static size_t compress_fixed_smem(int Q, int H, int R, bool split) {
    const int hmax = split ? CPT_HG : H;
    return (size_t)(R + 1) / 2 * 2 * sizeof(double) + (size_t)Q * sizeof(float2) + (size_t)hmax * Q * sizeof(float2) +
           (size_t)R * compress_hc(H, split) * sizeof(float) + 34 * 4 + 16;
}
// rings per slab: the largest of 32 / 16 / 8 KB slabs (at least one ring) that fits the budget: 200 KB
// for one CTA per row; a split row targets MIN_BLOCKS CTAs per SM (228 KB per SM, 1 KB reserved per CTA)
static int slab_rings_for(int Q, int H, int R, bool split) {
    const size_t ring = (size_t)Q * sizeof(float2);
    const size_t budget = split ? (Q >= 1024 ? 112 : 74) * 1024 : 200 * 1024;
    for (size_t slab : {32768u, 16384u, 8192u}) {
        const size_t sb = std::max(slab, ring);
        if (compress_fixed_smem(Q, H, R, split) + 2 * sb <= budget) return (int)std::min<size_t>(sb / ring, (size_t)R);
    }
    return 0;
}
// CTAs per row: 1 when the row's [H][Q] block fits, else groups of CPT_HG rings (needs 4 | H), else 0
static int compress_groups(int Q, int H, int R) {
    if (slab_rings_for(Q, H, R, false) > 0) return 1;
    if (H % 4 == 0 && slab_rings_for(Q, H, R, true) > 0) return (H + CPT_HG - 1) / CPT_HG;
    return 0;
}
static int compress_slab_rings(int Q, int H, int R) {
    const int ng = compress_groups(Q, H, R);
    return ng ? slab_rings_for(Q, H, R, ng > 1) : 0;
}
size_t compress_tc_smem(int Q, int H, int R) {
    const int sr = compress_slab_rings(Q, H, R);
    return compress_fixed_smem(Q, H, R, compress_groups(Q, H, R) > 1) + 2 * (size_t)std::max(sr, 1) * Q * sizeof(float2);
}

// TC layout needs a CTA's [hmax][Q] coefficient block in shared memory (R <= 256).
bool tc_supported(int Q, int H) { return compress_slab_rings(Q, H, 256) > 0; }

static int g_path = -1;
int resolve_path(int Q, int H) {
    if (g_path < 0) {
        const char *e = getenv("RSVD_PATH");
        g_path = PATH_AUTO;
        if (e && !strcmp(e, "simt")) g_path = PATH_SIMT;
        if (e && !strcmp(e, "tc")) g_path = PATH_TC;
    }
    if (g_path == PATH_SIMT) return PATH_SIMT;
    return tc_supported(Q, H) ? PATH_TC : PATH_SIMT;
}
void set_path(int p) { g_path = (p == PATH_SIMT || p == PATH_TC) ? p : PATH_AUTO; }

static std::atomic<int> g_precision{-1};
int resolve_precision() {
    int p = g_precision.load(std::memory_order_relaxed);
    if (p < 0) {
        const char *e = getenv("RSVD_PRECISION");
        p = (e && !strcmp(e, "fast")) ? PREC_FAST : PREC_FP32;
        g_precision.store(p, std::memory_order_relaxed);
    }
    return p;
}

template <int LOGQ, int HC, bool SPLIT>
static cudaError_t launch_compress_tc_qh(const float2 *rings, int64_t n, int R, const double *w, const double *U, int H,
                                         int side, void *blocks, const double *kr, const double *shifts, int S,
                                         cudaStream_t s) {
    const int Q = 1 << LOGQ;
    const int sr = compress_slab_rings(Q, H, R);
    const int ng = compress_groups(Q, H, R);
    if (sr < 1 || ng < 1 || n * ng > 0x7fffffffLL) return cudaErrorInvalidValue;
    const size_t smem = compress_tc_smem(Q, H, R);
    cudaError_t e = cudaFuncSetAttribute(compress_tc_kernel<LOGQ, HC, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    float *scales = const_cast<float *>(tc_scales(blocks, n, Q, H, side));
    compress_tc_kernel<LOGQ, HC, SPLIT><<<(unsigned)(n * ng), CptCfg<Q, SPLIT>::THREADS, smem, s>>>(
        rings, n, R, w, U, H, side, tc_kb(H), tc_op_rows(n, side), sr, ng, reinterpret_cast<__half *>(blocks), scales,
        kr, shifts, S);
    return cudaGetLastError();
}
template <int LOGQ>
static cudaError_t launch_compress_tc_q(const float2 *rings, int64_t n, int R, const double *w, const double *U, int H,
                                        int side, void *blocks, const double *kr, const double *shifts, int S,
                                        cudaStream_t s) {
    if (compress_groups(1 << LOGQ, H, R) > 1)
        return launch_compress_tc_qh<LOGQ, CPT_HG, true>(rings, n, R, w, U, H, side, blocks, kr, shifts, S, s);
    switch (compress_hc(H, false)) {
        case 8: return launch_compress_tc_qh<LOGQ, 8, false>(rings, n, R, w, U, H, side, blocks, kr, shifts, S, s);
        case 16: return launch_compress_tc_qh<LOGQ, 16, false>(rings, n, R, w, U, H, side, blocks, kr, shifts, S, s);
        case 24: return launch_compress_tc_qh<LOGQ, 24, false>(rings, n, R, w, U, H, side, blocks, kr, shifts, S, s);
        default: return launch_compress_tc_qh<LOGQ, 32, false>(rings, n, R, w, U, H, side, blocks, kr, shifts, S, s);
    }
}

#include "rsvd_compress_mma.cuh"

cudaError_t launch_compress_tc(const float2 *rings, int64_t n, int R, int Q, const double *w, const double *U, int H,
                               int side, float *blocks, const double *kr, const double *shifts, int S, cudaStream_t s) {
    if (!shifts) {
        bool launched = false;
        const cudaError_t e = launch_compress_mma(rings, n, R, Q, w, U, H, side, blocks, s, &launched);
        if (e != cudaSuccess || launched) return e;
    }
    switch (ilog2(Q)) {
        case 5: return launch_compress_tc_q<5>(rings, n, R, w, U, H, side, blocks, kr, shifts, S, s);
        case 6: return launch_compress_tc_q<6>(rings, n, R, w, U, H, side, blocks, kr, shifts, S, s);
        case 7: return launch_compress_tc_q<7>(rings, n, R, w, U, H, side, blocks, kr, shifts, S, s);
        case 8: return launch_compress_tc_q<8>(rings, n, R, w, U, H, side, blocks, kr, shifts, S, s);
        case 9: return launch_compress_tc_q<9>(rings, n, R, w, U, H, side, blocks, kr, shifts, S, s);
        default: return launch_compress_tc_q<10>(rings, n, R, w, U, H, side, blocks, kr, shifts, S, s);
    }
}

// canonical coefficients from the TC operand rows (hi + lo) / s, test / debug path
__global__ void unpack_tc_kernel(const __half *__restrict__ ops, const float *__restrict__ scales, int64_t n, int Q,
                                 int H, int side, int KB, int64_t op_rows, float2 *__restrict__ coeffs) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * (int64_t)Q * H) return;
    const int h = (int)(idx % H);
    const int q = (int)((idx / H) % Q);
    const int64_t row = idx / ((int64_t)H * Q);
    const int N = Q / 2;
    const int qq = q <= N ? q : Q - q;
    const int j = q <= N ? h : H + h;
    const int kb = j / 16, e = 2 * (j % 16);
    const int64_t r = side == RSVD_SIDE_TEMPLATE ? row : (row / 64) * 128 + row % 64;
    const int64_t sub = (int64_t)qq * KB + kb;
    const __half *hi = ops + (sub * op_rows + r) * 64 + e;
    const __half *lo = hi + 32;
    const float inv = 1.f / scales[row];
    float x = (__half2float(hi[0]) + __half2float(lo[0])) * inv;
    float y = (__half2float(hi[1]) + __half2float(lo[1])) * inv;
    float2 v = side == RSVD_SIDE_TEMPLATE ? make_float2(x, y) : make_float2(x, -y);   // alpha / beta_j
    if (q <= N) { if (side == RSVD_SIDE_IMAGE) v = c_conj(v); }
    else { if (side == RSVD_SIDE_TEMPLATE) v = c_conj(v); }
    coeffs[idx] = v;
}

cudaError_t launch_unpack_tc(const float *blocks, int64_t n, int Q, int H, int side, float2 *coeffs, cudaStream_t s) {
    const int64_t total = n * (int64_t)Q * H;
    unpack_tc_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(
        reinterpret_cast<const __half *>(blocks), tc_scales(blocks, n, Q, H, side), n, Q, H, side, tc_kb(H),
        tc_op_rows(n, side), coeffs);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ tensor maps + launch
// 4-D map of one side's operand rows: (64 fp16 = hi | lo, row, kb, q), box (64, box_rows, 1, 1), SWIZZLE_128B.
cudaError_t make_tc_operand_tmap(CUtensorMap *tm, const void *blocks, int64_t rows, int Q, int H, int side,
                                 int box_rows) {
    PFN_encodeTiled_tc enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    const int64_t op_rows = tc_op_rows(rows, side);
    const int KB = tc_kb(H);
    const cuuint64_t dims[4] = {64, (cuuint64_t)op_rows, (cuuint64_t)KB, (cuuint64_t)(Q / 2 + 1)};
    const cuuint64_t strides[3] = {128, (cuuint64_t)op_rows * 128, (cuuint64_t)op_rows * 128 * KB};
    const cuuint32_t box[4] = {64, (cuuint32_t)box_rows, 1, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void *>(blocks), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, (CUtensorMapL2promotion)RSVD_TC_L2PROMO,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// One chunk: images [m0, m0 + mc) (multiples of 128), templates [t0, t0 + tc) (multiples of 256).
cudaError_t launch_contract_tc(const CUtensorMap &tmA, const CUtensorMap &tmB, int H, int N, int Nout, int64_t m0,
                               int64_t t0, int64_t mc, int64_t tc, int64_t Mc, int64_t Tc, float *Upk, int nsms,
                               bool operands_fresh, int fmt, cudaStream_t s) {
    static std::atomic<uint64_t> attr0{0}, attr1{0}, attr2{0};
    auto kern = fmt == 1 ? contract_tc_kernel<1> : (fmt == 2 ? contract_tc_kernel<2> : contract_tc_kernel<0>);
    {
        const cudaError_t e = smem_attr_once((const void *)kern, (int)TC_SMEM, fmt == 1 ? attr1 : (fmt == 2 ? attr2 : attr0));
        if (e != cudaSuccess) return e;
    }
    const int mtl = (int)(mc / TC_PIMG), ntl = (int)(tc / TC_TT);
    const int ntiles = mtl * ntl;
    // q-groups per tile: as many as fit the CTA pairs of one wave (floor, so that every pair gets at
    // most one (tile, q-group) item -- a ceiling here gave a few pairs two items and doubled the launch)
    const int target = std::max(1, nsms / 2);
    int nqg = std::max(1, target / std::max(1, ntiles));
    nqg = std::min(nqg, N + 1);
    const int qg = (N + 1 + nqg - 1) / nqg;
    nqg = (N + 1 + qg - 1) / qg;
    const int nitems = ntiles * nqg;
    const int ncl = std::min(nitems, target);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * ncl));
    cfg.blockDim = dim3(TC_THREADS);
    cfg.dynamicSmemBytes = TC_SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tmA, tmB, tc_steps(H), tc_kb(H), N, mtl, ntl,
                                       (int)(m0 / TC_PIMG), (int)(t0 / TC_TT), qg, nqg, nitems, Mc, Tc, Upk, Nout,
                                       operands_fresh ? 1 : 0);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace rsvd

extern "C" void rsvd_set_path(int32_t path) { rsvd::set_path(path); }
extern "C" void rsvd_set_precision(int32_t precision) {
    rsvd::g_precision.store(precision == rsvd::PREC_FAST ? rsvd::PREC_FAST : rsvd::PREC_FP32);
}
extern "C" int32_t rsvd_precision(void) { return rsvd::resolve_precision(); }
extern "C" void rsvd_set_compress_mma(int32_t mode) {
    rsvd::g_compress_mma.store(mode < 0 || mode > 2 ? 1 : mode, std::memory_order_relaxed);
}
extern "C" int32_t rsvd_compress_mma_mode(void) { return rsvd::compress_mma_mode(); }
extern "C" int32_t rsvd_path_for(int32_t Q, int32_t H) { return rsvd::resolve_path(Q, H); }
