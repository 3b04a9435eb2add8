// rsvd_tc.cu -- tensor-core path of Step 2 (the q-batched complex contraction) on
// sm_100a: tcgen05.mma kind::tf32 with 3xTF32 error compensation, plus the compact block layout it
// consumes (written by compress) and the path selection.
//
// Real embedding of U_q[m,t] = sum_j alpha[q][j][m] beta[q][j][t] (alpha/beta: rsvd_compress.cu):
// two A rows per image and one B row per template,
//   A_re[m] = (Re a_j, -Im a_j)_j ,  A_im[m] = (Im a_j, Re a_j)_j ,  B[t] = (Re b_j, Im b_j)_j
//   D[m][t] = A_re . B = Re U ,  D[64 + m][t] = A_im . B = Im U.
// Each fp32 operand x = hi + lo (both TF32-rounded); D = Ahi Bhi + Ahi Blo + Alo Bhi recovers ~fp32
// accuracy (the dropped Alo Blo term is ~2^-22 relative).
//
// Block layout (compact TC layout; same bytes as the SIMT layout): K-major rows of interleaved
// complex fp32, 16 complex (128 B) per k-block row, pre-swizzled the way UMMA SWIZZLE_128B expects
// (16-byte chunk c of row r stored at chunk c ^ (r & 7)):
//   images    A[q][mtile][kb][64 rows][32 floats]    (mtile = 64 images, 8 KB per sub-tile)
//   templates B[q][ttile][kb][256 rows][32 floats]   (ttile = 256 templates, 32 KB per sub-tile)
// q = 0..N (N = Q/2), kb < KB = ceil(2H/16).  The in-shared-memory expansion to (Re, Im) rows and
// hi/lo parts preserves the position of every 16-byte chunk (64 + r = r mod 8), so producers copy
// chunk i of global to chunk i of shared memory with arithmetic only.
//
// contract_tc_kernel: one CTA per (64-image x 256-template tile, group of q), 13 warps:
//   warp 0      TMEM allocator + MMA issuer: per stage 4 k-steps x 3 tcgen05.mma (M=128, N=256, K=8)
//               into one of two 256-column TMEM accumulators; tcgen05.commit frees the smem stage /
//               signals the epilogue;
//   warps 1-4   epilogue: tcgen05.ld 32x32b of their 32 TMEM lanes; lanes 0-63 hold Re U, 64-127 Im U;
//               stores to the planar spectrum workspace (re plane | im plane), releases the accumulator;
//   warps 5-12  producers: LDG the compact (q, kb) sub-tiles (40 KB), expand to A hi/lo (2 x 16 KB) and
//               B hi/lo (2 x 32 KB) in a 2-deep shared-memory ring, fence.proxy.async, arrive.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "rsvd_common.cuh"

namespace rsvd {

constexpr int TC_THREADS = 13 * 32;
constexpr int TC_PROD_WARPS = 8;
constexpr int TC_STAGES = 2;
constexpr int TC_MT = 64;                           // images per tile
constexpr int TC_TT = 256;                          // templates per tile
constexpr uint32_t TC_A_BYTES = 128u * 128u;        // one of hi / lo: 128 rows x 128 B
constexpr uint32_t TC_B_BYTES = 256u * 128u;
constexpr uint32_t TC_STAGE_BYTES = 2 * TC_A_BYTES + 2 * TC_B_BYTES;    // 96 KB
constexpr size_t TC_SMEM = (size_t)TC_STAGES * TC_STAGE_BYTES + 1024 + 256;

int tc_kb(int H) { return (int)((2 * (int64_t)H + 15) / 16); }
int64_t tc_rows_pad_side(int64_t rows, int side) { return round_up(rows, side == RSVD_SIDE_TEMPLATE ? TC_TT : TC_MT); }
int64_t tc_rows_pad(int64_t rows) { return round_up(rows, 256); }
int64_t tc_block_bytes(int64_t rows, int Q, int H, int side) {
    return (int64_t)(Q / 2 + 1) * tc_kb(H) * tc_rows_pad_side(rows, side) * 128;
}

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFF) >> 4);          // start address
    d |= (uint64_t)1 << 16;                           // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;                 // SBO: 8-row atoms 1024 B apart
    d |= (uint64_t)1 << 46;                           // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                           // SWIZZLE_128B
    return d;
}

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_mma_tf32(uint32_t dtmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dtmem),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ float tf32_rna(float x) {       // hardware round-to-TF32 (one instruction)
    uint32_t u;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
    return __uint_as_float(u);
}
// x = hi + lo exactly (hi TF32-rounded; lo = x - hi has <= 13 significant bits and is fed as fp32:
// the tensor core keeps its top 11, an error <= 2^-22 |x|).
__device__ __forceinline__ void split4(float4 v, float4 &hi, float4 &lo) {
    hi.x = tf32_rna(v.x); lo.x = v.x - hi.x;
    hi.y = tf32_rna(v.y); lo.y = v.y - hi.y;
    hi.z = tf32_rna(v.z); lo.z = v.z - hi.z;
    hi.w = tf32_rna(v.w); lo.w = v.w - hi.w;
}

// ------------------------------------------------------------------ contraction kernel
// grid: ntiles_chunk * nqg; chunk tiles (Mc/64) x (Tc/256); item -> (tile, q-group).
// Upk planar: re plane [(n*Mc + ml)*Tc + tl], im plane at + N*Mc*Tc (floats).
__global__ void __launch_bounds__(TC_THREADS, 1) contract_tc_kernel(
    const float *__restrict__ Acmp, const float *__restrict__ Bcmp, int KB, int N, int64_t MT, int64_t NT,
    int64_t mt0, int64_t nt0, int ntl, int qg, int nqg, int64_t Mc, int64_t Tc, float *__restrict__ Upk) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char *base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint64_t *bars = reinterpret_cast<uint64_t *>(base + TC_STAGES * TC_STAGE_BYTES);
    uint64_t *full = bars, *empty = bars + TC_STAGES, *tfull = bars + 2 * TC_STAGES, *tempty = bars + 2 * TC_STAGES + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * TC_STAGES + 4);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int item = blockIdx.x;
    const int tile = item / nqg, qgi = item % nqg;
    const int mt_l = tile / ntl, nt_l = tile % ntl;
    const int64_t mt = mt0 + mt_l, nt = nt0 + nt_l;
    const int q_begin = qgi * qg;
    const int q_end = min(N + 1, q_begin + qg);
    const int nqi = max(0, q_end - q_begin);

    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < TC_STAGES; ++s) { mbar_init(full + s, TC_PROD_WARPS); mbar_init(empty + s, 1); }
            for (int a = 0; a < 2; ++a) { mbar_init(tfull + a, 1); mbar_init(tempty + a, 4); }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- MMA issuer
        if (lane == 0) {
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(256 >> 3) << 17) |
                                   ((uint32_t)(128 >> 4) << 24);
            int it = 0;
            for (int qi = 0; qi < nqi; ++qi) {
                const int acc = qi & 1;
                mbar_wait(tempty + acc, (((uint32_t)qi >> 1) & 1u) ^ 1u);
                tc_fence_after();
                const uint32_t dt = tmem + (uint32_t)(acc * 256);
                for (int kb = 0; kb < KB; ++kb, ++it) {
                    const int s = it % TC_STAGES;
                    mbar_wait(full + s, (uint32_t)(it / TC_STAGES) & 1u);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(base + s * TC_STAGE_BYTES);
                    const uint64_t a_hi = sw128_desc(sa), a_lo = sw128_desc(sa + TC_A_BYTES);
                    const uint64_t b_hi = sw128_desc(sa + 2 * TC_A_BYTES), b_lo = sw128_desc(sa + 2 * TC_A_BYTES + TC_B_BYTES);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t o = (uint64_t)(2 * k);          // +32 B per K=8 tf32 step
                        tc_mma_tf32(dt, a_hi + o, b_hi + o, idesc, (kb | k) ? 1u : 0u);
                        tc_mma_tf32(dt, a_hi + o, b_lo + o, idesc, 1u);
                        tc_mma_tf32(dt, a_lo + o, b_hi + o, idesc, 1u);
                    }
                    tc_commit(empty + s);          // stage free once these MMAs complete
                }
                tc_commit(tfull + acc);            // accumulator ready for the epilogue
            }
        }
    } else if (warp <= 4) {
        // ---------------- epilogue
        const int quad = warp & 3;                 // TMEM lane quadrant this warp may access
        const int row = quad * 32 + lane;
        const bool re_rows = row < 64;
        const int64_t ml = (int64_t)mt_l * TC_MT + (row & 63);
        float *const plane_re = Upk, *const plane_im = Upk + (int64_t)N * Mc * Tc;
        for (int qi = 0; qi < nqi; ++qi) {
            const int acc = qi & 1;
            mbar_wait(tfull + acc, ((uint32_t)qi >> 1) & 1u);
            tc_fence_after();
            const int q = q_begin + qi;
            // q = 0: Re U_0 -> re plane slot 0; q = N: Re U_N -> im plane slot 0; Im rows of both dropped
            const bool store = (q != 0 && q != N) || re_rows;
            float *plane = (q == N) ? plane_im : ((q == 0 || re_rows) ? plane_re : plane_im);
            const int n = (q == N) ? 0 : q;
            // workspace [n][t][m]: the 32 lanes hold 32 consecutive images -> each store is one 128-B line
            float *dst = plane + ((int64_t)n * Tc + (int64_t)nt_l * TC_TT) * Mc + ml;
            const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * 256);
#pragma unroll 1
            for (int c0 = 0; c0 < 256; c0 += 32) {
                uint32_t v[32];
                tmem_ld32(tbase + (uint32_t)c0, v);
                if (store) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) dst[(int64_t)(c0 + i) * Mc] = __uint_as_float(v[i]);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty + acc);
        }
    } else {
        // ---------------- producers: global compact tiles -> expanded hi/lo operand stages
        // Register ping-pong: the loads of stage it+1 are in flight while stage it waits for its smem
        // slot and is expanded, so one global-load latency is hidden per stage.
        const int pt = tid - 5 * 32;               // 0..255
        const int total = nqi * KB;
        auto load = [&](int it, float4 (&ra)[2], float4 (&rb)[8]) {
            const int q = q_begin + it / KB, kb = it % KB;
            const float4 *gA = reinterpret_cast<const float4 *>(
                Acmp + (((int64_t)q * MT + mt) * KB + kb) * (int64_t)(TC_MT * 32));
            const float4 *gB = reinterpret_cast<const float4 *>(
                Bcmp + (((int64_t)q * NT + nt) * KB + kb) * (int64_t)(TC_TT * 32));
#pragma unroll
            for (int i = 0; i < 2; ++i) ra[i] = __ldg(gA + pt + 256 * i);
#pragma unroll
            for (int i = 0; i < 8; ++i) rb[i] = __ldg(gB + pt + 256 * i);
        };
        auto expand = [&](int it, const float4 (&ra)[2], const float4 (&rb)[8]) {
            const int s = it % TC_STAGES;
            mbar_wait(empty + s, ((uint32_t)(it / TC_STAGES) & 1u) ^ 1u);
            float4 *sAhi = reinterpret_cast<float4 *>(base + s * TC_STAGE_BYTES);
            float4 *sAlo = sAhi + TC_A_BYTES / 16;
            float4 *sBhi = sAlo + TC_A_BYTES / 16;
            float4 *sBlo = sBhi + TC_B_BYTES / 16;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int idx = pt + 256 * i;               // image row idx/8, chunk position idx%8
                float4 hi, lo;
                split4(ra[i], hi, lo);
                sAhi[idx] = make_float4(hi.x, -hi.y, hi.z, -hi.w);     // A_re row: (Re a, -Im a)
                sAlo[idx] = make_float4(lo.x, -lo.y, lo.z, -lo.w);
                sAhi[512 + idx] = make_float4(hi.y, hi.x, hi.w, hi.z); // A_im row (row + 64, same chunk)
                sAlo[512 + idx] = make_float4(lo.y, lo.x, lo.w, lo.z);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int idx = pt + 256 * i;
                float4 hi, lo;
                split4(rb[i], hi, lo);
                sBhi[idx] = hi;
                sBlo[idx] = lo;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(full + s);
        };
        // L2 prefetch of the compact sub-tiles PF stages ahead (one bulk prefetch per operand), so the
        // ping-pong loads hit L2 instead of DRAM.
        constexpr int PF = 4;
        auto prefetch = [&](int it) {
            if (pt != 0 || it >= total) return;
            const int q = q_begin + it / KB, kb = it % KB;
            const float *gA = Acmp + (((int64_t)q * MT + mt) * KB + kb) * (int64_t)(TC_MT * 32);
            const float *gB = Bcmp + (((int64_t)q * NT + nt) * KB + kb) * (int64_t)(TC_TT * 32);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gA), "r"((uint32_t)(TC_MT * 128)) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gB), "r"((uint32_t)(TC_TT * 128)) : "memory");
        };
        for (int it = 1; it < PF; ++it) prefetch(it);
        float4 ra0[2], rb0[8], ra1[2], rb1[8];
        if (total > 0) load(0, ra0, rb0);
        for (int it = 0; it < total; it += 2) {
            prefetch(it + PF);
            if (it + 1 < total) load(it + 1, ra1, rb1);
            expand(it, ra0, rb0);
            if (it + 1 >= total) break;
            prefetch(it + 1 + PF);
            if (it + 2 < total) load(it + 2, ra0, rb0);
            expand(it + 1, ra1, rb1);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// ------------------------------------------------------------------ compact TC block emission (Step 1 tail)
// Emits the compact TC rows of one row (image or template) from its coefficients at[h][q] (smem,
// [H][Q]); 8 lanes write one 128-byte swizzled row (one 16-byte chunk each).
__device__ void emit_tc_rows(const float2 *at, int H, int Q, int KB, int side, int64_t row, int64_t ntiles,
                             float *__restrict__ blocks) {
    const int N = Q / 2;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int ch = tid & 7;
    const int rows_tile = side == RSVD_SIDE_TEMPLATE ? TC_TT : TC_MT;
    const int64_t tile = row / rows_tile;
    const int r = (int)(row % rows_tile);
    const int total = (N + 1) * KB;
    for (int idx = tid >> 3; idx < total; idx += nthr >> 3) {
        const int kb = idx % KB;
        const int q = idx / KB;
        float4 v;
        float2 c2[2];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const int j = kb * 16 + ch * 2 + jj;              // complex index of alpha/beta
            float2 a = make_float2(0.f, 0.f);
            if (j < H) {
                a = at[j * Q + q];
                if (side == RSVD_SIDE_IMAGE) a = c_conj(a);
            } else if (j < 2 * H) {
                a = at[(j - H) * Q + ((Q - q) & (Q - 1))];
                if (side == RSVD_SIDE_TEMPLATE) a = c_conj(a);
            }
            c2[jj] = a;
        }
        v = make_float4(c2[0].x, c2[0].y, c2[1].x, c2[1].y);
        const int64_t sub = ((int64_t)q * ntiles + tile) * KB + kb;
        *reinterpret_cast<float4 *>(blocks + (sub * rows_tile + r) * 32 + ((ch ^ (r & 7)) * 4)) = v;
    }
}

template <int LOGQ>
__global__ void __launch_bounds__(256) compress_tc_kernel(const float2 *__restrict__ rings, int64_t n, int R,
                                                          const double *__restrict__ w, const double *__restrict__ U,
                                                          int H, int side, int KB, int64_t ntiles,
                                                          float *__restrict__ blocks) {
    constexpr int Q = 1 << LOGQ;
    constexpr int L = 32;
    constexpr int E = Q / L;
    constexpr int HC = 16;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2 *tw = reinterpret_cast<float2 *>(smem_raw);       // [E][L]
    float2 *at = tw + E * L;                                 // [H][Q]
    float *up = reinterpret_cast<float *>(at + (size_t)H * Q);   // [R][HC]
    const int64_t row = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < E * L; i += 256) tw[i] = twiddle_N(i % L, i / L, Q);
    float2 stw[clog2(L)];
    lane_stage_twiddles<L>(lane, stw);
    const float2 *ring = rings + row * (int64_t)R * Q;
    const double invQ = 1.0 / (double)Q;
    for (int h0 = 0; h0 < H; h0 += HC) {
        const int hc = min(HC, H - h0);
        __syncthreads();
        for (int i = tid; i < R * HC; i += 256) {
            const int r = i / HC, hh = i % HC;
            up[i] = (hh < hc) ? (float)(U[(int64_t)r * H + h0 + hh] * sqrt(w[r]) * invQ) : 0.f;
        }
        __syncthreads();
        for (int j = tid; j < Q; j += 256) {
            float2 acc[HC];
#pragma unroll
            for (int hh = 0; hh < HC; ++hh) acc[hh] = make_float2(0.f, 0.f);
            for (int r = 0; r < R; ++r) {
                const float2 a = __ldg(ring + (int64_t)r * Q + j);
                const float4 *u4 = reinterpret_cast<const float4 *>(up + r * HC);
#pragma unroll
                for (int g = 0; g < HC / 4; ++g) {
                    const float4 u = u4[g];
                    acc[4 * g + 0].x = fmaf(u.x, a.x, acc[4 * g + 0].x); acc[4 * g + 0].y = fmaf(u.x, a.y, acc[4 * g + 0].y);
                    acc[4 * g + 1].x = fmaf(u.y, a.x, acc[4 * g + 1].x); acc[4 * g + 1].y = fmaf(u.y, a.y, acc[4 * g + 1].y);
                    acc[4 * g + 2].x = fmaf(u.z, a.x, acc[4 * g + 2].x); acc[4 * g + 2].y = fmaf(u.z, a.y, acc[4 * g + 2].y);
                    acc[4 * g + 3].x = fmaf(u.w, a.x, acc[4 * g + 3].x); acc[4 * g + 3].y = fmaf(u.w, a.y, acc[4 * g + 3].y);
                }
            }
#pragma unroll
            for (int hh = 0; hh < HC; ++hh)
                if (hh < hc) at[(h0 + hh) * Q + j] = acc[hh];
        }
    }
    __syncthreads();
    // in-place length-Q forward DFT of each principal ring, natural order
    for (int h = warp; h < H; h += 8) {
        float2 v[E];
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = at[h * Q + lane + L * e];
        fft_dist<E, L>(v, lane, tw, stw);
        __syncwarp();
        const int b = (int)(__brev((unsigned)lane) >> 27);
#pragma unroll
        for (int k1 = 0; k1 < E; ++k1) at[h * Q + k1 + E * b] = v[brev(k1, clog2(E))];
    }
    __syncthreads();
    emit_tc_rows(at, H, Q, KB, side, row, ntiles, blocks);
}

size_t compress_tc_smem(int Q, int H, int R) {
    return (size_t)Q * sizeof(float2) + (size_t)H * Q * sizeof(float2) + (size_t)R * 16 * sizeof(float);
}

// TC layout needs the whole [H][Q] coefficient block of a row in shared memory (R <= 256).
bool tc_supported(int Q, int H) { return compress_tc_smem(Q, H, 256) <= 200 * 1024; }

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

template <int LOGQ>
static cudaError_t launch_compress_tc_q(const float2 *rings, int64_t n, int R, const double *w, const double *U, int H,
                                        int side, float *blocks, cudaStream_t s) {
    const size_t smem = compress_tc_smem(1 << LOGQ, H, R);
    cudaError_t e = cudaFuncSetAttribute(compress_tc_kernel<LOGQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t ntiles = tc_rows_pad_side(n, side) / (side == RSVD_SIDE_TEMPLATE ? TC_TT : TC_MT);
    compress_tc_kernel<LOGQ><<<(unsigned)n, 256, smem, s>>>(rings, n, R, w, U, H, side, tc_kb(H), ntiles, blocks);
    return cudaGetLastError();
}

cudaError_t launch_compress_tc(const float2 *rings, int64_t n, int R, int Q, const double *w, const double *U, int H,
                               int side, float *blocks, cudaStream_t s) {
    switch (ilog2(Q)) {
        case 5: return launch_compress_tc_q<5>(rings, n, R, w, U, H, side, blocks, s);
        case 6: return launch_compress_tc_q<6>(rings, n, R, w, U, H, side, blocks, s);
        case 7: return launch_compress_tc_q<7>(rings, n, R, w, U, H, side, blocks, s);
        case 8: return launch_compress_tc_q<8>(rings, n, R, w, U, H, side, blocks, s);
        case 9: return launch_compress_tc_q<9>(rings, n, R, w, U, H, side, blocks, s);
        default: return launch_compress_tc_q<10>(rings, n, R, w, U, H, side, blocks, s);
    }
}

// canonical coefficients from compact TC blocks, test / debug path
__global__ void unpack_tc_kernel(const float *__restrict__ blocks, int64_t n, int Q, int H, int side, int KB,
                                 int64_t ntiles, float2 *__restrict__ coeffs) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * (int64_t)Q * H) return;
    const int h = (int)(idx % H);
    const int q = (int)((idx / H) % Q);
    const int64_t row = idx / ((int64_t)H * Q);
    const int N = Q / 2;
    const int qq = q <= N ? q : Q - q;
    const int j = q <= N ? h : H + h;
    const int kb = j / 16, ch = (j % 16) / 2, jj = j % 2;
    const int rows_tile = side == RSVD_SIDE_TEMPLATE ? TC_TT : TC_MT;
    const int r = (int)(row % rows_tile);
    const int64_t sub = ((int64_t)qq * ntiles + row / rows_tile) * KB + kb;
    const int64_t off = (sub * rows_tile + r) * 32 + (int64_t)((ch ^ (r & 7)) * 4) + 2 * jj;
    float2 v = make_float2(blocks[off], blocks[off + 1]);          // alpha_j / beta_j
    if (q <= N) { if (side == RSVD_SIDE_IMAGE) v = c_conj(v); }
    else { if (side == RSVD_SIDE_TEMPLATE) v = c_conj(v); }
    coeffs[idx] = v;
}

cudaError_t launch_unpack_tc(const float *blocks, int64_t n, int Q, int H, int side, float2 *coeffs, cudaStream_t s) {
    const int64_t total = n * (int64_t)Q * H;
    const int64_t ntiles = tc_rows_pad_side(n, side) / (side == RSVD_SIDE_TEMPLATE ? TC_TT : TC_MT);
    unpack_tc_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(blocks, n, Q, H, side, tc_kb(H), ntiles, coeffs);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ contraction launch (one chunk)
cudaError_t launch_contract_tc(const float *Acmp, const float *Bcmp, int H, int N, int64_t Mpad, int64_t Tpad,
                               int64_t m0, int64_t t0, int64_t mc, int64_t tc, int64_t Mc, int64_t Tc, float *Upk,
                               cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(contract_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TC_SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int KB = tc_kb(H);
    const int mtl = (int)(mc / TC_MT), ntl = (int)(tc / TC_TT);
    const int ntiles = mtl * ntl;
    const int target = 148;
    int nqg = std::max(1, (target + ntiles - 1) / ntiles);
    nqg = std::min(nqg, N + 1);
    const int qg = (N + 1 + nqg - 1) / nqg;
    nqg = (N + 1 + qg - 1) / qg;
    contract_tc_kernel<<<(unsigned)(ntiles * nqg), TC_THREADS, TC_SMEM, s>>>(
        Acmp, Bcmp, KB, N, Mpad / TC_MT, Tpad / TC_TT, m0 / TC_MT, t0 / TC_TT, ntl, qg, nqg, Mc, Tc, Upk);
    return cudaGetLastError();
}

}  // namespace rsvd

extern "C" void rsvd_set_path(int32_t path) { rsvd::set_path(path); }
extern "C" int32_t rsvd_path_for(int32_t Q, int32_t H) { return rsvd::resolve_path(Q, H); }
