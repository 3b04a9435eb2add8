// rsvd_tc.cu -- tensor-core path of Step 1 storage and Step 2 (the q-batched complex contraction,
// PAPER.md:672) on sm_100a: tcgen05.mma kind::tf32 with 3xTF32 error compensation.
//
// Real embedding of the complex contraction U_q[m,t] = sum_j alpha[q][j][m] beta[q][j][t]
// (alpha/beta as in rsvd_compress.cu):  A'[m][2j + c] = (Re, Im) alpha_j, and two B rows per template,
//   B'[2t][.]   = (Re beta_j, -Im beta_j)   ->  D[m][2t]   = Re U
//   B'[2t+1][.] = (Im beta_j,  Re beta_j)   ->  D[m][2t+1] = Im U
// Each fp32 operand x is split x = hi + lo with hi, lo TF32-rounded; D = Ahi Bhi + Ahi Blo + Alo Bhi
// recovers ~fp32 accuracy (the dropped Alo Blo term is ~2^-22 relative).
//
// Block layout (TC): 128-row x 32-float K-major sub-tiles stored pre-swizzled exactly as the
// UMMA SWIZZLE_128B canonical layout expects (16-byte chunk c of row r at chunk c ^ (r & 7)):
//   images    A[q][mtile][kb][hi|lo][128 rows][32]   (mtile = 128 images)
//   templates B[q][ttile][kb][hi|lo][256 rows][32]   (ttile = 128 templates = 256 B-rows)
// q = 0..N (N = Q/2), kb < KB = ceil(4H/32).  One stage of the contraction is then two contiguous
// bulk copies (cp.async.bulk, mbarrier complete_tx): 32 KB of A and 64 KB of B.
//
// contract_tc_kernel: one CTA per (128 x 128 pair tile, group of q), 6 warps:
//   warp 0  producer: bulk-copies (q, kb) stages into a 2-deep smem ring;
//   warp 1  TMEM allocator + MMA issuer: per stage 4 k-steps x 3 tcgen05.mma (M=128, N=256, K=8) into
//           one of two 256-column TMEM accumulators; tcgen05.commit releases smem / signals epilogue;
//   warps 2-5 epilogue: tcgen05.ld 32x32b of their 32 lanes, store U_q rows q-major to the spectrum
//           workspace (same layout as the SIMT contraction), release the accumulator.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "rsvd_common.cuh"

namespace rsvd {

constexpr int TC_THREADS = 192;
constexpr int TC_STAGES = 2;
constexpr uint32_t TC_A_BYTES = 2u * 128u * 128u;    // hi + lo, 128 rows x 128 B
constexpr uint32_t TC_B_BYTES = 2u * 256u * 128u;    // hi + lo, 256 rows x 128 B
constexpr uint32_t TC_STAGE_BYTES = TC_A_BYTES + TC_B_BYTES;
constexpr size_t TC_SMEM = (size_t)TC_STAGES * TC_STAGE_BYTES + 1024 + 256;

int tc_kb(int H) { return (int)((4 * (int64_t)H + 31) / 32); }
int64_t tc_rows_pad(int64_t rows) { return round_up(rows, 128); }
int64_t tc_block_bytes(int64_t rows, int Q, int H, int side) {
    return (int64_t)(Q / 2 + 1) * tc_kb(H) * 2 * tc_rows_pad(rows) * 128 * (side == RSVD_SIDE_TEMPLATE ? 2 : 1);
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
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
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

// ------------------------------------------------------------------ contraction kernel
// grid: ntiles_chunk * nqg.  Chunk tiles are (Mc/128) x (Tc/128); item -> (tile, q-group).
__global__ void __launch_bounds__(TC_THREADS, 1) contract_tc_kernel(
    const float *__restrict__ Atc, const float *__restrict__ Btc, int KB, int N, int64_t MT, int64_t NT, int64_t mt0,
    int64_t nt0, int ntl, int qg, int nqg, int64_t Mc, int64_t Tc, float2 *__restrict__ Upk) {
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

    if (warp == 1) {
        if (lane == 0) {
            for (int s = 0; s < TC_STAGES; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
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
        if (lane == 0) {
            int it = 0;
            for (int qi = 0; qi < nqi; ++qi) {
                const int q = q_begin + qi;
                for (int kb = 0; kb < KB; ++kb, ++it) {
                    const int s = it % TC_STAGES;
                    const uint32_t ph = (uint32_t)(it / TC_STAGES) & 1u;
                    mbar_wait(empty + s, ph ^ 1u);
                    unsigned char *sa = base + s * TC_STAGE_BYTES;
                    mbar_expect_tx(full + s, TC_STAGE_BYTES);
                    const float *ga = Atc + (((int64_t)q * MT + mt) * KB + kb) * (int64_t)(2 * 128 * 32);
                    const float *gb = Btc + (((int64_t)q * NT + nt) * KB + kb) * (int64_t)(2 * 256 * 32);
                    bulk_g2s(sa, ga, TC_A_BYTES, full + s);
                    bulk_g2s(sa + TC_A_BYTES, gb, TC_B_BYTES, full + s);
                }
            }
        }
    } else if (warp == 1) {
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
                    const uint64_t a_hi = sw128_desc(sa), a_lo = sw128_desc(sa + 128 * 128);
                    const uint64_t b_hi = sw128_desc(sa + TC_A_BYTES), b_lo = sw128_desc(sa + TC_A_BYTES + 256 * 128);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t o = (uint64_t)(2 * k);          // +32 B per K=8 tf32 step
                        tc_mma_tf32(dt, a_hi + o, b_hi + o, idesc, (kb | k) ? 1u : 0u);
                        tc_mma_tf32(dt, a_hi + o, b_lo + o, idesc, 1u);
                        tc_mma_tf32(dt, a_lo + o, b_hi + o, idesc, 1u);
                    }
                    tc_commit(empty + s);          // smem stage free once these MMAs complete
                }
                tc_commit(tfull + acc);            // accumulator ready for the epilogue
            }
        }
    } else {
        const int quad = warp & 3;                 // TMEM lane quadrant this warp may access
        const int row = quad * 32 + lane;
        for (int qi = 0; qi < nqi; ++qi) {
            const int acc = qi & 1;
            mbar_wait(tfull + acc, ((uint32_t)qi >> 1) & 1u);
            tc_fence_after();
            const int q = q_begin + qi;
            const int n = (q == N) ? 0 : q;
            float2 *dst = Upk + ((int64_t)n * Mc + (int64_t)mt_l * 128 + row) * Tc + (int64_t)nt_l * 128;
            const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * 256);
#pragma unroll 1
            for (int c0 = 0; c0 < 256; c0 += 32) {
                uint32_t v[32];
                tmem_ld32(tbase + (uint32_t)c0, v);
                float2 *d = dst + c0 / 2;
                if (q == 0) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) reinterpret_cast<float *>(d + i)[0] = __uint_as_float(v[2 * i]);
                } else if (q == N) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) reinterpret_cast<float *>(d + i)[1] = __uint_as_float(v[2 * i]);
                } else {
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        reinterpret_cast<float4 *>(d)[i] =
                            make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                        __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty + acc);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// ------------------------------------------------------------------ TC block emission (Step 1 tail)
__device__ __forceinline__ float tf32_rn(float x) {
    uint32_t u = __float_as_uint(x);
    if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x0FFFu + ((u >> 13) & 1u)) & 0xFFFFE000u;
    return __uint_as_float(u);
}

// Emits the TC blocks of one row (image or template) from its coefficients at[h][q] (smem, [H][Q]).
// 8 lanes write one 128-byte swizzled row (one 16-byte chunk each).
__device__ void emit_tc_rows(const float2 *at, int H, int Q, int KB, int side, int64_t row, int64_t ntiles,
                             float *__restrict__ blocks) {
    const int N = Q / 2;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int ch = tid & 7;
    const int64_t tile = row / 128;
    const int rr = (int)(row % 128);
    const int nc = side == RSVD_SIDE_TEMPLATE ? 2 : 1;          // B rows per template
    const int rows_tile = 128 * nc;
    const int total = (N + 1) * KB * nc;                      // (q, kb, c) rows; hi and lo both written
    for (int idx = tid >> 3; idx < total; idx += nthr >> 3) {
        const int c = idx % nc;
        const int kb = (idx / nc) % KB;
        const int q = idx / (nc * KB);
        const int r = rr * nc + c;                           // row inside the tile
        float v[4];
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
            if (side == RSVD_SIDE_IMAGE) { v[2 * jj] = a.x; v[2 * jj + 1] = a.y; }
            else if (c == 0) { v[2 * jj] = a.x; v[2 * jj + 1] = -a.y; }
            else { v[2 * jj] = a.y; v[2 * jj + 1] = a.x; }
        }
        const int64_t sub = (((int64_t)q * ntiles + tile) * KB + kb) * 2;   // hi sub-tile index
        const int64_t off = (int64_t)r * 32 + (int64_t)(((ch ^ (r & 7))) * 4);
        float4 hi, lo;
        hi.x = tf32_rn(v[0]); lo.x = tf32_rn(v[0] - hi.x);
        hi.y = tf32_rn(v[1]); lo.y = tf32_rn(v[1] - hi.y);
        hi.z = tf32_rn(v[2]); lo.z = tf32_rn(v[2] - hi.z);
        hi.w = tf32_rn(v[3]); lo.w = tf32_rn(v[3] - hi.w);
        *reinterpret_cast<float4 *>(blocks + sub * rows_tile * 32 + off) = hi;
        *reinterpret_cast<float4 *>(blocks + (sub + 1) * rows_tile * 32 + off) = lo;
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
    const int64_t nrows_tile = tc_rows_pad(n) / 128;
    compress_tc_kernel<LOGQ><<<(unsigned)n, 256, smem, s>>>(rings, n, R, w, U, H, side, tc_kb(H), nrows_tile, blocks);
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

// canonical coefficients from TC blocks (hi + lo), test / debug path
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
    const int nc = side == RSVD_SIDE_TEMPLATE ? 2 : 1;
    const int r = (int)(row % 128) * nc;                 // c = 0 row (template: (Re, -Im))
    const int64_t sub = (((int64_t)qq * ntiles + row / 128) * KB + kb) * 2;
    const int64_t off = (int64_t)r * 32 + (int64_t)((ch ^ (r & 7)) * 4) + 2 * jj;
    const int64_t rt = 128 * nc * 32;
    const float x = blocks[sub * rt + off] + blocks[(sub + 1) * rt + off];
    const float y = blocks[sub * rt + off + 1] + blocks[(sub + 1) * rt + off + 1];
    float2 v = side == RSVD_SIDE_IMAGE ? make_float2(x, y) : make_float2(x, -y);   // alpha_j / beta_j
    // undo the conj placement of the block layout
    if (q <= N) { if (side == RSVD_SIDE_IMAGE) v = c_conj(v); }
    else { if (side == RSVD_SIDE_TEMPLATE) v = c_conj(v); }
    coeffs[idx] = v;
}

cudaError_t launch_unpack_tc(const float *blocks, int64_t n, int Q, int H, int side, float2 *coeffs, cudaStream_t s) {
    const int64_t total = n * (int64_t)Q * H;
    unpack_tc_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(blocks, n, Q, H, side, tc_kb(H),
                                                                     tc_rows_pad(n) / 128, coeffs);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ contraction launch (one chunk)
cudaError_t launch_contract_tc(const float *Atc, const float *Btc, int H, int N, int64_t Mpad, int64_t Tpad,
                               int64_t m0, int64_t t0, int64_t mc, int64_t tc, int64_t Mc, int64_t Tc, float2 *Upk,
                               cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(contract_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TC_SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int KB = tc_kb(H);
    const int mtl = (int)(mc / 128), ntl = (int)(tc / 128);
    const int ntiles = mtl * ntl;
    const int target = 148;
    int nqg = std::max(1, (target + ntiles - 1) / ntiles);
    nqg = std::min(nqg, N + 1);
    const int qg = (N + 1 + nqg - 1) / nqg;
    nqg = (N + 1 + qg - 1) / qg;
    contract_tc_kernel<<<(unsigned)(ntiles * nqg), TC_THREADS, TC_SMEM, s>>>(
        Atc, Btc, KB, N, Mpad / 128, Tpad / 128, m0 / 128, t0 / 128, ntl, qg, nqg, Mc, Tc, Upk);
    return cudaGetLastError();
}

}  // namespace rsvd

extern "C" void rsvd_set_path(int32_t path) { rsvd::set_path(path); }
extern "C" int32_t rsvd_path_for(int32_t Q, int32_t H) { return rsvd::resolve_path(Q, H); }
