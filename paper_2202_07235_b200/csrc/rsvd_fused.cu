// rsvd_fused.cu -- rows a2-a4 (Step 2 contraction; Step 3 transform, :673; Step 4
// argmax / landscape, :504-517) as ONE persistent kernel with two CTA roles working on a ring of
// small, L2-sized spectrum buffers.
//
// Why: with one contraction launch and one transform launch per 128 MB chunk (rsvd_align.cu), the
// chunk does not fit the 126 MB L2 (most of it makes an HBM round trip) and the two kernels run one
// after the other, each paying a launch fill and tail.  Here the grid (one CTA per SM, clusters of
// two) is split once into
//   * KC contraction clusters (CTA pairs): tcgen05 kind::f16 MMAs (M = 256 rows = 128 images' Re/Im
//     rows, N = 128 templates, the error-compensated fp16 hi/lo split of rsvd_tc.cu), each owning a
//     fixed q-group of every chunk; TMA-fed 9-stage operand ring, 4 TMEM accumulators, 8 epilogue
//     warps that drain TMEM into the chunk's spectrum buffer;
//   * transform CTAs: the fft2 work items (rsvd_fft2.cuh: one template x 32 images, two groups of 8
//     warps, TMA-fed 3-slot ring) of every chunk, in a fixed global order.
// A chunk is one 128-image x 128-template pair tile (32 MB of spectrum at Q = 512).  Chunk c lives in
// buffer c % nbuf; two device counters per chunk order the roles:
//   cdone[c]  += 1 by every contraction epilogue warp once its stores of chunk c are done (release);
//             a transform CTA waits for cdone[c] == 2 * 8 * active clusters (acquire) before it
//             TMA-loads an item of chunk c;
//   tdone[c]  += 1 per transform item of chunk c once its data has landed in shared memory;
//             a contraction epilogue waits for tdone[c - nbuf] == items per chunk before it writes
//             chunk c into the buffer (spectrum reuse).
// Every wait is on work that precedes it in the global order, done by CTAs that are resident (one CTA
// per SM, grid <= the co-resident cluster count, checked before launch), so the schedule cannot
// deadlock.  The contraction and the transform overlap on different SMs; the spectrum ring
// (nbuf x 32 MB) is sized to stay in L2.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#define RSVD_TRACE_TU_FUSED
#include "rsvd_common.cuh"
#include "rsvd_fft2.cuh"
#include "rsvd_tcgen05.cuh"

namespace rsvd {

constexpr int FU_THREADS = 512;
constexpr int FU_TM = 128;                              // images per tile
constexpr int FU_TW = 128;                              // templates per tile (MMA N)
constexpr int FU_STAGES = 9;
constexpr uint32_t FU_A_BYTES = 128u * 128u;            // per CTA: 128 A rows x (32 hi + 32 lo) fp16
constexpr uint32_t FU_B_BYTES = 64u * 128u;             // per CTA: 64 B rows
constexpr uint32_t FU_STAGE_BYTES = FU_A_BYTES + FU_B_BYTES;
constexpr int FU_EPW = 8;                               // epilogue warps per CTA (2 per TMEM lane quadrant)
constexpr int FU_NACC = 4;                              // TMEM accumulators of FU_TW columns
constexpr int FU_IPC = FU_TW * (FU_TM / 32);            // transform items per chunk
constexpr size_t FU_C_SMEM = (size_t)FU_STAGES * FU_STAGE_BYTES + 1024;

struct FusedArgs {
    int N, KB, steps;
    int mtiles, nchunks;                // chunk c: template tile c / mtiles, image tile c % mtiles
    int KC, qg, nqg;                    // contraction clusters, q-group size, non-empty q-groups
    int nbuf;                           // spectrum buffers
    int64_t M, T;                       // valid images / templates of the call
    float *Upk;                         // nbuf x [2N rows][FU_TW][FU_TM] floats
    int *cdone, *tdone;                 // [nchunks] each, zeroed before the launch
    FftOut out;
};

__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(int *p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Spin (with back-off) until *p >= target.  Watchdog: a wait longer than 10 s can only be a broken
// schedule, so the kernel traps (the call then fails with a launch error) instead of hanging the GPU.
__device__ __forceinline__ void wait_counter(const int *p, int target) {
    if (ld_acquire(p) >= target) return;
    unsigned ns = 32;
    const uint64_t t0 = global_ns();
    while (ld_acquire(p) < target) {
        __nanosleep(ns);
        ns = ns < 512 ? 2 * ns : 512;
        if (global_ns() - t0 > 10000000000ull) __trap();
    }
}

// ------------------------------------------------------------------ contraction role (CTA pairs)
__device__ __forceinline__ void fused_contract(unsigned char *base, const CUtensorMap *tmA, const CUtensorMap *tmB,
                                               const FusedArgs &a, int cl) {
    uint64_t *bars = reinterpret_cast<uint64_t *>(base + FU_STAGES * FU_STAGE_BYTES);
    uint64_t *full = bars, *empty = bars + FU_STAGES, *tfull = bars + 2 * FU_STAGES,
             *tempty = bars + 2 * FU_STAGES + FU_NACC;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * FU_STAGES + 2 * FU_NACC);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_rank();
    const int N = a.N;
    const int q_begin = cl * a.qg, q_end = min(N + 1, q_begin + a.qg);
    const bool active = q_begin < q_end;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < FU_STAGES; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
        for (int x = 0; x < FU_NACC; ++x) { mbar_init(tfull + x, 1); mbar_init(tempty + x, 2 * FU_EPW); }
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

    if (active && warp == 0) {
        // ---------------- TMA producer (both CTAs): own 128 A rows + own 64 B rows per (q, kb)
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmA)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmB)) : "memory");
            uint64_t pol_stream, pol_keep;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
            int it = 0;
            for (int c = 0; c < a.nchunks; ++c) {
                const int nt = c / a.mtiles, mt = c - nt * a.mtiles;
                const int rowA = mt * 2 * FU_TM + (int)rank * 128;
                const int rowB = nt * FU_TW + (int)rank * 64;
                for (int q = q_begin; q < q_end; ++q) {
                    for (int kb = 0; kb < a.KB; ++kb, ++it) {
                        const int s = it % FU_STAGES;
                        mbar_wait(empty + s, ((uint32_t)(it / FU_STAGES) & 1u) ^ 1u);
                        const uint32_t fb = smem_u32(full + s);
                        if (rank == 0) mbar_expect_tx(full + s, 2 * FU_STAGE_BYTES);
                        const uint32_t fbl = rank == 0 ? fb : mapa_rank(fb, 0);
                        const uint32_t dst = smem_u32(base + s * FU_STAGE_BYTES);
                        tma_load_4d_pair(dst, tmA, 0, rowA, kb, q, fbl, pol_stream);
                        tma_load_4d_pair(dst + FU_A_BYTES, tmB, 0, rowB, kb, q, fbl, pol_keep);
                    }
                }
            }
            for (int k = 0; k < FU_STAGES && k < it; ++k) {          // drain: last MMA commits landed
                const int j = it - 1 - k;
                mbar_wait(empty + (j % FU_STAGES), (uint32_t)(j / FU_STAGES) & 1u);
            }
        }
    } else if (active && warp == 1) {
        // ---------------- MMA issuer (leader CTA)
        if (rank == 0 && lane == 0) {
            const uint32_t idesc = (1u << 4) | ((uint32_t)(FU_TW >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
            int it = 0, qi = 0;
            for (int c = 0; c < a.nchunks; ++c) {
                for (int q = q_begin; q < q_end; ++q, ++qi) {
                    const int acc = qi % FU_NACC;
                    mbar_wait(tempty + acc, (((uint32_t)(qi / FU_NACC)) & 1u) ^ 1u);
                    tc_fence_after();
                    const uint32_t dt = tmem + (uint32_t)(acc * FU_TW);
                    for (int kb = 0; kb < a.KB; ++kb, ++it) {
                        const int s = it % FU_STAGES;
                        mbar_wait(full + s, (uint32_t)(it / FU_STAGES) & 1u);
                        tc_fence_after();
                        const uint32_t sa = smem_u32(base + s * FU_STAGE_BYTES);
                        const uint64_t a_hi = sw128_desc(sa), a_lo = a_hi + 4;
                        const uint64_t b_hi = sw128_desc(sa + FU_A_BYTES), b_lo = b_hi + 4;
                        const int nst = min(2, a.steps - 2 * kb);
                        for (int k = 0; k < nst; ++k) {
                            const uint64_t o = (uint64_t)(2 * k);
                            tc_mma_f16_pair(dt, a_hi + o, b_hi + o, idesc, (kb | k) ? 1u : 0u);
                            tc_mma_f16_pair(dt, a_hi + o, b_lo + o, idesc, 1u);
                            tc_mma_f16_pair(dt, a_lo + o, b_hi + o, idesc, 1u);
                        }
                        tc_commit_pair(empty + s);
                    }
                    tc_commit_pair(tfull + acc);
                }
            }
        }
    } else if (active && warp >= 2 && warp < 2 + FU_EPW) {
        // ---------------- epilogue (both CTAs): TMEM -> spectrum buffer of the chunk
        const int ew = warp - 2;
        const int quad = warp & 3;                     // TMEM lane quadrant of this warp
        const int col0 = (ew >> 2) * (FU_TW / 2);      // this warp's half of the N columns
        const int row = quad * 32 + lane;
        const bool re_rows = row < 64;
        const int ml = (int)rank * 64 + (row & 63);
        const uint32_t te0 = rank == 0 ? smem_u32(tempty) : mapa_rank(smem_u32(tempty), 0);
        const int64_t plane = (int64_t)N * FU_TW * FU_TM;            // floats per plane
        uint64_t pol_ws;
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_ws));
        int qi = 0;
        for (int c = 0; c < a.nchunks; ++c) {
            if (c >= a.nbuf) {                          // the buffer's previous chunk has been read out
                if (lane == 0) wait_counter(a.tdone + (c - a.nbuf), FU_IPC);
                __syncwarp();
            }
            float *const buf = a.Upk + (int64_t)(c % a.nbuf) * 2 * plane;
            for (int q = q_begin; q < q_end; ++q, ++qi) {
                const int acc = qi % FU_NACC;
                mbar_wait(tfull + acc, ((uint32_t)(qi / FU_NACC)) & 1u);
                tc_fence_after();
                // q = 0: Re U_0 -> re plane slot 0; q = N: Re U_N -> im plane slot 0; their Im rows dropped
                const bool store = (q != 0 && q != N) || re_rows;
                const bool nyq = q == N;
                float *pl = (nyq || (q != 0 && !re_rows)) ? buf + plane : buf;
                const int n = nyq ? 0 : q;
                float *dst = pl + ((int64_t)n * FU_TW + col0) * FU_TM + ml;   // [n][t][m]
                const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * FU_TW + col0);
                uint32_t v[2][32];
                tmem_ld32(tbase, v[0]);
                tmem_wait_ld();
#pragma unroll
                for (int b = 0; b < FU_TW / 2 / 32; ++b) {
                    if (b + 1 < FU_TW / 2 / 32) tmem_ld32(tbase + (uint32_t)(32 * (b + 1)), v[(b + 1) & 1]);
                    if (store) {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(dst + (int64_t)(32 * b + i) * FU_TM),
                                         "f"(__uint_as_float(v[b & 1][i])), "l"(pol_ws)
                                         : "memory");
                    }
                    tmem_wait_ld();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(te0 + (uint32_t)(acc * 8));
            }
            // this warp's stores of chunk c are complete: publish them (release at gpu scope)
            __threadfence();
            __syncwarp();
            if (lane == 0) red_release_add(a.cdone + c, 1);
        }
    }
    tc_fence_before();
    cluster_sync_relaxed();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// ------------------------------------------------------------------ transform role (single CTAs)
template <int LOGN, int MODE>
__device__ __forceinline__ void fused_transform(unsigned char *base, const CUtensorMap *tmS, const FusedArgs &a,
                                                int tb, int nTc) {
    using C = Fft2Cfg<LOGN>;
    constexpr int N = C::N, TB = C::TB, G = C::G, GT = C::GT;
    float2 *Wn = reinterpret_cast<float2 *>(base + C::NSLOT * C::SLOT);
    float2 *Wq = Wn + N;
    uint64_t *full = reinterpret_cast<uint64_t *>(Wq + N / 2);
    uint64_t *empty = full + C::NSLOT;
    volatile int *tag = reinterpret_cast<volatile int *>(empty + C::NSLOT);      // [NSLOT] item issued into the slot
    volatile int *pending = tag + C::NSLOT;                                      // [NSLOT] item parked for its consumer
    const int tid = threadIdx.x;
    const int g = tid / GT, gt = tid - g * GT;
    const int warp = gt >> 5, lane = tid & 31;
    const int64_t total = (int64_t)a.nchunks * FU_IPC;
    const int cd_target = 2 * FU_EPW * a.nqg;
    auto id_of = [&](int i) { return (int64_t)tb + (int64_t)nTc * i; };
    struct Item { int c, tl, mg, nt, mt; int64_t t, m_first; int n_valid; bool real; };
    auto decode = [&](int64_t id) {
        Item it;
        it.c = (int)(id / FU_IPC);
        const int j = (int)(id - (int64_t)it.c * FU_IPC);
        it.tl = j / (FU_TM / TB);
        it.mg = j - it.tl * (FU_TM / TB);
        it.nt = it.c / a.mtiles;
        it.mt = it.c - it.nt * a.mtiles;
        it.t = (int64_t)it.nt * FU_TW + it.tl;
        it.m_first = (int64_t)it.mt * FU_TM + it.mg * TB;
        const int64_t nv = a.M - it.m_first;
        it.n_valid = (int)(nv < 0 ? 0 : (nv > TB ? TB : nv));
        it.real = it.t < a.T && it.n_valid > 0;
        return it;
    };
    // Issue item i into its slot (the slot is free).  Non-blocking form: when chunk c's spectrum is not
    // complete yet the item is parked in pending[slot] and its own consumer issues it later (blocking).
    // A thread therefore never blocks on a later chunk while an earlier item of its CTA still waits to
    // be issued or consumed -- the tdone counts of earlier chunks always make progress.
    auto try_issue = [&](int i, bool block) {               // one thread
        const int64_t id = id_of(i);
        const int sl = i % C::NSLOT;
        const Item it = decode(id);
        if (!block && ld_acquire(a.cdone + it.c) < cd_target) {
            pending[sl] = i;
            return;
        }
        wait_counter(a.cdone + it.c, cd_target);             // chunk c's spectrum is complete
        asm volatile("fence.proxy.async.global;" ::: "memory");
        const uint32_t bar = fr_smem(full + sl);
        if (!it.real) {
            tag[sl] = i;
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
            return;
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((uint32_t)C::UBYTES)
                     : "memory");
        const int row0 = (it.c % a.nbuf) * C::ROWS;
#pragma unroll
        for (int bx = 0; bx < C::NBOX; ++bx) {
            const uint32_t dst = fr_smem(base + (size_t)sl * C::SLOT + (size_t)bx * C::BOXR * TB * 4);
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                ::"r"(dst), "l"(reinterpret_cast<uint64_t>(tmS)), "r"(it.mg * TB), "r"(it.tl), "r"(row0 + bx * C::BOXR),
                "r"(bar)
                : "memory");
        }
        tag[sl] = i;
    };
    if (tid == 0) {
        for (int sl = 0; sl < C::NSLOT; ++sl) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(fr_smem(full + sl)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(fr_smem(empty + sl)), "r"(C::TASKS));
            tag[sl] = -1;
            pending[sl] = -1;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fft2_tables<LOGN>(Wn, Wq, tid, FU_THREADS);
    __syncthreads();
    if (tid == 0)
        for (int i = 0; i < C::NSLOT; ++i)
            if (id_of(i) < total) try_issue(i, false);
    __syncthreads();

    for (int i = g; id_of(i) < total; i += G) {
        const int sl = i % C::NSLOT;
        const Item it = decode(id_of(i));
        uint32_t stale[C::P2_PER];
        float smv[C::P2_PER];
        const float st = (it.real && a.out.sc_t) ? __ldg(a.out.sc_t + it.t) : 1.f;
        if (it.real) fft2_side<LOGN, MODE>(gt, it.m_first, it.n_valid, a.out, stale, smv);
        if (gt == 0) {
            while (tag[sl] != i)
                if (pending[sl] == i) {                      // parked by the slot's releaser: issue it now
                    pending[sl] = -1;
                    try_issue(i, true);
                }
        } else {
            while (tag[sl] != i) {}
        }
        fr_mbar_wait(full + sl, (uint32_t)(i / C::NSLOT) & 1u);
        if (gt == 0) red_release_add(a.tdone + it.c, 1);   // the item's spectrum lines have been read
        float *U = reinterpret_cast<float *>(base + (size_t)sl * C::SLOT);
        auto release = [&]() {
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(fr_smem(empty + sl)) : "memory");
            if (gt == 0 && id_of(i + C::NSLOT) < total) {
                fr_mbar_wait(empty + sl, (uint32_t)(i / C::NSLOT) & 1u);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                try_issue(i + C::NSLOT, false);
            }
        };
        if (it.real)
            fft2_item<LOGN, MODE>(U, gt, warp, lane, 1 + g, Wn, Wq, it.m_first, it.n_valid, it.t, st, stale, smv, a.out,
                                  release);
        else
            release();
    }
}

template <int LOGN, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(FU_THREADS, 1)
    align_fused_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const __grid_constant__ CUtensorMap tmS, const FusedArgs a) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char *base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    const int cl = (int)(blockIdx.x >> 1);
    if (cl < a.KC)
        fused_contract(base, &tmA, &tmB, a, cl);
    else
        fused_transform<LOGN, MODE>(base, &tmS, a, (int)blockIdx.x - 2 * a.KC, (int)gridDim.x - 2 * a.KC);
}

// 3-D view of the nbuf spectrum buffers (image, template, buffer * 2N + plane row), 32-image boxes
template <int LOGN>
static cudaError_t make_fused_spectrum_tmap(CUtensorMap *tm, const float *Upk, int nbuf) {
    using C = Fft2Cfg<LOGN>;
    PFN_encodeTiled_fr enc = encode_tiled_fn();
    if (!enc) return cudaErrorNotSupported;
    const cuuint64_t dims[3] = {(cuuint64_t)FU_TM, (cuuint64_t)FU_TW, (cuuint64_t)nbuf * C::ROWS};
    const cuuint64_t strides[2] = {(cuuint64_t)FU_TM * 4, (cuuint64_t)FU_TM * FU_TW * 4};
    const cuuint32_t box[3] = {(cuuint32_t)C::TB, 1u, (cuuint32_t)C::BOXR};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(Upk), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

static int env_int(const char *name, int dflt) {
    const char *e = getenv(name);
    return e ? atoi(e) : dflt;
}

int64_t fused_workspace_bytes(int Q, int nbuf) {
    return (int64_t)nbuf * Q * FU_TW * FU_TM * (int64_t)sizeof(float);          // 2N rows x 128 x 128 floats each
}
static int fused_nbuf() { return std::max(2, env_int("RSVD_FUSED_NBUF", 2)); }

template <int LOGN, int MODE>
static cudaError_t launch_fused_lm(const CUtensorMap &tmA, const CUtensorMap &tmB, FusedArgs a, cudaStream_t s,
                                   bool *launched) {
    const size_t smem = std::max(FU_C_SMEM + 256, Fft2Cfg<LOGN>::smem_bytes() + 64);
    static std::atomic<uint64_t> attr{0};
    cudaError_t e = smem_attr_once((const void *)align_fused_kernel<LOGN, MODE>, (int)smem, attr);
    if (e != cudaSuccess) return e;
    const int nsm = num_sms() & ~1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)nsm);
    cfg.blockDim = dim3(FU_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    int maxcl = 0;
    e = cudaOccupancyMaxActiveClusters(&maxcl, (const void *)align_fused_kernel<LOGN, MODE>, &cfg);
    if (e != cudaSuccess || maxcl * 2 < nsm) {                // not every CTA can be resident: not applicable
        (void)cudaGetLastError();
        return cudaSuccess;
    }
    CUtensorMap tmS;
    if ((e = make_fused_spectrum_tmap<LOGN>(&tmS, a.Upk, a.nbuf)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(a.cdone, 0, 2 * (size_t)a.nchunks * sizeof(int), s)) != cudaSuccess) return e;
    e = cudaLaunchKernelEx(&cfg, align_fused_kernel<LOGN, MODE>, tmA, tmB, tmS, a);
    if (e == cudaSuccess) *launched = true;
    return e;
}

template <int LOGN>
static cudaError_t launch_fused_l(int mode, const CUtensorMap &tmA, const CUtensorMap &tmB, const FusedArgs &a,
                                  cudaStream_t s, bool *launched) {
    if (mode == MODE_PAIR) return launch_fused_lm<LOGN, MODE_PAIR>(tmA, tmB, a, s, launched);
    if (mode == MODE_IMAGE) return launch_fused_lm<LOGN, MODE_IMAGE>(tmA, tmB, a, s, launched);
    return launch_fused_lm<LOGN, MODE_LANDSCAPE>(tmA, tmB, a, s, launched);
}

// The fused path for one align call on the TC layout: images [0, M) x templates [0, T) of the blocks,
// Q = 2N (Q_out = Q), every mode.  *launched = false (and cudaSuccess) when the path does not apply
// (fused disabled, Q not in [32, 512], workspace too small, or not all CTAs co-resident).
cudaError_t launch_align_fused(const void *alpha, int64_t M, const void *beta, int64_t T, int Q, int H, int mode,
                               void *work, int64_t work_bytes, const FftOut &out, cudaStream_t s, bool *launched) {
    *launched = false;
    if (!env_int("RSVD_FUSED", 0)) return cudaSuccess;
    const int N = Q / 2;
    const int LOGN = ilog2(N);
    if (LOGN < 4 || LOGN > 8) return cudaSuccess;
    const int nbuf = fused_nbuf();
    const int64_t mtiles = (M + FU_TM - 1) / FU_TM, ntiles = (T + FU_TW - 1) / FU_TW;
    const int64_t nchunks = mtiles * ntiles;
    if (nchunks > (1 << 30)) return cudaSuccess;
    const int64_t spec = fused_workspace_bytes(Q, nbuf);
    if (work_bytes < spec + 2 * nchunks * (int64_t)sizeof(int)) return cudaSuccess;
    const int nsm = num_sms() & ~1;
    int KC = env_int("RSVD_FUSED_KC", 14);
    KC = std::max(1, std::min(KC, nsm / 2 - 1));
    const int qg = (N + 1 + KC - 1) / KC;
    const int nqg = (N + 1 + qg - 1) / qg;
    cudaError_t e;
    CUtensorMap tmA, tmB;
    if ((e = make_tc_operand_tmap(&tmA, alpha, M, Q, H, RSVD_SIDE_IMAGE, 128)) != cudaSuccess) return e;
    if ((e = make_tc_operand_tmap(&tmB, beta, T, Q, H, RSVD_SIDE_TEMPLATE, 64)) != cudaSuccess) return e;
    FusedArgs a;
    a.N = N;
    a.KB = tc_kb(H);
    a.steps = (4 * H + 15) / 16;
    a.mtiles = (int)mtiles;
    a.nchunks = (int)nchunks;
    a.KC = KC;
    a.qg = qg;
    a.nqg = nqg;
    a.nbuf = nbuf;
    a.M = M;
    a.T = T;
    a.Upk = reinterpret_cast<float *>(work);
    a.cdone = reinterpret_cast<int *>(reinterpret_cast<char *>(work) + spec);
    a.tdone = a.cdone + nchunks;
    a.out = out;
    switch (LOGN) {
        case 4: return launch_fused_l<4>(mode, tmA, tmB, a, s, launched);
        case 5: return launch_fused_l<5>(mode, tmA, tmB, a, s, launched);
        case 6: return launch_fused_l<6>(mode, tmA, tmB, a, s, launched);
        case 7: return launch_fused_l<7>(mode, tmA, tmB, a, s, launched);
        default: return launch_fused_l<8>(mode, tmA, tmB, a, s, launched);
    }
}

}  // namespace rsvd
