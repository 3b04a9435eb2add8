// rsvd_compress_mma.cuh -- Step 1 (compress, PAPER.md:580-585 / :240-244) for the TC operand layout with
// the radial projection on the tensor cores.  Included by rsvd_tc.cu (uses its emit_tc_rows, at_pos,
// scale_for, tc_kb, tc_op_rows, encode_fn).
//
// The projection of one row (image or template) onto the H principal rings is a real GEMM:
//   D[m][h] = sum_r a[r][m] U'[r][h],   m = 2 psi + c (c = Re / Im of the sample a_r(psi)),
//   U'[r][h] = U[r][h] sqrt(w_r) / Q      (the same fp32-rounded basis as compress_tc_kernel),
// M = 2Q floats of each ring, K = R rings, N = H principal rings (padded to NPAD = 16 or 32).
// tcgen05.mma kind::tf32 (cta_group::1, M = 128 per tile, N = NPAD, K = 8 rings per instruction) with a
// three-term split for ~fp32 accuracy: a = a_hi + a_lo (a_hi = a truncated to tf32 -- what the tensor
// core reads from an fp32 operand --, a_lo the exact remainder), U' = U'_hi + U'_lo (rounded split),
// D = a_hi U'_hi + a_hi U'_lo + a_lo U'_hi (dropped a_lo U'_lo ~ 2^-21 relative).
// The rings stream from HBM once: TMA boxes of 8 rings x 512 floats (four M-tiles) land MN-major in
// the SWIZZLE_128B_BASE32B layout that tf32 MN-major operands need.  Each stage is used twice in place:
// the a_hi products read the raw stage, then four splitter warps overwrite it with a_lo for the a_lo
// product -- no second buffer, so all spare shared memory goes to TMA depth.  The row's accumulator (2Q/128 M-tiles x NPAD columns of TMEM, two buffers)
// is read by eight epilogue warps into the [H][Q] coefficient block in shared memory, which then takes
// the same length-Q DFTs, row scale and hi/lo operand emission as compress_tc_kernel.
//
// Warp roles (512 threads, one persistent CTA per SM, rows blockIdx.x, blockIdx.x + grid, ...):
//   warp 0      TMA producer;  warp 1  TMEM allocator + MMA issuer;  warps 4-7  tf32 splitters;
//   warps 8-15 + 2-3  epilogue (TMEM -> [H][Q] chunk, DFTs, scale, emission).
#pragma once
// (included inside namespace rsvd)

#ifndef CM_LAG
#define CM_LAG 3               // stages between a stage's phase-1 and phase-2 products
#endif
#ifndef RSVD_CM_PREFETCH
#define RSVD_CM_PREFETCH 0     // L2 prefetch of the next row (measured: doubles the HBM reads -- L2 thrash)
#endif
constexpr int CM_THREADS = 512;
constexpr int CM_KR = 8;                                   // rings per stage (tf32 MMA K)
constexpr int CM_HC = 8;                                   // principal rings per epilogue chunk
constexpr int CM_MAXST = 10;
constexpr size_t CM_SMEM_MAX = 227 * 1024;

// Stage = 8 rings x MC floats (MC = min(512, 2Q): up to four M-tiles), one TMA box; as many stages as
// fit next to the split basis, one [CM_HC][Q] coefficient chunk and the twiddles.
struct CmGeom {
    int Q, H, R, NPAD, RP32, MC, T, NPASS, NSLAB, COLS, ALLOC, NST;
    uint32_t stage_bytes;
    size_t fixed, smem;
};
static inline CmGeom cm_geom(int Q, int H, int R) {
    CmGeom g;
    g.Q = Q; g.H = H; g.R = R;
    g.NPAD = H <= 16 ? 16 : 32;
    g.RP32 = (R + 31) / 32 * 32;
    g.MC = std::min(512, 2 * Q);
    g.T = 2 * Q / 128;
    g.NPASS = 2 * Q / g.MC;
    g.NSLAB = (R + CM_KR - 1) / CM_KR;
    g.COLS = g.T * g.NPAD;                                 // TMEM columns per accumulator
    g.ALLOC = 32;
    while (g.ALLOC < 2 * g.COLS) g.ALLOC *= 2;
    g.stage_bytes = (uint32_t)(CM_KR * g.MC * 4);
    g.fixed = 1024 + 2 * (size_t)(g.RP32 / 32) * g.NPAD * 128 +
              (size_t)CM_HC * Q * 8 + (size_t)Q * 8 + 1024;
    g.NST = g.fixed < CM_SMEM_MAX ? (int)std::min<size_t>(CM_MAXST, (CM_SMEM_MAX - g.fixed) / g.stage_bytes) : 0;
    g.smem = g.fixed + (size_t)g.NST * g.stage_bytes;
    return g;
}
// shapes: 2Q >= 256, H <= 32 with 4 | H once it takes more than one epilogue chunk (operand quarters
// of 4 coefficients must not straddle chunks), more stages than the phase-2 lag, both TMEM buffers in
// 512 columns
static inline bool cm_supported(int Q, int H, int R) {
    if (2 * Q < 256 || 2 * Q > 2048 || H > 32 || (H > CM_HC && H % 4 != 0) || R > 256) return false;
    const CmGeom g = cm_geom(Q, H, R);
    return g.ALLOC <= 512 && g.NST > CM_LAG;      // phase 2 of stage i is issued after phase 1 of i + CM_LAG
}

// UMMA descriptor, MN-major SWIZZLE_128B_BASE32B (tf32): 128-B MN rows (32 elements), 4-row K groups
// SBO = 512 B apart, MN atoms of 32 elements LBO bytes apart.
__device__ __forceinline__ uint64_t mn_sw128b32_desc(uint32_t saddr, uint32_t lbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)(512 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)1 << 61;                                // SWIZZLE_128B_BASE32B
    return d;
}
__device__ __forceinline__ void tc_mma_tf32_1(uint32_t dtmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dtmem),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void cm_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void cm_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
// a = hi + lo with hi = a rounded to tf32 (10 explicit mantissa bits; low 13 bits zero) and lo exact
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u); }
// what kind::tf32 reads from an fp32 operand: the low 13 mantissa bits dropped (measured: a_lo = a - this
// passes the compress parity gate, a_lo = a - RNE(a) fails it)
__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

template <int LOGQ>
__global__ void __launch_bounds__(CM_THREADS, 1)
    compress_mma_kernel(const __grid_constant__ CUtensorMap tmR, const float2 *__restrict__ rings, int64_t n, int R,
                        const double *__restrict__ w, const double *__restrict__ U, int H, int NPAD, int NST,
                        int side, int KB, int64_t op_rows, __half *__restrict__ ops, float *__restrict__ scales) {
    constexpr int Q = 1 << LOGQ;
    constexpr int L = 32, E = Q / L;
    constexpr int MC = 2 * Q < 512 ? 2 * Q : 512;             // floats of a ring per stage
    constexpr int MT = MC / 128;                               // M-tiles per stage
    constexpr int T = 2 * Q / 128, NPASS = 2 * Q / MC;
    constexpr uint32_t SB = CM_KR * MC * 4;                    // stage bytes (TMA box)
    const int NSLAB = (R + CM_KR - 1) / CM_KR, RP32 = (R + 31) / 32 * 32;
    const int COLS = T * NPAD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char *bhi = base + (size_t)NST * SB;              // [RP32/32][NPAD][32] tf32, K-major SW128
    unsigned char *blo = bhi + (size_t)(RP32 / 32) * NPAD * 128;
    float2 *at = reinterpret_cast<float2 *>(blo + (size_t)(RP32 / 32) * NPAD * 128);   // [CM_HC][Q] chunk
    float2 *tw = at + (size_t)CM_HC * Q;                                              // [E][L]
    uint64_t *bars = reinterpret_cast<uint64_t *>(tw + Q);
    // per stage: full (TMA landed) -> mma1 (a_hi products done) -> split2 (a_lo in place) -> empty (a_lo
    // product done)
    uint64_t *full = bars, *mma1 = full + CM_MAXST, *split2 = mma1 + CM_MAXST;
    uint64_t *empty = split2 + CM_MAXST;
    uint64_t *tfull = empty + CM_MAXST, *tempty = tfull + 2, *amaxb = tempty + 2, *amaxf = amaxb + 2;
    float *amax_w = reinterpret_cast<float *>(amaxf + 2);                           // [2][4]
    float *red = amax_w + 8;                                                        // [34]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(red + 34);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const double invQ = 1.0 / (double)Q;
    uint32_t alloc = 32;
    while (alloc < (uint32_t)(2 * COLS)) alloc *= 2;

    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(full + s, 1); mbar_init(mma1 + s, 1); mbar_init(split2 + s, 4);
            mbar_init(empty + s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull + b, 1); mbar_init(tempty + b, 1); mbar_init(amaxb + b, 4); mbar_init(amaxf + b, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(alloc));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // U' split into tf32 hi / lo, K-major SWIZZLE_128B: element (n = h, k = r) of k-block r / 32 at byte
    // n * 128 + ((4 (r % 32) / 16) ^ (n % 8)) * 16 + (4 r) % 16 of the block
    for (int i = tid; i < RP32 * NPAD; i += CM_THREADS) {
        const int r = i / NPAD, h = i - r * NPAD;
        float v = 0.f;
        if (r < R && h < H) v = (float)(U[(int64_t)r * H + h] * sqrt(w[r]) * invQ);
        const float vh = tf32_hi(v);
        const int kk = r & 31;
        const uint32_t off = (uint32_t)(r >> 5) * NPAD * 128 + h * 128 + ((((kk * 4) >> 4) ^ (h & 7)) << 4) + ((kk * 4) & 15);
        *reinterpret_cast<float *>(bhi + off) = vh;
        *reinterpret_cast<float *>(blo + off) = v - vh;
    }
    for (int i = tid; i < E * L; i += CM_THREADS) tw[i] = twiddle_N(i % L, i / L, Q);
    // c = max_h sum_r |U[r][h]| sqrt(w_r) / Q (the bound compress_tc_kernel uses)
    float cmax = 0.f;
    for (int h = warp; h < H; h += CM_THREADS / 32) {
        double c = 0.0;
        for (int r = lane; r < R; r += 32) c += fabs(U[(int64_t)r * H + h]) * sqrt(w[r]);
#pragma unroll
        for (int off = 16; off; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
        cmax = fmaxf(cmax, (float)(c * invQ));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");      // B written by threads, read by the MMA
    tc_fence_before();
    cmax = block_max(cmax, red);                                      // (syncs the block)
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer (RSVD_CM_PREFETCH=1 also pulls the next row into L2: measured to
        // double the HBM reads -- 148 CTAs x 2 rows in flight do not fit L2 -- so off)
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmR)) : "memory");
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            const uint32_t row_bytes = (uint32_t)R * Q * 8u;
            (void)row_bytes;
            int it = 0;
            for (int64_t row = blockIdx.x; row < n; row += gridDim.x) {
#if RSVD_CM_PREFETCH
                if (row + gridDim.x < n) {
                    const char *nx = reinterpret_cast<const char *>(rings + (row + gridDim.x) * (int64_t)R * Q);
                    for (uint32_t o = 0; o < row_bytes; o += 65536u)
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nx + o),
                                     "r"(min(65536u, row_bytes - o))
                                     : "memory");
                }
#endif
                for (int p = 0; p < NPASS; ++p)
                    for (int j = 0; j < NSLAB; ++j, ++it) {
                        const int s = it % NST;
                        mbar_wait(empty + s, ((uint32_t)(it / NST) & 1u) ^ 1u);
                        mbar_expect_tx(full + s, SB);
                        asm volatile(
                            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                            " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(base + (size_t)s * SB)),
                            "l"(reinterpret_cast<uint64_t>(&tmR)), "r"(0), "r"(j * CM_KR), "r"(p * (MC / 32)),
                            "r"((int)row), "r"(smem_u32(full + s)), "l"(pol)
                            : "memory");
                    }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer: phase 1 of a stage (a_hi U'_hi + a_hi U'_lo per M-tile, a_hi being the
        // raw fp32 stage, which the tensor core reads as tf32 by truncation) as soon as it lands; phase 2
        // (a_lo U'_hi, after the splitters overwrote the stage with a_lo) CM_LAG stages later, so the
        // splitters' round trip overlaps the following stages' phase-1 products
        if (lane == 0) {
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | ((uint32_t)(NPAD >> 3) << 17) |
                                   ((uint32_t)(128 >> 4) << 24);
            const int SPR = NPASS * NSLAB;                            // stages per row
            int it = 0, k = 0;
            for (int64_t row = blockIdx.x; row < n; row += gridDim.x, ++k) {
                const int b = k & 1;
                mbar_wait(tempty + b, (((uint32_t)k >> 1) & 1u) ^ 1u);
                tc_fence_after();
                const int it0 = it;
                auto phase2 = [&](int i2) {                           // stage i2 of this row
                    const int s2 = i2 % NST, l2 = i2 - it0, p2 = l2 / NSLAB, j2 = l2 - p2 * NSLAB;
                    mbar_wait(split2 + s2, (uint32_t)(i2 / NST) & 1u);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(base + (size_t)s2 * SB);
                    const uint64_t bh = sw128_desc(smem_u32(bhi) + (uint32_t)(j2 >> 2) * NPAD * 128) + (uint64_t)(2 * (j2 & 3));
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt)
                        tc_mma_tf32_1(tmem + (uint32_t)(b * COLS + (p2 * MT + mt) * NPAD),
                                          mn_sw128b32_desc(sa + mt * 4096, 1024), bh, idesc, 1u);
                    cm_commit(empty + s2);                            // stage free once these complete
                };
                for (int l = 0; l < SPR; ++l, ++it) {
                    const int p = l / NSLAB, j = l - p * NSLAB, s = it % NST;
                    mbar_wait(full + s, (uint32_t)(it / NST) & 1u);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(base + (size_t)s * SB);
                    const uint64_t bh = sw128_desc(smem_u32(bhi) + (uint32_t)(j >> 2) * NPAD * 128) + (uint64_t)(2 * (j & 3));
                    const uint64_t bl = sw128_desc(smem_u32(blo) + (uint32_t)(j >> 2) * NPAD * 128) + (uint64_t)(2 * (j & 3));
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        const uint32_t d = tmem + (uint32_t)(b * COLS + (p * MT + mt) * NPAD);
                        const uint64_t ah = mn_sw128b32_desc(sa + mt * 4096, 1024);
                        tc_mma_tf32_1(d, ah, bh, idesc, j > 0 ? 1u : 0u);
                        tc_mma_tf32_1(d, ah, bl, idesc, 1u);
                    }
                    cm_commit(mma1 + s);                              // a_hi products done: stage may become a_lo
                    if (l >= CM_LAG) phase2(it - CM_LAG);
                }
                for (int l = SPR > CM_LAG ? SPR - CM_LAG : 0; l < SPR; ++l) phase2(it0 + l);
                cm_commit(tfull + b);                                 // the row's accumulator is complete
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ---------------- splitters: once a stage's phase-1 products are done, overwrite it with
        // a_lo = a - trunc_tf32(a) (exact); row max |Re|, |Im|
        const int t = tid - 128;
        constexpr int PER = SB / 16 / 128;                            // float4 per thread and stage
        const int SPR = NPASS * NSLAB;
        int it = 0, k = 0;
        for (int64_t row = blockIdx.x; row < n; row += gridDim.x, ++k) {
            float amax = 0.f;
            for (int l = 0; l < SPR; ++l, ++it) {
                const int s = it % NST;
                mbar_wait(mma1 + s, (uint32_t)(it / NST) & 1u);
                float4 *st = reinterpret_cast<float4 *>(base + (size_t)s * SB);
#pragma unroll
                for (int i = 0; i < PER; ++i) {
                    const float4 x = st[t + 128 * i];
                    amax = fmaxf(amax, fmaxf(fmaxf(fabsf(x.x), fabsf(x.y)), fmaxf(fabsf(x.z), fabsf(x.w))));
                    st[t + 128 * i] = make_float4(x.x - tf32_trunc(x.x), x.y - tf32_trunc(x.y), x.z - tf32_trunc(x.z),
                                                  x.w - tf32_trunc(x.w));
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) cm_arrive(split2 + s);
            }
#pragma unroll
            for (int off = 16; off; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
            const int b = k & 1;
            if (lane == 0) {
                mbar_wait(amaxf + b, (((uint32_t)k >> 1) & 1u) ^ 1u);
                amax_w[b * 4 + (warp - 4)] = amax;
                cm_arrive(amaxb + b);
            }
        }
    } else if (warp >= 8 || warp == 2 || warp == 3) {
        // ---------------- epilogue, per chunk of CM_HC principal rings: TMEM -> [hc][Q] (warps 8-15, one
        // TMEM lane quadrant each), DFTs (one ring per warp), emission (all ten warps)
        const bool tw8 = warp >= 8;
        const int e = tw8 ? tid - 256 : 256 + tid - 64, ew = tw8 ? warp - 8 : 6 + warp, quad = warp & 3;
        auto ebar = [&]() { asm volatile("bar.sync 1, 320;" ::: "memory"); };
        float2 stw[clog2(L)];
        lane_stage_twiddles<L>(lane, stw);
        float *atf = reinterpret_cast<float *>(at);
        int k = 0;
        for (int64_t row = blockIdx.x; row < n; row += gridDim.x, ++k) {
            const int b = k & 1;
            const uint32_t ph = ((uint32_t)k >> 1) & 1u;
            mbar_wait(amaxb + b, ph);
            const float amax = fmaxf(fmaxf(amax_w[b * 4], amax_w[b * 4 + 1]), fmaxf(amax_w[b * 4 + 2], amax_w[b * 4 + 3]));
            const float sc = scale_for(1.41421356f * (float)Q * amax * cmax * 1.0000002f);
            mbar_wait(tfull + b, ph);
            tc_fence_after();
            for (int h0 = 0; h0 < H; h0 += CM_HC) {
                const int hc = min(CM_HC, H - h0);
                const bool last = h0 + CM_HC >= H;
                ebar();                                   // the previous chunk's emission has read at[]
                if (h0 == 0 && e == 0) cm_arrive(amaxf + b);
                for (int i = ew >> 2; tw8 && i < T; i += 2) {
                    uint32_t v[8];
                    const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * COLS + i * NPAD + h0);
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                                   "=r"(v[7])
                                 : "r"(ta));
                    tmem_wait_ld();
                    const int m = 128 * i + 32 * quad + lane;     // float index 2 psi + c within the ring
#pragma unroll
                    for (int hh = 0; hh < CM_HC; ++hh)
                        if (hh < hc) atf[(size_t)hh * 2 * Q + m] = __uint_as_float(v[hh]);
                }
                if (last) tc_fence_before();
                ebar();                                   // chunk complete in at[]
                if (last && e == 0) cm_arrive(tempty + b);   // TMEM buffer b read out
                // in-place length-Q forward DFT of each principal ring, natural order (as compress_tc_kernel)
                if (ew < hc) {
                    float2 v[E];
#pragma unroll
                    for (int x = 0; x < E; ++x) v[x] = at[ew * Q + lane + L * x];
                    fft_dist<E, L>(v, lane, tw, stw);
                    __syncwarp();
                    const int bb = (int)(__brev((unsigned)lane) >> 27);
#pragma unroll
                    for (int k1 = 0; k1 < E; ++k1) at[ew * Q + at_pos(k1 + E * bb, E)] = v[brev(k1, clog2(E))];
                }
                ebar();
                if (h0 == 0 && e == 0) scales[row] = sc;
                // operand quarters of this chunk's coefficients (+ the zero padding once)
                // (one chunk: every quarter; several: 4 | H, so quarters never straddle chunks)
                const QuarterSet qs = H <= CM_HC ? QuarterSet{0, 4 * KB, 0, 0, 0, 0}
                                                 : QuarterSet{h0 / 4, (h0 + hc) / 4, (H + h0) / 4, (H + h0 + hc) / 4,
                                                              h0 == 0 ? H / 2 : 0, h0 == 0 ? 4 * KB : 0};
                emit_tc_rows(at, h0, H, Q, KB, side, row, op_rows, sc, qs, ops, e, 320);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(alloc));
    }
}

// 4-D view of one side's rings as fp32 (32-float MN rows, ring, 32-float block, row) for 8-ring x
// 256-float boxes in the tf32 MN-major SWIZZLE_128B_ATOM_32B layout
static cudaError_t make_rings_tmap(CUtensorMap *tm, const float2 *rings, int64_t n, int R, int Q) {
    PFN_encodeTiled_tc enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    const cuuint64_t dims[4] = {32, (cuuint64_t)R, (cuuint64_t)(2 * Q / 32), (cuuint64_t)n};
    const cuuint64_t strides[3] = {(cuuint64_t)Q * 8, 128, (cuuint64_t)R * Q * 8};
    const cuuint32_t box[4] = {32, (cuuint32_t)CM_KR, (cuuint32_t)(std::min(512, 2 * Q) / 32), 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float2 *>(rings), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int LOGQ>
static cudaError_t launch_compress_mma_q(const CUtensorMap &tm, const float2 *rings, int64_t n, int R, const double *w, const double *U,
                                         int H, int side, float *blocks, cudaStream_t s) {
    const CmGeom g = cm_geom(1 << LOGQ, H, R);
    static std::atomic<uint64_t> attr{0};
    cudaError_t e = smem_attr_once((const void *)compress_mma_kernel<LOGQ>, (int)CM_SMEM_MAX, attr);   // any shape
    if (e != cudaSuccess) return e;
    const int grid = (int)std::min<int64_t>(n, (int64_t)num_sms());
    compress_mma_kernel<LOGQ><<<grid, CM_THREADS, g.smem, s>>>(tm, rings, n, R, w, U, H, g.NPAD, g.NST, side, tc_kb(H),
                                                               tc_op_rows(n, side), reinterpret_cast<__half *>(blocks),
                                                               const_cast<float *>(tc_scales(blocks, n, 1 << LOGQ, H, side)));
    return cudaGetLastError();
}

static std::atomic<int> g_compress_mma{-1};
static int compress_mma_mode() {
    int m = g_compress_mma.load(std::memory_order_relaxed);
    if (m < 0) {
        const char *e = getenv("RSVD_COMPRESS_MMA");
        m = e ? atoi(e) : 1;
        g_compress_mma.store(m, std::memory_order_relaxed);
    }
    return m;
}
// Projection on the tensor cores where the shape fits and it is faster (RSVD_COMPRESS_MMA=0 forces
// compress_tc_kernel, =2 forces this kernel wherever the shape fits -- the tests use it).
static cudaError_t launch_compress_mma(const float2 *rings, int64_t n, int R, int Q, const double *w, const double *U,
                                       int H, int side, float *blocks, cudaStream_t s, bool *launched) {
    *launched = false;
    const int env = compress_mma_mode();
    // measured crossover (tools/gpu_compress_ab.sh): the FFMA2 projection of compress_tc_kernel is cheaper
    // at small H (H = 8: 2.26 vs 3.02 ms on Large-shape rows), the tensor cores win from H = 16 at
    // Q = 256 and above H = 16 at Q = 512 (H = 24: 3.27 vs 4.21 ms; H = 32, Q = 256: 0.41 vs 0.64 ms)
    const bool wins = H > 16 || (H == 16 && Q <= 256);
    if (!env || !cm_supported(Q, H, R) || (env == 1 && !wins)) return cudaSuccess;    // 2: force
    CUtensorMap tm;
    if (make_rings_tmap(&tm, rings, n, R, Q) != cudaSuccess) return cudaSuccess;    // shape the TMA cannot map
    cudaError_t e;
    switch (ilog2(Q)) {
        case 7: e = launch_compress_mma_q<7>(tm, rings, n, R, w, U, H, side, blocks, s); break;
        case 8: e = launch_compress_mma_q<8>(tm, rings, n, R, w, U, H, side, blocks, s); break;
        case 9: e = launch_compress_mma_q<9>(tm, rings, n, R, w, U, H, side, blocks, s); break;
        case 10: e = launch_compress_mma_q<10>(tm, rings, n, R, w, U, H, side, blocks, s); break;
        default: return cudaSuccess;
    }
    if (e == cudaSuccess) *launched = true;
    return e;
}

