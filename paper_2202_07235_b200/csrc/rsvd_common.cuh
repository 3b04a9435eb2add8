// rsvd_common.cuh -- shared device helpers of librsvd (CUDA path only; the oracle shares nothing).
//
// Holds: status/error plumbing, complex float2 arithmetic, and the distributed forward FFT used by
// both Step 1 (rsvd_compress: length-Q DFT of principal rings) and Step 3
// (rsvd_align: length-Q/2 DFT of the packed Hermitian spectrum).
//
// Distributed FFT layout ("four-step", N = L * E): a group of L lanes (L = min(32, N), a power of
// two) owns one length-N vector; lane l holds v[e] = x[l + L e], e < E.  fft_dist computes
//   X[k] = sum_n x[n] e^{-2 pi i n k / N}
// as (1) an in-register radix-2 DIF DFT of length E over e, (2) the twiddle W_N^{l k1},
// (3) a radix-2 DIF DFT of length L across lanes with warp shuffles.  On return lane l register
// brev_E(k1) holds X[k1 + E * brev_L(l)].
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "../../include/rsvd.h"

namespace rsvd {

// ------------------------------------------------------------------ status plumbing
void set_error(const std::string &msg);
rsvd_status fail(rsvd_status st, const std::string &msg);
rsvd_status cuda_check(cudaError_t e, const char *what);

// launch counter (rsvd_launch_count) and optional per-kernel event timing (rsvd_timing_*)
void count_launches(int n);
bool timing_enabled();
cudaEvent_t timing_event(cudaStream_t s);
void timing_span(cudaEvent_t a, cudaEvent_t b, int kind);
enum { TK_CONTRACT = 0, TK_FFT = 1, TK_COMPRESS = 2, TK_BASIS = 3, TK_FUSED = 4 };

// contraction path: FP32 SIMT (block layout "simt") or tcgen05 fp16 hi/lo split on CTA pairs (layout "tc").
// resolve_path(Q, H) is the single source of truth used by block sizing, compress and align.
enum { PATH_AUTO = 0, PATH_SIMT = 1, PATH_TC = 2 };
int resolve_path(int Q, int H);
bool tc_supported(int Q, int H);
int tc_kb(int H);
int64_t tc_rows_pad(int64_t rows);
int64_t tc_rows_pad_side(int64_t rows, int side);
int64_t tc_block_bytes(int64_t rows, int Q, int H, int side);
cudaError_t launch_compress_tc(const float2 *rings, int64_t n, int R, int Q, const double *w, const double *U, int H,
                               int side, float *blocks, const double *kr, const double *shifts, int S, cudaStream_t s);
cudaError_t launch_unpack_tc(const float *blocks, int64_t n, int Q, int H, int side, float2 *coeffs, cudaStream_t s);
cudaError_t make_tc_operand_tmap(CUtensorMap *tm, const void *blocks, int64_t rows, int Q, int H, int side,
                                 int box_rows = 128);
const float *tc_scales(const void *blocks, int64_t rows, int Q, int H, int side);
cudaError_t launch_contract_tc(const CUtensorMap &tmA, const CUtensorMap &tmB, int H, int N, int Nout, int64_t m0,
                               int64_t t0, int64_t mc, int64_t tc, int64_t Mc, int64_t Tc, float *Upk, int nsms,
                               bool operands_fresh, int fmt, cudaStream_t s);
// numeric precision of the TC align path: PREC_FP32 (error-compensated fp16 hi/lo, fp32 spectrum; the
// 1e-5 gate) or PREC_FAST (one fp16 MMA per product, fp16 spectrum; the <= 2e-3 gate of north_star)
enum { PREC_FP32 = 0, PREC_FAST = 1 };
#ifndef RSVD_SPLIT_SCALE
#define RSVD_SPLIT_SCALE (1.0f / 1048576.0f)     // split hi/lo spectrum: value x 2^-20 (fp16 range)
#endif
int resolve_precision();

// Per-device one-time kernel attribute (max dynamic shared memory): bit d of `done` is set once the
// attribute has been applied on device d.  The attribute is per device, so a process that launches on
// several GPUs sets it on each; concurrent first calls just set it twice (idempotent).
inline cudaError_t smem_attr_once(const void *fn, int bytes, std::atomic<uint64_t> &done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}
// SM count of the current device (cached per device)
inline int num_sms() {
    static std::atomic<int> cache[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    dev &= 63;
    int n = cache[dev].load(std::memory_order_relaxed);
    if (n <= 0) {
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        cache[dev].store(n, std::memory_order_relaxed);
    }
    return n;
}

// ------------------------------------------------------------------ optional CTA timeline (-DRSVD_TRACE)
// Diagnostic build only (tools/trace_align.py): every CTA of the two align kernels appends one record
// of %globaltimer stamps (entry, dependency wait passed, first work item ready, exit) to a per-TU
// device buffer, dumped by rsvd_trace_dump_<tu>.  Compiled out of the product library.
struct TraceRec { unsigned long long t0, t1, t2, t3; unsigned int kind_blk, key; };
#ifdef RSVD_TRACE
constexpr int TRACE_MAX = 1 << 20;
__device__ __forceinline__ unsigned long long trace_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define RSVD_TRACE_DEFINE(tu)                                                                          \
    static __device__ TraceRec g_trace[TRACE_MAX];                                                     \
    static __device__ unsigned int g_trace_n;                                                          \
    __device__ __forceinline__ void trace_put(const TraceRec &r) {                                     \
        const unsigned i = atomicAdd(&g_trace_n, 1u);                                                  \
        if (i < TRACE_MAX) g_trace[i] = r;                                                             \
    }                                                                                                  \
    extern "C" int rsvd_trace_dump_##tu(TraceRec *host, int max, int reset) {                          \
        unsigned n = 0;                                                                                \
        if (cudaDeviceSynchronize() != cudaSuccess) return -1;                                         \
        if (cudaMemcpyFromSymbol(&n, g_trace_n, sizeof(n)) != cudaSuccess) return -1;                  \
        n = n < (unsigned)TRACE_MAX ? n : (unsigned)TRACE_MAX;                                         \
        n = n < (unsigned)max ? n : (unsigned)max;                                                     \
        if (n && host && cudaMemcpyFromSymbol(host, g_trace, n * sizeof(TraceRec)) != cudaSuccess) return -1; \
        if (reset) {                                                                                   \
            const unsigned z = 0;                                                                      \
            if (cudaMemcpyToSymbol(g_trace_n, &z, sizeof(z)) != cudaSuccess) return -1;                \
        }                                                                                              \
        return (int)n;                                                                                 \
    }
#endif

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline bool is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }
inline int ilog2(int64_t x) {
    int r = 0;
    while ((int64_t(1) << r) < x) ++r;
    return r;
}
inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// Block layout constants (opaque to callers; rsvd_block_bytes / rsvd_blocks_unpack are the API).
// blocks: float2 [(Q/2 + 1)][Kpad][rows_pad], Kpad = round_up(2H, KPAD), rows_pad = round_up(rows, ROWPAD)
constexpr int KPAD = 16;
constexpr int ROWPAD = 64;
inline int64_t kpad_of(int H) { return round_up(2 * (int64_t)H, KPAD); }
inline int64_t rows_pad_of(int64_t rows) { return round_up(rows, ROWPAD); }

// ------------------------------------------------------------------ complex helpers
// On the device these are sm_100 packed-fp32 instructions (FADD2 / FMUL2 / FFMA2: two IEEE fp32
// lanes per instruction, operand swizzles, partial negation and scalar broadcast folded in), so a
// complex add costs one issue slot and a complex multiply two -- the FFT stages are issue-bound.
__host__ __device__ __forceinline__ float2 c_add(float2 a, float2 b) {
#ifdef __CUDA_ARCH__
    return __fadd2_rn(a, b);
#else
    return make_float2(a.x + b.x, a.y + b.y);
#endif
}
__host__ __device__ __forceinline__ float2 c_sub(float2 a, float2 b) {
#ifdef __CUDA_ARCH__
    return __fadd2_rn(a, make_float2(-b.x, -b.y));
#else
    return make_float2(a.x - b.x, a.y - b.y);
#endif
}
__host__ __device__ __forceinline__ float2 c_mul(float2 a, float2 b) {
#ifdef __CUDA_ARCH__
    // (a.x b.x - a.y b.y, a.x b.y + a.y b.x) = a.y * (-b.y, b.x) + a.x * b
    return __ffma2_rn(make_float2(a.y, a.y), make_float2(-b.y, b.x), __fmul2_rn(make_float2(a.x, a.x), b));
#else
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
#endif
}
// c * (s, s): a real scale of a complex value
__host__ __device__ __forceinline__ float2 c_scale(float2 a, float s) {
#ifdef __CUDA_ARCH__
    return __fmul2_rn(a, make_float2(s, s));
#else
    return make_float2(a.x * s, a.y * s);
#endif
}
__host__ __device__ __forceinline__ float2 c_conj(float2 a) { return make_float2(a.x, -a.y); }

// cos(2 pi i / 64) from a quarter-wave table of exact literals (compile-time folded when i is).
__host__ __device__ constexpr float cos64q(int i) {
    return i == 0 ? 1.00000000000000000000f : i == 1 ? 0.99518472667219692873f
         : i == 2 ? 0.98078528040323043058f : i == 3 ? 0.95694033573220882438f
         : i == 4 ? 0.92387953251128673848f : i == 5 ? 0.88192126434835504956f
         : i == 6 ? 0.83146961230254523567f : i == 7 ? 0.77301045336273699338f
         : i == 8 ? 0.70710678118654757274f : i == 9 ? 0.63439328416364548779f
         : i == 10 ? 0.55557023301960228867f : i == 11 ? 0.47139673682599780857f
         : i == 12 ? 0.38268343236508983729f : i == 13 ? 0.29028467725446233105f
         : i == 14 ? 0.19509032201612833135f : i == 15 ? 0.09801714032956077016f : 0.0f;
}
__host__ __device__ constexpr float cos64(int i) {
    return ((i & 63) <= 16) ? cos64q(i & 63)
         : ((i & 63) <= 32) ? -cos64q(32 - (i & 63))
         : ((i & 63) <= 48) ? -cos64q((i & 63) - 32) : cos64q(64 - (i & 63));
}
__host__ __device__ constexpr float sin64(int i) { return cos64(i - 16); }

__host__ __device__ constexpr int brev(int x, int bits) {
    int r = 0;
    for (int b = 0; b < bits; ++b) r |= ((x >> b) & 1) << (bits - 1 - b);
    return r;
}
__host__ __device__ constexpr int clog2(int x) { return x <= 1 ? 0 : 1 + clog2(x >> 1); }

// multiply by W_M^i = e^{-2 pi i * i / M} for compile-time M | 64 (M <= 64)
template <int M, int I>
__device__ __forceinline__ float2 c_mul_w(float2 d) {
    constexpr int idx = (I * (64 / M)) & 63;
    if constexpr (idx == 0) {
        return d;
    } else if constexpr (idx == 16) {           // e^{-i pi/2} = -i
        return make_float2(d.y, -d.x);
    } else if constexpr (idx == 32) {
        return make_float2(-d.x, -d.y);
    } else if constexpr (idx == 48) {           // +i
        return make_float2(-d.y, d.x);
    } else {
        return c_mul(d, make_float2(cos64(idx), -sin64(idx)));
    }
}

// In-register radix-2 DIF DFT of length E (E | 32): v[brev_E(k)] = sum_e v_in[e] W_E^{e k}.
template <int E, int SPAN, int START, int I>
struct DifBfly {
    static __device__ __forceinline__ void run(float2 (&v)[E]) {
        float2 a = v[START + I], b = v[START + I + SPAN];
        v[START + I] = c_add(a, b);
        v[START + I + SPAN] = c_mul_w<2 * SPAN, I>(c_sub(a, b));
        if constexpr (I + 1 < SPAN) DifBfly<E, SPAN, START, I + 1>::run(v);
    }
};
template <int E, int SPAN, int START>
struct DifGroup {
    static __device__ __forceinline__ void run(float2 (&v)[E]) {
        DifBfly<E, SPAN, START, 0>::run(v);
        if constexpr (START + 2 * SPAN < E) DifGroup<E, SPAN, START + 2 * SPAN>::run(v);
    }
};
template <int E, int SPAN>
struct DifStage {
    static __device__ __forceinline__ void run(float2 (&v)[E]) {
        DifGroup<E, SPAN, 0>::run(v);
        if constexpr (SPAN > 1) DifStage<E, SPAN / 2>::run(v);
    }
};
template <int E>
__device__ __forceinline__ void dif_reg(float2 (&v)[E]) {
    if constexpr (E > 1) DifStage<E, E / 2>::run(v);
}

// In-register radix-4 DIF DFT of length E in {4, 8, 16} (fewer nontrivial twiddles than radix-2 for
// E = 16): stage 1 = 4-point DFTs over v[i + E/4 l] times W_E^{i m}, stored at i + (E/4) m; stage 2 =
// 4- (E = 16) or 2-point (E = 8) DFTs over i.  Output order: v[dpos4<E>(k)] = X[k].
template <int E>
__host__ __device__ constexpr int dpos4(int k) {
    return E == 16 ? 4 * (k & 3) + (k >> 2) : (E == 8 ? 2 * (k & 3) + (k >> 2) : k);
}
__device__ __forceinline__ void dft4_inplace(float2 &x0, float2 &x1, float2 &x2, float2 &x3) {
    const float2 a = c_add(x0, x2), b = c_sub(x0, x2), c = c_add(x1, x3), d = c_sub(x1, x3);
    x0 = c_add(a, c);
    x1 = c_add(b, make_float2(d.y, -d.x));                   // b - i d
    x2 = c_sub(a, c);
    x3 = c_add(b, make_float2(-d.y, d.x));                   // b + i d
}
template <int E, int I>
struct Dif4Stage1 {
    static constexpr int SP = E / 4;
    static __device__ __forceinline__ void run(float2 (&v)[E]) {
        float2 x0 = v[I], x1 = v[I + SP], x2 = v[I + 2 * SP], x3 = v[I + 3 * SP];
        dft4_inplace(x0, x1, x2, x3);
        v[I] = x0;
        v[I + SP] = c_mul_w<E, I>(x1);
        v[I + 2 * SP] = c_mul_w<E, 2 * I>(x2);
        v[I + 3 * SP] = c_mul_w<E, 3 * I>(x3);
        if constexpr (I + 1 < SP) Dif4Stage1<E, I + 1>::run(v);
    }
};
template <int E>
__device__ __forceinline__ void dif4(float2 (&v)[E]) {
    static_assert(E == 4 || E == 8 || E == 16, "dif4: E in {4, 8, 16}");
    Dif4Stage1<E, 0>::run(v);
    if constexpr (E == 16) {
#pragma unroll
        for (int m = 0; m < 4; ++m) dft4_inplace(v[4 * m], v[4 * m + 1], v[4 * m + 2], v[4 * m + 3]);
    } else if constexpr (E == 8) {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const float2 a = v[2 * m], b = v[2 * m + 1];
            v[2 * m] = c_add(a, b);
            v[2 * m + 1] = c_sub(a, b);
        }
    }
}

// Radix-2 DIF DFT of length L across the lanes of an L-lane group (lanes l ^ h exchange).
// stw[s] = W_{2h}^{l & (h-1)} for stage s (h = L/2 >> s), computed by lane_stage_twiddles.
template <int E, int L>
__device__ __forceinline__ void dif_lanes(float2 (&v)[E], int l, const float2 (&stw)[clog2(L) > 0 ? clog2(L) : 1]) {
    // Select-free butterfly: lower lanes v + p, upper lanes (p - v) * tw, written as
    // (p + sgn v) * tw' with per-lane sgn = -1 / +1 and tw' = tw / 1.  The last stage (h = 1) has
    // tw = W_2^0 = 1 on every lane, so its multiply is skipped.
#pragma unroll
    for (int s = 0; s < clog2(L); ++s) {
        const int h = (L >> 1) >> s;
        const bool upper = (l & h) != 0;
        const float sgn = upper ? -1.f : 1.f;
        const float2 tw = upper ? stw[s] : make_float2(1.f, 0.f);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            float2 p;
            p.x = __shfl_xor_sync(0xffffffffu, v[e].x, h);
            p.y = __shfl_xor_sync(0xffffffffu, v[e].y, h);
            const float2 t = make_float2(fmaf(sgn, v[e].x, p.x), fmaf(sgn, v[e].y, p.y));
            v[e] = (h == 1) ? t : c_mul(t, tw);
        }
    }
}

template <int L>
__device__ __forceinline__ void lane_stage_twiddles(int l, float2 (&stw)[clog2(L) > 0 ? clog2(L) : 1]) {
#pragma unroll
    for (int s = 0; s < clog2(L); ++s) {
        const int h = (L >> 1) >> s;
        float sn, cs;
        sincospif((float)(l & (h - 1)) / (float)h, &sn, &cs);   // e^{-i pi j / h} = W_{2h}^j
        stw[s] = make_float2(cs, -sn);
    }
    if constexpr (clog2(L) == 0) stw[0] = make_float2(1.f, 0.f);
}

// W_N^{(l * k1) mod N} for k1 < E, stored at tw[k1 * L + l] (N = L * E).
__device__ __forceinline__ float2 twiddle_N(int l, int k1, int N) {
    float sn, cs;
    sincospif(2.0f * (float)((l * k1) & (N - 1)) / (float)N, &sn, &cs);
    return make_float2(cs, -sn);
}

// Full distributed forward FFT (see file header).  twN: pointer to this lane's column of the
// (k1, l) twiddle table (stride L), typically in shared memory.
template <int E, int L>
__device__ __forceinline__ void fft_dist(float2 (&v)[E], int l, const float2 *__restrict__ twN,
                                         const float2 (&stw)[clog2(L) > 0 ? clog2(L) : 1]) {
    dif_reg<E>(v);
#pragma unroll
    for (int k1 = 1; k1 < E; ++k1) {
        const int r = brev(k1, clog2(E));
        v[r] = c_mul(v[r], twN[k1 * L + l]);
    }
    dif_lanes<E, L>(v, l, stw);
}

}  // namespace rsvd
