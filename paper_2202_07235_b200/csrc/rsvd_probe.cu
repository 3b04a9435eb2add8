// rsvd_probe.cu -- measured FP32 peak of this GPU for the roofline denominators (SURVEY.md 8(d):
// "Pi_fp32 is measured on the box (sustained FFMA microbenchmark)").  Not part of the method.
//
// Every thread runs NCH independent dependency chains of the probed instruction on register operands
// (no memory traffic inside the loop), on 4 resident CTAs x 256 threads per SM.  The sustained rate is
// flops / elapsed time over a launch long enough (~100 ms) to settle under the power cap.
//   kind 0  FFMA  (scalar, 3-register form)        2 flops per lane per instruction
//   kind 1  FFMA2 (sm_100 packed fp32x2)           4 flops per lane per instruction
//   kind 2  FADD2 (sm_100 packed fp32x2 add)        2 flops per lane per instruction
//   kind 3  DFMA  (fp64)                            2 flops per lane per instruction (kernel-partials peak)
//   kind 4  DMMA  mma.sync m8n8k4 f64 (tensor core)  512 flops per warp per instruction
//   kind 5  DMMA  mma.sync m16n8k4 f64 (tensor core) 1024 flops per warp per instruction
#include <cuda_runtime.h>

#include "rsvd_common.cuh"

namespace rsvd {

constexpr int PR_THREADS = 256;
constexpr int PR_NCH = 8;

template <int KIND>
__global__ void __launch_bounds__(PR_THREADS) fp32_probe_kernel(int iters, float seed, float *__restrict__ sink) {
    float2 acc[PR_NCH];
    const float2 a = make_float2(seed * 1e-3f + 0.999f, 1.0001f - seed * 1e-3f);
    const float2 b = make_float2(seed * 1e-7f, -seed * 1e-7f);
#pragma unroll
    for (int c = 0; c < PR_NCH; ++c) acc[c] = make_float2((float)(threadIdx.x + c), (float)(blockIdx.x - c));
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int c = 0; c < PR_NCH; ++c) {
                if constexpr (KIND == 0) {
                    acc[c].x = fmaf(acc[c].x, a.x, b.x);
                    acc[c].y = fmaf(acc[c].y, a.y, b.y);
                } else if constexpr (KIND == 1) {
                    acc[c] = __ffma2_rn(acc[c], a, b);
                } else {
                    acc[c] = __fadd2_rn(acc[c], b);
                }
            }
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < PR_NCH; ++c) s += acc[c].x + acc[c].y;
    if (s == 1234.5678f) sink[threadIdx.x] = s;      // never true in practice; keeps the chains live
}

__global__ void __launch_bounds__(PR_THREADS) fp64_probe_kernel(int iters, double seed, double *__restrict__ sink) {
    double acc[2 * PR_NCH];
    const double a = seed * 1e-3 + 0.999, b = seed * 1e-7;
#pragma unroll
    for (int c = 0; c < 2 * PR_NCH; ++c) acc[c] = (double)(threadIdx.x + c);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int c = 0; c < 2 * PR_NCH; ++c) acc[c] = fma(acc[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 2 * PR_NCH; ++c) s += acc[c];
    if (s == 1234.5678) sink[threadIdx.x] = s;
}

// fp64 tensor-core probe: NCH independent accumulator fragments per warp, A/B fragments in registers
template <int SHAPE>   // 0: m8n8k4, 1: m16n8k4
__global__ void __launch_bounds__(PR_THREADS) dmma_probe_kernel(int iters, double seed, double *__restrict__ sink) {
    constexpr int NC = SHAPE == 0 ? 2 : 4;           // accumulator doubles per lane
    double acc[PR_NCH][NC];
    const double a0 = seed * 1e-3 + 0.999 + 1e-9 * threadIdx.x, a1 = 1.0001 - seed * 1e-3, b0 = seed * 1e-7;
#pragma unroll
    for (int c = 0; c < PR_NCH; ++c)
#pragma unroll
        for (int i = 0; i < NC; ++i) acc[c][i] = (double)(threadIdx.x + c + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int c = 0; c < PR_NCH; ++c) {
                if constexpr (SHAPE == 0) {
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                                 : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a0), "d"(b0));
                } else {
                    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0, %1, %2, %3}, {%4, %5}, {%6}, {%0, %1, %2, %3};"
                                 : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                                 : "d"(a0), "d"(a1), "d"(b0));
                }
            }
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < PR_NCH; ++c)
#pragma unroll
        for (int i = 0; i < NC; ++i) s += acc[c][i];
    if (s == 1234.5678) sink[threadIdx.x] = s;
}

template <int KIND>
static cudaError_t run_probe(int iters, cudaStream_t st, float *sink, float *ms) {
    const int grid = num_sms() * 4;
    cudaEvent_t e0, e1;
    cudaError_t e = cudaEventCreate(&e0);
    if (e != cudaSuccess) return e;
    if ((e = cudaEventCreate(&e1)) != cudaSuccess) { cudaEventDestroy(e0); return e; }
    if constexpr (KIND == 4 || KIND == 5) {
        dmma_probe_kernel<KIND - 4><<<grid, PR_THREADS, 0, st>>>(iters / 16, 0.5, reinterpret_cast<double *>(sink));
        cudaEventRecord(e0, st);
        dmma_probe_kernel<KIND - 4><<<grid, PR_THREADS, 0, st>>>(iters, 0.5, reinterpret_cast<double *>(sink));
    } else if constexpr (KIND == 3) {
        fp64_probe_kernel<<<grid, PR_THREADS, 0, st>>>(iters / 16, 0.5, reinterpret_cast<double *>(sink));
        cudaEventRecord(e0, st);
        fp64_probe_kernel<<<grid, PR_THREADS, 0, st>>>(iters, 0.5, reinterpret_cast<double *>(sink));
    } else {
        fp32_probe_kernel<KIND><<<grid, PR_THREADS, 0, st>>>(iters / 16, 0.5f, sink);      // warm-up
        cudaEventRecord(e0, st);
        fp32_probe_kernel<KIND><<<grid, PR_THREADS, 0, st>>>(iters, 0.5f, sink);
    }
    cudaEventRecord(e1, st);
    e = cudaEventSynchronize(e1);
    if (e == cudaSuccess) e = cudaEventElapsedTime(ms, e0, e1);
    if (e == cudaSuccess) e = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return e;
}

}  // namespace rsvd

extern "C" rsvd_status rsvd_probe_fp32(int32_t kind, int32_t iters, double *tflops, rsvd_stream_t stream) {
    using namespace rsvd;
    if (kind < 0 || kind > 5 || iters < 16 || !tflops) return fail(RSVD_ERR_ARG, "bad probe arguments");
    float *sink = nullptr;
    cudaError_t e = cudaMalloc(&sink, PR_THREADS * sizeof(double));
    if (e != cudaSuccess) return cuda_check(e, "probe sink");
    float ms = 0.f;
    cudaStream_t s = (cudaStream_t)stream;
    e = kind == 0 ? run_probe<0>(iters, s, sink, &ms)
      : kind == 1 ? run_probe<1>(iters, s, sink, &ms)
      : kind == 2 ? run_probe<2>(iters, s, sink, &ms) : kind == 3 ? run_probe<3>(iters, s, sink, &ms)
      : kind == 4 ? run_probe<4>(iters, s, sink, &ms) : run_probe<5>(iters, s, sink, &ms);
    cudaFree(sink);
    if (e != cudaSuccess) return cuda_check(e, "fp32 probe");
    const double lanes = (double)num_sms() * 4 * PR_THREADS;
    // flops per thread per iter (DMMA: a warp instruction's 2 M N K flops spread over its 32 lanes)
    const double per_iter = 4.0 * PR_NCH * (kind == 2 ? 2.0 : kind == 4 ? 512.0 / 32 : kind == 5 ? 1024.0 / 32 : 4.0);
    *tflops = lanes * (double)iters * per_iter / (ms * 1e-3) / 1e12;
    count_launches(2);
    return RSVD_OK;
}
