// L2 bandwidth probe: grid-strided 16-B loads / stores over an L2-resident buffer (default 48 MB),
// repeated; reports GB/s for read, write and 50/50 read+write.  Used to put the contraction's
// operand-read + spectrum-store traffic against a measured L2 ceiling.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void rd(const float4 *__restrict__ p, size_t n, int reps, float *sink) {
    float acc = 0.f;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            float4 v = __ldcg(p + i);
            acc += v.x + v.y + v.z + v.w;
        }
    if (acc == 1234.5f) *sink = acc;
}
__global__ void wr(float4 *__restrict__ p, size_t n, int reps) {
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
            __stcg(p + i, make_float4(r, i, 0, 1));
}
__global__ void rw(const float4 *__restrict__ a, float4 *__restrict__ b, size_t n, int reps) {
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            float4 v = __ldcg(a + i);
            v.x += 1.f;
            __stcg(b + i, v);
        }
}
int main(int argc, char **argv) {
    size_t mb = argc > 1 ? atoi(argv[1]) : 48;
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    size_t n = mb * (1 << 20) / 16;
    float4 *a, *b; float *sink;
    cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16); cudaMalloc(&sink, 4);
    cudaMemset(a, 0, n * 16); cudaMemset(b, 0, n * 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int reps = 20, blocks = nsm * 4, thr = 512;
    for (int k = 0; k < 3; ++k) {
        float ms;
        double bytes;
        rd<<<blocks, thr>>>(a, n, 2, sink);
        cudaEventRecord(e0); rd<<<blocks, thr>>>(a, n, reps, sink); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1); bytes = (double)n * 16 * reps;
        printf("%zu MB read  %8.1f GB/s\n", mb, bytes / ms * 1e-6);
        wr<<<blocks, thr>>>(b, n, 2);
        cudaEventRecord(e0); wr<<<blocks, thr>>>(b, n, reps); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%zu MB write %8.1f GB/s\n", mb, bytes / ms * 1e-6);
        rw<<<blocks, thr>>>(a, b, n / 2, 2);
        cudaEventRecord(e0); rw<<<blocks, thr>>>(a, b, n / 2, reps); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%zu MB r+w   %8.1f GB/s (read + write bytes)\n", mb, bytes / ms * 1e-6);
    }
    return 0;
}
// (appended) 4-byte coalesced stores and 1-D bulk (TMA) stores from shared memory
__global__ void wr4(float *__restrict__ p, size_t n, int reps) {
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
            __stcg(p + i, (float)r);
}
__global__ void wrbulk(char *__restrict__ p, size_t bytes, int reps, int chunk) {
    extern __shared__ __align__(128) char sb[];
    for (int i = threadIdx.x; i < chunk / 4; i += blockDim.x) reinterpret_cast<float *>(sb)[i] = (float)i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned s = (unsigned)__cvta_generic_to_shared(sb);
        for (int r = 0; r < reps; ++r)
            for (size_t off = (size_t)blockIdx.x * chunk; off + chunk <= bytes; off += (size_t)gridDim.x * chunk) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + off), "r"(s), "r"(chunk) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
            }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}
int main2(size_t mb) {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    size_t n = mb * (1 << 20) / 4;
    float *b; cudaMalloc(&b, n * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int reps = 20;
    cudaFuncSetAttribute(wrbulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int k = 0; k < 2; ++k) {
        float ms;
        const double bytes = (double)n * 4 * reps;
        wr4<<<nsm * 4, 512>>>(b, n, 2);
        cudaEventRecord(e0); wr4<<<nsm * 4, 512>>>(b, n, reps); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%zu MB write (4-B lanes)   %8.1f GB/s\n", mb, bytes / ms * 1e-6);
        for (int chunk : {4096, 16384}) {
            wrbulk<<<nsm, 32, chunk>>>((char *)b, n * 4, 2, chunk);
            cudaEventRecord(e0); wrbulk<<<nsm, 32, chunk>>>((char *)b, n * 4, reps, chunk); cudaEventRecord(e1); cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("%zu MB write (bulk %5d B) %8.1f GB/s  %s\n", mb, chunk, bytes / ms * 1e-6, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
struct Run2 { Run2() { const char *e = getenv("PROBE2"); if (e) { main2(atoi(e)); exit(0); } } } run2;
