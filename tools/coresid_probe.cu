// Probe: can a cluster kernel (2-CTA clusters, 192 threads, 168 regs, ~67 KB smem) and a plain kernel
// (256 threads, 128 regs, ~134 KB smem) run on the same SMs at the same time?  Each CTA spins for a
// fixed time and records (smid, start, end) from %globaltimer.
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ unsigned smid() { unsigned s; asm volatile("mov.u32 %0, %smid;" : "=r"(s)); return s; }
template <int TAG>
__device__ void spin(unsigned long long *rec, unsigned long long ns) {
    extern __shared__ unsigned char sm[];
    if (threadIdx.x == 0) {
        unsigned long long t0 = gt();
        sm[0] = 1;
        while (gt() - t0 < ns) {}
        rec[blockIdx.x * 3 + 0] = smid(); rec[blockIdx.x * 3 + 1] = t0; rec[blockIdx.x * 3 + 2] = gt();
    }
    __syncthreads();
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 2) kA(unsigned long long *rec, unsigned long long ns) { spin<0>(rec, ns); }
__global__ void __launch_bounds__(256, 2) kB(unsigned long long *rec, unsigned long long ns) { spin<1>(rec, ns); }
int main(int argc, char **argv) {
    int smemA = argc > 1 ? atoi(argv[1]) : 66816, smemB = argc > 2 ? atoi(argv[2]) : 134232, carve = argc > 3 ? atoi(argv[3]) : -1;
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(kA, cudaFuncAttributeMaxDynamicSharedMemorySize, smemA);
    cudaFuncSetAttribute(kB, cudaFuncAttributeMaxDynamicSharedMemorySize, smemB);
    if (carve >= 0) {
        cudaFuncSetAttribute(kA, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
        cudaFuncSetAttribute(kB, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
    }
    unsigned long long *ra, *rb; cudaMalloc(&ra, nsm * 24); cudaMalloc(&rb, nsm * 24);
    cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    const unsigned long long ns = 2000000;   // 2 ms
    for (int rep = 0; rep < 2; ++rep) {
        kB<<<nsm, 256, smemB, s2>>>(rb, ns);
        kA<<<nsm, 192, smemA, s1>>>(ra, ns);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    }
    std::vector<unsigned long long> a(nsm * 3), b(nsm * 3);
    cudaMemcpy(a.data(), ra, nsm * 24, cudaMemcpyDeviceToHost); cudaMemcpy(b.data(), rb, nsm * 24, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, aend = 0, bend = 0, astart = ~0ull;
    for (int i = 0; i < nsm; ++i) { t0 = std::min(t0, std::min(a[3*i+1], b[3*i+1])); }
    for (int i = 0; i < nsm; ++i) { aend = std::max(aend, a[3*i+2]); bend = std::max(bend, b[3*i+2]); astart = std::min(astart, a[3*i+1]); }
    int same = 0;
    for (int i = 0; i < nsm; ++i) for (int j = 0; j < nsm; ++j)
        if (a[3*i] == b[3*j] && a[3*i+1] < b[3*j+2] && b[3*j+1] < a[3*i+2]) { ++same; break; }
    printf("smemA %d smemB %d carve %d: B ends %.2f ms, A starts %.2f ms, A ends %.2f ms; A CTAs overlapping a B CTA on the same SM: %d / %d\n",
           smemA, smemB, carve, (bend - t0) * 1e-6, (astart - t0) * 1e-6, (aend - t0) * 1e-6, same, nsm);
    return 0;
}
