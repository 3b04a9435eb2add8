// tc_probe.cu -- standalone validation of the tcgen05 building blocks used by the TF32 contraction:
// K-major SWIZZLE_128B smem operands + UMMA descriptors, tcgen05.alloc / mma.kind::tf32 / commit to
// an mbarrier / tcgen05.ld 32x32b, on one 128 x N x K tile.  D[m][n] = sum_k A[m][k] B[n][k].
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -shared -Xcompiler -fPIC tools/tc_probe.cu -o tools/libtcprobe.so
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFF) >> 4);          // start address
    d |= (uint64_t)1 << 16;                           // LBO (ignored for swizzled K-major) = 1
    d |= (uint64_t)(1024 >> 4) << 32;                 // SBO = 1024 B between 8-row atoms
    d |= (uint64_t)1 << 46;                           // version = 1 (sm100)
    d |= (uint64_t)2 << 61;                           // SWIZZLE_128B
    return d;
}

template <int N>
__global__ void __launch_bounds__(128, 1) tc_probe_kernel(const float *A, const float *B, float *D, int K) {
    extern __shared__ __align__(1024) unsigned char smem[];
    // layout: A tiles [KB][128 rows][128 B], B tiles [KB][N rows][128 B], then mbarrier + tmem addr
    const int KB = K / 32;
    unsigned char *sA = smem;
    unsigned char *sB = smem + (size_t)KB * 128 * 128;
    uint64_t *mbar = reinterpret_cast<uint64_t *>(sB + (size_t)KB * N * 128);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(mbar + 1);
    const int tid = threadIdx.x, warp = tid >> 5;

    // fill swizzled tiles: element (r, k) -> r*128 + ((k/4) ^ (r&7))*16 + (k%4)*4 within k-block k/32
    for (int i = tid; i < 128 * K; i += 128) {
        const int r = i / K, k = i % K;
        const int kb = k / 32, kk = k % 32;
        float *dst = reinterpret_cast<float *>(sA + (size_t)kb * 128 * 128 + r * 128 + (((kk >> 2) ^ (r & 7)) << 4)) + (kk & 3);
        *dst = A[i];
    }
    for (int i = tid; i < N * K; i += 128) {
        const int r = i / K, k = i % K;
        const int kb = k / 32, kk = k % 32;
        float *dst = reinterpret_cast<float *>(sB + (size_t)kb * N * 128 + r * 128 + (((kk >> 2) ^ (r & 7)) << 4)) + (kk & 3);
        *dst = B[i];
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(1));
    }
    // make generic-proxy smem writes visible to the async proxy (tensor core)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    constexpr uint32_t NCOLS = N < 32 ? 32 : N;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(NCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (tid == 0) {
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        for (int kb = 0; kb < KB; ++kb) {
            const uint64_t da = sw128_desc(smem_u32(sA + (size_t)kb * 128 * 128));
            const uint64_t db = sw128_desc(smem_u32(sB + (size_t)kb * N * 128));
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const uint32_t acc = (kb | s) ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\t"
                    "setp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                    "l"(da + (uint64_t)(2 * s)), "l"(db + (uint64_t)(2 * s)), "r"(idesc), "r"(acc));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(mbar)));
    }
    // wait for the MMAs (phase 0)
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}\n"
                : "=r"(done)
                : "r"(smem_u32(mbar)), "r"(0));
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    // each warp reads its 32 TMEM lanes (rows 32w..32w+31), 32 columns at a time
    const int row = warp * 32 + (tid & 31);
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 32; ++j) D[(size_t)row * N + c0 + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(NCOLS));
}

extern "C" int tc_probe(const float *A, const float *B, float *D, int K, int N) {
    const size_t smem = (size_t)(K / 32) * (128 + N) * 128 + 64;
    cudaError_t e;
    if (N == 256) {
        cudaFuncSetAttribute(tc_probe_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        tc_probe_kernel<256><<<1, 128, smem>>>(A, B, D, K);
    } else if (N == 128) {
        cudaFuncSetAttribute(tc_probe_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        tc_probe_kernel<128><<<1, 128, smem>>>(A, B, D, K);
    } else {
        return -1;
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
    e = cudaDeviceSynchronize();
    return (int)e;
}
