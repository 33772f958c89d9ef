// tcgen05.mma kind::i8 throughput probe: one CTA per SM issues back-to-back MMAs (M = 128,
// K = 32, N = 64 / 128 / 256) from fixed shared-memory operands (no-swizzle K-major and
// 32-byte-swizzle K-major layouts) into TMEM, then one commit.  Reports int8 TOPS (2 ops/MAC).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o imma_rate imma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((addr & 0x3FFFF) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

__global__ void __launch_bounds__(128, 1) imma_loop(int iters, int N, int layout, int *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = i * 2654435761u;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint32_t a = su32(sm), b = su32(sm + 32768);
        // layout 0: no swizzle (LBO 128 between the two K core matrices, SBO 256 between 8-row groups);
        // layout 6: 32-byte swizzle (32-byte rows, SBO 256)
        const uint64_t da = layout == 0 ? desc(a, 128, 256, 0) : desc(a, 16, 256, 6);
        const uint64_t db = layout == 0 ? desc(b, 128, 256, 0) : desc(b, 16, 256, 6);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t d = tmem + (uint32_t)((u & 1) * 256);
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                             "l"(da), "l"(db), "r"(idesc), "r"(1));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.b32 %0, 1, 0, p;\n}\n"
                         : "=r"(done) : "r"(su32(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
    if (threadIdx.x == 0 && iters < 0) out[0] = 1;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int *o;
    cudaMalloc(&o, 4);
    cudaFuncSetAttribute(imma_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int iters = 4000;
    for (int layout : {0, 6}) {
        for (int N : {64, 128, 256}) {
            imma_loop<<<sms, 128, 100 * 1024>>>(10, N, layout, o);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            imma_loop<<<sms, 128, 100 * 1024>>>(iters, N, layout, o);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ops = 2.0 * 128.0 * N * 32.0 * 8.0 * iters * sms;
            printf("layout %d N %3d: %.0f TOPS (%s)\n", layout, N, ops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
