// TMA 2-D load throughput probe: a row-major fp32 matrix (n x 256, 2 GB) is streamed through a
// ring of S shared-memory stages by one producer thread per CTA (one CTA per SM); a consumer
// warp frees each stage as soon as it lands.  Box shapes: {32 cols x 128 rows} (the oz kernel's
// K chunk), {64 x 64}, {128 x 32}, {256 x 16}; swizzle 128B.  Prints GB/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_rate tma_rate.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.b32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(bar), "r"(par) : "memory");
}

__global__ void __launch_bounds__(64, 1) tma_stream(const __grid_constant__ CUtensorMap map, int bx, int by, int ncol,
                                                    int nrow, int S) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t full[16], empty[16];
    const int stage = bx * by * 4;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int tiles_x = ncol / bx, tiles_y = nrow / by;
    const long long total = (long long)tiles_x * tiles_y;
    // each CTA walks its row bands: (row band, col chunk) in row-band-major order
    if (threadIdx.x == 0) {
        long long g = 0;
        for (long long t = blockIdx.x; t < tiles_y; t += gridDim.x)
            for (int c = 0; c < tiles_x; ++c, ++g) {
                const int s = (int)(g % S);
                if (g >= S) wait(su32(&empty[s]), (uint32_t)(((g / S) - 1) & 1));
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(stage) : "memory");
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                                 su32(sm + s * stage)),
                             "l"(&map), "r"(su32(&full[s])), "r"(c * bx), "r"((int)(t * by))
                             : "memory");
            }
    } else if (threadIdx.x == 32) {
        long long g = 0;
        for (long long t = blockIdx.x; t < tiles_y; t += gridDim.x)
            for (int c = 0; c < tiles_x; ++c, ++g) {
                const int s = (int)(g % S);
                wait(su32(&full[s]), (uint32_t)((g / S) & 1));
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
            }
    }
    (void)total;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const long long n = 2000000, K = 256;
    float *A;
    cudaMalloc(&A, n * K * 4);
    cudaMemset(A, 0, n * K * 4);
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)p;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int shapes[3][2] = {{32, 64}, {32, 128}, {32, 256}};
    for (auto &sh : shapes) {
        const int bx = sh[0], by = sh[1];
        for (int S : {2, 4, 8}) {
            CUtensorMap m;
            const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)n};
            const cuuint64_t str[1] = {(cuuint64_t)K * 4};
            const cuuint32_t box[2] = {(cuuint32_t)(bx > 32 ? 32 : bx), (cuuint32_t)by};
            const cuuint32_t es[2] = {1, 1};
            // the 128B swizzle limits the inner box to 128 bytes: wider boxes are issued as bx/32 loads
            if (bx > 32) continue;
            enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, A, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            const int smem = S * bx * by * 4;
            cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            tma_stream<<<sms, 64, smem>>>(m, bx, by, (int)K, (int)n, S);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            tma_stream<<<sms, 64, smem>>>(m, bx, by, (int)K, (int)n, S);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("box %3d x %3d  stages %2d (%3d KB in flight): %.3f ms  %.0f GB/s  %s\n", bx, by, S, smem / 1024, ms,
                   n * K * 4 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
