// Gather-bandwidth probe: warps read random 512-byte rows (one float4 per lane, 8 rows in
// flight per warp) from a table of a given size -- the access pattern of the propagation
// SpMM's column slice.  Tables below L2 capacity measure the L2 -> SM gather ceiling, larger
// ones the DRAM gather ceiling.  Prints GB/s of gathered bytes.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void gather(const float4 *__restrict__ tab, const int *__restrict__ idx, long long E, float4 *out) {
    const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    float4 acc = make_float4(0, 0, 0, 0);
    for (long long e0 = w * 32; e0 < E; e0 += nw * 32) {
        const int my = idx[e0 + lane];
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(tab + (long long)__shfl_sync(~0u, my, j + u) * 32 + lane);
#pragma unroll
            for (int u = 0; u < 8; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
        }
    }
    if (acc.x == 123.456f) out[0] = acc;
}

int main() {
    const long long E = 1 << 24;
    int *idx;
    cudaMalloc(&idx, E * 4);
    float4 *out;
    cudaMalloc(&out, 16);
    const long long sizes_mb[] = {8, 32, 64, 96, 256, 1024, 4096};
    for (long long mb : sizes_mb) {
        const long long rows = mb * (1 << 20) / 512;
        float4 *tab;
        if (cudaMalloc(&tab, rows * 512) != cudaSuccess) break;
        cudaMemset(tab, 0, rows * 512);
        std::vector<int> h(E);
        unsigned long long s = 88172645463325252ull;
        for (long long i = 0; i < E; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (int)(s % rows); }
        cudaMemcpy(idx, h.data(), E * 4, cudaMemcpyHostToDevice);
        for (int bpsm : {4, 8}) {
            const int blocks = 148 * bpsm;
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            gather<<<blocks, 256>>>(tab, idx, E, out);
            cudaEventRecord(a);
            for (int it = 0; it < 5; ++it) gather<<<blocks, 256>>>(tab, idx, E, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("table %5lld MB  blocks/SM %d : %.1f GB/s gathered\n", mb, bpsm, 5.0 * E * 512 / (ms * 1e6));
        }
        cudaFree(tab);
    }
    return 0;
}
