// Gather probe on a real CSR pattern: warps gather 512-byte row slices of a table in the order
// of a CSR column-index array (one float4 per lane, 8 rows in flight per warp, slice-major like
// the propagation SpMM), with no epilogue.  Gives the gather ceiling of the graph's own access
// pattern (L2 locality of the real degree distribution) to compare the SpMM against.
// usage: gather_csr <col_idx.bin (int32)> <table_rows> <d (floats)>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void gather(const float4 *__restrict__ tab, const int *__restrict__ idx, long long E, int d4, int nsl,
                       float4 *out, unsigned long long *work) {
    const int lane = threadIdx.x & 31;
    float4 acc = make_float4(0, 0, 0, 0);
    const long long nchunks = (E + 31) / 32;
    while (true) {
        unsigned long long u = 0;
        if (lane == 0) u = atomicAdd(work, 1ull);
        u = __shfl_sync(~0u, u, 0);
        if ((long long)u >= nchunks * nsl) break;
        const int sl = (int)(u / nchunks);
        const long long e0 = (long long)(u % nchunks) * 32;
        const int cnt = (int)min(32LL, E - e0);
        const int my = idx[e0 + (lane < cnt ? lane : 0)];
        const float4 *base = tab + sl * 32 + lane;
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
            float4 v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = __ldg(base + (long long)__shfl_sync(~0u, my, j + q) * d4);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (j + q < cnt) { acc.x += v[q].x; acc.y += v[q].y; acc.z += v[q].z; acc.w += v[q].w; }
        }
    }
    if (acc.x == 123.456f) out[0] = acc;
}

int main(int argc, char **argv) {
    if (argc < 4) { fprintf(stderr, "usage: %s col_idx.bin rows d\n", argv[0]); return 1; }
    FILE *f = fopen(argv[1], "rb");
    fseek(f, 0, SEEK_END);
    const long long E = ftell(f) / 4;
    fseek(f, 0, SEEK_SET);
    std::vector<int> h(E);
    if (fread(h.data(), 4, E, f) != (size_t)E) return 1;
    fclose(f);
    const long long rows = atoll(argv[2]);
    const int d = atoi(argv[3]), d4 = d / 4, nsl = (d4 + 31) / 32;
    int *idx; float4 *tab, *out; unsigned long long *work;
    cudaMalloc(&idx, E * 4); cudaMalloc(&tab, rows * d * 4); cudaMalloc(&out, 16); cudaMalloc(&work, 8);
    cudaMemcpy(idx, h.data(), E * 4, cudaMemcpyHostToDevice);
    cudaMemset(tab, 0, rows * d * 4);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int bps : {4, 8}) {
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        float best = 1e9;
        for (int it = 0; it < 6; ++it) {
            cudaMemset(work, 0, 8);
            cudaEventRecord(a);
            gather<<<sms * bps, 256>>>(tab, idx, E, d4, nsl, out, work);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (it > 0 && ms < best) best = ms;
        }
        const double bytes = (double)E * nsl * 512.0;
        printf("E=%lld rows=%lld d=%d blocks/SM %d: %.3f ms  %.1f GB/s gathered\n", E, rows, d, bps, best, bytes / best / 1e6);
    }
    return 0;
}
