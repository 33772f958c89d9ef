// FP64 throughput probe: DFMA (CUDA cores) vs DMMA (mma.sync m8n8k4 f64).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double *out, int iters) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    const double b = 1.0000001, c = 1e-9;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 12345.0) out[0] = s;
}

__global__ void dmma_loop(double *out, int iters) {
    double acc[8][2];
    for (int j = 0; j < 8; ++j)
        for (int i = 0; i < 2; ++i) acc[j][i] = 0.0;
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[j][0]), "+d"(acc[j][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
    for (int j = 0; j < 8; ++j)
        for (int i = 0; i < 2; ++i) s += acc[j][i];
    if (s == 12345.0) out[0] = s;
}

int main() {
    double *o;
    cudaMalloc(&o, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 20000;
    for (int bps : {4, 8}) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        dfma_loop<<<sms * bps, 256>>>(o, 100);
        cudaEventRecord(e0);
        dfma_loop<<<sms * bps, 256>>>(o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 8 * iters * (double)sms * bps * 256;
        printf("DFMA blocks/SM %d: %.1f TFLOP/s\n", bps, fl / ms / 1e9);
        dmma_loop<<<sms * bps, 256>>>(o, 100);
        cudaEventRecord(e0);
        dmma_loop<<<sms * bps, 256>>>(o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        fl = 2.0 * 8 * 8 * 4 * 8 * iters * (double)sms * bps * 256 / 32;
        printf("DMMA blocks/SM %d: %.1f TFLOP/s\n", bps, fl / ms / 1e9);
    }
    return 0;
}
