// a5: random features of Alg. 1 L8-9 (Eq. R-prime; Eq. Ri, 466-468).
//
//   features_tc (gram_tc.cu): Zo = sqrt(d) Zhat Q^T on tcgen05 with 3xTF32 splitting
//     (fp32-accurate), epilogue R' = sqrt(e/d) (sin Zo || cos Zo) (accurate sincosf, the
//     arguments reach sqrt(d)) straight from TMEM.
//   colsum(4)_part_kernel + colsum_reduce_wide_kernel: r = sum_i R'[i] in fp64, fixed row ranges per
//     block and a fixed-order sum over blocks.
//   dinv_kernel: dinv_i = 1 / sqrt(max(R'[i] . r, 1e-12)) with r (fp64) staged in smem.
#include <algorithm>

#include "tpo_internal.cuh"

namespace tpo {
namespace {

constexpr int BM = 128, BN = 64;            // row / column granularity of the column-sum split
constexpr int ROW_GROUPS_MAX = 148 * 2;

// per-block fp64 column sums of R' over a fixed row range: grid (row groups, column blocks of
// 256), one column per thread, 4 independent accumulators over the rows (combined in order)
__global__ void colsum_part_kernel(const float *__restrict__ Rp, int64_t n, int D, int64_t rows_per,
                                   double *__restrict__ part) {
    const int j = blockIdx.y * blockDim.x + threadIdx.x;
    if (j >= D) return;
    const int64_t r0 = blockIdx.x * rows_per, r1 = min(n, r0 + rows_per);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int64_t i = r0;
    for (; i + 3 < r1; i += 4) {
        s0 += (double)Rp[i * D + j];
        s1 += (double)Rp[(i + 1) * D + j];
        s2 += (double)Rp[(i + 2) * D + j];
        s3 += (double)Rp[(i + 3) * D + j];
    }
    for (; i < r1; ++i) s0 += (double)Rp[i * D + j];
    part[blockIdx.x * (int64_t)D + j] = (s0 + s1) + (s2 + s3);
}

// the same partial column sums with 16-byte loads (D % 4 == 0): a thread owns 4 columns and the rows
// r0 + q, r0 + q + RL, ... of its block's range (q = its row lane), 8 rows in flight, summed in row
// order; the RL row lanes are combined in lane order (fixed, deterministic)
constexpr int CS4_RL = 4;
__global__ void __launch_bounds__(256) colsum4_part_kernel(const float4 *__restrict__ Rp4, int64_t n, int D4,
                                                           int64_t rows_per, double *__restrict__ part) {
    __shared__ double sm[CS4_RL][256][4];
    const int cq = threadIdx.x % 64, q = threadIdx.x / 64;       // column quad within a 256-column block
    const int j4 = blockIdx.y * 64 + cq;
    const int64_t r0 = blockIdx.x * rows_per, r1 = min(n, r0 + rows_per);
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    if (j4 < D4) {
        int64_t i = r0 + q;
        for (; i + 7 * CS4_RL < r1; i += 8 * CS4_RL) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = Rp4[(i + u * CS4_RL) * D4 + j4];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                s[0] += (double)v[u].x;
                s[1] += (double)v[u].y;
                s[2] += (double)v[u].z;
                s[3] += (double)v[u].w;
            }
        }
        for (; i < r1; i += CS4_RL) {
            const float4 v = Rp4[i * D4 + j4];
            s[0] += (double)v.x;
            s[1] += (double)v.y;
            s[2] += (double)v.z;
            s[3] += (double)v.w;
        }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) sm[q][cq][e] = s[e];
    __syncthreads();
    if (q == 0 && j4 < D4)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            double t = sm[0][cq][e];
#pragma unroll
            for (int qq = 1; qq < CS4_RL; ++qq) t += sm[qq][cq][e];
            part[blockIdx.x * (int64_t)(4 * D4) + 4 * j4 + e] = t;
        }
}

// r[j] = sum_g part[g][j] for many partials: 32 columns x 32 partial lanes per block, lane l sums
// g = l, l + 32, ... in order, the 32 lane sums are added in lane order (fixed, deterministic)
__global__ void __launch_bounds__(1024) colsum_reduce_wide_kernel(const double *__restrict__ part, int G, int D,
                                                                  double *__restrict__ r) {
    __shared__ double sm[32][33];
    const int c = threadIdx.x & 31, l = threadIdx.x >> 5;
    const int j = blockIdx.x * 32 + c;
    double s = 0.0;
    if (j < D)
        for (int g = l; g < G; g += 32) s += part[(int64_t)g * D + j];
    sm[l][c] = s;
    __syncthreads();
    if (l == 0 && j < D) {
        double t = sm[0][c];
        for (int q = 1; q < 32; ++q) t += sm[q][c];
        r[j] = t;
    }
}


__global__ void dinv_kernel(const float *__restrict__ Rp, int64_t n, int D, const double *__restrict__ r,
                            float *__restrict__ dinv) {
    extern __shared__ double rsh[];
    for (int j = threadIdx.x; j < D; j += blockDim.x) rsh[j] = r[j];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (row >= n) return;
    const float *x = Rp + row * D;
    double acc = 0.0;
    for (int j = lane; j < D; j += 32) acc = fma((double)x[j], rsh[j], acc);
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) dinv[row] = (float)(1.0 / sqrt(acc > 1e-12 ? acc : 1e-12));   // R6 floor
}

int row_groups_for(int64_t n, int d) {
    const int64_t col_tiles = cdiv(d, BN);
    const int64_t row_tiles = cdiv(std::max<int64_t>(n, 1), BM);
    const int64_t want = std::max<int64_t>(1, cdiv(ROW_GROUPS_MAX * 2, col_tiles));
    return (int)std::max<int64_t>(1, std::min<int64_t>({want, row_tiles, (int64_t)ROW_GROUPS_MAX * 4}));
}

void colsum_run(const float *Rp, int64_t n, int D, int G, double *part, double *r, cudaStream_t st) {
    const int64_t rows_per = cdiv(n, G);
    if (D % 4 == 0 && (reinterpret_cast<uintptr_t>(Rp) & 15) == 0)
        colsum4_part_kernel<<<dim3(G, cdiv(D, 256)), 256, 0, st>>>(reinterpret_cast<const float4 *>(Rp), n, D / 4,
                                                                  rows_per, part);
    else
        colsum_part_kernel<<<dim3(G, cdiv(D, 256)), 256, 0, st>>>(Rp, n, D, rows_per, part);
    TPO_LAUNCH_CHECK();
    colsum_reduce_wide_kernel<<<cdiv(D, 32), 1024, 0, st>>>(part, G, D, r);
    TPO_LAUNCH_CHECK();
}

// dinv_kernel fused with R''s row exponents and per-feature maxima (the integer-tensor-core
// products' statistics, see oz_rstats): a persistent warp per row (D = 32 NF), lane j reads the
// columns j + 32 i in the same order as dinv_kernel (so dinv is bit-identical), keeps its NF
// feature maxima in registers over all of its rows; block maxima -> atomicMax (order free).
// Also (spart != NULL) the block's partial s = sum_i dinv_i R'[i] (fp64, rows in a fixed order per
// lane, warps combined in order), the column sums 1^T R that a7's sign rule needs.
template <int NF>
__global__ void __launch_bounds__(256, 3) dinv_stats_kernel(const float *__restrict__ Rp, int64_t n, int D,
                                                         const double *__restrict__ r, float *__restrict__ dinv,
                                                         int32_t *__restrict__ rowE, uint32_t *__restrict__ featmax,
                                                         double *__restrict__ spart) {
    __shared__ double rsh[32 * NF];
    __shared__ double ssm[8][32 * NF];              // feature maxima, then the partial s
    for (int j = threadIdx.x; j < D; j += blockDim.x) rsh[j] = r[j];
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float fm[NF];
    double sa[NF];
#pragma unroll
    for (int i = 0; i < NF; ++i) {
        fm[i] = 0.f;
        sa[i] = 0.0;
    }
    for (int64_t r0 = (int64_t)blockIdx.x * 32 + w; r0 < n; r0 += (int64_t)gridDim.x * 32) {
        float x[4][NF];                                 // 4 rows in flight per warp
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t row = r0 + 8 * u;
#pragma unroll
            for (int i = 0; i < NF; ++i) x[u][i] = row < n ? Rp[row * D + lane + 32 * i] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t row = r0 + 8 * u;
            double acc = 0.0;
            float m = 0.f;
#pragma unroll
            for (int i = 0; i < NF; ++i) {
                acc = fma((double)x[u][i], rsh[lane + 32 * i], acc);
                const float a = fabsf(x[u][i]);
                m = fmaxf(m, a);
                fm[i] = fmaxf(fm[i], a);
            }
            for (int o = 16; o; o >>= 1) {
                acc += __shfl_xor_sync(0xffffffffu, acc, o);
                m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            }
            const float dv = (float)(1.0 / sqrt(acc > 1e-12 ? acc : 1e-12));   // R6 floor (all lanes)
            if (lane == 0 && row < n) {
                dinv[row] = dv;
                int e = 0;
                if (m > 0.f) frexpf(m, &e);
                rowE[row] = e;
            }
            if (spart && row < n)
#pragma unroll
                for (int i = 0; i < NF; ++i) sa[i] = fma((double)dv, (double)x[u][i], sa[i]);
        }
    }
#pragma unroll
    for (int i = 0; i < NF; ++i) ssm[w][lane + 32 * i] = (double)fm[i];
    __syncthreads();
    for (int j = threadIdx.x; j < D; j += blockDim.x) {
        float mm = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) mm = fmaxf(mm, (float)ssm[q][j]);
        atomicMax(&featmax[j], __float_as_uint(mm));
    }
    if (!spart) return;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NF; ++i) ssm[w][lane + 32 * i] = sa[i];
    __syncthreads();
    for (int j = threadIdx.x; j < D; j += blockDim.x) {
        double ss = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) ss += ssm[q][j];
        spart[(int64_t)blockIdx.x * D + j] = ss;
    }
}

}  // namespace

// r = sum_i R'[i] (fp64, deterministic), the same routine tpo_features uses.
void colsum_f64(const float *Rp, int64_t n, int64_t D, double *r, Arena &ar, cudaStream_t st) {
    const int G = row_groups_for(n, (int)(D / 2));
    const size_t mark = ar.off;
    double *part = ar.take<double>((size_t)G * D);
    if (n == 0) TPO_CUDA(cudaMemsetAsync(r, 0, sizeof(double) * D, st));
    else colsum_run(Rp, n, (int)D, G, part, r, st);
    ar.off = mark;
}

// r is staged in 8 * D bytes of dynamic shared memory: above the default 48 KB (D > 6144)
// the kernel must opt in to the larger carve-out first.
void launch_dinv(const float *Rp, int64_t n, int64_t D, const double *r, float *dinv, cudaStream_t st) {
    const size_t smem = sizeof(double) * (size_t)D;
    if (smem > 48 * 1024)
        TPO_CUDA(cudaFuncSetAttribute(dinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dinv_kernel<<<cdiv(n * 32, 256), 256, smem, st>>>(Rp, n, (int)D, r, dinv);
    TPO_LAUNCH_CHECK();
}

// dinv from a given (global) r: the per-row half of tpo_features (sharded path)
void dinv_from_r(const float *Rp, int64_t n, int64_t D, const double *r, float *dinv, cudaStream_t st) {
    if (n == 0) return;
    launch_dinv(Rp, n, D, r, dinv, st);
}

// R' of the given rows and their fp64 column sums (the shard's partial r)
void features_part(const float *Zhat, int64_t n, int64_t d, const float *Q, float *Rp, double *r_part, Arena &ar,
                   cudaStream_t st) {
    const int64_t D = 2 * d;
    if (n == 0) {
        TPO_CUDA(cudaMemsetAsync(r_part, 0, sizeof(double) * D, st));
        return;
    }
    {
        const size_t mark = ar.off;
        features_tc(Zhat, n, d, Q, Rp, ar, st);
        ar.off = mark;
    }
    colsum_f64(Rp, n, D, r_part, ar, st);
}

size_t features_ws_bytes(int64_t n, int64_t d) {
    Arena ar(nullptr, 0);
    ar.take<double>((size_t)row_groups_for(n, (int)d) * 2 * d);
    ar.take<double>(2 * d);
    return ar.off + features_tc_ws(n, d) + 256;
}

void features_impl(const float *Zhat, int64_t n, int64_t d, const float *Q, float *Rp, float *dinv, double *r_out,
                   Arena &ar, cudaStream_t st, int32_t *rowE, uint32_t *featmax, double *s_out) {
    const int D = (int)(2 * d);
    const int G = row_groups_for(n, (int)d);
    double *part = ar.take<double>((size_t)G * D);
    double *r = r_out ? r_out : ar.take<double>(D);
    if (n == 0) {
        TPO_CUDA(cudaMemsetAsync(r, 0, sizeof(double) * D, st));
        return;
    }
    {
        const size_t mark = ar.off;
        features_tc(Zhat, n, d, Q, Rp, ar, st);
        ar.off = mark;
    }
    colsum_run(Rp, n, D, G, part, r, st);
    if (rowE && featmax && D % 32 == 0 && D <= 512) {   // dinv + R' statistics in one pass
        TPO_CUDA(cudaMemsetAsync(featmax, 0, sizeof(uint32_t) * D, st));
        const unsigned grid = (unsigned)std::min<int64_t>(8 * sm_count(), cdiv(n, 32));
        double *spart = s_out ? ar.take<double>((size_t)grid * D) : nullptr;
        switch (D / 32) {
#define TPO_DS(NFV) case NFV: dinv_stats_kernel<NFV><<<grid, 256, 0, st>>>(Rp, n, D, r, dinv, rowE, featmax, spart); break;
            TPO_DS(1) TPO_DS(2) TPO_DS(3) TPO_DS(4) TPO_DS(5) TPO_DS(6) TPO_DS(7) TPO_DS(8)
            TPO_DS(9) TPO_DS(10) TPO_DS(11) TPO_DS(12) TPO_DS(13) TPO_DS(14) TPO_DS(15) TPO_DS(16)
#undef TPO_DS
        }
        TPO_LAUNCH_CHECK();
        if (s_out) {
            colsum_reduce_wide_kernel<<<cdiv(D, 32), 1024, 0, st>>>(spart, (int)grid, D, s_out);
            TPO_LAUNCH_CHECK();
        }
        return;
    }
    if (s_out) TPO_CUDA(cudaMemsetAsync(s_out, 0xFF, sizeof(double) * D, st));   // NaN: "not formed"
    launch_dinv(Rp, n, D, r, dinv, st);
    if (rowE && featmax) oz_rstats(Rp, n, D, rowE, featmax, st);
}

}  // namespace tpo
