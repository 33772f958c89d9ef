// a5: random features of Alg. 1 L8-9 (Eq. R-prime; Eq. Ri, 466-468).
//
//   features_kernel: Zo = sqrt(d) Zhat Q^T as a register-tiled fp32 GEMM (128 x 64 block tile,
//     8 x 4 per thread); the epilogue writes R' = sqrt(e/d) (sin Zo || cos Zo) (accurate
//     sincosf, arguments reach sqrt(d)) and accumulates fp64 column sums of R' for r.
//     Blocks are persistent over row tiles (fixed assignment), so each block emits one
//     partial column-sum vector; a second kernel adds the partials in block order.
//   dinv_kernel: dinv_i = 1 / sqrt(max(R'[i] . r, 1e-12)) with r (fp64) staged in smem.
#include <algorithm>

#include "tpo_internal.cuh"

namespace tpo {
namespace {

constexpr int BM = 128, BN = 64, BK = 16, NT = 256;
constexpr int RM = 8, RN = 4;               // per-thread micro tile (rows x cols)
constexpr int ROW_GROUPS_MAX = 148 * 2;

__global__ void __launch_bounds__(NT) features_kernel(const float *__restrict__ Zh, const float *__restrict__ Q,
                                                      int64_t n, int d, int row_groups, float *__restrict__ Rp,
                                                      double *__restrict__ colpart) {
    __shared__ float As[BK][BM + 4];     // As[k][row]
    __shared__ float Bs[BK][BN + 4];     // Bs[k][col]   (col j of Zo uses row j of Q)
    __shared__ double red[NT / 16][2 * BN];
    const int t = threadIdx.x;
    const int tr = t >> 4, tc = t & 15;  // 16 x 16 thread grid; rows tr*8.., cols tc + 16*j
    const int j0 = blockIdx.x * BN;
    const int D = 2 * d;
    const float sd = sqrtf((float)d);
    const double ampd = sqrt(exp(1.0) / (double)d);
    const float amp = (float)ampd;
    double csin[RN], ccos[RN];
#pragma unroll
    for (int j = 0; j < RN; ++j) csin[j] = ccos[j] = 0.0;
    const int64_t ntiles = (n + BM - 1) / BM;
    for (int64_t tile = blockIdx.y; tile < ntiles; tile += row_groups) {
        const int64_t i0 = tile * BM;
        float acc[RM][RN];
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
            for (int j = 0; j < RN; ++j) acc[i][j] = 0.f;
        for (int k0 = 0; k0 < d; k0 += BK) {
            // A tile 128 x 16: 2048 values, 8 per thread: row t>>1, k (t&1)*8..+7
            {
                const int r = t >> 1, kk = (t & 1) * 8;
                const int64_t row = i0 + r;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const int k = k0 + kk + c;
                    As[kk + c][r] = (row < n && k < d) ? Zh[row * d + k] : 0.f;
                }
            }
            // B tile 64 x 16 (rows j of Q): 1024 values, 4 per thread: j t>>2, k (t&3)*4..+3
            {
                const int r = t >> 2, kk = (t & 3) * 4;
                const int j = j0 + r;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int k = k0 + kk + c;
                    Bs[kk + c][r] = (j < d && k < d) ? Q[(int64_t)j * d + k] : 0.f;
                }
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < BK; ++k) {
                float a[RM], b[RN];
#pragma unroll
                for (int i = 0; i < RM; ++i) a[i] = As[k][tr * RM + i];
#pragma unroll
                for (int j = 0; j < RN; ++j) b[j] = Bs[k][tc + 16 * j];
#pragma unroll
                for (int i = 0; i < RM; ++i)
#pragma unroll
                    for (int j = 0; j < RN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
            }
            __syncthreads();
        }
        // epilogue
#pragma unroll
        for (int i = 0; i < RM; ++i) {
            const int64_t row = i0 + tr * RM + i;
            if (row >= n) continue;
#pragma unroll
            for (int j = 0; j < RN; ++j) {
                const int col = j0 + tc + 16 * j;
                if (col >= d) continue;
                float s, c;
                sincosf(sd * acc[i][j], &s, &c);
                const float rs = amp * s, rc = amp * c;
                Rp[row * D + col] = rs;
                Rp[row * D + d + col] = rc;
                csin[j] += (double)rs;
                ccos[j] += (double)rc;
            }
        }
    }
    // block reduction of the column sums over the 16 row-threads, fixed order
#pragma unroll
    for (int j = 0; j < RN; ++j) {
        red[tr][tc + 16 * j] = csin[j];
        red[tr][BN + tc + 16 * j] = ccos[j];
    }
    __syncthreads();
    if (t < 2 * BN) {
        double s = 0.0;
        for (int r = 0; r < NT / 16; ++r) s += red[r][t];
        const int col = j0 + (t % BN);
        if (col < d) {
            const int out_col = (t < BN) ? col : d + col;
            colpart[(int64_t)blockIdx.y * D + out_col] = s;
        }
    }
}

__global__ void colsum_reduce_kernel(const double *__restrict__ part, int G, int D, double *__restrict__ r) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= D) return;
    double s = 0.0;
    for (int g = 0; g < G; ++g) s += part[(int64_t)g * D + j];
    r[j] = s;
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

}  // namespace

size_t features_ws_bytes(int64_t n, int64_t d) {
    Arena ar(nullptr, 0);
    ar.take<double>((size_t)row_groups_for(n, (int)d) * 2 * d);
    ar.take<double>(2 * d);
    return ar.off + 256;
}

void features_impl(const float *Zhat, int64_t n, int64_t d, const float *Q, float *Rp, float *dinv, double *r_out,
                   Arena &ar, cudaStream_t st) {
    const int G = row_groups_for(n, (int)d);
    const int D = (int)(2 * d);
    double *part = ar.take<double>((size_t)G * D);
    double *r = r_out ? r_out : ar.take<double>(D);
    if (n == 0) {
        TPO_CUDA(cudaMemsetAsync(r, 0, sizeof(double) * D, st));
        return;
    }
    features_kernel<<<dim3(cdiv(d, BN), G), NT, 0, st>>>(Zhat, Q, n, (int)d, G, Rp, part);
    TPO_LAUNCH_CHECK();
    colsum_reduce_kernel<<<cdiv(D, 256), 256, 0, st>>>(part, G, D, r);
    TPO_LAUNCH_CHECK();
    const int TB = 256;
    dinv_kernel<<<cdiv(n * 32, TB), TB, sizeof(double) * D, st>>>(Rp, n, D, r, dinv);
    TPO_LAUNCH_CHECK();
}

}  // namespace tpo
