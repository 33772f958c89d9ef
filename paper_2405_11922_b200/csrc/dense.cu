// Tall-skinny dense products of the solver (a6-a8) with fp64 accumulation and a fixed-order
// cross-block reduction (no atomics): R'^T Y, Y^T Y and R' W of the implicit affinity
// (the n x n matrix is never formed) and of Alg. 2, whose right-hand sides
// have q = k or b <= a few hundred columns.
//
//   atb:  out[p x q] = sum_i (ra_i A[i,:])^T (rb_i B[i,:])
//         Thread owns TA columns of A (coalesced global loads) and a QT-wide chunk of B
//         (staged in smem, read as broadcasts); rows are split over a grid of row groups and
//         each block writes one fp64 partial that reduce_groups_kernel adds in group order.
//   aw:   out[i, :] = r_i A[i, :] W
//         A warp owns RW = 4 rows and a QT-wide chunk of W; lanes stride the reduction
//         dimension (coalesced loads of A), W is staged transposed in smem, and the lane
//         partials are combined by a fixed shuffle tree.
// Operands are widened to fp64 before multiplying.
#include <algorithm>

#include "tpo_internal.cuh"

namespace tpo {
namespace {

constexpr int NT = 256;
constexpr int TA = 2;          // A columns per thread in atb
constexpr int PT = NT * TA;    // A columns per block in atb
constexpr int QT = 16;         // q chunk (both kernels)
constexpr int RC = 32;         // rows per smem chunk in atb
constexpr int RW = 4;          // rows per warp in aw
constexpr int JT = 128;        // reduction-dimension tile in aw

template <class T>
__device__ __forceinline__ double wide(T x) { return (double)x; }

// ----------------------------------------------------------------------------------------
// atb
// ----------------------------------------------------------------------------------------
template <class TAt, class TBt>
__global__ void __launch_bounds__(NT) atb_kernel(const TAt *__restrict__ A, int64_t lda, const float *__restrict__ ra,
                                                 const TBt *__restrict__ B, int64_t ldb, const float *__restrict__ rb,
                                                 int64_t n, int p, int q, int64_t rows_per_group,
                                                 double *__restrict__ part) {
    __shared__ __align__(16) double Bs[RC][QT];
    __shared__ double Sa[RC];
    const int t = threadIdx.x;
    const int a0 = blockIdx.x * PT, b0 = blockIdx.y * QT;
    const int64_t g = blockIdx.z;
    const int64_t r_beg = g * rows_per_group, r_end = min(n, r_beg + rows_per_group);
    double acc[TA][QT];
#pragma unroll
    for (int i = 0; i < TA; ++i)
#pragma unroll
        for (int j = 0; j < QT; ++j) acc[i][j] = 0.0;
    int col[TA];
    bool cv[TA];
#pragma unroll
    for (int i = 0; i < TA; ++i) {
        col[i] = a0 + t + NT * i;
        cv[i] = col[i] < p;
    }
    for (int64_t r0 = r_beg; r0 < r_end; r0 += RC) {
        const int rows = (int)(r_end - r0 < RC ? r_end - r0 : RC);
        for (int e = t; e < RC * QT; e += NT) {
            const int r = e / QT, c = e - r * QT;
            double v = 0.0;
            if (r < rows && b0 + c < q) {
                v = wide(B[(r0 + r) * ldb + b0 + c]);
                if (rb) v *= (double)rb[r0 + r];
            }
            Bs[r][c] = v;
        }
        if (t < RC) Sa[t] = (t < rows) ? (ra ? (double)ra[r0 + t] : 1.0) : 0.0;
        __syncthreads();
#pragma unroll 4
        for (int r = 0; r < rows; ++r) {
            double av[TA];
#pragma unroll
            for (int i = 0; i < TA; ++i) av[i] = cv[i] ? Sa[r] * wide(A[(r0 + r) * lda + col[i]]) : 0.0;
#pragma unroll
            for (int j = 0; j < QT; j += 2) {
                const double2 bv = *reinterpret_cast<const double2 *>(&Bs[r][j]);
#pragma unroll
                for (int i = 0; i < TA; ++i) {
                    acc[i][j] = fma(av[i], bv.x, acc[i][j]);
                    acc[i][j + 1] = fma(av[i], bv.y, acc[i][j + 1]);
                }
            }
        }
        __syncthreads();
    }
    double *out = part + g * (int64_t)p * q;
#pragma unroll
    for (int i = 0; i < TA; ++i) {
        if (!cv[i]) continue;
#pragma unroll
        for (int j = 0; j < QT; ++j)
            if (b0 + j < q) out[(int64_t)col[i] * q + b0 + j] = acc[i][j];
    }
}

__global__ void reduce_groups_kernel(const double *__restrict__ part, int64_t G, int64_t len, double *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= len) return;
    double s = 0.0;
    for (int64_t g = 0; g < G; ++g) s += part[g * len + i];
    out[i] = s;
}

// ----------------------------------------------------------------------------------------
// aw
// ----------------------------------------------------------------------------------------
template <class TAt, class TO, int QW>
__global__ void __launch_bounds__(NT) aw_kernel(const TAt *__restrict__ A, int64_t lda, const float *__restrict__ rs,
                                                const double *__restrict__ W, int64_t n, int p, int q,
                                                TO *__restrict__ out, int64_t ldo) {
    __shared__ double Ws[QW][JT + 1];   // transposed W tile: Ws[c][j]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t row0 = ((int64_t)blockIdx.x * (NT / 32) + w) * RW;
    const int b0 = blockIdx.y * QW;
    double acc[RW][QW];
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int c = 0; c < QW; ++c) acc[r][c] = 0.0;
    for (int j0 = 0; j0 < p; j0 += JT) {
        // issue all loads of A for this tile first (RW x JT/32 per lane in flight)
        double av[JT / 32][RW];
#pragma unroll
        for (int jj = 0; jj < JT / 32; ++jj) {
            const int j = j0 + jj * 32 + lane;
#pragma unroll
            for (int r = 0; r < RW; ++r) {
                const int64_t row = row0 + r;
                av[jj][r] = (row < n && j < p) ? wide(A[row * lda + j]) : 0.0;
            }
        }
        for (int e = threadIdx.x; e < QW * JT; e += NT) {
            const int c = e / JT, j = e - c * JT;
            Ws[c][j] = (j0 + j < p && b0 + c < q) ? W[(int64_t)(j0 + j) * q + b0 + c] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int jj = 0; jj < JT / 32; ++jj) {
            const int j = jj * 32 + lane;
#pragma unroll
            for (int c = 0; c < QW; ++c) {
                const double wv = Ws[c][j];
#pragma unroll
                for (int r = 0; r < RW; ++r) acc[r][c] = fma(av[jj][r], wv, acc[r][c]);
            }
        }
        __syncthreads();
    }
    // fixed shuffle tree over the lanes
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int c = 0; c < QW; ++c) {
            double v = acc[r][c];
#pragma unroll
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            acc[r][c] = v;
        }
    if (lane < QW) {
#pragma unroll
        for (int r = 0; r < RW; ++r) {
            const int64_t row = row0 + r;
            if (row >= n || b0 + lane >= q) continue;
            double v = 0.0;
#pragma unroll
            for (int c = 0; c < QW; ++c)
                if (c == lane) v = acc[r][c];
            const double s = rs ? (double)rs[row] : 1.0;
            out[row * ldo + b0 + lane] = (TO)(s * v);
        }
    }
}

// Row groups of the split-over-rows products: about 4 blocks per SM of a 148-SM B200 in
// total (a fixed constant, so workspace queries need no device).
constexpr int64_t kBlocksTarget = 4 * 148;
int64_t atb_rows_per_group(int64_t n, int64_t p, int64_t q) {
    const int64_t tiles = cdiv(p, PT) * cdiv(q, QT);
    const int64_t want = std::max<int64_t>(1, cdiv(kBlocksTarget, tiles));
    const int64_t G = std::max<int64_t>(1, std::min<int64_t>(want, cdiv(std::max<int64_t>(n, 1), 4 * RC)));
    return cdiv(cdiv(std::max<int64_t>(n, 1), G), RC) * RC;
}

template <class TAt, class TBt>
void atb_run(const TAt *A, int64_t lda, const float *ra, const TBt *B, int64_t ldb, const float *rb, int64_t n,
             int64_t p, int64_t q, double *out, Arena &ar, cudaStream_t st) {
    if (n == 0) {
        TPO_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * p * q, st));
        return;
    }
    const int64_t rpg = atb_rows_per_group(n, p, q);
    const int64_t Gr = std::max<int64_t>(1, cdiv(n, rpg));
    const dim3 grid(cdiv(p, PT), cdiv(q, QT), Gr);
    if (Gr == 1) {
        atb_kernel<TAt, TBt><<<grid, NT, 0, st>>>(A, lda, ra, B, ldb, rb, n, (int)p, (int)q, rpg, out);
        TPO_LAUNCH_CHECK();
        return;
    }
    const size_t mark = ar.off;
    double *part = ar.take<double>(Gr * p * q);
    atb_kernel<TAt, TBt><<<grid, NT, 0, st>>>(A, lda, ra, B, ldb, rb, n, (int)p, (int)q, rpg, part);
    TPO_LAUNCH_CHECK();
    reduce_groups_kernel<<<cdiv(p * q, 256), 256, 0, st>>>(part, Gr, p * q, out);
    TPO_LAUNCH_CHECK();
    ar.off = mark;
}

template <class TAt, class TO>
void aw_run(const TAt *A, int64_t lda, const float *rs, const double *W, int64_t n, int64_t p, int64_t q, TO *out,
            int64_t ldo, cudaStream_t st) {
    if (n == 0 || q == 0) return;
    if (q <= 8) {
        const dim3 grid(cdiv(n, (NT / 32) * RW), cdiv(q, 8));
        aw_kernel<TAt, TO, 8><<<grid, NT, 0, st>>>(A, lda, rs, W, n, (int)p, (int)q, out, ldo);
    } else {
        const dim3 grid(cdiv(n, (NT / 32) * RW), cdiv(q, QT));
        aw_kernel<TAt, TO, QT><<<grid, NT, 0, st>>>(A, lda, rs, W, n, (int)p, (int)q, out, ldo);
    }
    TPO_LAUNCH_CHECK();
}

}  // namespace

size_t tsgemm_ws(int64_t n, int64_t p, int64_t q) {
    const int64_t Gr = std::max<int64_t>(1, cdiv(std::max<int64_t>(n, 1), atb_rows_per_group(n, p, q)));
    return align_up(sizeof(double) * (size_t)(Gr * p * q) + 1) + 512;
}

void tsgemm_AtB_f32f32(const float *A, int64_t lda, const float *rsA, const float *Bm, int64_t ldb,
                       const float *rsB, int64_t n, int64_t p, int64_t q, double *out, Arena &ar, cudaStream_t st) {
    atb_run<float, float>(A, lda, rsA, Bm, ldb, rsB, n, p, q, out, ar, st);
}
void tsgemm_AtB_f32f64(const float *A, int64_t lda, const float *rsA, const double *Bm, int64_t ldb, int64_t n,
                       int64_t p, int64_t q, double *out, Arena &ar, cudaStream_t st) {
    atb_run<float, double>(A, lda, rsA, Bm, ldb, nullptr, n, p, q, out, ar, st);
}
void tsgemm_AtB_f64f64(const double *A, int64_t lda, const double *Bm, int64_t ldb, int64_t n, int64_t p,
                       int64_t q, double *out, Arena &ar, cudaStream_t st) {
    atb_run<double, double>(A, lda, nullptr, Bm, ldb, nullptr, n, p, q, out, ar, st);
}

void tsgemm_AW_f32(const float *A, int64_t lda, const float *rs, const double *W, int64_t n, int64_t p, int64_t q,
                   float *out, int64_t ldo, cudaStream_t st) {
    aw_run<float, float>(A, lda, rs, W, n, p, q, out, ldo, st);
}
void tsgemm_AW_f64(const float *A, int64_t lda, const float *rs, const double *W, int64_t n, int64_t p, int64_t q,
                   double *out, int64_t ldo, cudaStream_t st) {
    aw_run<float, double>(A, lda, rs, W, n, p, q, out, ldo, st);
}
void tsgemm_AW_dd(const double *A, int64_t lda, const double *W, int64_t n, int64_t p, int64_t q, double *out,
                  int64_t ldo, cudaStream_t st) {
    aw_run<double, double>(A, lda, nullptr, W, n, p, q, out, ldo, st);
}

}  // namespace tpo
