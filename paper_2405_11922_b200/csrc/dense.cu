// Tall-skinny dense products of the solver (a6-a8) with fp64 accumulation and a fixed-order
// cross-block reduction (no atomics): the products R'^T Y, Y^T Y, R' W of the implicit
// affinity (never form the n x n matrix) and of Alg. 2.
//
//   atb:  out[p x q] = sum_i (ra_i A[i,:])^T (rb_i B[i,:])   rows split over a grid of
//         row groups; each block accumulates its rows in registers (fp64), writes one
//         partial, and a reduction kernel adds the partials in group order.
//   aw:   out[i, :] = r_i A[i, :] W                            (row tiles x column tiles)
//
// Both use a 64 x 64 output tile per 256-thread block, a 4 x 4 register micro-tile per
// thread, and a 16-deep smem k-slab.  Operands are widened to fp64 when staged.
#include <algorithm>

#include "tpo_internal.cuh"

namespace tpo {
namespace {

constexpr int TM = 64, TK = 16, NT = 256;

template <class T>
__device__ __forceinline__ double ld_wide(const T *p) { return (double)(*p); }

// ----------------------------------------------------------------------------------------
// atb: partial[g][a][b] = sum over rows i in group g of (ra_i A[i,a]) (rb_i B[i,b])
// ----------------------------------------------------------------------------------------
template <class TA, class TB>
__global__ void __launch_bounds__(NT) atb_kernel(const TA *__restrict__ A, int64_t lda, const float *__restrict__ ra,
                                                 const TB *__restrict__ B, int64_t ldb, const float *__restrict__ rb,
                                                 int64_t n, int p, int q, int64_t rows_per_group,
                                                 double *__restrict__ part) {
    __shared__ double As[TK][TM];
    __shared__ double Bs[TK][TM];
    const int t = threadIdx.x, ty = t >> 4, tx = t & 15;
    const int a0 = blockIdx.x * TM, b0 = blockIdx.y * TM;
    const int64_t g = blockIdx.z;
    const int64_t r_beg = g * rows_per_group, r_end = min(n, r_beg + rows_per_group);
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    // staging: 16 rows x 64 cols per operand = 1024 values, 4 per thread
    const int lr = t >> 4, lc = (t & 15) * 4;
    for (int64_t r0 = r_beg; r0 < r_end; r0 += TK) {
        const int64_t row = r0 + lr;
        const bool rv = row < r_end;
        const double sa = (rv && ra) ? (double)ra[row] : 1.0;
        const double sb = (rv && rb) ? (double)rb[row] : 1.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int ca = a0 + lc + c, cb = b0 + lc + c;
            As[lr][lc + c] = (rv && ca < p) ? sa * ld_wide(A + row * lda + ca) : 0.0;
            Bs[lr][lc + c] = (rv && cb < q) ? sb * ld_wide(B + row * ldb + cb) : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < TK; ++r) {
            double av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[r][i * 16 + ty];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[r][j * 16 + tx];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
    double *out = part + g * (int64_t)p * q;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int a = a0 + i * 16 + ty;
        if (a >= p) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int b = b0 + j * 16 + tx;
            if (b < q) out[(int64_t)a * q + b] = acc[i][j];
        }
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
// aw: out[i, b] = r_i sum_a A[i, a] W[a, b]    (A n x p, W p x q fp64)
// ----------------------------------------------------------------------------------------
template <class TA, class TO>
__global__ void __launch_bounds__(NT) aw_kernel(const TA *__restrict__ A, int64_t lda, const float *__restrict__ rs,
                                                const double *__restrict__ W, int64_t n, int p, int q,
                                                TO *__restrict__ out, int64_t ldo) {
    __shared__ double As[TK][TM];   // As[kk][row]
    __shared__ double Ws[TK][TM];   // Ws[kk][col]
    const int t = threadIdx.x, ty = t >> 4, tx = t & 15;
    const int64_t i0 = (int64_t)blockIdx.x * TM;
    const int b0 = blockIdx.y * TM;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    // A staging: 64 rows x 16 k: thread loads row (t >> 2), k (t & 3) * 4 .. +3
    const int ar = t >> 2, ak = (t & 3) * 4;
    // W staging: 16 k x 64 cols: thread loads k (t >> 4), cols (t & 15) * 4 .. +3
    const int wk = t >> 4, wc = (t & 15) * 4;
    for (int k0 = 0; k0 < p; k0 += TK) {
        const int64_t row = i0 + ar;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int kk = k0 + ak + c;
            As[ak + c][ar] = (row < n && kk < p) ? ld_wide(A + row * lda + kk) : 0.0;
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int kk = k0 + wk, col = b0 + wc + c;
            Ws[wk][wc + c] = (kk < p && col < q) ? W[(int64_t)kk * q + col] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < TK; ++r) {
            double av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[r][i * 16 + ty];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Ws[r][j * 16 + tx];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t row = i0 + i * 16 + ty;
        if (row >= n) continue;
        const double s = rs ? (double)rs[row] : 1.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int b = b0 + j * 16 + tx;
            if (b < q) out[row * ldo + b] = (TO)(s * acc[i][j]);
        }
    }
}

// Row groups of the split-over-rows products: about 4 blocks per SM of a 148-SM B200 in
// total (a fixed constant, so workspace queries need no device).
constexpr int64_t kBlocksTarget = 4 * 148;
int64_t atb_rows_per_group(int64_t n, int64_t p, int64_t q) {
    const int64_t tiles = cdiv(p, TM) * cdiv(q, TM);
    const int64_t want = std::max<int64_t>(1, cdiv(kBlocksTarget, tiles));
    const int64_t G = std::max<int64_t>(1, std::min<int64_t>(want, cdiv(n, 4 * TK)));
    return cdiv(cdiv(std::max<int64_t>(n, 1), G), TK) * TK;
}

template <class TA, class TB>
void atb_run(const TA *A, int64_t lda, const float *ra, const TB *B, int64_t ldb, const float *rb, int64_t n,
             int64_t p, int64_t q, double *out, Arena &ar, cudaStream_t st) {
    const int64_t tp = cdiv(p, TM), tq = cdiv(q, TM);
    const int64_t rpg = atb_rows_per_group(n, p, q);
    const int64_t Gr = std::max<int64_t>(1, cdiv(n, rpg));
    if (n == 0) {
        TPO_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * p * q, st));
        return;
    }
    if (Gr == 1) {
        atb_kernel<TA, TB><<<dim3(tp, tq, 1), NT, 0, st>>>(A, lda, ra, B, ldb, rb, n, (int)p, (int)q, rpg, out);
        TPO_LAUNCH_CHECK();
        return;
    }
    double *part = ar.take<double>(Gr * p * q);
    atb_kernel<TA, TB><<<dim3(tp, tq, Gr), NT, 0, st>>>(A, lda, ra, B, ldb, rb, n, (int)p, (int)q, rpg, part);
    TPO_LAUNCH_CHECK();
    reduce_groups_kernel<<<cdiv(p * q, 256), 256, 0, st>>>(part, Gr, p * q, out);
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
    if (n == 0) return;
    aw_kernel<float, float><<<dim3(cdiv(n, TM), cdiv(q, TM)), NT, 0, st>>>(A, lda, rs, W, n, (int)p, (int)q, out, ldo);
    TPO_LAUNCH_CHECK();
}
void tsgemm_AW_f64(const float *A, int64_t lda, const float *rs, const double *W, int64_t n, int64_t p, int64_t q,
                   double *out, int64_t ldo, cudaStream_t st) {
    if (n == 0) return;
    aw_kernel<float, double><<<dim3(cdiv(n, TM), cdiv(q, TM)), NT, 0, st>>>(A, lda, rs, W, n, (int)p, (int)q, out, ldo);
    TPO_LAUNCH_CHECK();
}
// fp64 A (used on the D x D Gram inside the subspace iteration)
void tsgemm_AW_dd(const double *A, int64_t lda, const double *W, int64_t n, int64_t p, int64_t q, double *out,
                  int64_t ldo, cudaStream_t st) {
    if (n == 0) return;
    aw_kernel<double, double><<<dim3(cdiv(n, TM), cdiv(q, TM)), NT, 0, st>>>(A, lda, nullptr, W, n, (int)p, (int)q, out, ldo);
    TPO_LAUNCH_CHECK();
}


}  // namespace tpo
