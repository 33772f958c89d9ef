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
#include <stdlib.h>

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


// ----------------------------------------------------------------------------------------
// Streaming variants for a fp32 A with 16-byte aligned rows (R' products): A slabs are staged
// into shared memory with cp.async (double buffered), each thread owns a 4 x 4 register tile
// (4 rows/columns of A strided by 32, 4 columns of the skinny side), fp64 FMA.
// ----------------------------------------------------------------------------------------
constexpr int SN = 128;        // threads
constexpr int SR = 128;        // rows (aw) or A columns (atb) per block
constexpr int SK = 32;         // slab depth
constexpr int SP = 36;         // smem pitch (floats) of an A slab row: conflict-free, 16 B aligned

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// out[i, b0 + c] = rs_i * sum_j A[i, j] W[j, b0 + c] with 2 column groups: a thread owns 2 rows
// (strided by 64) and CW = QW / 2 columns, so each fp32 element of A is widened twice (the F2F
// widening runs on the quarter-rate XU pipe; a 4-group tiling was bound by it) and QW may be
// any even width (k = 10 needs 10 columns, not 12).
template <class TO, int QW>
__global__ void __launch_bounds__(SN) aw2_stream_kernel(const float *__restrict__ A, int64_t lda,
                                                        const float *__restrict__ rs, const double *__restrict__ W,
                                                        int64_t n, int p, int q, TO *__restrict__ out, int64_t ldo) {
    constexpr int CW = QW / 2;
    static_assert(QW % 2 == 0, "aw2: even chunk width");
    __shared__ __align__(16) float As[2][SR * SP];
    __shared__ __align__(16) double Ws[2][SK * QW];
    const int t = threadIdx.x, rg = t >> 1, cg = t & 1;
    const int64_t i0 = (int64_t)blockIdx.x * SR;
    const int b0 = blockIdx.y * QW;
    const int nslab = (p + SK - 1) / SK;
    double acc[2][CW];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int c = 0; c < CW; ++c) acc[r][c] = 0.0;
    auto load = [&](int s, int buf) {
        const int k0 = s * SK;
#pragma unroll
        for (int m = 0; m < (SR * SK / 4) / SN; ++m) {
            const int ch = t + SN * m, row = ch >> 3, kc = (ch & 7) * 4;
            const int64_t gi = i0 + row;
            const bool ok = gi < n && k0 + kc < p;
            cp_async16(&As[buf][row * SP + kc], ok ? (const void *)(A + gi * lda + k0 + kc) : (const void *)A, ok);
        }
        for (int e = t; e < SK * QW; e += SN) {     // W slab by cp.async too (no synchronous loads)
            const int kk = e / QW, c = e - kk * QW;
            const bool ok = k0 + kk < p && b0 + c < q;
            const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(&Ws[buf][e]));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d),
                         "l"(ok ? (const void *)(W + (int64_t)(k0 + kk) * q + b0 + c) : (const void *)W),
                         "r"(ok ? 8 : 0)
                         : "memory");
        }
        cp_async_commit();
    };
    load(0, 0);
    for (int s = 0; s < nslab; ++s) {
        const int buf = s & 1;
        if (s + 1 < nslab) {
            load(s + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const float *a = As[buf];
        const double *w = Ws[buf];
#pragma unroll 8
        for (int kk = 0; kk < SK; ++kk) {
            const double a0 = (double)a[rg * SP + kk], a1 = (double)a[(rg + 64) * SP + kk];
#pragma unroll
            for (int c = 0; c < CW; ++c) {
                const double wv = w[kk * QW + cg * CW + c];
                acc[0][c] = fma(a0, wv, acc[0][c]);
                acc[1][c] = fma(a1, wv, acc[1][c]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int64_t row = i0 + rg + 64 * r;
        if (row >= n) continue;
        const double sc = rs ? (double)rs[row] : 1.0;
#pragma unroll
        for (int c = 0; c < CW; ++c) {
            const int col = b0 + cg * CW + c;
            if (col < q) out[row * ldo + col] = (TO)(sc * acc[r][c]);
        }
    }
}

// part[g][a][b0 + c] = sum over the rows of group g of (ra_i A[i, a]) B[i, b0 + c]
template <class TBt, int QW>
__global__ void __launch_bounds__(SN) atb_stream_kernel(const float *__restrict__ A, int64_t lda,
                                                        const float *__restrict__ ra, const TBt *__restrict__ B,
                                                        int64_t ldb, int64_t n, int p, int q, int64_t rows_per_group,
                                                        double *__restrict__ part) {
    constexpr int CW = QW / 4;
    __shared__ __align__(16) float As[2][SK * (SR + 4)];     // As[row][a], pitch SR + 4
    __shared__ __align__(16) double Bs[2][SK * QW];
    constexpr int AP = SR + 4;
    const int t = threadIdx.x, ag = t >> 2, bg = t & 3;
    const int a0 = blockIdx.x * SR, b0 = blockIdx.y * QW;
    const int64_t g = blockIdx.z;
    const int64_t r_beg = g * rows_per_group, r_end = min(n, r_beg + rows_per_group);
    const int nslab = r_end > r_beg ? (int)((r_end - r_beg + SK - 1) / SK) : 0;
    double acc[4][CW];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < CW; ++c) acc[r][c] = 0.0;
    auto load = [&](int s, int buf) {
        const int64_t k0 = r_beg + (int64_t)s * SK;
#pragma unroll
        for (int m = 0; m < (SR * SK / 4) / SN; ++m) {
            const int ch = t + SN * m, row = ch >> 5, ac = (ch & 31) * 4;
            const int64_t gi = k0 + row;
            const bool ok = gi < r_end && a0 + ac < p;
            cp_async16(&As[buf][row * AP + ac], ok ? (const void *)(A + gi * lda + a0 + ac) : (const void *)A, ok);
        }
        cp_async_commit();
        for (int e = t; e < SK * QW; e += SN) {
            const int kk = e / QW, c = e - kk * QW;
            const int64_t gi = k0 + kk;
            double v = 0.0;
            if (gi < r_end && b0 + c < q) {
                v = (double)B[gi * ldb + b0 + c];
                if (ra) v *= (double)ra[gi];
            }
            Bs[buf][e] = v;
        }
    };
    if (nslab > 0) load(0, 0);
    for (int s = 0; s < nslab; ++s) {
        const int buf = s & 1;
        if (s + 1 < nslab) {
            load(s + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const float *a = As[buf];
        const double *b = Bs[buf];
#pragma unroll 8
        for (int kk = 0; kk < SK; ++kk) {
            double av[4], bv[CW];
#pragma unroll
            for (int r = 0; r < 4; ++r) av[r] = (double)a[kk * AP + ag + 32 * r];
#pragma unroll
            for (int c = 0; c < CW; ++c) bv[c] = b[kk * QW + bg * CW + c];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < CW; ++c) acc[r][c] = fma(av[r], bv[c], acc[r][c]);
        }
        __syncthreads();
    }
    double *o = part + g * (int64_t)p * q;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int a = a0 + ag + 32 * r;
        if (a >= p) continue;
#pragma unroll
        for (int c = 0; c < CW; ++c) {
            const int col = b0 + bg * CW + c;
            if (col < q) o[(int64_t)a * q + col] = acc[r][c];
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
    if (n == 0 || lda % 4 != 0 || (reinterpret_cast<uintptr_t>(A) & 15u) != 0 || q > 16) {
        atb_run<float, double>(A, lda, rsA, Bm, ldb, nullptr, n, p, q, out, ar, st);
        return;
    }
    const int QW = q <= 8 ? 8 : 16;
    const int64_t tiles = cdiv(p, SR) * cdiv(q, QW);
    const int64_t want = std::max<int64_t>(1, cdiv(kBlocksTarget, tiles));
    const int64_t G0 = std::max<int64_t>(1, std::min<int64_t>(want, cdiv(n, 4 * SK)));
    const int64_t rpg = cdiv(cdiv(n, G0), SK) * SK;
    const int64_t Gr = std::max<int64_t>(1, cdiv(n, rpg));
    const size_t mark = ar.off;
    double *part = Gr == 1 ? out : ar.take<double>(Gr * p * q);
    const dim3 grid(cdiv(p, SR), cdiv(q, QW), Gr);
    if (QW == 8)
        atb_stream_kernel<double, 8><<<grid, SN, 0, st>>>(A, lda, rsA, Bm, ldb, n, (int)p, (int)q, rpg, part);
    else
        atb_stream_kernel<double, 16><<<grid, SN, 0, st>>>(A, lda, rsA, Bm, ldb, n, (int)p, (int)q, rpg, part);
    TPO_LAUNCH_CHECK();
    if (Gr > 1) {
        reduce_groups_kernel<<<cdiv(p * q, 256), 256, 0, st>>>(part, Gr, p * q, out);
        TPO_LAUNCH_CHECK();
    }
    ar.off = mark;
}
void tsgemm_AtB_f64f64(const double *A, int64_t lda, const double *Bm, int64_t ldb, int64_t n, int64_t p,
                       int64_t q, double *out, Arena &ar, cudaStream_t st) {
    atb_run<double, double>(A, lda, nullptr, Bm, ldb, nullptr, n, p, q, out, ar, st);
}

template <class TO>
void aw_f32_run(const float *A, int64_t lda, const float *rs, const double *W, int64_t n, int64_t p, int64_t q, TO *out,
                int64_t ldo, cudaStream_t st) {
    if (n == 0 || q == 0) return;
    if (lda % 4 != 0 || (reinterpret_cast<uintptr_t>(A) & 15u) != 0) {
        aw_run<float, TO>(A, lda, rs, W, n, p, q, out, ldo, st);
        return;
    }
    // 2 column groups, even chunk widths <= 22 (static smem) fitted to q
    const int64_t nch2 = cdiv(q, 22);
    const int QW2 = (int)(cdiv(cdiv(q, nch2), 2) * 2);
    const dim3 grid2((unsigned)cdiv(n, SR), (unsigned)cdiv(q, QW2));
#define TPO_AW2(QV) case QV: aw2_stream_kernel<TO, QV><<<grid2, SN, 0, st>>>(A, lda, rs, W, n, (int)p, (int)q, out, ldo); break;
    switch (QW2) {
        TPO_AW2(2) TPO_AW2(4) TPO_AW2(6) TPO_AW2(8) TPO_AW2(10) TPO_AW2(12) TPO_AW2(14) TPO_AW2(16)
        TPO_AW2(18) TPO_AW2(20)
        default: aw2_stream_kernel<TO, 22><<<grid2, SN, 0, st>>>(A, lda, rs, W, n, (int)p, (int)q, out, ldo); break;
    }
#undef TPO_AW2
    TPO_LAUNCH_CHECK();
}

void tsgemm_AW_f32(const float *A, int64_t lda, const float *rs, const double *W, int64_t n, int64_t p, int64_t q,
                   float *out, int64_t ldo, cudaStream_t st) {
    aw_f32_run<float>(A, lda, rs, W, n, p, q, out, ldo, st);
}
void tsgemm_AW_f64(const float *A, int64_t lda, const float *rs, const double *W, int64_t n, int64_t p, int64_t q,
                   double *out, int64_t ldo, cudaStream_t st) {
    if (ts64_enabled()) {
        ts_aw_f64(A, lda, rs, W, n, (int)p, (int)q, nullptr, out, ldo, st);
        return;
    }
    aw_f32_run<double>(A, lda, rs, W, n, p, q, out, ldo, st);
}
void tsgemm_AW_dd(const double *A, int64_t lda, const double *W, int64_t n, int64_t p, int64_t q, double *out,
                  int64_t ldo, cudaStream_t st) {
    aw_run<double, double>(A, lda, nullptr, W, n, p, q, out, ldo, st);
}

}  // namespace tpo
