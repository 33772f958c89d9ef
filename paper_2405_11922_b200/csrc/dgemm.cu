// Small and medium fp64 dense products of the host-sized linear algebra (Haar rotation of
// Alg. 1 L6-7; the D x D eigen-iteration of a7; CholeskyQR2), plus the
// device Cholesky-inverse that keeps CholeskyQR2 free of host round trips.
//
//   dgemm:     C = beta C + alpha op(A) B, row-major, op(A) = A (M x K) or A^T (A is K x M).
//              64 x 64 output tile per CTA, 16-deep K slabs staged in shared memory, each
//              thread owns a 4 x 4 register tile strided by 16 (conflict-free smem reads,
//              coalesced stores).  When the grid of output tiles cannot fill the GPU the K
//              range is split; each split writes an fp64 partial and splitk_reduce adds them
//              in split order (deterministic: no atomics).
//   chol_inv:  one CTA; for the b x b Gram g (b <= 112) of CholeskyQR: S = diag(g)^{-1/2},
//              S g S = C^T C (upper C), writes Ci = S C^{-1} so that V <- V Ci has orthonormal
//              columns; a non-SPD or non-finite pivot sets *flag (checked by the caller at its
//              next synchronisation point -> TPO_ENUMERIC).  A near-identity g (max|g - I| <=
//              1e-8, the second CholeskyQR pass) takes the first-order inverse I - F instead.
#include <algorithm>
#include <mutex>

#include "tpo_internal.cuh"

namespace tpo {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, NTH = 256;

// BNT = 64 (4 x 4 register tile per thread) or 32 (2 x 4, for skinny right-hand sides).
// The next K slab is prefetched into registers while the current one is multiplied.
template <bool TA, int BNT, int BK = 16>
__global__ void __launch_bounds__(NTH) dgemm_kernel(int64_t M, int64_t N, int64_t K, double alpha,
                                                    const double *__restrict__ A, int64_t lda,
                                                    const double *__restrict__ B, int64_t ldb, double beta,
                                                    double *__restrict__ C, int64_t ldc, int64_t kchunk,
                                                    double *__restrict__ part) {
    constexpr int TXN = BNT / 4, TYN = NTH / TXN, RM = BM / TYN;
    constexpr int NA = (BK * BM) / NTH, NB = (BK * BNT) / NTH;
    __shared__ double As[BK][BM + 1];
    __shared__ double Bs[BK][BNT + 1];
    const int t = threadIdx.x, tx = t % TXN, ty = t / TXN;
    const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BNT;
    const int64_t k0 = (int64_t)blockIdx.z * kchunk, k1 = min(K, k0 + kchunk);
    double acc[RM][4];
#pragma unroll
    for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    double ra[NA], rb[NB];
    auto fetch = [&](int64_t kk) {
#pragma unroll
        for (int r = 0; r < NA; ++r) {
            const int i = t + r * NTH;
            int k, m;
            if (TA) { k = i / BM; m = i % BM; } else { m = i / BK; k = i % BK; }
            const int64_t gk = kk + k, gm = m0 + m;
            ra[r] = (gk < k1 && gm < M) ? (TA ? A[gk * lda + gm] : A[gm * lda + gk]) : 0.0;
        }
#pragma unroll
        for (int r = 0; r < NB; ++r) {
            const int i = t + r * NTH;
            const int k = i / BNT, nn = i % BNT;
            const int64_t gk = kk + k, gn = n0 + nn;
            rb[r] = (gk < k1 && gn < N) ? B[gk * ldb + gn] : 0.0;
        }
    };
    if (k0 < k1) fetch(k0);
    for (int64_t kk = k0; kk < k1; kk += BK) {
#pragma unroll
        for (int r = 0; r < NA; ++r) {
            const int i = t + r * NTH;
            if (TA) As[i / BM][i % BM] = ra[r]; else As[i % BK][i / BK] = ra[r];
        }
#pragma unroll
        for (int r = 0; r < NB; ++r) {
            const int i = t + r * NTH;
            Bs[i / BNT][i % BNT] = rb[r];
        }
        __syncthreads();
        if (kk + BK < k1) fetch(kk + BK);
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            double av[RM], bv[4];
#pragma unroll
            for (int i = 0; i < RM; ++i) av[i] = As[k][ty + TYN * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[k][tx + TXN * j];
#pragma unroll
            for (int i = 0; i < RM; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < RM; ++i) {
        const int64_t gm = m0 + ty + TYN * i;
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t gn = n0 + tx + TXN * j;
            if (gn >= N) continue;
            if (part) {
                part[((int64_t)blockIdx.z * M + gm) * N + gn] = acc[i][j];
            } else {
                const double v = alpha * acc[i][j];
                C[gm * ldc + gn] = beta == 0.0 ? v : fma(beta, C[gm * ldc + gn], v);
            }
        }
    }
}

__global__ void splitk_reduce_kernel(const double *__restrict__ part, int64_t S, int64_t M, int64_t N, double alpha,
                                     double beta, double *__restrict__ C, int64_t ldc) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M * N) return;
    // 8 independent partial sums (split z mod 8) combined in a fixed order: deterministic and
    // 8 loads in flight
    double s8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int64_t z = 0;
    for (; z + 8 <= S; z += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) s8[j] += part[(z + j) * M * N + i];
    for (; z < S; ++z) s8[z & 7] += part[z * M * N + i];
    const double s = ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
    const int64_t r = i / N, c = i - r * N;
    const double v = alpha * s;
    C[r * ldc + c] = beta == 0.0 ? v : fma(beta, C[r * ldc + c], v);
}

// The same sum, one warp per output (lanes stride the splits, fixed shuffle tree): for few
// outputs and many splits.
__global__ void splitk_reduce_warp_kernel(const double *__restrict__ part, int64_t S, int64_t M, int64_t N,
                                          double alpha, double beta, double *__restrict__ C, int64_t ldc) {
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= M * N) return;
    double s = 0.0;
    for (int64_t z = lane; z < S; z += 32) s += part[z * M * N + i];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        const int64_t r = i / N, c = i - r * N;
        const double v = alpha * s;
        C[r * ldc + c] = beta == 0.0 ? v : fma(beta, C[r * ldc + c], v);
    }
}

void splitk_reduce(const double *part, int64_t S, int64_t M, int64_t N, double alpha, double beta, double *C,
                   int64_t ldc, cudaStream_t st) {
    if (S >= 64 && M * N <= 16384) {
        splitk_reduce_warp_kernel<<<cdiv(M * N * 32, 256), 256, 0, st>>>(part, S, M, N, alpha, beta, C, ldc);
    } else {
        splitk_reduce_kernel<<<cdiv(M * N, 256), 256, 0, st>>>(part, S, M, N, alpha, beta, C, ldc);
    }
    TPO_LAUNCH_CHECK();
}

int64_t splits_for(int64_t M, int64_t N, int64_t K) {
    const int64_t tiles = cdiv(M, BM) * cdiv(N, N <= 32 ? 32 : BN);
    const int64_t want = cdiv(2 * 148, tiles);
    return std::max<int64_t>(1, std::min<int64_t>(want, cdiv(K, 4 * BK)));
}

constexpr int CI_MAX = 112;

// ---------------------------------------------------------------------------------------
// Blocked chol_inv (one CTA of 256 threads, 16 x 16 blocks, b <= CI_MAX): Cholesky and
// triangular inverse with O(b / 16) block barriers (an unblocked one-barrier-per-step version
// was 2-3x slower).
//   Cholesky (upper, S g S = U^T U), per block column J = [j0, je):
//     (1) warp 0 factors the diagonal block (warp-synchronous right-looking steps),
//     (2) panel: U[J, c] <- U_JJ^{-T} U[J, c] for c >= je (thread per column, forward subst.),
//     (3) trailing: U[r][c] -= sum_{i in J} U[i][r] U[i][c] for je <= r <= c.
//   Inverse X = U^{-1}: warp w inverts diagonal block w (column per lane, back substitution),
//     then block rows I from the bottom: T[i][c] = sum_{l=ie}^{c} U[i][l] X[l][c] (c >= ie),
//     X[i][c] = -sum_{l=i}^{ie-1} X_II[i][l] T[l][c].
// ---------------------------------------------------------------------------------------
constexpr int CB = 16;

__global__ void __launch_bounds__(256, 1) chol_inv_blk_kernel(const double *__restrict__ g, int b,
                                                           double *__restrict__ Ci, int *__restrict__ flag) {
    extern __shared__ double sm[];
    const int p = b + 1, t = threadIdx.x, lane = t & 31, w = t >> 5;
    double *U = sm;                      // b x b (pitch p)
    double *X = sm + b * p;              // b x b (pitch p): inverse, then T scratch rows
    double *sc = X + b * p;              // b
    double *T = sc + b;                  // CB x b scratch
    double *rd = T + CB * b;             // b: 1 / U[i][i] (no fp64 divisions on the dependency chains)
    __shared__ int bad, far;
    if (t == 0) bad = 0, far = 0;
    __syncthreads();
    // Near-identity fast path (the second pass of CholeskyQR2): g = I + E with max|E| <= 1e-8
    // has the factor U = I + F + O(|E|^2), F = triu(E, 1) + diag(E) / 2, so U^{-1} = I - F to
    // O(|E|^2) <= 1e-16 -- no sequential factorisation needed.
    for (int i = t; i < b * b; i += 256) {
        const int r = i / b, c = i - r * b;
        const double e = g[i] - (r == c ? 1.0 : 0.0);
        if (!(fabs(e) <= 1e-8)) far = 1;
    }
    __syncthreads();
    if (!far) {
        for (int i = t; i < b * b; i += 256) {
            const int r = i / b, c = i - r * b;
            const double e = g[i] - (r == c ? 1.0 : 0.0);
            Ci[i] = c > r ? -e : (c == r ? 1.0 - 0.5 * e : 0.0);
        }
        return;
    }
    for (int i = t; i < b; i += 256) {
        const double d = g[(int64_t)i * b + i];
        sc[i] = (d > 0.0 && isfinite(d)) ? rsqrt(d) : 0.0;
    }
    __syncthreads();
    for (int i = t; i < b * b; i += 256) {
        const int r = i / b, c = i - r * b;
        U[r * p + c] = c >= r ? g[i] * sc[r] * sc[c] : 0.0;
        X[r * p + c] = 0.0;
    }
    __syncthreads();
    const int nb = (b + CB - 1) / CB;
    for (int J = 0; J < nb; ++J) {
        const int j0 = J * CB, je = min(b, j0 + CB);
        if (w == 0) {   // (1) diagonal block by warp 0, register-resident: lane owns column lane & 15 of
                        //     every other row from lane >> 4; row jj is broadcast by shuffles
            const int c = lane & 15, h = lane >> 4, bs = je - j0;
            double a[CB / 2];
#pragma unroll
            for (int m = 0; m < CB / 2; ++m) {
                const int r = h + 2 * m;
                a[m] = (r < bs && c < bs) ? U[(j0 + r) * p + j0 + c] : 0.0;
            }
#pragma unroll
            for (int jj = 0; jj < CB; ++jj) {
                if (jj >= bs) break;
                const int sh = (jj & 1) * 16;             // lanes holding row jj
                const double rowv = a[jj >> 1];
                double d = __shfl_sync(0xffffffffu, rowv, sh + jj);
                const bool ok = d > 0.0 && isfinite(d);
                if (!ok) d = 1.0;
                double inv = rsqrt(d);
                inv = inv * fma(-0.5 * d * inv, inv, 1.5);      // one Newton step: full fp64 accuracy
                const double piv = d * inv;
                const double uc = __shfl_sync(0xffffffffu, rowv, sh + c) * inv;
                double ur[CB / 2];
#pragma unroll
                for (int m = 0; m < CB / 2; ++m) ur[m] = __shfl_sync(0xffffffffu, rowv, sh + h + 2 * m) * inv;
#pragma unroll
                for (int m = 0; m < CB / 2; ++m) {
                    const int r = h + 2 * m;
                    if (r > jj && c >= r && c < bs) a[m] = fma(-ur[m], uc, a[m]);
                }
                if (h == (jj & 1)) {                      // the finished row jj of U
                    if (c == jj) a[jj >> 1] = piv;
                    else if (c > jj && c < bs) a[jj >> 1] = rowv * inv;
                }
                if (lane == 0) {
                    if (!ok) bad = 1;
                    rd[j0 + jj] = inv;
                }
            }
#pragma unroll
            for (int m = 0; m < CB / 2; ++m) {
                const int r = h + 2 * m;
                if (r < bs && c < bs && c >= r) U[(j0 + r) * p + j0 + c] = a[m];
            }
        }
        __syncthreads();
        for (int c = je + t; c < b; c += 256) {         // (2) panel: forward substitution per column
            double x[CB];
#pragma unroll
            for (int ii = 0; ii < CB; ++ii) x[ii] = j0 + ii < je ? U[(j0 + ii) * p + c] : 0.0;
#pragma unroll
            for (int ii = 0; ii < CB; ++ii) {
                const int i = j0 + ii;
                if (i >= je) break;
                double v = x[ii];
#pragma unroll
                for (int ll = 0; ll < ii; ++ll) v -= U[(j0 + ll) * p + i] * x[ll];
                x[ii] = v * rd[i];
            }
#pragma unroll
            for (int ii = 0; ii < CB; ++ii)
                if (j0 + ii < je) U[(j0 + ii) * p + c] = x[ii];
        }
        __syncthreads();
        const int w2 = b - je;                            // (3) trailing update, 16 threads per row
        for (int rr = t / 16; rr < w2; rr += 16) {
            const int r = je + rr;
            for (int c = r + (t & 15); c < b; c += 16) {
                double v = U[r * p + c];
                for (int i = j0; i < je; ++i) v -= U[i * p + r] * U[i * p + c];
                U[r * p + c] = v;
            }
        }
        __syncthreads();
    }
    // inverse of the diagonal blocks: warp w handles blocks w, w + 8, ...; lane = column,
    // the column's entries kept in registers while it is solved bottom-up
    for (int I = w; I < nb; I += 8) {
        const int i0 = I * CB, ie = min(b, i0 + CB);
        const int jj = lane, j = i0 + jj;
        if (lane < CB && j < ie) {
            double x[CB];
#pragma unroll
            for (int ii = 0; ii < CB; ++ii) x[ii] = 0.0;
#pragma unroll
            for (int ii = CB - 1; ii >= 0; --ii) {
                if (ii > jj) continue;
                const int i = i0 + ii;
                if (ii == jj) { x[ii] = rd[i]; continue; }
                double s2 = 0.0;
#pragma unroll
                for (int ll = ii + 1; ll < CB; ++ll)
                    if (ll <= jj) s2 += U[i * p + i0 + ll] * x[ll];
                x[ii] = -s2 * rd[i];
            }
#pragma unroll
            for (int ii = 0; ii < CB; ++ii)
                if (ii <= jj) X[(i0 + ii) * p + j] = x[ii];
        }
    }
    __syncthreads();
    for (int I = nb - 2; I >= 0; --I) {                  // off-diagonal block rows, bottom up
        const int i0 = I * CB, ie = min(b, i0 + CB), wc = b - ie;
        for (int e = t; e < CB * wc; e += 256) {          // T[i][c] = sum_{l=ie}^{c} U[i][l] X[l][c]
            const int ii = e / wc, c = ie + e % wc, i = i0 + ii;
            double s = 0.0;
            if (i < ie)
                for (int l = ie; l <= c; ++l) s += U[i * p + l] * X[l * p + c];
            T[ii * b + c] = s;
        }
        __syncthreads();
        for (int e = t; e < CB * wc; e += 256) {          // X[i][c] = -sum_{l=i}^{ie-1} X[i][l] T[l][c]
            const int ii = e / wc, c = ie + e % wc, i = i0 + ii;
            if (i >= ie) continue;
            double s = 0.0;
            for (int l = i; l < ie; ++l) s += X[i * p + l] * T[(l - i0) * b + c];
            X[i * p + c] = -s;
        }
        __syncthreads();
    }
    for (int i = t; i < b * b; i += 256) {
        const int r = i / b, c = i - r * b;
        Ci[i] = c >= r ? X[r * p + c] * sc[r] : 0.0;
    }
    if (t == 0) {
        bool z = false;
        for (int i = 0; i < b; ++i) z |= sc[i] == 0.0;
        if ((bad || z) && flag) *flag = 1;
    }
}


// ---- skinny C = A^T B (A: K x M, B: K x N, M, N <= 32, K large: the k x k products of Alg. 2)
// The dgemm tile (64 x 32) keeps only 20 % of its FMAs for M = N = 20; here a CTA owns the whole
// M x N output as a grid of TA x TB register tiles over its slice of the K rows, staged in
// 32-row chunks through a double-buffered cp.async ring; each CTA writes an fp64 partial that
// splitk_reduce adds in CTA order (deterministic).
constexpr int TS_RC = 32, TS_ST = 4;   // rows per chunk, ring stages
template <int TA, int TB>
__global__ void __launch_bounds__(256) tsatb_kernel(const double *__restrict__ A, int64_t lda,
                                                    const double *__restrict__ B, int64_t ldb, int64_t K, int M,
                                                    int N, int64_t rows_per, double *__restrict__ part) {
    extern __shared__ __align__(16) double tsm[];    // [TS_ST][TS_RC][M + N]
    const int W = M + N, t = threadIdx.x;
    const int QB = (N + TB - 1) / TB, PA = (M + TA - 1) / TA;
    const int ta = t / QB, tb = t - ta * QB;
    const bool active = ta < PA;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per, r1 = min(K, r0 + rows_per);
    const int nch = (int)((r1 - r0 + TS_RC - 1) / TS_RC);
    auto load = [&](int c, int buf) {
        double *S = tsm + (size_t)buf * TS_RC * W;
        const int64_t rb = r0 + (int64_t)c * TS_RC;
        for (int e = t; e < TS_RC * W; e += 256) {
            const int r = e / W, col = e - r * W;
            const bool v = rb + r < r1;
            const double *src = col < M ? A + (rb + r) * lda + col : B + (rb + r) * ldb + (col - M);
            const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(S + e));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d),
                         "l"(v ? (const void *)src : (const void *)A), "r"(v ? 8 : 0)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double acc[TA][TB];
#pragma unroll
    for (int i = 0; i < TA; ++i)
#pragma unroll
        for (int j = 0; j < TB; ++j) acc[i][j] = 0.0;
#pragma unroll
    for (int c = 0; c < TS_ST - 1; ++c) {
        if (c < nch) load(c, c);
        else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int c = 0; c < nch; ++c) {
        const int buf = c % TS_ST;
        asm volatile("cp.async.wait_group %0;" ::"n"(TS_ST - 2) : "memory");
        __syncthreads();
        if (c + TS_ST - 1 < nch) load(c + TS_ST - 1, (c + TS_ST - 1) % TS_ST);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        if (active) {
            const double *S = tsm + (size_t)buf * TS_RC * W;
#pragma unroll 8
            for (int r = 0; r < TS_RC; ++r) {
                double a[TA], b[TB];
#pragma unroll
                for (int i = 0; i < TA; ++i) a[i] = (ta * TA + i < M) ? S[r * W + ta * TA + i] : 0.0;
#pragma unroll
                for (int j = 0; j < TB; ++j) b[j] = (tb * TB + j < N) ? S[r * W + M + tb * TB + j] : 0.0;
#pragma unroll
                for (int i = 0; i < TA; ++i)
#pragma unroll
                    for (int j = 0; j < TB; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
            }
        }
    }
    if (!active) return;
    double *P = part + (size_t)blockIdx.x * M * N;
#pragma unroll
    for (int i = 0; i < TA; ++i)
#pragma unroll
        for (int j = 0; j < TB; ++j) {
            const int a = ta * TA + i, bcol = tb * TB + j;
            if (a < M && bcol < N) P[(size_t)a * N + bcol] = acc[i][j];
        }
}

template <int TA, int TB>
void launch_tsatb(int64_t G, const double *A, int64_t lda, const double *B, int64_t ldb, int64_t K, int M, int N,
                  int64_t rows_per, double *part, cudaStream_t st) {
    const size_t smem = sizeof(double) * TS_ST * TS_RC * (M + N);
    static std::once_flag once;
    std::call_once(once, [] {
        cudaFuncSetAttribute(tsatb_kernel<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(sizeof(double) * TS_ST * TS_RC * 64));
    });
    tsatb_kernel<TA, TB><<<(unsigned)G, 256, smem, st>>>(A, lda, B, ldb, K, M, N, rows_per, part);
    TPO_LAUNCH_CHECK();
}

}  // namespace

// Bound for every K and every M' <= M, N' <= N: S <= 296 / tiles + 1 and M N <= 4096 tiles,
// so the split-K partials hold at most 296 * 4096 + M N doubles.
size_t dgemm_ws(int64_t M, int64_t N, int64_t K) {
    (void)K;
    return align_up(sizeof(double) * (size_t)(2 * 148 * BM * BN + 2 * M * N) + 1) + 256;
}

void dgemm(bool transA, int64_t M, int64_t N, int64_t K, double alpha, const double *A, int64_t lda, const double *B,
           int64_t ldb, double beta, double *C, int64_t ldc, Arena &ar, cudaStream_t st) {
    if (M <= 0 || N <= 0) return;
    if (K <= 0) {   // empty sum: C = beta C
        splitk_reduce_kernel<<<cdiv(M * N, 256), 256, 0, st>>>(nullptr, 0, M, N, alpha, beta, C, ldc);
        TPO_LAUNCH_CHECK();
        return;
    }
    if (transA && M <= 32 && N <= 32 && K >= 8192) {    // skinny k x k products: tsatb
        const int64_t G = std::min<int64_t>(2 * 148, cdiv(K, 256));
        const int64_t rows_per = cdiv(K, G);
        const int64_t Gr = cdiv(K, rows_per);
        const size_t mark = ar.off;
        double *part = ar.take<double>(Gr * M * N);
        if (M <= 16 && N <= 16) launch_tsatb<1, 1>(Gr, A, lda, B, ldb, K, (int)M, (int)N, rows_per, part, st);
        else launch_tsatb<2, 2>(Gr, A, lda, B, ldb, K, (int)M, (int)N, rows_per, part, st);
        splitk_reduce(part, Gr, M, N, alpha, beta, C, ldc, st);
        ar.off = mark;
        return;
    }
    const int64_t S = splits_for(M, N, K);
    const int64_t kchunk = cdiv(cdiv(K, S), BK) * BK;
    const int64_t Sr = cdiv(K, kchunk);
    const bool skinny = N <= 32;
    const dim3 grid((unsigned)cdiv(M, BM), (unsigned)cdiv(N, skinny ? 32 : BN), (unsigned)Sr);
    const size_t mark = ar.off;
    double *part = Sr > 1 ? ar.take<double>(Sr * M * N) : nullptr;
    if (transA && skinny)
        dgemm_kernel<true, 32><<<grid, NTH, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, part);
    else if (transA)
        dgemm_kernel<true, 64><<<grid, NTH, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, part);
    else if (skinny)
        dgemm_kernel<false, 32, 32><<<grid, NTH, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, part);
    else
        dgemm_kernel<false, 64><<<grid, NTH, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kchunk, part);
    TPO_LAUNCH_CHECK();
    if (Sr > 1) splitk_reduce(part, Sr, M, N, alpha, beta, C, ldc, st);
    ar.off = mark;
}

void chol_inv_device(const double *g, int64_t b, double *Ci, int *flag, cudaStream_t st) {
    TPO_REQUIRE(b >= 1 && b <= CI_MAX, "chol_inv: block width out of range");
    const size_t smem = sizeof(double) * (size_t)(2 * b * (b + 1) + 2 * b + CB * b);
    TPO_CUDA(cudaFuncSetAttribute(chol_inv_blk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    chol_inv_blk_kernel<<<1, 256, smem, st>>>(g, (int)b, Ci, flag);
    TPO_LAUNCH_CHECK();
}

}  // namespace tpo
