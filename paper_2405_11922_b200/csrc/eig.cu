// a6-a7: implicit affinity product and the top-k singular triplets of R = diag(dinv) R'
// ("the top-k left and right singular vectors of R", Eq. init-HY).
//
// EXACT mode (R7): Gram G = R^T R (D x D, fp64 sums) once, then block subspace iteration
// with Rayleigh-Ritz on G (the D x D image of the implicit n x n affinity S~ = R R^T:
// both share their nonzero spectrum) until the top-k Ritz residuals fall below 1e-9 lambda_1;
// with a full-rank block (b = D) this is one Rayleigh-Ritz step, i.e. a dense eigensolve.
// Then Gamma = R Psi Sigma^{-1} and a CholeskyQR2 polish if ||Gamma^T Gamma - I||_max > 1e-6.
// HALKO mode: the randomised truncated SVD the paper cites, q power steps.
// Both modes end with the sign rule R8.
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include <stdio.h>
#include <chrono>

#include "tpo_internal.cuh"

namespace tpo {

void tsgemm_AW_dd(const double *A, int64_t lda, const double *W, int64_t n, int64_t p, int64_t q, double *out,
                  int64_t ldo, cudaStream_t st);

namespace {

// Column statistics of an n x k fp64 matrix: sum, sum |x|, argmax |x| (first index).  Stage 1:
// a block per fixed row range, warps own contiguous sub-ranges (rows in order), lanes own
// columns; warps are combined in order.  Stage 2 combines the blocks in order (strict '>'
// keeps the smallest index among equal magnitudes).  Deterministic.
constexpr int CS_WARPS = 8;
__global__ void __launch_bounds__(CS_WARPS * 32) colstats_part_kernel(const double *__restrict__ A, int64_t n, int k,
                                                                      int64_t rows_per, double *__restrict__ ps,
                                                                      double *__restrict__ pa, double *__restrict__ pm,
                                                                      int64_t *__restrict__ pi) {
    __shared__ double ss[CS_WARPS][128], sa[CS_WARPS][128], smx[CS_WARPS][128];
    __shared__ int64_t si[CS_WARPS][128];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t b0 = blockIdx.x * rows_per, b1 = min(n, b0 + rows_per);
    const int64_t per_w = (rows_per + CS_WARPS - 1) / CS_WARPS;
    const int64_t w0 = min(b1, b0 + w * per_w), w1 = min(b1, w0 + per_w);
    for (int c = lane; c < k; c += 32) {
        double s = 0.0, a = 0.0, best = -1.0;
        int64_t bi = 0;
        for (int64_t i = w0; i < w1; ++i) {
            const double v = A[i * k + c];
            s += v;
            a += fabs(v);
            if (fabs(v) > best) { best = fabs(v); bi = i; }
        }
        ss[w][c] = s; sa[w][c] = a; smx[w][c] = best; si[w][c] = bi;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < k; c += CS_WARPS * 32) {
        double s = 0.0, a = 0.0, best = -1.0;
        int64_t bi = 0;
        for (int ww = 0; ww < CS_WARPS; ++ww) {
            s += ss[ww][c];
            a += sa[ww][c];
            if (smx[ww][c] > best) { best = smx[ww][c]; bi = si[ww][c]; }
        }
        ps[blockIdx.x * (int64_t)k + c] = s;
        pa[blockIdx.x * (int64_t)k + c] = a;
        pm[blockIdx.x * (int64_t)k + c] = best;
        pi[blockIdx.x * (int64_t)k + c] = bi;
    }
}

// warp per column: lanes stride the block partials, fixed shuffle tree for the sums; the
// argmax keeps the larger magnitude, ties -> smaller row index (order independent)
__global__ void colstats_final_kernel(const double *__restrict__ ps, const double *__restrict__ pa,
                                      const double *__restrict__ pm, const int64_t *__restrict__ pi, int64_t G, int k,
                                      double *__restrict__ out_sum, double *__restrict__ out_abs,
                                      int64_t *__restrict__ out_arg) {
    const int c = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (c >= k) return;
    double s = 0.0, a = 0.0, best = -1.0;
    int64_t bi = INT64_MAX;
    for (int64_t g = lane; g < G; g += 32) {
        s += ps[g * k + c];
        a += pa[g * k + c];
        const double m = pm[g * k + c];
        const int64_t i = pi[g * k + c];
        if (m > best || (m == best && i < bi)) { best = m; bi = i; }
    }
    for (int o = 16; o; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        a += __shfl_xor_sync(0xffffffffu, a, o);
        const double om = __shfl_xor_sync(0xffffffffu, best, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (om > best || (om == best && oi < bi)) { best = om; bi = oi; }
    }
    if (lane == 0) {
        out_sum[c] = s;
        out_abs[c] = a;
        out_arg[c] = bi;
    }
}

__global__ void flip_cols_f64(double *__restrict__ A, int64_t n, int k, const int *__restrict__ sgn) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n * k) return;
    if (sgn[i % k] < 0) A[i] = -A[i];
}

// out = sgn(l) A (rounded to fp32): R8's column flips fused with the fp32 rounding of Gamma
__global__ void flip_cast_f64_f32(const double *__restrict__ A, int64_t n, int k, const int *__restrict__ sgn,
                                  float *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n * k) return;
    const double v = A[i];
    out[i] = (float)(sgn[i % k] < 0 ? -v : v);
}

__global__ void cast_f64_f32_k(const double *__restrict__ a, int64_t len, float *__restrict__ b) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < len) b[i] = (float)a[i];
}

__global__ void flip_cols_f32(float *__restrict__ A, int64_t n, int k, const int *__restrict__ sgn) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n * k) return;
    if (sgn[i % k] < 0) A[i] = -A[i];
}

__global__ void fill_f64(double *p, int64_t n, double v) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

__global__ void cast_f64_f32(const double *__restrict__ a, int64_t len, float *__restrict__ b) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < len) b[i] = (float)a[i];
}

template <class T>
T *to_dev(Arena &ar, const std::vector<T> &h, cudaStream_t st) {
    T *d = ar.take<T>(h.size());
    TPO_CUDA(cudaMemcpyAsync(d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, st));
    return d;
}

template <class T>
std::vector<T> to_host(const T *d, size_t len, cudaStream_t st) {
    std::vector<T> h(len);
    TPO_CUDA(cudaMemcpyAsync(h.data(), d, sizeof(T) * len, cudaMemcpyDeviceToHost, st));
    TPO_CUDA(cudaStreamSynchronize(st));
    return h;
}

// splitmix64 -> uniform in [-1, 1): the deterministic start block of the subspace iteration
double start_entry(uint64_t i) {
    uint64_t z = i + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

// CholeskyQR2 of a device fp64 matrix V (rows x b) in place (tmp: rows x b).  Each pass
// factors the column-equilibrated Gram S G S = C^T C (S = diag(G_ii^-1/2)), so V <- V S C^-1.
// For b <= 112 everything stays on the device (dgemm + one-CTA chol_inv); a failed
// factorisation sets *flag, which the caller checks at its next synchronisation point.
void cholqr2_f64(double *V, double *tmp, int64_t rows, int64_t b, int *flag, Arena &ar, cudaStream_t st) {
    for (int pass = 0; pass < 2; ++pass) {
        const size_t mark = ar.off;
        double *g = ar.take<double>(b * b);
        dgemm(true, b, b, rows, 1.0, V, b, V, b, 0.0, g, b, ar, st);
        double *ci = ar.take<double>(b * b);
        if (b <= 112) {
            chol_inv_device(g, b, ci, flag, st);
        } else {
            std::vector<double> gh = to_host(g, b * b, st), C(b * b), Ci(b * b), sc(b);
            for (int64_t i = 0; i < b; ++i) sc[i] = gh[i * b + i] > 0.0 ? 1.0 / sqrt(gh[i * b + i]) : 0.0;
            for (int64_t i = 0; i < b; ++i)
                for (int64_t j = 0; j < b; ++j) gh[i * b + j] *= sc[i] * sc[j];
            if (!host_cholesky_upper(b, gh.data(), C.data()))
                throw Error(TPO_ENUMERIC, "CholeskyQR2: Gram matrix not positive definite");
            host_upper_inverse(b, C.data(), Ci.data());
            for (int64_t i = 0; i < b; ++i)
                for (int64_t j = 0; j < b; ++j) Ci[i * b + j] *= sc[i];
            TPO_CUDA(cudaMemcpyAsync(ci, Ci.data(), sizeof(double) * b * b, cudaMemcpyHostToDevice, st));
            TPO_CUDA(cudaStreamSynchronize(st));
        }
        dgemm(false, rows, b, b, 1.0, V, b, ci, b, 0.0, tmp, b, ar, st);
        TPO_CUDA(cudaMemcpyAsync(V, tmp, sizeof(double) * rows * b, cudaMemcpyDeviceToDevice, st));
        ar.off = mark;
    }
}

// Reads the device failure flag of the CholeskyQR steps (synchronises the stream).
void check_flag(const int *flag, cudaStream_t st, const char *what) {
    int h = 0;
    TPO_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    TPO_CUDA(cudaStreamSynchronize(st));
    if (h) throw Error(TPO_ENUMERIC, std::string(what) + ": Gram matrix not positive definite");
}

// Gd = G - lam u u^T (deflation of the top eigenpair, see gram_topk)
__global__ void deflate_kernel(const double *__restrict__ G, const double *__restrict__ u,
                               const double *__restrict__ lam, int64_t D, double *__restrict__ Gd) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= D * D) return;
    const int64_t a = i / D, b = i - a * D;
    Gd[i] = G[i] - (*lam) * u[a] * u[b];
}

// u = r / ||r|| (one CTA, fixed-order tree); *zero = 1 when r = 0.
__global__ void __launch_bounds__(1024) unit_vec_kernel(const double *__restrict__ r, double *__restrict__ u,
                                                        int64_t D, int *__restrict__ zero) {
    __shared__ double s1[1024];
    const int t = threadIdx.x;
    double nr = 0.0;
    for (int64_t i = t; i < D; i += 1024) nr += r[i] * r[i];
    s1[t] = nr;
    __syncthreads();
    for (int o = 512; o; o >>= 1) {
        if (t < o) s1[t] += s1[t + o];
        __syncthreads();
    }
    if (!(s1[0] > 0.0)) {
        if (t == 0) *zero = 1;
        return;
    }
    const double inv = 1.0 / sqrt(s1[0]);
    for (int64_t i = t; i < D; i += 1024) u[i] = r[i] * inv;
}

// One power step finished on the device (one CTA, fixed-order tree): given gu = G u,
// lam = gu . u (Rayleigh quotient, u unit), u <- gu / ||gu||.
__global__ void __launch_bounds__(1024) power_step_kernel(const double *__restrict__ gu, double *__restrict__ u,
                                                          int64_t D, double *__restrict__ lam) {
    __shared__ double s1[1024], s2[1024];
    const int t = threadIdx.x;
    double nr = 0.0, ray = 0.0;
    for (int64_t i = t; i < D; i += 1024) {
        nr += gu[i] * gu[i];
        ray += gu[i] * u[i];
    }
    s1[t] = nr;
    s2[t] = ray;
    __syncthreads();
    for (int o = 512; o; o >>= 1) {
        if (t < o) { s1[t] += s1[t + o]; s2[t] += s2[t + o]; }
        __syncthreads();
    }
    const double inv = 1.0 / sqrt(s1[0]);
    for (int64_t i = t; i < D; i += 1024) u[i] = gu[i] * inv;
    if (t == 0) *lam = s2[0];
}

// out = s1 * GY - s2 * Y1 - (Y0 ? Y0 : 0): one step of the Chebyshev three-term recurrence
__global__ void cheb_kernel(const double *__restrict__ GY, const double *__restrict__ Y1,
                            const double *__restrict__ Y0, int64_t len, double s1, double s2,
                            double *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= len) return;
    double v = s1 * GY[i] - s2 * Y1[i];
    if (Y0) v -= Y0[i];
    out[i] = v;
}

// V[i, j] -= u[i] c[j]   (c = u^T V): keeps the block orthogonal to the deflated direction
__global__ void project_out_kernel(double *__restrict__ V, const double *__restrict__ u, const double *__restrict__ c,
                                   int64_t D, int b) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= D * b) return;
    const int64_t r = i / b;
    V[i] -= u[r] * c[i - r * b];
}

// res[l] = || GX[:, l] - w[l] X[:, l] ||  (one block per column, fixed tree)
__global__ void residual_kernel(const double *__restrict__ GX, const double *__restrict__ X,
                                const double *__restrict__ w, int64_t D, int k, double *__restrict__ res) {
    __shared__ double sh[256];
    const int l = blockIdx.x;
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < D; i += 256) {
        const double r = GX[i * k + l] - w[l] * X[i * k + l];
        acc += r * r;
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) res[l] = sqrt(sh[0]);
}

// Z = [u | V]  (D x (b+1))
__global__ void stack_kernel(const double *__restrict__ u, const double *__restrict__ V, int64_t D, int b,
                             double *__restrict__ Z) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= D * (b + 1)) return;
    const int64_t r = i / (b + 1), c = i - r * (b + 1);
    Z[i] = c == 0 ? u[r] : V[r * b + c - 1];
}

// Top-k eigenpairs of the symmetric D x D device matrix G = R^T R: lam (host, k), Psi64
// (device D x k).  u (device, unit norm) is the known top eigenvector r/||r|| of the trivial
// pair lambda = 1 (G r = R'^T 1 = r, since R'[i].r = dinv_i^-2).
//  * b + 1 >= D: one Rayleigh-Ritz step with the full basis = dense eigensolve on the host.
//  * otherwise Chebyshev-filtered block subspace iteration (degree m) on the deflated
//    Gd = G - u u^T with a block V (D x b) kept orthogonal to u, and after every filter a
//    Rayleigh-Ritz step with the FULL G on span([u, V]); stop when the top-k Ritz residuals
//    ||G z - theta z|| (computed explicitly) fall below 1e-9 theta_1 (sin theta <= residual / gap,
//    orders of magnitude below the 1e-4 parity bound and the fp32 rounding of Gamma).  The filter damps [0, theta_min] (theta_min
//    = smallest Ritz value of the block) and amplifies the wanted end of the spectrum; the
//    deflation keeps the lambda = 1 direction from swamping the block.
// Extra columns of the subspace block beyond k (b = k + extra).  The host Rayleigh-Ritz
// eigensolve costs O((b+1)^3) per round; on large (k = 50) extra = 50 / 32 / 24 / 16 all converged in
// the same 5 rounds while the top-k stage took 16.9 / 14.7 / 13.9 / 13.9 ms, so extra = 24 (16 for
// k < 24).  TPO_EIG_EXTRA overrides it within the workspace's bound max(k, 16) (measurement).
int64_t eig_block_extra(int64_t k) {
    if (const char *e = getenv("TPO_EIG_EXTRA")) {
        const int64_t v = atoll(e);
        if (v >= 8 && v <= std::max<int64_t>(k, 16)) return v;   // the workspace is sized for max(k, 16)
    }
    return std::max<int64_t>(16, std::min<int64_t>(k, 24));
}

void gram_topk(const double *G, double *u, int64_t D, int32_t k, std::vector<double> &lam, double *Psi64,
               Arena &ar, cudaStream_t st, int power_steps = 6) {
    const int64_t b = std::min<int64_t>(D - 1, k + eig_block_extra(k));
    if (b + 1 >= D || D <= 64) {
        std::vector<double> gh = to_host(G, D * D, st), w(D), V(D * k);
        host_sym_eig_top(D, gh.data(), k, w.data(), V.data());
        lam.assign(w.begin(), w.begin() + k);
        TPO_CUDA(cudaMemcpyAsync(Psi64, V.data(), sizeof(double) * D * k, cudaMemcpyHostToDevice, st));
        TPO_CUDA(cudaStreamSynchronize(st));
        return;
    }
    const int64_t bz = b + 1;
    double *Gd = ar.take<double>(D * D);
    double *V = ar.take<double>(D * b), *T = ar.take<double>(D * b);
    double *Y0 = ar.take<double>(D * b), *Y1 = ar.take<double>(D * b), *GY = ar.take<double>(D * b);
    double *Z = ar.take<double>(D * bz), *W = ar.take<double>(D * bz);
    double *cvec = ar.take<double>(b);
    // u = r/||r|| is the top eigenvector of the exact Gram; refine it to the top eigenvector of
    // the computed G by a few power steps (rate lambda_2 / lambda_1 ~ 0.03), then deflate
    // Gd = G - lambda_1 u u^T with lambda_1 = u^T G u.
    double *lam1 = ar.take<double>(1);
    int *flag = ar.take<int>(1);
    TPO_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
    for (int it = 0; it < power_steps; ++it) {
        dgemm(false, D, 1, D, 1.0, G, D, u, 1, 0.0, Y0, 1, ar, st);
        power_step_kernel<<<1, 1024, 0, st>>>(Y0, u, D, lam1);
        TPO_LAUNCH_CHECK();
    }
    deflate_kernel<<<cdiv(D * D, 256), 256, 0, st>>>(G, u, lam1, D, Gd);
    TPO_LAUNCH_CHECK();
    std::vector<double> v0(D * b);
    for (int64_t i = 0; i < D * b; ++i) v0[i] = start_entry((uint64_t)i);
    TPO_CUDA(cudaMemcpyAsync(V, v0.data(), sizeof(double) * D * b, cudaMemcpyHostToDevice, st));
    auto orth_against_u = [&]() {
        const size_t m2 = ar.off;
        dgemm(true, 1, b, D, 1.0, u, 1, V, b, 0.0, cvec, b, ar, st);
        ar.off = m2;
        project_out_kernel<<<cdiv(D * b, 256), 256, 0, st>>>(V, u, cvec, D, (int)b);
        TPO_LAUNCH_CHECK();
        cholqr2_f64(V, T, D, b, flag, ar, st);
    };
    orth_against_u();
    // 60 rounds; TPO_EIG_MAX_ROUNDS lowers the cap (tests of the no-convergence error only)
    const int max_rounds = [] {
        const char *e = getenv("TPO_EIG_MAX_ROUNDS");
        const int v = e ? atoi(e) : 60;
        return v >= 0 && v <= 60 ? v : 60;
    }();
    int m = 8;
    std::vector<double> w(bz), E(bz * bz);
    double bnd = 0.0;
    // Rayleigh-Ritz (a host eigensolve of the (b+1) x (b+1) projection) only where it can stop the
    // iteration: the residual falls by a steady factor per filter round (measured between the last
    // two Rayleigh-Ritz steps), so rounds whose predicted residual is still above the tolerance
    // filter and re-orthonormalise only; Rayleigh-Ritz runs when the predicted residual reaches the
    // tolerance.  Only for b + 1 >= 64, where the O(b^3) host eigensolve outweighs a filter round
    // (a wrong prediction costs one more round).  Stopping is always decided on explicit residuals.
    int last_rr = -1;
    double last_rel = 0.0, rate = 0.0;
    static const bool trace = getenv("TPO_TRACE_EIG") != nullptr;
    static cudaEvent_t tev[2] = {};   // trace only: created once, reused
    if (trace && !tev[0])
        for (auto &e : tev) TPO_CUDA(cudaEventCreate(&e));
    for (int round = 0; round <= max_rounds; ++round) {
        const auto t_round = std::chrono::steady_clock::now();
        if (trace) TPO_CUDA(cudaEventRecord(tev[0], st));
        if (round > 0) {   // Chebyshev filter p_m(Gd) V, damping [0, bnd]
            const double c = 0.5 * bnd, e = 0.5 * bnd;
            TPO_CUDA(cudaMemcpyAsync(Y0, V, sizeof(double) * D * b, cudaMemcpyDeviceToDevice, st));
            dgemm(false, D, b, D, 1.0, Gd, D, Y0, b, 0.0, GY, b, ar, st);
            cheb_kernel<<<cdiv(D * b, 256), 256, 0, st>>>(GY, Y0, nullptr, D * b, 1.0 / e, c / e, Y1);
            TPO_LAUNCH_CHECK();
            for (int j = 2; j <= m; ++j) {
                dgemm(false, D, b, D, 1.0, Gd, D, Y1, b, 0.0, GY, b, ar, st);
                cheb_kernel<<<cdiv(D * b, 256), 256, 0, st>>>(GY, Y1, Y0, D * b, 2.0 / e, 2.0 * c / e, Y0);
                TPO_LAUNCH_CHECK();
                std::swap(Y0, Y1);
            }
            TPO_CUDA(cudaMemcpyAsync(V, Y1, sizeof(double) * D * b, cudaMemcpyDeviceToDevice, st));
            orth_against_u();
            if (bz >= 64 && round < max_rounds && last_rr >= 1 && rate > 1.0 &&
                last_rel / pow(rate, (double)(round - last_rr)) > 1e-9)
                continue;                                  // predicted residual still above 1e-9
        }
        // Rayleigh-Ritz with the full G on Z = [u, V]
        stack_kernel<<<cdiv(D * bz, 256), 256, 0, st>>>(u, V, D, (int)b, Z);
        TPO_LAUNCH_CHECK();
        dgemm(false, D, bz, D, 1.0, G, D, Z, bz, 0.0, W, bz, ar, st);
        const size_t mark = ar.off;
        double *h = ar.take<double>(bz * bz);
        dgemm(true, bz, bz, D, 1.0, Z, bz, W, bz, 0.0, h, bz, ar, st);
        std::vector<double> H = to_host(h, bz * bz, st);
        host_sym_eig_top(bz, H.data(), bz, w.data(), E.data());
        // explicit residuals r_l = ||G x_l - w_l x_l|| of the top-k Ritz pairs (x = Z e, G x = W e)
        std::vector<double> Ek(bz * k), wk(w.begin(), w.begin() + k);
        for (int64_t a = 0; a < bz; ++a)
            for (int l = 0; l < k; ++l) Ek[a * k + l] = E[a * bz + l];
        double *ek = to_dev(ar, Ek, st), *dw = to_dev(ar, wk, st);
        double *gx = ar.take<double>(D * k), *res = ar.take<double>(k);
        dgemm(false, D, k, bz, 1.0, Z, bz, ek, k, 0.0, Psi64, k, ar, st);   // Ritz vectors x
        dgemm(false, D, k, bz, 1.0, W, bz, ek, k, 0.0, gx, k, ar, st);      // G x
        residual_kernel<<<k, 256, 0, st>>>(gx, Psi64, dw, D, k, res);
        TPO_LAUNCH_CHECK();
        const std::vector<double> rh = to_host(res, k, st);
        double rmax = 0.0;
        for (int l = 0; l < k; ++l) rmax = std::max(rmax, rh[l]);
        if (trace) {
            TPO_CUDA(cudaEventRecord(tev[1], st));
            TPO_CUDA(cudaEventSynchronize(tev[1]));
            float gpu_ms = 0.f;
            TPO_CUDA(cudaEventElapsedTime(&gpu_ms, tev[0], tev[1]));
            const double wall_ms =
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_round).count();
            fprintf(stderr, "[tpo eig] round %d degree %d rmax/w0 %.3e w0 %.6e wk %.6e wk+1 %.6e wb %.6e  "
                            "stream %.3f ms wall %.3f ms\n", round, round > 0 ? m : 0, rmax / fabs(w[0]), w[0],
                    w[k - 1], w[k], w[bz - 1], gpu_ms, wall_ms);
        }
        {
            const double rel = rmax / fabs(w[0]);
            if (last_rr >= 0 && rel > 0.0 && rel < last_rel)
                rate = pow(last_rel / rel, 1.0 / (double)(round - last_rr));
            last_rr = round;
            last_rel = rel;
        }
        if (rmax <= 1e-9 * fabs(w[0]) || round == max_rounds) {
            check_flag(flag, st, "top-k subspace iteration (CholeskyQR2)");
            if (!(rmax <= 1e-9 * fabs(w[0])))
                throw Error(TPO_ENUMERIC, "top-k subspace iteration did not converge in " + std::to_string(max_rounds) +
                                              " rounds: max Ritz residual / lambda_1 = " + std::to_string(rmax / fabs(w[0])));
            lam.assign(w.begin(), w.begin() + k);
            ar.off = mark;
            return;
        }
        bnd = std::max(w[bz - 1], 1e-6 * fabs(w[0]));
        // Degree: the filter grows the top deflated direction by T_m(x1), x1 = (w[1] - c) / e;
        // keep T_m(x1) <= 1e6 so the filtered block stays well conditioned for CholeskyQR2
        // (a wide spectrum converges in a few low-degree rounds anyway).
        {
            const double x1 = std::max(1.0, (w[1] - 0.5 * bnd) / (0.5 * bnd));
            m = 8;
            while (m > 1 && cosh(m * acosh(x1)) > 1e6) --m;
        }
        ar.off = mark;
    }
}

// signs of R8 from the column statistics, on the device (no host round trip)
__global__ void sign_rule_kernel(const double *__restrict__ s, const double *__restrict__ a,
                                 const int64_t *__restrict__ arg, const double *__restrict__ Gamma, int k,
                                 int *__restrict__ sgn) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= k) return;
    if (fabs(s[l]) < 1e-6 * a[l]) sgn[l] = Gamma[arg[l] * k + l] < 0.0 ? -1 : 1;
    else sgn[l] = s[l] < 0.0 ? -1 : 1;
}

// Sign rule R8 on (Gamma, Psi): sum_i Gamma[i,l] >= 0, else (near-zero sums) the sign of the
// largest-magnitude entry (smallest index among ties).  Flips are applied to both factors.
// out32 (optional): write sgn . Gamma rounded to fp32 there instead of flipping Gamma in place.
void apply_sign_rule(double *Gamma, int64_t n, int k, float *Psi, int64_t D, Arena &ar, cudaStream_t st,
                     float *out32 = nullptr) {
    const size_t mark = ar.off;
    const int64_t G = std::max<int64_t>(1, std::min<int64_t>(2 * 148, cdiv(n, 64)));
    const int64_t rows_per = cdiv(n, G);
    double *ps = ar.take<double>(G * k), *pa = ar.take<double>(G * k), *pm = ar.take<double>(G * k);
    int64_t *pi = ar.take<int64_t>(G * k);
    double *s = ar.take<double>(k), *a = ar.take<double>(k);
    int64_t *arg = ar.take<int64_t>(k);
    int *dsg = ar.take<int>(k);
    colstats_part_kernel<<<G, CS_WARPS * 32, 0, st>>>(Gamma, n, k, rows_per, ps, pa, pm, pi);
    TPO_LAUNCH_CHECK();
    colstats_final_kernel<<<cdiv((int64_t)k * 32, 256), 256, 0, st>>>(ps, pa, pm, pi, G, k, s, a, arg);
    TPO_LAUNCH_CHECK();
    sign_rule_kernel<<<cdiv(k, 128), 128, 0, st>>>(s, a, arg, Gamma, k, dsg);
    TPO_LAUNCH_CHECK();
    if (out32) flip_cast_f64_f32<<<cdiv(n * k, 256), 256, 0, st>>>(Gamma, n, k, dsg, out32);
    else flip_cols_f64<<<cdiv(n * k, 256), 256, 0, st>>>(Gamma, n, k, dsg);
    TPO_LAUNCH_CHECK();
    flip_cols_f32<<<cdiv(D * k, 256), 256, 0, st>>>(Psi, D, k, dsg);
    TPO_LAUNCH_CHECK();
    ar.off = mark;
}

// *dev = max |g - I| (one CTA, order-free max)
__global__ void gram_dev_kernel(const double *__restrict__ g, int k, double *__restrict__ dev) {
    __shared__ double sm[256];
    double m = 0.0;
    for (int i = threadIdx.x; i < k * k; i += blockDim.x) {
        const double dv = fabs(g[i] - ((i / k) == (i % k) ? 1.0 : 0.0));
        m = (dv > m || dv != dv) ? dv : m;                 // NaN propagates
    }
    sm[threadIdx.x] = m;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if ((int)threadIdx.x < o) {
            const double a = sm[threadIdx.x], b = sm[threadIdx.x + o];
            sm[threadIdx.x] = (b > a || b != b) ? b : a;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *dev = sm[0];
}

// X[i, :] <- X[i, :] Ci in place for an upper-triangular k x k Ci (k <= 128): a warp per row, the
// row in registers (lane: columns lane + 32 c), Ci in shared memory (entries below the diagonal
// read as 0)
template <int C>
__global__ void __launch_bounds__(256) apply_upper_rows_kernel(double *__restrict__ X, int64_t n, int k,
                                                               const double *__restrict__ Ci) {
    extern __shared__ double cs[];
    for (int i = threadIdx.x; i < k * k; i += blockDim.x) cs[i] = ((i / k) <= (i % k)) ? Ci[i] : 0.0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t row = wid; row < n; row += nw) {
        double x[C], acc[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int l = lane + 32 * c;
            x[c] = l < k ? X[row * k + l] : 0.0;
            acc[c] = 0.0;
        }
#pragma unroll
        for (int c0 = 0; c0 < C; ++c0) {
            for (int j = 0; j < 32; ++j) {
                const int a = 32 * c0 + j;
                if (a >= k) break;
                const double xa = __shfl_sync(0xffffffffu, x[c0], j);
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const int l = lane + 32 * c;
                    if (l < k) acc[c] = fma(xa, cs[a * k + l], acc[c]);
                }
            }
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int l = lane + 32 * c;
            if (l < k) X[row * k + l] = acc[c];
        }
    }
}

void apply_upper_rows(double *X, int64_t n, int k, const double *Ci, cudaStream_t st) {
    if (n == 0) return;
    const size_t smem = sizeof(double) * (size_t)k * k;
    const unsigned grid = (unsigned)std::min<int64_t>(8 * sm_count(), cdiv(n, 8));
#define TPO_AUR(CV)                                                                                          \
    {                                                                                                        \
        TPO_CUDA(cudaFuncSetAttribute(apply_upper_rows_kernel<CV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        apply_upper_rows_kernel<CV><<<grid, 256, smem, st>>>(X, n, k, Ci);                                \
    }
    if (k <= 32) TPO_AUR(1)
    else if (k <= 64) TPO_AUR(2)
    else TPO_AUR(4)
#undef TPO_AUR
    TPO_LAUNCH_CHECK();
}

// CholeskyQR polish of the fp64 n x k Gamma while its Gram is off identity by > 1e-6 (at most
// two corrections): G = Gamma^T Gamma, Ci = S C^{-1} (chol_inv), Gamma <- Gamma Ci (in place).
// The deviation max|G - I| is read back after each Gram: within 1e-6 Gamma is left as is; below
// 1e-2 one correction suffices (CholeskyQR leaves ||Gamma^T Gamma - I|| ~ kappa^2 u with kappa^2
// < 1.03, far below 1e-6), so the second Gram is skipped.
void polish_gamma(double *Gamma, int64_t n, int k, Arena &ar, cudaStream_t st) {
    const size_t mark = ar.off;
    double *g = ar.take<double>((size_t)k * k), *ci = ar.take<double>((size_t)k * k);
    double *dev = ar.take<double>(1);
    int *flag = ar.take<int>(1);
    TPO_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
    for (int pass = 0; pass < 2; ++pass) {
        if (ts64_enabled() && k <= 104) ts_atb_f64(Gamma, k, Gamma, k, n, k, k, g, ar, st);
        else dgemm(true, k, k, n, 1.0, Gamma, k, Gamma, k, 0.0, g, k, ar, st);
        if (k <= 112) {
            chol_inv_device(g, k, ci, flag, st);
        } else {
            std::vector<double> gh = to_host(g, (size_t)k * k, st), C((size_t)k * k), Ci((size_t)k * k);
            if (!host_cholesky_upper(k, gh.data(), C.data()))
                throw Error(TPO_ENUMERIC, "CholeskyQR2 polish: Gamma^T Gamma not positive definite");
            host_upper_inverse(k, C.data(), Ci.data());
            TPO_CUDA(cudaMemcpyAsync(ci, Ci.data(), sizeof(double) * k * k, cudaMemcpyHostToDevice, st));
        }
        gram_dev_kernel<<<1, 256, 0, st>>>(g, k, dev);
        TPO_LAUNCH_CHECK();
        double hdev = 1.0;
        TPO_CUDA(cudaMemcpyAsync(&hdev, dev, sizeof(double), cudaMemcpyDeviceToHost, st));
        TPO_CUDA(cudaStreamSynchronize(st));
        if (hdev <= 1e-6) break;
        if (!ts_xw_inplace_f64(Gamma, n, k, ci, st)) {       // k > 56: two column blocks, out of place
            const size_t m2 = ar.off;
            double *tmp = ar.take<double>((size_t)n * k);
            if (ts_xw_f64(Gamma, n, k, ci, tmp, st))
                TPO_CUDA(cudaMemcpyAsync(Gamma, tmp, sizeof(double) * n * k, cudaMemcpyDeviceToDevice, st));
            else
                apply_upper_rows(Gamma, n, k, ci, st);
            ar.off = m2;
        }
        if (hdev < 1e-2) break;
    }
    check_flag(flag, st, "CholeskyQR2 polish of Gamma");
    ar.off = mark;
}

// One-pass finish of the exact mode when s = 1^T R (D fp64) is known (tpo_run forms it in the dinv
// pass): the polish decision as polish_gamma (one Gram; within 1e-6 of I: W = I, below 1e-2: W =
// Ci, else not handled), R8's column sums of the final Gamma = G64 W from D-space,
// sum_i Gamma[i,l] = ((s^T Psi Sigma^-1) W)_l (exact arithmetic identity), decided on the host; a
// column whose |sum| is below 1e-6 sqrt(n) (where R8's fallback to the largest entry could apply:
// ||Gamma_l||_1 <= sqrt(n) for a unit column) is not handled.  Then Gamma = fp32(G64 W diag(sgn))
// in one fp64-tensor pass (or the sign flip fused with the rounding when W = I), no column-
// statistics pass.  Returns false (nothing written to Gamma) when not handled.
bool finish_fast(double *G64, int64_t n, int k, const double *Psi64, const std::vector<double> &sig,
                 const double *s_colsum, int64_t D, float *Psi, float *Gamma, Arena &ar, cudaStream_t st) {
    if (!ts64_enabled() || k > 104 || n == 0) return false;
    const size_t mark = ar.off;
    double *g = ar.take<double>((size_t)k * k), *ci = ar.take<double>((size_t)k * k);
    double *dev = ar.take<double>(1);
    int *flag = ar.take<int>(1);
    TPO_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
    ts_atb_f64(G64, k, G64, k, n, k, k, g, ar, st);
    if (k > 112) { ar.off = mark; return false; }
    chol_inv_device(g, k, ci, flag, st);
    gram_dev_kernel<<<1, 256, 0, st>>>(g, k, dev);
    TPO_LAUNCH_CHECK();
    double hdev = 1.0;
    int hflag = 0;
    std::vector<double> hs(D), hps((size_t)D * k), hci((size_t)k * k);
    TPO_CUDA(cudaMemcpyAsync(&hdev, dev, sizeof(double), cudaMemcpyDeviceToHost, st));
    TPO_CUDA(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    TPO_CUDA(cudaMemcpyAsync(hs.data(), s_colsum, sizeof(double) * D, cudaMemcpyDeviceToHost, st));
    TPO_CUDA(cudaMemcpyAsync(hps.data(), Psi64, sizeof(double) * D * k, cudaMemcpyDeviceToHost, st));
    TPO_CUDA(cudaMemcpyAsync(hci.data(), ci, sizeof(double) * k * k, cudaMemcpyDeviceToHost, st));
    TPO_CUDA(cudaStreamSynchronize(st));
    const bool ident = hdev <= 1e-6;
    if (!(hdev < 1e-2) || (!ident && hflag)) { ar.off = mark; return false; }   // NaN, far from I, failed pivot
    std::vector<double> t(k, 0.0), cs(k, 0.0);
    for (int64_t j = 0; j < D; ++j) {
        if (!std::isfinite(hs[j])) { ar.off = mark; return false; }           // s not formed
        for (int a = 0; a < k; ++a) t[a] += hs[j] * hps[(size_t)j * k + a];
    }
    for (int a = 0; a < k; ++a) t[a] /= sig[a];
    for (int l = 0; l < k; ++l) {
        if (ident) cs[l] = t[l];
        else
            for (int a = 0; a <= l; ++a) cs[l] += t[a] * hci[(size_t)a * k + l];   // Ci upper triangular
    }
    const double thr = 1e-6 * sqrt((double)n) * 1.01;
    std::vector<int> sg(k);
    for (int l = 0; l < k; ++l) {
        if (!(fabs(cs[l]) >= thr)) { ar.off = mark; return false; }
        sg[l] = cs[l] < 0.0 ? -1 : 1;
    }
    int *dsg = to_dev(ar, sg, st);
    flip_cols_f32<<<cdiv(D * k, 256), 256, 0, st>>>(Psi, D, k, dsg);
    TPO_LAUNCH_CHECK();
    if (ident) {
        flip_cast_f64_f32<<<cdiv(n * k, 256), 256, 0, st>>>(G64, n, k, dsg, Gamma);
        TPO_LAUNCH_CHECK();
    } else {
        for (int a = 0; a < k; ++a)
            for (int l = 0; l < k; ++l) hci[(size_t)a * k + l] = (a <= l ? hci[(size_t)a * k + l] : 0.0) * sg[l];
        double *w = to_dev(ar, hci, st);
        if (!ts_xw_f32out(G64, n, k, w, Gamma, st)) throw Error(TPO_ECUDA, "finish_fast: fp64 tensor path unavailable");
    }
    TPO_CUDA(cudaStreamSynchronize(st));
    ar.off = mark;
    return true;
}

// Psi / sigma column scaling on the device
__global__ void scale_cols_kernel(const double *__restrict__ A, int64_t rows, int k, const double *__restrict__ sig,
                                  double *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= rows * k) return;
    out[i] = A[i] / sig[i % k];
}

// Gamma = diag(dinv) R' Psi64 diag(1/sigma) in fp64, polished and sign-fixed, then rounded to
// fp32; Psi (fp32 out) = Psi64.
// Gamma_in (optional, n x k fp64): the left factor when the mode already has it (Halko: Y E_k);
// otherwise Gamma = R Psi Sigma^{-1} (exact mode: the same factor, the block being full rank).
void finish_factors(const float *Rp, const float *dinv, int64_t n, int64_t D, int k, const double *Psi64,
                    const std::vector<double> &sig, float *Gamma, float *Psi, Arena &ar, cudaStream_t st,
                    double *Gamma_in = nullptr, const int32_t *rowE = nullptr, const double *s_colsum = nullptr) {
    double *G64 = Gamma_in;
    if (!G64) {
        double *sd = to_dev(ar, sig, st);
        double *w = ar.take<double>((size_t)D * k);
        scale_cols_kernel<<<cdiv(D * k, 256), 256, 0, st>>>(Psi64, D, k, sd, w);
        TPO_LAUNCH_CHECK();
        G64 = ar.take<double>((size_t)n * k);
        const RhPlan gp = rh_plan_pre(rowE, Rp, n, D, k, ar, st);     // integer tensor cores when k > 32
        rh_apply(gp, Rp, dinv, w, n, D, k, G64, ar, st);
    }
    cast_f64_f32<<<cdiv(D * k, 256), 256, 0, st>>>(Psi64, D * k, Psi);
    TPO_LAUNCH_CHECK();
    if (s_colsum && !Gamma_in && finish_fast(G64, n, k, Psi64, sig, s_colsum, D, Psi, Gamma, ar, st)) return;
    polish_gamma(G64, n, k, ar, st);
    apply_sign_rule(G64, n, k, Psi, D, ar, st, Gamma);
    TPO_CUDA(cudaStreamSynchronize(st));
}

__global__ void copy2d_kernel(const double *__restrict__ src, int64_t lds, double *__restrict__ dst, int64_t ldd,
                              int64_t rows, int64_t cols, const double *__restrict__ sub, int64_t ldsub) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= rows * cols) return;
    const int64_t r = i / cols, c = i - r * cols;
    double v = src[r * lds + c];
    if (sub) v -= sub[r * ldsub + c];
    dst[r * ldd + c] = v;
}

}  // namespace

// panel width of the device Haar QR (<= 112, the one-CTA Cholesky-inverse limit; since the
// second CholeskyQR pass skips the factorisation, wide panels are fastest: d = 1000 takes
// 2.8 / 3.2 / 5.2 ms with 112 / 64 / 32 columns)
int64_t haar_panel(int64_t d) { return std::min<int64_t>(112, d); }

size_t haar_q_ws_bytes(int64_t d) {
    const int64_t bw = std::min<int64_t>(112, d);
    return 2 * align_up(sizeof(double) * d * d) + 3 * align_up(sizeof(double) * d * bw) +
           2 * align_up(sizeof(double) * bw * bw + 8) + dgemm_ws(d, bw, d) + 8192;
}

// Alg. 1 L6-7 on the device: Q of the unique QR (diag(R) > 0) of the d x d Gaussian G by
// block classical Gram-Schmidt with re-orthogonalisation (BCGS2) over 112-column panels, each
// panel orthonormalised by CholeskyQR2.  R is block upper triangular with upper triangular,
// positive-diagonal blocks, so Q is the same unique factor the host routine returns.  No
// host round trip until the final failure-flag check.
void haar_q_device(const double *G, bool G_on_device, int64_t d, float *Q_out, Arena &ar, cudaStream_t st) {
    const int64_t bw = haar_panel(d);
    double *A = ar.take<double>(d * d), *Q = ar.take<double>(d * d);
    double *P = ar.take<double>(d * bw), *T = ar.take<double>(d * bw), *Cm = ar.take<double>(d * bw);
    int *flag = ar.take<int>(1);
    TPO_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
    TPO_CUDA(cudaMemcpyAsync(A, G, sizeof(double) * d * d, G_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                             st));
    for (int64_t j0 = 0; j0 < d; j0 += bw) {
        const int64_t w = std::min<int64_t>(bw, d - j0);
        copy2d_kernel<<<cdiv(d * w, 256), 256, 0, st>>>(A + j0, d, P, w, d, w, nullptr, 0);
        TPO_LAUNCH_CHECK();
        for (int pass = 0; j0 > 0 && pass < 2; ++pass) {
            dgemm(true, j0, w, d, 1.0, Q, d, P, w, 0.0, Cm, w, ar, st);     // C = Q_<j^T P
            dgemm(false, d, w, j0, -1.0, Q, d, Cm, w, 1.0, P, w, ar, st);   // P -= Q_<j C
        }
        cholqr2_f64(P, T, d, w, flag, ar, st);
        copy2d_kernel<<<cdiv(d * w, 256), 256, 0, st>>>(P, w, Q + j0, d, d, w, nullptr, 0);
        TPO_LAUNCH_CHECK();
    }
    cast_f64_f32<<<cdiv(d * d, 256), 256, 0, st>>>(Q, d * d, Q_out);
    TPO_LAUNCH_CHECK();
    check_flag(flag, st, "Haar rotation (panel CholeskyQR2)");
}

size_t topk_eig_ws_bytes(int64_t n, int64_t D, int32_t k, int32_t mode, int32_t p) {
    const int64_t b = std::min<int64_t>(D, k + std::max<int64_t>(k, 16));
    const int64_t bh = k + p;
    size_t s = 0;
    s += align_up(sizeof(double) * D * D) + gram_tc_ws(n, D);
    s += align_up(sizeof(double) * D * D) + align_up(sizeof(double) * (n + D + 64));
    s += 8 * align_up(sizeof(double) * D * (std::max(b, bh) + 1)) + 8 * align_up(sizeof(double) * (b + 1) * (b + 1) + 8);
    s += 2 * align_up(sizeof(double) * D * k) + 2 * align_up(sizeof(double) * n * k) + dgemm_ws(n, k, k) +
         4 * align_up(sizeof(double) * 2 * 148 * k) + 8 * align_up(sizeof(double) * k * k);
    if (mode == TPO_EIG_HALKO) s += 3 * align_up(sizeof(double) * n * bh) + tsgemm_ws(n, D, bh) + tsgemm_ws(n, bh, bh);
    s += dgemm_ws(std::max(n, D), std::max(b, bh) + 1, 0) + 2 * align_up(sizeof(double) * (std::max(b, bh) + 1) * (std::max(b, bh) + 1));
    s += ts_atb_ws((int)k, (int)k);                      // the polish Gram Gamma^T Gamma (fp64 tensor path)
    s += rh_plan_ws(n) + rh_apply_ws(D, k);              // Gamma = R Psi Sigma^-1 on the integer tensor cores
    return s + 64 * 256;
}

// ---------------------------------------------------------------------------------------
// Pieces of the exact top-k for the row-sharded solver (the caller all-reduces partials).
// ---------------------------------------------------------------------------------------
size_t eig_from_gram_ws(int64_t D, int32_t k) {
    const int64_t b = std::min<int64_t>(D, k + std::max<int64_t>(k, 16));
    return align_up(sizeof(double) * D * D) + 8 * align_up(sizeof(double) * D * (b + 1)) +
           8 * align_up(sizeof(double) * (b + 1) * (b + 1) + 8) + dgemm_ws(D, b + 1, 0) + 2 * align_up(sizeof(double) * D) +
           64 * 256;
}

// Psi64 (D x k) and sigma (host, k) of the top-k eigenpairs of the global Gram G = R^T R, with
// u = r / ||r|| the known top direction (the same routine tpo_topk_eig runs after its Gram).
void eig_from_gram(const double *G, const double *r, int64_t D, int32_t k, double *Psi64, double *sigma, Arena &ar,
                   cudaStream_t st) {
    double *u = ar.take<double>(D);
    int *zflag = ar.take<int>(1);
    TPO_CUDA(cudaMemsetAsync(zflag, 0, sizeof(int), st));
    unit_vec_kernel<<<1, 1024, 0, st>>>(r, u, D, zflag);
    TPO_LAUNCH_CHECK();
    int zh = 0;
    TPO_CUDA(cudaMemcpyAsync(&zh, zflag, sizeof(int), cudaMemcpyDeviceToHost, st));
    TPO_CUDA(cudaStreamSynchronize(st));
    if (zh) throw Error(TPO_ENUMERIC, "top-k: R' has zero column sums");
    std::vector<double> lam;
    gram_topk(G, u, D, k, lam, Psi64, ar, st);
    for (int l = 0; l < k; ++l) {
        sigma[l] = sqrt(std::max(lam[l], 0.0));
        if (!(sigma[l] > 0.0)) throw Error(TPO_ENUMERIC, "top-k: sigma_k is zero (rank(R) < k)");
    }
}

// G64 = diag(dinv) R' Psi64 diag(1/sigma) on the given rows (fp64)
void gamma_rows(const float *Rp, const float *dinv, int64_t n, int64_t D, int k, const double *Psi64,
                const double *sigma, double *G64, Arena &ar, cudaStream_t st) {
    std::vector<double> ph = to_host(Psi64, (size_t)D * k, st);
    for (int64_t j = 0; j < D; ++j)
        for (int l = 0; l < k; ++l) ph[j * k + l] /= sigma[l];
    const size_t mark = ar.off;
    double *w = to_dev(ar, ph, st);
    if (n > 0) tsgemm_AW_f64(Rp, D, dinv, w, n, D, k, G64, k, st);
    TPO_CUDA(cudaStreamSynchronize(st));
    ar.off = mark;
}

// X <- X S C^{-1} for the global k x k Gram g = S^{-1} C^T C S^{-1} (one CholeskyQR step)
void apply_chol(double *X, int64_t n, int k, const double *g, Arena &ar, cudaStream_t st) {
    const size_t mark = ar.off;
    double *ci = ar.take<double>((size_t)k * k);
    int *flag = ar.take<int>(1);
    TPO_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
    if (k <= 112) {
        chol_inv_device(g, k, ci, flag, st);
    } else {
        std::vector<double> gh = to_host(g, (size_t)k * k, st), C((size_t)k * k), Ci((size_t)k * k);
        if (!host_cholesky_upper(k, gh.data(), C.data()))
            throw Error(TPO_ENUMERIC, "CholeskyQR: Gram not positive definite");
        host_upper_inverse(k, C.data(), Ci.data());
        TPO_CUDA(cudaMemcpyAsync(ci, Ci.data(), sizeof(double) * k * k, cudaMemcpyHostToDevice, st));
    }
    if (n > 0) {
        double *tmp = ar.take<double>((size_t)n * k);
        dgemm(false, n, k, k, 1.0, X, k, ci, k, 0.0, tmp, k, ar, st);
        TPO_CUDA(cudaMemcpyAsync(X, tmp, sizeof(double) * n * k, cudaMemcpyDeviceToDevice, st));
    }
    check_flag(flag, st, "CholeskyQR of Gamma");
    ar.off = mark;
}

// per-column sum, sum |x|, max |x| and its (global: + row0) row index over the given rows
void colstats_rows(const double *A, int64_t n, int k, int64_t row0, double *sum, double *abs_sum, double *maxabs,
                   int64_t *argmax, Arena &ar, cudaStream_t st) {
    const size_t mark = ar.off;
    const int64_t G = std::max<int64_t>(1, std::min<int64_t>(2 * 148, cdiv(std::max<int64_t>(n, 1), 64)));
    const int64_t rows_per = cdiv(std::max<int64_t>(n, 1), G);
    double *ps = ar.take<double>(G * k), *pa = ar.take<double>(G * k), *pm = ar.take<double>(G * k);
    int64_t *pi = ar.take<int64_t>(G * k);
    if (n == 0) {
        fill_f64<<<cdiv(G * k, 256), 256, 0, st>>>(ps, G * k, 0.0);
        fill_f64<<<cdiv(G * k, 256), 256, 0, st>>>(pa, G * k, 0.0);
        fill_f64<<<cdiv(G * k, 256), 256, 0, st>>>(pm, G * k, -1.0);
        TPO_LAUNCH_CHECK();
        TPO_CUDA(cudaMemsetAsync(pi, 0, sizeof(int64_t) * G * k, st));
    } else {
        colstats_part_kernel<<<G, CS_WARPS * 32, 0, st>>>(A, n, k, rows_per, ps, pa, pm, pi);
        TPO_LAUNCH_CHECK();
    }
    colstats_final_kernel<<<cdiv((int64_t)k * 32, 256), 256, 0, st>>>(ps, pa, pm, pi, G, k, sum, abs_sum, argmax);
    TPO_LAUNCH_CHECK();
    // max |x| per column: the value at the argmax (read back through the same partials)
    std::vector<double> hpm = to_host(pm, (size_t)(G * k), st);
    std::vector<int64_t> hpi = to_host(pi, (size_t)(G * k), st);
    std::vector<double> mx(k, -1.0);
    std::vector<int64_t> ai(k, INT64_MAX);
    for (int64_t g = 0; g < G; ++g)
        for (int c = 0; c < k; ++c) {
            const double m = hpm[g * k + c];
            const int64_t i = hpi[g * k + c];
            if (m > mx[c] || (m == mx[c] && i < ai[c])) { mx[c] = m; ai[c] = i; }
        }
    for (int c = 0; c < k; ++c) ai[c] = ai[c] == INT64_MAX ? row0 : ai[c] + row0;
    TPO_CUDA(cudaMemcpyAsync(maxabs, mx.data(), sizeof(double) * k, cudaMemcpyHostToDevice, st));
    TPO_CUDA(cudaMemcpyAsync(argmax, ai.data(), sizeof(int64_t) * k, cudaMemcpyHostToDevice, st));
    TPO_CUDA(cudaStreamSynchronize(st));
    ar.off = mark;
}

// flip the columns with signs_host[l] < 0 in G64 (n x k) and Psi (D x k, fp32; from Psi64 when
// given), then round G64 to fp32 Gamma
void gamma_final(double *G64, int64_t n, int k, const int *signs_host, float *Psi, const double *Psi64, int64_t D,
                 float *Gamma, Arena &ar, cudaStream_t st) {
    const size_t mark = ar.off;
    std::vector<int> sg(signs_host, signs_host + k);
    int *dsg = to_dev(ar, sg, st);
    if (Psi64) {
        cast_f64_f32<<<cdiv(D * k, 256), 256, 0, st>>>(Psi64, D * k, Psi);
        TPO_LAUNCH_CHECK();
    }
    flip_cols_f32<<<cdiv(D * k, 256), 256, 0, st>>>(Psi, D, k, dsg);
    TPO_LAUNCH_CHECK();
    if (n > 0) {
        flip_cols_f64<<<cdiv(n * k, 256), 256, 0, st>>>(G64, n, k, dsg);
        TPO_LAUNCH_CHECK();
        cast_f64_f32_k<<<cdiv(n * k, 256), 256, 0, st>>>(G64, n * k, Gamma);
        TPO_LAUNCH_CHECK();
    }
    TPO_CUDA(cudaStreamSynchronize(st));
    ar.off = mark;
}

void topk_eig_impl(const float *Rp, const float *dinv, int64_t n, int64_t D, int32_t k, int32_t mode, int32_t p,
                   int32_t q, const float *Omega, float *Gamma, double *sigma, float *Psi, Arena &ar,
                   cudaStream_t st, const double *r_colsum, RStats rs) {
    std::vector<double> lam;
    double *Psi64 = ar.take<double>(D * k);
    double *halko_gamma = nullptr;              // Halko mode: Gamma = Y E_k
    if (mode == TPO_EIG_EXACT) {
        double *G = ar.take<double>(D * D);
        double *u = ar.take<double>(D);
        const size_t mark = ar.off;
        gram_tc(Rp, dinv, n, D, G, ar, st);
        ar.off = mark;
        {   // u = r / ||r||, r = R'^T 1 (the top eigenvector of the trivial pair)
            double *r = const_cast<double *>(r_colsum);
            if (!r) {
                r = ar.take<double>(D);
                colsum_f64(Rp, n, D, r, ar, st);
            }
            int *zflag = ar.take<int>(1);
            TPO_CUDA(cudaMemsetAsync(zflag, 0, sizeof(int), st));
            unit_vec_kernel<<<1, 1024, 0, st>>>(r, u, D, zflag);
            TPO_LAUNCH_CHECK();
            int zh = 0;
            TPO_CUDA(cudaMemcpyAsync(&zh, zflag, sizeof(int), cudaMemcpyDeviceToHost, st));
            TPO_CUDA(cudaStreamSynchronize(st));
            if (zh) throw Error(TPO_ENUMERIC, "top-k: R' has zero column sums");
            ar.off = mark;
        }
        gram_topk(G, u, D, k, lam, Psi64, ar, st);
    } else {
        // Halko randomised SVD: Y = orth(R Omega); q x Y = orth(R (R^T Y)); B = R^T Y;
        // Rayleigh-Ritz through the eigendecomposition of B^T B = Y^T R R^T Y.
        const int64_t b = k + p;
        std::vector<float> om = to_host(Omega, D * b, st);
        std::vector<double> omd(om.begin(), om.end());
        double *Om = to_dev(ar, omd, st);
        double *Y = ar.take<double>(n * b), *T = ar.take<double>(n * b), *Bm = ar.take<double>(D * b);
        int *flag = ar.take<int>(1);
        TPO_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
        tsgemm_AW_f64(Rp, D, dinv, Om, n, D, b, Y, b, st);
        cholqr2_f64(Y, T, n, b, flag, ar, st);
        for (int it = 0; it < q; ++it) {
            const size_t mark = ar.off;
            tsgemm_AtB_f32f64(Rp, D, dinv, Y, b, n, D, b, Bm, ar, st);
            ar.off = mark;
            tsgemm_AW_f64(Rp, D, dinv, Bm, n, D, b, Y, b, st);
            cholqr2_f64(Y, T, n, b, flag, ar, st);
        }
        check_flag(flag, st, "randomised SVD (CholeskyQR2)");
        const size_t mark = ar.off;
        tsgemm_AtB_f32f64(Rp, D, dinv, Y, b, n, D, b, Bm, ar, st);     // B = R^T Y (D x b)
        double *g = ar.take<double>(b * b);
        tsgemm_AtB_f64f64(Bm, b, Bm, b, D, b, b, g, ar, st);           // B^T B (b x b)
        std::vector<double> gh = to_host(g, b * b, st), w(b), E(b * b);
        host_sym_eig_top(b, gh.data(), b, w.data(), E.data());
        lam.assign(w.begin(), w.begin() + k);
        std::vector<double> Ek(b * k);
        for (int64_t a = 0; a < b; ++a)
            for (int l = 0; l < k; ++l) Ek[a * k + l] = E[a * b + l];
        double *ek = to_dev(ar, Ek, st);
        // Y^T R = U S V^T with U = E, S^2 = w: Psi = V_k = B E_k S_k^{-1} (right singular vectors),
        // Gamma = Y U_k (left singular vectors of the rank-b approximation Y Y^T R, Halko et al.)
        tsgemm_AW_dd(Bm, b, ek, D, b, k, Psi64, k, st);
        std::vector<double> ps = to_host(Psi64, D * k, st);
        for (int64_t j = 0; j < D; ++j)
            for (int l = 0; l < k; ++l) ps[j * k + l] /= sqrt(std::max(w[l], 1e-300));
        TPO_CUDA(cudaMemcpyAsync(Psi64, ps.data(), sizeof(double) * D * k, cudaMemcpyHostToDevice, st));
        halko_gamma = ar.take<double>(n * k);
        dgemm(false, n, k, b, 1.0, Y, b, ek, k, 0.0, halko_gamma, k, ar, st);
        TPO_CUDA(cudaStreamSynchronize(st));
    }
    std::vector<double> sig(k);
    for (int l = 0; l < k; ++l) {
        sig[l] = sqrt(std::max(lam[l], 0.0));
        if (!(sig[l] > 0.0)) throw Error(TPO_ENUMERIC, "top-k: sigma_k is zero (rank(R) < k)");
        sigma[l] = sig[l];
    }
    finish_factors(Rp, dinv, n, D, k, Psi64, sig, Gamma, Psi, ar, st, halko_gamma, rs.rowE, rs.s_colsum);
}

// ---------------------------------------------------------------------------------------
// f3 "R-free" a7: the exact top-k (R7) of R = diag(dinv) R' without a
// materialised R'.  R' rows are recomputed from Zhat (Eq. R-prime; the features
// GEMM is row-local, so every recomputed row is bit-identical to the materialised one) in three
// sweeps of `chunk` rows: (1) r = R'^T 1; (2) dinv = (R' r)^{-1/2} (written out: the ONMF needs
// it) and G = sum_chunks R_c^T R_c (tcgen05 3xTF32 Gram per chunk, fp64 chunk sums added in chunk
// order); (3) Gamma = R Psi Sigma^-1 row by row.  Then the same device eigensolver of G, CholeskyQR
// polish and R8 sign rule as the materialised path.
// ---------------------------------------------------------------------------------------
size_t topk_rfree_ws(int64_t n, int64_t d, int32_t k, int64_t chunk) {
    const int64_t D = 2 * d, C = std::max<int64_t>(1, std::min(n, chunk));
    size_t s = align_up(sizeof(float) * (size_t)C * D) + 3 * align_up(sizeof(double) * D) +
               2 * align_up(sizeof(double) * D * D) + align_up(sizeof(double) * D * k) + align_up(sizeof(double) * n * k);
    s += std::max(std::max(features_ws_bytes(C, d), gram_tc_ws(C, D)), eig_from_gram_ws(D, k));
    s += 2 * align_up(sizeof(double) * n * k) + ts_atb_ws(k, k) + dgemm_ws(n, k, k) + 8 * align_up(sizeof(double) * k * k) +
         8 * align_up(sizeof(double) * 2 * 148 * k) + align_up(sizeof(double) * D * k);
    return s + 64 * 256;
}

namespace {
__global__ void add_to_f64_kernel(double *__restrict__ acc, const double *__restrict__ x, int64_t len) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < len) acc[i] += x[i];
}
}  // namespace

void topk_rfree_impl(const RSource &src, int64_t n, int32_t k, float *Gamma, double *sigma, float *Psi, float *dinv,
                     Arena &ar, cudaStream_t st) {
    const int64_t d = src.d, D = 2 * d, C = std::max<int64_t>(1, std::min(n, src.chunk));
    float *Rc = ar.take<float>((size_t)C * D);
    double *r = ar.take<double>(D), *rp = ar.take<double>(D);
    double *G = ar.take<double>((size_t)D * D), *Gc = ar.take<double>((size_t)D * D);
    double *Psi64 = ar.take<double>((size_t)D * k), *G64 = ar.take<double>((size_t)n * k);
    const size_t mark = ar.off;
    TPO_CUDA(cudaMemsetAsync(r, 0, sizeof(double) * D, st));
    TPO_CUDA(cudaMemsetAsync(G, 0, sizeof(double) * D * D, st));
    for (int64_t c0 = 0; c0 < n; c0 += C) {                 // sweep 1: r = R'^T 1
        const int64_t nc = std::min(C, n - c0);
        features_part(src.Zhat + c0 * d, nc, d, src.Q, Rc, rp, ar, st);
        ar.off = mark;
        add_to_f64_kernel<<<cdiv(D, 256), 256, 0, st>>>(r, rp, D);
        TPO_LAUNCH_CHECK();
    }
    for (int64_t c0 = 0; c0 < n; c0 += C) {                 // sweep 2: dinv, G = R^T R
        const int64_t nc = std::min(C, n - c0);
        features_part(src.Zhat + c0 * d, nc, d, src.Q, Rc, rp, ar, st);
        ar.off = mark;
        dinv_from_r(Rc, nc, D, r, dinv + c0, st);
        gram_tc(Rc, dinv + c0, nc, D, Gc, ar, st);
        ar.off = mark;
        add_to_f64_kernel<<<cdiv(D * D, 256), 256, 0, st>>>(G, Gc, D * D);
        TPO_LAUNCH_CHECK();
    }
    eig_from_gram(G, r, D, k, Psi64, sigma, ar, st);
    ar.off = mark;
    for (int64_t c0 = 0; c0 < n; c0 += C) {                 // sweep 3: Gamma = R Psi Sigma^-1
        const int64_t nc = std::min(C, n - c0);
        features_part(src.Zhat + c0 * d, nc, d, src.Q, Rc, rp, ar, st);
        ar.off = mark;
        gamma_rows(Rc, dinv + c0, nc, D, k, Psi64, sigma, G64 + c0 * k, ar, st);
        ar.off = mark;
    }
    cast_f64_f32<<<cdiv(D * k, 256), 256, 0, st>>>(Psi64, D * k, Psi);
    TPO_LAUNCH_CHECK();
    polish_gamma(G64, n, k, ar, st);
    apply_sign_rule(G64, n, k, Psi, D, ar, st, Gamma);
    TPO_CUDA(cudaStreamSynchronize(st));
}

// a6: out = dinv . R' (R'^T (dinv . Y)), the D x b intermediate summed in fp64.
void affinity_matvec_impl(const float *Rp, const float *dinv, int64_t n, int64_t D, const float *Y, int64_t b,
                          float *out, Arena &ar, cudaStream_t st) {
    if (ts64_enabled() && D % 4 == 0) {                  // fp64 tensor path (DMMA)
        ts_affinity(Rp, dinv, n, D, Y, b, out, ar, st);
        return;
    }
    double *W = ar.take<double>(D * b);
    tsgemm_AtB_f32f32(Rp, D, dinv, Y, b, nullptr, n, D, b, W, ar, st);
    tsgemm_AW_f32(Rp, D, dinv, W, n, D, b, out, b, st);
}

// ---------------------------------------------------------------------------------------
// f1: SVD-based attribute dimension reduction (Sec. 3.2.1, Eq. Xd):
// X' = Gamma Sigma of the exact top-d SVD of X (R14), computed as X Psi with Psi the top-d
// eigenvectors of the d_U x d_U Gram X^T X: the tcgen05 3xTF32 Gram (gram_tc with unit row
// weights), the device subspace iteration of the top-k solver started from the normalised
// column sums of X (refined by 30 power steps, then deflated), X Psi on the fp64 tensor path,
// the sign rule R8 on the columns of X' (X' = Gamma Sigma, so Gamma's rule), rounded to fp32.
// d == d_U is the pass-through X' = X.
// ---------------------------------------------------------------------------------------
__global__ void fill_f32_kernel(float *p, int64_t n, float v) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

size_t svd_reduce_ws_bytes(int64_t n, int64_t du, int64_t d) {
    return topk_eig_ws_bytes(n, du, (int32_t)d, TPO_EIG_EXACT, 0) + align_up(sizeof(double) * n * d) +
           align_up(sizeof(float) * n) + align_up(sizeof(float) * du * d) + align_up(sizeof(double) * du * d) + 4096;
}

void svd_reduce_impl(const float *X, int64_t n, int64_t du, int64_t d, float *Xr, double *sigma_host, Arena &ar,
                     cudaStream_t st) {
    if (d >= du) {
        TPO_CUDA(cudaMemcpyAsync(Xr, X, sizeof(float) * n * du, cudaMemcpyDeviceToDevice, st));
        TPO_CUDA(cudaStreamSynchronize(st));
        return;
    }
    float *ones = ar.take<float>(n);
    double *G = ar.take<double>(du * du), *u = ar.take<double>(du), *r = ar.take<double>(du);
    double *Psi64 = ar.take<double>(du * d), *X64 = ar.take<double>(n * d);
    float *Psi32 = ar.take<float>(du * d);
    int *zflag = ar.take<int>(1);
    fill_f32_kernel<<<cdiv(std::max<int64_t>(n, 1), 256), 256, 0, st>>>(ones, n, 1.0f);
    TPO_LAUNCH_CHECK();
    {
        const size_t mark = ar.off;
        gram_tc(X, ones, n, du, G, ar, st);              // X^T X
        ar.off = mark;
        colsum_f64(X, n, du, r, ar, st);                  // start direction: X^T 1
        ar.off = mark;
    }
    TPO_CUDA(cudaMemsetAsync(zflag, 0, sizeof(int), st));
    unit_vec_kernel<<<1, 1024, 0, st>>>(r, u, du, zflag);
    TPO_LAUNCH_CHECK();
    int zh = 0;
    TPO_CUDA(cudaMemcpyAsync(&zh, zflag, sizeof(int), cudaMemcpyDeviceToHost, st));
    TPO_CUDA(cudaStreamSynchronize(st));
    if (zh) {                                             // zero column sums: start from e_0-ish uniform
        std::vector<double> h((size_t)du, 1.0 / sqrt((double)du));
        TPO_CUDA(cudaMemcpyAsync(u, h.data(), sizeof(double) * du, cudaMemcpyHostToDevice, st));
        TPO_CUDA(cudaStreamSynchronize(st));
    }
    std::vector<double> lam;
    gram_topk(G, u, du, (int32_t)d, lam, Psi64, ar, st, 30);
    if (sigma_host)
        for (int64_t l = 0; l < d; ++l) sigma_host[l] = sqrt(std::max(lam[l], 0.0));
    tsgemm_AW_f64(X, du, nullptr, Psi64, n, du, d, X64, d, st);   // X Psi = Gamma Sigma
    cast_f64_f32<<<cdiv(du * d, 256), 256, 0, st>>>(Psi64, du * d, Psi32);
    TPO_LAUNCH_CHECK();
    apply_sign_rule(X64, n, (int)d, Psi32, du, ar, st, Xr);
    TPO_CUDA(cudaStreamSynchronize(st));
}

}  // namespace tpo
