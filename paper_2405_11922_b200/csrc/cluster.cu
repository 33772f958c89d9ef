// a8-a9: discretisation -- greedy orthogonal NMF (Alg. 2) and NCI
// generation (Alg. 3), fp64 arithmetic (R11), deterministic reductions.
//
// Per ONMF iteration (H first, then Ups; brackets of PAPER.md:564):
//   RtU = R'^T (dinv . Ups), UtU = Ups^T Ups             (split-over-rows fp64 products)
//   H   <- H . max(RtU,0) / (H UtU + eps)                 (h_update_kernel)
//   RH  = dinv . (R' H);  M = Ups^T RH                    (row-tiled product, split product)
//   Ups <- Ups . sqrt(max(RH,0) / (max(Ups M,0) + eps))   (ups_update_kernel, warp per row)
// Per NCI iteration (all on device, no host round trip; a device flag freezes the loop at
// the label fix-point, R10):
//   assign_kernel: l* = argmax_l Ups[i] . Phi[:,l] (ties -> smallest l), changed flag
//   count + per-cluster row sums (fixed row ranges per block, fixed-order reduction)
//   Phi[:,l] = sum_{i in C_l} Ups[i] / sqrt(|C_l|)
#include <math.h>

#include <algorithm>
#include <vector>

#include "tpo_internal.cuh"

namespace tpo {
namespace {

constexpr double EPS = 1e-12;   // R9

// u[l] for a runtime l from a register array (an unrolled select keeps u in registers)
template <int KM>
__device__ __forceinline__ double u_at(const double (&u)[KM], int l) {
    double v = 0.0;
#pragma unroll
    for (int a = 0; a < KM; ++a) v = a == l ? u[a] : v;
    return v;
}

__global__ void init_factors_kernel(const float *__restrict__ Gamma, int64_t n, const float *__restrict__ Psi,
                                    const double *__restrict__ sig, int64_t D, int k, double *__restrict__ U,
                                    double *__restrict__ H) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n * k) {
        const double g = (double)Gamma[i];
        U[i] = (g > 0.0 ? g : 0.0) + EPS;
    }
    if (i < D * k) {
        const double h = (double)Psi[i] * sig[i % k];
        H[i] = (h > 0.0 ? h : 0.0) + EPS;
    }
}

// Hn[j,l] = H[j,l] * max(RtU[j,l],0) / ((H UtU)[j,l] + eps)
__global__ void h_update_kernel(const double *__restrict__ H, const double *__restrict__ RtU,
                                const double *__restrict__ UtU, int64_t D, int k, double *__restrict__ Hn) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= D * k) return;
    const int64_t j = i / k;
    const int l = (int)(i - j * k);
    double s = 0.0;
    for (int a = 0; a < k; ++a) s = __dadd_rn(s, __dmul_rn(H[j * k + a], UtU[(int64_t)a * k + l]));
    const double num = RtU[i] > 0.0 ? RtU[i] : 0.0;
    Hn[i] = __dmul_rn(H[i], num) / __dadd_rn(s, EPS);
}

// Ups[i,l] *= sqrt(max(RH[i,l],0) / (max((Ups M)[i,l],0) + eps)); warp per row, the old row
// and M (k x k) staged in shared memory (k <= 128).
constexpr int UR = 8;     // rows per warp per pass (ups_update_kernel)

__global__ void __launch_bounds__(256) ups_update_kernel(double *__restrict__ U, const double *__restrict__ RH,
                                                         const double *__restrict__ M, int64_t n, int k) {
    extern __shared__ __align__(16) double msh[];    // [k * k] then rowbuf [8][k][UR] (rows innermost)
    double *rowbuf_all = msh + ((k * k + 1) & ~1);   // 16-byte aligned row buffers
    for (int i = threadIdx.x; i < k * k; i += blockDim.x) msh[i] = M[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t r0 = ((int64_t)blockIdx.x * 8 + w) * UR; r0 < n; r0 += (int64_t)gridDim.x * 8 * UR) {
        const int nr = (int)(n - r0 < UR ? n - r0 : UR);
        double *ubw = rowbuf_all + (size_t)w * UR * k;
        for (int e = lane; e < UR * k; e += 32) {        // coalesced read of the UR rows, stored [a][r]
            const int r = e / k, a = e - r * k;
            ubw[a * UR + r] = r < nr ? U[r0 * k + e] : 0.0;
        }
        __syncwarp();
        for (int l = lane; l < k; l += 32) {
            double sv[UR];
#pragma unroll
            for (int r = 0; r < UR; ++r) sv[r] = 0.0;
            for (int a = 0; a < k; ++a) {
                const double m = msh[a * k + l];
                double uv[UR];
#pragma unroll
                for (int r = 0; r < UR; r += 2) {
                    const double2 v2 = *reinterpret_cast<const double2 *>(ubw + a * UR + r);
                    uv[r] = v2.x;
                    uv[r + 1] = v2.y;
                }
#pragma unroll
                for (int r = 0; r < UR; ++r) sv[r] = fma(uv[r], m, sv[r]);
            }
#pragma unroll
            for (int r = 0; r < UR; ++r) {
                if (r >= nr) continue;
                const double rv = RH[(r0 + r) * k + l];
                const double num = rv > 0.0 ? rv : 0.0;
                const double den = (sv[r] > 0.0 ? sv[r] : 0.0) + EPS;
                U[(r0 + r) * k + l] = ubw[l * UR + r] * sqrt(num / den);
            }
        }
        __syncwarp();
    }
}

// The same update, thread per row with the old row in registers (k <= KM <= 64) and M read
// as shared-memory broadcasts; per (row, l) the same operation order (fma chain over a) as
// ups_update_kernel.
template <int KM>
__global__ void __launch_bounds__(256) ups_update_reg_kernel(double *__restrict__ U, const double *__restrict__ RH,
                                                             const double *__restrict__ M, int64_t n, int k) {
    __shared__ double msh[KM * KM];
    for (int i = threadIdx.x; i < k * k; i += blockDim.x) msh[i] = M[i];
    __syncthreads();
    const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (row >= n) return;
    double u[KM];
#pragma unroll
    for (int a = 0; a < KM; ++a) u[a] = a < k ? U[row * k + a] : 0.0;
    int l = 0;
    for (; l + 1 < k; l += 2) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int a = 0; a < KM; ++a)
            if (a < k) {
                s0 = fma(u[a], msh[a * k + l], s0);
                s1 = fma(u[a], msh[a * k + l + 1], s1);
            }
        const double r0 = RH[row * k + l], r1 = RH[row * k + l + 1];
        U[row * k + l] = __dmul_rn(u_at(u, l), sqrt((r0 > 0.0 ? r0 : 0.0) / __dadd_rn(s0 > 0.0 ? s0 : 0.0, EPS)));
        U[row * k + l + 1] =
            __dmul_rn(u_at(u, l + 1), sqrt((r1 > 0.0 ? r1 : 0.0) / __dadd_rn(s1 > 0.0 ? s1 : 0.0, EPS)));
    }
    for (; l < k; ++l) {
        double s0 = 0.0;
#pragma unroll
        for (int a = 0; a < KM; ++a)
            if (a < k) s0 = fma(u[a], msh[a * k + l], s0);
        const double r0 = RH[row * k + l];
        U[row * k + l] = __dmul_rn(u_at(u, l), sqrt((r0 > 0.0 ? r0 : 0.0) / __dadd_rn(s0 > 0.0 ? s0 : 0.0, EPS)));
    }
}

struct NciState {
    int32_t *changed;     // [0]: labels changed in the current iteration
    int32_t *done;        // [0]: fix-point reached (freezes the remaining iterations)
    int32_t *iters;       // [0]: iterations run
};

// l* = argmax_l sum_a Ups[i,a] Phi[a,l]; warp per row, Phi and the row in smem.
constexpr int AR = 8;     // rows per warp per pass (assign_kernel)

__global__ void __launch_bounds__(256) assign_kernel(const double *__restrict__ U, const double *__restrict__ Phi,
                                                     int64_t n, int k, int32_t *__restrict__ labels, NciState s) {
    if (*s.done) return;
    extern __shared__ __align__(16) double phs[];         // [k * k] then rowbuf [8][AR][k]
    double *rowbuf_all = phs + k * k;
    for (int i = threadIdx.x; i < k * k; i += blockDim.x) phs[i] = Phi[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    bool changed = false;
    // AR rows per warp at a time: each Phi element read from smem serves AR rows
    for (int64_t r0 = ((int64_t)blockIdx.x * 8 + w) * AR; r0 < n; r0 += (int64_t)gridDim.x * 8 * AR) {
        const int nr = (int)(n - r0 < AR ? n - r0 : AR);
        double *ubw = rowbuf_all + (size_t)w * AR * k;
        for (int r = 0; r < AR; ++r)
            for (int l = lane; l < k; l += 32) ubw[r * k + l] = r < nr ? U[(r0 + r) * k + l] : 0.0;
        __syncwarp();
        double best[AR];
        int arg[AR];
#pragma unroll
        for (int r = 0; r < AR; ++r) { best[r] = 0.0; arg[r] = 0x7fffffff; }
        for (int l = lane; l < k; l += 32) {
            double sc[AR];
#pragma unroll
            for (int r = 0; r < AR; ++r) sc[r] = 0.0;
            for (int a = 0; a < k; ++a) {
                const double ph = phs[a * k + l];
#pragma unroll
                for (int r = 0; r < AR; ++r) sc[r] = fma(ubw[r * k + a], ph, sc[r]);
            }
#pragma unroll
            for (int r = 0; r < AR; ++r)
                if (arg[r] == 0x7fffffff || sc[r] > best[r]) { best[r] = sc[r]; arg[r] = l; }
        }
#pragma unroll
        for (int r = 0; r < AR; ++r) {
            // warp argmax: larger score wins; equal scores -> smaller index
            for (int o = 16; o; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best[r], o);
                const int oa = __shfl_xor_sync(0xffffffffu, arg[r], o);
                if (oa != 0x7fffffff && (arg[r] == 0x7fffffff || ob > best[r] || (ob == best[r] && oa < arg[r]))) {
                    best[r] = ob;
                    arg[r] = oa;
                }
            }
            if (lane == 0 && r < nr) {
                if (labels[r0 + r] != arg[r]) changed = true;
                labels[r0 + r] = arg[r];
            }
        }
        __syncwarp();
    }
    if (changed) *s.changed = 1;
}

// Small-k variant (k <= 16): one thread per row, the row of Ups in registers, Phi in smem
// (same arithmetic and summation order as assign_kernel).
template <int KM>
__global__ void __launch_bounds__(128) assign_small_kernel(const double *__restrict__ U, const double *__restrict__ Phi,
                                                           int64_t n, int k, int32_t *__restrict__ labels, NciState s) {
    if (*s.done) return;
    __shared__ double phs[KM * KM];
    for (int i = threadIdx.x; i < k * k; i += blockDim.x) phs[i] = Phi[i];
    __syncthreads();
    const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (row >= n) return;
    double u[KM];
#pragma unroll
    for (int a = 0; a < KM; ++a) u[a] = a < k ? U[row * k + a] : 0.0;
    double best = 0.0;
    int arg = 0;
    int l = 0;
    for (; l + 3 < k; l += 4) {                 // four scores at once (independent chains)
        double sc0 = 0.0, sc1 = 0.0, sc2 = 0.0, sc3 = 0.0;
#pragma unroll
        for (int a = 0; a < KM; ++a)
            if (a < k) {
                const double ua = u[a];
                sc0 = fma(ua, phs[a * k + l], sc0);
                sc1 = fma(ua, phs[a * k + l + 1], sc1);
                sc2 = fma(ua, phs[a * k + l + 2], sc2);
                sc3 = fma(ua, phs[a * k + l + 3], sc3);
            }
        if (l == 0 || sc0 > best) { best = sc0; arg = l; }
        if (sc1 > best) { best = sc1; arg = l + 1; }
        if (sc2 > best) { best = sc2; arg = l + 2; }
        if (sc3 > best) { best = sc3; arg = l + 3; }
    }
    for (; l < k; ++l) {
        double sc = 0.0;
#pragma unroll
        for (int a = 0; a < KM; ++a)
            if (a < k) sc = fma(u[a], phs[a * k + l], sc);
        if (l == 0 || sc > best) { best = sc; arg = l; }
    }
    if (labels[row] != arg) *s.changed = 1;
    labels[row] = arg;
}

// Fused Alg. 3 pass for k <= KM <= 32: l*_i = argmax_l (Ups Phi)[i, l] (thread per row, the row
// in registers, Phi in smem; same arithmetic order as assign_kernel) AND the per-cluster sums
// of the next Phi in the same read of Ups.  Each warp owns a contiguous run of rows and adds
// them in row order into its own smem accumulators (lanes over columns); the warps of a block
// are combined in warp order -> part[b][l][a], cpart[b][l] (deterministic).
template <int KM, int NW>
__global__ void __launch_bounds__(NW * 32) nci_fused_kernel(const double *__restrict__ U, const double *__restrict__ Phi,
                                                        int64_t n, int k, int64_t rows_per_block,
                                                        int32_t *__restrict__ labels, NciState s,
                                                        double *__restrict__ part, int64_t *__restrict__ cpart) {
    if (*s.done) return;
    constexpr int NT = NW * 32;
    __shared__ double phs[KM * KM];
    __shared__ double acc[NW][KM][KM];
    __shared__ int cnt[NW][KM];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    for (int i = t; i < k * k; i += NT) phs[i] = Phi[i];
    for (int i = t; i < NW * KM * KM; i += NT) (&acc[0][0][0])[i] = 0.0;
    for (int i = t; i < NW * KM; i += NT) (&cnt[0][0])[i] = 0;
    __syncthreads();
    const int64_t b0 = blockIdx.x * rows_per_block, b1 = min(n, b0 + rows_per_block);
    const int64_t per_w = (rows_per_block + NW - 1) / NW;
    const int64_t w0 = min(b1, b0 + w * per_w), w1 = min(b1, w0 + per_w);
    bool changed = false;
    for (int64_t c0 = w0; c0 < w1; c0 += 32) {
        const int64_t row = c0 + lane;
        const bool ok = row < w1;
        double u[KM];
#pragma unroll
        for (int a = 0; a < KM; ++a) u[a] = (ok && a < k) ? U[row * k + a] : 0.0;
        double best = 0.0;
        int arg = 0;
        for (int l = 0; l < k; ++l) {
            double sc = 0.0;
#pragma unroll
            for (int a = 0; a < KM; ++a)
                if (a < k) sc = fma(u[a], phs[a * k + l], sc);   // fused multiply-add, as the oracle
            if (l == 0 || sc > best) { best = sc; arg = l; }
        }
        if (ok) {
            if (labels[row] != arg) changed = true;
            labels[row] = arg;
        }
        const int nr = (int)(w1 - c0 < 32 ? w1 - c0 : 32);
        for (int r = 0; r < nr; ++r) {          // rows in order: acc[l][a] += Ups[row, a]
            const int l = __shfl_sync(0xffffffffu, arg, r);
            if (lane < k) acc[w][l][lane] += U[(c0 + r) * k + lane];
            if (lane == 0) cnt[w][l] += 1;
            __syncwarp();
        }
    }
    if (__any_sync(0xffffffffu, changed) && lane == 0) *s.changed = 1;
    __syncthreads();
    for (int i = t; i < k * k; i += NT) {
        const int l = i / k, a = i - l * k;
        double v = 0.0;
        for (int ww = 0; ww < NW; ++ww) v += acc[ww][l][a];
        part[blockIdx.x * (int64_t)k * k + i] = v;
    }
    for (int l = t; l < k; l += NT) {
        int64_t c = 0;
        for (int ww = 0; ww < NW; ++ww) c += cnt[ww][l];
        cpart[blockIdx.x * (int64_t)k + l] = c;
    }
}

__global__ void nci_step_kernel(NciState s, int32_t *__restrict__ counts, int k) {
    // runs after assign: advance the iteration counter, freeze on a fix-point
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        if (!*s.done) {
            *s.iters += 1;
            if (!*s.changed) *s.done = 1;
            *s.changed = 0;
        }
    }
    (void)counts; (void)k;
}

// Per-block cluster sums over a fixed row range (k > 32 path): grid (blocks, 32-column chunks);
// each warp owns a contiguous run of the block's rows and adds them in row order into its own
// smem accumulators acc[w][l][lane] (lane = column of the chunk); warps are combined in order
// -> part[b][l][a], cpart[b][l] (deterministic, no atomics).
__global__ void cluster_sums_kernel(const double *__restrict__ U, const int32_t *__restrict__ labels, int64_t n,
                                    int k, int64_t rows_per_block, int nw, double *__restrict__ part,
                                    int64_t *__restrict__ cpart, const int32_t *__restrict__ done) {
    if (*done) return;
    extern __shared__ double sh[];
    double *acc = sh;                                          // [nw][k][32]
    int *cnt = reinterpret_cast<int *>(acc + (size_t)nw * k * 32);   // [nw][k]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nt = blockDim.x;
    for (int i = threadIdx.x; i < nw * k * 32; i += nt) acc[i] = 0.0;
    for (int i = threadIdx.x; i < nw * k; i += nt) cnt[i] = 0;
    __syncthreads();
    const int a = blockIdx.y * 32 + lane;
    const bool act = a < k;
    const int64_t b0 = blockIdx.x * rows_per_block, b1 = min(n, b0 + rows_per_block);
    const int64_t per_w = (rows_per_block + nw - 1) / nw;
    const int64_t w0 = min(b1, b0 + w * per_w), w1 = min(b1, w0 + per_w);
    double *my = acc + (size_t)w * k * 32 + lane;
    int *myc = cnt + w * k;
    int64_t i = w0;
    constexpr int CU = 16;                 // rows in flight per warp (the pass is memory-latency bound)
    for (; i + CU <= w1; i += CU) {
        int l[CU];
        double v[CU];
#pragma unroll
        for (int u = 0; u < CU; ++u) {
            l[u] = labels[i + u];
            v[u] = act ? U[(i + u) * k + a] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < CU; ++u) {
            my[l[u] * 32] += v[u];
            if (lane == 0 && blockIdx.y == 0) myc[l[u]] += 1;
        }
    }
    for (; i < w1; ++i) {
        const int l = labels[i];
        my[l * 32] += act ? U[i * k + a] : 0.0;
        if (lane == 0 && blockIdx.y == 0) myc[l] += 1;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < k * 32; e += nt) {
        const int l = e / 32, c = e % 32, col = blockIdx.y * 32 + c;
        if (col >= k) continue;
        double v = 0.0;
        for (int ww = 0; ww < nw; ++ww) v += acc[((size_t)ww * k + l) * 32 + c];
        part[blockIdx.x * (int64_t)k * k + (int64_t)l * k + col] = v;
    }
    if (blockIdx.y == 0)
        for (int l = threadIdx.x; l < k; l += nt) {
            int64_t c = 0;
            for (int ww = 0; ww < nw; ++ww) c += cnt[ww * k + l];
            cpart[blockIdx.x * (int64_t)k + l] = c;
        }
}

// Phi[a,l] = (sum_b part[b][l][a]) / sqrt(count_l)   (zero column for an empty cluster);
// one warp per entry, lanes stride the blocks, fixed shuffle tree.
__global__ void phi_kernel(const double *__restrict__ part, const int64_t *__restrict__ cpart, int64_t nb, int k,
                           double *__restrict__ Phi, const int32_t *__restrict__ done) {
    if (*done) return;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= (int64_t)k * k) return;
    const int l = (int)(wid / k), a = (int)(wid - (int64_t)l * k);
    double s = 0.0;
    int64_t c = 0;
    for (int64_t b = lane; b < nb; b += 32) {
        s += part[b * (int64_t)k * k + (int64_t)l * k + a];
        c += cpart[b * (int64_t)k + l];
    }
    for (int o = 16; o; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if (lane == 0) Phi[(int64_t)a * k + l] = c > 0 ? s / sqrt((double)c) : 0.0;
}

__global__ void fill_i32(int32_t *p, int64_t n, int32_t v) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

__global__ void eye_kernel(double *P, int k) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < k * k) P[i] = (i / k == i % k) ? 1.0 : 0.0;
}

int64_t cluster_rows_per_block(int64_t n) { return std::max<int64_t>(64, cdiv(std::max<int64_t>(n, 1), 4 * 148)); }

}  // namespace

// ---------------------------------------------------------------------------------------
// Pieces of Alg. 2 / Alg. 3 for the row-sharded solver (the caller all-reduces partials).
// ---------------------------------------------------------------------------------------
void onmf_init(const float *Gamma, int64_t n, const float *Psi, const double *sigma_host, int64_t D, int k, double *U,
               double *H, Arena &ar, cudaStream_t st) {
    const size_t mark = ar.off;
    double *sig = ar.take<double>(k);
    TPO_CUDA(cudaMemcpyAsync(sig, sigma_host, sizeof(double) * k, cudaMemcpyHostToDevice, st));
    const int64_t mx = std::max(n, D) * k;
    init_factors_kernel<<<cdiv(std::max<int64_t>(mx, 1), 256), 256, 0, st>>>(Gamma, n, Psi, sig, D, k, U, H);
    TPO_LAUNCH_CHECK();
    TPO_CUDA(cudaStreamSynchronize(st));
    ar.off = mark;
}

void onmf_h_update(double *H, const double *RtU, const double *UtU, int64_t D, int k, Arena &ar, cudaStream_t st) {
    const size_t mark = ar.off;
    double *Hn = ar.take<double>(D * k);
    h_update_kernel<<<cdiv(D * k, 256), 256, 0, st>>>(H, RtU, UtU, D, k, Hn);
    TPO_LAUNCH_CHECK();
    TPO_CUDA(cudaMemcpyAsync(H, Hn, sizeof(double) * D * k, cudaMemcpyDeviceToDevice, st));
    TPO_CUDA(cudaStreamSynchronize(st));
    ar.off = mark;
}

void onmf_u_update(double *U, const double *RH, const double *M, int64_t n, int k, cudaStream_t st) {
    if (n == 0) return;
    if (ts64_ups_enabled(k)) {
        ts_ups_update(U, RH, M, n, k, st);
        return;
    }
    if (k <= 16) {
        ups_update_reg_kernel<16><<<cdiv(n, 256), 256, 0, st>>>(U, RH, M, n, k);
    } else {
        const size_t ups_smem = sizeof(double) * ((size_t)k * k + 1 + (size_t)8 * UR * k);
        TPO_CUDA(cudaFuncSetAttribute(ups_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ups_smem));
        ups_update_kernel<<<(unsigned)std::min<int64_t>(cdiv(n, 8 * UR), 148 * 8), 256, ups_smem, st>>>(U, RH, M, n, k);
    }
    TPO_LAUNCH_CHECK();
}

// sums[l][a] = sum over the block partials, counts[l] (fp64) -- fixed order
__global__ void sums_reduce_kernel(const double *__restrict__ part, const int64_t *__restrict__ cpart, int64_t nb,
                                   int k, double *__restrict__ sums, double *__restrict__ counts) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < (int64_t)k * k) {
        double s = 0.0;
        for (int64_t b = 0; b < nb; ++b) s += part[b * (int64_t)k * k + i];
        sums[i] = s;
    }
    if (i < k) {
        int64_t c = 0;
        for (int64_t b = 0; b < nb; ++b) c += cpart[b * (int64_t)k + i];
        counts[i] = (double)c;
    }
}

// Phi[a][l] = sums[l][a] / sqrt(counts[l]) (zero column for an empty cluster)
__global__ void phi_from_sums_kernel(const double *__restrict__ sums, const double *__restrict__ counts, int k,
                                     double *__restrict__ Phi) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k * k) return;
    const int l = i / k, a = i - l * k;
    Phi[(int64_t)a * k + l] = counts[l] > 0.0 ? sums[i] / sqrt(counts[l]) : 0.0;
}

size_t nci_assign_part_ws(int64_t n, int k) {
    const int64_t nb = cdiv(std::max<int64_t>(n, 1), std::max<int64_t>(256, cdiv(cdiv(std::max<int64_t>(n, 1), 2 * 148), 256) * 256));
    return align_up(sizeof(double) * nb * k * k) + align_up(sizeof(int64_t) * nb * k) + 4 * 256;
}

// Alg. 3 assign on the shard's rows with the current Phi: labels, changed flag (device int,
// set to 1 when a label changes; the caller zeroes it), and the shard's cluster sums / counts.
void nci_assign_part(const double *U, const double *Phi, int64_t n, int k, int32_t *labels, int32_t *changed,
                     double *sums, double *counts, Arena &ar, cudaStream_t st) {
    const size_t mark = ar.off;
    int32_t *zero = ar.take<int32_t>(2);
    TPO_CUDA(cudaMemsetAsync(zero, 0, sizeof(int32_t) * 2, st));
    NciState s{changed, zero, zero + 1};
    const int64_t rpf = std::max<int64_t>(256, cdiv(cdiv(std::max<int64_t>(n, 1), 2 * 148), 256) * 256);
    const int64_t nbf = cdiv(std::max<int64_t>(n, 1), rpf);
    double *part = ar.take<double>(nbf * k * k);
    int64_t *cpart = ar.take<int64_t>(nbf * k);
    if (n == 0) {
        TPO_CUDA(cudaMemsetAsync(part, 0, sizeof(double) * nbf * k * k, st));
        TPO_CUDA(cudaMemsetAsync(cpart, 0, sizeof(int64_t) * nbf * k, st));
    } else if (k <= 32) {
        if (k <= 8) nci_fused_kernel<8, 8><<<nbf, 256, 0, st>>>(U, Phi, n, k, rpf, labels, s, part, cpart);
        else if (k <= 16) nci_fused_kernel<16, 8><<<nbf, 256, 0, st>>>(U, Phi, n, k, rpf, labels, s, part, cpart);
        else nci_fused_kernel<32, 4><<<nbf, 128, 0, st>>>(U, Phi, n, k, rpf, labels, s, part, cpart);
        TPO_LAUNCH_CHECK();
    } else {
        if (ts64_enabled() && k <= 104) {   // certified argmax on the fp64 tensor path (R13), as tpo_run's loop
            ts_assign(U, Phi, n, k, labels, s.changed, s.done, st);
        } else if (k <= 64) {
            assign_small_kernel<64><<<cdiv(n, 128), 128, 0, st>>>(U, Phi, n, k, labels, s);
        } else {
            const size_t phi_smem = sizeof(double) * ((size_t)k * k + (size_t)8 * AR * k);
            TPO_CUDA(cudaFuncSetAttribute(assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)phi_smem));
            assign_kernel<<<(unsigned)std::min<int64_t>(cdiv(n, 8 * AR), 148 * 8), 256, phi_smem, st>>>(U, Phi, n, k,
                                                                                                  labels, s);
        }
        TPO_LAUNCH_CHECK();
        const int sum_nw = (int)std::max<int64_t>(1, std::min<int64_t>(8, (200 * 1024) / ((int64_t)k * (32 * 8 + 4))));
        const size_t sum_smem = (size_t)sum_nw * k * (32 * sizeof(double) + sizeof(int));
        TPO_CUDA(cudaFuncSetAttribute(cluster_sums_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sum_smem));
        cluster_sums_kernel<<<dim3((unsigned)nbf, (unsigned)cdiv(k, 32)), sum_nw * 32, sum_smem, st>>>(
            U, labels, n, k, rpf, sum_nw, part, cpart, s.done);
        TPO_LAUNCH_CHECK();
    }
    sums_reduce_kernel<<<cdiv((int64_t)k * k, 256), 256, 0, st>>>(part, cpart, nbf, k, sums, counts);
    TPO_LAUNCH_CHECK();
    TPO_CUDA(cudaStreamSynchronize(st));
    ar.off = mark;
}

void nci_phi(const double *sums, const double *counts, int k, double *Phi, cudaStream_t st) {
    phi_from_sums_kernel<<<cdiv(k * k, 256), 256, 0, st>>>(sums, counts, k, Phi);
    TPO_LAUNCH_CHECK();
}

size_t cluster_ws_bytes(int64_t n, int64_t D, int32_t k) {
    Arena ar(nullptr, 0);
    ar.take<double>(n * k);          // Ups
    ar.take<double>(n * k);          // RH
    ar.take<double>(D * k * 2);      // H, Hn
    ar.take<double>(D * k);          // RtU
    ar.take<double>(k * k * 3);      // UtU, M, Phi
    ar.take<double>(k);
    ar.take<int32_t>(8);
    const int64_t nb = cdiv(std::max<int64_t>(n, 1), cluster_rows_per_block(n));
    ar.take<double>(nb * k * k);
    ar.take<int64_t>(nb * k);
    ar.take<char>(rh_plan_ws(n));
    ar.take<uint32_t>(D);
    size_t inner = std::max(std::max(std::max(onmf_ws_bytes(n, D, k), std::max(dgemm_ws(k, k, n), dgemm_ws(k, k, D))),
                                     ts_atb_ws(k, k)),
                            rh_apply_ws(D, k));
    if (oz_assign_supported(k)) inner = std::max(inner, oz_assign_ws(n, k));
    return ar.off + inner + 4096;
}

namespace {
__global__ void acc_f64_kernel(double *__restrict__ acc, const double *__restrict__ x, int64_t len) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < len) acc[i] += x[i];
}

int64_t rfree_chunk(const RSource &s, int64_t n) { return std::max<int64_t>(1, std::min(n, s.chunk)); }

// f3 Alg. 2 RtU = R'^T (dinv . Ups) (Eq. update-Q / update-Y) with R' rows
// recomputed from Zhat chunk by chunk (bit-identical rows: the features GEMM is row-local); the
// chunks' fp64 partials (fp64 tensor path) are added in chunk order, so the sum is deterministic
void rfree_rtu(const RSource &s, const float *dinv, const double *U, int64_t n, int64_t D, int k, double *RtU, Arena &ar,
               cudaStream_t st) {
    const int64_t C = rfree_chunk(s, n);
    const size_t mark0 = ar.off;
    float *Rc = ar.take<float>((size_t)C * D);
    double *rp = ar.take<double>(D), *Pc = ar.take<double>((size_t)D * k);
    const size_t mark = ar.off;
    TPO_CUDA(cudaMemsetAsync(RtU, 0, sizeof(double) * D * k, st));
    for (int64_t c0 = 0; c0 < n; c0 += C) {
        const int64_t nc = std::min(C, n - c0);
        features_part(s.Zhat + c0 * s.d, nc, s.d, s.Q, Rc, rp, ar, st);
        ar.off = mark;
        ts_rtu(Rc, nc, D, dinv + c0, U + c0 * k, k, Pc, ar, st);
        ar.off = mark;
        acc_f64_kernel<<<cdiv(D * k, 256), 256, 0, st>>>(RtU, Pc, D * k);
        TPO_LAUNCH_CHECK();
    }
    ar.off = mark0;
}

// f3 Alg. 2 RH = dinv . (R'H), row-local: each chunk's rows from its recomputed R' rows
void rfree_rh(const RSource &s, const float *dinv, const double *H, int64_t n, int64_t D, int k, double *RH, Arena &ar,
              cudaStream_t st) {
    const int64_t C = rfree_chunk(s, n);
    const size_t mark0 = ar.off;
    float *Rc = ar.take<float>((size_t)C * D);
    double *rp = ar.take<double>(D);
    const size_t mark = ar.off;
    for (int64_t c0 = 0; c0 < n; c0 += C) {
        const int64_t nc = std::min(C, n - c0);
        features_part(s.Zhat + c0 * s.d, nc, s.d, s.Q, Rc, rp, ar, st);
        ar.off = mark;
        rh_apply(RhPlan(), Rc, dinv + c0, H, nc, D, k, RH + c0 * k, ar, st);
        ar.off = mark;
    }
    ar.off = mark0;
}
}  // namespace

size_t rfree_pass_ws(int64_t n, int64_t d, int32_t k, int64_t chunk) {
    const int64_t D = 2 * d, C = std::max<int64_t>(1, std::min(n, chunk));
    return align_up(sizeof(float) * (size_t)C * D) + align_up(sizeof(double) * D) + align_up(sizeof(double) * D * k) +
           std::max(features_ws_bytes(C, d), ts_rtu_ws(0, D, k)) + 4096;
}

void cluster_impl(const float *Rp, const float *dinv, int64_t n, int64_t D, int32_t k, const float *Gamma,
                  const double *sigma, const float *Psi, int32_t Tf, int32_t Tg, int32_t *labels,
                  int32_t *iters_used, Arena &ar, cudaStream_t st, RStats rs, const RSource *src) {
    double *U = ar.take<double>(n * k);
    double *RH = ar.take<double>(n * k);
    double *H = ar.take<double>(D * k), *Hn = ar.take<double>(D * k);
    double *RtU = ar.take<double>(D * k);
    double *UtU = ar.take<double>(k * k), *M = ar.take<double>(k * k), *Phi = ar.take<double>(k * k);
    double *sig = ar.take<double>(k);
    int32_t *flags = ar.take<int32_t>(8);
    const int64_t rpb = cluster_rows_per_block(n);
    const int64_t nb = cdiv(std::max<int64_t>(n, 1), rpb);
    double *part = ar.take<double>(nb * k * k);
    int64_t *cpart = ar.take<int64_t>(nb * k);
    const RhPlan rhp = src ? RhPlan() : rh_plan_pre(rs.rowE, Rp, n, D, k, ar, st);
    const uint32_t *featmax = nullptr;                     // R''s per-feature maxima (oz R^T Ups), once per solve
    if (!src && oz_rtu_supported(n, D, k)) {
        if (rs.featmax) {
            featmax = rs.featmax;
        } else {
            uint32_t *fm = ar.take<uint32_t>(D);
            oz_featmax(Rp, n, D, fm, st);
            featmax = fm;
        }
    }
    const size_t mark = ar.off;

    TPO_CUDA(cudaMemcpyAsync(sig, sigma, sizeof(double) * k, cudaMemcpyHostToDevice, st));
    const int64_t mx = std::max(n, D) * k;
    init_factors_kernel<<<cdiv(mx, 256), 256, 0, st>>>(Gamma, n, Psi, sig, D, k, U, H);
    TPO_LAUNCH_CHECK();
    const size_t ups_smem = sizeof(double) * ((size_t)k * k + 1 + (size_t)8 * UR * k);
    TPO_CUDA(cudaFuncSetAttribute(ups_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ups_smem));
    for (int t = 0; t < Tf; ++t) {
        if (src) rfree_rtu(*src, dinv, U, n, D, k, RtU, ar, st);
        else onmf_rtu(Rp, n, D, dinv, U, k, RtU, ar, st, featmax);
        ar.off = mark;
        if (ts64_enabled() && k <= 104) ts_atb_f64(U, k, U, k, n, k, k, UtU, ar, st);
        else dgemm(true, k, k, n, 1.0, U, k, U, k, 0.0, UtU, k, ar, st);
        ar.off = mark;
        h_update_kernel<<<cdiv(D * k, 256), 256, 0, st>>>(H, RtU, UtU, D, k, Hn);
        TPO_LAUNCH_CHECK();
        std::swap(H, Hn);
        if (src) rfree_rh(*src, dinv, H, n, D, k, RH, ar, st);
        else rh_apply(rhp, Rp, dinv, H, n, D, k, RH, ar, st);
        ar.off = mark;
        // M = Ups^T (R H) = (R^T Ups)^T H = RtU^T H: the same product by associativity, from the
        // D x k factors instead of a pass over the n x k rows (RtU was formed from this Ups)
        dgemm(true, k, k, D, 1.0, RtU, k, H, k, 0.0, M, k, ar, st);
        ar.off = mark;
        if (ts64_ups_enabled(k)) {
            ts_ups_update(U, RH, M, n, k, st);
        } else {
            if (k <= 16)
                ups_update_reg_kernel<16><<<cdiv(n, 256), 256, 0, st>>>(U, RH, M, n, k);
            else
                ups_update_kernel<<<(unsigned)std::min<int64_t>(cdiv(n, 8 * UR), 148 * 8), 256, ups_smem, st>>>(U, RH, M,
                                                                                                              n, k);
            TPO_LAUNCH_CHECK();
        }
    }
    // Alg. 3
    ar.off = mark;
    const bool oa_on = oz_assign_supported(k);
    OzAssign oa;
    if (oa_on) oa = oz_assign_prepare(U, n, k, ar, st);      // Ups is fixed during Alg. 3
    NciState s{flags, flags + 1, flags + 2};
    TPO_CUDA(cudaMemsetAsync(flags, 0, sizeof(int32_t) * 8, st));
    fill_i32<<<cdiv(n, 256), 256, 0, st>>>(labels, n, -1);
    TPO_LAUNCH_CHECK();
    eye_kernel<<<cdiv(k * k, 256), 256, 0, st>>>(Phi, k);
    TPO_LAUNCH_CHECK();
    const size_t phi_smem = sizeof(double) * ((size_t)k * k + (size_t)8 * AR * k);
    const int sum_nw = (int)std::max<int64_t>(1, std::min<int64_t>(8, (200 * 1024) / ((int64_t)k * (32 * 8 + 4))));
    const size_t sum_smem = (size_t)sum_nw * k * (32 * sizeof(double) + sizeof(int));
    TPO_CUDA(cudaFuncSetAttribute(assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)phi_smem));
    TPO_CUDA(cudaFuncSetAttribute(cluster_sums_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sum_smem));
    // rows per block for the sums / fused passes: whole 32-row runs per warp, ~4 blocks per SM
    const int64_t rpf = std::max<int64_t>(rpb, cdiv(cdiv(n, 4 * 148), 256) * 256);
    const int64_t nbf = cdiv(n, rpf);
    for (int t = 0; t < Tg; ++t) {
        const bool last = t == Tg - 1;           // the last Phi update is never used
        if (k <= 32 && !last) {
            if (k <= 8) nci_fused_kernel<8, 8><<<nbf, 256, 0, st>>>(U, Phi, n, k, rpf, labels, s, part, cpart);
            else if (k <= 16) nci_fused_kernel<16, 8><<<nbf, 256, 0, st>>>(U, Phi, n, k, rpf, labels, s, part, cpart);
            else nci_fused_kernel<32, 4><<<nbf, 128, 0, st>>>(U, Phi, n, k, rpf, labels, s, part, cpart);
            TPO_LAUNCH_CHECK();
            nci_step_kernel<<<1, 32, 0, st>>>(s, nullptr, k);
            TPO_LAUNCH_CHECK();
            phi_kernel<<<cdiv((int64_t)k * k * 32, 256), 256, 0, st>>>(part, cpart, nbf, k, Phi, s.done);
            TPO_LAUNCH_CHECK();
            continue;
        }
        if (oa_on) {
            oz_assign(oa, U, Phi, labels, s.changed, s.done, st);
        } else if (ts64_enabled() && k > 32 && k <= 104) {
            ts_assign(U, Phi, n, k, labels, s.changed, s.done, st);
        } else {
            if (k <= 16)
                assign_small_kernel<16><<<cdiv(n, 128), 128, 0, st>>>(U, Phi, n, k, labels, s);
            else if (k <= 32)
                assign_small_kernel<32><<<cdiv(n, 128), 128, 0, st>>>(U, Phi, n, k, labels, s);
            else if (k <= 64)
                assign_small_kernel<64><<<cdiv(n, 128), 128, 0, st>>>(U, Phi, n, k, labels, s);
            else
                assign_kernel<<<(unsigned)std::min<int64_t>(cdiv(n, 8 * AR), 148 * 8), 256, phi_smem, st>>>(U, Phi, n,
                                                                                                      k, labels, s);
            TPO_LAUNCH_CHECK();
        }
        nci_step_kernel<<<1, 32, 0, st>>>(s, nullptr, k);
        TPO_LAUNCH_CHECK();
        if (last) break;
        cluster_sums_kernel<<<dim3((unsigned)nbf, (unsigned)cdiv(k, 32)), sum_nw * 32, sum_smem, st>>>(
            U, labels, n, k, rpf, sum_nw, part, cpart, s.done);
        TPO_LAUNCH_CHECK();
        phi_kernel<<<cdiv((int64_t)k * k * 32, 256), 256, 0, st>>>(part, cpart, nbf, k, Phi, s.done);
        TPO_LAUNCH_CHECK();
    }
    int32_t it = 0;
    TPO_CUDA(cudaMemcpyAsync(&it, s.iters, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    TPO_CUDA(cudaStreamSynchronize(st));
    if (iters_used) *iters_used = it;
}

}  // namespace tpo
