// a8: the two passes over R' of one greedy-orthogonal-NMF iteration (Alg. 2, PAPER.md:536-547;
// products bracketed as PAPER.md:564 so the n x n affinity is never formed), fp64 arithmetic
// (R11) with fp32 R' widened on load:
//
//   onmf_rtu:  RtU[a, l] = sum_i R'[i, a] (dinv_i Ups[i, l])          (D x k, reduce over n)
//              grid = (row groups, column blocks, k chunks); a thread owns CPT columns of R'
//              (coalesced loads, 4 rows in flight) and KC columns of Ups (dinv.Ups staged in
//              shared memory, read as broadcasts): CPT x KC fp64 accumulators.  Each CTA writes
//              an fp64 partial; onmf_reduce adds the row groups in order (deterministic).
//   (RH[i, l] = dinv_i sum_a R'[i, a] H[a, l] is tsgemm_AW_f64 in dense.cu.)
//
// Both are fp64-FMA bound on B200 (64 DFMA/clk/SM): n D k FMAs per pass.
#include <stdlib.h>

#include <algorithm>

#include "tpo_internal.cuh"

namespace tpo {
namespace {

constexpr int NTR = 128;                    // onmf_rtu block: 128 threads x CPT columns
constexpr int RT = 64;                      // rows of dinv.Ups staged per tile (onmf_rtu)

// part[g] = R'^T (dinv . U) over the rows of split g, with the R' rows and the Ups / dinv rows
// staged through an RS-stage cp.async ring (RTS rows per stage): the loads of the next stages
// are in flight while a stage is multiplied (a direct-load kernel keeping 4 rows per thread in
// flight was MLP-bound on HBM).  Per (column, l) the rows are accumulated in row order.
constexpr int RTS = 8, RS = 4;
__device__ __forceinline__ void cpa16(void *sm, const void *g, bool v) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(g), "r"(v ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cpa8(void *sm, const void *g, bool v) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(g), "r"(v ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cpa4(void *sm, const void *g, bool v) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(g), "r"(v ? 4 : 0) : "memory");
}
template <int CPT, int KC>
constexpr size_t rtu_pipe_smem() {
    return (size_t)RS * (RTS * NTR * CPT * 4 + RTS * KC * 8 + RTS * 4);
}

template <int CPT, int KC>
__global__ void __launch_bounds__(NTR, 2) onmf_rtu_pipe_kernel(const float *__restrict__ Rp, int64_t n, int D,
                                                              const float *__restrict__ dinv,
                                                              const double *__restrict__ U, int k, int64_t rows_per,
                                                              double *__restrict__ part) {
    constexpr int W = NTR * CPT;                      // columns of the block
    extern __shared__ __align__(16) uint8_t rsm[];
    float *Rs = reinterpret_cast<float *>(rsm);                                   // [RS][RTS][W]
    double *Ys = reinterpret_cast<double *>(rsm + (size_t)RS * RTS * W * 4);       // [RS][RTS][KC]
    float *ds = reinterpret_cast<float *>(rsm + (size_t)RS * (RTS * W * 4 + RTS * KC * 8));   // [RS][RTS]
    const int t = threadIdx.x;
    const int64_t g = blockIdx.x;
    const int a0 = blockIdx.y * W;
    const int k0 = blockIdx.z * KC;
    const int kc = min(KC, k - k0);
    const int64_t r0 = g * rows_per, r1 = min(n, r0 + rows_per);
    const int nst = (int)((r1 - r0 + RTS - 1) / RTS);
    const bool vec = (D % 4 == 0) && (a0 % 4 == 0);
    auto load = [&](int s) {
        const int buf = s % RS;
        const int64_t tb = r0 + (int64_t)s * RTS;
        float *R = Rs + (size_t)buf * RTS * W;
        if (vec) {
            for (int e = t; e < RTS * W / 4; e += NTR) {
                const int r = e / (W / 4), c4 = (e - r * (W / 4)) * 4;
                const bool v = tb + r < r1 && a0 + c4 < D;
                cpa16(R + r * W + c4, v ? (const void *)(Rp + (tb + r) * D + a0 + c4) : (const void *)Rp, v);
            }
        } else {
            for (int e = t; e < RTS * W; e += NTR) {
                const int r = e / W, c = e - r * W;
                const bool v = tb + r < r1 && a0 + c < D;
                cpa4(R + r * W + c, v ? (const void *)(Rp + (tb + r) * D + a0 + c) : (const void *)Rp, v);
            }
        }
        double *Y = Ys + (size_t)buf * RTS * KC;
        for (int e = t; e < RTS * KC; e += NTR) {
            const int r = e / KC, l = e - r * KC;
            const bool v = tb + r < r1 && l < kc;
            cpa8(Y + e, v ? (const void *)(U + (tb + r) * k + k0 + l) : (const void *)U, v);
        }
        if (t < RTS) {
            const bool v = tb + t < r1;
            cpa4(ds + buf * RTS + t, v ? (const void *)(dinv + tb + t) : (const void *)dinv, v);
        }
    };
    int col[CPT];
    bool cv[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        col[c] = a0 + t + NTR * c;
        cv[c] = col[c] < D;
    }
    double acc[CPT][KC];
#pragma unroll
    for (int c = 0; c < CPT; ++c)
#pragma unroll
        for (int l = 0; l < KC; ++l) acc[c][l] = 0.0;
#pragma unroll
    for (int s = 0; s < RS - 1; ++s) {
        if (s < nst) load(s);
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int s = 0; s < nst; ++s) {
        asm volatile("cp.async.wait_group %0;" ::"n"(RS - 2) : "memory");
        __syncthreads();
        const int buf = s % RS;
        double *Y = Ys + (size_t)buf * RTS * KC;
        for (int e = t; e < RTS * KC; e += NTR) Y[e] = (double)ds[buf * RTS + e / KC] * Y[e];   // dinv . Ups
        __syncthreads();
        if (s + RS - 1 < nst) load(s + RS - 1);
        asm volatile("cp.async.commit_group;" ::: "memory");
        const float *R = Rs + (size_t)buf * RTS * W;
#pragma unroll 2
        for (int r = 0; r < RTS; ++r) {
            double rv[CPT];
#pragma unroll
            for (int c = 0; c < CPT; ++c) rv[c] = (double)R[r * W + t + NTR * c];
#pragma unroll
            for (int l = 0; l < KC; ++l) {
                const double y = Y[r * KC + l];
#pragma unroll
                for (int c = 0; c < CPT; ++c) acc[c][l] = fma(rv[c], y, acc[c][l]);
            }
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        if (!cv[c]) continue;
#pragma unroll
        for (int l = 0; l < KC; ++l)
            if (l < kc) part[(g * D + col[c]) * (int64_t)k + k0 + l] = acc[c][l];
    }
}

// out[i] = sum_g part[g][i]: 8 independent partial sums (g mod 8) combined in a fixed order
__global__ void onmf_reduce_kernel(const double *__restrict__ part, int64_t G, int64_t len, double *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= len) return;
    double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int64_t g = 0;
    for (; g + 8 <= G; g += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) s[j] += part[(g + j) * len + i];
    for (; g < G; ++g) s[g & 7] += part[g * len + i];
    out[i] = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
}


// k-chunk widths that are instantiated (a chunk is padded up to the next one)
constexpr int KCS[] = {2, 4, 5, 8, 10, 12, 16, 20, 26, 32, 50};

int pick_kc(int need) {
    for (int v : KCS)
        if (v >= need) return v;
    return 50;
}

struct RtuPlan {
    int kc, nkc, cpt, ncb;
    int64_t G, rows_per;
};

RtuPlan rtu_plan(int64_t n, int D, int k) {
    RtuPlan p;
    // k chunks of <= 26 columns: each broadcast smem read of dinv.Ups feeds CPT FMAs, so a thread
    // owns >= 2 columns of R' whenever D allows (CPT x KC <= 64 accumulators: 2 CTAs / SM)
    p.nkc = (k + 25) / 26;
    p.kc = pick_kc((k + p.nkc - 1) / p.nkc);
    const int want = (D + NTR - 1) / NTR;               // columns per thread to cover D in one block
    const int cap = std::max(1, std::min(8, 64 / p.kc));
    int cpt = 1;
    while (cpt < want && cpt * 2 <= cap) cpt *= 2;
    p.cpt = cpt;
    p.ncb = (D + NTR * cpt - 1) / (NTR * cpt);
    const int64_t tiles = (int64_t)p.ncb * p.nkc;
    const int64_t want_g = std::max<int64_t>(1, (2 * 148 + tiles - 1) / tiles);   // one wave at 2 CTAs / SM (pipelined kernel)
    p.G = std::max<int64_t>(1, std::min<int64_t>(want_g, (std::max<int64_t>(n, 1) + RT - 1) / RT));
    p.rows_per = cdiv(cdiv(std::max<int64_t>(n, 1), p.G), 4) * 4;
    p.G = cdiv(std::max<int64_t>(n, 1), p.rows_per);
    return p;
}

template <int KC>
void launch_rtu(const RtuPlan &p, const float *Rp, int64_t n, int D, const float *dinv, const double *U, int k,
                double *part, cudaStream_t st) {
    const dim3 grid((unsigned)p.G, (unsigned)p.ncb, (unsigned)p.nkc);
    // only CPT x KC <= 64 (or CPT = 1) is planned (rtu_plan); the other combinations are not instantiated
    constexpr int C8 = 8 * KC <= 64 ? 8 : 1, C4 = 4 * KC <= 64 ? 4 : 1, C2 = 2 * KC <= 64 ? 2 : 1;
#define TPO_RTU_PIPE(CPTV)                                                                                   \
    {                                                                                                        \
        constexpr size_t sm = rtu_pipe_smem<CPTV, KC>();                                                     \
        TPO_CUDA(cudaFuncSetAttribute(onmf_rtu_pipe_kernel<CPTV, KC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
        onmf_rtu_pipe_kernel<CPTV, KC><<<grid, NTR, sm, st>>>(Rp, n, D, dinv, U, k, p.rows_per, part);      \
    }
    switch (p.cpt) {
        case 1: TPO_RTU_PIPE(1) break;
        case 2: TPO_RTU_PIPE(C2) break;
        case 4: TPO_RTU_PIPE(C4) break;
        default: TPO_RTU_PIPE(C8) break;
    }
#undef TPO_RTU_PIPE
    TPO_LAUNCH_CHECK();
}


#define TPO_KC_SWITCH(kc, F, ...)                      \
    switch (kc) {                                      \
        case 2: F<2>(__VA_ARGS__); break;              \
        case 4: F<4>(__VA_ARGS__); break;              \
        case 5: F<5>(__VA_ARGS__); break;              \
        case 8: F<8>(__VA_ARGS__); break;              \
        case 10: F<10>(__VA_ARGS__); break;            \
        case 12: F<12>(__VA_ARGS__); break;            \
        case 16: F<16>(__VA_ARGS__); break;            \
        case 20: F<20>(__VA_ARGS__); break;            \
        case 26: F<26>(__VA_ARGS__); break;            \
        case 32: F<32>(__VA_ARGS__); break;            \
        default: F<50>(__VA_ARGS__); break;            \
    }

}  // namespace

size_t onmf_ws_bytes(int64_t n, int64_t D, int32_t k) {
    const RtuPlan p = rtu_plan(n, (int)D, k);
    return std::max(std::max(align_up(sizeof(double) * (size_t)(p.G * D * k) + 1) + 256, ts_rtu_ws(n, D, k)),
                    align_up(sizeof(uint32_t) * (size_t)D + 1) + oz_rtu_ws(n, D, k));
}

// RtU = R'^T (dinv . U)   (D x k, fp64).  featmax (optional, from oz_featmax): R''s per-feature
// maxima when the caller keeps them across the iterations of one solve.
void onmf_rtu(const float *Rp, int64_t n, int64_t D, const float *dinv, const double *U, int k, double *RtU, Arena &ar,
              cudaStream_t st, const uint32_t *featmax, const unsigned long long *colmax) {
    if (dinv && oz_rtu_supported(n, D, k) && (reinterpret_cast<uintptr_t>(Rp) & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(U) & 15) == 0 && (reinterpret_cast<uintptr_t>(dinv) & 15) == 0) {
        const size_t mark = ar.off;
        if (!featmax) {
            uint32_t *fm = ar.take<uint32_t>(D);
            oz_featmax(Rp, n, D, fm, st);
            featmax = fm;
        }
        oz_rtu(Rp, n, D, dinv, U, k, featmax, RtU, ar, st, colmax);    // integer tensor cores (R16)
        ar.off = mark;
        return;
    }
    if (ts64_enabled()) {
        ts_rtu(Rp, n, D, dinv, U, k, RtU, ar, st);
        return;
    }
    const RtuPlan p = rtu_plan(n, (int)D, k);
    const size_t mark = ar.off;
    double *part = ar.take<double>(p.G * D * k);
    TPO_KC_SWITCH(p.kc, launch_rtu, p, Rp, n, (int)D, dinv, U, k, part, st);
    onmf_reduce_kernel<<<cdiv(D * k, 256), 256, 0, st>>>(part, p.G, D * k, RtU);
    TPO_LAUNCH_CHECK();
    ar.off = mark;
}


}  // namespace tpo
