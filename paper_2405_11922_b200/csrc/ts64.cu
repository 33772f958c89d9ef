// Tall-skinny fp64 products of the discretisation on the FP64 tensor path (DMMA,
// mma.sync.m8n8k4.f64): a7's Gamma = dinv . (R' Psi) / sigma (Eq. init-HY) and
// a8's Alg. 2 passes RtU = R'^T (dinv . Ups) (Eq. update-Q numerator),
// RH = dinv . (R' H) and the Ups update with den = Ups M (Eq. update-Y).
//
// R11 keeps the discretisation in fp64 arithmetic.  The B200's fp64 peak is the same on DFMA and
// DMMA (36-37 TFLOP/s measured), but a register-tiled DFMA kernel issues one
// instruction per 32 multiply-adds and plateaued at ~45 % of the fp64 pipe (issue / register
// bandwidth, profiles/r02_*); one DMMA does 256, so the fragments are fed from shared memory with
// a few loads per MMA.  fp32 operands (R') are staged as fp32 and widened when the fragment is
// loaded (1 conversion per 8 multiply-adds).  Every sum has a fixed order: deterministic.
// (Alg. 3's argmax scores keep their sequential fma order -- R13, bit-compared with the
// oracle -- and stay on the CUDA-core kernels of cluster.cu.)
#include <math.h>

#include <algorithm>
#include <type_traits>

#include "tpo_internal.cuh"

namespace tpo {
namespace {

constexpr double EPS_R9 = 1e-12;    // R9
constexpr int DM_NT = 256;          // 8 warps
constexpr int DM_BM = 256;          // rows per tile: 8 warps x 32 (4 m-tiles of 8)
constexpr int DM_BK = 32;           // K per stage (8 k-steps of 4)

enum { DM_STORE = 0, DM_UPS = 1, DM_ASSIGN = 2 };

struct DmArgs {
    const void *A;        // n x K (fp32 or fp64), leading dimension lda
    int64_t lda;
    const float *rs;      // STORE: row scale (dinv) or null
    const double *W;      // K x N, leading dimension ldw
    int64_t ldw;
    int64_t n;
    int K, N;
    double *out;          // STORE: n x N (ldo); UPS: Ups itself (= A, updated in place)
    float *out32;         // STORE: when set, the product is written as fp32 here instead of out
    int64_t ldo;
    const double *cs;     // STORE: column divisors (sigma) or null
    const double *RH;     // UPS: n x N
    int32_t *labels;      // ASSIGN: labels out; changed flag set when one changes; skipped when *done
    int32_t *changed;
    const int32_t *done;
};

// Alg. 3 certified argmax: the tensor-path scores of a row are accepted when their top-2 margin
// exceeds CERT_TOL relative to the best score (Ups and Phi are nonnegative, so every score carries a
// relative error <= k * 2^-53 ~ 1e-14 in either summation order); a row below it is rescored with
// the sequential fma of R13 (the oracle's arithmetic), so the labels are the oracle's.
constexpr double CERT_TOL = 1e-11;

__device__ __forceinline__ void top2_merge(double &b1, int &i1, double &b2, double v, int iv) {
    // (b1, i1): best (ties -> smaller index); b2: second-best value
    if (iv < 0) return;
    if (i1 < 0 || v > b1 || (v == b1 && iv < i1)) {
        if (i1 >= 0) b2 = fmax(b2, b1);
        b1 = v;
        i1 = iv;
    } else {
        b2 = fmax(b2, v);
    }
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(void *sm, const void *g, int bytes) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp8(void *sm, const void *g, bool v) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(g), "r"(v ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp4(void *sm, const void *g, bool v) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(g), "r"(v ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ uint32_t sm32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    uint64_t spins = 0;
    while (true) {
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.b32 %0, 1, 0, p;\n}\n"
                     : "=r"(done)
                     : "r"(sm32(bar)), "r"(parity)
                     : "memory");
        if (done) return;
        if (++spins > (1ull << 31)) __trap();            // watchdog: never hang the GPU
    }
}
// shared memory -> one contiguous global block (bulk-copy engine), tracked by bulk groups
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(sm32(src)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// one contiguous global block -> shared memory through the bulk-copy (1-D TMA) engine
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sm32(dst)),
                 "l"(src), "r"(bytes), "r"(sm32(bar))
                 : "memory");
}
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// A tile rows padded by 4 elements: the 8 rows x 4 columns of an m8n8k4 A fragment then hit
// distinct banks (fp32) / the minimum two wavefronts (fp64)
constexpr int DM_LDA = DM_BK + 4;

template <class TA, int NT>
constexpr size_t dm_smem() {
    return 2 * ((size_t)DM_BM * DM_LDA * sizeof(TA) + (size_t)DM_BK * 8 * NT * sizeof(double));
}

// out[i, l] = epi( sum_j A[i, j] W[j, l] ) for 256-row tiles (static round robin) and the column
// block [col0, col0 + 8 NT) (grid.y).  Warp w owns rows w*32 .. w*32+31 of a tile: 4 m-tiles x NT
// n-tiles of m8n8k4 accumulators.  The (tile, K-stage) steps form one cp.async pipeline.
template <class TA, int EPI, int NT>
__global__ void __launch_bounds__(DM_NT, 1) dm_rowgemm_kernel(DmArgs a) {
    if (EPI == DM_ASSIGN && *a.done) return;
    extern __shared__ __align__(16) unsigned char dsm[];
    constexpr int LDA = DM_LDA;
    constexpr int NBW = 8 * NT;
    TA *As = reinterpret_cast<TA *>(dsm);                                  // [2][DM_BM][LDA]
    double *Ws = reinterpret_cast<double *>(dsm + 2 * (size_t)DM_BM * LDA * sizeof(TA));   // [2][DM_BK][NBW]
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int gr = lane >> 2, gc = lane & 3;
    const int col0 = blockIdx.y * NBW;
    const TA *A = static_cast<const TA *>(a.A);
    const int nst = (a.K + DM_BK - 1) / DM_BK;
    const int64_t ntiles = (a.n + DM_BM - 1) / DM_BM;
    const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t Q = my_tiles * nst;
    const bool a16 = sizeof(TA) == 4 && (a.lda % 4) == 0 && ((reinterpret_cast<uintptr_t>(A) & 15u) == 0);
    const bool d16 = sizeof(TA) == 8 && (a.lda % 2) == 0 && ((reinterpret_cast<uintptr_t>(A) & 15u) == 0);
    auto load = [&](int64_t q, int buf) {
        const int64_t r0 = (blockIdx.x + (q / nst) * gridDim.x) * DM_BM;
        const int k0 = (int)(q % nst) * DM_BK;
        TA *as = As + (size_t)buf * DM_BM * LDA;
        double *ws = Ws + (size_t)buf * DM_BK * NBW;
        if (a16) {                          // fp32 rows in 16-byte chunks (8 per row)
#pragma unroll
            for (int i = 0; i < DM_BM * 8 / DM_NT; ++i) {
                const int c = tid + DM_NT * i, r = c >> 3, part = c & 7;
                const int64_t row = r0 + r;
                const int kc = k0 + part * 4;
                const int bytes = row < a.n ? 4 * max(0, min(4, a.K - kc)) : 0;
                cp16(as + r * LDA + part * 4, bytes ? (const void *)(A + row * a.lda + kc) : (const void *)A, bytes);
            }
        } else if (d16) {                   // fp64 rows in 16-byte chunks (16 per row): half the copies
#pragma unroll 4
            for (int i = 0; i < DM_BM * 16 / DM_NT; ++i) {
                const int c = tid + DM_NT * i, r = c >> 4, part = c & 15;
                const int64_t row = r0 + r;
                const int kc = k0 + part * 2;
                const int bytes = row < a.n ? 8 * max(0, min(2, a.K - kc)) : 0;
                cp16(as + r * LDA + part * 2, bytes ? (const void *)(A + row * a.lda + kc) : (const void *)A, bytes);
            }
        } else {                            // element copies (unaligned fp64 or fp32)
#pragma unroll 4
            for (int i = 0; i < DM_BM * DM_BK / DM_NT; ++i) {
                const int idx = tid + DM_NT * i, r = idx >> 5, c = idx & 31;
                const int64_t row = r0 + r;
                const bool v = row < a.n && k0 + c < a.K;
                if (sizeof(TA) == 8) cp8(as + r * LDA + c, v ? (const void *)(A + row * a.lda + k0 + c) : (const void *)A, v);
                else cp4(as + r * LDA + c, v ? (const void *)(A + row * a.lda + k0 + c) : (const void *)A, v);
            }
        }
        for (int idx = tid; idx < DM_BK * NBW; idx += DM_NT) {
            const int r = idx / NBW, c = idx - (idx / NBW) * NBW;
            const bool v = k0 + r < a.K && col0 + c < a.N;
            cp8(ws + idx, v ? a.W + (int64_t)(k0 + r) * a.ldw + col0 + c : a.W, v);
        }
        cp_commit();
    };
    double acc[4][NT][2];
    if (Q > 0) {
        load(0, 0);
        cp_wait_all();
        __syncthreads();
    }
    for (int64_t q = 0; q < Q; ++q) {
        const int buf = (int)(q & 1);
        const int s = (int)(q % nst);
        const int64_t r0 = (blockIdx.x + (q / nst) * gridDim.x) * DM_BM;
        if (q + 1 < Q) load(q + 1, buf ^ 1);
        if (s == 0) {
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
        }
        const TA *as = As + (size_t)buf * DM_BM * LDA + (w * 32 + gr) * LDA + gc;
        const double *ws = Ws + (size_t)buf * DM_BK * NBW + gc * NBW + gr;
#pragma unroll
        for (int k4 = 0; k4 < DM_BK / 4; ++k4) {
            double af[4], bf[NT];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) af[mt] = (double)as[mt * 8 * LDA + k4 * 4];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) bf[nt] = ws[k4 * 4 * NBW + nt * 8];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt], af[mt], bf[nt]);
        }
        if (EPI == DM_ASSIGN && s == nst - 1) {
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                const int64_t row = r0 + w * 32 + mt * 8 + gr;
                double b1 = 0.0, b2 = -1.0;
                int i1 = -1;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int col = nt * 8 + 2 * gc + h;
                        top2_merge(b1, i1, b2, acc[mt][nt][h], col < a.N ? col : -1);
                    }
#pragma unroll
                for (int o = 1; o < 4; o <<= 1) {       // the 4 lanes of this row (gc = 0..3)
                    const double ob1 = __shfl_xor_sync(0xffffffffu, b1, o), ob2 = __shfl_xor_sync(0xffffffffu, b2, o);
                    const int oi1 = __shfl_xor_sync(0xffffffffu, i1, o);
                    top2_merge(b1, i1, b2, ob1, oi1);
                    b2 = fmax(b2, ob2);
                }
                if (gc == 0 && row < a.n) {
                    int lab = i1;
                    if (!(b1 - b2 > CERT_TOL * fabs(b1))) {   // near tie (or a tie): R13 rescoring
                        const double *u = static_cast<const double *>(a.A) + row * a.lda;
                        double best = 0.0;
                        lab = 0;
                        for (int l = 0; l < a.N; ++l) {
                            double sc = 0.0;
                            for (int j = 0; j < a.K; ++j) sc = fma(u[j], a.W[(int64_t)j * a.ldw + l], sc);
                            if (l == 0 || sc > best) { best = sc; lab = l; }
                        }
                    }
                    if (a.labels[row] != lab) *a.changed = 1;
                    a.labels[row] = lab;
                }
            }
        }
        if (EPI != DM_ASSIGN && s == nst - 1) {   // epilogue of the tile: C[gr][2 gc + h] of each 8 x 8 tile
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                const int64_t row = r0 + w * 32 + mt * 8 + gr;
                if (row >= a.n) continue;
                const double rsv = (EPI == DM_STORE && a.rs) ? (double)a.rs[row] : 1.0;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int col = col0 + nt * 8 + 2 * gc + h;
                        if (col >= a.N) continue;
                        if (EPI == DM_STORE) {
                            double v = rsv * acc[mt][nt][h];
                            if (a.cs) v = v / a.cs[col];
                            if (a.out32) a.out32[row * a.ldo + col] = (float)v;
                            else a.out[row * a.ldo + col] = v;
                        } else {
                            const double rh = a.RH[row * a.N + col];
                            const double num = rh > 0.0 ? rh : 0.0;
                            const double dd = (acc[mt][nt][h] > 0.0 ? acc[mt][nt][h] : 0.0) + EPS_R9;
                            double *u = a.out + row * a.ldo + col;
                            *u = *u * sqrt(num / dd);
                        }
                    }
            }
        }
        if (q + 1 < Q) {
            cp_wait_all();
            __syncthreads();                // stage q+1 visible; everyone done with stage q's buffer
        }
    }
}

// Row-block products with a k x k right factor (K = N = k <= 104, k even), fp64 A = Ups stored
// densely: den = Ups M for the Ups update (Eq. update-Y) and the Alg. 3 scores Ups Phi.  W = M / Phi
// stays resident in shared memory; BM-row tiles of A (one contiguous block each) arrive by bulk copy
// into a 2-slot ring on mbarriers, the next tile in flight while one is multiplied.  Warp w owns the
// MTW m-tiles (8 rows each) w*MTW .. of a tile against all NT n-tiles.
template <int EPI, int NT, int MTW, int NS, int MINB>  // NS: ring slots; MINB: resident CTAs per SM
__global__ void __launch_bounds__(DM_NT, MINB) dm_rowk_kernel(DmArgs a) {
    if (EPI == DM_ASSIGN && *a.done) return;
    constexpr int BM = 8 * 8 * MTW;
    extern __shared__ __align__(128) unsigned char dsm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(dsm);                 // [2]
    const int k = a.N;
    double *Ws = reinterpret_cast<double *>(dsm + 128);                 // [k][k]
    double *ring = Ws + ((k * k + 15) / 16) * 16;                        // [NS][NB][BM * k]
    constexpr int NB = EPI == DM_UPS ? 2 : 1;                           // UPS slots: Ups tile, RH tile
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int gr = lane >> 2, gc = lane & 3;
    const double *A = static_cast<const double *>(a.A);
    const int64_t ntiles = (a.n + BM - 1) / BM;
    const int64_t my = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (tid == 0) {
        bar_init(full, 1);
        bar_init(full + 1, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = tid; i < k * k; i += DM_NT) Ws[i] = a.W[i];
    __syncthreads();
    auto issue = [&](int64_t j) {                    // thread 0: this CTA's j-th tile into slot j & 1
        const int64_t r0 = (blockIdx.x + j * gridDim.x) * BM;
        const int rows = (int)(a.n - r0 < BM ? a.n - r0 : BM);
        const uint32_t bytes = (uint32_t)rows * (uint32_t)k * 8u;
        double *slot = ring + (size_t)(j % NS) * NB * BM * k;
        bar_expect_tx(full + (j % NS), NB * bytes);
        bulk_g2s(slot, A + r0 * k, bytes, full + (j % NS));
        if (EPI == DM_UPS) bulk_g2s(slot + BM * k, a.RH + r0 * k, bytes, full + (j % NS));
    };
    if (tid == 0) {
        if (my > 0) issue(0);
        if (NS > 1 && my > 1) issue(1);
    }
    bool changed = false;
    for (int64_t j = 0; j < my; ++j) {
        const int64_t r0 = (blockIdx.x + j * gridDim.x) * BM;
        const int rows = (int)(a.n - r0 < BM ? a.n - r0 : BM);
        bar_wait(full + (j % NS), (uint32_t)((j / NS) & 1));
        double *as = ring + (size_t)(j % NS) * NB * BM * k;
        double acc[MTW][NT][2];
#pragma unroll
        for (int m = 0; m < MTW; ++m)
#pragma unroll
            for (int t = 0; t < NT; ++t) acc[m][t][0] = acc[m][t][1] = 0.0;
        for (int k4 = 0; k4 < (k + 3) / 4; ++k4) {
            const int kk = k4 * 4 + gc;
            double af[MTW], bf[NT];
#pragma unroll
            for (int m = 0; m < MTW; ++m) {
                const int r = (w * MTW + m) * 8 + gr;
                af[m] = (kk < k && r < rows) ? as[r * k + kk] : 0.0;
            }
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int col = t * 8 + gr;
                bf[t] = (kk < k && col < k) ? Ws[kk * k + col] : 0.0;
            }
#pragma unroll
            for (int m = 0; m < MTW; ++m)
#pragma unroll
                for (int t = 0; t < NT; ++t) dmma(acc[m][t], af[m], bf[t]);
        }
#pragma unroll
        for (int m = 0; m < MTW; ++m) {
            const int r = (w * MTW + m) * 8 + gr;
            const int64_t row = r0 + r;
            if (EPI == DM_UPS) {
                if (r >= rows) continue;
#pragma unroll
                for (int t = 0; t < NT; ++t)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int col = t * 8 + 2 * gc + h;
                        if (col >= k) continue;
                        const double rh = as[BM * k + r * k + col];
                        const double num = rh > 0.0 ? rh : 0.0;
                        const double dd = (acc[m][t][h] > 0.0 ? acc[m][t][h] : 0.0) + EPS_R9;
                        as[r * k + col] = as[r * k + col] * sqrt(num / dd);   // in the tile, stored below
                    }
            } else {   // DM_ASSIGN: certified argmax (see CERT_TOL)
                double b1 = 0.0, b2 = -1.0;
                int i1 = -1;
#pragma unroll
                for (int t = 0; t < NT; ++t)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int col = t * 8 + 2 * gc + h;
                        top2_merge(b1, i1, b2, acc[m][t][h], col < k ? col : -1);
                    }
#pragma unroll
                for (int o = 1; o < 4; o <<= 1) {
                    const double ob1 = __shfl_xor_sync(0xffffffffu, b1, o), ob2 = __shfl_xor_sync(0xffffffffu, b2, o);
                    const int oi1 = __shfl_xor_sync(0xffffffffu, i1, o);
                    top2_merge(b1, i1, b2, ob1, oi1);
                    b2 = fmax(b2, ob2);
                }
                if (gc == 0 && r < rows) {
                    int lab = i1;
                    if (!(b1 - b2 > CERT_TOL * fabs(b1))) {          // near tie: R13 rescoring
                        const double *u = as + (size_t)r * k;
                        double best = 0.0;
                        lab = 0;
                        for (int l = 0; l < k; ++l) {
                            double sc = 0.0;
                            for (int jj = 0; jj < k; ++jj) sc = fma(u[jj], Ws[jj * k + l], sc);
                            if (l == 0 || sc > best) { best = sc; lab = l; }
                        }
                    }
                    if (a.labels[row] != lab) changed = true;
                    a.labels[row] = lab;
                }
            }
        }
        if (EPI == DM_UPS) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // tile -> async proxy
        __syncthreads();                              // slot j & 1 is done (and, UPS, updated)
        if (tid == 0) {
            if (EPI == DM_UPS) {
                bulk_s2g(a.out + r0 * k, as, (uint32_t)rows * (uint32_t)k * 8u);
                bulk_wait_read();                     // the store has read the slot before it is refilled
            }
            if (j + NS < my) issue(j + NS);
        }
    }
    if (EPI == DM_UPS && tid == 0) bulk_wait_all();
    if (EPI == DM_ASSIGN && __any_sync(0xffffffffu, changed) && lane == 0) *a.changed = 1;
}

// part[b][d][l] = sum_{i in split b} R'[i, d] * (dinv_i Ups[i, l]) for D rows [d0, d0 + 256)
// (grid.z) and columns [col0, col0 + 8 NT) (grid.y): C (D x k) += R'^T (dinv . Ups) with the row
// index i as the reduction dimension.  Warp w owns D rows w*32 .. w*32+31 (4 m-tiles).
constexpr int RT_BK = 32;           // input rows per stage
constexpr int RT_DB = 256;          // D rows per CTA
constexpr int RT_LDR = RT_DB + 8;   // R_s[i][d] fp32 (fragment reads conflict-free)

template <int NT>
constexpr size_t rt_smem() {
    return 2 * ((size_t)RT_BK * RT_LDR * sizeof(float) + (size_t)RT_BK * 8 * NT * sizeof(double) + RT_BK * sizeof(float));
}

// TU: the right factor's type (fp64 Ups in Alg. 2; fp32 Y in the a6 product), staged as is and
// widened at the fragment load
template <int NT, class TU>
__global__ void __launch_bounds__(DM_NT, 1) dm_rtu_kernel(const float *__restrict__ Rp, int64_t n, int D,
                                                          const float *__restrict__ dinv, const TU *__restrict__ U,
                                                          int k, int64_t rows_per, double *__restrict__ part) {
    extern __shared__ __align__(16) unsigned char dsm[];
    constexpr int NBW = 8 * NT;
    float *Rs = reinterpret_cast<float *>(dsm);                                         // [2][RT_BK][RT_LDR]
    TU *Us = reinterpret_cast<TU *>(dsm + 2 * (size_t)RT_BK * RT_LDR * sizeof(float));   // [2][RT_BK][NBW]
    float *Ds = reinterpret_cast<float *>(dsm + 2 * (size_t)RT_BK * RT_LDR * sizeof(float) +
                                          2 * (size_t)RT_BK * NBW * sizeof(double));    // [2][RT_BK]
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int gr = lane >> 2, gc = lane & 3;
    const int col0 = blockIdx.y * NBW, d0 = blockIdx.z * RT_DB;
    const int64_t i0 = blockIdx.x * rows_per, i1 = min(n, i0 + rows_per);
    const bool r16 = (D % 4) == 0 && ((reinterpret_cast<uintptr_t>(Rp) & 15u) == 0);
    auto load = [&](int64_t b, int buf) {
        float *rs = Rs + (size_t)buf * RT_BK * RT_LDR;
        TU *us = Us + (size_t)buf * RT_BK * NBW;
        float *ds = Ds + buf * RT_BK;
        if (r16) {
#pragma unroll
            for (int i = 0; i < RT_BK * (RT_DB / 4) / DM_NT; ++i) {
                const int c = tid + DM_NT * i, r = c / (RT_DB / 4), part4 = c % (RT_DB / 4);
                const int64_t row = b + r;
                const int dc = d0 + part4 * 4;
                const int bytes = row < i1 ? 4 * max(0, min(4, D - dc)) : 0;
                cp16(rs + r * RT_LDR + part4 * 4, bytes ? (const void *)(Rp + row * D + dc) : (const void *)Rp, bytes);
            }
        } else {
            for (int idx = tid; idx < RT_BK * RT_DB; idx += DM_NT) {
                const int r = idx / RT_DB, c = idx % RT_DB;
                const int64_t row = b + r;
                const bool v = row < i1 && d0 + c < D;
                cp4(rs + r * RT_LDR + c, v ? (const void *)(Rp + row * D + d0 + c) : (const void *)Rp, v);
            }
        }
        for (int idx = tid; idx < RT_BK * NBW; idx += DM_NT) {
            const int r = idx / NBW, c = idx - (idx / NBW) * NBW;
            const int64_t row = b + r;
            const bool v = row < i1 && col0 + c < k;
            if (sizeof(TU) == 8) cp8(us + idx, v ? (const void *)(U + row * k + col0 + c) : (const void *)U, v);
            else cp4(us + idx, v ? (const void *)(U + row * k + col0 + c) : (const void *)U, v);
        }
        if (tid < RT_BK) cp4(ds + tid, (b + tid < i1) ? (const void *)(dinv + b + tid) : (const void *)dinv, b + tid < i1);
        cp_commit();
    };
    double acc[4][NT][2];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    if (i0 < i1) {
        load(i0, 0);
        cp_wait_all();
        __syncthreads();
        int buf = 0;
        for (int64_t b = i0; b < i1; b += RT_BK) {
            const bool more = b + RT_BK < i1;
            if (more) load(b + RT_BK, buf ^ 1);
            const float *rs = Rs + (size_t)buf * RT_BK * RT_LDR + gc * RT_LDR + w * 32 + gr;
            const TU *us = Us + (size_t)buf * RT_BK * NBW + gc * NBW + gr;
            const float *ds = Ds + buf * RT_BK + gc;
#pragma unroll
            for (int k4 = 0; k4 < RT_BK / 4; ++k4) {
                double af[4], bf[NT];
                const double dv = (double)ds[k4 * 4];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) af[mt] = (double)rs[k4 * 4 * RT_LDR + mt * 8];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) bf[nt] = dv * (double)us[k4 * 4 * NBW + nt * 8];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt], af[mt], bf[nt]);
            }
            if (more) {
                cp_wait_all();
                __syncthreads();
                buf ^= 1;
            }
        }
    }
    double *pp = part + (int64_t)blockIdx.x * D * k;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
        const int d = d0 + w * 32 + mt * 8 + gr;
        if (d >= D) continue;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int col = col0 + nt * 8 + 2 * gc + h;
                if (col < k) pp[(int64_t)d * k + col] = acc[mt][nt][h];
            }
    }
}

// part[b] = A^T B over the rows of split b (A: n x p, B: n x q, fp64, p, q <= 128): the k x k
// products of Alg. 2 (Ups^T Ups, Ups^T (R H)).  Output tiles (mt, nt) of 8 x 8: warp w owns the
// m-tiles w, w + 8 (< ceil(p/8)) against every n-tile; the row index is the reduction dimension,
// staged 32 rows at a time.
constexpr int AB_BK = 32;
template <int MT, int NTT, int S>    // m-tiles per warp (1 or 2), n-tiles (<= 13), ring stages
__global__ void __launch_bounds__(DM_NT, 1) dm_atb_kernel(const double *__restrict__ A, int64_t lda,
                                                          const double *__restrict__ B, int64_t ldb, int64_t n, int p,
                                                          int q, int64_t rows_per, double *__restrict__ part) {
    extern __shared__ __align__(16) unsigned char dsm[];
    constexpr int W = 8 * NTT + 4;                              // padded width (p, q <= 8 NTT)
    constexpr int STG = 2 * AB_BK * W;                          // doubles per stage: A then B
    double *ring = reinterpret_cast<double *>(dsm);             // [S][2][AB_BK][W]
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int gr = lane >> 2, gc = lane & 3;
    const int64_t i0 = blockIdx.x * rows_per, i1 = min(n, i0 + rows_per);
    const int64_t nch = i1 > i0 ? (i1 - i0 + AB_BK - 1) / AB_BK : 0;
    auto load = [&](int64_t c) {                                // chunk c into slot c % S (commits a group)
        if (c < nch) {
            double *as = ring + (size_t)(c % S) * STG, *bs = as + AB_BK * W;
            const int64_t b = i0 + c * AB_BK;
            for (int idx = tid; idx < AB_BK * p; idx += DM_NT) {
                const int r = idx / p, col = idx - (idx / p) * p;
                const bool v = b + r < i1;
                cp8(as + r * W + col, v ? A + (b + r) * lda + col : A, v);
            }
            for (int idx = tid; idx < AB_BK * q; idx += DM_NT) {
                const int r = idx / q, col = idx - (idx / q) * q;
                const bool v = b + r < i1;
                cp8(bs + r * W + col, v ? B + (b + r) * ldb + col : B, v);
            }
        }
        cp_commit();                                            // (an empty group past the end)
    };
    // zero the padding columns once (never written by the loads)
    for (int idx = tid; idx < S * STG; idx += DM_NT) ring[idx] = 0.0;
    __syncthreads();
    double acc[MT][NTT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int t = 0; t < NTT; ++t) acc[m][t][0] = acc[m][t][1] = 0.0;
    const int mtiles = (p + 7) / 8;
#pragma unroll
    for (int c = 0; c < S - 1; ++c) load(c);
    for (int64_t c = 0; c < nch; ++c) {
        asm volatile("cp.async.wait_group %0;" ::"n"(S - 2) : "memory");   // chunk c has landed
        __syncthreads();                                         // ... for every thread; slot (c-1)%S is free
        load(c + S - 1);
        const double *as = ring + (size_t)(c % S) * STG + gc * W + gr;
        const double *bs = as + AB_BK * W;
#pragma unroll
        for (int k4 = 0; k4 < AB_BK / 4; ++k4) {
            double af[MT], bf[NTT];
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                const int mt = w + 8 * m;
                af[m] = mt < mtiles ? as[k4 * 4 * W + mt * 8] : 0.0;
            }
#pragma unroll
            for (int t = 0; t < NTT; ++t) bf[t] = bs[k4 * 4 * W + t * 8];
#pragma unroll
            for (int m = 0; m < MT; ++m)
#pragma unroll
                for (int t = 0; t < NTT; ++t) dmma(acc[m][t], af[m], bf[t]);
        }
    }
    cp_wait_all();
    double *pp = part + (int64_t)blockIdx.x * p * q;
#pragma unroll
    for (int m = 0; m < MT; ++m) {
        const int row = (w + 8 * m) * 8 + gr;
        if (row >= p) continue;
#pragma unroll
        for (int t = 0; t < NTT; ++t)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int col = t * 8 + 2 * gc + h;
                if (col < q) pp[(int64_t)row * q + col] = acc[m][t][h];
            }
    }
}

// The same A^T B with A, B stored densely (lda = p, ldb = q): a 32-row chunk of each is one
// contiguous block, fetched by one bulk copy (cp.async.bulk) into an S-stage ring completed on
// mbarriers -- one instruction per 12.8 KB instead of one per element (the element-wise cp.async
// version was LSU-issue bound, 1.0 ms for 2M x 50).  Fragment reads use the unpadded row stride.
// A CTA's rows are whole chunks except the last CTA's tail, which is staged element-wise with
// zero fill.  A Gram (B == A, `same`) stages each chunk once and reads both fragments from it.
template <int MT, int NTT, int S>
__global__ void __launch_bounds__(DM_NT, 1) dm_atb_bulk_kernel(const double *__restrict__ A, const double *__restrict__ B,
                                                               int64_t n, int p, int q, int64_t rows_per, bool same,
                                                               double *__restrict__ part) {
    extern __shared__ __align__(128) unsigned char dsm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(dsm);                        // [S]
    double *ring = reinterpret_cast<double *>(dsm + 128);                       // [S][AB_BK * (p + q)] (same: p)
    const int stage = AB_BK * (same ? p : p + q);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int gr = lane >> 2, gc = lane & 3;
    const int64_t i0 = blockIdx.x * rows_per, i1 = min(n, i0 + rows_per);
    const int64_t nfull = i1 > i0 ? (i1 - i0) / AB_BK : 0;
    const int tail = i1 > i0 ? (int)((i1 - i0) - nfull * AB_BK) : 0;
    if (tid == 0)
        for (int sI = 0; sI < S; ++sI) bar_init(full + sI, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    auto issue = [&](int64_t c) {                      // thread 0: full chunk c into slot c % S
        double *as = ring + (size_t)(c % S) * stage, *bs = as + AB_BK * p;
        const int64_t b = i0 + c * AB_BK;
        const uint32_t ba = (uint32_t)(AB_BK * p * 8), bb = (uint32_t)(AB_BK * q * 8);
        bar_expect_tx(full + c % S, same ? ba : ba + bb);
        bulk_g2s(as, A + b * p, ba, full + c % S);
        if (!same) bulk_g2s(bs, B + b * q, bb, full + c % S);
    };
    if (tid == 0)
        for (int64_t c = 0; c < S && c < nfull; ++c) issue(c);
    double acc[MT][NTT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int t = 0; t < NTT; ++t) acc[m][t][0] = acc[m][t][1] = 0.0;
    const int mtiles = (p + 7) / 8, ntiles = (q + 7) / 8;
    auto compute = [&](const double *as, const double *bs) {
#pragma unroll
        for (int k4 = 0; k4 < AB_BK / 4; ++k4) {
            double af[MT], bf[NTT];
            const int r = k4 * 4 + gc;
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                const int col = (w + 8 * m) * 8 + gr;
                af[m] = col < p ? as[r * p + col] : 0.0;
            }
#pragma unroll
            for (int t = 0; t < NTT; ++t) {
                const int col = t * 8 + gr;
                bf[t] = (t < ntiles && col < q) ? bs[r * q + col] : 0.0;
            }
#pragma unroll
            for (int m = 0; m < MT; ++m)
#pragma unroll
                for (int t = 0; t < NTT; ++t) dmma(acc[m][t], af[m], bf[t]);
        }
    };
    for (int64_t c = 0; c < nfull; ++c) {
        bar_wait(full + c % S, (uint32_t)((c / S) & 1));
        const double *as = ring + (size_t)(c % S) * stage;
        compute(as, same ? as : as + AB_BK * p);
        __syncthreads();                               // every thread is done with slot c % S
        if (tid == 0 && c + S < nfull) issue(c + S);
    }
    if (tail > 0) {                                    // the last rows: element-wise, zero-filled
        double *as = ring, *bs = ring + AB_BK * p;     // slots 0 (and 1) are free: all bulk copies consumed
        const int64_t b = i0 + nfull * AB_BK;
        for (int idx = tid; idx < AB_BK * p; idx += DM_NT) {
            const int r = idx / p;
            as[idx] = r < tail ? A[(b + r) * p + (idx - r * p)] : 0.0;
        }
        for (int idx = tid; idx < AB_BK * q; idx += DM_NT) {
            const int r = idx / q;
            bs[idx] = r < tail ? B[(b + r) * q + (idx - r * q)] : 0.0;
        }
        __syncthreads();
        compute(as, bs);
    }
    (void)mtiles;
    double *pp = part + (int64_t)blockIdx.x * p * q;
#pragma unroll
    for (int m = 0; m < MT; ++m) {
        const int row = (w + 8 * m) * 8 + gr;
        if (row >= p) continue;
#pragma unroll
        for (int t = 0; t < NTT; ++t)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int col = t * 8 + 2 * gc + h;
                if (col < q) pp[(int64_t)row * q + col] = acc[m][t][h];
            }
    }
}

// out[i] = sum_g part[g][i] in g order; 16 partials loaded ahead of their (in-order) adds, so the
// few threads of a k x k reduction are not bound by one L2 round trip per partial
__global__ void reduce_parts_kernel(const double *__restrict__ part, int64_t G, int64_t len, double *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= len) return;
    constexpr int U = 16;
    double s = 0.0;
    int64_t g = 0;
    for (; g + U <= G; g += U) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcg(part + (g + u) * len + i);
#pragma unroll
        for (int u = 0; u < U; ++u) s += v[u];
    }
    for (; g < G; ++g) s += part[g * len + i];
    out[i] = s;
}

int sm_count_cached() {
    static int v = 0;
    if (!v) v = sm_count();
    return v;
}

// column blocks of 8 NT <= 56 columns (NT <= 7), as few blocks as possible
void col_tiling(int N, int &NT, int &nblk) {
    nblk = std::max(1, (N + 55) / 56);
    NT = std::max(1, ((N + nblk - 1) / nblk + 7) / 8);
}

#define TPO_NT13(F, NT, ...)                          \
    switch (NT) {                                     \
        case 1: F<1>(__VA_ARGS__); break;             \
        case 2: F<2>(__VA_ARGS__); break;             \
        case 3: F<3>(__VA_ARGS__); break;             \
        case 4: F<4>(__VA_ARGS__); break;             \
        case 5: F<5>(__VA_ARGS__); break;             \
        case 6: F<6>(__VA_ARGS__); break;             \
        case 7: F<7>(__VA_ARGS__); break;             \
        case 8: F<8>(__VA_ARGS__); break;             \
        case 9: F<9>(__VA_ARGS__); break;             \
        case 10: F<10>(__VA_ARGS__); break;           \
        case 11: F<11>(__VA_ARGS__); break;           \
        case 12: F<12>(__VA_ARGS__); break;           \
        default: F<13>(__VA_ARGS__); break;           \
    }

template <class TA, int EPI, int NT>
void dm_launch(const DmArgs &a, int nblk, cudaStream_t st) {
    const size_t sm = dm_smem<TA, NT>();
    TPO_CUDA(cudaFuncSetAttribute(dm_rowgemm_kernel<TA, EPI, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const int64_t tiles = cdiv(std::max<int64_t>(a.n, 1), DM_BM);
    const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, cdiv(sm_count_cached(), nblk)));
    dm_rowgemm_kernel<TA, EPI, NT><<<dim3((unsigned)gx, (unsigned)nblk), DM_NT, sm, st>>>(a);
    TPO_LAUNCH_CHECK();
}
template <int NT>
void dm_store_f32(const DmArgs &a, int nblk, cudaStream_t st) { dm_launch<float, DM_STORE, NT>(a, nblk, st); }
template <int NT>
void dm_store_f64(const DmArgs &a, int nblk, cudaStream_t st) { dm_launch<double, DM_STORE, NT>(a, nblk, st); }
// the Ups update reads whole rows of Ups (den = Ups M) and overwrites them: one column block
template <int NT>
void dm_ups(const DmArgs &a, cudaStream_t st) { dm_launch<double, DM_UPS, NT>(a, 1, st); }
template <int NT>
void dm_assign(const DmArgs &a, cudaStream_t st) { dm_launch<double, DM_ASSIGN, NT>(a, 1, st); }

// resident-W row-block kernel (dense fp64 Ups, even k): 16 rows per warp for k <= 64, else 8
template <int EPI, int NT>
void dm_rowk_launch(const DmArgs &a, cudaStream_t st) {
    const int k = a.N;
    auto go = [&](auto mtw_tag, auto ns_tag, auto minb_tag) {
        constexpr int MTW = decltype(mtw_tag)::value, NS = decltype(ns_tag)::value;
        constexpr int MINB = decltype(minb_tag)::value;
        constexpr int BM = 64 * MTW;
        constexpr int NB = EPI == DM_UPS ? 2 : 1;
        const size_t sm = 128 + sizeof(double) * (((size_t)k * k + 15) / 16 * 16 + (size_t)NS * NB * BM * k);
        TPO_CUDA(cudaFuncSetAttribute(dm_rowk_kernel<EPI, NT, MTW, NS, MINB>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        const int64_t tiles = cdiv(std::max<int64_t>(a.n, 1), BM);
        const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)MINB * sm_count_cached()));
        dm_rowk_kernel<EPI, NT, MTW, NS, MINB><<<gx, DM_NT, sm, st>>>(a);
        TPO_LAUNCH_CHECK();
    };
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    using I3 = std::integral_constant<int, 3>;
    // ASSIGN: 128-row tiles for k <= 64.  UPS: 64-row tile pairs (Ups, RH).  The UPS epilogue (an fp64
    // divide and square root per element) is as long as the tile's DMMA product, so several CTAs per SM
    // with one slot each (one CTA's epilogue and store beside another's product and load) beat one CTA
    // with a two-slot ring: as many CTAs as the k x k factor and one tile pair let fit (<= 227 KB / SM).
    if (EPI != DM_UPS) {
        if (k <= 64) go(I2(), I2(), I1());
        else go(I1(), I2(), I1());
    } else {
        const size_t per = 1024 + 128 + sizeof(double) * (((size_t)k * k + 15) / 16 * 16 + (size_t)2 * 64 * k);
        if (3 * per <= 227 * 1024) go(I1(), I1(), I3());
        else if (2 * per <= 227 * 1024) go(I1(), I1(), I2());
        else go(I1(), I1(), I1());
    }
}
template <int NT>
void dm_rowk_ups(const DmArgs &a, cudaStream_t st) { dm_rowk_launch<DM_UPS, NT>(a, st); }
template <int NT>
void dm_rowk_assign(const DmArgs &a, cudaStream_t st) { dm_rowk_launch<DM_ASSIGN, NT>(a, st); }
bool rowk_ok(const double *A, int k) { return k % 2 == 0 && (reinterpret_cast<uintptr_t>(A) & 15u) == 0; }
bool rowk_ups_ok(const double *U, const double *RH, int k) {
    return rowk_ok(U, k) && (reinterpret_cast<uintptr_t>(RH) & 15u) == 0;
}

template <int NT, class TU>
void dm_rtu_launch_t(const float *Rp, int64_t n, int D, const float *dinv, const TU *U, int k, int64_t rows_per, int G,
                     int nblk, double *part, cudaStream_t st) {
    const size_t sm = rt_smem<NT>();
    TPO_CUDA(cudaFuncSetAttribute(dm_rtu_kernel<NT, TU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    dm_rtu_kernel<NT, TU><<<dim3((unsigned)G, (unsigned)nblk, (unsigned)cdiv(D, RT_DB)), DM_NT, sm, st>>>(Rp, n, D, dinv,
                                                                                                       U, k, rows_per, part);
    TPO_LAUNCH_CHECK();
}
template <int NT>
void dm_rtu_launch(const float *Rp, int64_t n, int D, const float *dinv, const double *U, const float *U32, int k,
                   int64_t rows_per, int G, int nblk, double *part, cudaStream_t st) {
    if (U32) dm_rtu_launch_t<NT, float>(Rp, n, D, dinv, U32, k, rows_per, G, nblk, part, st);
    else dm_rtu_launch_t<NT, double>(Rp, n, D, dinv, U, k, rows_per, G, nblk, part, st);
}

}  // namespace

namespace {
template <int MT, int NTT>
void dm_atb_launch(const double *A, int64_t lda, const double *B, int64_t ldb, int64_t n, int p, int q, int64_t rows_per,
                   int G, double *part, cudaStream_t st) {
    constexpr int S = NTT <= 8 ? 4 : 3;                         // ring depth within ~220 KB
    const size_t sm = (size_t)S * 2 * AB_BK * (8 * NTT + 4) * sizeof(double);
    TPO_CUDA(cudaFuncSetAttribute(dm_atb_kernel<MT, NTT, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    dm_atb_kernel<MT, NTT, S><<<G, DM_NT, sm, st>>>(A, lda, B, ldb, n, p, q, rows_per, part);
    TPO_LAUNCH_CHECK();
}
template <int MT, int NTT>
void dm_atb_bulk_launch(const double *A, const double *B, int64_t n, int p, int q, int64_t rows_per, int G, double *part,
                        cudaStream_t st) {
    constexpr int S = 4;
    const bool same = A == B && p == q;
    // the tail's element-wise staging uses AB_BK * (p + q) doubles of the (S-slot) ring in either case
    const size_t sm = 128 + (size_t)std::max(S * AB_BK * (same ? p : p + q), AB_BK * (p + q)) * sizeof(double);
    TPO_CUDA(cudaFuncSetAttribute(dm_atb_bulk_kernel<MT, NTT, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    dm_atb_bulk_kernel<MT, NTT, S><<<G, DM_NT, sm, st>>>(A, B, n, p, q, rows_per, same, part);
    TPO_LAUNCH_CHECK();
}
template <int NTT>
void dm_atb_mt(int mt, const double *A, int64_t lda, const double *B, int64_t ldb, int64_t n, int p, int q,
               int64_t rows_per, int G, double *part, cudaStream_t st) {
    // dense rows (lda = p, ldb = q), 16-byte aligned bases: one bulk copy per 32-row chunk
    const bool bulk = lda == p && ldb == q && ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15u) == 0;
    if (bulk) {
        if (mt <= 8) dm_atb_bulk_launch<1, NTT>(A, B, n, p, q, rows_per, G, part, st);
        else dm_atb_bulk_launch<2, NTT>(A, B, n, p, q, rows_per, G, part, st);
        return;
    }
    if (mt <= 8) dm_atb_launch<1, NTT>(A, lda, B, ldb, n, p, q, rows_per, G, part, st);
    else dm_atb_launch<2, NTT>(A, lda, B, ldb, n, p, q, rows_per, G, part, st);
}
}  // namespace

// two row splits per SM: a Gram chunk ring is small enough for two resident CTAs, whose DMMA chains
// and bulk copies interleave
constexpr int AB_SPLITS_PER_SM = 2;
size_t ts_atb_ws(int p, int q) {
    return align_up(sizeof(double) * (size_t)AB_SPLITS_PER_SM * sm_count_cached() * p * q) + 256;
}

// out (p x q fp64) = A^T B, A n x p, B n x q fp64 (p, q <= 128): fixed-order split over rows
void ts_atb_f64(const double *A, int64_t lda, const double *B, int64_t ldb, int64_t n, int p, int q, double *out,
                Arena &ar, cudaStream_t st) {
    const int64_t rows_per =
        cdiv(cdiv(std::max<int64_t>(n, 1), (int64_t)AB_SPLITS_PER_SM * sm_count_cached()), AB_BK) * AB_BK;
    const int G = (int)cdiv(std::max<int64_t>(n, 1), rows_per);
    const size_t mark = ar.off;
    double *part = ar.take<double>((size_t)G * p * q);
    const int mt = (p + 7) / 8;
    TPO_NT13(dm_atb_mt, (std::max(p, q) + 7) / 8, mt, A, lda, B, ldb, n, p, q, rows_per, G, part, st);
    reduce_parts_kernel<<<cdiv((int64_t)p * q, 256), 256, 0, st>>>(part, G, (int64_t)p * q, out);
    TPO_LAUNCH_CHECK();
    ar.off = mark;
}

bool ts64_enabled() {
    const char *e = getenv("TPO_TS64");
    return !(e && e[0] == '0');
}
// (k <= 64: two 64-row Ups / RH slots and the resident k x k M fit shared memory; up to 104 with one)
bool ts64_ups_enabled(int k) { return ts64_enabled() && k > 16 && k <= 104 && k % 2 == 0; }

// out = diag(rs) A W diag(1/cs): A n x K fp32 (lda), W K x N fp64 (ldw = N), out n x N fp64 (ldo)
void ts_aw_f64(const float *A, int64_t lda, const float *rs, const double *W, int64_t n, int K, int N,
               const double *cs, double *out, int64_t ldo, cudaStream_t st) {
    if (n == 0 || N == 0) return;
    DmArgs a{};
    a.A = A; a.lda = lda; a.rs = rs; a.W = W; a.ldw = N; a.n = n; a.K = K; a.N = N; a.out = out; a.ldo = ldo; a.cs = cs;
    int NT, nblk;
    col_tiling(N, NT, nblk);
    TPO_NT13(dm_store_f32, NT, a, nblk, st);
}

// X <- X W in place (X n x k fp64, W k x k fp64) on the fp64 tensor path when the k columns form
// one column block (k <= 56: every CTA reads its rows whole before writing them, like the Ups
// update); returns false (nothing done) otherwise.
bool ts_xw_inplace_f64(double *X, int64_t n, int k, const double *W, cudaStream_t st) {
    if (!ts64_enabled()) return false;
    int NT, nblk;
    col_tiling(k, NT, nblk);
    if (nblk != 1) return false;
    if (n == 0) return true;
    DmArgs a{};
    a.A = X; a.lda = k; a.W = W; a.ldw = k; a.n = n; a.K = k; a.N = k; a.out = X; a.ldo = k;
    TPO_NT13(dm_store_f64, NT, a, 1, st);
    return true;
}

// out32 = fp32(X W) (X n x k fp64, W k x k) on the fp64 tensor path, k <= 104
bool ts_xw_f32out(const double *X, int64_t n, int k, const double *W, float *out32, cudaStream_t st) {
    if (!ts64_enabled() || k > 104) return false;
    if (n == 0) return true;
    int NT, nblk;
    col_tiling(k, NT, nblk);
    DmArgs a{};
    a.A = X; a.lda = k; a.W = W; a.ldw = k; a.n = n; a.K = k; a.N = k; a.out32 = out32; a.ldo = k;
    TPO_NT13(dm_store_f64, NT, a, nblk, st);
    return true;
}

// out = X W (X n x k fp64, W k x k, out n x k; out != X) on the fp64 tensor path, k <= 104
bool ts_xw_f64(const double *X, int64_t n, int k, const double *W, double *out, cudaStream_t st) {
    if (!ts64_enabled() || k > 104) return false;
    if (n == 0) return true;
    int NT, nblk;
    col_tiling(k, NT, nblk);
    DmArgs a{};
    a.A = X; a.lda = k; a.W = W; a.ldw = k; a.n = n; a.K = k; a.N = k; a.out = out; a.ldo = k;
    TPO_NT13(dm_store_f64, NT, a, nblk, st);
    return true;
}

// Ups <- Ups . sqrt(max(RH,0) / (max(Ups M,0) + eps))  (Eq. update-Y with the R9 clamps), in place;
// k <= 104 (13 n-tiles of accumulators per warp)
void ts_ups_update(double *U, const double *RH, const double *M, int64_t n, int k, cudaStream_t st) {
    if (n == 0) return;
    DmArgs a{};
    a.A = U; a.lda = k; a.W = M; a.ldw = k; a.n = n; a.K = k; a.N = k; a.out = U; a.ldo = k; a.RH = RH;
    if (rowk_ups_ok(U, RH, k)) {
        TPO_NT13(dm_rowk_ups, (k + 7) / 8, a, st);
        return;
    }
    TPO_NT13(dm_ups, (k + 7) / 8, a, st);
}

// Alg. 3 assignment (Eq. ell-ast) for k <= 104: labels = argmax_l (Ups Phi)[i, l]
// with ties -> smallest l, scores on the fp64 tensor path, certified (CERT_TOL) or rescored by R13's
// sequential fma; *changed = 1 when a label changes; nothing when *done.
void ts_assign(const double *U, const double *Phi, int64_t n, int k, int32_t *labels, int32_t *changed,
               const int32_t *done, cudaStream_t st) {
    if (n == 0) return;
    DmArgs a{};
    a.A = U; a.lda = k; a.W = Phi; a.ldw = k; a.n = n; a.K = k; a.N = k;
    a.labels = labels; a.changed = changed; a.done = done;
    if (rowk_ok(U, k)) {
        TPO_NT13(dm_rowk_assign, (k + 7) / 8, a, st);
        return;
    }
    TPO_NT13(dm_assign, (k + 7) / 8, a, st);
}

size_t ts_rtu_ws(int64_t n, int64_t D, int k) {
    (void)n;
    return align_up(sizeof(double) * (size_t)sm_count_cached() * D * k) + 256;   // >= G * D * k
}

namespace {
void rtu_run(const float *Rp, int64_t n, int64_t D, const float *dinv, const double *U, const float *U32, int k,
             double *RtU, Arena &ar, cudaStream_t st) {
    int NT, nblk;
    col_tiling(k, NT, nblk);
    const int nz = (int)cdiv(D, RT_DB);
    const int64_t want = std::max<int64_t>(1, sm_count_cached() / (nblk * nz));
    const int64_t rows_per = cdiv(cdiv(std::max<int64_t>(n, 1), want), RT_BK) * RT_BK;
    const int G = (int)cdiv(std::max<int64_t>(n, 1), rows_per);
    const size_t mark = ar.off;
    double *part = ar.take<double>((size_t)G * D * k);
    TPO_NT13(dm_rtu_launch, NT, Rp, n, (int)D, dinv, U, U32, k, rows_per, G, nblk, part, st);
    reduce_parts_kernel<<<cdiv(D * k, 256), 256, 0, st>>>(part, G, D * k, RtU);
    TPO_LAUNCH_CHECK();
    ar.off = mark;
}
}  // namespace

// RtU = R'^T (dinv . Ups) (D x k fp64)
void ts_rtu(const float *Rp, int64_t n, int64_t D, const float *dinv, const double *U, int k, double *RtU, Arena &ar,
            cudaStream_t st) {
    rtu_run(Rp, n, D, dinv, U, nullptr, k, RtU, ar, st);
}

// a6 on the fp64 tensor path (Theorem 1, bracketing 564): W = R'^T (dinv . Y)
// (D x b, fp64), out = dinv . (R' W) rounded to fp32
size_t ts_affinity_ws(int64_t D, int64_t b) {
    return align_up(sizeof(double) * (size_t)D * b) + ts_rtu_ws(0, D, (int)b) + 256;
}
void ts_affinity(const float *Rp, const float *dinv, int64_t n, int64_t D, const float *Y, int64_t b, float *out,
                 Arena &ar, cudaStream_t st) {
    double *W = ar.take<double>((size_t)D * b);
    rtu_run(Rp, n, D, dinv, nullptr, Y, (int)b, W, ar, st);
    if (n == 0) return;
    DmArgs a{};
    a.A = Rp; a.lda = D; a.rs = dinv; a.W = W; a.ldw = b; a.n = n; a.K = (int)D; a.N = (int)b; a.out32 = out; a.ldo = b;
    int NT, nblk;
    col_tiling((int)b, NT, nblk);
    TPO_NT13(dm_store_f32, NT, a, nblk, st);
}

namespace {
__global__ void add_f64_kernel(double *__restrict__ acc, const double *__restrict__ x, int64_t len) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < len) acc[i] += x[i];
}
}  // namespace

// ---------------------------------------------------------------------------------------
// f3 "R-free" a6: S~Y without materialising R' for all n rows.  R' rows are
// recomputed from Zhat (Eq. R-prime: tcgen05 3xTF32 GEMM + sincos) in chunks of
// `chunk` rows in each of three sweeps -- r = sum_i R'[i]; W = sum_chunks R'_c^T (dinv_c . Y_c);
// out_c = dinv_c . (R'_c W) -- so the working set is chunk x 2d floats instead of n x 2d (10 GB at
// xl).  The chunk sums of r and W are added in chunk order (deterministic).  The cost is three
// feature evaluations per application (an O(n d^2) GEMM + 2nd sincos each) for half the bytes.
// ---------------------------------------------------------------------------------------
size_t ts_affinity_rfree_ws(int64_t n, int64_t d, int64_t b, int64_t chunk) {
    const int64_t D = 2 * d, C = std::max<int64_t>(1, std::min(n, chunk));
    return align_up(sizeof(float) * (size_t)C * D) + align_up(sizeof(float) * (size_t)C) + 3 * align_up(sizeof(double) * D) +
           2 * align_up(sizeof(double) * (size_t)D * b) + std::max(features_ws_bytes(C, d), ts_rtu_ws(0, D, (int)b)) + 4096;
}

void ts_affinity_rfree(const float *Zhat, int64_t n, int64_t d, const float *Q, const float *Y, int64_t b, float *out,
                       int64_t chunk, Arena &ar, cudaStream_t st) {
    const int64_t D = 2 * d, C = std::max<int64_t>(1, std::min(n, chunk));
    float *Rc = ar.take<float>((size_t)C * D), *dc = ar.take<float>((size_t)C);
    double *r = ar.take<double>(D), *rp = ar.take<double>(D);
    double *W = ar.take<double>((size_t)D * b), *Wc = ar.take<double>((size_t)D * b);
    const size_t mark = ar.off;
    TPO_CUDA(cudaMemsetAsync(r, 0, sizeof(double) * D, st));
    TPO_CUDA(cudaMemsetAsync(W, 0, sizeof(double) * D * b, st));
    for (int64_t c0 = 0; c0 < n; c0 += C) {                // sweep 1: r
        const int64_t nc = std::min(C, n - c0);
        features_part(Zhat + c0 * d, nc, d, Q, Rc, rp, ar, st);
        ar.off = mark;
        add_f64_kernel<<<cdiv(D, 256), 256, 0, st>>>(r, rp, D);
        TPO_LAUNCH_CHECK();
    }
    for (int64_t c0 = 0; c0 < n; c0 += C) {                // sweep 2: W = R^T Y
        const int64_t nc = std::min(C, n - c0);
        features_part(Zhat + c0 * d, nc, d, Q, Rc, rp, ar, st);
        ar.off = mark;
        dinv_from_r(Rc, nc, D, r, dc, st);
        rtu_run(Rc, nc, D, dc, nullptr, Y + c0 * b, (int)b, Wc, ar, st);
        ar.off = mark;
        add_f64_kernel<<<cdiv(D * b, 256), 256, 0, st>>>(W, Wc, D * b);
        TPO_LAUNCH_CHECK();
    }
    for (int64_t c0 = 0; c0 < n; c0 += C) {                // sweep 3: out = R W
        const int64_t nc = std::min(C, n - c0);
        features_part(Zhat + c0 * d, nc, d, Q, Rc, rp, ar, st);
        ar.off = mark;
        dinv_from_r(Rc, nc, D, r, dc, st);
        DmArgs a{};
        a.A = Rc; a.lda = D; a.rs = dc; a.W = W; a.ldw = b; a.n = nc; a.K = (int)D; a.N = (int)b;
        a.out32 = out + c0 * b; a.ldo = b;
        int NT, nblk;
        col_tiling((int)b, NT, nblk);
        TPO_NT13(dm_store_f32, NT, a, nblk, st);
    }
}

}  // namespace tpo
