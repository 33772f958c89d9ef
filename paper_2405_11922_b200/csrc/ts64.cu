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

#include "tpo_internal.cuh"

namespace tpo {
namespace {

constexpr double EPS_R9 = 1e-12;    // R9
constexpr int DM_NT = 256;          // 8 warps
constexpr int DM_BM = 256;          // rows per tile: 8 warps x 32 (4 m-tiles of 8)
constexpr int DM_BK = 32;           // K per stage (8 k-steps of 4)

enum { DM_STORE = 0, DM_UPS = 1 };

struct DmArgs {
    const void *A;        // n x K (fp32 or fp64), leading dimension lda
    int64_t lda;
    const float *rs;      // STORE: row scale (dinv) or null
    const double *W;      // K x N, leading dimension ldw
    int64_t ldw;
    int64_t n;
    int K, N;
    double *out;          // STORE: n x N (ldo); UPS: Ups itself (= A, updated in place)
    int64_t ldo;
    const double *cs;     // STORE: column divisors (sigma) or null
    const double *RH;     // UPS: n x N
};

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
        } else {                            // element copies (fp64 A, or unaligned fp32)
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
        if (s == nst - 1) {                 // epilogue of the tile: C[gr][2 gc + h] of each 8 x 8 tile
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
                            a.out[row * a.ldo + col] = v;
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

template <int NT>
__global__ void __launch_bounds__(DM_NT, 1) dm_rtu_kernel(const float *__restrict__ Rp, int64_t n, int D,
                                                          const float *__restrict__ dinv, const double *__restrict__ U,
                                                          int k, int64_t rows_per, double *__restrict__ part) {
    extern __shared__ __align__(16) unsigned char dsm[];
    constexpr int NBW = 8 * NT;
    float *Rs = reinterpret_cast<float *>(dsm);                                         // [2][RT_BK][RT_LDR]
    double *Us = reinterpret_cast<double *>(dsm + 2 * (size_t)RT_BK * RT_LDR * sizeof(float));   // [2][RT_BK][NBW]
    float *Ds = reinterpret_cast<float *>(Us + 2 * RT_BK * NBW);                       // [2][RT_BK]
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int gr = lane >> 2, gc = lane & 3;
    const int col0 = blockIdx.y * NBW, d0 = blockIdx.z * RT_DB;
    const int64_t i0 = blockIdx.x * rows_per, i1 = min(n, i0 + rows_per);
    const bool r16 = (D % 4) == 0 && ((reinterpret_cast<uintptr_t>(Rp) & 15u) == 0);
    auto load = [&](int64_t b, int buf) {
        float *rs = Rs + (size_t)buf * RT_BK * RT_LDR;
        double *us = Us + (size_t)buf * RT_BK * NBW;
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
            cp8(us + idx, v ? (const void *)(U + row * k + col0 + c) : (const void *)U, v);
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
            const double *us = Us + (size_t)buf * RT_BK * NBW + gc * NBW + gr;
            const float *ds = Ds + buf * RT_BK + gc;
#pragma unroll
            for (int k4 = 0; k4 < RT_BK / 4; ++k4) {
                double af[4], bf[NT];
                const double dv = (double)ds[k4 * 4];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) af[mt] = (double)rs[k4 * 4 * RT_LDR + mt * 8];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) bf[nt] = dv * us[k4 * 4 * NBW + nt * 8];
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
constexpr int AB_MAXT = 16;         // up to 128 columns
template <int MT, int NTT>          // m-tiles per warp (1 or 2), n-tiles (<= 16)
__global__ void __launch_bounds__(DM_NT, 1) dm_atb_kernel(const double *__restrict__ A, int64_t lda,
                                                          const double *__restrict__ B, int64_t ldb, int64_t n, int p,
                                                          int q, int64_t rows_per, double *__restrict__ part) {
    extern __shared__ __align__(16) unsigned char dsm[];
    constexpr int PW = 8 * AB_MAXT + 4, QW = 8 * NTT + 4;      // padded widths (fragment reads)
    double *As = reinterpret_cast<double *>(dsm);               // [2][AB_BK][PW]
    double *Bs = As + 2 * AB_BK * PW;                           // [2][AB_BK][QW]
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int gr = lane >> 2, gc = lane & 3;
    const int64_t i0 = blockIdx.x * rows_per, i1 = min(n, i0 + rows_per);
    auto load = [&](int64_t b, int buf) {
        double *as = As + (size_t)buf * AB_BK * PW, *bs = Bs + (size_t)buf * AB_BK * QW;
        for (int idx = tid; idx < AB_BK * p; idx += DM_NT) {
            const int r = idx / p, c = idx - (idx / p) * p;
            const bool v = b + r < i1;
            cp8(as + r * PW + c, v ? A + (b + r) * lda + c : A, v);
        }
        for (int idx = tid; idx < AB_BK * q; idx += DM_NT) {
            const int r = idx / q, c = idx - (idx / q) * q;
            const bool v = b + r < i1;
            cp8(bs + r * QW + c, v ? B + (b + r) * ldb + c : B, v);
        }
        cp_commit();
    };
    // zero the padding columns once (never written by the loads)
    for (int idx = tid; idx < 2 * AB_BK * PW; idx += DM_NT) As[idx] = 0.0;
    for (int idx = tid; idx < 2 * AB_BK * QW; idx += DM_NT) Bs[idx] = 0.0;
    __syncthreads();
    double acc[MT][NTT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int t = 0; t < NTT; ++t) acc[m][t][0] = acc[m][t][1] = 0.0;
    const int mtiles = (p + 7) / 8;
    if (i0 < i1) {
        load(i0, 0);
        cp_wait_all();
        __syncthreads();
        int buf = 0;
        for (int64_t b = i0; b < i1; b += AB_BK) {
            const bool more = b + AB_BK < i1;
            if (more) load(b + AB_BK, buf ^ 1);
            const double *as = As + (size_t)buf * AB_BK * PW + gc * PW + gr;
            const double *bs = Bs + (size_t)buf * AB_BK * QW + gc * QW + gr;
#pragma unroll
            for (int k4 = 0; k4 < AB_BK / 4; ++k4) {
                double af[MT], bf[NTT];
#pragma unroll
                for (int m = 0; m < MT; ++m) {
                    const int mt = w + 8 * m;
                    af[m] = mt < mtiles ? as[k4 * 4 * PW + mt * 8] : 0.0;
                }
#pragma unroll
                for (int t = 0; t < NTT; ++t) bf[t] = bs[k4 * 4 * QW + t * 8];
#pragma unroll
                for (int m = 0; m < MT; ++m)
#pragma unroll
                    for (int t = 0; t < NTT; ++t) dmma(acc[m][t], af[m], bf[t]);
            }
            if (more) {
                cp_wait_all();
                __syncthreads();
                buf ^= 1;
            }
        }
    }
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

__global__ void reduce_parts_kernel(const double *__restrict__ part, int64_t G, int64_t len, double *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= len) return;
    double s = 0.0;
    for (int64_t g = 0; g < G; ++g) s += part[g * len + i];
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
// the Ups update reads whole rows of Ups (den = Ups M) and overwrites them: one column block
template <int NT>
void dm_ups(const DmArgs &a, cudaStream_t st) { dm_launch<double, DM_UPS, NT>(a, 1, st); }

template <int NT>
void dm_rtu_launch(const float *Rp, int64_t n, int D, const float *dinv, const double *U, int k, int64_t rows_per,
                   int G, int nblk, double *part, cudaStream_t st) {
    const size_t sm = rt_smem<NT>();
    TPO_CUDA(cudaFuncSetAttribute(dm_rtu_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    dm_rtu_kernel<NT><<<dim3((unsigned)G, (unsigned)nblk, (unsigned)cdiv(D, RT_DB)), DM_NT, sm, st>>>(Rp, n, D, dinv, U, k,
                                                                                                   rows_per, part);
    TPO_LAUNCH_CHECK();
}

}  // namespace

namespace {
template <int MT, int NTT>
void dm_atb_launch(const double *A, int64_t lda, const double *B, int64_t ldb, int64_t n, int p, int q, int64_t rows_per,
                   int G, double *part, cudaStream_t st) {
    const size_t sm = 2 * sizeof(double) * ((size_t)AB_BK * (8 * AB_MAXT + 4) + (size_t)AB_BK * (8 * NTT + 4));
    TPO_CUDA(cudaFuncSetAttribute(dm_atb_kernel<MT, NTT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    dm_atb_kernel<MT, NTT><<<G, DM_NT, sm, st>>>(A, lda, B, ldb, n, p, q, rows_per, part);
    TPO_LAUNCH_CHECK();
}
template <int NTT>
void dm_atb_mt(int mt, const double *A, int64_t lda, const double *B, int64_t ldb, int64_t n, int p, int q,
               int64_t rows_per, int G, double *part, cudaStream_t st) {
    if (mt <= 8) dm_atb_launch<1, NTT>(A, lda, B, ldb, n, p, q, rows_per, G, part, st);
    else dm_atb_launch<2, NTT>(A, lda, B, ldb, n, p, q, rows_per, G, part, st);
}
}  // namespace

size_t ts_atb_ws(int p, int q) { return align_up(sizeof(double) * (size_t)sm_count_cached() * p * q) + 256; }

// out (p x q fp64) = A^T B, A n x p, B n x q fp64 (p, q <= 128): fixed-order split over rows
void ts_atb_f64(const double *A, int64_t lda, const double *B, int64_t ldb, int64_t n, int p, int q, double *out,
                Arena &ar, cudaStream_t st) {
    const int64_t rows_per = cdiv(cdiv(std::max<int64_t>(n, 1), sm_count_cached()), AB_BK) * AB_BK;
    const int G = (int)cdiv(std::max<int64_t>(n, 1), rows_per);
    const size_t mark = ar.off;
    double *part = ar.take<double>((size_t)G * p * q);
    const int mt = (p + 7) / 8;
    TPO_NT13(dm_atb_mt, (q + 7) / 8, mt, A, lda, B, ldb, n, p, q, rows_per, G, part, st);
    reduce_parts_kernel<<<cdiv((int64_t)p * q, 256), 256, 0, st>>>(part, G, (int64_t)p * q, out);
    TPO_LAUNCH_CHECK();
    ar.off = mark;
}

bool ts64_enabled() {
    const char *e = getenv("TPO_TS64");
    return !(e && e[0] == '0');
}
bool ts64_ups_enabled(int k) {
    const char *e = getenv("TPO_TS64_UPS");
    return ts64_enabled() && e && e[0] == '1' && k > 16 && k <= 104;
}

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

// Ups <- Ups . sqrt(max(RH,0) / (max(Ups M,0) + eps))  (Eq. update-Y with the R9 clamps), in place;
// k <= 104 (13 n-tiles of accumulators per warp)
void ts_ups_update(double *U, const double *RH, const double *M, int64_t n, int k, cudaStream_t st) {
    if (n == 0) return;
    DmArgs a{};
    a.A = U; a.lda = k; a.W = M; a.ldw = k; a.n = n; a.K = k; a.N = k; a.out = U; a.ldo = k; a.RH = RH;
    TPO_NT13(dm_ups, (k + 7) / 8, a, st);
}

size_t ts_rtu_ws(int64_t n, int64_t D, int k) {
    (void)n;
    return align_up(sizeof(double) * (size_t)sm_count_cached() * D * k) + 256;   // >= G * D * k
}

// RtU = R'^T (dinv . Ups) (D x k fp64)
void ts_rtu(const float *Rp, int64_t n, int64_t D, const float *dinv, const double *U, int k, double *RtU, Arena &ar,
            cudaStream_t st) {
    int NT, nblk;
    col_tiling(k, NT, nblk);
    const int nz = (int)cdiv(D, RT_DB);
    const int64_t want = std::max<int64_t>(1, sm_count_cached() / (nblk * nz));
    const int64_t rows_per = cdiv(cdiv(std::max<int64_t>(n, 1), want), RT_BK) * RT_BK;
    const int G = (int)cdiv(std::max<int64_t>(n, 1), rows_per);
    const size_t mark = ar.off;
    double *part = ar.take<double>((size_t)G * D * k);
    TPO_NT13(dm_rtu_launch, NT, Rp, n, (int)D, dinv, U, k, rows_per, G, nblk, part, st);
    reduce_parts_kernel<<<cdiv(D * k, 256), 256, 0, st>>>(part, G, D * k, RtU);
    TPO_LAUNCH_CHECK();
    ar.off = mark;
}

}  // namespace tpo
