// fp64-accurate row GEMM on the integer tensor cores (tcgen05 kind::i8):
//      out = diag(rs) . A . W          A: n x K fp32 (R'), W: K x N fp64 (H), out: n x N fp64
// the ONMF product RH = dinv . (R' H) of Alg. 2, and Gamma = R Psi Sigma^-1.
//
// Error-free splitting (Ozaki scheme, integer form).  Row i of A is scaled by 2^-E_i (E_i: the
// smallest power of two above max_j |A_ij|) and written as a 49-bit fixed-point number with a
// bias:  F'_ij = trunc(A_ij 2^(48 - E_i)) + 2^48 in [0, 2^49), cut into 7 unsigned 7-bit digits
// A'_p (p = 0 most significant).  Column l of W is scaled by 2^-E_l and cut into 7 signed 7-bit
// digits B_q of trunc(|W_jl| 2^(49 - E_l)) (sign on every digit).  Then
//      A_ij W_jl ~= 2^(E_i + E_l - 97) sum_{p,q} A'_p B_q 2^(7 (12 - p - q)) - (bias term)
// and the products of equal weight s = p + q are summed EXACTLY in one int32 TMEM accumulator
// acc_s (<= 7 K 127^2 < 2^31 for K <= 256 ... 19,000).  Pairs with p + q > 7 are dropped (their sum
// is below 2^-44 of max|A_i| max|W_l| K).  The bias 2^48 = 64 * 2^42 lives in digit 0 only, so it
// is removed exactly per accumulator: acc_s -= 64 sum_j B_s[j, l].  The epilogue combines the 8
// accumulators in int64 (hi = acc_0..3, lo = acc_4..7, both < 2^53), converts with one fp64
// rounding (fma(hi, 2^28, lo)), scales by powers of two (exact) and by rs_i (one rounding).
// Accuracy: |error| <~ 2^-44 K max|A_i| max|W_l| -- within a few units of fp64 DMMA's own
// rounding (K 2^-53 sum |A||W|) on these operands; parity is checked against an fp64 reference
// (tests/test_gpu_reduce.py) and, end to end, by the bit-exact Alg. 3 labels.
//
// Kernel (persistent, one CTA per SM, 448 threads):
//   warp 0      TMA producer: W's digit image once (bulk copy, resident in smem), then per
//               (row tile of 128, K chunk of 32) the fp32 A chunk (SWIZZLE_128B box) into a ring
//   warp 1      MMA issuer: per K chunk 34 tcgen05.mma kind::i8 (u8 x s8 -> s32), M = 128, N = NP,
//               K = 32, into the 8 accumulators acc_s (TMEM columns s * NP)
//   warps 2-9   slicers: fp32 chunk -> 7 digit planes (K-major, no-swizzle core-matrix layout)
//   warps 10-13 epilogue: TMEM -> int64 -> fp64 -> out (rows of the tile, TMEM lane quarter warp % 4)
#include <cuda.h>

#include <algorithm>

#include "tc_ptx.cuh"
#include "tpo_internal.cuh"

namespace tpo {
namespace {

constexpr int OZ_M = 128;                 // rows per tile
constexpr int OZ_KC = 32;                 // K chunk (fp32 columns) = one kind::i8 MMA K
constexpr int OZ_STG = 3;                 // fp32 staging stages
constexpr int OZ_SL = 7;                  // digits per operand
constexpr int OZ_SMAX = 7;                // kept digit pairs: p + q <= OZ_SMAX
constexpr int OZ_NACC = OZ_SMAX + 1;      // accumulators acc_0 .. acc_7
constexpr int OZ_STAGE_BYTES = OZ_M * OZ_KC * 4;      // 16 KB
constexpr int OZ_PLANE = OZ_M * OZ_KC;                // one digit plane of a chunk: 4 KB
constexpr int OZ_SBUF = OZ_SL * OZ_PLANE;             // 28 KB
constexpr int OZ_SLICERS = 8;
constexpr int OZ_EPI = 4;
constexpr int OZ_THREADS = 32 * (2 + OZ_SLICERS + OZ_EPI);
constexpr size_t OZ_B_MAX = 112 * 1024;               // resident digit image of W

struct OzArgs {
    int64_t n, ldo;
    int K, N, NP, Kp;        // Kp: K rounded up to OZ_KC; NP: N rounded up to 16
    int64_t ntiles;
    const int32_t *rowE;     // [n]
    const int32_t *colE;     // [NP]
    const int32_t *corr;     // [OZ_NACC][NP]
    const uint8_t *Bimg;     // [OZ_SL][NP x Kp] digit image (smem layout)
    const float *rs;         // [n] or null
    double *out;
};

__device__ __forceinline__ uint64_t desc_kmajor_noswz(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr & 0x3FFFF) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;                    // version (sm_100)
    return d;                                   // layout type 0: no swizzle (core matrices)
}

// kind::i8: s32 accumulate, A unsigned 8-bit, B signed 8-bit, both K-major, M x N
constexpr uint32_t idesc_i8(int M, int N) {
    return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
            tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int32_t *v) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = (int32_t)r[i];
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// 28 low bits -> 4 bytes of 7-bit digits (byte 0 = least significant digit)
__device__ __forceinline__ uint32_t spread7x4(uint32_t x) {
    return (x & 0x7Fu) | ((x << 1) & 0x7F00u) | ((x << 2) & 0x7F0000u) | ((x << 3) & 0x7F000000u);
}

// Digits of 4 consecutive elements of one row -> the 7 digit-plane words (byte e = element e).
__device__ __forceinline__ void slice4(const float4 a, float sc1, float sc2, uint32_t (&w)[OZ_SL]) {
    const float av[4] = {a.x, a.y, a.z, a.w};
    uint32_t L[4], H[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float x = (av[e] * sc1) * sc2;                       // exact: power-of-two scales
        long long f;
        asm("cvt.rzi.s64.f32 %0, %1;" : "=l"(f) : "f"(x));         // trunc(A 2^(48-E)), |f| < 2^48
        const unsigned long long fp = (unsigned long long)(f + (1ll << 48));   // biased, < 2^49
        L[e] = spread7x4((uint32_t)fp & 0x0FFFFFFFu);              // digits 6, 5, 4, 3
        H[e] = spread7x4((uint32_t)(fp >> 28));                    // digits 2, 1, 0
    }
    const uint32_t t0 = __byte_perm(L[0], L[1], 0x5140), t1 = __byte_perm(L[2], L[3], 0x5140);
    const uint32_t u0 = __byte_perm(L[0], L[1], 0x7362), u1 = __byte_perm(L[2], L[3], 0x7362);
    w[6] = __byte_perm(t0, t1, 0x5410);
    w[5] = __byte_perm(t0, t1, 0x7632);
    w[4] = __byte_perm(u0, u1, 0x5410);
    w[3] = __byte_perm(u0, u1, 0x7632);
    const uint32_t h0 = __byte_perm(H[0], H[1], 0x5140), h1 = __byte_perm(H[2], H[3], 0x5140);
    const uint32_t g0 = __byte_perm(H[0], H[1], 0x7362), g1 = __byte_perm(H[2], H[3], 0x7362);
    w[2] = __byte_perm(h0, h1, 0x5410);
    w[1] = __byte_perm(h0, h1, 0x7632);
    w[0] = __byte_perm(g0, g1, 0x5410);
}

__device__ __forceinline__ float pow2f(int e) {       // 2^e for -126 <= e <= 127
    return __int_as_float((e + 127) << 23);
}
__device__ __forceinline__ double pow2d(int e) {      // 2^e for -1022 <= e <= 1023
    return __longlong_as_double((long long)(e + 1023) << 52);
}

template <int NP>
__global__ void __launch_bounds__(OZ_THREADS, 1) oz_aw_kernel(const __grid_constant__ CUtensorMap mapA, OzArgs g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t bbytes = (uint32_t)OZ_SL * NP * g.Kp;
    const uint32_t stage_off = (bbytes + 1023) & ~1023u;
    const uint32_t slice_off = stage_off + OZ_STG * OZ_STAGE_BYTES;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + slice_off + 2 * OZ_SBUF);
    // bars: bfull, afull[STG], aempty[STG], sready[2], sfree[2], tfull, tempty
    uint64_t *bfull = bars, *afull = bars + 1, *aempty = afull + OZ_STG, *sready = aempty + OZ_STG;
    uint64_t *sfree = sready + 2, *tfull = sfree + 2, *tempty = tfull + 1;
    int32_t *sh_corr = reinterpret_cast<int32_t *>(tempty + 1);   // [OZ_NACC][NP]
    int32_t *sh_colE = sh_corr + OZ_NACC * NP;                    // [NP]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sh_colE + NP);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nkc = g.Kp / OZ_KC;
    constexpr uint32_t TMEM_COLS = (OZ_NACC * NP <= 128) ? 128 : (OZ_NACC * NP <= 256 ? 256 : 512);

    if (threadIdx.x == 0) {
        mbar_init(smem_u32(bfull), 1);
        for (int s = 0; s < OZ_STG; ++s) {
            mbar_init(smem_u32(&afull[s]), 1);
            mbar_init(smem_u32(&aempty[s]), OZ_SLICERS);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&sready[b]), OZ_SLICERS);
            mbar_init(smem_u32(&sfree[b]), 1);
        }
        mbar_init(smem_u32(tfull), 1);
        mbar_init(smem_u32(tempty), OZ_EPI);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    }
    for (int i = threadIdx.x; i < OZ_NACC * NP; i += blockDim.x) sh_corr[i] = g.corr[i];
    for (int i = threadIdx.x; i < NP; i += blockDim.x) sh_colE[i] = g.colE[i];
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ---------------- producer ----------------
        if (lane == 0) {
            const uint32_t bar = smem_u32(bfull);
            mbar_expect_tx(bar, bbytes);
            for (uint32_t o = 0; o < bbytes; o += 32768)
                bulk_g2s(smem_u32(smem) + o, g.Bimg + o, std::min<uint32_t>(32768, bbytes - o), bar);
            int64_t gc = 0;
            for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
                for (int c = 0; c < nkc; ++c, ++gc) {
                    const int s = (int)(gc % OZ_STG);
                    const int64_t j = gc / OZ_STG;
                    if (j > 0) mbar_wait(smem_u32(&aempty[s]), (uint32_t)((j - 1) & 1));
                    const uint32_t full = smem_u32(&afull[s]);
                    mbar_expect_tx(full, OZ_STAGE_BYTES);
                    tma_load_2d(smem_u32(smem + stage_off + s * OZ_STAGE_BYTES), &mapA, full, c * OZ_KC,
                                (int)(t * OZ_M));
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        constexpr uint32_t idesc = idesc_i8(OZ_M, NP);
        mbar_wait(smem_u32(bfull), 0);
        const uint32_t bres = smem_u32(smem);
        const uint32_t sbo_b = 8u * (uint32_t)g.Kp;                   // 8 rows of W's image
        int64_t gc = 0;
        int i = 0;
        for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x, ++i) {
            if (i > 0) mbar_wait(smem_u32(tempty), (uint32_t)((i - 1) & 1));
            fence_after();
            for (int c = 0; c < nkc; ++c, ++gc) {
                const int b = (int)(gc & 1);
                mbar_wait(smem_u32(&sready[b]), (uint32_t)((gc >> 1) & 1));
                fence_after();
                if (lane == 0) {
                    const uint32_t abase = smem_u32(smem + slice_off + b * OZ_SBUF);
#pragma unroll
                    for (int p = 0; p < OZ_SL; ++p) {
                        const uint64_t da = desc_kmajor_noswz(abase + p * OZ_PLANE, 128, 256);
#pragma unroll
                        for (int q = 0; q < OZ_SL; ++q) {
                            if (p + q > OZ_SMAX) continue;
                            const int s = p + q;
                            const uint64_t db = desc_kmajor_noswz(
                                bres + (uint32_t)q * NP * g.Kp + (uint32_t)c * (OZ_KC * 8), 128, sbo_b);
                            const bool first = (c == 0) && (p == (s > OZ_SL - 1 ? s - (OZ_SL - 1) : 0));
                            mma_i8(tmem_base + (uint32_t)(s * NP), da, db, idesc, first ? 0u : 1u);
                        }
                    }
                    mma_commit(smem_u32(&sfree[b]));
                    if (c == nkc - 1) mma_commit(smem_u32(tfull));
                }
                __syncwarp();
            }
        }
    } else if (warp < 2 + OZ_SLICERS) {
        // ---------------- slicers: 16 rows per warp ----------------
        const int sw = warp - 2;
        int64_t gc = 0;
        for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
            float sc1[2], sc2[2];
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const int64_t row = t * OZ_M + 16 * sw + 8 * rr + (lane >> 2);
                const int E = row < g.n ? g.rowE[row] : 0;
                const int sh = 48 - E;                                 // scale 2^(48 - E) in two steps
                const int h1 = sh / 2;
                sc1[rr] = pow2f(h1);
                sc2[rr] = pow2f(sh - h1);
            }
            for (int c = 0; c < nkc; ++c, ++gc) {
                const int s = (int)(gc % OZ_STG);
                const int b = (int)(gc & 1);
                mbar_wait(smem_u32(&afull[s]), (uint32_t)((gc / OZ_STG) & 1));
                if (gc >= 2) mbar_wait(smem_u32(&sfree[b]), (uint32_t)(((gc >> 1) - 1) & 1));
                const uint8_t *stg = smem + stage_off + s * OZ_STAGE_BYTES;
                uint8_t *sb = smem + slice_off + b * OZ_SBUF;
#pragma unroll
                for (int rr = 0; rr < 2; ++rr) {
                    const int r = 16 * sw + 8 * rr + (lane >> 2);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int c16 = 4 * h + (lane & 3);                   // 16-byte chunk of the fp32 row
                        const float4 a = *reinterpret_cast<const float4 *>(stg + r * 128 + ((c16 ^ (r & 7)) << 4));
                        uint32_t w[OZ_SL];
                        slice4(a, sc1[rr], sc2[rr], w);
                        const int kb = 16 * h + 4 * (lane & 3);               // byte (= element) in the K chunk
                        const uint32_t off = (uint32_t)((r >> 3) * 256 + (kb >> 4) * 128 + (r & 7) * 16 + (kb & 15));
#pragma unroll
                        for (int p = 0; p < OZ_SL; ++p) *reinterpret_cast<uint32_t *>(sb + p * OZ_PLANE + off) = w[p];
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(smem_u32(&aempty[s]));
                    mbar_arrive(smem_u32(&sready[b]));
                }
            }
        }
    } else {
        // ---------------- epilogue ----------------
        const int q4 = warp & 3;
        int i = 0;
        for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x, ++i) {
            mbar_wait(smem_u32(tfull), (uint32_t)(i & 1));
            fence_after();
            const int64_t row = t * OZ_M + 32 * q4 + lane;
            const bool ok = row < g.n;
            const int E = ok ? g.rowE[row] : 0;
            const double rsc = (ok && g.rs ? (double)g.rs[row] : 1.0);
            double *orow = g.out + (ok ? row : 0) * g.ldo;
#pragma unroll 1
            for (int cb = 0; cb < NP; cb += 8) {
                int32_t v[OZ_NACC][8];
#pragma unroll
                for (int s = 0; s < OZ_NACC; ++s)
                    tmem_ld8(tmem_base + ((uint32_t)(32 * q4) << 16) + (uint32_t)(s * NP + cb), v[s]);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int l = cb + j;
                    long long hi = 0, lo = 0;
#pragma unroll
                    for (int s = 0; s < 4; ++s) hi = hi * 128 + (long long)(v[s][j] - sh_corr[s * NP + l]);
#pragma unroll
                    for (int s = 4; s < OZ_NACC; ++s) lo = lo * 128 + (long long)(v[s][j] - sh_corr[s * NP + l]);
                    const double cval = fma((double)hi, 268435456.0, (double)lo) * pow2d(E + sh_colE[l] - 62);
                    if (ok && l < g.N) orow[l] = cval * rsc;
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(tempty));
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                     : "memory");
    }
}

// E_i = smallest e with max_j |A_ij| < 2^e (0 for a zero row); one warp per row.
__global__ void oz_rowexp_kernel(const float *__restrict__ A, int64_t lda, int64_t n, int K, int32_t *__restrict__ E) {
    const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    float m = 0.f;
    for (int j = lane; j < K; j += 32) m = fmaxf(m, fabsf(A[row * lda + j]));
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) {
        int e = 0;
        if (m > 0.f) frexpf(m, &e);          // m = f 2^e, f in [0.5, 1): m < 2^e
        E[row] = e;
    }
}

// W (K x N fp64, row-major) -> digit image [OZ_SL][NP x Kp] in the kernel's shared-memory layout,
// column exponents E_l and the bias corrections corr[s][l] = 64 sum_j B_s[j, l] (s < OZ_SL).
// One block per padded column l.
__global__ void oz_bprep_kernel(const double *__restrict__ W, int K, int N, int NP, int Kp, uint8_t *__restrict__ img,
                                int32_t *__restrict__ colE, int32_t *__restrict__ corr) {
    const int l = blockIdx.x;
    __shared__ double red[32];
    __shared__ int sred[OZ_SL][32];
    double m = 0.0;
    if (l < N)
        for (int j = threadIdx.x; j < K; j += blockDim.x) m = fmax(m, fabs(W[(int64_t)j * N + l]));
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    int E = 0;
    if (red[0] > 0.0) frexp(red[0], &E);
    int dsum[OZ_SL];
#pragma unroll
    for (int q = 0; q < OZ_SL; ++q) dsum[q] = 0;
    const double scale = ldexp(1.0, 49 - E);
    for (int j = threadIdx.x; j < Kp; j += blockDim.x) {
        const double w = (l < N && j < K) ? W[(int64_t)j * N + l] : 0.0;
        const long long f = (long long)(fabs(w) * scale);          // trunc, < 2^49 (exact scaling)
        const int sg = w < 0.0 ? -1 : 1;
        const int64_t off = (int64_t)(l >> 3) * (8 * Kp) + (j >> 4) * 128 + (l & 7) * 16 + (j & 15);
#pragma unroll
        for (int q = 0; q < OZ_SL; ++q) {
            const int d = sg * (int)((f >> (7 * (OZ_SL - 1 - q))) & 127);
            img[(int64_t)q * NP * Kp + off] = (uint8_t)(int8_t)d;
            dsum[q] += d;
        }
    }
#pragma unroll
    for (int q = 0; q < OZ_SL; ++q) {
        int v = dsum[q];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0) sred[q][threadIdx.x >> 5] = v;
    }
    __syncthreads();
    if (threadIdx.x < OZ_NACC) {
        int v = 0;
        if (threadIdx.x < OZ_SL)
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += sred[threadIdx.x][w];
        corr[threadIdx.x * NP + l] = 64 * v;
    }
    if (threadIdx.x == 0) colE[l] = E;
}

CUtensorMap oz_map(const float *A, int64_t n, int64_t K, int64_t lda) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)lda * sizeof(float)};
    const cuuint32_t box[2] = {OZ_KC, OZ_M};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(A), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(TPO_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

int oz_np(int N) { return (N + 15) / 16 * 16; }
int oz_kp(int64_t K) { return (int)((K + OZ_KC - 1) / OZ_KC * OZ_KC); }

size_t oz_smem(int NP, int Kp) {
    const size_t b = ((size_t)OZ_SL * NP * Kp + 1023) & ~size_t(1023);
    return 1024 + b + OZ_STG * OZ_STAGE_BYTES + 2 * OZ_SBUF + 16 * 8 + sizeof(int32_t) * (OZ_NACC + 1) * NP + 16;
}

template <int NP>
void oz_launch(const CUtensorMap &map, const OzArgs &a, cudaStream_t st) {
    const size_t sm = oz_smem(NP, a.Kp);
    TPO_CUDA(cudaFuncSetAttribute(oz_aw_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const int grid = (int)std::min<int64_t>(a.ntiles, sm_count());
    oz_aw_kernel<NP><<<grid, OZ_THREADS, sm, st>>>(map, a);
    TPO_LAUNCH_CHECK();
}

}  // namespace

bool oz_enabled() {
    const char *e = getenv("TPO_OZ");
    return !(e && e[0] == '0');
}

bool oz_aw_supported(int64_t K, int N) {
    if (K < 1 || N < 1 || N > 64 || K > 16384) return false;
    if ((size_t)OZ_SL * oz_np(N) * oz_kp(K) > OZ_B_MAX) return false;
    return oz_smem(oz_np(N), oz_kp(K)) <= 227 * 1024;
}

size_t oz_aw_ws(int64_t K, int N) {
    Arena ar(nullptr, 0);
    const int NP = oz_np(N), Kp = oz_kp(K);
    ar.take<uint8_t>((size_t)OZ_SL * NP * Kp);
    ar.take<int32_t>(NP);
    ar.take<int32_t>((size_t)OZ_NACC * NP);
    return ar.off + 256;
}

void oz_rowexp(const float *A, int64_t lda, int64_t n, int K, int32_t *E, cudaStream_t st) {
    if (n == 0) return;
    oz_rowexp_kernel<<<cdiv(n * 32, 256), 256, 0, st>>>(A, lda, n, K, E);
    TPO_LAUNCH_CHECK();
}

// out = diag(rs) A W (n x N fp64, ldo) on the integer tensor cores; rowE from oz_rowexp(A).
void oz_aw_f64(const float *A, int64_t lda, const float *rs, const int32_t *rowE, const double *W, int64_t n, int K,
               int N, double *out, int64_t ldo, Arena &ar, cudaStream_t st) {
    if (n == 0 || N == 0) return;
    TPO_REQUIRE(oz_aw_supported(K, N), "oz_aw_f64: unsupported shape");
    TPO_REQUIRE(lda % 4 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0, "oz_aw_f64: A must be 16-byte aligned");
    const size_t mark = ar.off;
    const int NP = oz_np(N), Kp = oz_kp(K);
    uint8_t *img = ar.take<uint8_t>((size_t)OZ_SL * NP * Kp);
    int32_t *colE = ar.take<int32_t>(NP);
    int32_t *corr = ar.take<int32_t>((size_t)OZ_NACC * NP);
    oz_bprep_kernel<<<NP, 256, 0, st>>>(W, K, N, NP, Kp, img, colE, corr);
    TPO_LAUNCH_CHECK();
    OzArgs a{};
    a.n = n; a.ldo = ldo; a.K = K; a.N = N; a.NP = NP; a.Kp = Kp;
    a.ntiles = cdiv(n, OZ_M);
    a.rowE = rowE; a.colE = colE; a.corr = corr; a.Bimg = img; a.rs = rs; a.out = out;
    const CUtensorMap map = oz_map(A, n, K, lda);
    switch (NP) {
        case 16: oz_launch<16>(map, a, st); break;
        case 32: oz_launch<32>(map, a, st); break;
        case 48: oz_launch<48>(map, a, st); break;
        default: oz_launch<64>(map, a, st); break;
    }
    ar.off = mark;
}

// Alg. 2's RH = dinv . (R' H) for every ONMF iteration of one solve: R''s row exponents once, then
// the integer-tensor-core product (or the fp64 DMMA path when the shape is not supported).
RhPlan rh_plan_at(int32_t *rowE, const float *Rp, int64_t n, int64_t D, int k, cudaStream_t st) {
    RhPlan p;
    p.oz = oz_enabled() && n > 0 && D % 4 == 0 && oz_aw_supported(D, k) &&
           (reinterpret_cast<uintptr_t>(Rp) & 15) == 0;
    p.rowE = rowE;
    if (p.oz) oz_rowexp(Rp, D, n, (int)D, p.rowE, st);
    return p;
}
RhPlan rh_plan(const float *Rp, int64_t n, int64_t D, int k, Arena &ar, cudaStream_t st) {
    return rh_plan_at(ar.take<int32_t>(std::max<int64_t>(n, 1)), Rp, n, D, k, st);
}
size_t rh_plan_ws(int64_t n) { return align_up(sizeof(int32_t) * (size_t)std::max<int64_t>(n, 1) + 1); }
size_t rh_apply_ws(int64_t D, int k) { return oz_aw_supported(D, k) ? oz_aw_ws(D, k) : 0; }

void rh_apply(const RhPlan &p, const float *Rp, const float *dinv, const double *H, int64_t n, int64_t D, int k,
              double *RH, Arena &ar, cudaStream_t st) {
    if (n == 0) return;
    if (p.oz) oz_aw_f64(Rp, D, dinv, p.rowE, H, n, (int)D, k, RH, k, ar, st);
    else tsgemm_AW_f64(Rp, D, dinv, H, n, D, k, RH, k, st);
}

}  // namespace tpo
