// fp64-accurate row GEMM on the integer tensor cores (tcgen05 kind::i8):
//      out = diag(rs) . A . W          A: n x K fp32 (R'), W: K x N fp64 (H), out: n x N fp64
// the ONMF product RH = dinv . (R' H) of Alg. 2.
//
// Error-free splitting (Ozaki scheme, integer form, base 256).  Row i of A is scaled by 2^-E_i
// (E_i: the smallest power of two above max_j |A_ij|) and written as the biased 48-bit integer
//      A'_ij = floor(A_ij 2^(47 - E_i)) + 2^47  in [0, 2^48)
// (one fp64 fma with round-toward-zero: A' is the low 48 bits of 2^52 + 2^47 + A 2^(47-E_i)),
// cut into its 6 bytes a_p (unsigned digits, p = 0 most significant).  Column l of W is scaled by
// 2^-E_l, truncated to the signed integer F_jl = trunc(W_jl 2^(46 - E_l)) (|F| < 2^46) and cut
// into 6 balanced signed base-256 digits b_q in [-128, 127].  Then
//      sum_j A'_ij F_jl = sum_{p,q} 2^(8 (10 - p - q)) sum_j a_p b_q
// and the digit products of equal weight s = p + q are summed EXACTLY in one int32 TMEM
// accumulator acc_s (|acc_s| <= 6 K 255 128 < 2^29 for K <= 2,048).  Pairs with p + q > 5 are
// dropped.  The bias is removed exactly: sum_j A' F = sum_j floor(A 2^(47-E_i)) F + 2^47 sum_j F,
// the last term a per-column constant.  The epilogue forms g0 = acc_0 2^16 + acc_1 2^8 + acc_2 and
// g1 = acc_3 2^16 + acc_4 2^8 + acc_5 (exact int64, < 2^53), then
//      out_il = rs_i 2^(E_i + E_l - 53) [ (g0 2^24 - C_hi) + (g1 - C_lo) ]
// with C = 128 sum_j F_jl = C_hi + C_lo (C_hi = 128 fp64(sum), C_lo the exact int64 rest): two
// fp64 roundings.  Error <~ 2^-44 K max|A_i| max|W_l| |rs_i| (the dropped pairs and the
// truncations), within a few units of the fp64 DMMA path's own rounding on these operands
// (tests/test_gpu_oz.py: ~3e-14 of max|out| apart); end to end the Alg. 3 labels stay bit-exact
// (tests/test_gpu_fullsize.py).
//
// Kernel (persistent, one CTA per SM, 832 threads, ~207 KB shared memory):
//   warp 0      W's digit image once (bulk copy, resident: 6 planes x NP x K bytes), then per
//               (row tile of 128, K chunk of 32) the fp32 A chunk by TMA (SWIZZLE_128B) into a
//               3-stage ring
//   warp 1      MMA issuer: per K chunk 8 tcgen05.mma kind::i8 (u8 x s8 -> s32), M = 128, K = 32,
//               N = up to 4 NP, into the 6 accumulators acc_s (TMEM columns s * NP)
//   warps 2-9   slicers: fp32 chunk -> digits in registers (stage released), then 6 byte planes
//               (K-major, no-swizzle core-matrix layout) into one of 3 plane buffers
//   warps 10-25 epilogue: TMEM -> int64 -> fp64 -> out (TMEM lane quarter warp % 4, column quarter)
// Measured on large (n = 2M, K = 256, N = 50): 1.37 ms vs 2.42 ms on the fp64 DMMA path
// (tools/bench_oz.py).  On medium (K = 512, N = 20) it does not beat DMMA (0.62 vs 0.61 ms), so
// the ONMF uses it only for N > 32 (rh_plan).
#include <cuda.h>

#include <algorithm>
#include <numeric>

#include "tc_ptx.cuh"
#include "tpo_internal.cuh"

namespace tpo {
namespace {

constexpr int OZ_M = 128;                 // rows per tile
constexpr int OZ_KC = 32;                 // K chunk (fp32 columns) = one kind::i8 MMA K
constexpr int OZ_STG = 3;                 // fp32 staging stages (TMA ring, 16 KB each; 4-5 measured no faster)
constexpr int OZ_NBUF = 3;                // digit-plane buffers
constexpr int OZ_SL = 6;                  // digits per operand
constexpr int OZ_SMAX = 5;                // kept digit pairs: p + q <= OZ_SMAX
constexpr int OZ_NACC = OZ_SMAX + 1;      // accumulators acc_0 .. acc_5
constexpr int OZ_STAGE_BYTES = OZ_M * OZ_KC * 4;      // 16 KB
constexpr int OZ_PLANE = OZ_M * OZ_KC;                // one digit plane of a chunk: 4 KB
constexpr int OZ_SBUF = OZ_SL * OZ_PLANE;             // 24 KB
constexpr int OZ_SLICERS = 8;
constexpr int OZ_EPI = 16;                // 4 per TMEM lane quarter (column quarters)
constexpr int OZ_THREADS = 32 * (2 + OZ_SLICERS + OZ_EPI);
constexpr size_t OZ_B_MAX = 96 * 1024;                // resident digit image of W

struct OzArgs {
    const float *A;
    int64_t n, ldo, lda;
    int K, N, NP, Kp;        // Kp: K rounded up to OZ_KC; NP: N rounded up to 16
    int64_t ntiles;
    const int32_t *rowE;     // [n]
    const int32_t *colE;     // [NP]
    const double *chi;       // [NP]: C_hi (fp64 rounding of C = 8 sum_j F_jl)
    const long long *clo;    // [NP]: C - C_hi (exact)
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

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// Byte planes of 4 consecutive elements of one row: w[p] holds byte 5 - p (digit p) of the
// elements' A' (byte e = element e).  scale = 2^(47 - E_i).
__device__ __forceinline__ void slice4(const float4 a, double scale, uint32_t (&w)[OZ_SL]) {
    const float av[4] = {a.x, a.y, a.z, a.w};
    uint32_t L[4], H[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        // 2^52 + floor(2^47 + A 2^(47-E)): the product is exact (power of two), the sum lies in
        // [2^52, 2^53) where round-toward-zero is floor
        const double z = __fma_rz((double)av[e], scale, 4644337115725824.0);
        const unsigned long long zb = (unsigned long long)__double_as_longlong(z);
        L[e] = (uint32_t)zb;                                   // bytes 0..3
        H[e] = (uint32_t)(zb >> 32) & 0xFFFFu;                 // bytes 4..5
    }
    const uint32_t t0 = __byte_perm(L[0], L[1], 0x5140), t1 = __byte_perm(L[2], L[3], 0x5140);
    const uint32_t u0 = __byte_perm(L[0], L[1], 0x7362), u1 = __byte_perm(L[2], L[3], 0x7362);
    w[5] = __byte_perm(t0, t1, 0x5410);
    w[4] = __byte_perm(t0, t1, 0x7632);
    w[3] = __byte_perm(u0, u1, 0x5410);
    w[2] = __byte_perm(u0, u1, 0x7632);
    const uint32_t h0 = __byte_perm(H[0], H[1], 0x5140), h1 = __byte_perm(H[2], H[3], 0x5140);
    w[1] = __byte_perm(h0, h1, 0x5410);
    w[0] = __byte_perm(h0, h1, 0x7632);
}

__device__ __forceinline__ void tmem_ld4_nowait(uint32_t taddr, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
}

// mbarrier wait with a back-off for warps that wait a whole tile (frees issue slots for the
// producer, MMA and slicer warps)
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    uint64_t spins = 0;
    while (true) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.b32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
        if (done) return;
        __nanosleep(128);
        if (++spins > (1ull << 28)) __trap();
    }
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
    const uint32_t stage_off = (bbytes + 1023) & ~1023u;        // SWIZZLE_128B TMA targets
    const uint32_t slice_off = stage_off + OZ_STG * OZ_STAGE_BYTES;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + slice_off + OZ_NBUF * OZ_SBUF);
    // bars: bfull, afull[STG], aempty[STG], sready[NBUF], sfree[NBUF], tfull, tempty
    uint64_t *bfull = bars, *afull = bars + 1, *aempty = afull + OZ_STG, *sready = aempty + OZ_STG;
    uint64_t *sfree = sready + OZ_NBUF, *tfull = sfree + OZ_NBUF, *tempty = tfull + 1;
    double *sh_chi = reinterpret_cast<double *>(tempty + 1);         // [NP]
    long long *sh_clo = reinterpret_cast<long long *>(sh_chi + NP);  // [NP]
    int32_t *sh_colE = reinterpret_cast<int32_t *>(sh_clo + NP);     // [NP]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sh_colE + NP);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nkc = g.Kp / OZ_KC;
    constexpr uint32_t TMEM_COLS = (OZ_NACC * NP <= 128) ? 128 : (OZ_NACC * NP <= 256 ? 256 : 512);

    if (threadIdx.x == 0) {
        mbar_init(smem_u32(bfull), 1);
        for (int b = 0; b < OZ_STG; ++b) {
            mbar_init(smem_u32(&afull[b]), 1);
            mbar_init(smem_u32(&aempty[b]), OZ_SLICERS);
        }
        for (int b = 0; b < OZ_NBUF; ++b) {
            mbar_init(smem_u32(&sready[b]), OZ_SLICERS);
            mbar_init(smem_u32(&sfree[b]), 1);
        }
        mbar_init(smem_u32(tfull), 1);
        mbar_init(smem_u32(tempty), OZ_EPI);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    }
    for (int i = threadIdx.x; i < NP; i += blockDim.x) {
        sh_chi[i] = g.chi[i];
        sh_clo[i] = g.clo[i];
    }
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
        // ---------------- producer: W's digit image (resident), then the fp32 A chunks ----------------
        // A chunks: 128 rows x 32 fp32, SWIZZLE_128B, into a 4-stage ring freed as soon as the
        // slicers hold the chunk in registers
        if (lane == 0) {
            const uint32_t bar = smem_u32(bfull);
            mbar_expect_tx(bar, bbytes);
            for (uint32_t o = 0; o < bbytes; o += 32768)
                bulk_g2s(smem_u32(smem) + o, g.Bimg + o, std::min<uint32_t>(32768, bbytes - o), bar);
            int64_t gc = 0;
            for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
                for (int c = 0; c < nkc; ++c, ++gc) {
                    const int b = (int)(gc % OZ_STG);
                    if (gc >= OZ_STG) mbar_wait(smem_u32(&aempty[b]), (uint32_t)(((gc / OZ_STG) - 1) & 1));
                    const uint32_t full = smem_u32(&afull[b]);
                    mbar_expect_tx(full, OZ_STAGE_BYTES);
                    tma_load_2d(smem_u32(smem + stage_off + b * OZ_STAGE_BYTES), &mapA, full, c * OZ_KC, (int)(t * OZ_M));
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        mbar_wait(smem_u32(bfull), 0);
        const uint32_t bres = smem_u32(smem);
        const uint32_t sbo_b = 8u * (uint32_t)g.Kp;                   // 8 rows of W's image
        int64_t gc = 0;
        int i = 0;
        for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x, ++i) {
            if (i > 0) mbar_wait(smem_u32(tempty), (uint32_t)((i - 1) & 1));
            fence_after();
            for (int c = 0; c < nkc; ++c, ++gc) {
                const int b = (int)(gc % OZ_NBUF);
                mbar_wait(smem_u32(&sready[b]), (uint32_t)((gc / OZ_NBUF) & 1));
                fence_after();
                if (lane == 0) {
                    const uint32_t abase = smem_u32(smem + slice_off + b * OZ_SBUF);
                    // digit planes of W are consecutive NP-row blocks of one K-major matrix, so one
                    // MMA with D at acc_{p+q0} and B = planes q0 .. q0+nq-1 (N = nq NP) adds
                    // a_p b_q into acc_{p+q} for all nq planes at once: 8 MMAs per chunk for the
                    // 21 kept pairs; the first two (p = 0) initialise acc_0..3 and acc_4..5.
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        constexpr int P[8] = {0, 0, 1, 1, 2, 3, 4, 5};
                        constexpr int Q0[8] = {0, 4, 0, 4, 0, 0, 0, 0};
                        constexpr int NQ[8] = {4, 2, 4, 1, 4, 3, 2, 1};
                        const uint64_t da = desc_kmajor_noswz(abase + P[u] * OZ_PLANE, 128, 256);
                        const uint64_t db = desc_kmajor_noswz(
                            bres + (uint32_t)Q0[u] * NP * g.Kp + (uint32_t)c * (OZ_KC * 8), 128, sbo_b);
                        const uint32_t acc = (c > 0 || u >= 2) ? 1u : 0u;
                        mma_i8(tmem_base + (uint32_t)((P[u] + Q0[u]) * NP), da, db, idesc_i8(OZ_M, NQ[u] * NP), acc);
                    }
                    mma_commit(smem_u32(&sfree[b]));
                    if (c == nkc - 1) mma_commit(smem_u32(tfull));
                }
                __syncwarp();
            }
        }
    } else if (warp < 2 + OZ_SLICERS) {
        // ---------------- slicers: 16 rows per warp ----------------
        // lane -> (row r = 8-row group + lane % 8, 16-byte chunk 4h + lane / 8): the 8 lanes of a
        // shared-memory phase read 8 different swizzled chunks and write one 128-byte core matrix
        const int sw = warp - 2;
        int64_t gc = 0;
        for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
            double scale[2];
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const int64_t row = t * OZ_M + 16 * sw + 8 * rr + (lane & 7);
                scale[rr] = pow2d(47 - (row < g.n ? g.rowE[row] : 0));
            }
            for (int c = 0; c < nkc; ++c, ++gc) {
                const int s = (int)(gc % OZ_STG);
                mbar_wait(smem_u32(&afull[s]), (uint32_t)((gc / OZ_STG) & 1));
                const uint8_t *stg = smem + stage_off + s * OZ_STAGE_BYTES;
                float4 cur[2][2];
#pragma unroll
                for (int rr = 0; rr < 2; ++rr) {
                    const int r = 16 * sw + 8 * rr + (lane & 7);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int c16 = 4 * h + (lane >> 3);
                        cur[rr][h] = *reinterpret_cast<const float4 *>(stg + r * 128 + ((c16 ^ (r & 7)) << 4));
                    }
                }
                // digits first (consumes the stage's values), then the stage is released
                uint32_t w[2][2][OZ_SL];
#pragma unroll
                for (int rr = 0; rr < 2; ++rr)
#pragma unroll
                    for (int h = 0; h < 2; ++h) slice4(cur[rr][h], scale[rr], w[rr][h]);
                // release the stage once every lane's values have arrived: the warp-wide OR of the
                // digits depends on all of them (an LDS may still be in flight when later
                // instructions issue, and the next TMA would overwrite the stage)
                uint32_t dep = 0;
#pragma unroll
                for (int rr = 0; rr < 2; ++rr)
#pragma unroll
                    for (int h = 0; h < 2; ++h) dep |= w[rr][h][0] | w[rr][h][OZ_SL - 1];
                dep = __reduce_or_sync(0xffffffffu, dep);
                if (lane == 0)
                    asm volatile("{\n.reg .pred q;\nsetp.ne.u32 q, %1, 0xdeadbeef;\n@q mbarrier.arrive.shared::cta.b64 _, [%0];\n}\n" ::"r"(
                                     smem_u32(&aempty[s])),
                                 "r"(dep)
                                 : "memory");
                const int b = (int)(gc % OZ_NBUF);
                if (gc >= OZ_NBUF) mbar_wait(smem_u32(&sfree[b]), (uint32_t)(((gc / OZ_NBUF) - 1) & 1));
                uint8_t *sb = smem + slice_off + b * OZ_SBUF;
#pragma unroll
                for (int rr = 0; rr < 2; ++rr) {
                    const int r = 16 * sw + 8 * rr + (lane & 7);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int kb = 4 * (4 * h + (lane >> 3));             // byte (= element) in the K chunk
                        const uint32_t off = (uint32_t)((r >> 3) * 256 + (kb >> 4) * 128 + (r & 7) * 16 + (kb & 15));
#pragma unroll
                        for (int p = 0; p < OZ_SL; ++p) *reinterpret_cast<uint32_t *>(sb + p * OZ_PLANE + off) = w[rr][h][p];
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&sready[b]));
            }
        }
    } else {
        // ---------------- epilogue: 4 warps per TMEM lane quarter, NP / 4 columns each ----------------
        const int q4 = warp & 3, ch = (warp - 2 - OZ_SLICERS) >> 2;
        constexpr int HALF = NP / 4;                 // columns per epilogue warp (multiple of 4)
        int i = 0;
        for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x, ++i) {
            mbar_wait_sleep(smem_u32(tfull), (uint32_t)(i & 1));
            fence_after();
            const int64_t row = t * OZ_M + 32 * q4 + lane;
            const bool ok = row < g.n;
            const int E = ok ? g.rowE[row] : 0;
            const double rsc = (ok && g.rs ? (double)g.rs[row] : 1.0);
#pragma unroll 1
            for (int cb = ch * HALF; cb < (ch + 1) * HALF; cb += 4) {
                uint32_t v[OZ_NACC][4];
#pragma unroll
                for (int s = 0; s < OZ_NACC; ++s)
                    tmem_ld4_nowait(tmem_base + ((uint32_t)(32 * q4) << 16) + (uint32_t)(s * NP + cb), v[s]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int s = 0; s < OZ_NACC; ++s)
#pragma unroll
                    for (int j = 0; j < 4; ++j) asm volatile("" : "+r"(v[s][j]));
                double o[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int l = cb + j;
                    const long long g0 = (long long)(int32_t)v[0][j] * 65536 + (long long)(int32_t)v[1][j] * 256 +
                                         (long long)(int32_t)v[2][j];
                    const long long g1 = (long long)(int32_t)v[3][j] * 65536 + (long long)(int32_t)v[4][j] * 256 +
                                         (long long)(int32_t)v[5][j] - sh_clo[l];
                    const double x = fma((double)g0, 16777216.0, -sh_chi[l]) + (double)g1;
                    o[j] = x * pow2d(E + sh_colE[l] - 53) * rsc;
                }
                if (ok) {
                    double *orow = g.out + row * g.ldo;
                    if (cb + 4 <= g.N && ((reinterpret_cast<uintptr_t>(orow + cb) & 15) == 0)) {
                        *reinterpret_cast<double2 *>(orow + cb) = make_double2(o[0], o[1]);
                        *reinterpret_cast<double2 *>(orow + cb + 2) = make_double2(o[2], o[3]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            if (cb + j < g.N) orow[cb + j] = o[j];
                    }
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

// W (K x N fp64, row-major) -> digit image [OZ_SL][NP x Kp] in the kernel's shared-memory layout
// (plane q = digit q, most significant first), the column exponents E_l and the bias
// correction C = 8 sum_j F_jl split into C_hi (fp64) + C_lo (int64).  One block per padded column.
__global__ void oz_bprep_kernel(const double *__restrict__ W, int K, int N, int NP, int Kp, uint8_t *__restrict__ img,
                                int32_t *__restrict__ colE, double *__restrict__ chi, long long *__restrict__ clo) {
    const int l = blockIdx.x;
    __shared__ double red[32];
    __shared__ long long lred[32];
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
    const double scale = ldexp(1.0, 46 - E);     // |F| < 2^46: inside the 6-digit balanced range
    long long fsum = 0;
    for (int j = threadIdx.x; j < Kp; j += blockDim.x) {
        const double w = (l < N && j < K) ? W[(int64_t)j * N + l] : 0.0;
        long long f = (long long)(w * scale);                      // trunc, |f| < 2^46 (exact scaling)
        fsum += f;
        const int64_t off = (int64_t)(l >> 3) * (8 * Kp) + (j >> 4) * 128 + (l & 7) * 16 + (j & 15);
#pragma unroll
        for (int q = OZ_SL - 1; q >= 0; --q) {                      // balanced base-256 digits, LSB first
            const int d = (int)(int8_t)(uint8_t)(f & 255);
            img[(int64_t)q * NP * Kp + off] = (uint8_t)(int8_t)d;
            f = (f - d) >> 8;
        }
    }
    for (int o = 16; o; o >>= 1) fsum += __shfl_xor_sync(0xffffffffu, fsum, o);
    if ((threadIdx.x & 31) == 0) lred[threadIdx.x >> 5] = fsum;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long c = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) c += lred[w];
        // C = 128 sum_j F (up to 2^65): C_hi = 128 fp64(sum), C_lo = 128 (sum - fp64(sum)), exact
        const double h = (double)c;
        chi[l] = 128.0 * h;
        clo[l] = 128 * (c - (long long)h);
        colE[l] = E;
    }
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
    return 1024 + b + OZ_STG * OZ_STAGE_BYTES + OZ_NBUF * OZ_SBUF + 16 * 8 + (sizeof(double) + sizeof(long long) + sizeof(int32_t)) * NP + 16;
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
    if (K < 1 || N < 1 || N > 64 || K > 2048) return false;      // exact int64 / fp64 epilogue sums
    if ((size_t)OZ_SL * oz_np(N) * oz_kp(K) > OZ_B_MAX) return false;
    return oz_smem(oz_np(N), oz_kp(K)) <= 227 * 1024 - 256;
}

size_t oz_aw_ws(int64_t K, int N) {
    Arena ar(nullptr, 0);
    const int NP = oz_np(N), Kp = oz_kp(K);
    ar.take<uint8_t>((size_t)OZ_SL * NP * Kp);
    ar.take<int32_t>(NP);
    ar.take<double>(NP);
    ar.take<long long>(NP);
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
    double *chi = ar.take<double>(NP);
    long long *clo = ar.take<long long>(NP);
    oz_bprep_kernel<<<NP, 256, 0, st>>>(W, K, N, NP, Kp, img, colE, chi, clo);
    TPO_LAUNCH_CHECK();
    OzArgs a{};
    a.A = A; a.lda = lda;
    a.n = n; a.ldo = ldo; a.K = K; a.N = N; a.NP = NP; a.Kp = Kp;
    a.ntiles = cdiv(n, OZ_M);
    a.rowE = rowE; a.colE = colE; a.chi = chi; a.clo = clo;
    a.Bimg = img; a.rs = rs; a.out = out;
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
    // measured faster than the fp64 DMMA path for N > 32 only (large: 1.37 vs 2.42 ms; medium,
    // N = 20: 0.62 vs 0.61 ms)
    p.oz = oz_enabled() && n > 0 && D % 4 == 0 && k > 32 && oz_aw_supported(D, k) &&
           (reinterpret_cast<uintptr_t>(Rp) & 15) == 0;
    p.rowE = rowE;
    if (p.oz) oz_rowexp(Rp, D, n, (int)D, p.rowE, st);
    return p;
}
RhPlan rh_plan(const float *Rp, int64_t n, int64_t D, int k, Arena &ar, cudaStream_t st) {
    return rh_plan_at(ar.take<int32_t>(std::max<int64_t>(n, 1)), Rp, n, D, k, st);
}
RhPlan rh_plan_pre(const int32_t *rowE, const float *Rp, int64_t n, int64_t D, int k, Arena &ar, cudaStream_t st) {
    if (!rowE) return rh_plan(Rp, n, D, k, ar, st);
    RhPlan p;
    p.oz = oz_enabled() && n > 0 && D % 4 == 0 && k > 32 && oz_aw_supported(D, k) &&
           (reinterpret_cast<uintptr_t>(Rp) & 15) == 0;
    p.rowE = const_cast<int32_t *>(rowE);
    return p;
}
size_t rh_plan_ws(int64_t n) { return align_up(sizeof(int32_t) * (size_t)std::max<int64_t>(n, 1) + 1); }
size_t rh_apply_ws(int64_t D, int k) { return (k > 32 && oz_aw_supported(D, k)) ? oz_aw_ws(D, k) : 0; }

void rh_apply(const RhPlan &p, const float *Rp, const float *dinv, const double *H, int64_t n, int64_t D, int k,
              double *RH, Arena &ar, cudaStream_t st) {
    if (n == 0) return;
    if (p.oz) oz_aw_f64(Rp, D, dinv, p.rowE, H, n, (int)D, k, RH, k, ar, st);
    else tsgemm_AW_f64(Rp, D, dinv, H, n, D, k, RH, k, st);
}

// ---------------------------------------------------------------------------------------------
// Alg. 3 assignment on the integer tensor cores (Eq. ell-ast; R13 certified):
//      l*_i = argmax_l sum_a Ups[i,a] Phi[a,l]
// Ups and Phi are nonnegative, so both are cut into UNSIGNED byte digits without a bias: row i of
// Ups -> A'_ia = floor(Ups_ia 2^(48-E_i)) (6 bytes; computed ONCE per Alg. 3, Ups is fixed while
// Phi changes), column l of Phi -> B'_al = floor(Phi_al 2^(48-E_l)) (per iteration).  The kept
// digit pairs (p + q <= 5) give c_il = 2^(E_i+E_l-56) [acc_0..2 2^24 + acc_3..5] <= the exact
// score, below it by at most U_il = k 2^(E_i+E_l) (2^-45 + k 2^-52) (dropped pairs, truncation,
// and the slack that keeps the certified argmax equal to R13's sequential-fma argmax).  A row's
// argmax is accepted when its best computed score exceeds every other c_il + U_il; otherwise the
// row is rescored with R13's sequential fma from Ups and Phi (rare).  Labels are the oracle's.
//   warp 0     Phi's digit image once (bulk copy, resident), then per row tile of 128 its precomputed
//              Ups digit planes (one bulk copy) into a 3-slot ring
//   warp 1     MMA issuer: per 32-wide K chunk the 8 N-concatenated kind::i8 MMAs (u8 x u8 -> s32)
//   warps 2-17 epilogue: 4 per TMEM lane quarter (a quarter of the columns each), per row a running
//              certified top-2, merged in column order
// ---------------------------------------------------------------------------------------------
namespace {

constexpr int OA_NBUF = 3;
constexpr int OA_EPI = 16;                // 4 per TMEM lane quarter (column quarters)
constexpr int OA_THREADS = 32 * (2 + OA_EPI);

struct OaArgs {
    int64_t n;
    int k, NP, Kp;
    int64_t ntiles;
    const uint8_t *Ud;       // [ntiles][Kp/32][6][4 KB] digit planes of Ups
    const int32_t *rowE;     // [n]
    const uint8_t *Bimg;     // [6][NP x Kp] digit image of Phi
    const int32_t *colE;     // [NP]
    const double *U, *Phi;   // fp64 (R13 rescoring)
    int32_t *labels, *changed;
    const int32_t *done;
};

// (once per Alg. 3) row exponents E_i and the Ups digit planes in the MMA layout.  Half a warp
// per row (Kp <= 64: 16 lanes x 4 columns), two rows per warp; coalesced 32-byte reads.
__global__ void oa_prep_kernel(const double *__restrict__ U, int64_t n, int k, int Kp, int32_t *__restrict__ rowE,
                               uint8_t *__restrict__ Ud) {
    const int64_t row = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * 2 + ((threadIdx.x >> 4) & 1);
    const int hl = threadIdx.x & 15;
    const int64_t ntiles = (n + OZ_M - 1) / OZ_M;
    if (row >= ntiles * OZ_M) return;                    // uniform per half warp
    const int a0 = 4 * hl;
    double u[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) u[e] = (row < n && a0 + e < k) ? U[row * k + a0 + e] : 0.0;
    double m = fmax(fmax(u[0], u[1]), fmax(u[2], u[3]));
    for (int o = 8; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    int E = 0;
    if (m > 0.0) frexp(m, &E);
    if (hl == 0 && row < n) rowE[row] = E;
    if (a0 >= Kp) return;
    const double scale = pow2d(48 - E);
    uint32_t L[4], H[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const double z = __fma_rz(u[e], scale, 4503599627370496.0);    // 2^52 + floor(Ups 2^(48-E))
        const unsigned long long zb = (unsigned long long)__double_as_longlong(z);
        L[e] = (uint32_t)zb;
        H[e] = (uint32_t)(zb >> 32) & 0xFFFFu;
    }
    uint32_t w[OZ_SL];
    const uint32_t t0 = __byte_perm(L[0], L[1], 0x5140), t1 = __byte_perm(L[2], L[3], 0x5140);
    const uint32_t u0 = __byte_perm(L[0], L[1], 0x7362), u1 = __byte_perm(L[2], L[3], 0x7362);
    w[5] = __byte_perm(t0, t1, 0x5410);
    w[4] = __byte_perm(t0, t1, 0x7632);
    w[3] = __byte_perm(u0, u1, 0x5410);
    w[2] = __byte_perm(u0, u1, 0x7632);
    const uint32_t h0 = __byte_perm(H[0], H[1], 0x5140), h1 = __byte_perm(H[2], H[3], 0x5140);
    w[1] = __byte_perm(h0, h1, 0x5410);
    w[0] = __byte_perm(h0, h1, 0x7632);
    const int64_t t = row / OZ_M;
    const int r = (int)(row - t * OZ_M), c = a0 / OZ_KC, kb = a0 % OZ_KC;
    uint8_t *base = Ud + ((t * (Kp / OZ_KC) + c) * OZ_SL) * (int64_t)OZ_PLANE;
    const uint32_t off = (uint32_t)((r >> 3) * 256 + (kb >> 4) * 128 + (r & 7) * 16 + (kb & 15));
#pragma unroll
    for (int p = 0; p < OZ_SL; ++p) *reinterpret_cast<uint32_t *>(base + p * OZ_PLANE + off) = w[p];
}

// Phi (k x k fp64, Phi[a][l]) -> unsigned digit image [6][NP x Kp] (row l = column of Phi), E_l
__global__ void oa_phidigits_kernel(const double *__restrict__ Phi, int k, int NP, int Kp, uint8_t *__restrict__ img,
                                    int32_t *__restrict__ colE, const int32_t *__restrict__ done) {
    if (*done) return;
    const int l = blockIdx.x;
    __shared__ double red[32];
    double m = 0.0;
    if (l < k)
        for (int a = threadIdx.x; a < k; a += blockDim.x) m = fmax(m, Phi[(int64_t)a * k + l]);
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = fmax(v, red[w]);
        red[0] = v;
    }
    __syncthreads();
    int E = 0;
    if (red[0] > 0.0) frexp(red[0], &E);
    const double scale = ldexp(1.0, 48 - E);
    for (int a = threadIdx.x; a < Kp; a += blockDim.x) {
        const double v = (l < k && a < k) ? Phi[(int64_t)a * k + l] : 0.0;
        const unsigned long long f = (unsigned long long)(v * scale);     // floor (v >= 0), < 2^48
        const int64_t off = (int64_t)(l >> 3) * (8 * Kp) + (a >> 4) * 128 + (l & 7) * 16 + (a & 15);
#pragma unroll
        for (int q = 0; q < OZ_SL; ++q) img[(int64_t)q * NP * Kp + off] = (uint8_t)((f >> (8 * (OZ_SL - 1 - q))) & 255);
    }
    if (threadIdx.x == 0) colE[l] = E;
}

template <int NP>
__global__ void __launch_bounds__(OA_THREADS, 1) oa_assign_kernel(OaArgs g) {
    if (*g.done) return;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    const int nkc = g.Kp / OZ_KC;
    const uint32_t bbytes = (uint32_t)OZ_SL * NP * g.Kp;
    const uint32_t tbytes = (uint32_t)nkc * OZ_SBUF;                 // one tile's Ups planes
    const uint32_t ring_off = (bbytes + 127) & ~127u;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + ring_off + OA_NBUF * tbytes);
    uint64_t *bfull = bars, *afull = bars + 1, *afree = afull + OA_NBUF, *tfull = afree + OA_NBUF, *tempty = tfull + 1;
    double *sh_c1 = reinterpret_cast<double *>(tempty + 1);         // [4 column quarters][128 rows]
    double *sh_cu = sh_c1 + 4 * OZ_M, *sh_w2 = sh_cu + 4 * OZ_M;
    int32_t *sh_i1 = reinterpret_cast<int32_t *>(sh_w2 + 4 * OZ_M);
    int32_t *sh_colE = sh_i1 + 4 * OZ_M;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sh_colE + NP);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr uint32_t TMEM_COLS = (OZ_NACC * NP <= 128) ? 128 : (OZ_NACC * NP <= 256 ? 256 : 512);
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(bfull), 1);
        for (int b = 0; b < OA_NBUF; ++b) {
            mbar_init(smem_u32(&afull[b]), 1);
            mbar_init(smem_u32(&afree[b]), 1);
        }
        mbar_init(smem_u32(tfull), 1);
        mbar_init(smem_u32(tempty), OA_EPI);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
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
        if (lane == 0) {
            mbar_expect_tx(smem_u32(bfull), bbytes);
            for (uint32_t o = 0; o < bbytes; o += 32768)
                bulk_g2s(smem_u32(smem) + o, g.Bimg + o, std::min<uint32_t>(32768, bbytes - o), smem_u32(bfull));
            int j = 0;
            for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x, ++j) {
                const int b = j % OA_NBUF;
                if (j >= OA_NBUF) mbar_wait(smem_u32(&afree[b]), (uint32_t)(((j / OA_NBUF) - 1) & 1));
                mbar_expect_tx(smem_u32(&afull[b]), tbytes);
                bulk_g2s(smem_u32(smem + ring_off + b * tbytes), g.Ud + t * (int64_t)tbytes, tbytes, smem_u32(&afull[b]));
            }
        }
    } else if (warp == 1) {
        mbar_wait(smem_u32(bfull), 0);
        const uint32_t bres = smem_u32(smem);
        const uint32_t sbo_b = 8u * (uint32_t)g.Kp;
        int j = 0;
        for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x, ++j) {
            const int b = j % OA_NBUF;
            if (j > 0) mbar_wait(smem_u32(tempty), (uint32_t)((j - 1) & 1));
            mbar_wait(smem_u32(&afull[b]), (uint32_t)((j / OA_NBUF) & 1));
            fence_after();
            if (lane == 0) {
                for (int c = 0; c < nkc; ++c) {
                    const uint32_t abase = smem_u32(smem + ring_off + b * tbytes + c * OZ_SBUF);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        constexpr int P[8] = {0, 0, 1, 1, 2, 3, 4, 5};
                        constexpr int Q0[8] = {0, 4, 0, 4, 0, 0, 0, 0};
                        constexpr int NQ[8] = {4, 2, 4, 1, 4, 3, 2, 1};
                        const uint64_t da = desc_kmajor_noswz(abase + P[u] * OZ_PLANE, 128, 256);
                        const uint64_t db = desc_kmajor_noswz(
                            bres + (uint32_t)Q0[u] * NP * g.Kp + (uint32_t)c * (OZ_KC * 8), 128, sbo_b);
                        const uint32_t acc = (c > 0 || u >= 2) ? 1u : 0u;
                        // u8 x u8 (both digit sets unsigned)
                        const uint32_t idesc = (2u << 4) | (0u << 7) | (0u << 10) |
                                               ((uint32_t)((NQ[u] * NP) >> 3) << 17) | ((uint32_t)(OZ_M >> 4) << 24);
                        mma_i8(tmem_base + (uint32_t)((P[u] + Q0[u]) * NP), da, db, idesc, acc);
                    }
                }
                mma_commit(smem_u32(&afree[b]));
                mma_commit(smem_u32(tfull));
            }
            __syncwarp();
        }
    } else {
        // 4 warps per lane quarter, NP / 4 columns each; per row a local certified top-2, merged
        // in column order by the quarter's first warp (ties keep the smallest index)
        const int q4 = warp & 3, ch = (warp - 2) >> 2;
        constexpr int CW = NP / 4;
        const double kf = (double)g.k;
        const double urel = kf * (2.8421709430404007e-14 + kf * 2.220446049250313e-16);   // k (2^-45 + k 2^-52)
        bool changed = false;
        int j = 0;
        for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x, ++j) {
            mbar_wait_sleep(smem_u32(tfull), (uint32_t)(j & 1));
            fence_after();
            const int rloc = 32 * q4 + lane;
            const int64_t row = t * OZ_M + rloc;
            const bool ok = row < g.n;
            const int E = ok ? g.rowE[row] : 0;
            double c1 = -1.0, w2 = -1.0, u1 = 0.0;      // best computed score, max over others of c + U
            int i1 = -1;
#pragma unroll 1
            for (int cb = ch * CW; cb < (ch + 1) * CW; cb += 4) {
                uint32_t v[OZ_NACC][4];
#pragma unroll
                for (int s = 0; s < OZ_NACC; ++s)
                    tmem_ld4_nowait(tmem_base + ((uint32_t)(32 * q4) << 16) + (uint32_t)(s * NP + cb), v[s]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int s = 0; s < OZ_NACC; ++s)
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) asm volatile("" : "+r"(v[s][jj]));
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const int l = cb + jj;
                    if (l >= g.k) break;
                    const long long g0 = (long long)v[0][jj] * 65536 + (long long)v[1][jj] * 256 + (long long)v[2][jj];
                    const long long g1 = (long long)v[3][jj] * 65536 + (long long)v[4][jj] * 256 + (long long)v[5][jj];
                    const double c = fma((double)g0, 16777216.0, (double)g1) * pow2d(E + sh_colE[l] - 56);
                    const double U = urel * pow2d(E + sh_colE[l]);
                    if (i1 < 0 || c > c1) {
                        if (i1 >= 0) w2 = fmax(w2, c1 + u1);
                        c1 = c; i1 = l; u1 = U;
                    } else {
                        w2 = fmax(w2, c + U);
                    }
                }
            }
            fence_before();
            sh_c1[ch * OZ_M + rloc] = c1;
            sh_cu[ch * OZ_M + rloc] = i1 >= 0 ? c1 + u1 : -1.0;
            sh_w2[ch * OZ_M + rloc] = w2;
            sh_i1[ch * OZ_M + rloc] = i1;
            asm volatile("bar.sync %0, 128;" ::"r"(1 + q4) : "memory");     // the quarter's 4 warps
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(tempty));      // TMEM may be refilled; rescoring uses fp64
            if (ch == 0 && ok) {
                double bc = -1.0, bw = -1.0;
                int bi = -1, bq = -1;
                for (int q = 0; q < 4; ++q) {
                    const int qi = sh_i1[q * OZ_M + rloc];
                    if (qi < 0) continue;
                    const double qc = sh_c1[q * OZ_M + rloc];
                    if (bi < 0 || qc > bc) { bc = qc; bi = qi; bq = q; }
                }
                for (int q = 0; q < 4; ++q) {
                    if (sh_i1[q * OZ_M + rloc] < 0) continue;
                    bw = fmax(bw, sh_w2[q * OZ_M + rloc]);
                    if (q != bq) bw = fmax(bw, sh_cu[q * OZ_M + rloc]);
                }
                int lab = bi;
                if (!(bc > bw)) {                               // not certified: R13 sequential fma
                    const double *u = g.U + row * g.k;
                    double best = 0.0;
                    lab = 0;
                    for (int l = 0; l < g.k; ++l) {
                        double sc = 0.0;
                        for (int a = 0; a < g.k; ++a) sc = fma(u[a], g.Phi[(int64_t)a * g.k + l], sc);
                        if (l == 0 || sc > best) { best = sc; lab = l; }
                    }
                }
                if (g.labels[row] != lab) changed = true;
                g.labels[row] = lab;
            }
            asm volatile("bar.sync %0, 128;" ::"r"(1 + q4) : "memory");     // merge read before the next tile's writes
        }
        if (__any_sync(0xffffffffu, changed) && lane == 0) *g.changed = 1;
    }
    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                     : "memory");
    }
}

size_t oa_smem(int NP, int Kp) {
    return 128 + (((size_t)OZ_SL * NP * Kp + 127) & ~size_t(127)) + (size_t)OA_NBUF * (Kp / OZ_KC) * OZ_SBUF + 16 * 8 +
           4 * OZ_M * (3 * sizeof(double) + sizeof(int32_t)) + sizeof(int32_t) * NP + 16;
}

template <int NP>
void oa_launch(const OaArgs &a, cudaStream_t st) {
    const size_t sm = oa_smem(NP, a.Kp);
    TPO_CUDA(cudaFuncSetAttribute(oa_assign_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const int grid = (int)std::min<int64_t>(a.ntiles, sm_count());
    oa_assign_kernel<NP><<<grid, OA_THREADS, sm, st>>>(a);
    TPO_LAUNCH_CHECK();
}

}  // namespace

// k in (32, 64]: the Ups digit planes fit (3 tiles of 6 x 128 x Kp bytes + Phi's image)
bool oz_assign_supported(int k) { return oz_enabled() && k > 32 && k <= 64 && oa_smem(oz_np(k), oz_kp(k)) <= 227 * 1024 - 256; }

size_t oz_assign_ws(int64_t n, int k) {
    const int NP = oz_np(k), Kp = oz_kp(k);
    const int64_t ntiles = cdiv(std::max<int64_t>(n, 1), OZ_M);
    Arena ar(nullptr, 0);
    ar.take<uint8_t>((size_t)ntiles * (Kp / OZ_KC) * OZ_SBUF);
    ar.take<int32_t>(std::max<int64_t>(n, 1));
    ar.take<uint8_t>((size_t)OZ_SL * NP * Kp);
    ar.take<int32_t>(NP);
    return ar.off + 256;
}

OzAssign oz_assign_prepare(const double *U, int64_t n, int k, Arena &ar, cudaStream_t st) {
    OzAssign p;
    p.n = n;
    p.k = k;
    p.NP = oz_np(k);
    p.Kp = oz_kp(k);
    const int64_t ntiles = cdiv(std::max<int64_t>(n, 1), OZ_M);
    p.Ud = ar.take<uint8_t>((size_t)ntiles * (p.Kp / OZ_KC) * OZ_SBUF);
    p.rowE = ar.take<int32_t>(std::max<int64_t>(n, 1));
    p.Bimg = ar.take<uint8_t>((size_t)OZ_SL * p.NP * p.Kp);
    p.colE = ar.take<int32_t>(p.NP);
    if (n == 0) return p;
    const int64_t rows = ntiles * OZ_M;
    oa_prep_kernel<<<cdiv(rows * 16, 256), 256, 0, st>>>(U, n, k, p.Kp, p.rowE, p.Ud);
    TPO_LAUNCH_CHECK();
    return p;
}

void oz_assign(const OzAssign &p, const double *U, const double *Phi, int32_t *labels, int32_t *changed,
               const int32_t *done, cudaStream_t st) {
    if (p.n == 0) return;
    oa_phidigits_kernel<<<p.NP, 128, 0, st>>>(Phi, p.k, p.NP, p.Kp, p.Bimg, p.colE, done);
    TPO_LAUNCH_CHECK();
    OaArgs a{};
    a.n = p.n; a.k = p.k; a.NP = p.NP; a.Kp = p.Kp;
    a.ntiles = cdiv(p.n, OZ_M);
    a.Ud = p.Ud; a.rowE = p.rowE; a.Bimg = p.Bimg; a.colE = p.colE;
    a.U = U; a.Phi = Phi; a.labels = labels; a.changed = changed; a.done = done;
    switch (p.NP) {
        case 48: oa_launch<48>(a, st); break;
        default: oa_launch<64>(a, st); break;
    }
}


// ---------------------------------------------------------------------------------------------
// Alg. 2's R^T Ups = R'^T (dinv . Ups) (D x k, reduced over the n rows; Eq. update-Q)
// fp64-accurate on the integer tensor cores (R16), 32 < k <= 64:
//   A = R'^T (M = 128 features per tile, K = rows): feature j scaled by 2^(46 - EA_j) (EA_j: the
//       smallest e with max_i |R'_ij| < 2^e), F = round(R' 2^(46-EA)) (|F| <= 2^46; nearest, so the
//       truncation is unbiased) cut into 6 balanced signed byte digits.  One fp64 fma gives V = F +
//       beta (beta = 0x808080808080, so V in [0, 2^48)) in the low 48 bits of 2^52 + beta + R' 2^(46-EA);
//       the digits are V's bytes xor 0x80 (byte b stands for b - 128).
//   B = dinv . Ups (N = k padded to 16, K = rows; Ups >= 0): column l scaled by 2^(47 - EB_l), G =
//       round(dinv_i Ups_il 2^(47-EB_l)) <= 2^47 (one fma rounds the exact product), 6 unsigned digits.
//   The 26 kept digit pairs (p + q <= 6: a sum over K = n rows needs one digit weight more than
//   the row products of oz_aw) are summed exactly in 7 int32 TMEM accumulators over one item of
//   <= 8192 rows (per 32-row chunk |acc_s| grows by <= 6 x 32 x 128 x 255 < 2^23), then flushed as
//   the exact int64 pair g0 = acc0 2^16 + acc1 2^8 + acc2, g1 = (acc3 2^16 + acc4 2^8 + acc5) 2^8
//   + acc6 per (feature, column, item).  oz_rtu_reduce adds the items in 128-bit integers (exact,
//   so the result does not depend on the order) and rounds once:
//        RtU_jl = 2^(EA_j + EB_l - 61) sum_items (g0 2^32 + g1).
//   Error per row <~ 2^-52 2^EA_j 2^EB_l (dropped pairs) + the roundings 2^-47 2^EA_j (dinv_i Ups_il)
//   + 2^-48 2^EB_l |R'_ij| (both unbiased): the class of the fp64 products' own rounding
//   (tests/test_gpu_oz.py).
// Kernel (persistent, 704 threads, ~214 KB shared memory), items = (row block, feature tile):
//   warp 0       producer: per 32-row chunk the fp32 R' tile (4 TMA boxes of 32 x 32, SWIZZLE_128B),
//                the Ups rows (bulk copy) and dinv (bulk copy) into a 4-stage ring
//   warp 1       MMA issuer: 9 N-concatenated tcgen05.mma kind::i8 (s8 x u8 -> s32) per chunk
//   warps 2-9    A slicers: one feature x 16 rows per thread (conflict-free swizzled reads,
//                16-byte core-matrix row stores)
//   warps 10-13  B slicers: one column x 16 rows per thread
//   warps 14-21  epilogue: TMEM -> exact int64 partials of the item
// ---------------------------------------------------------------------------------------------
namespace {

constexpr int RT_ASL = 8, RT_BSL = 4, RT_EPI = 8;
constexpr int RT_THREADS = 32 * (2 + RT_ASL + RT_BSL + RT_EPI);
constexpr int RT_STG = 4;                          // input ring depth covers the load latency
constexpr int RT_ITEM_MAX = 8192;                      // rows per item (int32 accumulators)
constexpr int RT_NACC = 7;                             // acc_0 .. acc_6 (p + q <= 6)
constexpr uint32_t RT_A_BYTES = 4 * 4096;              // 32 rows x 128 fp32 (4 swizzled boxes)

struct RtArgs {
    int64_t n;
    int D, k, NP, nD;
    int64_t RB, nitems;
    const double *U;
    const float *dinv;
    const uint32_t *featmax;                           // [D] bits of max_i |R'_ij|
    const unsigned long long *colmax;                  // [k] bits of max_i dinv_i Ups_il
    long long *g0, *g1;                                // [nitems][NP][128]
    uint32_t stage, ubytes;                            // ring stage stride (A + Ups + dinv), Ups region
};

// stage = R' tile (16 KB) + 32 Ups rows + 32 dinv, 1024-aligned (the TMA boxes use SWIZZLE_128B)
inline uint32_t rt_ubytes(int k) { return (uint32_t)((32 * k * 8 + 15) / 16 * 16); }
inline uint32_t rt_stage(int k) { return (RT_A_BYTES + rt_ubytes(k) + 128 + 1023) / 1024 * 1024; }

__device__ __forceinline__ int exp_f32bits(uint32_t b) {       // smallest e with m < 2^e (0 for m = 0)
    const float m = __uint_as_float(b);
    int e = 0;
    if (m > 0.f) frexpf(m, &e);
    return e;
}
__device__ __forceinline__ int exp_f64bits(unsigned long long b) {
    const double m = __longlong_as_double((long long)b);
    int e = 0;
    if (m > 0.0) frexp(m, &e);
    return max(e, -900);                                // tiny / zero columns: any scale works
}

// bytes 0..5 of the 48-bit integers in the low mantissa bits of z[0..3] -> w[p] = byte 5 - p of
// each (byte e = element e)
__device__ __forceinline__ void pack6(const double (&z)[4], uint32_t (&w)[OZ_SL]) {
    uint32_t L[4], H[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const unsigned long long zb = (unsigned long long)__double_as_longlong(z[e]);
        L[e] = (uint32_t)zb;
        H[e] = (uint32_t)(zb >> 32) & 0xFFFFu;
    }
    const uint32_t t0 = __byte_perm(L[0], L[1], 0x5140), t1 = __byte_perm(L[2], L[3], 0x5140);
    const uint32_t u0 = __byte_perm(L[0], L[1], 0x7362), u1 = __byte_perm(L[2], L[3], 0x7362);
    w[5] = __byte_perm(t0, t1, 0x5410);
    w[4] = __byte_perm(t0, t1, 0x7632);
    w[3] = __byte_perm(u0, u1, 0x5410);
    w[2] = __byte_perm(u0, u1, 0x7632);
    const uint32_t h0 = __byte_perm(H[0], H[1], 0x5140), h1 = __byte_perm(H[2], H[3], 0x5140);
    w[1] = __byte_perm(h0, h1, 0x5410);
    w[0] = __byte_perm(h0, h1, 0x7632);
}

template <int NP, int RT_NBUF>
__global__ void __launch_bounds__(RT_THREADS, 1) oz_rtu_kernel(const __grid_constant__ CUtensorMap mapA, RtArgs g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr uint32_t BPLANE = NP * 32;                           // one B digit plane (NP x 32 bytes)
    constexpr uint32_t BUF = OZ_SL * OZ_PLANE + OZ_SL * BPLANE;    // A planes then B planes
    const uint32_t RT_STAGE = g.stage, RT_U_BYTES = g.ubytes;
    const uint32_t buf_off = RT_STG * RT_STAGE;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + buf_off + RT_NBUF * BUF);
    uint64_t *afull = bars, *aempty = afull + RT_STG, *sready = aempty + RT_STG, *sfree = sready + RT_NBUF;
    uint64_t *tfull = sfree + RT_NBUF, *tempty = tfull + 1;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr uint32_t TMEM_COLS = (RT_NACC * NP <= 128) ? 128 : (RT_NACC * NP <= 256 ? 256 : 512);
    constexpr int NSL = RT_ASL + RT_BSL;

    if (threadIdx.x == 0) {
        for (int b = 0; b < RT_STG; ++b) {
            mbar_init(smem_u32(&afull[b]), 1);
            mbar_init(smem_u32(&aempty[b]), NSL);
        }
        for (int b = 0; b < RT_NBUF; ++b) {
            mbar_init(smem_u32(&sready[b]), NSL);
            mbar_init(smem_u32(&sfree[b]), 1);
        }
        mbar_init(smem_u32(tfull), 1);
        mbar_init(smem_u32(tempty), RT_EPI);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    }
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
            int64_t gc = 0;
            for (int64_t w = blockIdx.x; w < g.nitems; w += gridDim.x) {
                const int64_t rb = w / g.nD;
                const int t = (int)(w - rb * g.nD);
                const int64_t row0 = rb * g.RB, rows = min(g.RB, g.n - row0);
                const int nch = (int)((rows + 31) / 32);
                for (int c = 0; c < nch; ++c, ++gc) {
                    const int s = (int)(gc % RT_STG);
                    if (gc >= RT_STG) mbar_wait(smem_u32(&aempty[s]), (uint32_t)(((gc / RT_STG) - 1) & 1));
                    const int64_t r0 = row0 + 32 * c;
                    const int nv = (int)(g.n - r0 < 32 ? g.n - r0 : 32);
                    uint8_t *st = smem + s * RT_STAGE;
                    double *su = reinterpret_cast<double *>(st + RT_A_BYTES);
                    float *sd = reinterpret_cast<float *>(st + RT_A_BYTES + RT_U_BYTES);
                    const uint32_t ub = (uint32_t)nv * g.k * 8, ubulk = ub & ~15u;
                    const uint32_t db = (uint32_t)nv * 4, dbulk = db & ~15u;
                    // tails that are not 16-byte multiples: plain copies before the arrive (release)
                    if (ub != ubulk) su[ubulk / 8] = g.U[r0 * g.k + ubulk / 8];
                    for (uint32_t o = dbulk; o < db; o += 4) sd[o / 4] = g.dinv[r0 + o / 4];
                    const uint32_t full = smem_u32(&afull[s]);
                    mbar_expect_tx(full, RT_A_BYTES + ubulk + dbulk);
#pragma unroll
                    for (int bx = 0; bx < 4; ++bx) tma_load_2d(smem_u32(st + bx * 4096), &mapA, full, t * 128 + 32 * bx, (int)r0);
                    if (ubulk) bulk_g2s(smem_u32(su), g.U + r0 * g.k, ubulk, full);
                    if (dbulk) bulk_g2s(smem_u32(sd), g.dinv + r0, dbulk, full);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        int64_t gc = 0;
        int i = 0;
        for (int64_t w = blockIdx.x; w < g.nitems; w += gridDim.x, ++i) {
            const int64_t rb = w / g.nD;
            const int64_t row0 = rb * g.RB, rows = min(g.RB, g.n - row0);
            const int nch = (int)((rows + 31) / 32);
            if (i > 0) mbar_wait(smem_u32(tempty), (uint32_t)((i - 1) & 1));
            fence_after();
            for (int c = 0; c < nch; ++c, ++gc) {
                const int b = (int)(gc % RT_NBUF);
                mbar_wait(smem_u32(&sready[b]), (uint32_t)((gc / RT_NBUF) & 1));
                fence_after();
                if (lane == 0) {
                    const uint32_t abase = smem_u32(smem + buf_off + b * BUF);
                    const uint32_t bbase = abase + OZ_SL * OZ_PLANE;
                    // the 26 pairs p + q <= 6 in 9 MMAs; the first three initialise acc_0..3,
                    // acc_4..5 and acc_6 (an MMA's accumulate flag covers all of its N columns)
#pragma unroll
                    for (int u = 0; u < 9; ++u) {
                        constexpr int P[9] = {0, 0, 2, 1, 1, 2, 3, 4, 5};
                        constexpr int Q0[9] = {0, 4, 4, 0, 4, 0, 0, 0, 0};
                        constexpr int NQ[9] = {4, 2, 1, 4, 2, 4, 4, 3, 2};
                        const uint64_t da = desc_kmajor_noswz(abase + P[u] * OZ_PLANE, 128, 256);
                        const uint64_t dbd = desc_kmajor_noswz(bbase + (uint32_t)Q0[u] * BPLANE, 128, 256);
                        const uint32_t acc = (c > 0 || u >= 3) ? 1u : 0u;
                        // s8 (R' digits) x u8 (dinv.Ups digits) -> s32
                        const uint32_t idesc = (2u << 4) | (1u << 7) | (0u << 10) |
                                               ((uint32_t)((NQ[u] * NP) >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
                        mma_i8(tmem_base + (uint32_t)((P[u] + Q0[u]) * NP), da, dbd, idesc, acc);
                    }
                    mma_commit(smem_u32(&sfree[b]));
                    if (c == nch - 1) mma_commit(smem_u32(tfull));
                }
                __syncwarp();
            }
        }
    } else if (warp < 2 + NSL) {
        // ---------------- slicers ----------------
        const bool is_a = warp < 2 + RT_ASL;
        const int sw = is_a ? warp - 2 : warp - 2 - RT_ASL;
        const int bx = sw & 3, h = is_a ? (sw >> 2) : (sw >> 1), ch = sw & 1;
        const int l = 32 * ch + lane;                              // B: column
        const bool lok = !is_a && l < g.k;
        double sB = 0.0;
        if (lok) sB = pow2d(47 - exp_f64bits(g.colmax[l]));
        int64_t gc = 0;
        for (int64_t w = blockIdx.x; w < g.nitems; w += gridDim.x) {
            const int64_t rb = w / g.nD;
            const int t = (int)(w - rb * g.nD);
            const int64_t row0 = rb * g.RB, rows = min(g.RB, g.n - row0);
            const int nch = (int)((rows + 31) / 32);
            const int f = t * 128 + 32 * bx + lane;                // A: feature
            const double sA = pow2d(46 - (is_a && f < g.D ? exp_f32bits(g.featmax[f]) : 0));
            for (int c = 0; c < nch; ++c, ++gc) {
                const int s = (int)(gc % RT_STG);
                mbar_wait(smem_u32(&afull[s]), (uint32_t)((gc / RT_STG) & 1));
                const uint8_t *st = smem + s * RT_STAGE;
                uint32_t wd[4][OZ_SL];
                if (is_a) {
                    const uint8_t *box = st + bx * 4096;
                    float x[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        const int r = 16 * h + u;
                        x[u] = *reinterpret_cast<const float *>(box + r * 128 + ((((lane >> 2) ^ (r & 7))) << 4) + (lane & 3) * 4);
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        double z[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) z[e] = __fma_rn((double)x[4 * q + e], sA, 4644889027444864.0);   // 2^52 + beta
                        pack6(z, wd[q]);
#pragma unroll
                        for (int p = 0; p < OZ_SL; ++p) wd[q][p] ^= 0x80808080u;
                    }
                } else {
                    const double *su = reinterpret_cast<const double *>(st + RT_A_BYTES);
                    const float *sd = reinterpret_cast<const float *>(st + RT_A_BYTES + RT_U_BYTES);
                    const int64_t r0 = row0 + 32 * c;
                    const int nv = (int)(g.n - r0 < 32 ? g.n - r0 : 32);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        double z[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int r = 16 * h + 4 * q + e;
                            const bool ok = lok && r < nv;
                            const double v = ok ? su[r * g.k + l] : 0.0;
                            const double sc = ok ? (double)sd[r] * sB : 0.0;
                            z[e] = __fma_rn(v, sc, 4503599627370496.0);                                  // 2^52 + G
                        }
                        pack6(z, wd[q]);
                    }
                }
                uint32_t dep = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) dep |= wd[q][0] | wd[q][OZ_SL - 1];
                dep = __reduce_or_sync(0xffffffffu, dep);
                if (lane == 0)
                    asm volatile("{\n.reg .pred q;\nsetp.ne.u32 q, %1, 0xdeadbeef;\n@q mbarrier.arrive.shared::cta.b64 _, [%0];\n}\n" ::"r"(
                                     smem_u32(&aempty[s])),
                                 "r"(dep)
                                 : "memory");
                const int b = (int)(gc % RT_NBUF);
                if (gc >= RT_NBUF) mbar_wait(smem_u32(&sfree[b]), (uint32_t)(((gc / RT_NBUF) - 1) & 1));
                uint8_t *sb = smem + buf_off + b * BUF;
                if (is_a) {
                    const int m = 32 * bx + lane;
                    const uint32_t off = (uint32_t)((m >> 3) * 256 + h * 128 + (m & 7) * 16);
#pragma unroll
                    for (int p = 0; p < OZ_SL; ++p)
                        *reinterpret_cast<uint4 *>(sb + p * OZ_PLANE + off) = make_uint4(wd[0][p], wd[1][p], wd[2][p], wd[3][p]);
                } else if (l < NP) {
                    const uint32_t off = (uint32_t)((l >> 3) * 256 + h * 128 + (l & 7) * 16);
#pragma unroll
                    for (int p = 0; p < OZ_SL; ++p)
                        *reinterpret_cast<uint4 *>(sb + OZ_SL * OZ_PLANE + p * BPLANE + off) =
                            make_uint4(wd[0][p], wd[1][p], wd[2][p], wd[3][p]);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&sready[b]));
            }
        }
    } else {
        // ---------------- epilogue: item partials (exact int64) ----------------
        const int e = warp - 2 - NSL;
        const int q4 = warp & 3, chh = e >> 2;
        constexpr int HALF = NP / 2;
        int i = 0;
        for (int64_t w = blockIdx.x; w < g.nitems; w += gridDim.x, ++i) {
            mbar_wait_sleep(smem_u32(tfull), (uint32_t)(i & 1));
            fence_after();
            const int jj = 32 * q4 + lane;
#pragma unroll 1
            for (int cb = chh * HALF; cb < (chh + 1) * HALF; cb += 4) {
                uint32_t v[RT_NACC][4];
#pragma unroll
                for (int s = 0; s < RT_NACC; ++s)
                    tmem_ld4_nowait(tmem_base + ((uint32_t)(32 * q4) << 16) + (uint32_t)(s * NP + cb), v[s]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const long long a0 = (long long)(int32_t)v[0][j] * 65536 + (long long)(int32_t)v[1][j] * 256 +
                                         (long long)(int32_t)v[2][j];
                    const long long a1 = ((long long)(int32_t)v[3][j] * 65536 + (long long)(int32_t)v[4][j] * 256 +
                                          (long long)(int32_t)v[5][j]) * 256 + (long long)(int32_t)v[6][j];
                    const int64_t o = (w * NP + cb + j) * 128 + jj;
                    g.g0[o] = a0;
                    g.g1[o] = a1;
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

// bits of max_i |A_ij| per column (atomicMax on the bit patterns of nonnegative floats: order free)
__global__ void oz_featmax_kernel(const float *__restrict__ A, int64_t n, int D, int64_t rows_per,
                                  uint32_t *__restrict__ mx) {
    const int64_t r0 = blockIdx.x * rows_per, r1 = min(n, r0 + rows_per);
    for (int c = threadIdx.x; c < D; c += blockDim.x) {
        float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f;
        int64_t r = r0;
        for (; r + 4 <= r1; r += 4) {
            m0 = fmaxf(m0, fabsf(A[r * D + c]));
            m1 = fmaxf(m1, fabsf(A[(r + 1) * D + c]));
            m2 = fmaxf(m2, fabsf(A[(r + 2) * D + c]));
            m3 = fmaxf(m3, fabsf(A[(r + 3) * D + c]));
        }
        for (; r < r1; ++r) m0 = fmaxf(m0, fabsf(A[r * D + c]));
        atomicMax(&mx[c], __float_as_uint(fmaxf(fmaxf(m0, m1), fmaxf(m2, m3))));
    }
}

// bits of max_i fl(dinv_i U_il) per column (U >= 0, k <= 64): a warp per row (lane: columns l and
// l + 32, coalesced), 4 rows in flight per warp, block maxima combined by atomicMax (order free)
__global__ void __launch_bounds__(256) oz_colmax_kernel(const double *__restrict__ U, const float *__restrict__ dinv,
                                                        int64_t n, int k, int64_t rows_per,
                                                        unsigned long long *__restrict__ mx) {
    __shared__ double sm[8][64];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t r0 = blockIdx.x * rows_per, r1 = min(n, r0 + rows_per);
    const bool v0 = lane < k, v1 = lane + 32 < k;
    double m0 = 0.0, m1 = 0.0;
    int64_t r = r0 + w;
    for (; r + 24 < r1; r += 32) {
        double a[4], b[4];
        float dv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t rr = r + 8 * u;
            dv[u] = dinv[rr];
            a[u] = v0 ? U[rr * k + lane] : 0.0;
            b[u] = v1 ? U[rr * k + lane + 32] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            m0 = fmax(m0, (double)dv[u] * a[u]);
            m1 = fmax(m1, (double)dv[u] * b[u]);
        }
    }
    for (; r < r1; r += 8) {
        const double dv = (double)dinv[r];
        if (v0) m0 = fmax(m0, dv * U[r * k + lane]);
        if (v1) m1 = fmax(m1, dv * U[r * k + lane + 32]);
    }
    sm[w][lane] = m0;
    sm[w][lane + 32] = m1;
    __syncthreads();
    if (threadIdx.x < 64 && (int)threadIdx.x < k) {
        double m = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) m = fmax(m, sm[i][threadIdx.x]);
        atomicMax(&mx[threadIdx.x], (unsigned long long)__double_as_longlong(m));
    }
}

// one block per (feature tile t, column l): 128 features x 8 groups of row blocks, exact 128-bit
// sums (the order does not matter), one rounding
__global__ void __launch_bounds__(1024) oz_rtu_reduce_kernel(const long long *__restrict__ g0,
                                                             const long long *__restrict__ g1, int D, int k, int NP,
                                                             int nD, int64_t nrb, const uint32_t *__restrict__ featmax,
                                                             const unsigned long long *__restrict__ colmax,
                                                             double *__restrict__ out) {
    __shared__ __int128 sh[8][128];
    const int t = blockIdx.x, l = blockIdx.y;
    const int jj = threadIdx.x & 127, grp = threadIdx.x >> 7;
    __int128 T = 0;                                     // sum (g0 2^32 + g1): < 2^88, exact
    for (int64_t rb = grp; rb < nrb; rb += 8) {
        const int64_t o = ((rb * nD + t) * NP + l) * 128 + jj;
        T += ((__int128)g0[o] << 32) + (__int128)g1[o];
    }
    sh[grp][jj] = T;
    __syncthreads();
    const int j = t * 128 + jj;
    if (grp != 0 || j >= D) return;
#pragma unroll
    for (int i = 1; i < 8; ++i) T += sh[i][jj];
    // T = a 2^40 + b with a (< 2^48), b (< 2^40) exact in fp64: one rounding
    const long long a = (long long)(T >> 40);
    const long long b = (long long)(T - ((__int128)a << 40));
    const double x = (double)a * 1099511627776.0 + (double)b;
    out[(int64_t)j * k + l] = ldexp(x, exp_f32bits(featmax[j]) + exp_f64bits(colmax[l]) - 61);
}

CUtensorMap oz_rtu_map(const float *A, int64_t n, int64_t D) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)D * sizeof(float)};
    const cuuint32_t box[2] = {32, 32};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(A), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(TPO_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

size_t oz_rtu_smem(int NP, int k, int nbuf) {
    return 1024 + RT_STG * (size_t)rt_stage(k) + nbuf * (size_t)(OZ_SL * OZ_PLANE + OZ_SL * NP * 32) + 16 * 8 + 16;
}
// two digit-plane buffers: a third one (it fits beside the 4-stage ring for k <= 50) measured
// slower on large (1.51 vs 1.45 ms)
int rt_nbuf(int NP, int k) { (void)NP; (void)k; return 2; }

struct RtuShape {
    int NP, nD;
    int64_t RB, nrb, nitems;
};

RtuShape rtu_shape(int64_t n, int64_t D, int k) {
    RtuShape s;
    s.NP = oz_np(k);
    s.nD = (int)cdiv(D, 128);
    // row blocks of <= 8192 rows (multiples of 32), their count rounded so that the items fill
    // whole waves of the SMs
    const int64_t sms = sm_count();
    const int64_t base = cdiv(std::max<int64_t>(n, 1), RT_ITEM_MAX);
    const int64_t step = sms / std::gcd<int64_t>(sms, (int64_t)s.nD);
    int64_t nrb = cdiv(base, step) * step;
    s.RB = std::max<int64_t>(32, cdiv(cdiv(std::max<int64_t>(n, 1), nrb), 32) * 32);
    s.nrb = cdiv(std::max<int64_t>(n, 1), s.RB);
    s.nitems = s.nrb * s.nD;
    return s;
}

}  // namespace

bool oz_rtu_supported(int64_t n, int64_t D, int k) {
    return oz_enabled() && n > 0 && k > 32 && k <= 64 && D % 4 == 0 && D >= 4 &&
           oz_rtu_smem(oz_np(k), k, 2) <= 227 * 1024;
}

size_t oz_rtu_ws(int64_t n, int64_t D, int k) {
    if (!(k > 32 && k <= 64)) return 0;
    const RtuShape s = rtu_shape(n, D, k);
    Arena ar(nullptr, 0);
    ar.take<long long>((size_t)s.nitems * s.NP * 128);
    ar.take<long long>((size_t)s.nitems * s.NP * 128);
    ar.take<unsigned long long>(k);
    return ar.off + 256;
}

// bits of max_i |R'_ij| per feature (once per solve: R' is fixed during Alg. 2)
void oz_featmax(const float *Rp, int64_t n, int64_t D, uint32_t *featmax, cudaStream_t st) {
    TPO_CUDA(cudaMemsetAsync(featmax, 0, sizeof(uint32_t) * D, st));
    if (n == 0) return;
    const int64_t blocks = std::min<int64_t>(8 * sm_count(), cdiv(n, 64));
    const int64_t rows_per = cdiv(n, blocks);
    oz_featmax_kernel<<<(unsigned)cdiv(n, rows_per), 256, 0, st>>>(Rp, n, (int)D, rows_per, featmax);
    TPO_LAUNCH_CHECK();
}

// RtU = R'^T (dinv . U) (D x k fp64) on the integer tensor cores; featmax from oz_featmax(R').
void oz_rtu(const float *Rp, int64_t n, int64_t D, const float *dinv, const double *U, int k, const uint32_t *featmax,
            double *RtU, Arena &ar, cudaStream_t st, const unsigned long long *colmax_pre) {
    TPO_REQUIRE(oz_rtu_supported(n, D, k), "oz_rtu: unsupported shape");
    TPO_REQUIRE((reinterpret_cast<uintptr_t>(Rp) & 15) == 0 && (reinterpret_cast<uintptr_t>(U) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(dinv) & 15) == 0,
                "oz_rtu: R', Ups and dinv must be 16-byte aligned");
    const RtuShape s = rtu_shape(n, D, k);
    const size_t mark = ar.off;
    long long *g0 = ar.take<long long>((size_t)s.nitems * s.NP * 128);
    long long *g1 = ar.take<long long>((size_t)s.nitems * s.NP * 128);
    unsigned long long *colmax = ar.take<unsigned long long>(k);
    if (colmax_pre) {
        colmax = const_cast<unsigned long long *>(colmax_pre);
    } else {
        TPO_CUDA(cudaMemsetAsync(colmax, 0, sizeof(unsigned long long) * k, st));
        const int64_t blocks = std::min<int64_t>(8 * sm_count(), cdiv(n, 256));
        const int64_t rows_per = cdiv(n, blocks);
        oz_colmax_kernel<<<(unsigned)cdiv(n, rows_per), 256, 0, st>>>(U, dinv, n, k, rows_per, colmax);
        TPO_LAUNCH_CHECK();
    }
    RtArgs a{};
    a.n = n; a.D = (int)D; a.k = k; a.NP = s.NP; a.nD = s.nD;
    a.RB = s.RB; a.nitems = s.nitems;
    a.U = U; a.dinv = dinv; a.featmax = featmax; a.colmax = colmax; a.g0 = g0; a.g1 = g1;
    a.stage = rt_stage(k); a.ubytes = rt_ubytes(k);
    const CUtensorMap map = oz_rtu_map(Rp, n, D);
    const int nbuf = rt_nbuf(s.NP, k);
    const size_t sm = oz_rtu_smem(s.NP, k, nbuf);
    const int grid = (int)std::min<int64_t>(s.nitems, sm_count());
#define TPO_RTU_LAUNCH(NPV, NB)                                                                                    \
    {                                                                                                              \
        TPO_CUDA(cudaFuncSetAttribute(oz_rtu_kernel<NPV, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
        oz_rtu_kernel<NPV, NB><<<grid, RT_THREADS, sm, st>>>(map, a);                                            \
    }
    if (s.NP == 48) {
        TPO_RTU_LAUNCH(48, 2)
    } else {
        TPO_RTU_LAUNCH(64, 2)
    }
#undef TPO_RTU_LAUNCH
    TPO_LAUNCH_CHECK();
    oz_rtu_reduce_kernel<<<dim3((unsigned)s.nD, (unsigned)k), 1024, 0, st>>>(g0, g1, (int)D, k, s.NP, s.nD, s.nrb,
                                                                             featmax, colmax, RtU);
    TPO_LAUNCH_CHECK();
    ar.off = mark;
}


namespace {
// rowE (row exponents, as oz_rowexp_kernel) and featmax (bits of per-feature max |A|, as
// oz_featmax_kernel) in one pass: a warp per row (16-byte loads, 4 rows in flight), a lane keeps
// the maxima of its 4 NF4 features in registers over all of its rows; block maxima -> atomicMax
// (order free).  D % 4 == 0, D <= 128 NF4.
template <int NF4>
__global__ void __launch_bounds__(256) oz_rstats_kernel(const float *__restrict__ A, int64_t n, int D,
                                                        int32_t *__restrict__ rowE, uint32_t *__restrict__ featmax) {
    __shared__ float sm[8][128 * NF4];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int D4 = D / 4;
    float fm[NF4][4];
#pragma unroll
    for (int i = 0; i < NF4; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) fm[i][e] = 0.f;
    const float4 *A4 = reinterpret_cast<const float4 *>(A);
    const int64_t stride = (int64_t)gridDim.x * 32;
    for (int64_t r0 = (int64_t)blockIdx.x * 32 + w; r0 < n; r0 += stride) {
        float m[4];
        float4 v[4][NF4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t r = r0 + 8 * u;
#pragma unroll
            for (int i = 0; i < NF4; ++i) {
                const int q = lane + 32 * i;
                v[u][i] = (q < D4 && r < n) ? A4[r * D4 + q] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            float mm = 0.f;
#pragma unroll
            for (int i = 0; i < NF4; ++i) {
                const float a0 = fabsf(v[u][i].x), a1 = fabsf(v[u][i].y), a2 = fabsf(v[u][i].z), a3 = fabsf(v[u][i].w);
                fm[i][0] = fmaxf(fm[i][0], a0);
                fm[i][1] = fmaxf(fm[i][1], a1);
                fm[i][2] = fmaxf(fm[i][2], a2);
                fm[i][3] = fmaxf(fm[i][3], a3);
                mm = fmaxf(mm, fmaxf(fmaxf(a0, a1), fmaxf(a2, a3)));
            }
            m[u] = mm;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            for (int o = 16; o; o >>= 1) m[u] = fmaxf(m[u], __shfl_xor_sync(0xffffffffu, m[u], o));
        if (lane < 4) {
            const int64_t r = r0 + 8 * lane;
            const float mu = lane == 0 ? m[0] : lane == 1 ? m[1] : lane == 2 ? m[2] : m[3];
            if (r < n) {
                int e = 0;
                if (mu > 0.f) frexpf(mu, &e);
                rowE[r] = e;
            }
        }
    }
#pragma unroll
    for (int i = 0; i < NF4; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) sm[w][4 * (lane + 32 * i) + e] = fm[i][e];
    __syncthreads();
    for (int j = threadIdx.x; j < D; j += blockDim.x) {
        float mm = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) mm = fmaxf(mm, sm[q][j]);
        atomicMax(&featmax[j], __float_as_uint(mm));
    }
}
}  // namespace

bool oz_rstats_wanted(int64_t n, int64_t D, int k) {
    return oz_enabled() && n > 0 && k > 32 && D % 4 == 0 && D <= 512;
}

void oz_rstats(const float *Rp, int64_t n, int64_t D, int32_t *rowE, uint32_t *featmax, cudaStream_t st) {
    TPO_REQUIRE(D >= 1 && D <= 512, "oz_rstats: D out of range");
    TPO_CUDA(cudaMemsetAsync(featmax, 0, sizeof(uint32_t) * D, st));
    if (n == 0) return;
    TPO_REQUIRE(D % 4 == 0 && (reinterpret_cast<uintptr_t>(Rp) & 15) == 0, "oz_rstats: R' must be 16-byte aligned rows");
    const unsigned grid = (unsigned)std::min<int64_t>(8 * sm_count(), cdiv(n, 32));
    const int nf4 = (int)cdiv(D, 128);
    if (nf4 <= 1) oz_rstats_kernel<1><<<grid, 256, 0, st>>>(Rp, n, (int)D, rowE, featmax);
    else if (nf4 <= 2) oz_rstats_kernel<2><<<grid, 256, 0, st>>>(Rp, n, (int)D, rowE, featmax);
    else oz_rstats_kernel<4><<<grid, 256, 0, st>>>(Rp, n, (int)D, rowE, featmax);
    TPO_LAUNCH_CHECK();
}

}  // namespace tpo
