// a7 step 1: Gram G = R^T R = R'^T diag(dinv^2) R' (D x D) on the 5th-generation tensor cores.
//
// R = dinv . R' is first split into TF32 halves (R = R_hi + R_lo, R_hi = rna-tf32(R), both
// stored fp32), then each 128 x 128 upper-triangular output tile accumulates
//      R_lo^T R_hi + R_hi^T R_lo + R_hi^T R_hi          ("3xTF32", fp32-accurate products)
// with tcgen05.mma kind::tf32 (both operands MN-major straight out of row-major R, staged by
// TMA with the 128-byte / 32-byte-atom swizzle), fp32 accumulators in TMEM.  Every SEG k-blocks (128 rows) the
// accumulator (every SEG k-blocks = 128 rows) is drained by 8 epilogue warps into fp64 registers (double-buffered TMEM, so
// the MMAs of the next segment overlap the drain), and the fp64 tile partials of the row
// splits are summed in split order by a second kernel (deterministic, no atomics).
//
// Warp roles (320 threads): warp 0 TMA producer, warp 1 MMA issuer (+ TMEM owner),
// warps 2..9 epilogue (TMEM lane quarter = warp % 4, column half = (warp - 2) / 4).
#include <cuda.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "tpo_internal.cuh"
#include "tc_ptx.cuh"

namespace tpo {
namespace {

constexpr int TILE = 128;          // output tile (M = N = 128)
constexpr int KB = 32;             // rows per k-block (4 MMAs of K = 8)
constexpr int STAGES = 3;
constexpr int SEG = 4;             // k-blocks per fp32 accumulation segment (128 rows)
constexpr int SLAB = 32 * KB * 4;  // one 32-column x 32-row fp32 slab (4 KB)
constexpr int OPER = 4 * SLAB;     // one 128-column operand tile (16 KB)
constexpr int STAGE_BYTES = 4 * OPER;   // A_hi, A_lo, B_hi, B_lo
constexpr int NTHREADS = 320;
constexpr int TMEM_COLS = 256;

// UMMA shared-memory descriptor for a 32-bit MN-major operand.  32-bit MN-major operands use the
// "128-byte swizzle with 32-byte atomicity" layout (descriptor layout type 1, TMA mode
// SWIZZLE_128B_ATOM_32B): 128-byte rows, 32-byte chunks XOR-swizzled over 4-row atoms.
// LBO = byte stride between 32-element (128 B) MN slabs, SBO = byte stride between 4-row K
// atoms (512 B); version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr & 0x3FFFF) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)1 << 61;     // SWIZZLE_128B_BASE32B
    return d;
}

// Instruction descriptor: kind::tf32, fp32 accumulate, A and B MN-major, M x N.
constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(
            tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

struct GramArgs {
    int n_tiles;        // T = ceil(D / 128)
    int ksplit;         // row splits
    int64_t rows_per;   // rows per split (multiple of KB)
    int64_t n;
    double *part;       // [ksplit][pairs][128][128]
};

__device__ __forceinline__ void pair_of(int p, int T, int &ta, int &tb) {
    int a = 0;
    while (p >= T - a) { p -= T - a; ++a; }
    ta = a;
    tb = a + p;
}

__global__ void __launch_bounds__(NTHREADS, 1)
gram_tc_kernel(const __grid_constant__ CUtensorMap map_hi, const __grid_constant__ CUtensorMap map_lo, GramArgs g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE_BYTES);
    // bars: full[STAGES], empty[STAGES], tfull[2], tempty[2]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * STAGES + 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    const int pairs = g.n_tiles * (g.n_tiles + 1) / 2;
    const int split = blockIdx.x % g.ksplit;
    const int pidx = blockIdx.x / g.ksplit;
    int ta, tb;
    pair_of(pidx, g.n_tiles, ta, tb);
    const bool diag = (ta == tb);
    const int64_t r0 = (int64_t)split * g.rows_per;
    const int64_t r1 = min(g.n, r0 + g.rows_per);
    const int nkb = r1 > r0 ? (int)((r1 - r0 + KB - 1) / KB) : 0;
    const int nseg = (nkb + SEG - 1) / SEG;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&bars[s]), 1);
            mbar_init(smem_u32(&bars[STAGES + s]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&bars[2 * STAGES + b]), 1);
            mbar_init(smem_u32(&bars[2 * STAGES + 2 + b]), 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_hi) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_lo) : "memory");
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
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            const uint32_t bytes = diag ? 2 * OPER : 4 * OPER;
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % STAGES, j = kb / STAGES;
                if (j > 0) mbar_wait(smem_u32(&bars[STAGES + s]), (j - 1) & 1);
                const uint32_t full = smem_u32(&bars[s]);
                mbar_expect_tx(full, bytes);
                const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
                const int y = (int)(r0 + (int64_t)kb * KB);
                for (int c = 0; c < 4; ++c) {
                    tma_load_2d(base + 0 * OPER + c * SLAB, &map_hi, full, ta * TILE + 32 * c, y);
                    tma_load_2d(base + 1 * OPER + c * SLAB, &map_lo, full, ta * TILE + 32 * c, y);
                    if (!diag) {
                        tma_load_2d(base + 2 * OPER + c * SLAB, &map_hi, full, tb * TILE + 32 * c, y);
                        tma_load_2d(base + 3 * OPER + c * SLAB, &map_lo, full, tb * TILE + 32 * c, y);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        constexpr uint32_t idesc = idesc_tf32(TILE, TILE);
        for (int seg = 0; seg < nseg; ++seg) {
            const int buf = seg & 1, use = seg >> 1;
            if (use > 0) mbar_wait(smem_u32(&bars[2 * STAGES + 2 + buf]), (use - 1) & 1);
            fence_after();
            const uint32_t tmem_d = tmem_base + buf * TILE;
            const int kb0 = seg * SEG, kb1 = min(nkb, kb0 + SEG);
            for (int kb = kb0; kb < kb1; ++kb) {
                const int s = kb % STAGES, j = kb / STAGES;
                mbar_wait(smem_u32(&bars[s]), j & 1);
                fence_after();
                if (lane == 0) {
                    const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
                    const uint32_t ahi = base, alo = base + OPER;
                    const uint32_t bhi = diag ? ahi : base + 2 * OPER, blo = diag ? alo : base + 3 * OPER;
#pragma unroll
                    for (int kk = 0; kk < KB / 8; ++kk) {
                        const uint32_t off = kk * 1024;
                        const uint64_t dAhi = umma_desc(ahi + off, SLAB, 512);
                        const uint64_t dAlo = umma_desc(alo + off, SLAB, 512);
                        const uint64_t dBhi = umma_desc(bhi + off, SLAB, 512);
                        const uint64_t dBlo = umma_desc(blo + off, SLAB, 512);
                        const uint32_t first = (kb == kb0 && kk == 0) ? 0u : 1u;
                        mma_tf32(tmem_d, dAlo, dBhi, idesc, first);
                        mma_tf32(tmem_d, dAhi, dBlo, idesc, 1u);
                        mma_tf32(tmem_d, dAhi, dBhi, idesc, 1u);
                    }
                    mma_commit(smem_u32(&bars[STAGES + s]));          // frees the smem stage
                    if (kb == kb1 - 1) mma_commit(smem_u32(&bars[2 * STAGES + buf]));   // segment done
                }
                __syncwarp();
            }
        }
    } else {
        // ---------------- epilogue: TMEM -> fp64 registers ----------------
        const int q = warp & 3, h = (warp - 2) >> 2;
        double acc[64];
#pragma unroll
        for (int i = 0; i < 64; ++i) acc[i] = 0.0;
        for (int seg = 0; seg < nseg; ++seg) {
            const int buf = seg & 1, use = seg >> 1;
            mbar_wait(smem_u32(&bars[2 * STAGES + buf]), use & 1);
            fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + buf * TILE + 64 * h;
            float v[32];
            tmem_ld32(taddr, v);
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[i] += (double)v[i];
            tmem_ld32(taddr + 32, v);
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[32 + i] += (double)v[i];
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bars[2 * STAGES + 2 + buf]));
        }
        double *out = g.part + (((int64_t)split * pairs + pidx) * TILE + (32 * q + lane)) * TILE + 64 * h;
#pragma unroll
        for (int i = 0; i < 64; i += 2) *reinterpret_cast<double2 *>(out + i) = make_double2(acc[i], acc[i + 1]);
    }
    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                     : "memory");
    }
}

// G[a][b] = sum_s part[s][pair(min tile, max tile)][..]; lower triangle mirrored from the upper.
__global__ void gram_reduce_kernel(const double *__restrict__ part, int D, int T, int ksplit, double *__restrict__ G) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)D * D) return;
    int a = (int)(i / D), b = (int)(i - (int64_t)a * D);
    if (a > b) { const int t = a; a = b; b = t; }
    const int ta = a / TILE, tb = b / TILE;
    const int pidx = ta * T - ta * (ta - 1) / 2 + (tb - ta);
    const int64_t pairs = (int64_t)T * (T + 1) / 2;
    const int64_t off = ((int64_t)pidx * TILE + (a - ta * TILE)) * TILE + (b - tb * TILE);
    double s = 0.0;
    for (int k = 0; k < ksplit; ++k) s += part[k * pairs * TILE * TILE + off];
    G[i] = s;
}

// R_hi = rna-tf32(dinv . R'), R_lo = dinv . R' - R_hi   (fp32 bit patterns)
__global__ void split_tf32_kernel(const float4 *__restrict__ Rp, const float *__restrict__ dinv, int64_t n, int D4,
                                  float4 *__restrict__ hi, float4 *__restrict__ lo) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n * D4) return;
    const float s = dinv[i / D4];
    const float4 x = Rp[i];
    float v[4] = {x.x * s, x.y * s, x.z * s, x.w * s}, h[4], l[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        uint32_t t;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(v[j]));
        h[j] = __uint_as_float(t);
        l[j] = v[j] - h[j];
    }
    hi[i] = make_float4(h[0], h[1], h[2], h[3]);
    lo[i] = make_float4(l[0], l[1], l[2], l[3]);
}

CUtensorMap make_map(const float *base, int64_t n, int64_t D) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)D * sizeof(float)};
    const cuuint32_t box[2] = {32, KB};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(TPO_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

struct GramPlan {
    int T, pairs, ksplit;
    int64_t rows_per;
};

GramPlan plan(int64_t n, int64_t D) {
    GramPlan p;
    p.T = (int)cdiv(D, TILE);
    p.pairs = p.T * (p.T + 1) / 2;
    const int64_t kblocks = std::max<int64_t>(1, cdiv(n, KB));
    int64_t ks = std::max<int64_t>(1, 148 / p.pairs);
    ks = std::min<int64_t>(ks, kblocks);
    p.rows_per = cdiv(kblocks, ks) * KB;
    p.ksplit = (int)std::max<int64_t>(1, cdiv(std::max<int64_t>(n, 1), p.rows_per));
    return p;
}


// =========================================================================================
// a5 on the tensor cores: Zo = sqrt(d) Zhat Q^T with 3xTF32 (K-major operands: Zhat rows and
// Q rows are both contiguous along the reduction index l), fp32 accumulation in TMEM over
// the d-term dot products, epilogue R' = sqrt(e/d) (sin Zo || cos Zo) straight from TMEM.
// Warps: 0 TMA producer, 1 MMA issuer (+ TMEM owner), 2..5 epilogue (lane quarter = warp % 4).
// =========================================================================================
constexpr int FT_M = 128, FT_N = 128, FT_KB = 32, FT_STAGES = 3;
constexpr int FT_OPER = FT_M * FT_KB * 4;          // 16 KB: 128 rows x 32 fp32 (128 B rows)
constexpr int FT_STAGE = 4 * FT_OPER;              // A_hi, A_lo, B_hi, B_lo
constexpr int FT_EPI = 8;                          // epilogue warps: 2 per TMEM lane quarter
constexpr int FT_THREADS = 32 * (2 + FT_EPI);

// sin / cos of an fp32 argument without the XU conversions of sincosf's reduction: k = rint(x 2/pi)
// by the 1.5 2^23 magic addition (the quadrant is the low bits of its pattern), r = x - k pi/2 with a
// two-part pi/2 (fma; |k| small, so r is accurate to ~1e-15), Cephes minimax polynomials on
// [-pi/4, pi/4] (~1 ulp).  |x| >= 2^17 (never reached here: |x| <= sqrt(d) for unit rows) falls
// back to sincosf.
__device__ __forceinline__ void sincos_fast(float x, float *sn, float *cs) {
    if (!(fabsf(x) < 131072.f)) {
        sincosf(x, sn, cs);
        return;
    }
    const float t = fmaf(x, 0.636619772367581343f, 12582912.f);       // 1.5 * 2^23 + rint(x 2/pi)
    const int q = __float_as_int(t) & 3;
    const float k = t - 12582912.f;
    float r = fmaf(-k, 1.57079637050628662109375f, x);
    r = fmaf(-k, -4.37113900018624283e-8f, r);
    const float z = r * r;
    const float sr = fmaf(r * z, fmaf(z, fmaf(z, -1.9515295891e-4f, 8.3321608736e-3f), -1.6666654611e-1f), r);
    const float cr = fmaf(z * z, fmaf(z, fmaf(z, 2.443315711809948e-5f, -1.388731625493765e-3f), 4.166664568298827e-2f),
                          fmaf(-0.5f, z, 1.0f));
    const float a = (q & 1) ? cr : sr, b = (q & 1) ? sr : cr;
    *sn = (q & 2) ? -a : a;
    *cs = ((q + 1) & 2) ? -b : b;
}

// K-major operand, 128-byte swizzle: 8-row x 128-byte atoms stacked along M/N at SBO = 1 KB.
__device__ __forceinline__ uint64_t umma_desc_kmajor(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr & 0x3FFFF) >> 4);
    d |= (uint64_t)1 << 16;                       // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;             // SBO
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;                       // SWIZZLE_128B
    return d;
}

constexpr uint32_t idesc_tf32_kmajor(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// Persistent: grid = min(tiles, SMs); a CTA walks the 128 x 128 output tiles t = blockIdx.x +
// i * gridDim.x (row tile = t / ncol, so the concurrently running CTAs share A row tiles in
// L2).  Two TMEM accumulators (2 x 128 columns): the MMA warp fills buffer i & 1 while the eight
// epilogue warps (two per TMEM lane quarter, half of the 32-column chunks each) drain the other
// one (sincos + stores), so the epilogue overlaps the MMAs.
// Barriers: full[s] / empty[s] per smem stage (TMA <-> MMA), tfull[a] (MMA commit -> epilogue),
// tempty[a] (8 epilogue warps -> MMA).
__global__ void __launch_bounds__(FT_THREADS, 1)
features_tc_kernel(const __grid_constant__ CUtensorMap mz_hi, const __grid_constant__ CUtensorMap mz_lo,
                   const __grid_constant__ CUtensorMap mq_hi, const __grid_constant__ CUtensorMap mq_lo, int64_t n,
                   int d, float *__restrict__ Rp) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + FT_STAGES * FT_STAGE);   // full[S], empty[S], tfull[2], tempty[2]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * FT_STAGES + 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nkb = (d + FT_KB - 1) / FT_KB;
    const int ncol = (d + FT_N - 1) / FT_N;
    const int64_t nrow = (n + FT_M - 1) / FT_M;
    const int64_t ntiles = nrow * ncol;
    if (threadIdx.x == 0) {
        for (int s = 0; s < FT_STAGES; ++s) {
            mbar_init(smem_u32(&bars[s]), 1);
            mbar_init(smem_u32(&bars[FT_STAGES + s]), 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(smem_u32(&bars[2 * FT_STAGES + a]), 1);
            mbar_init(smem_u32(&bars[2 * FT_STAGES + 2 + a]), FT_EPI);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(2 * FT_N)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (warp == 0) {
        if (lane == 0) {
            int64_t g = 0;                                   // k-blocks issued by this CTA
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int64_t i0 = (t / ncol) * FT_M;
                const int j0 = (int)(t % ncol) * FT_N;
                for (int kb = 0; kb < nkb; ++kb, ++g) {
                    const int s = (int)(g % FT_STAGES);
                    const int64_t j = g / FT_STAGES;
                    if (j > 0) mbar_wait(smem_u32(&bars[FT_STAGES + s]), (uint32_t)((j - 1) & 1));
                    const uint32_t full = smem_u32(&bars[s]);
                    mbar_expect_tx(full, FT_STAGE);
                    const uint32_t base = smem_u32(smem + s * FT_STAGE);
                    tma_load_2d(base + 0 * FT_OPER, &mz_hi, full, kb * FT_KB, (int)i0);
                    tma_load_2d(base + 1 * FT_OPER, &mz_lo, full, kb * FT_KB, (int)i0);
                    tma_load_2d(base + 2 * FT_OPER, &mq_hi, full, kb * FT_KB, j0);
                    tma_load_2d(base + 3 * FT_OPER, &mq_lo, full, kb * FT_KB, j0);
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = idesc_tf32_kmajor(FT_M, FT_N);
        int64_t g = 0;
        int i = 0;                                           // tiles of this CTA
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const int a = i & 1;
            if (i >= 2) {                                    // the epilogue drained this buffer (tile i - 2)
                mbar_wait(smem_u32(&bars[2 * FT_STAGES + 2 + a]), (uint32_t)(((i >> 1) - 1) & 1));
                fence_after();
            }
            const uint32_t acc = tmem_base + (uint32_t)(a * FT_N);
            for (int kb = 0; kb < nkb; ++kb, ++g) {
                const int s = (int)(g % FT_STAGES);
                const int64_t j = g / FT_STAGES;
                mbar_wait(smem_u32(&bars[s]), (uint32_t)(j & 1));
                fence_after();
                if (lane == 0) {
                    const uint32_t base = smem_u32(smem + s * FT_STAGE);
#pragma unroll
                    for (int kk = 0; kk < FT_KB / 8; ++kk) {
                        const uint32_t off = kk * 32;        // 8 fp32 of K inside the 128-byte atom
                        const uint64_t ah = umma_desc_kmajor(base + off), al = umma_desc_kmajor(base + FT_OPER + off);
                        const uint64_t bh = umma_desc_kmajor(base + 2 * FT_OPER + off);
                        const uint64_t bl = umma_desc_kmajor(base + 3 * FT_OPER + off);
                        mma_tf32(acc, al, bh, idesc, (kb | kk) ? 1u : 0u);
                        mma_tf32(acc, ah, bl, idesc, 1u);
                        mma_tf32(acc, ah, bh, idesc, 1u);
                    }
                    mma_commit(smem_u32(&bars[FT_STAGES + s]));
                    if (kb == nkb - 1) mma_commit(smem_u32(&bars[2 * FT_STAGES + a]));
                }
                __syncwarp();
            }
        }
    } else {
        const int q = warp & 3, half = (warp - 2) >> 2;
        float *tb = reinterpret_cast<float *>(smem + FT_STAGES * FT_STAGE + 256) + (warp - 2) * 1024;   // 32 x 32
        const float sd = sqrtf((float)d);
        const float amp = (float)sqrt(exp(1.0) / (double)d);
        const int64_t D = 2 * (int64_t)d;
        int i = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const int a = i & 1;
            const int64_t i0 = (t / ncol) * FT_M;
            const int j0 = (int)(t % ncol) * FT_N;
            mbar_wait(smem_u32(&bars[2 * FT_STAGES + a]), (uint32_t)((i >> 1) & 1));
            fence_after();
            const int64_t row = i0 + 32 * q + lane;
#pragma unroll 1
            for (int c = half * (FT_N / 64); c < (half + 1) * (FT_N / 64); ++c) {
                float v[32];
                tmem_ld32(tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(a * FT_N) + 32 * c, v);
                const int jb = j0 + 32 * c;
                if (jb + 32 > d && row >= n) continue;     // (the full-width path stores whole rows)
                float *ps = Rp + row * D + jb, *pc = Rp + row * D + d + jb;
                if (jb + 32 <= d) {
                    // lane = row: transpose the 32 x 32 block through the warp's smem buffer (XOR
                    // swizzle, conflict-free) so that every store writes one row's 128 contiguous
                    // bytes instead of 32 rows x 16 bytes
#pragma unroll
                    for (int tt = 0; tt < 32; ++tt) {
                        float sn, cs;
                        sincos_fast(sd * v[tt], &sn, &cs);
                        tb[lane * 32 + (tt ^ lane)] = amp * sn;
                        v[tt] = amp * cs;
                    }
                    __syncwarp();
                    const int64_t rb0 = i0 + 32 * q;
#pragma unroll 4
                    for (int rr = 0; rr < 32; ++rr)
                        if (rb0 + rr < n) Rp[(rb0 + rr) * D + jb + lane] = tb[rr * 32 + (lane ^ rr)];
                    __syncwarp();
#pragma unroll
                    for (int tt = 0; tt < 32; ++tt) tb[lane * 32 + (tt ^ lane)] = v[tt];
                    __syncwarp();
#pragma unroll 4
                    for (int rr = 0; rr < 32; ++rr)
                        if (rb0 + rr < n) Rp[(rb0 + rr) * D + d + jb + lane] = tb[rr * 32 + (lane ^ rr)];
                    __syncwarp();
                } else {
#pragma unroll
                    for (int tt = 0; tt < 32; ++tt) {
                        if (jb + tt < d) {
                            float sn, cs;
                            sincos_fast(sd * v[tt], &sn, &cs);
                            ps[tt] = amp * sn;
                            pc[tt] = amp * cs;
                        }
                    }
                }
            }
            fence_before();                                  // TMEM reads done before the MMA reuses it
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bars[2 * FT_STAGES + 2 + a]));
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * FT_N)
                     : "memory");
    }
}

// hi = rna-tf32(x), lo = x - hi   (plain split, no row scale)
__global__ void split_plain_kernel(const float4 *__restrict__ x, int64_t len4, float4 *__restrict__ hi,
                                   float4 *__restrict__ lo) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= len4) return;
    const float4 v4 = x[i];
    const float v[4] = {v4.x, v4.y, v4.z, v4.w};
    float h[4], l[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        uint32_t t;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(v[j]));
        h[j] = __uint_as_float(t);
        l[j] = v[j] - h[j];
    }
    hi[i] = make_float4(h[0], h[1], h[2], h[3]);
    lo[i] = make_float4(l[0], l[1], l[2], l[3]);
}

CUtensorMap make_map_kmajor(const float *base, int64_t rows, int64_t K, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)K * sizeof(float)};
    const cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(TPO_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

}  // namespace

size_t features_tc_ws(int64_t n, int64_t d) {
    return 2 * align_up(sizeof(float) * n * d) + 2 * align_up(sizeof(float) * d * d) + 1024;
}

// R'[:, 0:d] = sqrt(e/d) sin(sqrt(d) Zhat Q^T), R'[:, d:2d] = sqrt(e/d) cos(...)   (d % 4 == 0)
void features_tc(const float *Zhat, int64_t n, int64_t d, const float *Q, float *Rp, Arena &ar, cudaStream_t st) {
    float *zh = ar.take<float>(n * d), *zl = ar.take<float>(n * d);
    float *qh = ar.take<float>(d * d), *ql = ar.take<float>(d * d);
    split_plain_kernel<<<cdiv(n * d / 4, 256), 256, 0, st>>>((const float4 *)Zhat, n * d / 4, (float4 *)zh,
                                                           (float4 *)zl);
    TPO_LAUNCH_CHECK();
    split_plain_kernel<<<cdiv(d * d / 4, 256), 256, 0, st>>>((const float4 *)Q, d * d / 4, (float4 *)qh, (float4 *)ql);
    TPO_LAUNCH_CHECK();
    const CUtensorMap a_hi = make_map_kmajor(zh, n, d, FT_M), a_lo = make_map_kmajor(zl, n, d, FT_M);
    const CUtensorMap b_hi = make_map_kmajor(qh, d, d, FT_N), b_lo = make_map_kmajor(ql, d, d, FT_N);
    const size_t smem = FT_STAGES * FT_STAGE + 1024 + 256 + FT_EPI * 4096;   // + the epilogue transpose buffers
    static std::once_flag once;
    std::call_once(once, [&] {
        cudaFuncSetAttribute(features_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    const int64_t tiles = cdiv(n, FT_M) * cdiv(d, FT_N);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(tiles, sm_count()));
    features_tc_kernel<<<grid, FT_THREADS, smem, st>>>(a_hi, a_lo, b_hi, b_lo, n, (int)d, Rp);
    TPO_LAUNCH_CHECK();
}

size_t gram_tc_ws(int64_t n, int64_t D) {
    const GramPlan p = plan(n, D);
    return 2 * align_up(sizeof(float) * n * D) + align_up(sizeof(double) * p.ksplit * p.pairs * TILE * TILE) + 1024;
}

// G (D x D fp64, device) = R'^T diag(dinv^2) R'.  Requires D % 4 == 0 (TMA row pitch).
void gram_tc(const float *Rp, const float *dinv, int64_t n, int64_t D, double *G, Arena &ar, cudaStream_t st) {
    const GramPlan p = plan(n, D);
    float *hi = ar.take<float>(n * D), *lo = ar.take<float>(n * D);
    double *part = ar.take<double>((size_t)p.ksplit * p.pairs * TILE * TILE);
    split_tf32_kernel<<<cdiv(n * (D / 4), 256), 256, 0, st>>>((const float4 *)Rp, dinv, n, (int)(D / 4),
                                                            (float4 *)hi, (float4 *)lo);
    TPO_LAUNCH_CHECK();
    const CUtensorMap mh = make_map(hi, n, D), ml = make_map(lo, n, D);
    const size_t smem = STAGES * STAGE_BYTES + 1024 + 256;
    static std::once_flag once;
    std::call_once(once, [&] {
        cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    GramArgs a{p.T, p.ksplit, p.rows_per, n, part};
    gram_tc_kernel<<<p.pairs * p.ksplit, NTHREADS, smem, st>>>(mh, ml, a);
    TPO_LAUNCH_CHECK();
    gram_reduce_kernel<<<cdiv(D * D, 256), 256, 0, st>>>(part, (int)D, p.T, p.ksplit, G);
    TPO_LAUNCH_CHECK();
}

}  // namespace tpo
