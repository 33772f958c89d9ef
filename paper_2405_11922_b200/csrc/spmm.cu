// a1-a3: MSA propagation (Lemma 1 / Eq. PX; hop update Eq. update-Z,
// PAPER.md:454, bracketed L (L^T Z) as PAPER.md:456) on sm_100a.
//
// Data layout and fusion:
//   * The iterate is kept pre-scaled, P = s_u . Z (s_u = D_U^{-1/2}), in the caller's Z
//     buffer, so that neither SpMM gathers a per-edge scale:
//        SpMM-1 (rows of B^T, V side):   Q[v] = s_v[v]^2 * sum_{u in N(v)} w_uv P[u]
//        SpMM-2 (rows of B,   U side):   Z[u] = c X[u] + alpha s_u[u] sum_{v in N(u)} w_uv Q[v]
//                                         P[u] = s_u[u] Z[u]      (hops 1..T-1)
//     which is Z <- c X + alpha L (L^T Z) with L = D_U^{-1/2} B D_V^{-1/2} (Eq. L).
//     The last hop writes Z and fuses the row L2 normalisation (Eq. Z) when d <= 128.
//   * One warp gathers one 128-float column slice of a CSR row with 128-bit loads
//     (lane l owns float4 column l of the slice); 8 neighbour rows are in flight per warp.
//     Work is ordered slice-major, so for d > 128 the rows gathered at any time come from one
//     128-column slice of the dense operand (a slice of the V-side block is m x 512 B).
//   * Work items: consecutive short rows are grouped into row blocks of about CHUNK edges
//     (a new block starts where floor(row_ptr / CHUNK) changes), processed by one warp as a
//     single edge stream -- 8 gathers in flight regardless of row boundaries, rows flushed
//     through the epilogue as the stream crosses them (empty rows included).  Rows longer
//     than CHUNK edges are split into CHUNK-edge items that write partial sums, added in
//     chunk order by a fix-up kernel (deterministic: no float atomics anywhere).
#include <stdlib.h>

#include <algorithm>

#include "tpo_internal.cuh"

namespace tpo {
namespace {

constexpr int CHUNK = 256;           // edges per long-row chunk; also the row-block grouping grain
constexpr int kCounters = 64;        // persistent-warp work counters zeroed together
#ifndef TPO_L2_HINTS
#define TPO_L2_HINTS 1
#endif
constexpr int WPB = 8;               // warps per block
constexpr int UNR = 8;               // neighbour rows in flight per warp

enum Epi { EPI_V = 0, EPI_U = 1, EPI_FINAL = 2, EPI_RAW = 3 };

struct Sched {
    int64_t *offsets;      // [n_rows+1] packed exclusive scan: (items << 32) | slots
    int4 *items;           // {row, chunk, slot or -1, nchunks}
    int4 *slots;           // {row, chunk, nchunks, first slot}
    int64_t max_items, max_slots;
};

__device__ __forceinline__ int64_t packed_total(const int64_t *offsets, int64_t n) { return offsets[n]; }

// ---------------------------------------------------------------------------------------
// degrees -> scales (a1).  s = 1/sqrt(sum of weights), 1/sqrt(0) := 0 (R3).
// ---------------------------------------------------------------------------------------
__global__ void degree_scale_kernel(const int64_t *__restrict__ rowptr, const float *__restrict__ val,
                                    int64_t n, float *__restrict__ s) {
    const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const int64_t b = rowptr[row], e = rowptr[row + 1];
    double deg;
    if (val == nullptr) {
        deg = (double)(e - b);
    } else {
        double acc = 0.0;
        for (int64_t i = b + lane; i < e; i += 32) acc += (double)val[i];
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        deg = acc;
    }
    if (lane == 0) s[row] = deg > 0.0 ? (float)(1.0 / sqrt(deg)) : 0.0f;
}

// unweighted degrees: a thread per row (deg = row length; the same value as degree_scale_kernel)
__global__ void degree_scale_unw_kernel(const int64_t *__restrict__ rowptr, int64_t n, float *__restrict__ s) {
    const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (row >= n) return;
    const double deg = (double)(rowptr[row + 1] - rowptr[row]);
    s[row] = deg > 0.0 ? (float)(1.0 / sqrt(deg)) : 0.0f;
}

// weighted degrees in fp64 (sharded path: the V-side sums are all-reduced across ranks)
__global__ void degree_kernel(const int64_t *__restrict__ rowptr, const float *__restrict__ val, int64_t n,
                              double *__restrict__ deg) {
    const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const int64_t b = rowptr[row], e = rowptr[row + 1];
    double acc = 0.0;
    if (val == nullptr) {
        acc = lane == 0 ? (double)(e - b) : 0.0;
    } else {
        for (int64_t i = b + lane; i < e; i += 32) acc += (double)val[i];
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) deg[row] = acc;
}

__global__ void inv_sqrt_kernel(const double *__restrict__ deg, int64_t n, float *__restrict__ s) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) s[i] = deg[i] > 0.0 ? (float)(1.0 / sqrt(deg[i])) : 0.0f;
}

// Q[r] *= s[r]^2 (the V-side scale of a reduce-scattered slice)
__global__ void vscale_kernel(float4 *__restrict__ Q, const float *__restrict__ s, int64_t rows, int d4) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= rows * d4) return;
    const float v = s[i / d4];
    const float s2 = v * v;
    float4 q = Q[i];
    Q[i] = make_float4(q.x * s2, q.y * s2, q.z * s2, q.w * s2);
}

// ---------------------------------------------------------------------------------------
// Work schedule: items per row, packed exclusive scan, fill.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ bool row_is_long(const int64_t *rowptr, int64_t r) {
    return rowptr[r + 1] - rowptr[r] > CHUNK;
}
// A short row starts a row block at row 0, after a long row, or where floor(rowptr / CHUNK)
// changes.  Packed count: (items << 32) | slots.
__global__ void sched_count_kernel(const int64_t *__restrict__ rowptr, int64_t n, int64_t *__restrict__ cnt) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int64_t len = rowptr[r + 1] - rowptr[r];
    if (len > CHUNK) {
        const int64_t nch = (len + CHUNK - 1) / CHUNK;
        cnt[r] = (nch << 32) | nch;
        return;
    }
    const bool start = r == 0 || row_is_long(rowptr, r - 1) || (rowptr[r] / CHUNK != rowptr[r - 1] / CHUNK);
    cnt[r] = start ? (int64_t(1) << 32) : 0;
}

constexpr int SCAN_T = 1024, SCAN_I = 4, SCAN_TILE = SCAN_T * SCAN_I;

__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t *sh, int64_t &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int64_t w = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        sh[lane + 32] = w;   // inclusive warp totals
    }
    __syncthreads();
    const int64_t before = (wid ? sh[32 + wid - 1] : 0) + x - v;
    total = sh[32 + (blockDim.x >> 5) - 1];
    __syncthreads();
    return before;
}

__global__ void scan_tile_sums(const int64_t *__restrict__ in, int64_t n, int64_t *__restrict__ sums) {
    __shared__ int64_t sh[64];
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_I;
    int64_t s = 0;
    for (int i = 0; i < SCAN_I; ++i) s += (base + i < n) ? in[base + i] : 0;
    int64_t tot;
    block_exclusive_scan(s, sh, tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void scan_sums_single(int64_t *__restrict__ sums, int64_t nb) {
    __shared__ int64_t sh[64];
    int64_t carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += SCAN_T) {
        const int64_t i = b0 + threadIdx.x;
        const int64_t v = i < nb ? sums[i] : 0;
        int64_t tot;
        const int64_t ex = block_exclusive_scan(v, sh, tot);
        if (i < nb) sums[i] = carry + ex;
        carry += tot;
    }
}

__global__ void scan_apply(const int64_t *__restrict__ in, int64_t n, const int64_t *__restrict__ sums,
                           int64_t *__restrict__ out, int64_t *__restrict__ out_total) {
    __shared__ int64_t sh[64];
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_I;
    int64_t v[SCAN_I], s = 0;
    for (int i = 0; i < SCAN_I; ++i) {
        v[i] = (base + i < n) ? in[base + i] : 0;
        s += v[i];
    }
    int64_t tot;
    int64_t run = block_exclusive_scan(s, sh, tot) + sums[blockIdx.x];
    for (int i = 0; i < SCAN_I; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1) *out_total = run;
}

// items: {row, chunk, slot, nchunks} for long-row chunks; {first row, 0, -1, 0} for a row
// block (its rows end where the next item starts).
__global__ void sched_fill_kernel(const int64_t *__restrict__ rowptr, const int64_t *__restrict__ offsets,
                                  int64_t n, int4 *__restrict__ items, int4 *__restrict__ slots) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int64_t off = offsets[r], nxt = (r + 1 < n) ? offsets[r + 1] : offsets[n];
    const int64_t it0 = off >> 32;
    const int nit = (int)((nxt >> 32) - it0);
    if (nit == 0) return;
    const int64_t len = rowptr[r + 1] - rowptr[r];
    if (len <= CHUNK) {
        items[it0] = make_int4((int)r, 0, -1, 0);
        return;
    }
    const int sl0 = (int)(off & 0xffffffffLL);
    for (int j = 0; j < nit; ++j) {
        items[it0 + j] = make_int4((int)r, j, sl0 + j, nit);
        slots[sl0 + j] = make_int4((int)r, j, nit, sl0);
    }
}

// ---------------------------------------------------------------------------------------
// Gather SpMM + fused epilogues.
// ---------------------------------------------------------------------------------------
struct SpmmArgs {
    const int64_t *rowptr;
    const int32_t *col;
    const float *val;
    const float4 *src;        // gathered operand, row stride d4 float4
    int d4, nslices;          // nslices: 32-float4 slices (fix-up granularity)
    int ngroups;              // column groups of SL slices (gather granularity)
    Sched sch;
    int64_t n_rows;
    float4 *partials;         // [slots][d4]
    // epilogue
    const float *scale;       // s_v (EPI_V) or s_u (EPI_U / EPI_FINAL)
    const float4 *X;
    float c, alpha;
    float4 *out;              // Q (EPI_V), P (EPI_U), Z (EPI_FINAL)
    float4 *out_hat;          // Zhat (EPI_FINAL, fused when nslices == 1), else null
    unsigned long long *work; // persistent-warp work counter of this launch (zeroed)
    unsigned *arrive;         // per (long row, column group) chunk-arrival counters (zeroed once per
                              // propagation; each launch adds nchunks), or null: separate fix-up kernel
    int reserve_sms;          // SMs left free (blocks placed on them exit) for concurrent side-stream work
    int smid_limit;           // = SMs - reserve_sms, set at launch
    // column-group kernel only: the gathered table holds src_rows rows in LPE-float4 groups; the
    // output is written in out_L-float4 groups of out_rows rows (out_L = d4: row-major)
    int64_t src_rows, out_rows;
    int out_L;
};

// Packed fp32x2 arithmetic (FADD2 / FFMA2 on sm_100a): two lanes of a float4 per instruction,
// each lane rounded exactly as the scalar operation.
__device__ __forceinline__ unsigned long long pk(float x, float y) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
    return r;
}
__device__ __forceinline__ void upk(unsigned long long r, float &x, float &y) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(r));
}
__device__ __forceinline__ float4 f4fma(float w, float4 v, float4 a) {
    const unsigned long long ww = pk(w, w);
    unsigned long long lo = pk(a.x, a.y), hi = pk(a.z, a.w);
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(lo) : "l"(ww), "l"(pk(v.x, v.y)));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(hi) : "l"(ww), "l"(pk(v.z, v.w)));
    upk(lo, a.x, a.y);
    upk(hi, a.z, a.w);
    return a;
}
__device__ __forceinline__ float4 f4add(float4 a, float4 v) {
    unsigned long long lo = pk(a.x, a.y), hi = pk(a.z, a.w);
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(lo) : "l"(pk(v.x, v.y)));
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(hi) : "l"(pk(v.z, v.w)));
    upk(lo, a.x, a.y);
    upk(hi, a.z, a.w);
    return a;
}

// One warp gathers the SL float4 columns c4[0..SL) (stride 32) of the CSR rows in edges
// [beg, end) into acc[].
// L2 residency hints.  The gathered operand is re-read by many edges: loads carry an
// evict_last cache policy; the outputs (and X) are touched once per hop: streaming stores /
// loads (evict-first), so they do not push the gathered column group out of L2.
__device__ __forceinline__ uint64_t l2_keep_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ float4 ld_keep(const float4 *p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float4 gather_ld(const float4 *p) {
#if TPO_L2_HINTS
    return ld_keep(p, l2_keep_policy());
#else
    return __ldg(p);
#endif
}
// base + ro float4 in one IMAD.WIDE.U32
__device__ __forceinline__ const float4 *row_addr(const float4 *base, uint32_t ro) {
    const float4 *p;
    asm("mad.wide.u32 %0, %1, 16, %2;" : "=l"(p) : "r"(ro), "l"(base));
    return p;
}
__device__ __forceinline__ void st_stream(float4 *p, float4 v) {
#if TPO_L2_HINTS
    __stcs(p, v);
#else
    *p = v;
#endif
}

// Loads are unconditional: lanes past the end of an edge batch hold a valid (clamped) column
// and inactive column lanes read a clamped in-range address (`base`); neither is accumulated
// or stored.  Row offsets col * d4 are 32-bit (every gathered table has < 2^31 float4).
template <bool WEIGHTED, int SL, int UE>
__device__ __forceinline__ void gather_rows(const SpmmArgs &a, int64_t beg, int64_t end, const float4 *const (&base)[SL],
                                            float4 (&acc)[SL]) {
    const int lane = threadIdx.x & 31;
    constexpr int U = UE;
#pragma unroll
    for (int s = 0; s < SL; ++s) acc[s] = make_float4(0.f, 0.f, 0.f, 0.f);
    const uint32_t d4 = (uint32_t)a.d4;
    for (int64_t e0 = beg; e0 < end; e0 += 32) {
        const int cnt = (int)(end - e0 < 32 ? end - e0 : 32);
        const uint32_t myoff = (uint32_t)__ldg(a.col + e0 + (lane < cnt ? lane : 0)) * d4;
        // weight 0 past the batch end (the clamped row is read but adds +0)
        const float myw = lane < cnt ? (WEIGHTED ? __ldg(a.val + e0 + lane) : 1.f) : 0.f;
        for (int j = 0; j < cnt; j += U) {
            float4 v[U][SL];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t ro = __shfl_sync(0xffffffffu, myoff, j + u);
#pragma unroll
                for (int s = 0; s < SL; ++s) v[u][s] = gather_ld(row_addr(base[s], ro));
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const float w = __shfl_sync(0xffffffffu, myw, j + u);
#pragma unroll
                for (int s = 0; s < SL; ++s) acc[s] = f4fma(w, v[u][s], acc[s]);
            }
        }
    }
}

// Epilogue of one output row from its gathered sum `acc`; x (this lane's float4 of X[row])
// and s (the row's degree scale) are preloaded by the caller.
template <int EPI>
__device__ __forceinline__ void epilogue_v(const SpmmArgs &a, int64_t row, int c4, bool act, float4 acc, float4 x,
                                           float s) {
    const int64_t o = row * (int64_t)a.d4 + c4;
    if (EPI == EPI_RAW) {
        if (act) st_stream(a.out + o, acc);
        return;
    }
    if (EPI == EPI_V) {
        const float s2 = s * s;
        if (act) st_stream(a.out + o, make_float4(acc.x * s2, acc.y * s2, acc.z * s2, acc.w * s2));
        return;
    }
    const float g = a.alpha * s;
    float4 z;
    z.x = fmaf(a.c, x.x, g * acc.x);
    z.y = fmaf(a.c, x.y, g * acc.y);
    z.z = fmaf(a.c, x.z, g * acc.z);
    z.w = fmaf(a.c, x.w, g * acc.w);
    if (EPI == EPI_U) {
        if (act) st_stream(a.out + o, make_float4(s * z.x, s * z.y, s * z.z, s * z.w));
        return;
    }
    // EPI_FINAL
    if (act) st_stream(a.out + o, z);
    if (a.out_hat != nullptr) {            // only when nslices == 1: the warp owns the row
        float ss = act ? z.x * z.x + z.y * z.y + z.z * z.z + z.w * z.w : 0.f;
        for (int off = 16; off; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
        const float inv = ss > 0.f ? 1.0f / sqrtf(ss) : 0.f;
        if (act) st_stream(a.out_hat + o, make_float4(z.x * inv, z.y * inv, z.z * inv, z.w * inv));
    }
}

template <int EPI>
__device__ __forceinline__ float4 load_x(const SpmmArgs &a, int64_t row, int c4, bool act) {
    if (EPI == EPI_V || EPI == EPI_RAW || !act) return make_float4(0.f, 0.f, 0.f, 0.f);
#if TPO_L2_HINTS
    return __ldcs(a.X + row * (int64_t)a.d4 + c4);
#else
    return __ldg(a.X + row * (int64_t)a.d4 + c4);
#endif
}

template <int EPI>
__device__ __forceinline__ void epilogue(const SpmmArgs &a, int64_t row, int c4, bool act, float4 acc) {
    epilogue_v<EPI>(a, row, c4, act, acc, load_x<EPI>(a, row, c4, act), EPI == EPI_RAW ? 0.f : a.scale[row]);
}

// Epilogue of one output row over the warp's SL column slices; the fused row normalisation
// (EPI_FINAL with out_hat) is only used when one slice covers the whole row (nslices == 1).
template <int EPI, int SL>
__device__ __forceinline__ void epilogue_sl(const SpmmArgs &a, int64_t row, const int (&c4)[SL], const bool (&act)[SL],
                                            const float4 (&acc)[SL], const float4 (&x)[SL], float s) {
#pragma unroll
    for (int q = 0; q < SL; ++q) epilogue_v<EPI>(a, row, c4[q], act[q], acc[q], x[q], s);
}

template <int EPI, int SL>
__device__ __forceinline__ void load_x_sl(const SpmmArgs &a, int64_t row, const int (&c4)[SL], const bool (&act)[SL],
                                          float4 (&x)[SL]) {
#pragma unroll
    for (int q = 0; q < SL; ++q) x[q] = load_x<EPI>(a, row, c4[q], act[q]);
}

// One warp streams the edges of rows [r0, r1) (all short) for its SL column slices, flushing
// each row through the epilogue as the stream crosses its end; empty rows are flushed with 0.
template <int EPI, bool WEIGHTED, int SL, int UE>
__device__ __forceinline__ void process_row_block(const SpmmArgs &a, int64_t r0, int64_t r1, const int (&c4)[SL],
                                                  const bool (&act)[SL], const float4 *const (&base)[SL]) {
    const int lane = threadIdx.x & 31;
    constexpr int U = UE;
    const uint32_t d4 = (uint32_t)a.d4;
    const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t rb = r0; rb < r1; rb += 32) {
        const int nb = (int)(r1 - rb < 32 ? r1 - rb : 32);
        const int64_t e_beg = a.rowptr[rb];
        // edge positions relative to e_beg (a batch of <= 32 short rows has <= 32 * CHUNK edges)
        const int my_end = lane < nb ? (int)(a.rowptr[rb + 1 + lane] - e_beg) : 0;   // end of row rb + lane
        const float my_s = (EPI != EPI_RAW && lane < nb) ? a.scale[rb + lane] : 0.f;
        const int n_e = __shfl_sync(0xffffffffu, my_end, nb - 1);
        int cur = 0;
        int cur_end = __shfl_sync(0xffffffffu, my_end, 0);
        float4 xcur[SL], acc[SL];
        load_x_sl<EPI, SL>(a, rb, c4, act, xcur);
#pragma unroll
        for (int q = 0; q < SL; ++q) acc[q] = zero;
        for (int k0 = 0; k0 < n_e; k0 += 32) {
            const int cnt = n_e - k0 < 32 ? n_e - k0 : 32;
            const uint32_t myoff = (uint32_t)__ldg(a.col + e_beg + k0 + (lane < cnt ? lane : 0)) * d4;
            float myw = 1.f;
            if (WEIGHTED) myw = lane < cnt ? __ldg(a.val + e_beg + k0 + lane) : 0.f;
            for (int j = 0; j < cnt; j += U) {
                float4 v[U][SL];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t ro = __shfl_sync(0xffffffffu, myoff, j + u);
#pragma unroll
                    for (int q = 0; q < SL; ++q) v[u][q] = gather_ld(row_addr(base[q], ro));
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (j + u >= cnt) break;
                    const int e = k0 + j + u;
                    while (e >= cur_end) {               // warp-uniform: flush finished rows
                        epilogue_sl<EPI, SL>(a, rb + cur, c4, act, acc, xcur, __shfl_sync(0xffffffffu, my_s, cur));
#pragma unroll
                        for (int q = 0; q < SL; ++q) acc[q] = zero;
                        ++cur;
                        cur_end = __shfl_sync(0xffffffffu, my_end, cur);
                        load_x_sl<EPI, SL>(a, rb + cur, c4, act, xcur);
                    }
                    const float w = WEIGHTED ? __shfl_sync(0xffffffffu, myw, j + u) : 1.f;
#pragma unroll
                    for (int q = 0; q < SL; ++q) acc[q] = WEIGHTED ? f4fma(w, v[u][q], acc[q]) : f4add(acc[q], v[u][q]);
                }
            }
        }
        while (cur < nb) {                               // last row of the batch and empty rows
            epilogue_sl<EPI, SL>(a, rb + cur, c4, act, acc, xcur, __shfl_sync(0xffffffffu, my_s, cur));
#pragma unroll
            for (int q = 0; q < SL; ++q) acc[q] = zero;
            ++cur;
            if (cur < nb) load_x_sl<EPI, SL>(a, rb + cur, c4, act, xcur);
        }
    }
}

// One work unit: item `item` of the schedule for column group `grp`.
template <int EPI, bool WEIGHTED, int SL, int UE>
__device__ __forceinline__ void spmm_unit(const SpmmArgs &a, int grp, int64_t item, int64_t n_items) {
    const int lane = threadIdx.x & 31;
    const int4 it = a.sch.items[item];
    int c4[SL];
    bool act[SL];
    const float4 *base[SL];
#pragma unroll
    for (int q = 0; q < SL; ++q) {
        c4[q] = (grp * SL + q) * 32 + lane;
        act[q] = c4[q] < a.d4;
        base[q] = a.src + (act[q] ? c4[q] : a.d4 - 1);
    }
    if (it.w == 0) {                                     // row block
        const int64_t r1 = item + 1 < n_items ? (int64_t)a.sch.items[item + 1].x : a.n_rows;
        process_row_block<EPI, WEIGHTED, SL, UE>(a, it.x, r1, c4, act, base);
        return;
    }
    const int64_t rb = a.rowptr[it.x], re = a.rowptr[it.x + 1];   // chunk of a long row
    const int64_t beg = rb + (int64_t)it.y * CHUNK;
    const int64_t end = min(re, beg + CHUNK);
    float4 acc[SL];
    gather_rows<WEIGHTED, SL, UE>(a, beg, end, base, acc);
#pragma unroll
    for (int q = 0; q < SL; ++q)
        if (act[q]) a.partials[(int64_t)it.z * a.d4 + c4[q]] = acc[q];
    if (a.arrive == nullptr) return;
    // the last chunk to arrive finishes the row: partials added in chunk order (the same sum as
    // the fix-up kernel, whichever warp does it)
    __threadfence();
    const int slot0 = it.z - it.y;
    unsigned old = 0;
    if (lane == 0) old = atomicAdd(a.arrive + (int64_t)slot0 * a.ngroups + grp, 1u);
    old = __shfl_sync(0xffffffffu, old, 0);
    if ((int)(old % (unsigned)it.w) != it.w - 1) return;
    __threadfence();
#pragma unroll
    for (int q = 0; q < SL; ++q) {
        float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (act[q]) {
            const float4 *pp = a.partials + (int64_t)slot0 * a.d4 + c4[q];
            for (int j = 0; j < it.w; ++j) s4 = f4add(s4, __ldcg(pp + (int64_t)j * a.d4));
        }
        epilogue<EPI>(a, it.x, c4[q], act[q], s4);
    }
}

// Persistent warps: the grid is the resident capacity (SMs x MINB blocks); each warp takes the
// next work unit from a device counter (*a.work, zeroed before the launch).  Units are ordered
// group-major, so concurrently running warps work on the same column group (its gathered
// working set stays L2-resident) -- and no block holds its slot while one slow warp finishes.
// Which warp runs a unit does not change its result (each unit is computed by one warp in a
// fixed order), so results stay deterministic.
template <int EPI, bool WEIGHTED, int SL, int MINB, int UE = (UNR / SL > 0 ? UNR / SL : 1)>
__global__ void __launch_bounds__(WPB * 32, MINB) spmm_kernel(SpmmArgs a) {
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    if ((int)smid >= a.smid_limit) return;            // a reserved SM: leave it to the side stream
    const int lane = threadIdx.x & 31;
    const int64_t tot = packed_total(a.sch.offsets, a.n_rows);
    const int64_t n_items = tot >> 32;
    const int64_t units = n_items * a.ngroups;
    while (true) {
        unsigned long long u = 0;
        if (lane == 0) u = atomicAdd(a.work, 1ull);
        u = __shfl_sync(0xffffffffu, u, 0);
        if ((int64_t)u >= units) return;
        const int grp = (int)((int64_t)u / n_items);
        spmm_unit<EPI, WEIGHTED, SL, UE>(a, grp, (int64_t)u - (int64_t)grp * n_items, n_items);
    }
}

template <int EPI>
__global__ void __launch_bounds__(WPB * 32) fixup_kernel(SpmmArgs a) {
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t tot = packed_total(a.sch.offsets, a.n_rows);
    const int64_t n_slots = tot & 0xffffffffLL;
    const int slice = (int)(gw / a.sch.max_slots);
    const int64_t slot = gw - (int64_t)slice * a.sch.max_slots;
    if (slot >= n_slots) return;
    const int4 s = a.sch.slots[slot];
    if (s.y != 0) return;                       // the warp of chunk 0 finishes the row
    const int c4 = slice * 32 + lane;
    const bool act = c4 < a.d4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (act) {
        const float4 *p = a.partials + (int64_t)slot * a.d4 + c4;
        int j = 0;
        for (; j + 16 <= s.z; j += 16) {               // 16 loads in flight, added in chunk order
            float4 v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) v[u] = p[(int64_t)(j + u) * a.d4];
#pragma unroll
            for (int u = 0; u < 16; ++u) acc = f4add(acc, v[u]);
        }
        for (; j + 4 <= s.z; j += 4) {
            float4 v0 = p[(int64_t)(j + 0) * a.d4], v1 = p[(int64_t)(j + 1) * a.d4];
            float4 v2 = p[(int64_t)(j + 2) * a.d4], v3 = p[(int64_t)(j + 3) * a.d4];
            acc = f4add(acc, v0); acc = f4add(acc, v1); acc = f4add(acc, v2); acc = f4add(acc, v3);
        }
        for (; j < s.z; ++j) acc = f4add(acc, p[(int64_t)j * a.d4]);
    }
    epilogue<EPI>(a, s.x, c4, act, acc);
}

// ---------------------------------------------------------------------------------------
// Column-group SpMM (propagation on tables too large for L2 at full width).  The gathered table
// is stored in column groups of LPE float4 ("blocked": [group][row][LPE float4]); the work is
// ordered group-major, so while the warps work on group g every gathered row comes from one
// rows x 16*LPE-byte slice of the table, which stays L2-resident where the full-width table
// (1 GB for the large config's P) does not.  A warp gathers E = 32 / LPE edges per load
// instruction (lane sg * LPE + sl loads float4 sl of edge sg of the stream), accumulates per
// lane, and folds the E partial sums of a row with an xor butterfly when the edge stream
// crosses the row's end (fp addition is commutative, so every lane of a group holds the same
// sum; the order is fixed by the edge positions: deterministic).  Outputs are written in
// out_L-float4 groups (out_L = d4: row-major Z on the last hop).
// ---------------------------------------------------------------------------------------
template <int LPE>
__device__ __forceinline__ float4 fold_edges(float4 a) {
#pragma unroll
    for (int o = LPE; o < 32; o <<= 1) {
        a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
        a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
        a.z += __shfl_xor_sync(0xffffffffu, a.z, o);
        a.w += __shfl_xor_sync(0xffffffffu, a.w, o);
    }
    return a;
}

// epilogue of one output row (lanes of edge slot 0 only): o = the row's output offset
template <int EPI>
__device__ __forceinline__ void gepilogue(const SpmmArgs &a, int64_t o, float4 acc, float4 x, float s) {
    if (EPI == EPI_RAW) {
        st_stream(a.out + o, acc);
        return;
    }
    if (EPI == EPI_V) {
        const float s2 = s * s;
        st_stream(a.out + o, make_float4(acc.x * s2, acc.y * s2, acc.z * s2, acc.w * s2));
        return;
    }
    const float g = a.alpha * s;
    float4 z;
    z.x = fmaf(a.c, x.x, g * acc.x);
    z.y = fmaf(a.c, x.y, g * acc.y);
    z.z = fmaf(a.c, x.z, g * acc.z);
    z.w = fmaf(a.c, x.w, g * acc.w);
    if (EPI == EPI_U) st_stream(a.out + o, make_float4(s * z.x, s * z.y, s * z.z, s * z.w));
    else st_stream(a.out + o, z);
}

template <int EPI>
__device__ __forceinline__ float4 gload_x(const SpmmArgs &a, int64_t row, int c4, bool lead) {
    if (EPI == EPI_V || EPI == EPI_RAW || !lead) return make_float4(0.f, 0.f, 0.f, 0.f);
#if TPO_L2_HINTS
    return __ldcs(a.X + row * (int64_t)a.d4 + c4);
#else
    return __ldg(a.X + row * (int64_t)a.d4 + c4);
#endif
}

template <int EPI, bool WEIGHTED, int LPE, int UMAX>
__device__ __forceinline__ void gspmm_unit(const SpmmArgs &a, int grp, int64_t item, int64_t n_items) {
    constexpr int E = 32 / LPE;                       // edges per load instruction
    constexpr int U = (32 / E) < UMAX ? (32 / E) : UMAX;   // load instructions in flight (E * U divides 32)
    const int lane = threadIdx.x & 31, sg = lane / LPE, sl = lane % LPE;
    const bool lead = sg == 0;
    const int c4 = grp * LPE + sl;
    const float4 *base = a.src + (int64_t)grp * a.src_rows * LPE + sl;
    const int64_t o_lane = (int64_t)(c4 / a.out_L) * a.out_rows * a.out_L + (c4 % a.out_L);
    const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
    const int4 it = a.sch.items[item];
    if (it.w == 0) {                                   // row block: one edge stream over its rows
        const int64_t r0 = it.x;
        const int64_t r1 = item + 1 < n_items ? (int64_t)a.sch.items[item + 1].x : a.n_rows;
        for (int64_t rb = r0; rb < r1; rb += 32) {
            const int nb = (int)(r1 - rb < 32 ? r1 - rb : 32);
            const int64_t e_beg = a.rowptr[rb];
            const int my_end = lane < nb ? (int)(a.rowptr[rb + 1 + lane] - e_beg) : 0;
            const float my_s = (EPI != EPI_RAW && lane < nb) ? a.scale[rb + lane] : 0.f;
            const int n_e = __shfl_sync(0xffffffffu, my_end, nb - 1);
            int cur = 0;
            int cur_end = __shfl_sync(0xffffffffu, my_end, 0);
            float4 acc = zero;
            float4 xcur = gload_x<EPI>(a, rb, c4, lead);
            auto flush = [&]() {                        // warp-uniform: row rb + cur is complete
                const float s = __shfl_sync(0xffffffffu, my_s, cur);
                const float4 tot = fold_edges<LPE>(acc);
                if (lead) gepilogue<EPI>(a, o_lane + (rb + cur) * a.out_L, tot, xcur, s);
                acc = zero;
                ++cur;
                cur_end = __shfl_sync(0xffffffffu, my_end, cur < nb ? cur : nb - 1);
                if (cur < nb) xcur = gload_x<EPI>(a, rb + cur, c4, lead);
            };
            for (int k0 = 0; k0 < n_e; k0 += 32) {
                const int cnt = n_e - k0 < 32 ? n_e - k0 : 32;
                const uint32_t mycol = (uint32_t)__ldg(a.col + e_beg + k0 + (lane < cnt ? lane : cnt - 1));
                const float myw = WEIGHTED ? (lane < cnt ? __ldg(a.val + e_beg + k0 + lane) : 0.f) : 1.f;
                for (int j = 0; j < cnt; j += E * U) {
                    float4 v[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int idx = j + u * E + sg;
                        const uint32_t ro = __shfl_sync(0xffffffffu, mycol, idx < cnt ? idx : cnt - 1) * LPE;
                        v[u] = gather_ld(row_addr(base, ro));
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (j + u * E >= cnt) break;            // warp-uniform
                        const int idx = j + u * E + sg;
                        const float w = WEIGHTED ? __shfl_sync(0xffffffffu, myw, idx < cnt ? idx : cnt - 1) : 1.f;
                        const int e = k0 + idx;
                        bool pend = idx < cnt;
                        while (true) {
                            if (pend && e < cur_end) {
                                acc = WEIGHTED ? f4fma(w, v[u], acc) : f4add(acc, v[u]);
                                pend = false;
                            }
                            if (!__any_sync(0xffffffffu, pend)) break;
                            flush();
                        }
                    }
                }
            }
            while (cur < nb) flush();                   // the last row and trailing empty rows
        }
        return;
    }
    // one CHUNK-edge chunk of a long row -> partial sum; the last chunk to arrive finishes the row
    const int64_t rbe = a.rowptr[it.x], re = a.rowptr[it.x + 1];
    const int64_t beg = rbe + (int64_t)it.y * CHUNK;
    const int64_t end = min(re, beg + CHUNK);
    float4 acc = zero;
    for (int64_t e0 = beg; e0 < end; e0 += 32) {
        const int cnt = (int)(end - e0 < 32 ? end - e0 : 32);
        const uint32_t mycol = (uint32_t)__ldg(a.col + e0 + (lane < cnt ? lane : cnt - 1));
        const float myw = WEIGHTED ? (lane < cnt ? __ldg(a.val + e0 + lane) : 0.f) : 1.f;
        for (int j = 0; j < cnt; j += E * U) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int idx = j + u * E + sg;
                const uint32_t ro = __shfl_sync(0xffffffffu, mycol, idx < cnt ? idx : cnt - 1) * LPE;
                v[u] = gather_ld(row_addr(base, ro));
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int idx = j + u * E + sg;
                const float w = WEIGHTED ? __shfl_sync(0xffffffffu, myw, idx < cnt ? idx : cnt - 1) : 1.f;
                if (idx < cnt) acc = WEIGHTED ? f4fma(w, v[u], acc) : f4add(acc, v[u]);
            }
        }
    }
    const float4 tot = fold_edges<LPE>(acc);
    if (lead) a.partials[(int64_t)it.z * a.d4 + c4] = tot;
    __threadfence();
    const int slot0 = it.z - it.y;
    unsigned old = 0;
    if (lane == 0) old = atomicAdd(a.arrive + (int64_t)slot0 * a.ngroups + grp, 1u);
    old = __shfl_sync(0xffffffffu, old, 0);
    if ((int)(old % (unsigned)it.w) != it.w - 1) return;
    __threadfence();
    if (!lead) return;
    float4 s4 = zero;
    const float4 *pp = a.partials + (int64_t)slot0 * a.d4 + c4;
    for (int j = 0; j < it.w; ++j) s4 = f4add(s4, __ldcg(pp + (int64_t)j * a.d4));
    const float s = EPI == EPI_RAW ? 0.f : a.scale[it.x];
    gepilogue<EPI>(a, o_lane + (int64_t)it.x * a.out_L, s4, gload_x<EPI>(a, it.x, c4, true), s);
}

// Persistent warps over (column group, work item) units, group-major (see spmm_kernel).
template <int EPI, bool WEIGHTED, int LPE, int UMAX, int MINB>
__global__ void __launch_bounds__(WPB * 32, MINB) gspmm_kernel(SpmmArgs a) {
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    if ((int)smid >= a.smid_limit) return;
    const int lane = threadIdx.x & 31;
    const int64_t n_items = packed_total(a.sch.offsets, a.n_rows) >> 32;
    const int64_t units = n_items * a.ngroups;
    while (true) {
        unsigned long long u = 0;
        if (lane == 0) u = atomicAdd(a.work, 1ull);
        u = __shfl_sync(0xffffffffu, u, 0);
        if ((int64_t)u >= units) return;
        const int grp = (int)((int64_t)u / n_items);
        gspmm_unit<EPI, WEIGHTED, LPE, UMAX>(a, grp, (int64_t)u - (int64_t)grp * n_items, n_items);
    }
}

// P0 = s_u . (c X) for T >= 1; for T == 0, Z = c X (and Zhat = rownorm, see below).
// out_L: column-group width of the output layout (d4: row-major).
__global__ void init_scaled_kernel(const float4 *__restrict__ X, const float *__restrict__ su, int64_t n, int d4,
                                   float c, int scale_rows, float4 *__restrict__ out, int out_L) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n * d4) return;
    const int64_t row = i / d4;
    const int c4 = (int)(i - row * d4);
    const float s = scale_rows ? su[row] * c : c;
    const float4 x = X[i];
    out[(int64_t)(c4 / out_L) * n * out_L + row * out_L + (c4 % out_L)] = make_float4(s * x.x, s * x.y, s * x.z, s * x.w);
}

// Zhat = Z / ||Z|| row-wise (warp per row), zero rows stay zero (R4).
__global__ void rownorm_kernel(const float4 *__restrict__ Z, int64_t n, int d4, float4 *__restrict__ Zh) {
    const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const float4 *z = Z + row * d4;
    float ss = 0.f;
    for (int j = lane; j < d4; j += 32) {
        const float4 v = z[j];
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float inv = ss > 0.f ? 1.0f / sqrtf(ss) : 0.f;
    for (int j = lane; j < d4; j += 32) {
        const float4 v = z[j];
        Zh[row * d4 + j] = make_float4(v.x * inv, v.y * inv, v.z * inv, v.w * inv);
    }
}

struct SchedBufs {
    Sched s;
    int64_t *cnt, *tilesums;
};

SchedBufs sched_alloc(Arena &ar, int64_t n_rows, int64_t nnz) {
    SchedBufs b;
    b.s.max_items = n_rows + 2 * (nnz / CHUNK) + 1;
    b.s.max_slots = 2 * (nnz / CHUNK) + 1;
    b.s.offsets = ar.take<int64_t>(n_rows + 1);
    b.s.items = ar.take<int4>(b.s.max_items);
    b.s.slots = ar.take<int4>(b.s.max_slots);
    b.cnt = ar.take<int64_t>(n_rows + 1);
    b.tilesums = ar.take<int64_t>(cdiv(n_rows + 1, SCAN_TILE) + 1);
    return b;
}

void sched_build(SchedBufs &b, const int64_t *rowptr, int64_t n_rows, cudaStream_t st) {
    const int T = 256;
    sched_count_kernel<<<cdiv(n_rows, T), T, 0, st>>>(rowptr, n_rows, b.cnt);
    TPO_LAUNCH_CHECK();
    const int64_t nb = cdiv(n_rows, SCAN_TILE);
    scan_tile_sums<<<nb, SCAN_T, 0, st>>>(b.cnt, n_rows, b.tilesums);
    TPO_LAUNCH_CHECK();
    scan_sums_single<<<1, SCAN_T, 0, st>>>(b.tilesums, nb);
    TPO_LAUNCH_CHECK();
    scan_apply<<<nb, SCAN_T, 0, st>>>(b.cnt, n_rows, b.tilesums, b.s.offsets, b.s.offsets + n_rows);
    TPO_LAUNCH_CHECK();
    sched_fill_kernel<<<cdiv(n_rows, T), T, 0, st>>>(rowptr, b.s.offsets, n_rows, b.s.items, b.s.slots);
    TPO_LAUNCH_CHECK();
}

// Row-major kernel: one 128-float column slice per warp (SL = 1) with 4 resident blocks per SM,
// measured best on small (d = 1000), medium (d = 256) and large (d = 128) against SL = 2 / 3-4
// blocks and 16 rows in flight.
template <int EPI, bool W>
void spmm_launch_rm(SpmmArgs a, int64_t max_items, cudaStream_t st) {
    constexpr int MINB = 4;
    a.ngroups = a.nslices;
    const int64_t blocks = cdiv(max_items * a.ngroups, WPB);
    // persistent warps: at most the resident capacity (SMs x MINB blocks of WPB warps)
    const int nsm = sm_count();
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)nsm * MINB));
    // the reserve applies only to a full-capacity grid (blocks on every SM, so the blocks of the
    // non-reserved SMs exist and drain the work queue); a smaller grid keeps every block
    a.smid_limit = (int64_t)grid == (int64_t)nsm * MINB ? std::max(1, nsm - std::max(0, a.reserve_sms)) : (1 << 30);
    spmm_kernel<EPI, W, 1, MINB><<<grid, WPB * 32, 0, st>>>(a);
    TPO_LAUNCH_CHECK();
}

template <int EPI>
void spmm_launch(const SpmmArgs &a, int64_t max_items, int64_t max_slots, bool weighted, cudaStream_t st) {
    if (weighted) spmm_launch_rm<EPI, true>(a, max_items, st);
    else spmm_launch_rm<EPI, false>(a, max_items, st);
    if (a.arrive) return;                 // long rows finished by their last chunk (fused fix-up)
    const int64_t fw = max_slots * a.nslices;
    fixup_kernel<EPI><<<cdiv(fw, WPB), WPB * 32, 0, st>>>(a);
    TPO_LAUNCH_CHECK();
}

// Column-group kernel launch: LPE = a.ngroups' group width (a.d4 / a.ngroups); needs a.arrive.
template <int EPI, bool W, int UMAX, int MINB>
void gspmm_launch(SpmmArgs a, int lpe, int64_t max_items, cudaStream_t st) {
    a.ngroups = a.d4 / lpe;
    const int64_t blocks = cdiv(max_items * a.ngroups, WPB);
    const int nsm = sm_count();
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)nsm * MINB));
    a.smid_limit = (int64_t)grid == (int64_t)nsm * MINB ? std::max(1, nsm - std::max(0, a.reserve_sms)) : (1 << 30);
    switch (lpe) {
        case 4: gspmm_kernel<EPI, W, 4, UMAX, MINB><<<grid, WPB * 32, 0, st>>>(a); break;
        case 8: gspmm_kernel<EPI, W, 8, UMAX, MINB><<<grid, WPB * 32, 0, st>>>(a); break;
        case 16: gspmm_kernel<EPI, W, 16, UMAX, MINB><<<grid, WPB * 32, 0, st>>>(a); break;
        default: gspmm_kernel<EPI, W, 32, UMAX, MINB><<<grid, WPB * 32, 0, st>>>(a); break;
    }
    TPO_LAUNCH_CHECK();
}

// (8 loads in flight per warp, 3 resident blocks per SM): measured faster than (4, 4)
template <int EPI>
void gspmm(const SpmmArgs &a, int lpe, int64_t max_items, bool weighted, cudaStream_t st) {
    if (weighted) gspmm_launch<EPI, true, 8, 3>(a, lpe, max_items, st);
    else gspmm_launch<EPI, false, 8, 3>(a, lpe, max_items, st);
}

// Column-group width (float4) of a gathered table of `rows` rows: the widest group whose slice
// (rows x 16 * L bytes) fits the L2 budget, among the widths dividing d4 (>= 4: 64-byte pieces,
// two DRAM sectors).  0 = no group width divides d4 (the row-major kernel is used).
// TPO_SPMM_L = "Lp,Lq" overrides both choices (tuning and the per-width parity tests).
constexpr double kL2SliceBudget = 64.0 * (1 << 20);
int group_width(int64_t rows, int d4) {
    for (int L = 32; L >= 4; L >>= 1)
        if (d4 % L == 0 && (double)rows * L * 16.0 <= kL2SliceBudget) return L;
    return d4 % 4 == 0 ? 4 : 0;
}
void choose_widths(int64_t n, int64_t m, int d4, int &Lp, int &Lq) {
    // measured (large, medium): every column-group layout is slower than the row-major slice
    // kernel (per-group index re-reads, shuffles and row folds cost more than the L2 locality
    // saves), so the row-major layout is the default; group_width() is kept for the override.
    Lp = Lq = 0;
    (void)n; (void)m;
    if (const char *e = getenv("TPO_SPMM_L")) {
        int a = 0, b = 0;
        if (sscanf(e, "%d,%d", &a, &b) == 2) {
            auto ok = [&](int L) { return L == 0 || ((L == 4 || L == 8 || L == 16 || L == 32) && d4 % L == 0); };
            if (ok(a) && ok(b)) { Lp = a; Lq = b; }
        }
    }
    // both row-major (the slice-major row-major kernel) when either table cannot be grouped or
    // both fit L2 at full width in 32-float4 slices
    if (Lp == 0 || Lq == 0) Lp = Lq = 0;
}

}  // namespace

size_t propagate_ws_bytes(int64_t n_u, int64_t n_v, int64_t nnz, int64_t d) {
    Arena ar(nullptr, 0);
    ar.take<float>(n_v * d);                      // Q (V-side block)
    ar.take<float>(n_u);
    ar.take<float>(n_v);
    sched_alloc(ar, n_u, nnz);
    sched_alloc(ar, n_v, nnz);
    ar.take<float>((2 * (nnz / CHUNK) + 1) * d);  // partials (shared by both SpMMs)
    ar.take<unsigned long long>(kCounters);       // persistent-warp work counters
    const int64_t ncnt = std::max<int64_t>((d / 4 + 31) / 32, d / 16);   // slices or column groups
    ar.take<unsigned>((2 * (nnz / CHUNK) + 1) * ncnt);  // chunk-arrival counters (U side)
    ar.take<unsigned>((2 * (nnz / CHUNK) + 1) * ncnt);  // (V side)
    return ar.off + 256;
}

void propagate_impl(const tpo_csr_t &B, const tpo_csr_t &Bt, const float *X, int64_t d, float alpha,
                    int32_t T, float *Z, float *Zhat, Arena &ar, cudaStream_t st, int reserve_sms,
                    int reserve_launches, cudaEvent_t b_cols_ready) {
    const int64_t n = B.n_rows, m = B.n_cols, nnz = B.nnz;
    const int d4 = (int)(d / 4);
    const float c = alpha < 1.0f ? 1.0f - alpha : 1.0f;    // R1
    float *Qv = ar.take<float>(m * d);
    float *su = ar.take<float>(n);
    float *sv = ar.take<float>(m);
    SchedBufs sb = sched_alloc(ar, n, nnz);
    SchedBufs sbt = sched_alloc(ar, m, nnz);
    float *partials = ar.take<float>((2 * (nnz / CHUNK) + 1) * d);
    unsigned long long *work = ar.take<unsigned long long>(kCounters);
    const int64_t ncnt = std::max<int64_t>((d4 + 31) / 32, d4 / 4);
    unsigned *arr_u = ar.take<unsigned>(sb.s.max_slots * ncnt), *arr_v = ar.take<unsigned>(sbt.s.max_slots * ncnt);
    TPO_CUDA(cudaMemsetAsync(arr_u, 0, sizeof(unsigned) * sb.s.max_slots * ncnt, st));
    TPO_CUDA(cudaMemsetAsync(arr_v, 0, sizeof(unsigned) * sbt.s.max_slots * ncnt, st));
    int launches = 0;
    auto counter = [&]() {        // a zeroed counter per SpMM launch (the pool is re-zeroed when it wraps)
        if (launches % kCounters == 0) TPO_CUDA(cudaMemsetAsync(work, 0, sizeof(unsigned long long) * kCounters, st));
        return work + (launches++ % kCounters);
    };

    const int TB = 256;
    if (n > 0) {
        if (B.val) degree_scale_kernel<<<cdiv(n * 32, TB), TB, 0, st>>>(B.row_ptr, B.val, n, su);
        else degree_scale_unw_kernel<<<cdiv(n, TB), TB, 0, st>>>(B.row_ptr, n, su);
    }
    TPO_LAUNCH_CHECK();
    if (m > 0) {
        if (Bt.val) degree_scale_kernel<<<cdiv(m * 32, TB), TB, 0, st>>>(Bt.row_ptr, Bt.val, m, sv);
        else degree_scale_unw_kernel<<<cdiv(m, TB), TB, 0, st>>>(Bt.row_ptr, m, sv);
    }
    TPO_LAUNCH_CHECK();
    if (n == 0) return;
    if (T == 0) {
        init_scaled_kernel<<<cdiv(n * d4, TB), TB, 0, st>>>((const float4 *)X, su, n, d4, c, 0, (float4 *)Z, d4);
        TPO_LAUNCH_CHECK();
        if (Zhat) rownorm_kernel<<<cdiv(n * 32, TB), TB, 0, st>>>((const float4 *)Z, n, d4, (float4 *)Zhat);
        TPO_LAUNCH_CHECK();
        return;
    }
    sched_build(sb, B.row_ptr, n, st);
    if (m > 0) sched_build(sbt, Bt.row_ptr, m, st);
    // Layouts: Lp / Lq = column-group widths of the iterate P (n rows, gathered by SpMM-1) and of
    // the V-side block Q (m rows, gathered by SpMM-2); 0 = row-major with the slice kernel.
    int Lp = 0, Lq = 0;
    choose_widths(n, m, d4, Lp, Lq);
    const bool grouped = Lp > 0;
    init_scaled_kernel<<<cdiv(n * d4, TB), TB, 0, st>>>((const float4 *)X, su, n, d4, c, 1, (float4 *)Z,
                                                        grouped ? Lp : d4);
    TPO_LAUNCH_CHECK();

    const int nslices = (d4 + 31) / 32;
    for (int t = 0; t < T; ++t) {
        const bool last = (t == T - 1);
        if (m > 0) {
            SpmmArgs a{};
            a.rowptr = Bt.row_ptr; a.col = Bt.col_idx; a.val = Bt.val;
            a.src = (const float4 *)Z; a.d4 = d4; a.nslices = nslices;
            a.sch = sbt.s; a.n_rows = m; a.partials = (float4 *)partials;
            a.scale = sv; a.out = (float4 *)Qv;
            a.arrive = arr_v;
            a.reserve_sms = launches < reserve_launches ? reserve_sms : 0;
            a.work = counter();
            if (grouped) {
                a.src_rows = n; a.out_rows = m; a.out_L = Lq;
                gspmm<EPI_V>(a, Lp, sbt.s.max_items, Bt.val != nullptr, st);
            } else {
                spmm_launch<EPI_V>(a, sbt.s.max_items, sbt.s.max_slots, Bt.val != nullptr, st);
            }
        } else {
            TPO_CUDA(cudaMemsetAsync(Qv, 0, sizeof(float) * 0, st));
        }
        // B's column ids may still be in flight (host inputs): nothing before the first U-side SpMM reads them
        if (t == 0 && b_cols_ready) TPO_CUDA(cudaStreamWaitEvent(st, b_cols_ready, 0));
        SpmmArgs a{};
        a.rowptr = B.row_ptr; a.col = B.col_idx; a.val = B.val;
        a.src = (const float4 *)Qv; a.d4 = d4; a.nslices = nslices;
        a.sch = sb.s; a.n_rows = n; a.partials = (float4 *)partials;
        a.scale = su; a.X = (const float4 *)X; a.c = c; a.alpha = alpha;
        a.out = (float4 *)Z;
        a.arrive = arr_u;
        a.reserve_sms = launches < reserve_launches ? reserve_sms : 0;
        a.work = counter();
        if (grouped) {
            a.src_rows = m; a.out_rows = n; a.out_L = last ? d4 : Lp;
            if (last) gspmm<EPI_FINAL>(a, Lq, sb.s.max_items, B.val != nullptr, st);
            else gspmm<EPI_U>(a, Lq, sb.s.max_items, B.val != nullptr, st);
            if (last && Zhat) {
                rownorm_kernel<<<cdiv(n * 32, TB), TB, 0, st>>>((const float4 *)Z, n, d4, (float4 *)Zhat);
                TPO_LAUNCH_CHECK();
            }
        } else if (last) {
            a.out_hat = (nslices == 1 && Zhat) ? (float4 *)Zhat : nullptr;
            spmm_launch<EPI_FINAL>(a, sb.s.max_items, sb.s.max_slots, B.val != nullptr, st);
            if (Zhat && nslices > 1) {
                rownorm_kernel<<<cdiv(n * 32, TB), TB, 0, st>>>((const float4 *)Z, n, d4, (float4 *)Zhat);
                TPO_LAUNCH_CHECK();
            }
        } else {
            spmm_launch<EPI_U>(a, sb.s.max_items, sb.s.max_slots, B.val != nullptr, st);
        }
    }
}

// ------------------------------------------------------------------------------------------
// Sharded propagation pieces (U rows split across ranks; collectives done by the caller).
// ------------------------------------------------------------------------------------------
size_t shard_spmm_ws_bytes(int64_t n_rows, int64_t nnz, int64_t d) {
    Arena ar(nullptr, 0);
    sched_alloc(ar, n_rows, nnz);
    ar.take<float>((2 * (nnz / CHUNK) + 1) * d);
    ar.take<unsigned long long>(1);
    return ar.off + 256;
}

void shard_degrees_impl(const tpo_csr_t &Bp, const tpo_csr_t &Btp, double *deg_u, double *deg_v, cudaStream_t st) {
    const int TB = 256;
    if (Bp.n_rows > 0) degree_kernel<<<cdiv(Bp.n_rows * 32, TB), TB, 0, st>>>(Bp.row_ptr, Bp.val, Bp.n_rows, deg_u);
    TPO_LAUNCH_CHECK();
    if (Btp.n_rows > 0) degree_kernel<<<cdiv(Btp.n_rows * 32, TB), TB, 0, st>>>(Btp.row_ptr, Btp.val, Btp.n_rows, deg_v);
    TPO_LAUNCH_CHECK();
}

void shard_start_impl(const double *deg_u, const double *deg_v, int64_t n_p, int64_t m, const float *Xp, int64_t d,
                      float alpha, float *s_u, float *s_v, float *Pp, cudaStream_t st) {
    const int TB = 256;
    const float c = alpha < 1.0f ? 1.0f - alpha : 1.0f;
    if (n_p > 0) inv_sqrt_kernel<<<cdiv(n_p, TB), TB, 0, st>>>(deg_u, n_p, s_u);
    TPO_LAUNCH_CHECK();
    if (m > 0) inv_sqrt_kernel<<<cdiv(m, TB), TB, 0, st>>>(deg_v, m, s_v);
    TPO_LAUNCH_CHECK();
    const int d4 = (int)(d / 4);
    if (n_p > 0) init_scaled_kernel<<<cdiv(n_p * d4, TB), TB, 0, st>>>((const float4 *)Xp, s_u, n_p, d4, c, 1, (float4 *)Pp, d4);
    TPO_LAUNCH_CHECK();
}

void shard_vside_impl(const tpo_csr_t &Btp, const float *Pp, int64_t d, float *Qpart, Arena &ar, cudaStream_t st) {
    const int64_t m = Btp.n_rows;
    if (m == 0) return;
    const int d4 = (int)(d / 4);
    SchedBufs sb = sched_alloc(ar, m, Btp.nnz);
    float *partials = ar.take<float>((2 * (Btp.nnz / CHUNK) + 1) * d);
    sched_build(sb, Btp.row_ptr, m, st);
    SpmmArgs a{};
    a.rowptr = Btp.row_ptr; a.col = Btp.col_idx; a.val = Btp.val;
    a.src = (const float4 *)Pp; a.d4 = d4; a.nslices = (d4 + 31) / 32;
    a.sch = sb.s; a.n_rows = m; a.partials = (float4 *)partials;
    a.out = (float4 *)Qpart;
    a.work = ar.take<unsigned long long>(1);
    TPO_CUDA(cudaMemsetAsync(a.work, 0, sizeof(unsigned long long), st));
    spmm_launch<EPI_RAW>(a, sb.s.max_items, sb.s.max_slots, Btp.val != nullptr, st);
}

// Row movers of the touched-row exchange: dst[i] = src[idx[i]] and
// dst[idx[i]] (+)= src[i] for d/4 float4 per row (idx unique within one call: no races).
namespace {
__global__ void rows_gather_kernel(const float4 *__restrict__ src, const int32_t *__restrict__ idx, int64_t nidx,
                                   int d4, float4 *__restrict__ dst) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nidx * d4) return;
    const int64_t r = i / d4;
    const int c = (int)(i - r * d4);
    dst[i] = src[(int64_t)idx[r] * d4 + c];
}
__global__ void rows_scatter_kernel(float4 *__restrict__ dst, const int32_t *__restrict__ idx, int64_t nidx, int d4,
                                    const float4 *__restrict__ src, int accumulate) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nidx * d4) return;
    const int64_t r = i / d4;
    const int c = (int)(i - r * d4);
    float4 *p = dst + (int64_t)idx[r] * d4 + c;
    const float4 v = src[i];
    if (accumulate) *p = f4add(*p, v);
    else *p = v;
}
}  // namespace

void rows_gather_impl(const float *src, const int32_t *idx, int64_t nidx, int64_t d, float *dst, cudaStream_t st) {
    if (nidx == 0) return;
    const int d4 = (int)(d / 4);
    rows_gather_kernel<<<cdiv(nidx * d4, 256), 256, 0, st>>>((const float4 *)src, idx, nidx, d4, (float4 *)dst);
    TPO_LAUNCH_CHECK();
}
void rows_scatter_impl(float *dst, const int32_t *idx, int64_t nidx, int64_t d, const float *src, bool accumulate,
                       cudaStream_t st) {
    if (nidx == 0) return;
    const int d4 = (int)(d / 4);
    rows_scatter_kernel<<<cdiv(nidx * d4, 256), 256, 0, st>>>((float4 *)dst, idx, nidx, d4, (const float4 *)src,
                                                               accumulate ? 1 : 0);
    TPO_LAUNCH_CHECK();
}

// T = 0 on a shard: Z = c X, Zhat = rownorm(Z) (no exchange)
void propagate_local_t0(const float *Xp, int64_t n_p, int64_t d, float alpha, float *Zp, float *Zhat_p, cudaStream_t st) {
    if (n_p == 0) return;
    const int d4 = (int)(d / 4);
    const float c = alpha < 1.0f ? 1.0f - alpha : 1.0f;
    init_scaled_kernel<<<cdiv(n_p * d4, 256), 256, 0, st>>>((const float4 *)Xp, nullptr, n_p, d4, c, 0, (float4 *)Zp, d4);
    TPO_LAUNCH_CHECK();
    if (Zhat_p) rownorm_kernel<<<cdiv(n_p * 32, 256), 256, 0, st>>>((const float4 *)Zp, n_p, d4, (float4 *)Zhat_p);
    TPO_LAUNCH_CHECK();
}

void shard_vscale_impl(float *Q, const float *s_v, int64_t rows, int64_t d, cudaStream_t st) {
    const int d4 = (int)(d / 4);
    if (rows == 0) return;
    vscale_kernel<<<cdiv(rows * d4, 256), 256, 0, st>>>((float4 *)Q, s_v, rows, d4);
    TPO_LAUNCH_CHECK();
}

void shard_uside_impl(const tpo_csr_t &Bp, const float *Q, const float *Xp, int64_t d, float alpha, const float *s_u,
                      bool last, float *Zp, float *Zhat_p, Arena &ar, cudaStream_t st) {
    const int64_t n = Bp.n_rows;
    if (n == 0) return;
    const int d4 = (int)(d / 4);
    const int nslices = (d4 + 31) / 32;
    SchedBufs sb = sched_alloc(ar, n, Bp.nnz);
    float *partials = ar.take<float>((2 * (Bp.nnz / CHUNK) + 1) * d);
    sched_build(sb, Bp.row_ptr, n, st);
    SpmmArgs a{};
    a.rowptr = Bp.row_ptr; a.col = Bp.col_idx; a.val = Bp.val;
    a.src = (const float4 *)Q; a.d4 = d4; a.nslices = nslices;
    a.sch = sb.s; a.n_rows = n; a.partials = (float4 *)partials;
    a.scale = s_u; a.X = (const float4 *)Xp; a.c = alpha < 1.0f ? 1.0f - alpha : 1.0f; a.alpha = alpha;
    a.out = (float4 *)Zp;
    a.work = ar.take<unsigned long long>(1);
    TPO_CUDA(cudaMemsetAsync(a.work, 0, sizeof(unsigned long long), st));
    if (last) {
        a.out_hat = (nslices == 1 && Zhat_p) ? (float4 *)Zhat_p : nullptr;
        spmm_launch<EPI_FINAL>(a, sb.s.max_items, sb.s.max_slots, Bp.val != nullptr, st);
        if (Zhat_p && nslices > 1) {
            rownorm_kernel<<<cdiv(n * 32, 256), 256, 0, st>>>((const float4 *)Zp, n, d4, (float4 *)Zhat_p);
            TPO_LAUNCH_CHECK();
        }
    } else {
        spmm_launch<EPI_U>(a, sb.s.max_items, sb.s.max_slots, Bp.val != nullptr, st);
    }
}

}  // namespace tpo
