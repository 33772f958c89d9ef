// Internal helpers of libtpo (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <exception>
#include <string>

#include "../../include/tpo.h"

namespace tpo {

// Thread-local last error message (the only global mutable state of the library).
void set_error(const std::string &msg);

struct Error : public std::exception {
    int code;
    std::string msg;
    Error(int c, std::string m) : code(c), msg(std::move(m)) {}
    const char *what() const noexcept override { return msg.c_str(); }
};

#define TPO_REQUIRE(cond, msg)                                                   \
    do {                                                                         \
        if (!(cond)) throw ::tpo::Error(TPO_EINVAL, std::string(__func__) + ": " + (msg)); \
    } while (0)

#define TPO_CUDA(call)                                                           \
    do {                                                                         \
        cudaError_t _e = (call);                                                 \
        if (_e != cudaSuccess)                                                   \
            throw ::tpo::Error(TPO_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

// Every kernel launch is followed by TPO_LAUNCH_CHECK(), which also counts it (thread-local
// counter read by tpo_launch_count(); used by bench.py's gpu_launches).
void count_launch();
#define TPO_LAUNCH_CHECK()            \
    do {                              \
        ::tpo::count_launch();        \
        TPO_CUDA(cudaGetLastError()); \
    } while (0)

// Runs f(); converts exceptions into TPO error codes + the last-error message.
template <class F>
int guarded(F &&f) {
    try {
        f();
        return TPO_OK;
    } catch (const Error &e) {
        set_error(e.msg);
        return e.code;
    } catch (const std::exception &e) {
        set_error(std::string("internal: ") + e.what());
        return TPO_ECUDA;
    } catch (...) {
        set_error("internal: unknown exception");
        return TPO_ECUDA;
    }
}

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Bump allocator over the caller's workspace.
struct Arena {
    char *base;
    size_t cap, off = 0;
    bool dry;                       // dry run: only measures
    Arena(void *b, size_t c) : base(static_cast<char *>(b)), cap(c), dry(b == nullptr) {}
    template <class T>
    T *take(size_t count) {
        size_t bytes = align_up(count * sizeof(T) + 1);
        size_t at = off;
        off += bytes;
        if (dry) return nullptr;
        if (off > cap) throw Error(TPO_ENOMEM, "workspace too small: need at least " + std::to_string(off) + " bytes");
        return reinterpret_cast<T *>(base + at);
    }
};

inline cudaStream_t as_stream(void *s) { return static_cast<cudaStream_t>(s); }

int sm_count();

// ----------------------------------------------------------------------------------------
// Module entry points (implemented in the .cu files; called by tpo_api.cu)
// ----------------------------------------------------------------------------------------
// reserve_sms: SMs the persistent SpMM grids of the first reserve_launches SpMM launches leave
// free (tpo_run keeps some for the Haar rotation running beside the propagation on a side stream).
void propagate_impl(const tpo_csr_t &B, const tpo_csr_t &Bt, const float *X, int64_t d, float alpha,
                    int32_t T, float *Z, float *Zhat, Arena &ar, cudaStream_t st, int reserve_sms = 0,
                    int reserve_launches = 1 << 30, cudaEvent_t b_cols_ready = nullptr);
// sharded propagation pieces (spmm.cu)
size_t shard_spmm_ws_bytes(int64_t n_rows, int64_t nnz, int64_t d);
void propagate_local_t0(const float *Xp, int64_t n_p, int64_t d, float alpha, float *Zp, float *Zhat_p, cudaStream_t st);
// library-owned NCCL communicator (comm.cu)
void comm_unique_id(void *id);
void *comm_create(const void *id, int rank, int world, int device);
void comm_destroy(void *comm);
int comm_world(const void *comm);
int comm_rank(const void *comm);
size_t propagate_sharded_ws_bytes(int64_t n_p, int64_t m, int64_t nnz_p, int64_t d, int world);
void propagate_sharded_impl(void *comm, const tpo_csr_t &Bp, const tpo_csr_t &Btp, const float *Xp, int64_t d,
                            float alpha, int32_t T, float *Zp, float *Zhat_p, Arena &ar, cudaStream_t st);
size_t run_sharded_ws_bytes(int64_t n_p, int64_t m, int64_t nnz_p, int64_t d, int32_t k, int world);
void run_sharded_impl(void *comm, const tpo_csr_t &Bp, const tpo_csr_t &Btp, const float *Xp, int64_t d, float alpha,
                      int32_t T, int32_t k, const double *Gdev, int64_t row0, int32_t Tf, int32_t Tg, int32_t *labels_p,
                      int32_t *iters_used, double *timings_ms, Arena &ar, cudaStream_t st);
void shard_degrees_impl(const tpo_csr_t &Bp, const tpo_csr_t &Btp, double *deg_u, double *deg_v, cudaStream_t st);
void shard_start_impl(const double *deg_u, const double *deg_v, int64_t n_p, int64_t m, const float *Xp, int64_t d,
                      float alpha, float *s_u, float *s_v, float *Pp, cudaStream_t st);
void shard_vside_impl(const tpo_csr_t &Btp, const float *Pp, int64_t d, float *Qpart, Arena &ar, cudaStream_t st);
void shard_vscale_impl(float *Q, const float *s_v, int64_t rows, int64_t d, cudaStream_t st);
void shard_uside_impl(const tpo_csr_t &Bp, const float *Q, const float *Xp, int64_t d, float alpha, const float *s_u,
                      bool last, float *Zp, float *Zhat_p, Arena &ar, cudaStream_t st);
// rowE / featmax (optional, both or neither): R''s row exponents and per-feature maxima (see
// oz_rstats), formed in the dinv pass when D % 32 == 0 and D <= 512
// s_out (optional, with rowE / featmax): s = sum_i dinv_i R'[i] (D fp64); NaN-filled when not formed
void features_impl(const float *Zhat, int64_t n, int64_t d, const float *Q, float *Rp, float *dinv,
                   double *r_out, Arena &ar, cudaStream_t st, int32_t *rowE = nullptr, uint32_t *featmax = nullptr,
                   double *s_out = nullptr);
void affinity_matvec_impl(const float *Rp, const float *dinv, int64_t n, int64_t D, const float *Y,
                          int64_t b, float *out, Arena &ar, cudaStream_t st);
// Per-R' statistics of the integer-tensor-core products (oz.cu), computed once per R' inside
// tpo_run and shared by the top-k (Gamma = R Psi Sigma^-1) and the discretisation (RH, R^T Ups):
// rowE[i] = row exponents of R', featmax[j] = bits of max_i |R'_ij|; NULL members: not computed.
struct RStats {
    const int32_t *rowE = nullptr;
    const uint32_t *featmax = nullptr;
    const double *s_colsum = nullptr;   // s = sum_i dinv_i R'[i] = 1^T R (D fp64): a7's sign rule from D-space
};
// one pass over R' for both (rowE: n, featmax: D); only when k > 32 and D <= 512
bool oz_rstats_wanted(int64_t n, int64_t D, int k);
void oz_rstats(const float *Rp, int64_t n, int64_t D, int32_t *rowE, uint32_t *featmax, cudaStream_t st);
// r_colsum: r = sum_i R'[i] (2d fp64, device) from tpo_features, or NULL to recompute it.
void topk_eig_impl(const float *Rp, const float *dinv, int64_t n, int64_t D, int32_t k, int32_t mode,
                   int32_t p, int32_t q, const float *Omega, float *Gamma, double *sigma, float *Psi,
                   Arena &ar, cudaStream_t st, const double *r_colsum = nullptr, RStats rs = RStats());
void colsum_f64(const float *Rp, int64_t n, int64_t D, double *r, Arena &ar, cudaStream_t st);
size_t features_ws_bytes(int64_t n, int64_t d);
// f3 "R-free": R' rows recomputed from Zhat (Eq. R-prime) in chunks of `chunk`
// rows wherever a pass needs them, instead of a materialised n x 2d R'
struct RSource {
    const float *Zhat = nullptr;   // n x d fp32
    int64_t d = 0;
    const float *Q = nullptr;      // d x d fp32 (the Haar rotation)
    int64_t chunk = 0;
};
size_t rfree_pass_ws(int64_t n, int64_t d, int32_t k, int64_t chunk);
void cluster_impl(const float *Rp, const float *dinv, int64_t n, int64_t D, int32_t k, const float *Gamma,
                  const double *sigma, const float *Psi, int32_t Tf, int32_t Tg, int32_t *labels,
                  int32_t *iters_used, Arena &ar, cudaStream_t st, RStats rs = RStats(),
                  const RSource *src = nullptr);
// f3 a7: the exact top-k with R' recomputed from Zhat (sweeps: r, then dinv and the Gram, then Gamma)
size_t topk_rfree_ws(int64_t n, int64_t d, int32_t k, int64_t chunk);
void topk_rfree_impl(const RSource &src, int64_t n, int32_t k, float *Gamma, double *sigma, float *Psi, float *dinv,
                     Arena &ar, cudaStream_t st);

// G: d x d fp64, on the device when G_on_device, else host memory
void haar_q_device(const double *G, bool G_on_device, int64_t d, float *Q_out, Arena &ar, cudaStream_t st);

// Pieces of a5-a9 for the row-sharded solver (the caller all-reduces the
// partials between them).  features.cu:
void features_part(const float *Zhat, int64_t n, int64_t d, const float *Q, float *Rp, double *r_part, Arena &ar,
                   cudaStream_t st);
void dinv_from_r(const float *Rp, int64_t n, int64_t D, const double *r, float *dinv, cudaStream_t st);
// eig.cu: top-k of a given (global) Gram; Gamma pieces on the shard's rows
void eig_from_gram(const double *G, const double *r, int64_t D, int32_t k, double *Psi64, double *sigma, Arena &ar,
                   cudaStream_t st);
size_t eig_from_gram_ws(int64_t D, int32_t k);
void gamma_rows(const float *Rp, const float *dinv, int64_t n, int64_t D, int k, const double *Psi64,
                const double *sigma, double *G64, Arena &ar, cudaStream_t st);
void apply_chol(double *X, int64_t n, int k, const double *g, Arena &ar, cudaStream_t st);
void colstats_rows(const double *A, int64_t n, int k, int64_t row0, double *sum, double *abs_sum, double *maxabs,
                   int64_t *argmax, Arena &ar, cudaStream_t st);
void gamma_final(double *G64, int64_t n, int k, const int *signs_host, float *Psi, const double *Psi64, int64_t D,
                 float *Gamma, Arena &ar, cudaStream_t st);
// cluster.cu
void onmf_init(const float *Gamma, int64_t n, const float *Psi, const double *sigma_host, int64_t D, int k, double *U,
               double *H, Arena &ar, cudaStream_t st);
void onmf_h_update(double *H, const double *RtU, const double *UtU, int64_t D, int k, Arena &ar, cudaStream_t st);
void onmf_u_update(double *U, const double *RH, const double *M, int64_t n, int k, cudaStream_t st);
void nci_assign_part(const double *U, const double *Phi, int64_t n, int k, int32_t *labels, int32_t *changed,
                     double *sums, double *counts, Arena &ar, cudaStream_t st);
size_t nci_assign_part_ws(int64_t n, int k);
void nci_phi(const double *sums, const double *counts, int k, double *Phi, cudaStream_t st);
size_t haar_q_ws_bytes(int64_t d);
// touched-row exchange row movers (spmm.cu)
void rows_gather_impl(const float *src, const int32_t *idx, int64_t nidx, int64_t d, float *dst, cudaStream_t st);
void rows_scatter_impl(float *dst, const int32_t *idx, int64_t nidx, int64_t d, const float *src, bool accumulate,
                       cudaStream_t st);
// f4 evaluation and monitors (eval.cu)
size_t eval_ws_bytes(int32_t ka, int32_t kb);
void eval_impl(const int32_t *pred, const int32_t *truth, int64_t n, int32_t ka, int32_t kb, double *metrics, Arena &ar,
               cudaStream_t st);
size_t objective_ws_bytes(int64_t n, int64_t D, int32_t k);
void objective_impl(const float *Rp, const float *dinv, int64_t n, int64_t D, int32_t k, const int32_t *labels,
                    const double *Ups, double *out, Arena &ar, cudaStream_t st);
// f1 SVD attribute reduction (eig.cu)
size_t svd_reduce_ws_bytes(int64_t n, int64_t du, int64_t d);
void svd_reduce_impl(const float *X, int64_t n, int64_t du, int64_t d, float *Xr, double *sigma_host, Arena &ar,
                     cudaStream_t st);

// ----------------------------------------------------------------------------------------
// Dense building blocks (dense.cu)
// ----------------------------------------------------------------------------------------
// out[p x q] (fp64, device) = sum_i (rs[i] * A[i, :])^T B[i, :], A fp32 n x p (lda), B fp32 or
// fp64 n x q; deterministic split over rows with a fixed-order fp64 reduction.
void tsgemm_AtB_f32f32(const float *A, int64_t lda, const float *rsA, const float *Bm, int64_t ldb,
                       const float *rsB, int64_t n, int64_t p, int64_t q, double *out, Arena &ar,
                       cudaStream_t st);
void tsgemm_AtB_f32f64(const float *A, int64_t lda, const float *rsA, const double *Bm, int64_t ldb,
                       int64_t n, int64_t p, int64_t q, double *out, Arena &ar, cudaStream_t st);
void tsgemm_AtB_f64f64(const double *A, int64_t lda, const double *Bm, int64_t ldb, int64_t n, int64_t p,
                       int64_t q, double *out, Arena &ar, cudaStream_t st);
// Out[n x q] = rs[i] * (A[i, :] W) with A fp32 n x p, W fp64 p x q; output fp32 or fp64.
void tsgemm_AW_f32(const float *A, int64_t lda, const float *rs, const double *W, int64_t n, int64_t p,
                   int64_t q, float *out, int64_t ldo, cudaStream_t st);
void tsgemm_AW_f64(const float *A, int64_t lda, const float *rs, const double *W, int64_t n, int64_t p,
                   int64_t q, double *out, int64_t ldo, cudaStream_t st);
void tsgemm_AW_dd(const double *A, int64_t lda, const double *W, int64_t n, int64_t p, int64_t q, double *out,
                  int64_t ldo, cudaStream_t st);
// Symmetric Gram G = sum_i w_i^2 A[i]^T A[i] (D x D fp64, full matrix written).
// tcgen05 3xTF32 Gram with fp64 segment accumulation (gram_tc.cu).
void gram_tc(const float *Rp, const float *dinv, int64_t n, int64_t D, double *G, Arena &ar, cudaStream_t st);
size_t gram_tc_ws(int64_t n, int64_t D);
// R' = sqrt(e/d) (sin || cos)(sqrt(d) Zhat Q^T) on tcgen05 (3xTF32), R' only (gram_tc.cu).
void features_tc(const float *Zhat, int64_t n, int64_t d, const float *Q, float *Rp, Arena &ar, cudaStream_t st);
size_t features_tc_ws(int64_t n, int64_t d);
size_t tsgemm_ws(int64_t n, int64_t p, int64_t q);
// fp64 C = beta C + alpha op(A) B (row-major; op(A) = A^T when transA, A is then K x M);
// deterministic split-K (dgemm.cu).  Workspace <= dgemm_ws(M, N, K).
void dgemm(bool transA, int64_t M, int64_t N, int64_t K, double alpha, const double *A, int64_t lda,
           const double *B, int64_t ldb, double beta, double *C, int64_t ldc, Arena &ar, cudaStream_t st);
size_t dgemm_ws(int64_t M, int64_t N, int64_t K);
// ONMF passes over R' (onmf.cu): RtU = R'^T (dinv . U) (D x k), fp64 (RH = dinv . (R' H) is tsgemm_AW_f64).
void onmf_rtu(const float *Rp, int64_t n, int64_t D, const float *dinv, const double *U, int k, double *RtU,
              Arena &ar, cudaStream_t st, const uint32_t *featmax = nullptr,
              const unsigned long long *colmax = nullptr);
size_t onmf_ws_bytes(int64_t n, int64_t D, int32_t k);
// fp64 tensor-path (DMMA) products of the discretisation (ts64.cu).  ts64_enabled(): TPO_TS64=0
// selects the CUDA-core kernels of dense.cu / onmf.cu / cluster.cu (A/B measurement only).
bool ts64_enabled();
// the DMMA Ups update (den = Ups M, resident M, bulk-copied Ups / RH tiles): even 16 < k <= 104
bool ts64_ups_enabled(int k);
size_t ts_atb_ws(int p, int q);
void ts_assign(const double *U, const double *Phi, int64_t n, int k, int32_t *labels, int32_t *changed,
               const int32_t *done, cudaStream_t st);
// out (p x q) = A^T B for n x p / n x q fp64 A, B (p, q <= 104) on the fp64 tensor path
void ts_atb_f64(const double *A, int64_t lda, const double *B, int64_t ldb, int64_t n, int p, int q, double *out,
                Arena &ar, cudaStream_t st);
// fp64-accurate out = diag(rs) A W on the integer tensor cores (oz.cu; Ozaki digit splitting):
// A n x K fp32 (lda % 4 == 0, 16-byte aligned), W K x N fp64, out n x N fp64; N <= 64 and the
// digit image of W (7 x N x K bytes) <= 112 KB.  rowE = oz_rowexp(A) (per-row exponents).
bool oz_enabled();
bool oz_aw_supported(int64_t K, int N);
size_t oz_aw_ws(int64_t K, int N);
void oz_rowexp(const float *A, int64_t lda, int64_t n, int K, int32_t *E, cudaStream_t st);
void oz_aw_f64(const float *A, int64_t lda, const float *rs, const int32_t *rowE, const double *W, int64_t n, int K,
               int N, double *out, int64_t ldo, Arena &ar, cudaStream_t st);
// Alg. 2's RtU = R'^T (dinv . Ups) (D x k fp64) on the integer tensor cores (oz.cu), 32 < k <= 64:
// featmax = bits of R''s per-feature max |R'| (oz_featmax, once per solve).
bool oz_rtu_supported(int64_t n, int64_t D, int k);
size_t oz_rtu_ws(int64_t n, int64_t D, int k);
void oz_featmax(const float *Rp, int64_t n, int64_t D, uint32_t *featmax, cudaStream_t st);
// colmax_pre (optional): bits of max_i dinv_i U_il already formed (the Ups update's fused maxima)
void oz_rtu(const float *Rp, int64_t n, int64_t D, const float *dinv, const double *U, int k, const uint32_t *featmax,
            double *RtU, Arena &ar, cudaStream_t st, const unsigned long long *colmax_pre = nullptr);
// Alg. 3 assignment on the integer tensor cores (oz.cu), 32 < k <= 64: Ups digits prepared once
// per solve (Ups is fixed during Alg. 3), then one certified argmax per iteration.
struct OzAssign {
    int64_t n = 0;
    int k = 0, NP = 0, Kp = 0;
    uint8_t *Ud = nullptr, *Bimg = nullptr;
    int32_t *rowE = nullptr, *colE = nullptr;
};
bool oz_assign_supported(int k);
size_t oz_assign_ws(int64_t n, int k);
OzAssign oz_assign_prepare(const double *U, int64_t n, int k, Arena &ar, cudaStream_t st);
void oz_assign(const OzAssign &p, const double *U, const double *Phi, int32_t *labels, int32_t *changed,
               const int32_t *done, cudaStream_t st);
struct RhPlan {
    bool oz = false;
    int32_t *rowE = nullptr;
};
RhPlan rh_plan(const float *Rp, int64_t n, int64_t D, int k, Arena &ar, cudaStream_t st);
RhPlan rh_plan_at(int32_t *rowE, const float *Rp, int64_t n, int64_t D, int k, cudaStream_t st);
// the plan with precomputed row exponents (oz_rstats), or computed into the arena when NULL
RhPlan rh_plan_pre(const int32_t *rowE, const float *Rp, int64_t n, int64_t D, int k, Arena &ar, cudaStream_t st);
size_t rh_plan_ws(int64_t n);
size_t rh_apply_ws(int64_t D, int k);
void rh_apply(const RhPlan &p, const float *Rp, const float *dinv, const double *H, int64_t n, int64_t D, int k,
              double *RH, Arena &ar, cudaStream_t st);
void ts_aw_f64(const float *A, int64_t lda, const float *rs, const double *W, int64_t n, int K, int N,
               const double *cs, double *out, int64_t ldo, cudaStream_t st);
void ts_ups_update(double *U, const double *RH, const double *M, int64_t n, int k, cudaStream_t st);
bool ts_xw_inplace_f64(double *X, int64_t n, int k, const double *W, cudaStream_t st);
bool ts_xw_f64(const double *X, int64_t n, int k, const double *W, double *out, cudaStream_t st);
bool ts_xw_f32out(const double *X, int64_t n, int k, const double *W, float *out32, cudaStream_t st);
size_t ts_rtu_ws(int64_t n, int64_t D, int k);
size_t ts_affinity_ws(int64_t D, int64_t b);
size_t ts_affinity_rfree_ws(int64_t n, int64_t d, int64_t b, int64_t chunk);
void ts_affinity_rfree(const float *Zhat, int64_t n, int64_t d, const float *Q, const float *Y, int64_t b, float *out,
                       int64_t chunk, Arena &ar, cudaStream_t st);
void ts_affinity(const float *Rp, const float *dinv, int64_t n, int64_t D, const float *Y, int64_t b, float *out,
                 Arena &ar, cudaStream_t st);
void ts_rtu(const float *Rp, int64_t n, int64_t D, const float *dinv, const double *U, int k, double *RtU, Arena &ar,
            cudaStream_t st);

// Ci = S C^{-1} for the b x b Gram g (S g S = C^T C, S = diag(g)^{-1/2}), b <= 128; one CTA;
// a failed pivot sets *flag (device int) instead of throwing (dgemm.cu).
void chol_inv_device(const double *g, int64_t b, double *Ci, int *flag, cudaStream_t st);

// ----------------------------------------------------------------------------------------
// Host fp64 dense linear algebra (host_linalg.cpp)
// ----------------------------------------------------------------------------------------
void host_qr_positive(int64_t rows, int64_t cols, const double *A, double *Q, double *R);
// Symmetric eigendecomposition: all eigenvalues (descending) in w, the eigenvectors of the
// top `nvec` eigenvalues in the columns of V (D x nvec, row-major).
void host_sym_eig_top(int64_t D, const double *A, int64_t nvec, double *w, double *V);
// Cholesky A = C^T C (upper C), returns false if not SPD.
bool host_cholesky_upper(int64_t k, const double *A, double *C);
// Inverse of an upper-triangular matrix.
void host_upper_inverse(int64_t k, const double *C, double *Ci);

}  // namespace tpo
