/*
 * tpo.h -- C-ABI of libtpo, the B200 (sm_100a) implementation of the TPO hot path
 * ("Effective Clustering on Large Attributed Bipartite Graphs", arXiv 2405.11922).
 *
 * Citations are PAPER.md line numbers of the paper's LaTeX source plus the equation /
 * algorithm label; "R<n>" names a reading of a silent or garbled passage listed in
 * DESIGN.md ("Readings").
 *
 * Conventions for every entry point
 * ---------------------------------
 *  - Pointers are DEVICE pointers unless marked (host).  Dense matrices are row-major.
 *    Dense float/double device buffers must be 16-byte aligned.
 *  - Ownership: the caller allocates and owns every buffer; the library never frees
 *    caller memory and keeps no pointer after a call returns.  The only objects the
 *    library owns are the opaque communicator handles of tpo_comm_create (freed by
 *    tpo_comm_destroy).
 *  - Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Calls enqueue on it and return without synchronising, except those marked [sync],
 *    which copy small fp64 matrices to the host, factor them there and copy back; [sync]
 *    calls return after their work has completed.
 *  - Workspace: calls that take (ws, ws_bytes) have a size query tpo_<name>_ws(...);
 *    a smaller ws_bytes returns TPO_ENOMEM.  ws must be 256-byte aligned.
 *  - Errors: the int return is 0 (TPO_OK) or a negative TPO_E* code; no C++ exception
 *    crosses the ABI.  tpo_last_error() returns a thread-local message describing the
 *    last failure.  On error the contents of output buffers are unspecified.
 *  - Determinism: no floating-point atomics; every cross-thread reduction has a fixed
 *    order, so identical inputs give bitwise-identical outputs on the same GPU model.
 *  - Thread safety: concurrent calls on different streams with disjoint buffers are
 *    allowed; the only global mutable state is thread-local (last-error slot, launch count).
 */
#ifndef TPO_H
#define TPO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TPO_ABI_VERSION 1

enum {
    TPO_OK = 0,
    TPO_EINVAL = -1,    /* bad shape, null pointer, range, alignment, unknown mode       */
    TPO_ECUDA = -2,     /* a CUDA runtime call or kernel launch failed                     */
    TPO_ENOMEM = -3,    /* ws_bytes below the size query                                   */
    TPO_ENCCL = -4,     /* an NCCL call failed (multi-GPU entry points)                    */
    TPO_ENUMERIC = -5   /* non-SPD Gram in CholeskyQR, zero singular value, non-finite     */
};

/* Sparse bipartite adjacency B_U or its transpose, in CSR.
 * row_ptr: int64 [n_rows+1] (device), monotone, row_ptr[0] = 0, row_ptr[n_rows] = nnz;
 * col_idx: int32 [nnz] (device), each < n_cols; val: fp32 [nnz] (device) non-negative edge
 * weights w(u_i, v_j), or NULL for unit weights.  Duplicate (row, col) pairs must have
 * been merged by the caller. */
typedef struct tpo_csr {
    int64_t n_rows, n_cols, nnz;
    const int64_t *row_ptr;
    const int32_t *col_idx;
    const float *val;
} tpo_csr_t;

int tpo_abi_version(void);
const char *tpo_last_error(void);
/* Number of CUDA kernels this library has launched from the calling host thread (monotone
 * thread-local counter; for launch accounting in benchmarks). */
uint64_t tpo_launch_count(void);

/* ---------------------------------------------------------------------------------------
 * a1-a3  MSA propagation.  Lemma 1 / Eq. PX truncated at gamma = T
 * hops, with L = D_U^{-1/2} B D_V^{-1/2} (Eq. L) and the
 * hop update of Eq. update-Z bracketed as L (L^T Z):
 *      Z_0 = c X ;   Z <- c X + alpha * L (L^T Z)   (T times),   c = 1 - alpha  (R1;
 *      c = 1 when alpha = 1), then Zhat[i] = Z[i] / ||Z[i]|| (Eq. Z),
 *      zero rows stay zero (R4).  D_U, D_V are the weighted degrees,
 *      1/sqrt(0) := 0 (R3).
 *   B  : n_u x n_v CSR;  Bt: the same edges as an n_v x n_u CSR (B^T).
 *   X  : n_u x d fp32 (input, not modified).  d >= 4, d % 4 == 0.
 *   Z  : n_u x d fp32 out (raw Z, prefactor c); also used as the iterate in place.
 *   Zhat: n_u x d fp32 out, or NULL.
 *   alpha in [0, 1], T >= 0.
 * Workspace: tpo_propagate_ws(n_u, n_v, nnz, d).
 * Errors: TPO_EINVAL (shapes of B/Bt/X disagree, Bt.nnz != B.nnz, alpha/T/d out of range,
 * null or misaligned pointers, max(n_u, n_v) * d/4 >= 2^32: the SpMM gathers use 32-bit row
 * offsets), TPO_ENOMEM, TPO_ECUDA.
 * --------------------------------------------------------------------------------------- */
size_t tpo_propagate_ws(int64_t n_u, int64_t n_v, int64_t nnz, int64_t d);
int tpo_propagate(const tpo_csr_t *B, const tpo_csr_t *Bt, const float *X, int64_t d,
                  float alpha, int32_t T, float *Z, float *Zhat,
                  void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------------------
 * a1-a3 sharded across GPUs (one process per GPU).  The rank owns the
 * contiguous U slice [u0, u1) (n_p rows): Bp = those rows of B (global V column ids) and
 * Btp = Bp^T (m x n_p, local U column ids).  The CALLER runs the collectives:
 *    deg_v <- all-reduce(sum) of the shard partials        (once)
 *    per hop:  Qpart = tpo_shard_vside(Btp, P)              (m x d, raw sums B_p^T P_p)
 *              Qslice = reduce-scatter(sum) of Qpart over V
 *              tpo_shard_vscale(Qslice, s_v slice)          (Q[v] *= s_v[v]^2)
 *              Q = all-gather(Qslice)                        (m x d)
 *              tpo_shard_uside(Bp, Q, ...)                   (P, or Z and Zhat at the last hop)
 * which reproduces tpo_propagate on the full graph (the sum of the shard partials of
 * B^T (s_u . Z) over ranks is the full product).  T = 0 needs no exchange: Z = (1-alpha) X.
 *   tpo_shard_degrees: deg_u (n_p fp64 out) weighted row sums of Bp; deg_v (m fp64 out) the
 *     shard's partial V degrees (row sums of Btp).
 *   tpo_shard_start: s_u = deg_u^-1/2, s_v = deg_v^-1/2 (global deg_v; 1/sqrt(0) := 0), fp32;
 *     Pp = s_u . (1 - alpha) Xp (n_p x d), the pre-scaled iterate.
 *   tpo_shard_uside: last = 0 -> Zp <- P = s_u . (c Xp + alpha s_u . B_p Q);
 *     last = 1 -> Zp <- Z = c Xp + alpha s_u . B_p Q, Zhat_p <- rownorm(Z) (may be NULL).
 * Workspace of vside / uside: tpo_shard_ws(rows of the CSR, nnz, d).
 * --------------------------------------------------------------------------------------- */
size_t tpo_shard_ws(int64_t n_rows, int64_t nnz, int64_t d);
int tpo_shard_degrees(const tpo_csr_t *Bp, const tpo_csr_t *Btp, double *deg_u, double *deg_v,
                      void *stream);
int tpo_shard_start(const double *deg_u, const double *deg_v, int64_t n_p, int64_t m, const float *Xp,
                    int64_t d, float alpha, float *s_u, float *s_v, float *Pp, void *stream);
int tpo_shard_vside(const tpo_csr_t *Btp, const float *Pp, int64_t d, float *Qpart, void *ws,
                    size_t ws_bytes, void *stream);
int tpo_shard_vscale(float *Q, const float *s_v, int64_t rows, int64_t d, void *stream);
int tpo_shard_uside(const tpo_csr_t *Bp, const float *Q, const float *Xp, int64_t d, float alpha,
                    const float *s_u, int32_t last, float *Zp, float *Zhat_p, void *ws,
                    size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------------------
 * Touched-row exchange of the sharded propagation: instead of reduce-scattering
 * and all-gathering the whole m x d V-side block, rank p sends only the rows of V its U slice
 * touches (the non-empty rows of Btp) to their owners and receives back only those rows of Q;
 * the caller runs the all-to-all exchanges (NCCL / gloo) and these row movers pack / unpack them.
 *   tpo_rows_gather:  dst[i] = src[idx[i]]            (nidx rows of d floats)
 *   tpo_rows_scatter: dst[idx[i]] = src[i], or += when accumulate != 0; idx must not repeat
 *                     within one call (the caller adds the ranks' blocks one call at a time, in
 *                     rank order: a fixed summation order).
 * d % 4 == 0; src / dst 16-byte aligned device pointers; idx device int32.  Errors: TPO_EINVAL.
 * --------------------------------------------------------------------------------------- */
int tpo_rows_gather(const float *src, const int32_t *idx, int64_t nidx, int64_t d, float *dst, void *stream);
int tpo_rows_scatter(float *dst, const int32_t *idx, int64_t nidx, int64_t d, const float *src, int32_t accumulate,
                     void *stream);

/* ---------------------------------------------------------------------------------------
 * Library-owned NCCL communicator and the sharded propagation with its
 * collectives inside the library (§8e).  NCCL is resolved at run time (libnccl.so.2, e.g. the copy
 * PyTorch loaded); TPO_ENCCL when it is unavailable or a call fails.
 *   tpo_comm_unique_id: (host) 128-byte ncclUniqueId out (rank 0 creates it and shares it).
 *   tpo_comm_create:    one communicator per rank on `device`; *comm is an opaque handle owned by
 *                       the library until tpo_comm_destroy.
 *   tpo_propagate_sharded: a1-a3 for the rank's U slice (Bp = its rows of B with global V ids,
 *                       Btp = Bp^T with local U ids, Xp its rows of X) on `stream`: all-reduce of the
 *                       V degrees, then per hop B_p^T P_p -> ncclReduceScatter over V slices ->
 *                       s_v^2 -> ncclAllGather -> U side; Zp (n_p x d) raw Z, Zhat_p rownorm or NULL.
 *                       The same result as tpo_propagate on the whole graph.  Workspace:
 *                       tpo_propagate_sharded_ws(n_p, n_v, nnz_p, d, world).
 * --------------------------------------------------------------------------------------- */
int tpo_comm_unique_id(void *id);
int tpo_comm_create(const void *id, int32_t rank, int32_t world, int32_t device, void **comm);
int tpo_comm_destroy(void *comm);
size_t tpo_propagate_sharded_ws(int64_t n_p, int64_t n_v, int64_t nnz_p, int64_t d, int32_t world);
int tpo_propagate_sharded(void *comm, const tpo_csr_t *Bp, const tpo_csr_t *Btp, const float *Xp, int64_t d, float alpha,
                          int32_t T, float *Zp, float *Zhat_p, void *ws, size_t ws_bytes, void *stream);
/* tpo_run_sharded: the whole hot path (as tpo_run) on the rank's U slice [row0, row0 + n_p) with every
 * collective inside the library: the sharded propagation, then features, the exact top-k, ONMF and
 * NCI with the fp64 partials all-reduced in between (r, the Gram, Gamma^T Gamma and the polish
 * decision, the sign rule's column statistics and largest entries, R'^T Ups, Ups^T Ups, Ups^T RH,
 * the cluster sums, counts and changed flag), so every rank's replicated factors are identical and
 * its labels are the single-GPU path's.  G: d x d fp64 (device), the same on every rank.
 * labels_p: n_p int32 out; iters_used: (host) Alg. 3 iterations or NULL; timings_ms: (host) 4
 * stage times {propagate, features, topk, cluster} or NULL.  [sync]
 * Workspace: tpo_run_sharded_ws(n_p, n_v, nnz_p, d, k, world). */
size_t tpo_run_sharded_ws(int64_t n_p, int64_t n_v, int64_t nnz_p, int64_t d, int32_t k, int32_t world);
int tpo_run_sharded(void *comm, const tpo_csr_t *Bp, const tpo_csr_t *Btp, const float *Xp, int64_t d, float alpha,
                    int32_t T, int32_t k, const double *G, int64_t row0, int32_t Tf, int32_t Tg, int32_t *labels_p,
                    int32_t *iters_used, double *timings_ms, void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------------------
 * a4  Haar rotation, Alg. 1 L6-7: Q = the Q factor of the QR
 * decomposition of the d x d Gaussian matrix G, sign-fixed so that diag(R) > 0, which
 * makes Q Haar-distributed and unique.  Host-only, fp64.
 *   G: (host) d x d fp64 in;  Q: (host) d x d fp64 out.  Errors: TPO_EINVAL.
 * --------------------------------------------------------------------------------------- */
int tpo_haar_q(const double *G, int64_t d, double *Q);
/* The same factor computed on the device (block Gram-Schmidt with re-orthogonalisation over
 * 112-column panels, each panel by CholeskyQR2; the QR with diag(R) > 0 is unique, so this is
 * the Q of tpo_haar_q up to rounding), written as fp32 for tpo_features.
 *   G: (host) d x d fp64;  Q: d x d fp32 out (device).  [sync].
 * Workspace: tpo_haar_q_dev_ws(d).  Errors: TPO_EINVAL, TPO_ENOMEM, TPO_ECUDA, TPO_ENUMERIC. */
size_t tpo_haar_q_dev_ws(int64_t d);
int tpo_haar_q_dev(const double *G, int64_t d, float *Q, void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------------------
 * a5  Random features (Alg. 1 L8-9; Eq. R-prime; Eq. Ri 466-468):
 *      Zo = sqrt(d) * Zhat * Q^T ;  R' = sqrt(e/d) * ( sin(Zo) || cos(Zo) )   (n x 2d,
 *      sin in columns [0,d), cos in [d,2d));  r = sum_i R'[i] (fp64);
 *      dinv[i] = 1 / sqrt(max(R'[i] . r, 1e-12))   (R6)     so that R = diag(dinv) R'.
 *   Zhat: n x d fp32, d % 4 == 0;  Q: d x d fp32 (from tpo_haar_q);  Rp: n x 2d fp32 out;
 *   The GEMM Zhat Q^T runs on tcgen05 with 3xTF32 splitting (fp32-accurate products).
 *   dinv: n fp32 out;  r_out: 2d fp64 out (device) or NULL.
 * Workspace: tpo_features_ws(n, d).  Errors: TPO_EINVAL, TPO_ENOMEM, TPO_ECUDA.
 * --------------------------------------------------------------------------------------- */
size_t tpo_features_ws(int64_t n, int64_t d);
int tpo_features(const float *Zhat, int64_t n, int64_t d, const float *Q, float *Rp,
                 float *dinv, double *r_out, void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------------------
 * a6  Implicit affinity product: out = S~ Y with S~ = R R^T = diag(dinv) R' R'^T diag(dinv)
 * (R R^T approximates the MSA matrix S, Theorem 1); evaluated as
 * dinv . (R' (R'^T (dinv . Y))) so the n x n matrix is never formed.
 *   Rp: n x D fp32;  dinv: n fp32;  Y: n x b fp32;  out: n x b fp32 out (may not alias Y).
 *   Both products run on the fp64 tensor path (DMMA); the D x b intermediate R'^T (dinv . Y) is
 *   fp64 and reduced across the GPU in a fixed order.
 * Workspace: tpo_affinity_matvec_ws(n, D, b).  Errors: TPO_EINVAL, TPO_ENOMEM, TPO_ECUDA.
 * --------------------------------------------------------------------------------------- */
size_t tpo_affinity_matvec_ws(int64_t n, int64_t D, int64_t b);
int tpo_affinity_matvec(const float *Rp, const float *dinv, int64_t n, int64_t D,
                        const float *Y, int64_t b, float *out, void *ws, size_t ws_bytes,
                        void *stream);

/* "R-free" a6: the same S~Y from Zhat and Q instead of R' -- R' rows are
 * recomputed (tcgen05 features GEMM + sincos) in chunks of chunk_rows rows (<= 0: 262,144) in three
 * sweeps (r, then W = R^T Y, then dinv . R'W), so only chunk_rows x 2d floats of R' ever exist.
 *   Zhat: n x d fp32 (d % 4 == 0);  Q: d x d fp32;  Y, out: n x b fp32.
 * Workspace: tpo_affinity_matvec_rfree_ws(n, d, b, chunk_rows).  Errors: TPO_EINVAL, TPO_ENOMEM, TPO_ECUDA. */
size_t tpo_affinity_matvec_rfree_ws(int64_t n, int64_t d, int64_t b, int64_t chunk_rows);
int tpo_affinity_matvec_rfree(const float *Zhat, int64_t n, int64_t d, const float *Q, const float *Y, int64_t b,
                              float *out, int64_t chunk_rows, void *ws, size_t ws_bytes, void *stream);

/* "R-free" a7: tpo_topk_eig's exact mode (R7) from Zhat and Q instead of R' --
 * R' rows are recomputed (Eq. R-prime; tcgen05 features GEMM + sincos, row-local,
 * so each recomputed row equals the materialised one bit for bit) in chunks of chunk_rows rows
 * (<= 0: 262,144) in three sweeps: r = R'^T 1; dinv = (R' r)^{-1/2} and the Gram G = R^T R (fp64
 * chunk sums added in chunk order); Gamma = R Psi Sigma^-1 (Eq. init-HY).  Then
 * the same eigensolver of G, CholeskyQR polish and R8 sign rule as tpo_topk_eig.
 *   Zhat: n x d fp32 device (d % 4 == 0);  Q: d x d fp32 device;  Gamma: n x k fp32 device out;
 *   sigma: k fp64 HOST out;  Psi: 2d x k fp32 device out;  dinv: n fp32 device out (Eq. dinv).
 * Workspace: tpo_topk_eig_rfree_ws(n, d, k, chunk_rows).  Errors: TPO_EINVAL, TPO_ENOMEM, TPO_ECUDA,
 * TPO_ENUMERIC (as tpo_topk_eig).  Synchronises the stream. */
size_t tpo_topk_eig_rfree_ws(int64_t n, int64_t d, int32_t k, int64_t chunk_rows);
int tpo_topk_eig_rfree(const float *Zhat, int64_t n, int64_t d, const float *Q, int32_t k, float *Gamma,
                       double *sigma, float *Psi, float *dinv, int64_t chunk_rows, void *ws, size_t ws_bytes,
                       void *stream);

/* "R-free" a8-a9: tpo_cluster (Alg. 2 ONMF, then Alg. 3 NCI rounding,
 * PAPER.md:536-604) with R' rows recomputed from Zhat and Q in chunks of chunk_rows rows in each of
 * the two R' passes of an ONMF iteration (R'^T (dinv . Ups), then dinv . (R' H)); the chunks' fp64
 * partials of R'^T (dinv . Ups) are added in chunk order (deterministic).  Both products run on the
 * fp64 tensor path (DMMA).  Alg. 3 does not touch R'.
 *   Zhat: n x d fp32;  Q: d x d fp32;  dinv: n fp32 (e.g. from tpo_topk_eig_rfree);  Gamma: n x k
 *   fp32;  sigma: k fp64 HOST;  Psi: 2d x k fp32;  labels: n int32 device out;  iters_used: host
 *   int32 out (Alg. 3 iterations), may be NULL.
 * Workspace: tpo_cluster_rfree_ws(n, d, k, chunk_rows).  Errors: TPO_EINVAL, TPO_ENOMEM, TPO_ECUDA. */
size_t tpo_cluster_rfree_ws(int64_t n, int64_t d, int32_t k, int64_t chunk_rows);
int tpo_cluster_rfree(const float *Zhat, int64_t n, int64_t d, const float *Q, const float *dinv, int32_t k,
                      const float *Gamma, const double *sigma, const float *Psi, int32_t Tf, int32_t Tg,
                      int32_t *labels, int32_t *iters_used, int64_t chunk_rows, void *ws, size_t ws_bytes,
                      void *stream);

/* ---------------------------------------------------------------------------------------
 * a7  Top-k singular triplets of R = diag(dinv) R' -- "the top-k left and right singular
 * vectors of R" and its top-k singular values (Eq. init-HY).
 *   mode TPO_EIG_EXACT (R7): the exact top-k.  Gram G = R^T R (D x D, fp64 cross-block
 *     sums), its top-k eigenpairs by a Chebyshev-filtered block subspace iteration on the
 *     device (fp64; the trivial pair u = r/||r||, G r = R'^T 1 = r, deflated; Rayleigh-Ritz
 *     with the full G; stop at max Ritz residual <= 1e-9 lambda_1, else TPO_ENUMERIC after
 *     60 rounds), Gamma = R Psi Sigma^{-1}, CholeskyQR2 polish when
 *     ||Gamma^T Gamma - I||_max > 1e-6.
 *   mode TPO_EIG_HALKO: the randomised truncated SVD the paper cites (Halko et al.,
 *     PAPER.md:574) with b = k + p columns, q power iterations, orthonormalisation by
 *     CholeskyQR2, Rayleigh-Ritz on the host.  Omega (D x b fp32) is its Gaussian test
 *     matrix.  An approximation of the EXACT result (exact only when it has converged).
 *   Both modes apply the sign rule R8 (column sums of Gamma >= 0).
 *   Rp: n x D fp32;  dinv: n fp32;  1 <= k <= min(n, D) (HALKO: k + p <= min(n, D)).
 *   Gamma: n x k fp32 out;  sigma: (host) k fp64 out, descending;  Psi: D x k fp32 out.
 * [sync].  Workspace: tpo_topk_eig_ws(n, D, k, mode, p).
 * Errors: TPO_EINVAL, TPO_ENOMEM, TPO_ECUDA, TPO_ENUMERIC (sigma_k == 0, non-SPD Gram, the
 * subspace iteration not converged).
 * --------------------------------------------------------------------------------------- */
enum { TPO_EIG_EXACT = 0, TPO_EIG_HALKO = 1 };
/* a7 step 1 on its own: G = R^T R = R'^T diag(dinv^2) R' (D x D fp64 out, full symmetric
 * matrix), the Gram of the exact mode.  tcgen05 kind::tf32 with 3xTF32 splitting of R
 * (fp32-accurate products), fp32 accumulation over 128-row segments, fp64 across segments.
 *   Rp: n x D fp32, D % 4 == 0;  dinv: n fp32;  G: D x D fp64 out (device).
 * Workspace: tpo_gram_ws(n, D).  Errors: TPO_EINVAL, TPO_ENOMEM, TPO_ECUDA. */
size_t tpo_gram_ws(int64_t n, int64_t D);
int tpo_gram(const float *Rp, const float *dinv, int64_t n, int64_t D, double *G, void *ws,
             size_t ws_bytes, void *stream);
size_t tpo_topk_eig_ws(int64_t n, int64_t D, int32_t k, int32_t mode, int32_t p);
int tpo_topk_eig(const float *Rp, const float *dinv, int64_t n, int64_t D, int32_t k,
                 int32_t mode, int32_t p, int32_t q, const float *Omega,
                 float *Gamma, double *sigma, float *Psi, void *ws, size_t ws_bytes,
                 void *stream);

/* ---------------------------------------------------------------------------------------
 * a8-a9  Discretisation: greedy orthogonal NMF (Alg. 2, Eqs. update-Q /
 * update-Y PAPER.md:553-560, products bracketed as PAPER.md:564), initialised from the
 * top-k triplets (Eq. init-HY) with the R9 clamps
 *     Ups = max(Gamma,0)+eps, H = max(Psi Sigma,0)+eps, eps = 1e-12,
 *     H   <- H   . max(R^T Ups,0) / (H (Ups^T Ups) + eps)
 *     Ups <- Ups . sqrt( max(R H,0) / (max(Ups (Ups^T (R H)),0) + eps) ),
 * T_f times (H first), then NCI generation (Alg. 3): Phi = I; T_g times
 * l*_i = argmax_l Ups[i].Phi[:,l] (Eq. ell-ast, ties -> smallest l), Y one-hot with unit
 * columns (Eqs. Y-update, y-norm), Phi = Ups^T Y; early stop on a
 * repeated labelling (R10).  All arithmetic fp64 or fp64-accurate: for 32 < k <= 64 the products
 * R H, R^T Ups and Alg. 3's scores run on the integer tensor cores (error-free byte-digit
 * splitting, R16; R^T Ups keeps the 26 digit pairs p + q <= 6, exact 128-bit cross-block sums),
 * the Alg. 3 argmax certified against the sequential fma of R13.
 *   Rp: n x D fp32;  dinv: n fp32;  Gamma: n x k fp32;  sigma: (host) k fp64;
 *   Psi: D x k fp32;  Tf >= 0, Tg >= 1;  labels: n int32 out in [0,k);
 *   iters_used: (host) int32 out, iterations of Alg. 3 actually run (may be NULL).
 * [sync].  Workspace: tpo_cluster_ws(n, D, k).  Errors: TPO_EINVAL, TPO_ENOMEM, TPO_ECUDA.
 * --------------------------------------------------------------------------------------- */
size_t tpo_cluster_ws(int64_t n, int64_t D, int32_t k);
int tpo_cluster(const float *Rp, const float *dinv, int64_t n, int64_t D, int32_t k,
                const float *Gamma, const double *sigma, const float *Psi, int32_t Tf,
                int32_t Tg, int32_t *labels, int32_t *iters_used, void *ws,
                size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------------------
 * Row GEMM of Alg. 2 / a7:  out = diag(rs) A W   (RH = dinv . (R' H), PAPER.md:552-560;
 * Gamma = R Psi Sigma^-1).  A: n x K fp32 row-major (16-byte aligned rows,
 * K % 4 == 0);  rs: n fp32 (NULL = 1);  W: K x N fp64;  out: n x N fp64 (all device).
 * fp64-accurate: when N <= 64 and 6 N K <= 96 KB (and TPO_OZ != 0) on the integer tensor cores
 * (tcgen05 kind::i8, Ozaki digit splitting: 6 byte digits per operand, exact int32 sums of
 * the digit products of equal weight, error <~ 2^-44 K max|A_i| max|W_l|), otherwise on the fp64
 * tensor path (DMMA).  Workspace: tpo_rowgemm_f64_ws(n, K, N).  Errors: TPO_EINVAL, TPO_ENOMEM,
 * TPO_ECUDA.  Asynchronous on `stream`.
 * --------------------------------------------------------------------------------------- */
size_t tpo_rowgemm_f64_ws(int64_t n, int64_t K, int32_t N);
int tpo_rowgemm_f64(const float *A, int64_t n, int64_t K, const float *rs, const double *W, int32_t N,
                    double *out, void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------------------
 * a5-a9 sharded across GPUs: the rank owns the contiguous U rows [u0, u1)
 * (n_p rows) of Zhat / R' / dinv / Gamma / Ups / labels; the CALLER all-reduces (sum) the
 * marked partials between the calls (NCCL on GPUs via torch.distributed), so the replicated
 * D x D / D x k / k x k quantities are identical on every rank:
 *   tpo_shard_features  R'_p = features of Zhat_p (Eqs. R-prime) and
 *                       r_part = sum_{i in p} R'[i] (2d fp64)                   -> all-reduce r
 *   tpo_shard_dinv      dinv_p[i] = 1/sqrt(max(R'[i] . r, 1e-12)) (Eq. Ri, 466-468; R6)
 *   tpo_gram            G_part = R_p^T R_p (D x D fp64)                          -> all-reduce G
 *   tpo_eig_from_gram   Psi64 (D x k fp64), sigma (host) = the exact top-k of R from the
 *                       global Gram (Eq. init-HY; R7) [sync]
 *   tpo_shard_gamma     Gamma64_p = diag(dinv_p) R'_p Psi64 diag(1/sigma) (n_p x k fp64) [sync]
 *   tpo_shard_atb64     out = A_p^T B_p (k x k fp64; A_p, B_p n_p x k fp64)      -> all-reduce
 *                       (Gamma^T Gamma for the CholeskyQR polish; Ups^T Ups, Ups^T RH in Alg. 2)
 *   tpo_shard_apply_chol X_p <- X_p S C^{-1} for the global Gram g = S^-1 C^T C S^-1 [sync]
 *   tpo_shard_colstats  per-column sum, sum|x|, max|x| and its GLOBAL row index (row0 = u0)
 *                       of Gamma64_p: sums -> all-reduce; (max, index) -> all-gather, the
 *                       caller keeps the largest magnitude, ties -> smallest index (R8) [sync]
 *   tpo_shard_gamma_final flips the columns with signs[l] < 0 (host int32 k) in Gamma64_p and
 *                       Psi (Psi = fp32 copy of Psi64 when Psi64 != NULL), rounds Gamma_p to
 *                       fp32 [sync]
 *   tpo_shard_onmf_init Ups_p = max(Gamma_p,0)+eps, H = max(Psi Sigma,0)+eps (R9) [sync]
 *   tpo_shard_onmf_rtu  RtU_part = R'_p^T (dinv_p . Ups_p) (D x k fp64)          -> all-reduce
 *   tpo_onmf_h_update   H <- H . max(RtU,0) / (H UtU + eps) (Eq. update-Q) [sync]
 *   tpo_shard_onmf_rh   RH_p = dinv_p . (R'_p H) (n_p x k fp64)
 *   tpo_shard_onmf_u_update Ups_p <- Ups_p . sqrt(max(RH_p,0) / (max(Ups_p M,0) + eps))
 *                       (Eq. update-Y; M = all-reduced Ups^T RH)
 *   tpo_shard_nci_assign labels_p = argmax_l (Ups_p Phi)[i, l] (Eq. ell-ast, PAPER.md:625-627,
 *                       ties -> smallest l); *changed (device int32, zeroed by the caller) set
 *                       to 1 when a label changes; sums[l][a] = sum_{i in C_l, i in p} Ups[i,a]
 *                       (k x k fp64) and counts[l] (k fp64)             -> all-reduce all three [sync]
 *   tpo_nci_phi         Phi[a][l] = sums[l][a] / sqrt(counts[l]) (empty -> 0)
 * Pointers are device pointers except those marked (host).  Workspace: tpo_shard_solver_ws
 * (n_p, d, k) bytes serve every call that takes one.  Errors: TPO_EINVAL (shapes, null or
 * misaligned pointers), TPO_ENOMEM, TPO_ECUDA, TPO_ENUMERIC (non-SPD Gram, sigma_k == 0).
 * --------------------------------------------------------------------------------------- */
size_t tpo_shard_solver_ws(int64_t n_p, int64_t d, int32_t k);
int tpo_shard_features(const float *Zhat_p, int64_t n_p, int64_t d, const float *Q, float *Rp_p,
                       double *r_part, void *ws, size_t ws_bytes, void *stream);
int tpo_shard_dinv(const float *Rp_p, int64_t n_p, int64_t D, const double *r, float *dinv_p,
                   void *stream);
int tpo_eig_from_gram(const double *G, const double *r, int64_t D, int32_t k, double *Psi64,
                      double *sigma, void *ws, size_t ws_bytes, void *stream);
int tpo_shard_gamma(const float *Rp_p, const float *dinv_p, int64_t n_p, int64_t D, int32_t k,
                    const double *Psi64, const double *sigma, double *Gamma64_p, void *ws,
                    size_t ws_bytes, void *stream);
int tpo_shard_atb64(const double *A_p, const double *B_p, int64_t n_p, int32_t k, double *out,
                    void *ws, size_t ws_bytes, void *stream);
int tpo_shard_apply_chol(double *X_p, int64_t n_p, int32_t k, const double *g, void *ws,
                         size_t ws_bytes, void *stream);
int tpo_shard_colstats(const double *A_p, int64_t n_p, int32_t k, int64_t row0, double *sum,
                       double *abs_sum, double *maxabs, int64_t *argmax, void *ws, size_t ws_bytes,
                       void *stream);
int tpo_shard_gamma_final(double *Gamma64_p, int64_t n_p, int32_t k, const int32_t *signs,
                          const double *Psi64, int64_t D, float *Psi, float *Gamma_p, void *ws,
                          size_t ws_bytes, void *stream);
int tpo_shard_onmf_init(const float *Gamma_p, int64_t n_p, const float *Psi, const double *sigma,
                        int64_t D, int32_t k, double *U_p, double *H, void *ws, size_t ws_bytes,
                        void *stream);
int tpo_shard_onmf_rtu(const float *Rp_p, const float *dinv_p, const double *U_p, int64_t n_p,
                       int64_t D, int32_t k, double *RtU_part, void *ws, size_t ws_bytes,
                       void *stream);
int tpo_onmf_h_update(double *H, const double *RtU, const double *UtU, int64_t D, int32_t k,
                      void *ws, size_t ws_bytes, void *stream);
int tpo_shard_onmf_rh(const float *Rp_p, const float *dinv_p, const double *H, int64_t n_p,
                      int64_t D, int32_t k, double *RH_p, void *stream);
int tpo_shard_onmf_u_update(double *U_p, const double *RH_p, const double *M, int64_t n_p,
                            int32_t k, void *stream);
int tpo_shard_nci_assign(const double *U_p, const double *Phi, int64_t n_p, int32_t k,
                         int32_t *labels_p, int32_t *changed, double *sums, double *counts,
                         void *ws, size_t ws_bytes, void *stream);
int tpo_nci_phi(const double *sums, const double *counts, int32_t k, double *Phi, void *stream);

/* ---------------------------------------------------------------------------------------
 * Evaluation and monitors.
 * tpo_eval: ARI, NMI and ACC of a predicted labelling against ground truth (Evaluation Metrics,
 *   PAPER.md:2448-2462): the k_pred x k_true contingency table is counted on the device (exact
 *   integer counts), the metrics are evaluated from it on the host in fp64; ACC matches
 *   predicted to true labels with the Hungarian algorithm; NMI is the standard
 *   sqrt-normalised form (reading R15: the printed numerator omits |U| inside the logarithm).
 *   pred, truth: n int32 (device), values in [0, k_pred) / [0, k_true);
 *   metrics: (host) 3 fp64 out {ARI, NMI, ACC}.  k_pred * k_true <= 49152.  [sync]
 *   Workspace: tpo_eval_ws(k_pred, k_true).  Errors: TPO_EINVAL (also a label out of range).
 * tpo_objective: the Lemma 4 monitor (Eq. obj5) of a labelling: out[0] =
 *   ||R^T Y||_F^2 = Tr(Y^T R R^T Y) for the NCI matrix Y of `labels` (columns 1/sqrt|C_l| on C_l;
 *   the discretisation's objective, <= sum_{l<=k} sigma_l^2 by Ky Fan), and, when Ups (n x k fp64,
 *   device) is given, out[1] = ||R^T Ups||_F^2, so that |Tr((Y Y^T - Ups Ups^T) R R^T)| =
 *   |out[0] - out[1]|.  R = diag(dinv) R' as in tpo_cluster.  out: (host) 1 or 2 fp64.  [sync]
 *   Workspace: tpo_objective_ws(n, D, k).  Errors: TPO_EINVAL (also a label out of range).
 * Target side V: clustering V instead of U is the same calls with the roles of B
 *   and B^T swapped and X = X_V: tpo_run(Bt, B, X_V, ...).
 * --------------------------------------------------------------------------------------- */
size_t tpo_eval_ws(int32_t k_pred, int32_t k_true);
int tpo_eval(const int32_t *pred, const int32_t *truth, int64_t n, int32_t k_pred, int32_t k_true, double *metrics,
             void *ws, size_t ws_bytes, void *stream);
size_t tpo_objective_ws(int64_t n, int64_t D, int32_t k);
int tpo_objective(const float *Rp, const float *dinv, int64_t n, int64_t D, int32_t k, const int32_t *labels,
                  const double *Ups, double *out, void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------------------
 * SVD-based attribute dimension reduction (Sec. 3.2.1, Eq. Xd; the step the
 * paper's default "TPO" runs before Alg. 1): X' = Gamma Sigma of the exact
 * top-d SVD X ~ Gamma Sigma Psi^T (R14: exact, as R7), computed as X Psi (Psi = top-d
 * eigenvectors of X^T X; tcgen05 3xTF32 Gram, device subspace iteration, fp64 product), each
 * column's sign fixed by R8 (column sum >= 0).  Lemma 3 bounds the MSA
 * error of propagating X' instead of X by sigma_{d+1}^2.  d == d_u copies X (pass-through).
 *   X: n x d_u fp32 (d_u % 4 == 0);  Xr: n x d fp32 out (the input X of tpo_propagate / tpo_run);
 *   sigma: (host) d fp64 out (descending singular values of X), or NULL.  1 <= d <= min(n, d_u).
 * [sync].  Workspace: tpo_svd_reduce_ws(n, d_u, d).
 * Errors: TPO_EINVAL, TPO_ENOMEM, TPO_ECUDA, TPO_ENUMERIC (subspace iteration not converged).
 * --------------------------------------------------------------------------------------- */
size_t tpo_svd_reduce_ws(int64_t n, int64_t d_u, int64_t d);
int tpo_svd_reduce(const float *X, int64_t n, int64_t d_u, int64_t d, float *Xr, double *sigma, void *ws,
                   size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------------------
 * Whole hot path (Fig. overview): propagate -> Haar Q from G -> features ->
 * top-k (mode) -> cluster.  G: d x d fp64 on the DEVICE (the Gaussian input of Alg. 1 L6,
 * resident like X; the Haar QR of Alg. 1 L7 runs inside the call, beside the propagation).  Omega: D x (k+p) fp32 (HALKO only, else
 * NULL).  labels: n int32 out.  timings_ms: (host) 4 doubles out {propagate, features,
 * topk, cluster} measured with CUDA events on `stream`, or NULL.
 * [sync].  Workspace: tpo_run_ws(n_u, n_v, nnz, d, k, mode, p).
 * --------------------------------------------------------------------------------------- */
size_t tpo_run_ws(int64_t n_u, int64_t n_v, int64_t nnz, int64_t d, int32_t k, int32_t mode,
                  int32_t p);
int tpo_run(const tpo_csr_t *B, const tpo_csr_t *Bt, const float *X, int64_t d, float alpha,
            int32_t T, int32_t k, const double *G, int32_t eig_mode, const float *Omega,
            int32_t p, int32_t q, int32_t Tf, int32_t Tg, int32_t *labels,
            double *timings_ms, void *ws, size_t ws_bytes, void *stream);

/* The same path end to end from HOST inputs: B, Bt (row_ptr, col_idx, val), X and G are host
 * pointers (pinned memory lets the copies run asynchronously), labels a host int32 array of
 * n_u.  Inside the call the inputs are copied to device buffers carved from the workspace --
 * G first, on the Haar side stream, so the Haar QR of Alg. 1 L7 runs while the CSRs and X
 * are still being copied (no SMs are held back for it) -- then the path runs as tpo_run and the
 * labels are copied back.  Omega (HALKO only) stays a device pointer.  timings_ms[0] includes
 * the input copies.  [sync].  Workspace: tpo_run_host_ws(..., weighted = B->val != NULL). */
size_t tpo_run_host_ws(int64_t n_u, int64_t n_v, int64_t nnz, int64_t d, int32_t k, int32_t mode,
                       int32_t p, int32_t weighted);
int tpo_run_host(const tpo_csr_t *B, const tpo_csr_t *Bt, const float *X, int64_t d, float alpha,
                 int32_t T, int32_t k, const double *G, int32_t eig_mode, const float *Omega,
                 int32_t p, int32_t q, int32_t Tf, int32_t Tg, int32_t *labels,
                 double *timings_ms, void *ws, size_t ws_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* TPO_H */
