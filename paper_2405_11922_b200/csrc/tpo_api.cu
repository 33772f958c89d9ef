// C-ABI entry points of libtpo (include/tpo.h): argument validation, workspace carving,
// error translation.  All arithmetic lives in the module files.
#include <string.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include <stdio.h>
#include <stdlib.h>

#include "tpo_internal.cuh"

namespace tpo {

size_t propagate_ws_bytes(int64_t n_u, int64_t n_v, int64_t nnz, int64_t d);
size_t features_ws_bytes(int64_t n, int64_t d);
size_t topk_eig_ws_bytes(int64_t n, int64_t D, int32_t k, int32_t mode, int32_t p);
size_t cluster_ws_bytes(int64_t n, int64_t D, int32_t k);

namespace {
thread_local std::string g_last_error;
thread_local uint64_t g_launches = 0;
}

void set_error(const std::string &msg) { g_last_error = msg; }
void count_launch() { ++g_launches; }

int sm_count() {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
    return v;
}

namespace {

void check_ptr(const void *p, const char *name, bool need_align = true) {
    TPO_REQUIRE(p != nullptr, std::string(name) + " is NULL");
    if (need_align) TPO_REQUIRE(aligned16(p), std::string(name) + " is not 16-byte aligned");
}

void check_csr(const tpo_csr_t *A, const char *name) {
    TPO_REQUIRE(A != nullptr, std::string(name) + " is NULL");
    TPO_REQUIRE(A->n_rows >= 0 && A->n_cols >= 0 && A->nnz >= 0, std::string(name) + ": negative size");
    TPO_REQUIRE(A->n_rows < (int64_t(1) << 31) && A->n_cols < (int64_t(1) << 31), std::string(name) + ": more than 2^31-1 rows/cols");
    TPO_REQUIRE(A->row_ptr != nullptr, std::string(name) + ".row_ptr is NULL");
    TPO_REQUIRE(A->nnz == 0 || A->col_idx != nullptr, std::string(name) + ".col_idx is NULL");
}

// The SpMM gathers address a row of the gathered table with a 32-bit float4 offset
// (col * d/4 for a row-major table, col * group width for a column-group table), so every
// gathered table must hold fewer than 2^32 float4.
void check_gather_range(int64_t rows, int64_t d, const char *what) {
    TPO_REQUIRE(rows * (d / 4) < (int64_t(1) << 32),
                std::string(what) + ": rows x d/4 >= 2^32 exceeds the SpMM's 32-bit gather offsets");
}

void check_ws(void *ws, size_t have, size_t need) {
    if (have < need) throw Error(TPO_ENOMEM, "workspace too small: " + std::to_string(have) + " < " + std::to_string(need));
    TPO_REQUIRE(ws != nullptr || need == 0, "ws is NULL");
    TPO_REQUIRE((reinterpret_cast<uintptr_t>(ws) & 255u) == 0, "ws is not 256-byte aligned");
}

void check_propagate(const tpo_csr_t *B, const tpo_csr_t *Bt, const float *X, int64_t d, float alpha, int32_t T,
                     const float *Z, const float *Zhat) {
    check_csr(B, "B");
    check_csr(Bt, "Bt");
    TPO_REQUIRE(B->n_rows == Bt->n_cols && B->n_cols == Bt->n_rows, "Bt is not shaped as the transpose of B");
    TPO_REQUIRE(B->nnz == Bt->nnz, "B.nnz != Bt.nnz");
    TPO_REQUIRE(d >= 4 && d % 4 == 0, "d must be a positive multiple of 4");
    TPO_REQUIRE(alpha >= 0.0f && alpha <= 1.0f, "alpha must lie in [0, 1]");
    TPO_REQUIRE(T >= 0, "T must be >= 0");
    check_gather_range(B->n_rows, d, "Z (gathered by the V-side SpMM)");
    check_gather_range(B->n_cols, d, "the V-side block (gathered by the U-side SpMM)");
    if (B->n_rows > 0) {
        check_ptr(X, "X");
        check_ptr(Z, "Z");
    }
    if (Zhat) check_ptr(Zhat, "Zhat");
}

}  // namespace
}  // namespace tpo

using namespace tpo;

extern "C" {

int tpo_abi_version(void) { return TPO_ABI_VERSION; }

const char *tpo_last_error(void) { return tpo::g_last_error.c_str(); }

uint64_t tpo_launch_count(void) { return tpo::g_launches; }

size_t tpo_propagate_ws(int64_t n_u, int64_t n_v, int64_t nnz, int64_t d) {
    return propagate_ws_bytes(n_u, n_v, nnz, d);
}

int tpo_propagate(const tpo_csr_t *B, const tpo_csr_t *Bt, const float *X, int64_t d, float alpha, int32_t T,
                  float *Z, float *Zhat, void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        check_propagate(B, Bt, X, d, alpha, T, Z, Zhat);
        check_ws(ws, ws_bytes, tpo_propagate_ws(B->n_rows, B->n_cols, B->nnz, d));
        Arena ar(ws, ws_bytes);
        propagate_impl(*B, *Bt, X, d, alpha, T, Z, Zhat, ar, as_stream(stream));
    });
}

size_t tpo_shard_ws(int64_t n_rows, int64_t nnz, int64_t d) { return shard_spmm_ws_bytes(n_rows, nnz, d); }

int tpo_shard_degrees(const tpo_csr_t *Bp, const tpo_csr_t *Btp, double *deg_u, double *deg_v, void *stream) {
    return guarded([&] {
        check_csr(Bp, "Bp");
        check_csr(Btp, "Btp");
        TPO_REQUIRE(Bp->n_rows == Btp->n_cols && Bp->n_cols == Btp->n_rows && Bp->nnz == Btp->nnz,
                    "Btp is not shaped as the transpose of Bp");
        if (Bp->n_rows) TPO_REQUIRE(deg_u != nullptr, "deg_u is NULL");
        if (Btp->n_rows) TPO_REQUIRE(deg_v != nullptr, "deg_v is NULL");
        shard_degrees_impl(*Bp, *Btp, deg_u, deg_v, as_stream(stream));
    });
}

int tpo_shard_start(const double *deg_u, const double *deg_v, int64_t n_p, int64_t m, const float *Xp, int64_t d,
                    float alpha, float *s_u, float *s_v, float *Pp, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n_p >= 0 && m >= 0, "negative size");
        TPO_REQUIRE(d >= 4 && d % 4 == 0, "d must be a positive multiple of 4");
        TPO_REQUIRE(alpha >= 0.0f && alpha <= 1.0f, "alpha must lie in [0, 1]");
        if (n_p) {
            check_ptr(Xp, "Xp");
            check_ptr(Pp, "Pp");
            TPO_REQUIRE(deg_u && s_u, "deg_u / s_u is NULL");
        }
        if (m) TPO_REQUIRE(deg_v && s_v, "deg_v / s_v is NULL");
        shard_start_impl(deg_u, deg_v, n_p, m, Xp, d, alpha, s_u, s_v, Pp, as_stream(stream));
    });
}

int tpo_shard_vside(const tpo_csr_t *Btp, const float *Pp, int64_t d, float *Qpart, void *ws, size_t ws_bytes,
                    void *stream) {
    return guarded([&] {
        check_csr(Btp, "Btp");
        TPO_REQUIRE(d >= 4 && d % 4 == 0, "d must be a positive multiple of 4");
        check_gather_range(Btp->n_cols, d, "Pp (gathered by the V-side SpMM)");
        if (Btp->n_rows) check_ptr(Qpart, "Qpart");
        if (Btp->n_cols) check_ptr(Pp, "Pp");
        check_ws(ws, ws_bytes, tpo_shard_ws(Btp->n_rows, Btp->nnz, d));
        Arena ar(ws, ws_bytes);
        shard_vside_impl(*Btp, Pp, d, Qpart, ar, as_stream(stream));
    });
}

int tpo_shard_vscale(float *Q, const float *s_v, int64_t rows, int64_t d, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(rows >= 0 && d >= 4 && d % 4 == 0, "bad shape");
        if (rows) {
            check_ptr(Q, "Q");
            TPO_REQUIRE(s_v != nullptr, "s_v is NULL");
        }
        shard_vscale_impl(Q, s_v, rows, d, as_stream(stream));
    });
}

int tpo_shard_uside(const tpo_csr_t *Bp, const float *Q, const float *Xp, int64_t d, float alpha, const float *s_u,
                    int32_t last, float *Zp, float *Zhat_p, void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        check_csr(Bp, "Bp");
        TPO_REQUIRE(d >= 4 && d % 4 == 0, "d must be a positive multiple of 4");
        check_gather_range(Bp->n_cols, d, "Q (gathered by the U-side SpMM)");
        TPO_REQUIRE(alpha >= 0.0f && alpha <= 1.0f, "alpha must lie in [0, 1]");
        if (Bp->n_rows) {
            check_ptr(Xp, "Xp");
            check_ptr(Zp, "Zp");
            TPO_REQUIRE(s_u != nullptr, "s_u is NULL");
        }
        if (Bp->n_cols) check_ptr(Q, "Q");
        if (Zhat_p) check_ptr(Zhat_p, "Zhat_p");
        check_ws(ws, ws_bytes, tpo_shard_ws(Bp->n_rows, Bp->nnz, d));
        Arena ar(ws, ws_bytes);
        shard_uside_impl(*Bp, Q, Xp, d, alpha, s_u, last != 0, Zp, Zhat_p, ar, as_stream(stream));
    });
}

int tpo_haar_q(const double *G, int64_t d, double *Q) {
    return guarded([&] {
        TPO_REQUIRE(G != nullptr && Q != nullptr, "G and Q must be host pointers");
        TPO_REQUIRE(d >= 1, "d must be >= 1");
        host_qr_positive(d, d, G, Q, nullptr);
    });
}

size_t tpo_haar_q_dev_ws(int64_t d) { return haar_q_ws_bytes(d); }

int tpo_haar_q_dev(const double *G, int64_t d, float *Q, void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(G != nullptr, "G (host) is NULL");
        TPO_REQUIRE(d >= 1, "d must be >= 1");
        check_ptr(Q, "Q");
        check_ws(ws, ws_bytes, tpo_haar_q_dev_ws(d));
        Arena ar(ws, ws_bytes);
        cudaStream_t st = as_stream(stream);
        haar_q_device(G, false, d, Q, ar, st);
        TPO_CUDA(cudaStreamSynchronize(st));
    });
}

size_t tpo_features_ws(int64_t n, int64_t d) { return features_ws_bytes(n, d); }

int tpo_features(const float *Zhat, int64_t n, int64_t d, const float *Q, float *Rp, float *dinv, double *r_out,
                 void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n >= 0, "n must be >= 0");
        TPO_REQUIRE(d >= 4 && d <= 8192 && d % 4 == 0, "d must be a multiple of 4 in [4, 8192]");
        if (n > 0) {
            check_ptr(Zhat, "Zhat");
            check_ptr(Rp, "Rp");
            check_ptr(dinv, "dinv");
        }
        check_ptr(Q, "Q");
        check_ws(ws, ws_bytes, tpo_features_ws(n, d));
        Arena ar(ws, ws_bytes);
        features_impl(Zhat, n, d, Q, Rp, dinv, r_out, ar, as_stream(stream));
    });
}

size_t tpo_affinity_matvec_ws(int64_t n, int64_t D, int64_t b) {
    return std::max(align_up(sizeof(double) * D * b) + tsgemm_ws(n, D, b), ts_affinity_ws(D, b)) + 1024;
}

int tpo_affinity_matvec(const float *Rp, const float *dinv, int64_t n, int64_t D, const float *Y, int64_t b,
                        float *out, void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n >= 1 && D >= 1 && b >= 1, "n, D, b must be >= 1");
        check_ptr(Rp, "Rp");
        check_ptr(dinv, "dinv");
        check_ptr(Y, "Y");
        check_ptr(out, "out");
        TPO_REQUIRE(out != Y, "out may not alias Y");
        check_ws(ws, ws_bytes, tpo_affinity_matvec_ws(n, D, b));
        Arena ar(ws, ws_bytes);
        affinity_matvec_impl(Rp, dinv, n, D, Y, b, out, ar, as_stream(stream));
    });
}

size_t tpo_affinity_matvec_rfree_ws(int64_t n, int64_t d, int64_t b, int64_t chunk_rows) {
    return ts_affinity_rfree_ws(n, d, b, chunk_rows > 0 ? chunk_rows : (int64_t)1 << 18);
}

int tpo_affinity_matvec_rfree(const float *Zhat, int64_t n, int64_t d, const float *Q, const float *Y, int64_t b,
                              float *out, int64_t chunk_rows, void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n >= 1 && d >= 4 && d % 4 == 0 && b >= 1, "need n >= 1, d a positive multiple of 4, b >= 1");
        check_ptr(Zhat, "Zhat");
        check_ptr(Q, "Q");
        check_ptr(Y, "Y", false);
        check_ptr(out, "out", false);
        const int64_t chunk = chunk_rows > 0 ? chunk_rows : (int64_t)1 << 18;
        check_ws(ws, ws_bytes, tpo_affinity_matvec_rfree_ws(n, d, b, chunk));
        Arena ar(ws, ws_bytes);
        ts_affinity_rfree(Zhat, n, d, Q, Y, b, out, chunk, ar, as_stream(stream));
    });
}

static int64_t rfree_chunk_rows(int64_t chunk_rows) { return chunk_rows > 0 ? chunk_rows : (int64_t)1 << 18; }

size_t tpo_topk_eig_rfree_ws(int64_t n, int64_t d, int32_t k, int64_t chunk_rows) {
    return topk_rfree_ws(n, d, k, rfree_chunk_rows(chunk_rows));
}

int tpo_topk_eig_rfree(const float *Zhat, int64_t n, int64_t d, const float *Q, int32_t k, float *Gamma, double *sigma,
                       float *Psi, float *dinv, int64_t chunk_rows, void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n >= 1 && d >= 4 && d % 4 == 0, "need n >= 1 and d a positive multiple of 4");
        TPO_REQUIRE(k >= 1 && k <= 128 && k <= n && k <= 2 * d, "k must lie in [1, min(n, 2d, 128)]");
        check_ptr(Zhat, "Zhat");
        check_ptr(Q, "Q");
        check_ptr(Gamma, "Gamma");
        check_ptr(Psi, "Psi");
        check_ptr(dinv, "dinv");
        TPO_REQUIRE(sigma != nullptr, "sigma (host) is NULL");
        const int64_t chunk = rfree_chunk_rows(chunk_rows);
        check_ws(ws, ws_bytes, tpo_topk_eig_rfree_ws(n, d, k, chunk));
        Arena ar(ws, ws_bytes);
        RSource src;
        src.Zhat = Zhat; src.d = d; src.Q = Q; src.chunk = chunk;
        topk_rfree_impl(src, n, k, Gamma, sigma, Psi, dinv, ar, as_stream(stream));
    });
}

size_t tpo_cluster_rfree_ws(int64_t n, int64_t d, int32_t k, int64_t chunk_rows) {
    return cluster_ws_bytes(n, 2 * d, k) + rfree_pass_ws(n, d, k, rfree_chunk_rows(chunk_rows));
}

int tpo_cluster_rfree(const float *Zhat, int64_t n, int64_t d, const float *Q, const float *dinv, int32_t k,
                      const float *Gamma, const double *sigma, const float *Psi, int32_t Tf, int32_t Tg, int32_t *labels,
                      int32_t *iters_used, int64_t chunk_rows, void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n >= 1 && d >= 4 && d % 4 == 0, "need n >= 1 and d a positive multiple of 4");
        TPO_REQUIRE(k >= 1 && k <= 128 && k <= n && k <= 2 * d, "k must lie in [1, min(n, 2d, 128)]");
        TPO_REQUIRE(Tf >= 0 && Tg >= 1, "need Tf >= 0 and Tg >= 1");
        check_ptr(Zhat, "Zhat");
        check_ptr(Q, "Q");
        check_ptr(dinv, "dinv");
        check_ptr(Gamma, "Gamma");
        check_ptr(Psi, "Psi");
        check_ptr(labels, "labels");
        TPO_REQUIRE(sigma != nullptr, "sigma (host) is NULL");
        const int64_t chunk = rfree_chunk_rows(chunk_rows);
        check_ws(ws, ws_bytes, tpo_cluster_rfree_ws(n, d, k, chunk));
        Arena ar(ws, ws_bytes);
        RSource src;
        src.Zhat = Zhat; src.d = d; src.Q = Q; src.chunk = chunk;
        cluster_impl(nullptr, dinv, n, 2 * d, k, Gamma, sigma, Psi, Tf, Tg, labels, iters_used, ar, as_stream(stream),
                     RStats(), &src);
    });
}

size_t tpo_gram_ws(int64_t n, int64_t D) { return gram_tc_ws(n, D) + 1024; }

int tpo_gram(const float *Rp, const float *dinv, int64_t n, int64_t D, double *G, void *ws, size_t ws_bytes,
             void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n >= 1 && D >= 4 && D % 4 == 0, "need n >= 1 and D a positive multiple of 4");
        check_ptr(Rp, "Rp");
        check_ptr(dinv, "dinv");
        check_ptr(G, "G");
        check_ws(ws, ws_bytes, tpo_gram_ws(n, D));
        Arena ar(ws, ws_bytes);
        gram_tc(Rp, dinv, n, D, G, ar, as_stream(stream));
    });
}

size_t tpo_topk_eig_ws(int64_t n, int64_t D, int32_t k, int32_t mode, int32_t p) {
    return topk_eig_ws_bytes(n, D, k, mode, p);
}

int tpo_topk_eig(const float *Rp, const float *dinv, int64_t n, int64_t D, int32_t k, int32_t mode, int32_t p,
                 int32_t q, const float *Omega, float *Gamma, double *sigma, float *Psi, void *ws, size_t ws_bytes,
                 void *stream) {
    return guarded([&] {
        TPO_REQUIRE(mode == TPO_EIG_EXACT || mode == TPO_EIG_HALKO, "unknown eig mode");
        TPO_REQUIRE(n >= 1 && D >= 1, "n and D must be >= 1");
        TPO_REQUIRE(k >= 1 && k <= n && k <= D, "k must lie in [1, min(n, D)]");
        TPO_REQUIRE(k <= 128, "k must be <= 128");
        if (mode == TPO_EIG_HALKO) {
            TPO_REQUIRE(p >= 0 && q >= 0, "p and q must be >= 0");
            TPO_REQUIRE(k + p <= n && k + p <= D, "k + p must be <= min(n, D)");
            check_ptr(Omega, "Omega");
        }
        check_ptr(Rp, "Rp");
        check_ptr(dinv, "dinv");
        check_ptr(Gamma, "Gamma");
        check_ptr(Psi, "Psi");
        TPO_REQUIRE(sigma != nullptr, "sigma (host) is NULL");
        check_ws(ws, ws_bytes, tpo_topk_eig_ws(n, D, k, mode, p));
        Arena ar(ws, ws_bytes);
        cudaStream_t st = as_stream(stream);
        topk_eig_impl(Rp, dinv, n, D, k, mode, p, q, Omega, Gamma, sigma, Psi, ar, st);
        TPO_CUDA(cudaStreamSynchronize(st));
    });
}

size_t tpo_cluster_ws(int64_t n, int64_t D, int32_t k) { return cluster_ws_bytes(n, D, k); }

int tpo_cluster(const float *Rp, const float *dinv, int64_t n, int64_t D, int32_t k, const float *Gamma,
                const double *sigma, const float *Psi, int32_t Tf, int32_t Tg, int32_t *labels, int32_t *iters_used,
                void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n >= 1 && D >= 1, "n and D must be >= 1");
        TPO_REQUIRE(k >= 1 && k <= 128 && k <= n && k <= D, "k must lie in [1, min(n, D, 128)]");
        TPO_REQUIRE(Tf >= 0 && Tg >= 1, "need Tf >= 0 and Tg >= 1");
        check_ptr(Rp, "Rp");
        check_ptr(dinv, "dinv");
        check_ptr(Gamma, "Gamma");
        check_ptr(Psi, "Psi");
        check_ptr(labels, "labels");
        TPO_REQUIRE(sigma != nullptr, "sigma (host) is NULL");
        check_ws(ws, ws_bytes, tpo_cluster_ws(n, D, k));
        Arena ar(ws, ws_bytes);
        cluster_impl(Rp, dinv, n, D, k, Gamma, sigma, Psi, Tf, Tg, labels, iters_used, ar, as_stream(stream));
    });
}

int tpo_comm_unique_id(void *id) {
    return guarded([&] {
        TPO_REQUIRE(id != nullptr, "id is NULL");
        comm_unique_id(id);
    });
}

int tpo_comm_create(const void *id, int32_t rank, int32_t world, int32_t device, void **comm) {
    return guarded([&] {
        TPO_REQUIRE(id != nullptr && comm != nullptr, "id / comm is NULL");
        TPO_REQUIRE(world >= 1 && rank >= 0 && rank < world, "need 0 <= rank < world");
        *comm = comm_create(id, rank, world, device);
    });
}

int tpo_comm_destroy(void *comm) {
    return guarded([&] { comm_destroy(comm); });
}

size_t tpo_propagate_sharded_ws(int64_t n_p, int64_t n_v, int64_t nnz_p, int64_t d, int32_t world) {
    return propagate_sharded_ws_bytes(n_p, n_v, nnz_p, d, std::max<int32_t>(world, 1));
}

int tpo_propagate_sharded(void *comm, const tpo_csr_t *Bp, const tpo_csr_t *Btp, const float *Xp, int64_t d, float alpha,
                          int32_t T, float *Zp, float *Zhat_p, void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(comm != nullptr, "comm is NULL");
        check_csr(Bp, "Bp");
        check_csr(Btp, "Btp");
        TPO_REQUIRE(Bp->n_rows == Btp->n_cols && Bp->n_cols == Btp->n_rows && Bp->nnz == Btp->nnz,
                    "Btp is not shaped as the transpose of Bp");
        TPO_REQUIRE(d >= 4 && d % 4 == 0, "d must be a positive multiple of 4");
        TPO_REQUIRE(alpha >= 0.0f && alpha <= 1.0f, "alpha must lie in [0, 1]");
        TPO_REQUIRE(T >= 0, "T must be >= 0");
        check_gather_range(Btp->n_cols, d, "Pp (gathered by the V-side SpMM)");
        check_gather_range(Bp->n_cols, d, "Q (gathered by the U-side SpMM)");
        if (Bp->n_rows) {
            check_ptr(Xp, "Xp");
            check_ptr(Zp, "Zp");
        }
        if (Zhat_p) check_ptr(Zhat_p, "Zhat_p");
        check_ws(ws, ws_bytes, tpo_propagate_sharded_ws(Bp->n_rows, Bp->n_cols, Bp->nnz, d, comm_world(comm)));
        Arena ar(ws, ws_bytes);
        propagate_sharded_impl(comm, *Bp, *Btp, Xp, d, alpha, T, Zp, Zhat_p, ar, as_stream(stream));
    });
}

size_t tpo_run_sharded_ws(int64_t n_p, int64_t n_v, int64_t nnz_p, int64_t d, int32_t k, int32_t world) {
    return run_sharded_ws_bytes(n_p, n_v, nnz_p, d, k, std::max<int32_t>(world, 1));
}

int tpo_run_sharded(void *comm, const tpo_csr_t *Bp, const tpo_csr_t *Btp, const float *Xp, int64_t d, float alpha,
                    int32_t T, int32_t k, const double *G, int64_t row0, int32_t Tf, int32_t Tg, int32_t *labels_p,
                    int32_t *iters_used, double *timings_ms, void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(comm != nullptr, "comm is NULL");
        check_csr(Bp, "Bp");
        check_csr(Btp, "Btp");
        TPO_REQUIRE(Bp->n_rows == Btp->n_cols && Bp->n_cols == Btp->n_rows && Bp->nnz == Btp->nnz,
                    "Btp is not shaped as the transpose of Bp");
        TPO_REQUIRE(d >= 4 && d % 4 == 0, "d must be a positive multiple of 4");
        TPO_REQUIRE(alpha >= 0.0f && alpha <= 1.0f, "alpha must lie in [0, 1]");
        TPO_REQUIRE(T >= 0 && Tf >= 0 && Tg >= 1 && row0 >= 0, "T, Tf >= 0, Tg >= 1, row0 >= 0");
        TPO_REQUIRE(k >= 1 && k <= 2 * d && k <= 128, "need 1 <= k <= min(2d, 128)");
        check_gather_range(Btp->n_cols, d, "Pp (gathered by the V-side SpMM)");
        check_gather_range(Bp->n_cols, d, "Q (gathered by the U-side SpMM)");
        check_ptr(G, "G");
        if (Bp->n_rows) {
            check_ptr(Xp, "Xp");
            TPO_REQUIRE(labels_p != nullptr, "labels_p is NULL");
        }
        check_ws(ws, ws_bytes, tpo_run_sharded_ws(Bp->n_rows, Bp->n_cols, Bp->nnz, d, k, comm_world(comm)));
        Arena ar(ws, ws_bytes);
        run_sharded_impl(comm, *Bp, *Btp, Xp, d, alpha, T, k, G, row0, Tf, Tg, labels_p, iters_used, timings_ms, ar,
                         as_stream(stream));
    });
}

int tpo_rows_gather(const float *src, const int32_t *idx, int64_t nidx, int64_t d, float *dst, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(nidx >= 0 && d >= 4 && d % 4 == 0, "need nidx >= 0 and d a positive multiple of 4");
        if (nidx > 0) {
            check_ptr(src, "src");
            check_ptr(dst, "dst");
            TPO_REQUIRE(idx != nullptr, "idx is NULL");
        }
        rows_gather_impl(src, idx, nidx, d, dst, as_stream(stream));
    });
}

int tpo_rows_scatter(float *dst, const int32_t *idx, int64_t nidx, int64_t d, const float *src, int32_t accumulate,
                     void *stream) {
    return guarded([&] {
        TPO_REQUIRE(nidx >= 0 && d >= 4 && d % 4 == 0, "need nidx >= 0 and d a positive multiple of 4");
        if (nidx > 0) {
            check_ptr(src, "src");
            check_ptr(dst, "dst");
            TPO_REQUIRE(idx != nullptr, "idx is NULL");
        }
        rows_scatter_impl(dst, idx, nidx, d, src, accumulate != 0, as_stream(stream));
    });
}

size_t tpo_eval_ws(int32_t k_pred, int32_t k_true) { return eval_ws_bytes(k_pred, k_true); }

int tpo_eval(const int32_t *pred, const int32_t *truth, int64_t n, int32_t k_pred, int32_t k_true, double *metrics,
             void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n >= 0, "n must be >= 0");
        TPO_REQUIRE(k_pred >= 1 && k_true >= 1 && (int64_t)k_pred * k_true <= 48 * 1024,
                    "k_pred, k_true must be >= 1 with k_pred * k_true <= 49152");
        TPO_REQUIRE(metrics != nullptr, "metrics is NULL");
        if (n > 0) {
            TPO_REQUIRE(pred != nullptr, "pred is NULL");
            TPO_REQUIRE(truth != nullptr, "truth is NULL");
        }
        check_ws(ws, ws_bytes, tpo_eval_ws(k_pred, k_true));
        Arena ar(ws, ws_bytes);
        eval_impl(pred, truth, n, k_pred, k_true, metrics, ar, as_stream(stream));
    });
}

size_t tpo_objective_ws(int64_t n, int64_t D, int32_t k) { return objective_ws_bytes(n, D, k); }

int tpo_objective(const float *Rp, const float *dinv, int64_t n, int64_t D, int32_t k, const int32_t *labels,
                  const double *Ups, double *out, void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n >= 1 && D >= 4 && D % 4 == 0, "need n >= 1 and D a positive multiple of 4");
        TPO_REQUIRE(k >= 1, "k must be >= 1");
        check_ptr(Rp, "Rp");
        check_ptr(dinv, "dinv", false);
        TPO_REQUIRE(labels != nullptr, "labels is NULL");
        TPO_REQUIRE(out != nullptr, "out is NULL");
        if (Ups) check_ptr(Ups, "Ups");
        check_ws(ws, ws_bytes, tpo_objective_ws(n, D, k));
        Arena ar(ws, ws_bytes);
        objective_impl(Rp, dinv, n, D, k, labels, Ups, out, ar, as_stream(stream));
    });
}

size_t tpo_svd_reduce_ws(int64_t n, int64_t d_u, int64_t d) { return svd_reduce_ws_bytes(n, d_u, d); }

int tpo_svd_reduce(const float *X, int64_t n, int64_t d_u, int64_t d, float *Xr, double *sigma, void *ws,
                   size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n >= 1, "n must be >= 1");
        TPO_REQUIRE(d_u >= 4 && d_u % 4 == 0, "d_u must be a positive multiple of 4");
        TPO_REQUIRE(d >= 1 && d <= d_u && d <= n, "d must lie in [1, min(n, d_u)]");
        check_ptr(X, "X");
        check_ptr(Xr, "Xr");
        check_ws(ws, ws_bytes, tpo_svd_reduce_ws(n, d_u, d));
        Arena ar(ws, ws_bytes);
        svd_reduce_impl(X, n, d_u, d, Xr, sigma, ar, as_stream(stream));
    });
}

size_t tpo_run_ws(int64_t n_u, int64_t n_v, int64_t nnz, int64_t d, int32_t k, int32_t mode, int32_t p) {
    const int64_t D = 2 * d;
    size_t s = 0;
    s += 2 * align_up(sizeof(float) * n_u * d);          // Z, Zhat
    s += align_up(sizeof(float) * n_u * D) + align_up(sizeof(float) * n_u);   // Rp, dinv
    s += align_up(sizeof(float) * d * d);                // Q
    s += align_up(sizeof(float) * n_u * k) + align_up(sizeof(float) * D * k);   // Gamma, Psi
    s += align_up(sizeof(double) * D);                                           // r
    s += align_up(sizeof(int32_t) * n_u + 1) + align_up(sizeof(uint32_t) * D + 1);  // R' row exponents, feature maxima
    s += align_up(sizeof(double) * D + 1);                                        // s = 1^T R
    s += align_up(haar_q_ws_bytes(d));                   // Haar Q runs beside the propagation
    size_t stage = std::max(std::max(tpo_propagate_ws(n_u, n_v, nnz, d), tpo_features_ws(n_u, d)),
                            std::max(tpo_topk_eig_ws(n_u, D, k, mode, p), tpo_cluster_ws(n_u, D, k)));
    return s + stage + 8 * 256;
}

// ------------------------------------------------------------------------------------------
// Row-sharded solver pieces (a5-a9); the caller all-reduces the partials between calls.
// ------------------------------------------------------------------------------------------
size_t tpo_shard_solver_ws(int64_t n_p, int64_t d, int32_t k) {
    const int64_t D = 2 * d;
    size_t s = features_ws_bytes(n_p, d);
    s = std::max(s, eig_from_gram_ws(D, k));
    s = std::max(s, nci_assign_part_ws(n_p, k));
    s = std::max(s, onmf_ws_bytes(n_p, D, k));
    s = std::max(s, ts_atb_ws(k, k) + align_up(sizeof(double) * (size_t)k * k));
    s = std::max(s, dgemm_ws(std::max<int64_t>(n_p, k), k, n_p) + align_up(sizeof(double) * (size_t)(n_p * k + k * k)));
    return s + 64 * 256 + align_up(sizeof(double) * (size_t)(D * k + 4 * 2 * 148 * k));
}

int tpo_shard_features(const float *Zhat_p, int64_t n_p, int64_t d, const float *Q, float *Rp_p, double *r_part,
                       void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n_p >= 0 && d >= 4 && d % 4 == 0, "bad n_p / d");
        check_ptr(Q, "Q");
        check_ptr(r_part, "r_part");
        if (n_p > 0) { check_ptr(Zhat_p, "Zhat_p"); check_ptr(Rp_p, "Rp_p"); }
        Arena ar(ws, ws_bytes);
        features_part(Zhat_p, n_p, d, Q, Rp_p, r_part, ar, as_stream(stream));
    });
}

int tpo_shard_dinv(const float *Rp_p, int64_t n_p, int64_t D, const double *r, float *dinv_p, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n_p >= 0 && D >= 1, "bad n_p / D");
        check_ptr(r, "r");
        if (n_p > 0) { check_ptr(Rp_p, "Rp_p"); check_ptr(dinv_p, "dinv_p", false); }
        dinv_from_r(Rp_p, n_p, D, r, dinv_p, as_stream(stream));
    });
}

int tpo_eig_from_gram(const double *G, const double *r, int64_t D, int32_t k, double *Psi64, double *sigma,
                      void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(D >= 1 && k >= 1 && k <= D && k <= 128, "need 1 <= k <= min(D, 128)");
        check_ptr(G, "G");
        check_ptr(r, "r");
        check_ptr(Psi64, "Psi64");
        TPO_REQUIRE(sigma != nullptr, "sigma (host) is NULL");
        check_ws(ws, ws_bytes, eig_from_gram_ws(D, k));
        Arena ar(ws, ws_bytes);
        eig_from_gram(G, r, D, k, Psi64, sigma, ar, as_stream(stream));
    });
}

int tpo_shard_gamma(const float *Rp_p, const float *dinv_p, int64_t n_p, int64_t D, int32_t k, const double *Psi64,
                    const double *sigma, double *Gamma64_p, void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n_p >= 0 && D >= 1 && k >= 1, "bad shapes");
        check_ptr(Psi64, "Psi64");
        TPO_REQUIRE(sigma != nullptr, "sigma (host) is NULL");
        if (n_p > 0) { check_ptr(Rp_p, "Rp_p"); check_ptr(dinv_p, "dinv_p", false); check_ptr(Gamma64_p, "Gamma64_p"); }
        Arena ar(ws, ws_bytes);
        gamma_rows(Rp_p, dinv_p, n_p, D, k, Psi64, sigma, Gamma64_p, ar, as_stream(stream));
    });
}

int tpo_shard_atb64(const double *A_p, const double *B_p, int64_t n_p, int32_t k, double *out, void *ws,
                    size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n_p >= 0 && k >= 1, "bad shapes");
        check_ptr(out, "out");
        cudaStream_t st = as_stream(stream);
        if (n_p == 0) {
            TPO_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * k * k, st));
            return;
        }
        check_ptr(A_p, "A_p");
        check_ptr(B_p, "B_p");
        Arena ar(ws, ws_bytes);
        if (ts64_enabled() && k <= 104) ts_atb_f64(A_p, k, B_p, k, n_p, k, k, out, ar, st);
        else dgemm(true, k, k, n_p, 1.0, A_p, k, B_p, k, 0.0, out, k, ar, st);
    });
}

int tpo_shard_apply_chol(double *X_p, int64_t n_p, int32_t k, const double *g, void *ws, size_t ws_bytes,
                         void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n_p >= 0 && k >= 1, "bad shapes");
        check_ptr(g, "g");
        if (n_p > 0) check_ptr(X_p, "X_p");
        Arena ar(ws, ws_bytes);
        apply_chol(X_p, n_p, k, g, ar, as_stream(stream));
    });
}

int tpo_shard_colstats(const double *A_p, int64_t n_p, int32_t k, int64_t row0, double *sum, double *abs_sum,
                       double *maxabs, int64_t *argmax, void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n_p >= 0 && k >= 1 && k <= 128, "bad shapes");
        check_ptr(sum, "sum"); check_ptr(abs_sum, "abs_sum"); check_ptr(maxabs, "maxabs"); check_ptr(argmax, "argmax");
        if (n_p > 0) check_ptr(A_p, "A_p");
        Arena ar(ws, ws_bytes);
        colstats_rows(A_p, n_p, k, row0, sum, abs_sum, maxabs, argmax, ar, as_stream(stream));
    });
}

int tpo_shard_gamma_final(double *Gamma64_p, int64_t n_p, int32_t k, const int32_t *signs, const double *Psi64,
                          int64_t D, float *Psi, float *Gamma_p, void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n_p >= 0 && k >= 1 && D >= 1, "bad shapes");
        TPO_REQUIRE(signs != nullptr, "signs (host) is NULL");
        check_ptr(Psi, "Psi");
        if (n_p > 0) { check_ptr(Gamma64_p, "Gamma64_p"); check_ptr(Gamma_p, "Gamma_p"); }
        Arena ar(ws, ws_bytes);
        gamma_final(Gamma64_p, n_p, k, reinterpret_cast<const int *>(signs), Psi, Psi64, D, Gamma_p, ar,
                    as_stream(stream));
    });
}

int tpo_shard_onmf_init(const float *Gamma_p, int64_t n_p, const float *Psi, const double *sigma, int64_t D, int32_t k,
                        double *U_p, double *H, void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n_p >= 0 && k >= 1 && D >= 1, "bad shapes");
        TPO_REQUIRE(sigma != nullptr, "sigma (host) is NULL");
        check_ptr(Psi, "Psi"); check_ptr(H, "H");
        if (n_p > 0) { check_ptr(Gamma_p, "Gamma_p"); check_ptr(U_p, "U_p"); }
        Arena ar(ws, ws_bytes);
        onmf_init(Gamma_p, n_p, Psi, sigma, D, k, U_p, H, ar, as_stream(stream));
    });
}

int tpo_shard_onmf_rtu(const float *Rp_p, const float *dinv_p, const double *U_p, int64_t n_p, int64_t D, int32_t k,
                       double *RtU_part, void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n_p >= 0 && k >= 1 && D >= 1, "bad shapes");
        check_ptr(RtU_part, "RtU_part");
        cudaStream_t st = as_stream(stream);
        if (n_p == 0) {
            TPO_CUDA(cudaMemsetAsync(RtU_part, 0, sizeof(double) * D * k, st));
            return;
        }
        check_ptr(Rp_p, "Rp_p"); check_ptr(dinv_p, "dinv_p", false); check_ptr(U_p, "U_p");
        Arena ar(ws, ws_bytes);
        onmf_rtu(Rp_p, n_p, D, dinv_p, U_p, k, RtU_part, ar, st);
    });
}

int tpo_onmf_h_update(double *H, const double *RtU, const double *UtU, int64_t D, int32_t k, void *ws,
                      size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(D >= 1 && k >= 1, "bad shapes");
        check_ptr(H, "H"); check_ptr(RtU, "RtU"); check_ptr(UtU, "UtU");
        Arena ar(ws, ws_bytes);
        onmf_h_update(H, RtU, UtU, D, k, ar, as_stream(stream));
    });
}

size_t tpo_rowgemm_f64_ws(int64_t n, int64_t K, int32_t N) {
    if (n < 0 || K < 1 || N < 1) return 0;
    return align_up(sizeof(int32_t) * (size_t)std::max<int64_t>(n, 1)) + oz_aw_ws(K, N) + 1024;
}

int tpo_rowgemm_f64(const float *A, int64_t n, int64_t K, const float *rs, const double *W, int32_t N, double *out,
                    void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n >= 0 && K >= 1 && N >= 1 && K % 4 == 0, "bad shapes (K % 4 == 0 required)");
        check_ptr(W, "W");
        if (n == 0) return;
        check_ptr(A, "A"); check_ptr(out, "out");
        cudaStream_t st = as_stream(stream);
        if (oz_enabled() && oz_aw_supported(K, N)) {
            Arena ar(ws, ws_bytes);
            int32_t *rowE = ar.take<int32_t>(n);
            oz_rowexp(A, K, n, (int)K, rowE, st);
            oz_aw_f64(A, K, rs, rowE, W, n, (int)K, N, out, N, ar, st);
        } else {
            tsgemm_AW_f64(A, K, rs, W, n, K, N, out, N, st);
        }
    });
}

int tpo_shard_onmf_rh(const float *Rp_p, const float *dinv_p, const double *H, int64_t n_p, int64_t D, int32_t k,
                      double *RH_p, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n_p >= 0 && k >= 1 && D >= 1, "bad shapes");
        check_ptr(H, "H");
        if (n_p == 0) return;
        check_ptr(Rp_p, "Rp_p"); check_ptr(dinv_p, "dinv_p", false); check_ptr(RH_p, "RH_p");
        tsgemm_AW_f64(Rp_p, D, dinv_p, H, n_p, D, k, RH_p, k, as_stream(stream));
    });
}

int tpo_shard_onmf_u_update(double *U_p, const double *RH_p, const double *M, int64_t n_p, int32_t k, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n_p >= 0 && k >= 1 && k <= 128, "bad shapes");
        check_ptr(M, "M");
        if (n_p == 0) return;
        check_ptr(U_p, "U_p"); check_ptr(RH_p, "RH_p");
        onmf_u_update(U_p, RH_p, M, n_p, k, as_stream(stream));
    });
}

int tpo_shard_nci_assign(const double *U_p, const double *Phi, int64_t n_p, int32_t k, int32_t *labels_p,
                         int32_t *changed, double *sums, double *counts, void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(n_p >= 0 && k >= 1 && k <= 128, "bad shapes");
        check_ptr(Phi, "Phi"); check_ptr(changed, "changed", false); check_ptr(sums, "sums"); check_ptr(counts, "counts");
        if (n_p > 0) { check_ptr(U_p, "U_p"); check_ptr(labels_p, "labels_p", false); }
        check_ws(ws, ws_bytes, nci_assign_part_ws(n_p, k));
        Arena ar(ws, ws_bytes);
        nci_assign_part(U_p, Phi, n_p, k, labels_p, changed, sums, counts, ar, as_stream(stream));
    });
}

int tpo_nci_phi(const double *sums, const double *counts, int32_t k, double *Phi, void *stream) {
    return guarded([&] {
        TPO_REQUIRE(k >= 1, "bad k");
        check_ptr(sums, "sums"); check_ptr(counts, "counts"); check_ptr(Phi, "Phi");
        nci_phi(sums, counts, k, Phi, as_stream(stream));
    });
}

// SMs left to the Haar rotation while the first (persistent) propagation kernels run beside
// it; TPO_HAAR_RESERVE="sms,launches" overrides (tuning)
static void haar_reserve(int &sms, int &launches) {
    sms = 16;
    launches = 1 << 30;
    if (const char *e = getenv("TPO_HAAR_RESERVE")) {
        int a = 0, b = 0;
        if (sscanf(e, "%d,%d", &a, &b) == 2 && a >= 0 && b >= 0) { sms = a; launches = b; }
    }
}

// The whole path on device inputs (B, Bt, X, G).  The Haar side stream starts after `g_ready`
// (recorded on `st` once G is on the device); with `haar_first` its kernels are queued before
// the propagation's (host inputs: the Haar QR runs while the CSRs and X are still being copied).
struct RunRes {   // events and the Haar side stream of tpo_run / tpo_run_host (see run_res)
    cudaEvent_t ev[5] = {}, join = nullptr, g_ready = nullptr, x_done = nullptr, b_ready = nullptr;
    cudaStream_t side = nullptr, copy = nullptr;
    RunRes() {
        for (auto &e : ev) TPO_CUDA(cudaEventCreate(&e));
        TPO_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
        TPO_CUDA(cudaEventCreateWithFlags(&g_ready, cudaEventDisableTiming));
        TPO_CUDA(cudaEventCreateWithFlags(&x_done, cudaEventDisableTiming));
        TPO_CUDA(cudaEventCreateWithFlags(&b_ready, cudaEventDisableTiming));
        TPO_CUDA(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
        int lo = 0, hi = 0;   // highest priority: the latency-bound Haar chain interleaves with the SpMMs
        TPO_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        TPO_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, hi));
    }
    ~RunRes() {
        for (auto &e : ev) if (e) cudaEventDestroy(e);
        if (join) cudaEventDestroy(join);
        if (g_ready) cudaEventDestroy(g_ready);
        if (x_done) cudaEventDestroy(x_done);
        if (b_ready) cudaEventDestroy(b_ready);
        if (side) cudaStreamDestroy(side);
        if (copy) cudaStreamDestroy(copy);
    }
};

// One RunRes per (host thread, device), created on first use and reused: no event / stream
// creation inside a timed call.
static RunRes &run_res() {
    int dev = 0;
    TPO_CUDA(cudaGetDevice(&dev));
    thread_local std::map<int, std::unique_ptr<RunRes>> cache;
    auto &r = cache[dev];
    if (!r) r.reset(new RunRes());
    return *r;
}

static void run_body(const tpo_csr_t *B, const tpo_csr_t *Bt, const float *X, int64_t d, float alpha, int32_t T,
                     int32_t k, const double *G, bool haar_first, cudaEvent_t g_ready, int32_t eig_mode,
                     const float *Omega, int32_t p, int32_t q, int32_t Tf, int32_t Tg, int32_t *labels,
                     double *timings_ms, Arena &ar, cudaStream_t st, RunRes &res, int res_sms, int res_launches,
                     cudaEvent_t b_cols_ready = nullptr) {
    const int64_t n = B->n_rows, D = 2 * d;
    float *Z = ar.take<float>(n * d), *Zh = ar.take<float>(n * d);
    float *Rp = ar.take<float>(n * D), *dinv = ar.take<float>(n);
    float *Qd = ar.take<float>(d * d);
    float *Gamma = ar.take<float>(n * k), *Psi = ar.take<float>(D * k);
    double *r = ar.take<double>(D);
    int32_t *rowE = ar.take<int32_t>(n);
    uint32_t *featmax = ar.take<uint32_t>(D);
    double *s_colsum = ar.take<double>(D);
    const size_t haar_bytes = align_up(haar_q_ws_bytes(d));
    Arena har(ar.dry ? nullptr : ar.base + ar.off, haar_bytes);
    ar.take<char>(haar_bytes - 256);
    const size_t mark = ar.off;
    cudaEvent_t *ev = res.ev;
    cudaEvent_t join = res.join;
    cudaStream_t side = res.side;
    // Alg. 1 L6-7 depends only on G: it runs on a side stream beside the propagation.  With
    // device inputs the propagation is queued first, so its persistent kernels take their SMs
    // (all but the reserved ones) before the Haar kernels arrive.
    auto haar = [&] {
        TPO_CUDA(cudaStreamWaitEvent(side, g_ready, 0));
        haar_q_device(G, true, d, Qd, har, side);
        TPO_CUDA(cudaEventRecord(join, side));
    };
    if (haar_first) haar();
    propagate_impl(*B, *Bt, X, d, alpha, T, Z, Zh, ar, st, res_sms, res_launches, b_cols_ready);
    ar.off = mark;
    if (!haar_first) haar();
    TPO_CUDA(cudaEventRecord(ev[1], st));
    TPO_CUDA(cudaStreamWaitEvent(st, join, 0));
    RStats rs;                  // R''s row exponents / feature maxima (in the dinv pass), shared by a7 and a8
    if (oz_rstats_wanted(n, D, k)) {
        features_impl(Zh, n, d, Qd, Rp, dinv, r, ar, st, rowE, featmax, s_colsum);
        rs.rowE = rowE;
        rs.featmax = featmax;
        rs.s_colsum = s_colsum;
    } else {
        features_impl(Zh, n, d, Qd, Rp, dinv, r, ar, st);
    }
    ar.off = mark;
    TPO_CUDA(cudaEventRecord(ev[2], st));
    std::vector<double> sig(k);
    topk_eig_impl(Rp, dinv, n, D, k, eig_mode, p, q, Omega, Gamma, sig.data(), Psi, ar, st, r, rs);
    ar.off = mark;
    TPO_CUDA(cudaEventRecord(ev[3], st));
    cluster_impl(Rp, dinv, n, D, k, Gamma, sig.data(), Psi, Tf, Tg, labels, nullptr, ar, st, rs);
    TPO_CUDA(cudaEventRecord(ev[4], st));
    TPO_CUDA(cudaStreamSynchronize(st));
    if (timings_ms)
        for (int i = 0; i < 4; ++i) {
            float ms = 0.f;
            TPO_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
            timings_ms[i] = ms;
        }
}

static void check_run(const tpo_csr_t *B, int64_t d, int32_t k) {
    const int64_t n = B->n_rows, D = 2 * d;
    TPO_REQUIRE(n >= 1, "empty U side");
    TPO_REQUIRE(k >= 1 && k <= 128 && k <= n && k <= D, "k must lie in [1, min(n, 2d, 128)]");
}

int tpo_run(const tpo_csr_t *B, const tpo_csr_t *Bt, const float *X, int64_t d, float alpha, int32_t T, int32_t k,
            const double *G, int32_t eig_mode, const float *Omega, int32_t p, int32_t q, int32_t Tf, int32_t Tg,
            int32_t *labels, double *timings_ms, void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        check_propagate(B, Bt, X, d, alpha, T, X, nullptr);
        check_ptr(G, "G");
        check_run(B, d, k);
        check_ptr(labels, "labels");
        check_ws(ws, ws_bytes, tpo_run_ws(B->n_rows, B->n_cols, B->nnz, d, k, eig_mode, p));
        cudaStream_t st = as_stream(stream);
        Arena ar(ws, ws_bytes);
        RunRes &res = run_res();
        TPO_CUDA(cudaEventRecord(res.ev[0], st));
        int res_sms = 0, res_launches = 0;
        haar_reserve(res_sms, res_launches);
        run_body(B, Bt, X, d, alpha, T, k, G, false, res.ev[0], eig_mode, Omega, p, q, Tf, Tg, labels, timings_ms, ar,
                 st, res, res_sms, res_launches);
    });
}

size_t tpo_run_host_ws(int64_t n_u, int64_t n_v, int64_t nnz, int64_t d, int32_t k, int32_t mode, int32_t p,
                       int32_t weighted) {
    size_t s = align_up(sizeof(int64_t) * (n_u + 1)) + align_up(sizeof(int64_t) * (n_v + 1));
    s += 2 * align_up(sizeof(int32_t) * nnz);
    if (weighted) s += 2 * align_up(sizeof(float) * nnz);
    s += align_up(sizeof(float) * n_u * d) + align_up(sizeof(double) * d * d) + align_up(sizeof(int32_t) * n_u);
    return s + tpo_run_ws(n_u, n_v, nnz, d, k, mode, p) + 8 * 256;
}

int tpo_run_host(const tpo_csr_t *B, const tpo_csr_t *Bt, const float *X, int64_t d, float alpha, int32_t T,
                 int32_t k, const double *G, int32_t eig_mode, const float *Omega, int32_t p, int32_t q, int32_t Tf,
                 int32_t Tg, int32_t *labels, double *timings_ms, void *ws, size_t ws_bytes, void *stream) {
    return guarded([&] {
        check_propagate(B, Bt, X, d, alpha, T, X, nullptr);
        TPO_REQUIRE(G != nullptr, "G is NULL");
        TPO_REQUIRE(labels != nullptr, "labels is NULL");
        TPO_REQUIRE((B->val == nullptr) == (Bt->val == nullptr), "B and Bt must both carry weights or neither");
        check_run(B, d, k);
        const int64_t n = B->n_rows, m = B->n_cols, nnz = B->nnz;
        const int weighted = B->val != nullptr;
        check_ws(ws, ws_bytes, tpo_run_host_ws(n, m, nnz, d, k, eig_mode, p, weighted));
        cudaStream_t st = as_stream(stream);
        Arena ar(ws, ws_bytes);
        int64_t *brp = ar.take<int64_t>(n + 1), *trp = ar.take<int64_t>(m + 1);
        int32_t *bci = ar.take<int32_t>(nnz), *tci = ar.take<int32_t>(nnz);
        float *bv = weighted ? ar.take<float>(nnz) : nullptr, *tv = weighted ? ar.take<float>(nnz) : nullptr;
        float *Xd = ar.take<float>(n * d);
        double *Gd = ar.take<double>(d * d);
        int32_t *lab = ar.take<int32_t>(n);
        RunRes &res = run_res();
        TPO_CUDA(cudaEventRecord(res.ev[0], st));
        // inputs in the order the path consumes them: G (the Haar QR starts as soon as it lands;
        // the copy engine serves the copies in issue order), the CSRs (degrees, schedules), X
        auto h2d = [&](void *dst, const void *src, size_t bytes) {
            if (bytes) TPO_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        };
        h2d(Gd, G, sizeof(double) * d * d);
        TPO_CUDA(cudaEventRecord(res.g_ready, st));
        h2d(brp, B->row_ptr, sizeof(int64_t) * (n + 1));
        // unweighted: B's column ids are first read by hop 1's U-side SpMM, so they are copied on a
        // side copy stream after X, during the degrees, schedules and hop 1's V-side SpMM
        if (weighted) h2d(bci, B->col_idx, sizeof(int32_t) * nnz);
        h2d(trp, Bt->row_ptr, sizeof(int64_t) * (m + 1));
        h2d(tci, Bt->col_idx, sizeof(int32_t) * nnz);
        if (weighted) {
            h2d(bv, B->val, sizeof(float) * nnz);
            h2d(tv, Bt->val, sizeof(float) * nnz);
        }
        h2d(Xd, X, sizeof(float) * n * d);
        cudaEvent_t b_cols_ready = nullptr;
        if (!weighted && nnz > 0) {
            TPO_CUDA(cudaEventRecord(res.x_done, st));
            TPO_CUDA(cudaStreamWaitEvent(res.copy, res.x_done, 0));
            TPO_CUDA(cudaMemcpyAsync(bci, B->col_idx, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, res.copy));
            TPO_CUDA(cudaEventRecord(res.b_ready, res.copy));
            b_cols_ready = res.b_ready;
        }
        const tpo_csr_t Bd{n, m, nnz, brp, bci, bv}, Btd{m, n, nnz, trp, tci, tv};
        // the Haar rotation runs during the input copies: no SMs are held back for it
        int res_sms = 0, res_launches = 0;
        if (const char *e = getenv("TPO_HOST_RESERVE")) {
            int a = 0, b = 0;
            if (sscanf(e, "%d,%d", &a, &b) == 2 && a >= 0 && b >= 0) { res_sms = a; res_launches = b; }
        }
        run_body(&Bd, &Btd, Xd, d, alpha, T, k, Gd, true, res.g_ready, eig_mode, Omega, p, q, Tf, Tg, lab, timings_ms,
                 ar, st, res, res_sms, res_launches, b_cols_ready);
        if (b_cols_ready) TPO_CUDA(cudaStreamWaitEvent(st, b_cols_ready, 0));   // joined even when T = 0
        TPO_CUDA(cudaMemcpyAsync(labels, lab, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
        TPO_CUDA(cudaStreamSynchronize(st));
    });
}

}  // extern "C"
