// Library-owned NCCL communicator and the sharded propagation with its collectives inside the
// library (SURVEY.md §8b "tpo_comm_create / tpo_comm_destroy / *_sharded(comm)", §8e).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2: the copy the process already loaded, e.g.
// PyTorch's, else the system one), so libtpo.so carries no link-time NCCL dependency and loads on
// machines without it; only tpo_comm_* and tpo_propagate_sharded need it.
//
// tpo_propagate_sharded runs, on the caller's stream, exactly the exchange of SURVEY.md §8e:
//   deg_v <- ncclAllReduce(sum) of the shard partials                              (once)
//   per hop:  Qpart = B_p^T P_p (m x d)  ->  ncclReduceScatter(sum) over V slices
//             Qslice *= s_v^2            ->  ncclAllGather  ->  U side of the rank's rows
// (Eq. update-Z, bracketed L (L^T Z)).
#include <dlfcn.h>
#include <nccl.h>

#include <math.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "tpo_internal.cuh"

namespace tpo {
namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*ReduceScatter)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    const char *(*GetErrorString)(ncclResult_t);
};

const NcclApi &nccl() {
    static NcclApi api{};
    static std::string err;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);   // already loaded (torch)?
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = "libnccl.so.2 not found";
            return;
        }
        auto sym = [&](const char *name) {
            void *p = dlsym(h, name);
            if (!p) err = std::string("NCCL symbol missing: ") + name;
            return p;
        };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
        api.ReduceScatter = reinterpret_cast<decltype(api.ReduceScatter)>(sym("ncclReduceScatter"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    });
    if (!err.empty()) throw Error(TPO_ENCCL, err);
    return api;
}

#define TPO_NCCL(call)                                                                                  \
    do {                                                                                                \
        ncclResult_t _r = (call);                                                                       \
        if (_r != ncclSuccess) throw ::tpo::Error(TPO_ENCCL, std::string(#call) + ": " + nccl().GetErrorString(_r)); \
    } while (0)

struct Comm {
    ncclComm_t nc;
    int rank, world, device;
};

}  // namespace

void comm_unique_id(void *id) {
    ncclUniqueId u;
    TPO_NCCL(nccl().GetUniqueId(&u));
    memcpy(id, &u, sizeof(u));
}

void *comm_create(const void *id, int rank, int world, int device) {
    const NcclApi &api = nccl();
    ncclUniqueId u;
    memcpy(&u, id, sizeof(u));
    TPO_CUDA(cudaSetDevice(device));
    Comm *c = new Comm{nullptr, rank, world, device};
    const ncclResult_t r = api.CommInitRank(&c->nc, world, u, rank);
    if (r != ncclSuccess) {
        delete c;
        throw Error(TPO_ENCCL, std::string("ncclCommInitRank: ") + api.GetErrorString(r));
    }
    return c;
}

void comm_destroy(void *comm) {
    Comm *c = static_cast<Comm *>(comm);
    if (!c) return;
    const ncclResult_t r = nccl().CommDestroy(c->nc);
    delete c;
    if (r != ncclSuccess) throw Error(TPO_ENCCL, std::string("ncclCommDestroy: ") + nccl().GetErrorString(r));
}

int comm_world(const void *comm) { return static_cast<const Comm *>(comm)->world; }
int comm_rank(const void *comm) { return static_cast<const Comm *>(comm)->rank; }

size_t propagate_sharded_ws_bytes(int64_t n_p, int64_t m, int64_t nnz_p, int64_t d, int world) {
    const int64_t mp = (m + world - 1) / world;
    Arena ar(nullptr, 0);
    ar.take<double>(n_p);                     // deg_u
    ar.take<double>(m);                       // deg_v
    ar.take<float>(n_p);                      // s_u
    ar.take<float>(m);                        // s_v
    ar.take<float>(mp * world);               // s_v padded
    ar.take<float>(mp * world * d);           // Qpart
    ar.take<float>(mp * d);                   // Qslice
    ar.take<float>(mp * world * d);           // Q
    return ar.off + std::max(shard_spmm_ws_bytes(m, nnz_p, d), shard_spmm_ws_bytes(n_p, nnz_p, d)) + 1024;
}

void propagate_sharded_impl(void *comm, const tpo_csr_t &Bp, const tpo_csr_t &Btp, const float *Xp, int64_t d,
                            float alpha, int32_t T, float *Zp, float *Zhat_p, Arena &ar, cudaStream_t st) {
    Comm *c = static_cast<Comm *>(comm);
    const NcclApi &api = nccl();
    const int64_t n_p = Bp.n_rows, m = Bp.n_cols;
    const int world = c->world;
    const int64_t mp = (m + world - 1) / world;
    double *deg_u = ar.take<double>(n_p), *deg_v = ar.take<double>(m);
    float *s_u = ar.take<float>(n_p), *s_v = ar.take<float>(m), *s_v_pad = ar.take<float>(mp * world);
    float *Qpart = ar.take<float>(mp * world * d), *Qslice = ar.take<float>(mp * d), *Q = ar.take<float>(mp * world * d);
    const size_t mark = ar.off;
    shard_degrees_impl(Bp, Btp, deg_u, deg_v, st);
    TPO_NCCL(api.AllReduce(deg_v, deg_v, (size_t)m, ncclFloat64, ncclSum, c->nc, st));     // global D_V
    // s_u, s_v and P_0 = s_u (c X) into Zp (the iterate lives in Zp's buffer)
    shard_start_impl(deg_u, deg_v, n_p, m, Xp, d, alpha, s_u, s_v, Zp, st);
    if (T == 0) {                                  // no exchange: Z = c X, Zhat = rownorm(X)
        propagate_local_t0(Xp, n_p, d, alpha, Zp, Zhat_p, st);
        return;
    }
    TPO_CUDA(cudaMemsetAsync(s_v_pad, 0, sizeof(float) * mp * world, st));
    TPO_CUDA(cudaMemcpyAsync(s_v_pad, s_v, sizeof(float) * m, cudaMemcpyDeviceToDevice, st));
    TPO_CUDA(cudaMemsetAsync(Qpart, 0, sizeof(float) * mp * world * d, st));   // padding rows stay zero
    for (int t = 0; t < T; ++t) {
        const bool last = t == T - 1;
        shard_vside_impl(Btp, Zp, d, Qpart, ar, st);
        ar.off = mark;
        TPO_NCCL(api.ReduceScatter(Qpart, Qslice, (size_t)(mp * d), ncclFloat32, ncclSum, c->nc, st));
        shard_vscale_impl(Qslice, s_v_pad + (int64_t)c->rank * mp, mp, d, st);
        TPO_NCCL(api.AllGather(Qslice, Q, (size_t)(mp * d), ncclFloat32, c->nc, st));
        shard_uside_impl(Bp, Q, Xp, d, alpha, s_u, last, Zp, last ? Zhat_p : nullptr, ar, st);
        ar.off = mark;
    }
}

// ---------------------------------------------------------------------------------------
// The whole hot path on a rank's U slice with every collective inside the library (SURVEY.md
// §8e "an all-reduce of the d x k Gram matrices"): sharded propagation, then a5-a9 with the fp64
// partials all-reduced in between -- r, the Gram R^T R, Gamma^T Gamma for the CholeskyQR polish
// (and its decision), the sign rule's column statistics (all-reduce) and largest-magnitude entries
// (all-gather; R8 applied identically on every rank), R'^T Ups, Ups^T Ups, Ups^T (R H) per Alg. 2
// iteration, and the cluster sums, counts and changed flag per Alg. 3 iteration.  Every D x D,
// D x k and k x k quantity is replicated, so each rank's steps are the single-GPU ones.
// ---------------------------------------------------------------------------------------
namespace {
__global__ void eye_f64_kernel(double *P, int k) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < k * k) P[i] = (i / k == i % k) ? 1.0 : 0.0;
}
__global__ void fill_i32_kernel(int32_t *p, int64_t n, int32_t v) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}
}  // namespace

size_t run_sharded_ws_bytes(int64_t n_p, int64_t m, int64_t nnz_p, int64_t d, int32_t k, int world) {
    const int64_t D = 2 * d;
    size_t s = propagate_sharded_ws_bytes(n_p, m, nnz_p, d, world);
    s += 2 * align_up(sizeof(float) * (size_t)n_p * d) + align_up(sizeof(float) * (size_t)d * d);
    s += align_up(sizeof(float) * (size_t)n_p * D) + align_up(sizeof(float) * (size_t)n_p + 1) + align_up(sizeof(double) * D);
    s += align_up(sizeof(double) * (size_t)D * D) + 3 * align_up(sizeof(double) * (size_t)D * k) + align_up(sizeof(float) * D * k);
    s += 3 * align_up(sizeof(double) * (size_t)n_p * k) + align_up(sizeof(float) * (size_t)n_p * k);
    s += 8 * align_up(sizeof(double) * (size_t)k * k) + 8 * align_up(sizeof(double) * (size_t)k) + 1024;
    s += rh_plan_ws(n_p) + align_up(sizeof(uint32_t) * (size_t)D + 1);
    size_t inner = std::max(features_ws_bytes(n_p, d), gram_tc_ws(std::max<int64_t>(n_p, 1), D));
    inner = std::max(inner, eig_from_gram_ws(D, k));
    inner = std::max(inner, haar_q_ws_bytes(d));
    inner = std::max(inner, nci_assign_part_ws(n_p, k));
    inner = std::max(inner, onmf_ws_bytes(n_p, D, k));
    inner = std::max(inner, rh_apply_ws(D, k));
    inner = std::max(inner, ts_atb_ws(k, k) + dgemm_ws(k, k, std::max<int64_t>(n_p, 1)));
    inner = std::max(inner, dgemm_ws(k, k, D));
    inner = std::max(inner, align_up(sizeof(double) * (size_t)(4 * 2 * 148 * k)) + 4096);
    return s + inner + 64 * 256;
}

void run_sharded_impl(void *comm, const tpo_csr_t &Bp, const tpo_csr_t &Btp, const float *Xp, int64_t d, float alpha,
                      int32_t T, int32_t k, const double *Gdev, int64_t row0, int32_t Tf, int32_t Tg, int32_t *labels_p,
                      int32_t *iters_used, double *timings_ms, Arena &ar, cudaStream_t st) {
    Comm *c = static_cast<Comm *>(comm);
    const NcclApi &api = nccl();
    const int64_t n_p = Bp.n_rows, D = 2 * d;
    const int world = c->world;
    cudaEvent_t ev[5];
    for (auto &e : ev) TPO_CUDA(cudaEventCreate(&e));
    auto allreduce = [&](double *p, size_t len) { TPO_NCCL(api.AllReduce(p, p, len, ncclFloat64, ncclSum, c->nc, st)); };
    float *Zp = ar.take<float>(n_p * d), *Zh = ar.take<float>(n_p * d), *Q = ar.take<float>(d * d);
    float *Rp = ar.take<float>(n_p * D), *dinv = ar.take<float>(n_p + 1);
    double *r = ar.take<double>(D), *Gd = ar.take<double>(D * D), *Psi64 = ar.take<double>(D * k);
    double *RtU = ar.take<double>(D * k), *H = ar.take<double>(D * k);
    float *Psi = ar.take<float>(D * k);
    double *G64 = ar.take<double>(n_p * k), *U = ar.take<double>(n_p * k), *RH = ar.take<double>(n_p * k);
    float *Gam = ar.take<float>(n_p * k);
    double *g = ar.take<double>(k * k), *UtU = ar.take<double>(k * k), *M = ar.take<double>(k * k),
           *Phi = ar.take<double>(k * k), *sums = ar.take<double>(k * k);
    double *cs = ar.take<double>(k), *ca = ar.take<double>(k), *cmax = ar.take<double>(k), *counts = ar.take<double>(k);
    int64_t *carg = ar.take<int64_t>(k);
    double *vals_all = ar.take<double>((size_t)world * k);
    int64_t *idx_all = ar.take<int64_t>((size_t)world * k);
    int32_t *changed = ar.take<int32_t>(2);
    int32_t *rowE = ar.take<int32_t>(std::max<int64_t>(n_p, 1));
    uint32_t *featmax = ar.take<uint32_t>(D);           // R''s per-feature maxima (oz R^T Ups), once per solve
    const size_t mark = ar.off;
    auto atb = [&](const double *A, const double *B, double *out) {
        if (n_p == 0) { TPO_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * k * k, st)); return; }
        if (ts64_enabled() && k <= 104) ts_atb_f64(A, k, B, k, n_p, k, k, out, ar, st);
        else dgemm(true, k, k, n_p, 1.0, A, k, B, k, 0.0, out, k, ar, st);
        ar.off = mark;
    };
    TPO_CUDA(cudaEventRecord(ev[0], st));
    // a1-a3
    propagate_sharded_impl(comm, Bp, Btp, Xp, d, alpha, T, Zp, Zh, ar, st);
    ar.off = mark;
    TPO_CUDA(cudaEventRecord(ev[1], st));
    // a4-a5: Q replicated from G; R'_p, r (all-reduce), dinv_p
    haar_q_device(Gdev, true, d, Q, ar, st);
    ar.off = mark;
    features_part(Zh, n_p, d, Q, Rp, r, ar, st);
    ar.off = mark;
    allreduce(r, (size_t)D);
    if (n_p > 0) dinv_from_r(Rp, n_p, D, r, dinv, st);
    TPO_CUDA(cudaEventRecord(ev[2], st));
    // a7: Gram (all-reduce), replicated eigensolve, Gamma rows, polish, sign rule
    if (n_p > 0) gram_tc(Rp, dinv, n_p, D, Gd, ar, st);
    else TPO_CUDA(cudaMemsetAsync(Gd, 0, sizeof(double) * D * D, st));
    ar.off = mark;
    allreduce(Gd, (size_t)(D * D));
    std::vector<double> sigma(k);
    eig_from_gram(Gd, r, D, k, Psi64, sigma.data(), ar, st);
    ar.off = mark;
    gamma_rows(Rp, dinv, n_p, D, k, Psi64, sigma.data(), G64, ar, st);
    ar.off = mark;
    std::vector<double> gh((size_t)k * k);
    for (int p = 0; p < 3; ++p) {                         // CholeskyQR polish while ||G^T G - I|| > 1e-6
        atb(G64, G64, g);
        allreduce(g, (size_t)k * k);
        TPO_CUDA(cudaMemcpyAsync(gh.data(), g, sizeof(double) * k * k, cudaMemcpyDeviceToHost, st));
        TPO_CUDA(cudaStreamSynchronize(st));
        double dev = 0.0;
        for (int i = 0; i < k; ++i)
            for (int j = 0; j < k; ++j) dev = std::max(dev, fabs(gh[(size_t)i * k + j] - (i == j ? 1.0 : 0.0)));
        if (dev <= 1e-6 || p == 2) break;
        apply_chol(G64, n_p, k, g, ar, st);
        ar.off = mark;
    }
    colstats_rows(G64, n_p, k, row0, cs, ca, cmax, carg, ar, st);
    ar.off = mark;
    allreduce(cs, (size_t)k);
    allreduce(ca, (size_t)k);
    TPO_NCCL(api.AllGather(cmax, vals_all, (size_t)k, ncclFloat64, c->nc, st));
    TPO_NCCL(api.AllGather(carg, idx_all, (size_t)k, ncclInt64, c->nc, st));
    std::vector<double> hs(k), ha(k), hv((size_t)world * k);
    std::vector<int64_t> hi((size_t)world * k);
    TPO_CUDA(cudaMemcpyAsync(hs.data(), cs, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    TPO_CUDA(cudaMemcpyAsync(ha.data(), ca, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    TPO_CUDA(cudaMemcpyAsync(hv.data(), vals_all, sizeof(double) * world * k, cudaMemcpyDeviceToHost, st));
    TPO_CUDA(cudaMemcpyAsync(hi.data(), idx_all, sizeof(int64_t) * world * k, cudaMemcpyDeviceToHost, st));
    TPO_CUDA(cudaStreamSynchronize(st));
    std::vector<int> signs(k, 1);                          // R8 from the global statistics
    for (int l = 0; l < k; ++l) {
        if (fabs(hs[l]) < 1e-6 * ha[l]) {
            double best = -1.0, bv = 0.0;
            int64_t bi = INT64_MAX;
            for (int q = 0; q < world; ++q) {
                const double mv = fabs(hv[(size_t)q * k + l]);
                const int64_t iv = hi[(size_t)q * k + l];
                if (mv > best || (mv == best && iv < bi)) { best = mv; bi = iv; bv = hv[(size_t)q * k + l]; }
            }
            signs[l] = bv < 0.0 ? -1 : 1;
        } else {
            signs[l] = hs[l] < 0.0 ? -1 : 1;
        }
    }
    gamma_final(G64, n_p, k, signs.data(), Psi, Psi64, D, Gam, ar, st);
    ar.off = mark;
    TPO_CUDA(cudaEventRecord(ev[3], st));
    // a8 (Alg. 2)
    onmf_init(Gam, n_p, Psi, sigma.data(), D, k, U, H, ar, st);
    ar.off = mark;
    const RhPlan rhp = rh_plan_at(rowE, Rp, n_p, D, k, st);
    if (oz_rtu_supported(n_p, D, k)) oz_featmax(Rp, n_p, D, featmax, st);
    else featmax = nullptr;
    for (int t = 0; t < Tf; ++t) {
        if (n_p > 0) onmf_rtu(Rp, n_p, D, dinv, U, k, RtU, ar, st, featmax);
        else TPO_CUDA(cudaMemsetAsync(RtU, 0, sizeof(double) * D * k, st));
        ar.off = mark;
        allreduce(RtU, (size_t)(D * k));
        atb(U, U, UtU);
        allreduce(UtU, (size_t)k * k);
        onmf_h_update(H, RtU, UtU, D, k, ar, st);
        ar.off = mark;
        rh_apply(rhp, Rp, dinv, H, n_p, D, k, RH, ar, st);
        ar.off = mark;
        // M = Ups^T R H = RtU^T H (RtU is already the all-reduced global product): no pass over
        // the rows and no all-reduce
        dgemm(true, k, k, D, 1.0, RtU, k, H, k, 0.0, M, k, ar, st);
        ar.off = mark;
        onmf_u_update(U, RH, M, n_p, k, st);
    }
    // a9 (Alg. 3)
    eye_f64_kernel<<<cdiv((int64_t)k * k, 256), 256, 0, st>>>(Phi, k);
    TPO_LAUNCH_CHECK();
    if (n_p > 0) fill_i32_kernel<<<cdiv(n_p, 256), 256, 0, st>>>(labels_p, n_p, -1);
    TPO_LAUNCH_CHECK();
    int32_t iters = 0;
    for (int t = 0; t < Tg; ++t) {
        TPO_CUDA(cudaMemsetAsync(changed, 0, sizeof(int32_t), st));
        nci_assign_part(U, Phi, n_p, k, labels_p, changed, sums, counts, ar, st);
        ar.off = mark;
        TPO_NCCL(api.AllReduce(changed, changed, 1, ncclInt32, ncclSum, c->nc, st));
        int32_t ch = 0;
        TPO_CUDA(cudaMemcpyAsync(&ch, changed, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        TPO_CUDA(cudaStreamSynchronize(st));
        ++iters;
        if (ch == 0 || t == Tg - 1) break;
        allreduce(sums, (size_t)k * k);
        allreduce(counts, (size_t)k);
        nci_phi(sums, counts, k, Phi, st);
    }
    TPO_CUDA(cudaEventRecord(ev[4], st));
    TPO_CUDA(cudaEventSynchronize(ev[4]));
    if (iters_used) *iters_used = iters;
    if (timings_ms)
        for (int i = 0; i < 4; ++i) {
            float ms = 0.f;
            TPO_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
            timings_ms[i] = ms;
        }
    for (auto &e : ev) cudaEventDestroy(e);
}

}  // namespace tpo
