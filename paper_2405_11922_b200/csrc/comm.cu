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

#include <algorithm>
#include <mutex>
#include <string>

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

}  // namespace tpo
