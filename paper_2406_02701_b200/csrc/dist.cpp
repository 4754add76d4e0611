// 2D block-cyclic schedule + NCCL (dlopen) for the distributed MPCRTile
// Cholesky.  NCCL is resolved at run time from whichever libnccl.so.2 the
// process already has (torch's) or the system one, so the library itself has
// no link-time NCCL dependency and still loads on a CPU-only machine.
#include "dist.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

namespace mpcr {

std::vector<DistAction> dist_schedule(int rank, int P, int Q, int64_t NT, const int* prec) {
    std::vector<DistAction> out;
    const int world = P * Q;
    auto p = [&](int64_t i, int64_t j) { return prec ? prec[j * NT + i] : 2; };
    for (int64_t k = 0; k < NT; ++k) {
        const int kk = static_cast<int>(k);
        const int dk = dist_owner(k, k, P, Q);
        if (dk == rank) out.push_back({DA_POTRF, kk, kk, kk, dk, p(k, k)});
        if (k + 1 == NT) break;
        if (world > 1) out.push_back({DA_BCAST_DIAG, kk, kk, kk, dk, 2});
        for (int64_t i = k + 1; i < NT; ++i)
            if (dist_owner(i, k, P, Q) == rank)
                out.push_back({DA_TRSM, kk, static_cast<int>(i), kk, rank, p(i, k)});
        if (world > 1)
            for (int64_t i = k + 1; i < NT; ++i)
                out.push_back({DA_BCAST_PANEL, kk, static_cast<int>(i), kk, dist_owner(i, k, P, Q),
                               p(i, k)});
        for (int64_t j = k + 1; j < NT; ++j)
            for (int64_t i = j; i < NT; ++i)
                if (dist_owner(i, j, P, Q) == rank)
                    out.push_back({DA_UPDATE, kk, static_cast<int>(i), static_cast<int>(j), rank,
                                   p(i, j)});
    }
    return out;
}

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = dlerror() ? dlerror() : "libnccl.so.2 not found";
            return;
        }
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(dlsym(h, "ncclBroadcast"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(h, "ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    });
    if (!api.GetUniqueId || !api.CommInitRank || !api.Broadcast || !api.AllReduce)
        fail(MP_NCCL_ERROR, "NCCL unavailable: " + (err.empty() ? std::string("missing symbols") : err));
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(MP_NCCL_ERROR, std::string(what) + ": " +
                                (nccl().GetErrorString ? nccl().GetErrorString(r) : "error"));
}

}  // namespace

void dist_bcast(Dist* d, void* buf, size_t bytes, int root, cudaStream_t s) {
    if (!d || d->world == 1) return;
    nccl_check(nccl().Broadcast(buf, buf, bytes, ncclUint8, root, static_cast<ncclComm_t>(d->comm), s),
               "ncclBroadcast");
}
void dist_group_start(Dist* d) {
    if (d && d->world > 1) nccl_check(nccl().GroupStart(), "ncclGroupStart");
}
void dist_group_end(Dist* d) {
    if (d && d->world > 1) nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
}
void dist_allreduce_min_u64(Dist* d, int64_t* buf, cudaStream_t s) {
    if (!d || d->world == 1) return;
    nccl_check(nccl().AllReduce(buf, buf, 1, ncclUint64, ncclMin, static_cast<ncclComm_t>(d->comm), s),
               "ncclAllReduce");
}
void dist_allreduce_sum_f64(Dist* d, double* buf, size_t n, cudaStream_t s) {
    if (!d || d->world == 1) return;
    nccl_check(nccl().AllReduce(buf, buf, n, ncclFloat64, ncclSum, static_cast<ncclComm_t>(d->comm), s),
               "ncclAllReduce");
}

}  // namespace mpcr

using namespace mpcr;

extern "C" {

mp_status mp_nccl_unique_id(unsigned char* out128) {
    try {
        ncclUniqueId id;
        nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out128, &id, sizeof(id));
        return MP_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.status;
    }
}

mp_status mp_dist_create(mp_ctx ctx, int rank, int world, int P, int Q, const unsigned char* uid128,
                         mp_dist* out) {
    try {
        if (!ctx || !out) fail(MP_INVALID_PARAM, "null argument");
        if (P < 1 || Q < 1 || P * Q != world || rank < 0 || rank >= world)
            fail(MP_INVALID_PARAM, "dist: need P * Q == world and 0 <= rank < world");
        auto* d = new mp_dist_s();
        d->ctx = ctx;
        d->rank = rank;
        d->world = world;
        d->P = P;
        d->Q = Q;
        if (world > 1) {
            if (!uid128) {
                delete d;
                fail(MP_INVALID_PARAM, "dist: unique id required for world > 1");
            }
            ncclUniqueId id;
            std::memcpy(&id, uid128, sizeof(id));
            ncclComm_t comm;
            MP_CUDA(cudaSetDevice(ctx->device));
            try {
                nccl_check(nccl().CommInitRank(&comm, world, id, rank), "ncclCommInitRank");
            } catch (...) {
                delete d;
                throw;
            }
            d->comm = comm;
        }
        *out = d;
        return MP_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.status;
    }
}

mp_status mp_dist_destroy(mp_dist d) {
    if (!d) return MP_OK;
    if (d->comm && nccl().CommDestroy) nccl().CommDestroy(static_cast<ncclComm_t>(d->comm));
    delete d;
    return MP_OK;
}

int mp_dist_owner(int64_t i, int64_t j, int P, int Q) { return dist_owner(i, j, P, Q); }

mp_status mp_dist_schedule(int rank, int P, int Q, int64_t NT, const int* precisions,
                           int32_t* actions, int64_t capacity, int64_t* count) {
    try {
        if (P < 1 || Q < 1 || rank < 0 || rank >= P * Q || NT < 1)
            fail(MP_INVALID_PARAM, "dist schedule: bad grid");
        const auto s = dist_schedule(rank, P, Q, NT, precisions);
        if (count) *count = static_cast<int64_t>(s.size());
        if (actions) {
            if (capacity < static_cast<int64_t>(s.size())) fail(MP_INVALID_PARAM, "dist schedule: buffer too small");
            std::memcpy(actions, s.data(), s.size() * sizeof(DistAction));
        }
        return MP_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.status;
    }
}

}  // extern "C"
