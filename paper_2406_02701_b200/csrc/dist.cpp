// 2D block-cyclic schedule + NCCL (dlopen) for the distributed MPCRTile
// Cholesky.  NCCL is resolved at run time from whichever libnccl.so.2 the
// process already has (torch's) or the system one, so the library itself has
// no link-time NCCL dependency and still loads on a CPU-only machine.
#include "dist.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <type_traits>

namespace mpcr {

std::vector<DistAction> dist_schedule(int rank, int P, int Q, int64_t NT, const int* prec) {
    std::vector<DistAction> out;
    const int world = P * Q;
    const int pr = rank / Q, pc = rank % Q;
    auto p = [&](int64_t i, int64_t j) { return prec ? prec[j * NT + i] : 2; };
    for (int64_t k = 0; k < NT; ++k) {
        const int kk = static_cast<int>(k);
        const int dk = dist_owner(k, k, P, Q);
        if (dk == rank) out.push_back({DA_POTRF, kk, kk, kk, dk, p(k, k), DC_WORLD});
        if (k + 1 == NT) break;
        // L_kk^-1 down process column k mod Q (the column's TRSM owners)
        if (P > 1 && pc == static_cast<int>(k % Q)) out.push_back({DA_BCAST_DIAG, kk, kk, kk, dk, 2, DC_COL});
        for (int64_t i = k + 1; i < NT; ++i)
            if (dist_owner(i, k, P, Q) == rank)
                out.push_back({DA_TRSM, kk, static_cast<int>(i), kk, rank, p(i, k), DC_WORLD});
        if (world > 1)
            for (int64_t i = k + 1; i < NT; ++i) {
                const int ii = static_cast<int>(i);
                // along process row i mod P from the owner (i mod P, k mod Q) ...
                if (Q > 1 && pr == static_cast<int>(i % P))
                    out.push_back({DA_BCAST_PANEL, kk, ii, kk, dist_owner(i, k, P, Q), p(i, k), DC_ROW});
                // ... then down process column i mod Q from (i mod P, i mod Q)
                if (P > 1 && pc == static_cast<int>(i % Q))
                    out.push_back({DA_BCAST_PANEL, kk, ii, kk, dist_owner(i, i, P, Q), p(i, k), DC_COL});
            }
        for (int64_t j = k + 1; j < NT; ++j)
            for (int64_t i = j; i < NT; ++i)
                if (dist_owner(i, j, P, Q) == rank)
                    out.push_back({DA_UPDATE, kk, static_cast<int>(i), static_cast<int>(j), rank, p(i, j),
                                   DC_WORLD});
    }
    return out;
}

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
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
        auto sym = [&](auto& f, const char* name) { f = reinterpret_cast<std::decay_t<decltype(f)>>(dlsym(h, name)); };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.CommAbort, "ncclCommAbort");
        sym(api.CommSplit, "ncclCommSplit");
        sym(api.CommGetAsyncError, "ncclCommGetAsyncError");
        sym(api.Broadcast, "ncclBroadcast");
        sym(api.AllReduce, "ncclAllReduce");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.GetErrorString, "ncclGetErrorString");
    });
    if (!api.GetUniqueId || !api.CommInitRank || !api.Broadcast || !api.AllReduce || !api.CommSplit)
        fail(MP_NCCL_ERROR, "NCCL unavailable: " + (err.empty() ? std::string("missing symbols") : err));
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(MP_NCCL_ERROR, std::string(what) + ": " +
                                (nccl().GetErrorString ? nccl().GetErrorString(r) : "error"));
}

}  // namespace

// ---- single-GPU simulation of the ranks ---------------------------------------
// All ranks live in one process on one GPU, each with its own context
// (streams) and host thread.  A broadcast is a device copy from the root's
// buffer, ordered by events: the receivers wait on the root's event and copy
// on their own stream; the root's stream waits until every copy is done
// before it may overwrite the buffer.  The host threads only rendezvous to
// exchange pointers and events (no kernel ever waits on another rank's).
struct SimGroup {
    int world = 1, P = 1, Q = 1;
    int refs = 0;
    std::mutex mu;
    std::condition_variable cv;
    struct Slot {
        const void* src = nullptr;
        cudaEvent_t ready = nullptr;
        int arrived = 0;
        std::vector<cudaEvent_t> done;
        std::vector<uint64_t> vals;  // allreduce: contributions (8-byte words) by rank
        int left = 0;                // allreduce: ranks that have not read the result yet
    };
    std::map<std::tuple<int, int, int>, Slot> slots;  // (comm, color, seq)
};

namespace {

int comm_color(const Dist* d, DistComm c) { return c == DC_ROW ? d->pr() : c == DC_COL ? d->pc() : 0; }
int comm_size(const Dist* d, DistComm c) { return c == DC_ROW ? d->Q : c == DC_COL ? d->P : d->world; }

void sim_bcast(Dist* d, void* buf, size_t bytes, int root, DistComm c, cudaStream_t s) {
    SimGroup& g = *d->sim;
    const auto key = std::make_tuple(static_cast<int>(c), comm_color(d, c), d->sim_seq[c]++);
    const int size = comm_size(d, c);
    std::unique_lock<std::mutex> lk(g.mu);
    SimGroup::Slot& sl = g.slots[key];
    if (d->rank == root) {
        MP_CUDA(cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming));
        MP_CUDA(cudaEventRecord(sl.ready, s));
        sl.src = buf;
        g.cv.notify_all();
        g.cv.wait(lk, [&] { return static_cast<int>(sl.done.size()) == size - 1; });
        for (cudaEvent_t e : sl.done) {
            MP_CUDA(cudaStreamWaitEvent(s, e, 0));
            cudaEventDestroy(e);
        }
        cudaEventDestroy(sl.ready);
        g.slots.erase(key);
    } else {
        g.cv.wait(lk, [&] { return sl.src != nullptr; });
        MP_CUDA(cudaStreamWaitEvent(s, sl.ready, 0));
        MP_CUDA(cudaMemcpyAsync(buf, sl.src, bytes, cudaMemcpyDeviceToDevice, s));
        cudaEvent_t e;
        MP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        MP_CUDA(cudaEventRecord(e, s));
        sl.done.push_back(e);
        g.cv.notify_all();
    }
}

// Small allreduce on the host: every rank's contribution, combined in rank order.
template <typename T, typename F>
void sim_allreduce(Dist* d, T* buf, size_t n, cudaStream_t s, F combine) {
    static_assert(sizeof(T) == sizeof(uint64_t), "8-byte words");
    SimGroup& g = *d->sim;
    std::vector<T> mine(n), out(n);
    MP_CUDA(cudaMemcpyAsync(mine.data(), buf, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    const auto key = std::make_tuple(static_cast<int>(DC_WORLD), 0, d->sim_seq[DC_WORLD]++);
    {
        std::unique_lock<std::mutex> lk(g.mu);
        SimGroup::Slot& sl = g.slots[key];
        if (sl.vals.empty()) {
            sl.vals.resize(n * g.world);
            sl.left = g.world;
        }
        std::memcpy(&sl.vals[d->rank * n], mine.data(), n * sizeof(T));
        ++sl.arrived;
        g.cv.notify_all();
        g.cv.wait(lk, [&] { return sl.arrived >= g.world; });
        for (size_t q = 0; q < n; ++q) {
            T acc, v;
            std::memcpy(&acc, &sl.vals[q], sizeof(T));
            for (int r = 1; r < g.world; ++r) {
                std::memcpy(&v, &sl.vals[r * n + q], sizeof(T));
                acc = combine(acc, v);
            }
            out[q] = acc;
        }
        if (--sl.left == 0) g.slots.erase(key);
    }
    MP_CUDA(cudaMemcpy(buf, out.data(), n * sizeof(T), cudaMemcpyHostToDevice));
}

ncclComm_t comm_of(Dist* d, DistComm c) {
    return static_cast<ncclComm_t>(c == DC_ROW ? d->row_comm : c == DC_COL ? d->col_comm : d->comm);
}

}  // namespace

void dist_bcast(Dist* d, void* buf, size_t bytes, int root, DistComm c, cudaStream_t s) {
    if (!d || d->world == 1 || comm_size(d, c) == 1) return;
    if (d->sim) {
        sim_bcast(d, buf, bytes, root, c, s);
        return;
    }
    // root's index in the sub-communicator: row members are ordered by
    // process column, column members by process row
    const int r = c == DC_ROW ? root % d->Q : c == DC_COL ? root / d->Q : root;
    nccl_check(nccl().Broadcast(buf, buf, bytes, ncclUint8, r, comm_of(d, c), s), "ncclBroadcast");
}
void dist_group_start(Dist* d) {
    if (d && d->world > 1 && !d->sim) nccl_check(nccl().GroupStart(), "ncclGroupStart");
}
void dist_group_end(Dist* d) {
    if (d && d->world > 1 && !d->sim) nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
}
void dist_allreduce_min_u64(Dist* d, int64_t* buf, cudaStream_t s) {
    if (!d || d->world == 1) return;
    if (d->sim) {
        sim_allreduce(d, reinterpret_cast<uint64_t*>(buf), 1, s, [](uint64_t a, uint64_t b) { return a < b ? a : b; });
        return;
    }
    nccl_check(nccl().AllReduce(buf, buf, 1, ncclUint64, ncclMin, static_cast<ncclComm_t>(d->comm), s),
               "ncclAllReduce");
}
void dist_allreduce_sum_f64(Dist* d, double* buf, size_t n, cudaStream_t s) {
    if (!d || d->world == 1) return;
    if (d->sim) {
        sim_allreduce(d, buf, n, s, [](double a, double b) { return a + b; });
        return;
    }
    nccl_check(nccl().AllReduce(buf, buf, n, ncclFloat64, ncclSum, static_cast<ncclComm_t>(d->comm), s),
               "ncclAllReduce");
}

void dist_wait(Dist* d, cudaStream_t s) {
    if (!d || d->world == 1 || d->sim || !nccl().CommGetAsyncError) {
        MP_CUDA(cudaStreamSynchronize(s));
        return;
    }
    static const double limit = [] {
        const char* e = getenv("MPCR_DIST_TIMEOUT_S");
        return e ? atof(e) : 1800.0;
    }();
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        const cudaError_t q = cudaStreamQuery(s);
        if (q == cudaSuccess) return;
        if (q != cudaErrorNotReady) MP_CUDA(q);
        for (void* cm : {d->comm, d->row_comm, d->col_comm}) {
            if (!cm) continue;
            ncclResult_t ar = ncclSuccess;
            nccl().CommGetAsyncError(static_cast<ncclComm_t>(cm), &ar);
            if (ar != ncclSuccess && ar != ncclInProgress) {
                for (void* x : {d->comm, d->row_comm, d->col_comm})
                    if (x && nccl().CommAbort) nccl().CommAbort(static_cast<ncclComm_t>(x));
                d->comm = d->row_comm = d->col_comm = nullptr;
                fail(MP_NCCL_ERROR, std::string("NCCL asynchronous error on rank ") + std::to_string(d->rank) +
                                        ": " + (nccl().GetErrorString ? nccl().GetErrorString(ar) : "error") +
                                        " (communicators aborted)");
            }
        }
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) {
            for (void* x : {d->comm, d->row_comm, d->col_comm})
                if (x && nccl().CommAbort) nccl().CommAbort(static_cast<ncclComm_t>(x));
            d->comm = d->row_comm = d->col_comm = nullptr;
            fail(MP_NCCL_ERROR, "distributed factorization did not finish within MPCR_DIST_TIMEOUT_S on rank " +
                                    std::to_string(d->rank) + " (communicators aborted)");
        }
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
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
            // row and column communicators: members ordered by
            // process column / row, so a root's index is its column / row
            try {
                ncclComm_t rc = nullptr, cc = nullptr;
                nccl_check(nccl().CommSplit(comm, rank / Q, rank % Q, &rc, nullptr), "ncclCommSplit(row)");
                nccl_check(nccl().CommSplit(comm, rank % Q, rank / Q, &cc, nullptr), "ncclCommSplit(col)");
                d->row_comm = rc;
                d->col_comm = cc;
            } catch (...) {
                mp_dist_destroy(d);
                throw;
            }
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
    for (void* c : {d->row_comm, d->col_comm, d->comm})
        if (c && nccl().CommDestroy) nccl().CommDestroy(static_cast<ncclComm_t>(c));
    if (d->sim) {
        bool last;
        {
            std::lock_guard<std::mutex> lk(d->sim->mu);
            last = --d->sim->refs == 0;
        }
        if (last) delete d->sim;
    }
    delete d;
    return MP_OK;
}

// world handles over one GPU, rank r on ctxs[r] (each with its own streams);
// the ranks run concurrently from `world` host threads.
mp_status mp_dist_create_sim(mp_ctx* ctxs, int world, int P, int Q, mp_dist* out) {
    try {
        if (!ctxs || !out) fail(MP_INVALID_PARAM, "null argument");
        if (P < 1 || Q < 1 || P * Q != world) fail(MP_INVALID_PARAM, "dist: need P * Q == world");
        auto* g = new SimGroup();
        g->world = world;
        g->P = P;
        g->Q = Q;
        g->refs = world;
        for (int r = 0; r < world; ++r) {
            if (!ctxs[r]) fail(MP_INVALID_PARAM, "null context");
            auto* d = new mp_dist_s();
            d->ctx = ctxs[r];
            d->rank = r;
            d->world = world;
            d->P = P;
            d->Q = Q;
            d->sim = g;
            out[r] = d;
        }
        return MP_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.status;
    }
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
