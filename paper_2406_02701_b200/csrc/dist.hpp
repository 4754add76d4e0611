// Distributed MPCRTile Cholesky: 2D block-cyclic schedule and NCCL plumbing.
//
// Tile (i, j), i >= j, lives on rank (i mod P) * Q + (j mod Q) of a P x Q
// process grid.  Every rank derives its action list from the
// same host-only schedule: the GPU executor (tile.cpp) and the CPU/gloo test
// executor (tests/test_dist_cpu.py, through mp_dist_schedule) run the
// identical plan, so the CPU test pins the distributed algorithm bit-for-bit
// against the single-process oracle.
#pragma once

#include <cstdint>
#include <vector>

#include "internal.hpp"

namespace mpcr {

enum DistOp : int32_t {
    DA_POTRF = 1,        // factor diagonal tile (k, k) (owner only)
    DA_BCAST_DIAG = 2,   // broadcast the step's diagonal factor/inverse from `root` (all ranks)
    DA_TRSM = 3,         // panel tile (i, k) (owner only)
    DA_BCAST_PANEL = 4,  // broadcast panel tile (i, k) in precision `prec` from `root` (all ranks)
    DA_UPDATE = 5,       // A_ij -= L_ik L_jk^T, (i, j) owned
};

struct DistAction {
    int32_t op, k, i, j, root, prec;
};

inline int dist_owner(int64_t i, int64_t j, int P, int Q) {
    return static_cast<int>((i % P) * Q + (j % Q));
}

// The per-rank action list in execution order.  prec: tile-precision grid
// (column-major NT x NT); world == 1 yields no broadcasts.
std::vector<DistAction> dist_schedule(int rank, int P, int Q, int64_t NT, const int* prec);

struct Dist {
    Ctx* ctx = nullptr;
    int rank = 0, world = 1, P = 1, Q = 1;
    void* comm = nullptr;  // ncclComm_t
};

// Collectives on the context stream (NCCL, resolved with dlopen at first use).
void dist_bcast(Dist* d, void* buf, size_t bytes, int root, cudaStream_t s);
void dist_group_start(Dist* d);
void dist_group_end(Dist* d);
void dist_allreduce_min_u64(Dist* d, int64_t* buf, cudaStream_t s);  // -1 is the largest
void dist_allreduce_sum_f64(Dist* d, double* buf, size_t n, cudaStream_t s);

}  // namespace mpcr

struct mp_dist_s : mpcr::Dist {};
