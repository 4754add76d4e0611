// Distributed MPCRTile Cholesky: 2D block-cyclic schedule and the collective
// plumbing (NCCL, or a single-GPU simulation of the ranks for tests).
//
// Tile (i, j), i >= j, lives on rank (i mod P) * Q + (j mod Q) of a P x Q
// process grid.  Per step k the data moves along the grid's
// rows and columns only:
//   * L_kk's FP64 inverse travels down process column k mod Q (the TRSM
//     owners of tile column k);
//   * every panel tile L_ik travels along process row i mod P (the owners of
//     the row-i updates A_ij, k < j <= i, read it as the A operand) and then
//     down process column i mod Q (the owners of the column-i updates A_mi,
//     m >= i, read it as the B operand) from rank (i mod P, i mod Q), which
//     holds it after the row broadcast: P + Q - 2 copies per tile.
// Every rank derives its action list from the same host-only schedule; the
// GPU executor (tile.cpp) and the CPU/gloo test executor
// (tests/test_dist_cpu.py, through mp_dist_schedule) run the identical plan.
// The collectives follow one global order (step, diagonal, then per panel
// tile row then column), each rank issuing the subsequence it takes part in,
// so no communicator can deadlock against another.
#pragma once

#include <cstdint>
#include <vector>

#include "internal.hpp"

namespace mpcr {

enum DistOp : int32_t {
    DA_POTRF = 1,        // factor diagonal tile (k, k) (owner only)
    DA_BCAST_DIAG = 2,   // broadcast the step's diagonal inverse from `root` (column k mod Q)
    DA_TRSM = 3,         // panel tile (i, k) (owner only)
    DA_BCAST_PANEL = 4,  // broadcast panel tile (i, k) in precision `prec` from `root` over `comm`
    DA_UPDATE = 5,       // A_ij -= L_ik L_jk^T, (i, j) owned
};
enum DistComm : int32_t { DC_WORLD = 0, DC_ROW = 1, DC_COL = 2 };

struct DistAction {
    int32_t op, k, i, j, root, prec, comm;  // root: global rank
};

inline int dist_owner(int64_t i, int64_t j, int P, int Q) {
    return static_cast<int>((i % P) * Q + (j % Q));
}

// The per-rank action list in execution order.  prec: tile-precision grid
// (column-major NT x NT); world == 1 yields no broadcasts.
std::vector<DistAction> dist_schedule(int rank, int P, int Q, int64_t NT, const int* prec);

struct SimGroup;

struct Dist {
    Ctx* ctx = nullptr;
    int rank = 0, world = 1, P = 1, Q = 1;
    void* comm = nullptr;      // ncclComm_t over all ranks
    void* row_comm = nullptr;  // ranks of this process row (P x Q grid row rank / Q), ordered by column
    void* col_comm = nullptr;  // ranks of this process column, ordered by row
    SimGroup* sim = nullptr;   // single-GPU simulation of the ranks (tests), instead of NCCL
    int sim_seq[3] = {0, 0, 0};  // collectives issued per communicator (simulation)
    int pr() const { return rank / Q; }
    int pc() const { return rank % Q; }
};

// Collectives (NCCL, resolved with dlopen at first use; or the simulation).
// bcast: root is a global rank; comm selects the world / row / column
// communicator the caller belongs to.
void dist_bcast(Dist* d, void* buf, size_t bytes, int root, DistComm comm, cudaStream_t s);
void dist_group_start(Dist* d);
void dist_group_end(Dist* d);
void dist_allreduce_min_u64(Dist* d, int64_t* buf, cudaStream_t s);  // -1 is the largest
void dist_allreduce_sum_f64(Dist* d, double* buf, size_t n, cudaStream_t s);
// Wait for stream s on the host while polling the communicators for
// asynchronous NCCL errors (a rank that died mid-broadcast); on an error or
// after MPCR_DIST_TIMEOUT_S seconds the communicators are aborted and
// MP_NCCL_ERROR is raised instead of hanging.
void dist_wait(Dist* d, cudaStream_t s);

}  // namespace mpcr

struct mp_dist_s : mpcr::Dist {};
