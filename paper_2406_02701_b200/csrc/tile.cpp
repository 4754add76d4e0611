// MPCRTile on the device, and its mixed-precision tiled
// Cholesky scheduler.
//
// Storage: one slab per precision; every tile is one contiguous
// rows_per_tile x cols_per_tile column-major buffer inside the slab of its
// precision (so a single 3-D TMA map addresses every FP16 tile).
//
// Tiled Cholesky (right-looking, lower), per step k — the device version of
// the reference composition in oracle/ref_shim.cpp:ref_tile_chol:
//   1. POTRF of A_kk in its compute precision (cooperative kernel), then
//      TRTRI of the stored factor in FP64 -> Linv.
//   2. Linv rounded once to each panel precision present.
//   3. TRSM as GEMM: L_ik = A_ik * Linv^T in p_ik (tcgen05 FP16 for half
//      tiles), written to the panel buffer of p_ik and back to the tile.
//   4. Panel tiles converted once to every precision their consumers need
//      (A_ik.converted(p_ij) of the reference composition).
//   5. Trailing update A_ij -= L_ik L_jk^T, one grouped launch per precision
//      (lower triangle only on diagonal tiles).
// All per-step work lists are built on the host once per factorization and
// uploaded in one copy; the step loop is launch-only (no host sync).
#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "batch.hpp"
#include "dist.hpp"
#include "gemm_dmma.hpp"
#include "gemm_tc.hpp"
#include "ozaki.hpp"
#include "internal.hpp"

using namespace mpcr;

struct mp_tile_s {
    Ctx* ctx = nullptr;
    mp_dist_s* dist = nullptr;  // distributed over a process grid (null: single GPU)
    int64_t rows = 0, cols = 0, br = 0, bc = 0, tr = 0, tc = 0;
    std::vector<mp_precision> prec;  // tile (i, j) at j * tr + i
    std::vector<int64_t> slot;
    void* slab[3] = {nullptr, nullptr, nullptr};
    int64_t nslot[3] = {0, 0, 0};
    // scheduler workspace (grown on demand)
    void* panel[3] = {nullptr, nullptr, nullptr};
    void* digits = nullptr;  // INT8 digit planes of FP16 panel tiles [2][tr][S][br][br]
    int32_t* rexp = nullptr;  // their row exponents [2][tr][br]
    int32_t* ndig = nullptr;  // digits each 128-row block of them needs [gens][tr][ceil(br / 128)]
    void* backup[3] = {nullptr, nullptr, nullptr};  // jittered-NLL copy of the input slabs
    void* work = nullptr;  // FP64 + FP32 diagonal work, two Linv generations, info (WorkLayout)
    void* lists = nullptr;
    size_t lists_bytes = 0;
    TrtriPlan* trtri[2] = {nullptr, nullptr};  // FP64 inverse plans, one per Linv generation
    std::vector<cudaEvent_t> events;  // lookahead stream ordering (built on first chol)
    // the whole factorization as one CUDA graph (captured on the second
    // chol of this tile, replayed afterwards)
    cudaGraphExec_t graph = nullptr;
    uint64_t graph_scr_gen = 0;  // Ctx::scr_gen the graph's scratch pointers belong to
    int64_t graph_launches = 0;
    int chol_runs = 0;
    bool graph_failed = false;

    int64_t tt() const { return br * bc; }
    mp_precision p(int64_t i, int64_t j) const { return prec[j * tr + i]; }
    bool has(int64_t i, int64_t j) const { return slot[j * tr + i] >= 0; }
    void* ptr(int64_t i, int64_t j) const {
        const mp_precision q = p(i, j);
        if (!has(i, j)) return nullptr;
        return static_cast<char*>(slab[q]) + slot[j * tr + i] * tt() * elem_bytes(q);
    }
    int rank() const { return dist ? dist->rank : 0; }
    ~mp_tile_s() {
        for (int q = 0; q < 3; ++q) {
            if (slab[q]) cudaFree(slab[q]);
            if (panel[q]) cudaFree(panel[q]);
        }
        if (digits) cudaFree(digits);
        if (rexp) cudaFree(rexp);
        if (ndig) cudaFree(ndig);
        for (void* b : backup)
            if (b) cudaFree(b);
        if (work) cudaFree(work);
        if (lists) cudaFree(lists);
        for (TrtriPlan* p : trtri) trtri_plan_destroy(p);
        for (cudaEvent_t e : events) cudaEventDestroy(e);
        if (graph) cudaGraphExecDestroy(graph);
    }
};

namespace {

#define MP_API_BEGIN try {
#define MP_API_END                                       \
    return MP_OK;                                        \
    }                                                    \
    catch (const mpcr::Error& e) {                       \
        mpcr::g_last_error = e.what();                   \
        return e.status;                                 \
    }                                                    \
    catch (const std::exception& e) {                    \
        mpcr::g_last_error = e.what();                   \
        return MP_INTERNAL_ERROR;                        \
    }

mp_tile_s& T_(mp_tile t) {
    if (!t) fail(MP_INVALID_PARAM, "null MPCRTile");
    if (t->ctx) bind_device(t->ctx);
    return *t;
}

// Diagonal-tile workspace of the scheduler.  Linv (FP64) and its FP32 /
// FP16 hi+lo roundings come in two generations by step parity: the tail
// TRSM of panel k (lookahead stream) still reads Linv_k while the critical
// stream's POTRF/TRTRI of step k+1 writes Linv_{k+1}.
struct WorkLayout {
    size_t nn;
    explicit WorkLayout(int64_t nb) : nn(static_cast<size_t>(nb) * nb) {}
    double* dwork(void* w) const { return static_cast<double*>(w); }            // 8 nn
    float* swork(void* w) const { return reinterpret_cast<float*>(b(w) + 8 * nn); }  // 4 nn
    size_t gen(int g) const { return 12 * nn + static_cast<size_t>(g) * 16 * nn; }
    double* linv64(void* w, int g) const { return reinterpret_cast<double*>(b(w) + gen(g)); }
    float* linvS(void* w, int g) const { return reinterpret_cast<float*>(b(w) + gen(g) + 8 * nn); }
    uint16_t* linvH(void* w, int g) const { return reinterpret_cast<uint16_t*>(b(w) + gen(g) + 12 * nn); }
    uint16_t* linvHlo(void* w, int g) const { return reinterpret_cast<uint16_t*>(b(w) + gen(g) + 14 * nn); }
    int64_t* info(void* w) const { return reinterpret_cast<int64_t*>(b(w) + gen(2) + 64); }
    size_t bytes() const { return gen(2) + 256; }
    static char* b(void* w) { return static_cast<char*>(w); }
};

// Panel generations (step k uses generation k mod 3): the lookahead panel of
// step k+1 is produced while the trailing update still reads panel k, and
// with paired steps (below) the bulk update of an even step k runs during
// step k+1, still reading panel k while panel k+2 is produced.
constexpr int PANEL_GENS = 4;

void ensure_panels(mp_tile_s& t) {
    for (int q = 0; q < 3; ++q)
        if (!t.panel[q])
            MP_CUDA(cudaMalloc(&t.panel[q], PANEL_GENS * static_cast<size_t>(t.tr) * t.tt() * elem_bytes((mp_precision)q)));
    if (!t.digits && ozaki_enabled()) {
        MP_CUDA(cudaMalloc(&t.digits, PANEL_GENS * static_cast<size_t>(t.tr) * OZ_SLICES * t.tt()));
        MP_CUDA(cudaMalloc(&t.rexp, PANEL_GENS * static_cast<size_t>(t.tr) * t.br * sizeof(int32_t)));
        MP_CUDA(cudaMalloc(&t.ndig, PANEL_GENS * static_cast<size_t>(t.tr) * ((t.br + 127) / 128) * sizeof(int32_t)));
    }
    if (!t.work) MP_CUDA(cudaMalloc(&t.work, WorkLayout(t.br).bytes()));
    if (t.events.empty()) {
        t.events.resize(6 * t.tr + 4);
        for (auto& e : t.events) MP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
}

template <typename V>
void append(std::vector<char>& buf, const std::vector<V>& v, size_t& off) {
    off = (buf.size() + 255) / 256 * 256;
    buf.resize(off + v.size() * sizeof(V));
    if (!v.empty()) std::memcpy(buf.data() + off, v.data(), v.size() * sizeof(V));
}

// Device work lists of one trailing-update part (offsets into the list
// buffer + counts): tcgen05 FP16 (FP16 tiles; FP32 tiles fed by two FP16
// panel tiles), INT8 digits (FP64 tiles fed by two FP16 panel tiles), SIMT
// FP16 (tile sizes the tcgen05 path cannot map), and DMMA for every other
// FP32 / FP64 tile, keyed [A panel precision][B panel precision][C: FP32, FP64]
// with the panel tiles read natively (widened exactly on load).
// With paired steps a list belongs to one source panel (src 0: the panel of
// the previous, even step whose update was deferred; src 1: the step's own
// panel); tcf / tcf16s hold the tiles that take both panels in one pass
// (two K segments, one read-modify-write of C).
struct UpLists {
    size_t tc = 0, tc16s = 0, simt16 = 0, oz = 0, oz32 = 0, dm[3][3][2] = {}, tcf = 0, tcf16s = 0;
    int64_t n_tc = 0, n_tc16s = 0, n_simt16 = 0, n_oz = 0, n_oz_lower = 0, n_oz_two = 0, n_oz32 = 0, n_oz32_lower = 0,
            n_oz32_two = 0, n_dm[3][3][2] = {}, n_tcf = 0, n_tcf16s = 0;
};

struct StepLists {
    bool potrf = false;
    bool need_linv[3] = {false, false, false};
    // panel TRSM lists, [0]: tile k+1 (the head: the next diagonal SYRK and
    // the next column's first tile need it), [1]: the rest of the column
    size_t trsm_tc[2] = {0, 0}, trsm_p[2][3] = {};
    int64_t n_trsm_tc[2] = {0, 0}, n_trsm_p[2][3] = {};
    size_t wb[3] = {0, 0, 0};
    int64_t n_wb[3] = {0, 0, 0};
    // panel conversions, [0]: copies read by the lookahead updates (tile
    // column k+1), [1]: the rest (read by the bulk update only), [2]: the
    // head tile's share of [0], made on the critical path right after its TRSM
    size_t cv[3][3][3] = {};
    int64_t n_cv[3][3][3] = {};
    size_t digits[3] = {0, 0, 0};  // INT8 digit slicing of FP16 panel tiles (same split)
    int64_t n_digits[3] = {0, 0, 0};
    size_t digits32[3] = {0, 0, 0};  // ... and of FP32 panel tiles
    int64_t n_digits32[3] = {0, 0, 0};
    // [0: tile column k+1 below tile k+2, 1: the rest (bulk), 2: tile (k+1, k+1),
    //  3: tile column k+2 of a paired step below its diagonal, 4: tile (k+2, k+1)
    //  (the next step's head tile), 5: tile (k+2, k+2) of a paired step]
    //  [source panel].  Parts 4 and 5 run first on the lookahead stream: the
    //  next head TRSM and diagonal SYRK wait for them, not for the columns.
    UpLists up[6][2];
    bool diag_bcast = false;  // receive / send L_kk^-1 down this process column
    struct Bcast {
        int i, root, comm;
    };
    // panel broadcasts in schedule order (row then column per tile), [0]: the
    // head tile k+1 (critical path), [1]: the rest of the column
    std::vector<Bcast> bcasts[2];
};

}  // namespace

namespace mpcr {

// Tiled Cholesky of an MPCRTile in place.  Returns the global failing column
// (or -1); the caller maps it to MP_NOT_POSITIVE_DEFINITE.
//
// Lookahead (depth 1) on two streams: the critical path — update of tile
// column k+1 with panel k, then POTRF/TRTRI/TRSM/conversions of panel k+1 —
// runs on the high-priority stream while the bulk of step k's trailing update
// runs on the context stream.  Panels alternate between two buffers by step
// parity.  MPCR_LOOKAHEAD=0 serialises everything on one stream.
int64_t tile_chol_inplace(Ctx* c, mp_tile_s& t) {
    cudaStream_t s = c->stream;
    const int64_t nb = t.br, NT = t.tr, tt = t.tt();
    ensure_panels(t);
    const size_t nn = static_cast<size_t>(nb) * nb;
    const WorkLayout WL(nb);
    int64_t* dinfo = WL.info(t.work);
    auto read_info = [&]() {
        int64_t info = -1;
        MP_CUDA(cudaMemcpyAsync(&info, dinfo, sizeof(info), cudaMemcpyDeviceToHost, s));
        // multi-rank: poll NCCL for asynchronous errors instead of blocking
        dist_wait(t.dist, s);
        return info;
    };
    // Graph replay: the factorization of this tile was captured once (lists,
    // pointers and streams do not change over the tile's life).  Profiling
    // and multi-rank runs stay eager.  MPCR_GRAPH=0 disables graphs.
    static const bool graph_env = [] {
        const char* e = getenv("MPCR_GRAPH");
        return !(e && e[0] == '0');
    }();
    // multi-rank (real NCCL) factorizations are captured too: NCCL
    // collectives are graph-capturable; the single-GPU rank simulation is not
    // (its host rendezvous), and MPCR_DIST_GRAPH=0 keeps NCCL runs eager
    static const bool dist_graph_env = [] {
        const char* e = getenv("MPCR_DIST_GRAPH");
        return !(e && e[0] == '0');
    }();
    const bool multi = t.dist && t.dist->world > 1;
    const bool want_graph =
        graph_env && !c->prof.enabled && !(multi && (t.dist->sim || !dist_graph_env));
    if (t.graph && t.graph_scr_gen != c->scr_gen) {
        // a context scratch slot the graph captured (POTRF barriers / leaf
        // inverses, 3xTF32 splits) was reallocated since: re-capture
        MP_CUDA(cudaStreamSynchronize(s));
        MP_CUDA(cudaGraphExecDestroy(t.graph));
        t.graph = nullptr;
    }
    if (want_graph && t.graph) {
        MP_CUDA(cudaGraphLaunch(t.graph, s));
        c->launches += t.graph_launches;
        return read_info();
    }
    const bool tc_ok = (nb % 8) == 0;  // TMA stride alignment for FP16 tiles
    static const bool lookahead_env = [] {
        const char* e = getenv("MPCR_LOOKAHEAD");
        return !(e && e[0] == '0');
    }();
    const bool la = lookahead_env && NT > 1;
    cudaStream_t sl = la ? c->hi : s;  // critical-path stream

    auto pan = [&](mp_precision q, int64_t i, int64_t k) -> void* {
        return static_cast<char*>(t.panel[q]) + ((k % PANEL_GENS) * NT + i) * tt * elem_bytes(q);
    };

    // ---- host plan: the rank's action list (dist.hpp) turned into grouped
    //      per-step work lists (single GPU: P = Q = 1, no broadcasts) --------
    const int P = t.dist ? t.dist->P : 1, Q = t.dist ? t.dist->Q : 1, rank = t.rank();
    std::vector<int> pgrid(t.prec.begin(), t.prec.end());
    const auto sched = dist_schedule(rank, P, Q, NT, pgrid.data());
    struct UpAcc {
        std::vector<TcProblem> tc, tc16s, tcf, tcf16s;
        std::vector<TileProblem> simt16;
        std::vector<OzProblem> oz;           // FP64 tiles fed by FP16 panels: INT8 digit products
        std::vector<OzProblem> oz32;         // FP32 tiles fed by FP32 (or FP32 + FP16) panels: the same
        std::vector<TileProblem> dm[3][3][2];  // DMMA, native panel precisions
    };
    // FP32 tiles whose two panel tiles are both FP16: the FP16 tensor-core
    // GEMM with an FP32 accumulator/output (exact products; what 3xTF32
    // reduces to when the low halves are zero)
    auto half_into_single = [&](int64_t i, int64_t j, int64_t k) {
        return tc_ok && t.p(i, k) == MP_HALF && t.p(j, k) == MP_HALF;
    };
    // Operand precision the update of a tile of precision q reads panel tile
    // (i, k) in: FP16 tiles take FP16 copies (A_ik.converted(half), the
    // reference composition); FP32 and FP64 tiles are updated on DMMA, which
    // widens FP16 / FP32 panel tiles exactly on load (an FP64 panel tile is
    // rounded to FP32 first for an FP32 tile, as the reference's
    // converted(single)).
    auto opnd_prec = [&](mp_precision q, int64_t i, int64_t k) -> mp_precision {
        const mp_precision r = t.p(i, k);
        if (q == MP_HALF) return MP_HALF;
        if (q == MP_SINGLE && r == MP_DOUBLE) return MP_SINGLE;
        return r;
    };
    // FP64 tiles fed by two FP16 panel tiles: the INT8 tensor cores (exact digits)
    const bool oz_ok = tc_ok && (nb % 16) == 0 && ozaki_enabled();
    auto ozaki64 = [&](int64_t i, int64_t j, int64_t k) {
        return oz_ok && t.p(i, k) == MP_HALF && t.p(j, k) == MP_HALF;
    };
    // FP32 tiles fed by FP32 panel tiles (or one FP32 and one FP16): INT8
    // digits of the FP32 / FP16 panel tiles, FP64 combination, one rounding to
    // FP32 -- the tensor cores instead of DMMA (MPCR_OZAKI32=0: DMMA).  Digits
    // of an FP32 row are exact down to 2^-41 of the row's largest entry.
    static const bool oz32_env = [] {
        const char* e = getenv("MPCR_OZAKI32");
        return !(e && e[0] == '0');
    }();
    auto ozaki32 = [&](int64_t i, int64_t j, int64_t k) {
        return oz_ok && oz32_env && nb <= 1024 && !(t.p(i, k) == MP_HALF && t.p(j, k) == MP_HALF) &&
               t.p(i, k) != MP_DOUBLE &&
               t.p(j, k) != MP_DOUBLE;
    };
    // the update of tile (i, j) by panel k reads INT8 digits of the panel tiles
    auto uses_digits = [&](int64_t i, int64_t j, int64_t k) {
        const mp_precision q = t.p(i, j);
        return (q == MP_DOUBLE && ozaki64(i, j, k)) || (q == MP_SINGLE && ozaki32(i, j, k));
    };
    const int64_t dig_tile = OZ_SLICES * tt;  // bytes of one tile's digit planes
    auto dig = [&](int64_t i, int64_t k) -> int8_t* {
        return static_cast<int8_t*>(t.digits) + ((k % PANEL_GENS) * NT + i) * dig_tile;
    };
    auto rex = [&](int64_t i, int64_t k) -> int32_t* { return t.rexp + ((k % PANEL_GENS) * NT + i) * nb; };
    const int64_t NDB = (nb + 127) / 128;  // digit-count blocks per tile
    auto ndg = [&](int64_t i, int64_t k) -> int32_t* { return t.ndig + ((k % PANEL_GENS) * NT + i) * NDB; };
    struct StepAcc {
        std::vector<TcProblem> trsm_tc[2];
        std::vector<TileProblem> trsm_p[2][3];
        std::vector<CopyItem> wb[3], cv[3][3][3];
        std::vector<OzSliceItem> digits[3], digits32[3];
        UpAcc up[6][2];
    };
    // Head/tail split of the panel TRSM (single GPU with lookahead): the head
    // tile runs on the critical-path stream, the rest of the column on the
    // lookahead stream next to the column update it feeds.  MPCR_TRSM_SPLIT=0
    // keeps the whole column on the critical path.
    static const bool tsplit_env = [] {
        const char* e = getenv("MPCR_TRSM_SPLIT");
        return !(e && e[0] == '0');
    }();
    // (also without lookahead, on one stream: the same launches, serialised)
    const bool tsplit = tsplit_env && NT > 1;
    std::vector<StepAcc> acc(NT);
    std::vector<StepLists> steps(NT);
    const size_t nn0 = static_cast<size_t>(nb) * nb;
    (void)nn0;
    auto linv = [&](int q, int64_t k) -> const void* {  // Linv_k rounded to p = q
        const int g = static_cast<int>(k & 1);
        return q == MP_HALF ? static_cast<const void*>(WL.linvH(t.work, g))
               : q == MP_SINGLE ? static_cast<const void*>(WL.linvS(t.work, g))
                                : static_cast<const void*>(WL.linv64(t.work, g));
    };
    // Paired steps (MPCR_PAIR_STEPS=0 turns them off): the trailing update of
    // an even step k is deferred into step k+1, where tensor-core tiles take
    // both panels in one pass (K = 2 nb, C read and written once instead of
    // twice, rounded once).  Tile column k+2 of an odd step k leaves the
    // paired bulk for the lookahead stream (part 3), so neither of the next
    // two critical chains waits on the paired bulk that precedes them; the
    // panel, digit and exponent buffers live in four generations (panel k+1
    // is produced while the bulk still reads panels k-2 and k-1).
    static const bool pair_env = [] {
        const char* e = getenv("MPCR_PAIR_STEPS");
        return !(e && e[0] == '0');
    }();
    const bool pair_steps = pair_env && NT > 2;
    // tile columns whose updates from panel k run on the lookahead streams:
    // their operand copies / digits are made with the panel, not with the bulk
    auto la_col = [&](int64_t k, int64_t j) { return j == k + 1 || (pair_steps && j == k + 2); };
    auto consumers = [&](int64_t k, int64_t i, StepAcc& A) {
        // every rank receives every panel tile: convert it once to each
        // precision the rank's own consumers (A_ij.converted(p) operands)
        // need.  Copies read by the lookahead updates (tile column k+1, and
        // k+2 with paired steps) are made on the critical path ([0]); the rest
        // with the bulk update ([1]).
        const mp_precision q = t.p(i, k);
        bool need[2][3] = {{false, false, false}, {false, false, false}};
        for (int64_t j = k + 1; j <= i; ++j)  // A operand of (owned) row-i updates
            if (t.has(i, j) && !uses_digits(i, j, k))
                need[la_col(k, j) ? 0 : 1][opnd_prec(t.p(i, j), i, k)] = true;
        for (int64_t m = i; m < NT; ++m)  // B operand of (owned) column-i updates
            if (t.has(m, i) && !uses_digits(m, i, k))
                need[la_col(k, i) ? 0 : 1][opnd_prec(t.p(m, i), i, k)] = true;
        const int h0 = (tsplit && i == k + 1) ? 2 : 0;  // the head tile's part-0 work
        for (int r = 0; r < 3; ++r) {
            if (r == q) continue;
            const int h = need[0][r] ? h0 : need[1][r] ? 1 : -1;
            if (h >= 0) A.cv[h][q][r].push_back(CopyItem{pan(q, i, k), pan((mp_precision)r, i, k)});
        }
        bool need_dig[2] = {false, false};
        for (int64_t j = k + 1; j <= i; ++j)
            if (t.has(i, j) && uses_digits(i, j, k)) need_dig[la_col(k, j) ? 0 : 1] = true;
        for (int64_t m = i; m < NT; ++m)
            if (t.has(m, i) && uses_digits(m, i, k)) need_dig[la_col(k, i) ? 0 : 1] = true;
        const int hd = need_dig[0] ? h0 : need_dig[1] ? 1 : -1;
        if (hd >= 0) {  // from the panel tile's own precision (FP16 or FP32)
            const bool f32 = q != MP_HALF;
            (f32 ? A.digits32 : A.digits)[hd].push_back(OzSliceItem{pan(f32 ? MP_SINGLE : MP_HALF, i, k), dig(i, k),
                                                                    rex(i, k), ndg(i, k), nb, nb, nb, nb, tt, 0, 0});
        }
    };
    std::vector<char> have(NT * NT, 0);  // panel tile (i, k) present on this rank (conversions made)
    struct TcCand {
        int64_t ks;
        int part, kind, src;  // kind 0: FP16 tile, 1: FP32 tile fed by FP16 panels
        TcProblem p;
    };
    std::vector<TcCand> tc_cand;
    // INT8-digit candidates (kind 0: FP64 tile, 1: FP32 tile); digit tiles are
    // indexed over all panel generations (gen * NT + row)
    struct OzCand {
        int64_t ks;
        int part, kind, src;
        int64_t i, j;
        OzProblem p;
    };
    std::vector<OzCand> oz_cand;
    auto gtile = [&](int64_t i, int64_t k) { return static_cast<int32_t>((k % PANEL_GENS) * NT + i); };
    for (const DistAction& a : sched) {
        StepAcc& A = acc[a.k];
        StepLists& L = steps[a.k];
        const int64_t k = a.k, i = a.i, j = a.j;
        const mp_precision q = static_cast<mp_precision>(a.prec);
        switch (a.op) {
            case DA_POTRF:
                L.potrf = true;
                break;
            case DA_TRSM: {
                L.need_linv[q] = true;
                const int hb = (tsplit && i == k + 1) ? 0 : 1;
                if (q == MP_HALF && tc_ok)
                    // A = matrix tile (i,k) in the FP16 slab, C = panel16[i]
                    A.trsm_tc[hb].push_back(TcProblem{static_cast<int32_t>(t.slot[k * NT + i]), 0,
                                                      static_cast<int32_t>(i), 0});
                else  // FP32 / FP64 tiles (and FP16 when nb % 8): the FP64 inverse
                    A.trsm_p[hb][q].push_back(TileProblem{t.ptr(i, k), linv(q == MP_HALF ? MP_HALF : MP_DOUBLE, k),
                                                          pan(q, i, k), 0, 0});
                A.wb[q].push_back(CopyItem{pan(q, i, k), t.ptr(i, k)});
                if (P * Q == 1) consumers(k, i, A);
                break;
            }
            case DA_BCAST_DIAG:
                L.diag_bcast = true;
                break;
            case DA_BCAST_PANEL:
                L.bcasts[(tsplit && i == k + 1) ? 0 : 1].push_back({static_cast<int>(i), a.root, a.comm});
                if (!have[k * NT + i]) consumers(k, i, A);
                have[k * NT + i] = 1;
                break;
            case DA_UPDATE: {
                // paired steps: an even step's update of tiles j >= k+2 runs in
                // step k+1 (source 0) next to that step's own update (source 1)
                const bool defer = pair_steps && (k % 2 == 0) && j >= k + 2;
                const int64_t ks = defer ? k + 1 : k;
                const int src = defer ? 0 : 1;
                int part;  // see StepLists::up
                if (j == ks + 1)
                    part = i == j ? 2 : i == ks + 2 ? 4 : 0;
                else if (pair_steps && ks % 2 == 1 && j == ks + 2)
                    part = i == j ? 5 : 3;
                else
                    part = 1;
                UpAcc& U = acc[ks].up[part][src];
                const int32_t lo = (i == j) ? 1 : 0;
                const TcProblem tp{static_cast<int32_t>(i), static_cast<int32_t>(j),
                                   static_cast<int32_t>(t.slot[j * NT + i]), lo};
                if (q == MP_HALF && tc_ok)
                    tc_cand.push_back({ks, part, 0, src, tp});
                else if (q == MP_HALF)
                    U.simt16.push_back(TileProblem{pan(MP_HALF, i, k), pan(MP_HALF, j, k), t.ptr(i, j), lo, 0});
                else if (q == MP_SINGLE && half_into_single(i, j, k))
                    tc_cand.push_back({ks, part, 1, src, tp});
                else if ((q == MP_DOUBLE && ozaki64(i, j, k)) || (q == MP_SINGLE && ozaki32(i, j, k)))
                    oz_cand.push_back({ks, part, q == MP_SINGLE ? 1 : 0, src, i, j,
                                       OzProblem{gtile(i, k), gtile(j, k), t.ptr(i, j), lo, -1, -1, 0}});
                else {
                    const mp_precision pa = opnd_prec(q, i, k), pb = opnd_prec(q, j, k);
                    U.dm[pa][pb][q == MP_DOUBLE ? 1 : 0].push_back(
                        TileProblem{pan(pa, i, k), pan(pb, j, k), t.ptr(i, j), lo, 0});
                }
                break;
            }
            default:
                break;
        }
    }
    // tensor-core candidates: a tile with both sources of the same kind in one
    // step goes to the fused two-panel list, otherwise to its source's list
    {
        std::sort(tc_cand.begin(), tc_cand.end(), [](const TcCand& x, const TcCand& y) {
            if (x.ks != y.ks) return x.ks < y.ks;
            if (x.part != y.part) return x.part < y.part;
            if (x.p.a_tile != y.p.a_tile) return x.p.a_tile < y.p.a_tile;
            if (x.p.b_tile != y.p.b_tile) return x.p.b_tile < y.p.b_tile;
            return x.src < y.src;
        });
        for (size_t q = 0; q < tc_cand.size(); ++q) {
            const TcCand& x = tc_cand[q];
            const bool both = q + 1 < tc_cand.size() && tc_cand[q + 1].ks == x.ks && tc_cand[q + 1].part == x.part &&
                              tc_cand[q + 1].p.a_tile == x.p.a_tile && tc_cand[q + 1].p.b_tile == x.p.b_tile;
            if (both && tc_cand[q + 1].kind == x.kind) {
                UpAcc& U = acc[x.ks].up[x.part][1];
                (x.kind == 0 ? U.tcf : U.tcf16s).push_back(x.p);
                ++q;
                continue;
            }
            UpAcc& U = acc[x.ks].up[x.part][x.src];
            (x.kind == 0 ? U.tc : U.tc16s).push_back(x.p);
        }
    }
    // INT8-digit tiles with both sources in one step take both panels in one
    // pass (C read and written once): src 0's digits first, then src 1's
    {
        std::sort(oz_cand.begin(), oz_cand.end(), [](const OzCand& x, const OzCand& y) {
            if (x.ks != y.ks) return x.ks < y.ks;
            if (x.part != y.part) return x.part < y.part;
            if (x.kind != y.kind) return x.kind < y.kind;
            if (x.j != y.j) return x.j < y.j;
            if (x.i != y.i) return x.i < y.i;
            return x.src < y.src;
        });
        for (size_t q = 0; q < oz_cand.size(); ++q) {
            const OzCand& x = oz_cand[q];
            const bool both = q + 1 < oz_cand.size() && oz_cand[q + 1].ks == x.ks && oz_cand[q + 1].part == x.part &&
                              oz_cand[q + 1].kind == x.kind && oz_cand[q + 1].i == x.i && oz_cand[q + 1].j == x.j;
            if (both) {
                OzProblem f = x.p;
                f.a_tile2 = oz_cand[q + 1].p.a_tile;
                f.b_tile2 = oz_cand[q + 1].p.b_tile;
                UpAcc& U = acc[x.ks].up[x.part][1];
                (x.kind ? U.oz32 : U.oz).push_back(f);
                ++q;
                continue;
            }
            UpAcc& U = acc[x.ks].up[x.part][x.src];
            (x.kind ? U.oz32 : U.oz).push_back(x.p);
        }
    }
    // FP16 update tiles of a step in groups of G tile columns, rows within a
    // group, the group's columns within a row: each panel tile L_ik serves G
    // consecutive tiles and the group's G tiles L_jk stay in L2, so the panel
    // (256 MB at n=131072, twice the L2) is not re-read from HBM per column.
    // Tiles of one step are independent, so the factor is unchanged.
    static const int upd_group = [] {
        const char* e = getenv("MPCR_UPDATE_GROUP");
        return e ? std::max(1, atoi(e)) : 8;
    }();
    auto grouped = [](const TcProblem& x, const TcProblem& y) {
        const int gx = x.b_tile / upd_group, gy = y.b_tile / upd_group;
        if (gx != gy) return gx < gy;
        if (x.a_tile != y.a_tile) return x.a_tile < y.a_tile;
        return x.b_tile < y.b_tile;
    };
    for (int64_t k = 0; k < NT; ++k)
        for (int w = 0; w < 6; ++w)
            for (int sc = 0; sc < 2; ++sc) {
                std::stable_sort(acc[k].up[w][sc].tc.begin(), acc[k].up[w][sc].tc.end(), grouped);
                std::stable_sort(acc[k].up[w][sc].tcf.begin(), acc[k].up[w][sc].tcf.end(), grouped);
            }
    std::vector<char> buf;
    for (int64_t k = 0; k < NT; ++k) {
        StepLists& L = steps[k];
        StepAcc& A = acc[k];
        for (int hb = 0; hb < 2; ++hb) {
            append(buf, A.trsm_tc[hb], L.trsm_tc[hb]);
            L.n_trsm_tc[hb] = A.trsm_tc[hb].size();
            for (int q = 0; q < 3; ++q) {
                append(buf, A.trsm_p[hb][q], L.trsm_p[hb][q]);
                L.n_trsm_p[hb][q] = A.trsm_p[hb][q].size();
            }
        }
        for (int q = 0; q < 3; ++q) {
            append(buf, A.wb[q], L.wb[q]);
            L.n_wb[q] = A.wb[q].size();
            for (int r = 0; r < 3; ++r)
                for (int h = 0; h < 3; ++h) {
                    append(buf, A.cv[h][q][r], L.cv[h][q][r]);
                    L.n_cv[h][q][r] = A.cv[h][q][r].size();
                }
        }
        for (int h = 0; h < 3; ++h) {
            append(buf, A.digits[h], L.digits[h]);
            L.n_digits[h] = A.digits[h].size();
            append(buf, A.digits32[h], L.digits32[h]);
            L.n_digits32[h] = A.digits32[h].size();
        }
        for (int w = 0; w < 6; ++w)
            for (int sc = 0; sc < 2; ++sc) {
                const UpAcc& U = A.up[w][sc];
                UpLists& D = L.up[w][sc];
                append(buf, U.tc, D.tc);
                D.n_tc = U.tc.size();
                append(buf, U.tc16s, D.tc16s);
                D.n_tc16s = U.tc16s.size();
                append(buf, U.tcf, D.tcf);
                D.n_tcf = U.tcf.size();
                append(buf, U.tcf16s, D.tcf16s);
                D.n_tcf16s = U.tcf16s.size();
                append(buf, U.simt16, D.simt16);
                D.n_simt16 = U.simt16.size();
                // diagonal (lower-only) problems first: the kernel enumerates
                // only their live units
                for (int w32 = 0; w32 < 2; ++w32) {
                    std::vector<OzProblem> oz = w32 ? U.oz32 : U.oz;
                    const auto lower_end = std::stable_partition(
                        oz.begin(), oz.end(), [](const OzProblem& o) { return o.lower_only != 0; });
                    (w32 ? D.n_oz32_lower : D.n_oz_lower) = lower_end - oz.begin();
                    (w32 ? D.n_oz32_two : D.n_oz_two) =
                        std::count_if(oz.begin(), oz.end(), [](const OzProblem& o) { return o.a_tile2 >= 0; });
                    append(buf, oz, w32 ? D.oz32 : D.oz);
                    (w32 ? D.n_oz32 : D.n_oz) = oz.size();
                }
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b)
                        for (int c2 = 0; c2 < 2; ++c2) {
                            append(buf, U.dm[a][b][c2], D.dm[a][b][c2]);
                            D.n_dm[a][b][c2] = U.dm[a][b][c2].size();
                        }
            }
    }
    // final clean-up lists: upper part of diagonal tiles, strictly-upper tiles
    std::vector<void*> diag_ptrs[3], upper_ptrs[3];
    for (int64_t j = 0; j < NT; ++j)
        for (int64_t i = 0; i <= j; ++i)
            if (t.has(i, j)) (i == j ? diag_ptrs : upper_ptrs)[t.p(i, j)].push_back(t.ptr(i, j));
    size_t off_diag[3], off_upper[3];
    for (int q = 0; q < 3; ++q) {
        append(buf, diag_ptrs[q], off_diag[q]);
        append(buf, upper_ptrs[q], off_upper[q]);
    }
    if (buf.size() > t.lists_bytes) {
        if (t.lists) MP_CUDA(cudaFree(t.lists));
        MP_CUDA(cudaMalloc(&t.lists, buf.size()));
        t.lists_bytes = buf.size();
    }
    char* dl = static_cast<char*>(t.lists);
    MP_CUDA(cudaMemcpyAsync(dl, buf.data(), buf.size(), cudaMemcpyHostToDevice, s));

    // ---- workspace ------------------------------------------------------------
    double* dwork = WL.dwork(t.work);
    float* swork = WL.swork(t.work);
    // the TRTRI plans (FP64 inverse of dwork into either Linv generation) are built once
    for (int g = 0; g < 2; ++g)
        if (!t.trtri[g]) t.trtri[g] = trtri_plan_create(c, s, dwork, nb, WL.linv64(t.work, g), nb, nb);

    // ---- panel k: factor A_kk, invert, TRSM the tile column, distribute and
    //      convert the panel for its consumers ---------------------------------
    // consumer-precision copies of panel k ([0] lookahead tiles, [1] bulk) and
    // the hi/lo TF32 splits of its FP32 tiles, stored transposed (K-major)
    auto convert_panel = [&](int64_t k, int h, cudaStream_t st) {
        const StepLists& L = steps[k];
        for (int q = 0; q < 3; ++q)
            for (int r = 0; r < 3; ++r)
                if (L.n_cv[h][q][r])
                    launch_batched_convert(c, st, (mp_precision)q, (mp_precision)r,
                                           reinterpret_cast<const CopyItem*>(dl + L.cv[h][q][r]),
                                           L.n_cv[h][q][r], tt);
        if (L.n_digits32[h])
            launch_oz_slices_f32(c, st, reinterpret_cast<const OzSliceItem*>(dl + L.digits32[h]), L.n_digits32[h], nb,
                                 nb);
        if (L.n_digits[h]) {
            launch_oz_slices(c, st, reinterpret_cast<const OzSliceItem*>(dl + L.digits[h]), L.n_digits[h], nb, nb);
            static const bool dbg = getenv("MPCR_DEBUG_NDIG") != nullptr;  // diagnostics (eager runs only)
            if (dbg && h == 1) {
                std::vector<int32_t> nd(NT * NDB);
                MP_CUDA(cudaMemcpyAsync(nd.data(), ndg(0, k), nd.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
                MP_CUDA(cudaStreamSynchronize(st));
                int hist[8] = {};  // per 128-row block
                for (int64_t i = k + 1; i < NT; ++i)
                    for (int64_t b = 0; b < NDB; ++b) hist[std::min(7, std::max(0, nd[i * NDB + b]))]++;
                std::fprintf(stderr, "[mpcr] step %lld digits:", static_cast<long long>(k));
                for (int q = 0; q < 8; ++q) std::fprintf(stderr, " %d", hist[q]);
                std::fprintf(stderr, "\n");
            }
        }
    };
    // write the factor of tile column k back from the panel into the tiles
    auto write_back = [&](int64_t k, cudaStream_t st) {
        const StepLists& L = steps[k];
        for (int q = 0; q < 3; ++q)
            if (L.n_wb[q])
                launch_batched_convert(c, st, (mp_precision)q, (mp_precision)q,
                                       reinterpret_cast<const CopyItem*>(dl + L.wb[q]), L.n_wb[q], tt);
    };

    // TRSM as GEMM of one part of the column: panel_q[i] = A_ik * Linv_q^T
    auto trsm_part = [&](int64_t k, int hb, cudaStream_t st) {
        const StepLists& L = steps[k];
        if (L.n_trsm_tc[hb]) {
            TcGemm g;
            g.pc = MP_HALF;
            g.ta = false;
            g.tb = true;
            g.m = g.n = g.k = nb;
            g.alpha = 1.0;
            g.beta = 0.0;
            g.A = t.slab[MP_HALF];
            g.lda = nb;
            g.a_tiles = t.nslot[MP_HALF];
            g.a_tile_stride = tt;
            g.B = WL.linvH(t.work, static_cast<int>(k & 1));
            g.B2 = WL.linvHlo(t.work, static_cast<int>(k & 1));
            g.ldb = nb;
            g.b_tiles = 1;
            g.b_tile_stride = tt;
            g.C = pan(MP_HALF, 0, k);
            g.ldc = nb;
            g.c_tiles = NT;
            g.c_tile_stride = tt;
            g.problems = reinterpret_cast<const TcProblem*>(dl + L.trsm_tc[hb]);
            g.count = L.n_trsm_tc[hb];
            g.k_tri = true;  // Linv^T is upper triangular: skip its zero K blocks
            launch_tc_gemm(c, st, g);
        }
        for (int q = 0; q < 3; ++q) {
            if (!L.n_trsm_p[hb][q]) continue;
            const auto* probs = reinterpret_cast<const TileProblem*>(dl + L.trsm_p[hb][q]);
            if (q != MP_HALF) {
                // FP32 / FP64 panel tiles: one grouped DMMA launch, A_ik (FP32
                // widened exactly on load, or FP64) times the FP64 inverse, each
                // CTA's K loop cut at the triangle; FP32 tiles rounded once from
                // the FP64 result.  (An explicit inverse applied in TF32/FP32
                // carries cond(L_kk) * u_32 into the panel; in FP64 it does not.)
                DmmaArgs d{false, true, nb, nb, nb, 1.0, 0.0, nullptr, nb, nullptr, nb, nullptr, nb, false,
                           probs, (mp_precision)q};
                d.pout = (mp_precision)q;
                d.k_tri = true;
                d.pin_b = MP_DOUBLE;
                d.exclusive = hb == 0;  // the head tile is on the critical path
                d.allow_ksplit = hb == 0;  // one tile on every rank: grouping-independent
                ProfScope ps(c, MP_PROF_TRSM, st, static_cast<double>(nb) * nb * nb * L.n_trsm_p[hb][q]);
                launch_dmma_gemm(c, st, d, L.n_trsm_p[hb][q]);
                continue;
            }
            GroupedGemm g{(mp_precision)q, (mp_precision)q, true, nb, nb, nb, nb, nb, nb, 1.0, 0.0, probs,
                          L.n_trsm_p[hb][q]};
            launch_grouped_gemm(c, st, g);
        }
    };

    // Distributed: panel tiles of one part along their process rows (one NCCL
    // group), then down their process columns (a second group: a column
    // root receives the tile in the row broadcast).
    auto broadcast = [&](int64_t k, int part, cudaStream_t st) {
        const auto& B = steps[k].bcasts[part];
        for (int c : {DC_ROW, DC_COL}) {
            bool any = false;
            for (const auto& br : B) any = any || br.comm == c;
            if (!any) continue;
            dist_group_start(t.dist);
            for (const auto& br : B)
                if (br.comm == c) {
                    const mp_precision q = t.p(br.i, k);
                    dist_bcast(t.dist, pan(q, br.i, k), tt * elem_bytes(q), br.root, static_cast<DistComm>(c), st);
                }
            dist_group_end(t.dist);
        }
    };
    // Panel k, critical part (stream st): factor A_kk, invert, round Linv to
    // the panel precisions, TRSM of the head tile (k+1) and its lookahead
    // conversions.  Without the head/tail split the whole column follows here.
    auto panel_head = [&](int64_t k, cudaStream_t st, cudaEvent_t before_trsm) {
        const StepLists& L = steps[k];
        const mp_precision pk = t.p(k, k);
        void* akk = t.ptr(k, k);
        const int lg = static_cast<int>(k & 1);  // Linv generation of this step
        double* linv64 = WL.linv64(t.work, lg);
        TrtriPlan* trtri = t.trtri[lg];
        if (!L.potrf) {
            // not the owner: nothing to factor
        } else if (pk == MP_DOUBLE) {
            // POTRF in place, its 64x64 block inverses straight into Linv
            launch_potrf_lower(c, st, MP_DOUBLE, akk, nb, nb, dinfo, k * nb, linv64, nb);
            if (k + 1 < NT) {
                MP_CUDA(cudaMemcpyAsync(dwork, akk, nn * sizeof(double), cudaMemcpyDeviceToDevice, st));
                launch_trtri_plan(c, st, trtri, true);
            }
        } else {
            if (pk == MP_SINGLE) {
                launch_potrf_lower(c, st, MP_SINGLE, akk, nb, nb, dinfo, k * nb);
            } else {
                launch_convert(c, st, MP_HALF, akk, nb, MP_SINGLE, swork, nb, nb, nb);
                launch_potrf_lower(c, st, MP_SINGLE, swork, nb, nb, dinfo, k * nb);
                launch_convert(c, st, MP_SINGLE, swork, nb, MP_HALF, akk, nb, nb, nb);
            }
            if (k + 1 < NT) {  // inverse of the stored (rounded) factor, in FP64
                launch_convert(c, st, pk, akk, nb, MP_DOUBLE, dwork, nb, nb, nb);
                launch_trtri_plan(c, st, trtri, false);
            }
        }
        if (k + 1 == NT) return;
        // distributed: the FP64 inverse of L_kk travels down process column k mod Q
        if (L.diag_bcast)
            dist_bcast(t.dist, linv64, nn * sizeof(double), dist_owner(k, k, P, Q), DC_COL, st);
        // Linv rounded to the panel precisions (the reference rounds U_kk to
        // p_ik before trsm: U_kk.converted(p_ik)).  FP16 panels apply the
        // inverse as hi + lo FP16 halves accumulated in one FP32 accumulator:
        // an explicit inverse rounded to FP16 alone has a backward error
        // ~cond(L_kk) * 2^-11 and loses definiteness where the reference's
        // substitution does not.
        if (L.need_linv[MP_HALF]) {
            if (L.n_trsm_tc[0] + L.n_trsm_tc[1])
                launch_split_f16(c, st, linv64, WL.linvH(t.work, lg), WL.linvHlo(t.work, lg),
                                 static_cast<int64_t>(nn));
            else
                launch_convert(c, st, MP_DOUBLE, linv64, nb, MP_HALF, WL.linvH(t.work, lg), nb, nb, nb);
        }

        // the tile column has its update from step k-1
        if (before_trsm) MP_CUDA(cudaStreamWaitEvent(st, before_trsm, 0));
        trsm_part(k, 0, st);
        broadcast(k, 0, st);  // distributed: the head tile to its row and column
        convert_panel(k, 2, st);
    };
    // Panel k, the rest of the column (stream st): TRSM, broadcasts, lookahead
    // conversions.
    auto panel_tail = [&](int64_t k, cudaStream_t st) {
        if (k + 1 == NT) return;
        trsm_part(k, 1, st);
        broadcast(k, 1, st);  // distributed: the rest of the column
        convert_panel(k, 0, st);
    };

    // ---- trailing update A_ij -= L_ik L_jk^T of one part of step k ------------
    // (with paired steps, odd k also applies the deferred update of panel k-1:
    // its source-0 lists first, then source 1, then the two-panel lists)
    auto tc_update = [&](mp_precision pc, size_t off, int64_t cnt, int64_t kp, bool both, int tiles_per_cta,
                         cudaStream_t st) {
        TcGemm g;
        g.pc = pc;
        g.ta = false;
        g.tb = true;
        g.m = g.n = g.k = nb;
        g.alpha = -1.0;
        g.beta = 1.0;
        g.A = g.B = pan(MP_HALF, 0, both ? kp - 1 : kp);
        if (both) {  // C -= L_{k-1} L_{k-1}^T + L_k L_k^T in one pass
            g.A2 = g.B2 = pan(MP_HALF, 0, kp);
            g.two_panels = true;
        }
        g.lda = g.ldb = nb;
        g.a_tiles = g.b_tiles = NT;
        g.a_tile_stride = g.b_tile_stride = tt;
        g.C = t.slab[pc];
        g.ldc = nb;
        g.c_tiles = t.nslot[pc];
        g.c_tile_stride = tt;
        g.problems = reinterpret_cast<const TcProblem*>(dl + off);
        g.count = cnt;
        g.tiles_per_cta = tiles_per_cta;
        launch_tc_gemm(c, st, g);
    };
    auto update_phase = [&](int64_t k, int part, cudaStream_t st, int tiles_per_cta) {
        for (int sc = 0; sc < 2; ++sc) {
            const UpLists& U = steps[k].up[part][sc];
            const int64_t kp = sc == 0 ? k - 1 : k;  // the source panel's step
            if (U.n_tc16s) tc_update(MP_SINGLE, U.tc16s, U.n_tc16s, kp, false, tiles_per_cta, st);  // FP32 tiles, FP16 panels
            if (U.n_tc) tc_update(MP_HALF, U.tc, U.n_tc, kp, false, tiles_per_cta, st);
            if (U.n_simt16) {  // FP16 tiles of a size the tcgen05 maps cannot take
                GroupedGemm g{MP_HALF, MP_HALF, true, nb, nb, nb, nb, nb, nb, -1.0, 1.0,
                              reinterpret_cast<const TileProblem*>(dl + U.simt16), U.n_simt16};
                launch_grouped_gemm(c, st, g);
            }
            // FP64 tiles from FP16 panels (exact INT8 digit products) and FP32
            // tiles from FP32 panels (digits exact to 2^-41 of each row's max)
            for (int w32 = 0; w32 < 2; ++w32) {
                const int64_t cnt = w32 ? U.n_oz32 : U.n_oz;
                if (!cnt) continue;
                OzGemm o;
                o.A = o.B = t.digits;  // every generation: problems carry gen * NT + row
                o.a_tiles = o.b_tiles = PANEL_GENS * NT;
                o.a_slice_stride = o.b_slice_stride = tt;
                o.kpad = nb;
                o.m = o.n = o.k = nb;
                o.ldc = nb;
                o.alpha = -1.0;
                o.beta = 1.0;
                o.c_single = w32 == 1;
                o.problems = reinterpret_cast<const OzProblem*>(dl + (w32 ? U.oz32 : U.oz));
                o.count = cnt;
                o.n_lower = w32 ? U.n_oz32_lower : U.n_oz_lower;
                o.n_two = w32 ? U.n_oz32_two : U.n_oz_two;
                o.rexp_a = o.rexp_b = t.rexp;
                o.ndig_a = o.ndig_b = t.ndig;
                o.ndig_stride_a = o.ndig_stride_b = NDB;
                o.rexp_stride_a = o.rexp_stride_b = nb;
                launch_oz_gemm(c, st, o);
            }
            // FP32 / FP64 tiles on DMMA: exact products of the widened panel
            // tiles, FP64 accumulation, one rounding into the tile
            for (int pa = 0; pa < 3; ++pa)
                for (int pb = 0; pb < 3; ++pb)
                    for (int c2 = 0; c2 < 2; ++c2) {
                        const int64_t cnt = U.n_dm[pa][pb][c2];
                        if (!cnt) continue;
                        DmmaArgs d{false, true, nb, nb, nb, -1.0, 1.0, nullptr, nb, nullptr, nb, nullptr, nb, false,
                                   reinterpret_cast<const TileProblem*>(dl + U.dm[pa][pb][c2]), (mp_precision)pa};
                        d.pin_b = pb;
                        d.pout = c2 ? MP_DOUBLE : MP_SINGLE;
                        // single critical-path tiles (alone in their launch on every rank)
                        d.exclusive = part == 2 || part == 4 || part == 5;
                        d.allow_ksplit = d.exclusive;
                        ProfScope ps(c, c2 ? MP_PROF_GEMM_F64 : MP_PROF_GEMM_F32, st,
                                     2.0 * static_cast<double>(nb) * nb * nb * cnt);
                        launch_dmma_gemm(c, st, d, cnt);
                    }
            if (sc == 1) {  // tiles that take both panels in one pass
                if (U.n_tcf16s) tc_update(MP_SINGLE, U.tcf16s, U.n_tcf16s, k, true, tiles_per_cta, st);
                if (U.n_tcf) tc_update(MP_HALF, U.tcf, U.n_tcf, k, true, tiles_per_cta, st);
            }
        }
    };

    auto issue_all = [&]() {
        MP_CUDA(cudaMemsetAsync(dinfo, 0xFF, sizeof(int64_t), s));  // -1: no failure
        // Linv's strictly upper part stays zero for the whole factorization
        for (int g = 0; g < 2; ++g) MP_CUDA(cudaMemsetAsync(WL.linv64(t.work, g), 0, nn * sizeof(double), s));
        // ---- issue.  Per step k, three streams:
        //   s   : wait panel k; bulk conversions of panel k; update of everything
        //         but tile column k+1 (bulk); write tile column k back
        //   sl2 : wait panel k and bulk k-1; update of column k+1 below the diagonal;
        //         then (head/tail split) wait the head of panel k+1, TRSM and
        //         conversions of the rest of tile column k+1
        //   sl  : wait bulk k-1; SYRK of A_{k+1,k+1}; POTRF + TRTRI of panel k+1;
        //         wait sl2; TRSM + conversions of the head tile (k+2, k+1)
        //   The chain POTRF -> TRSM(head) -> SYRK -> POTRF is the critical path;
        //   the bulk GEMMs hand SMs back every few tiles so it is never starved.
        static const int tpc_env = [] {
            const char* e = getenv("MPCR_TILES_PER_CTA");
            return e ? atoi(e) : 24;
        }();
        const int bulk_tpc = la ? tpc_env : 0;
        cudaStream_t sl2 = la ? c->hi2 : s;
        cudaEvent_t* ev_panel = t.events.data();          // NT
        cudaEvent_t* ev_rest = t.events.data() + NT;      // NT
        cudaEvent_t ev_join = t.events[3 * NT + 1], ev_join2 = t.events[3 * NT + 2];
        cudaEvent_t* ev_head = t.events.data() + 3 * NT + 4;  // NT
        cudaEvent_t* ev_cv = t.events.data() + 4 * NT + 4;    // NT
        cudaEvent_t* ev_hu = t.events.data() + 5 * NT + 4;    // NT: parts 4 and 5 of step k done
        // MPCR_CONVERT_SIDE=1: the bulk's operand copies and digit planes of
        // panel k on a side stream as soon as the panel exists, next to the
        // bulk update of the previous step.  Off: measured neutral at
        // n = 131072 (1155-1162 TF/s either way, tools/r02_gpu24.sh) -- the
        // side kernels wait for SMs behind the persistent bulk GEMM.
        static const bool cv_side_env = [] {
            const char* e = getenv("MPCR_CONVERT_SIDE");
            return e && e[0] == '1';
        }();
        const bool cv_side = la && cv_side_env;
        cudaStream_t scv = cv_side ? c->aux[0] : s;
        // panel k: head on the critical-path stream, tail on the lookahead stream
        auto panel_phase = [&](int64_t k, cudaEvent_t before_trsm) {
            panel_head(k, sl, before_trsm);
            if (tsplit) {
                MP_CUDA(cudaEventRecord(ev_head[k], sl));
                MP_CUDA(cudaStreamWaitEvent(sl2, ev_head[k], 0));
                panel_tail(k, sl2);
                MP_CUDA(cudaEventRecord(ev_panel[k], sl2));
            } else {
                panel_tail(k, sl);
                if (la) MP_CUDA(cudaEventRecord(ev_panel[k], sl));
            }
        };
        if (la) {
            MP_CUDA(cudaEventRecord(ev_join, s));
            MP_CUDA(cudaStreamWaitEvent(sl, ev_join, 0));
            MP_CUDA(cudaStreamWaitEvent(sl2, ev_join, 0));
        }
        static const bool dbg_host = getenv("MPCR_DEBUG_HOST") != nullptr;
        const auto th0 = std::chrono::steady_clock::now();
        std::vector<double> th;
        panel_phase(0, nullptr);
        // MPCR_WB_ASYNC=1 (off by default: measured 0.5-0.8 % slower at n=65536 and 131072,
        // the high-priority copy steals SMs from the bulk GEMM; tools/ab_wb_async.sh):
        // write-back of tile column k off the bulk stream: on sl2 right after the tail of
        // panel k+1 (ev_panel[k+1] is recorded before it, so bulk k+1 does not wait on it).
        // The panel buffer of generation k is next written by panel k + PANEL_GENS, whose
        // head TRSM waits an ev_hu recorded on sl2 after this copy and whose tail runs on sl2.
        static const bool wb_env = [] {
            const char* e = getenv("MPCR_WB_ASYNC");
            return e && e[0] == '1';
        }();
        const bool wb_async = wb_env && tsplit;
        for (int64_t k = 0; k < NT; ++k) {
            if (la) MP_CUDA(cudaStreamWaitEvent(s, ev_panel[k], 0));
            // MPCR_CHAIN_ONLY=1 (diagnostic; the factor is meaningless): skip
            // the bulk update so a timing measures the critical chain alone
            static const bool chain_only = getenv("MPCR_CHAIN_ONLY") != nullptr;
            if (!chain_only) {
                if (cv_side) {
                    MP_CUDA(cudaStreamWaitEvent(scv, ev_panel[k], 0));
                    convert_panel(k, 1, scv);
                    MP_CUDA(cudaEventRecord(ev_cv[k], scv));
                    MP_CUDA(cudaStreamWaitEvent(s, ev_cv[k], 0));
                } else {
                    convert_panel(k, 1, s);
                }
                update_phase(k, 1, s, bulk_tpc);
            }
            if (!wb_async || k + 1 >= NT) write_back(k, s);
            if (la) MP_CUDA(cudaEventRecord(ev_rest[k], s));
            if (k + 1 < NT) {
                // after a paired bulk (odd k-1) the lookahead work of step k
                // touches only columns that bulk left to the lookahead stream
                const bool after_bulk = k >= 1 && !(pair_steps && (k - 1) % 2 == 1);
                if (la) {
                    MP_CUDA(cudaStreamWaitEvent(sl2, ev_panel[k], 0));
                    if (after_bulk) MP_CUDA(cudaStreamWaitEvent(sl2, ev_rest[k - 1], 0));
                }
                // the next head tile (and a paired step's tile (k+2, k+2)) first:
                // the critical stream waits for these, not for the whole columns
                update_phase(k, 4, sl2, 0);
                update_phase(k, 5, sl2, 0);
                if (la) MP_CUDA(cudaEventRecord(ev_hu[k], sl2));
                update_phase(k, 0, sl2, 0);
                update_phase(k, 3, sl2, 0);  // paired odd step: tile column k+2
                if (la && after_bulk) MP_CUDA(cudaStreamWaitEvent(sl, ev_rest[k - 1], 0));
                update_phase(k, 2, sl, 0);
                panel_phase(k + 1, la ? ev_hu[k] : nullptr);
                if (wb_async) write_back(k, sl2);
            }
            if (dbg_host)
                th.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th0).count());
        }
        if (dbg_host) {
            std::fprintf(stderr, "[mpcr] host issue per step (ms):");
            for (size_t q = 0; q < th.size(); q += 4) std::fprintf(stderr, " %zu:%.2f", q, th[q]);
            std::fprintf(stderr, "\n");
        }
        if (la) {
            MP_CUDA(cudaEventRecord(ev_join, sl));
            MP_CUDA(cudaEventRecord(ev_join2, sl2));
            MP_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
            MP_CUDA(cudaStreamWaitEvent(s, ev_join2, 0));
        }
        // ---- zero everything above the diagonal (lower L output) ------------------
        for (int q = 0; q < 3; ++q) {
            if (!diag_ptrs[q].empty())
                launch_batched_zero(c, s, (mp_precision)q, reinterpret_cast<void* const*>(dl + off_diag[q]),
                                    diag_ptrs[q].size(), tt, true, nb);
            if (!upper_ptrs[q].empty())
                launch_batched_zero(c, s, (mp_precision)q, reinterpret_cast<void* const*>(dl + off_upper[q]),
                                    upper_ptrs[q].size(), tt, false, nb);
        }
    };
    const bool capture = want_graph && t.chol_runs > 0 && !t.graph_failed;
    if (capture) {
        const int64_t l0 = c->launches;
        cudaGraph_t g = nullptr;
        MP_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
        bool ok = true;
        try {
            issue_all();
        } catch (const Error&) {
            ok = false;
        }
        if (cudaStreamEndCapture(s, &g) != cudaSuccess) ok = false;
        if (ok && cudaGraphInstantiate(&t.graph, g, 0) != cudaSuccess) {
            ok = false;
            t.graph = nullptr;
        }
        if (g) cudaGraphDestroy(g);
        if (ok) {
            t.graph_launches = c->launches - l0;
            t.graph_scr_gen = c->scr_gen;
            MP_CUDA(cudaGraphLaunch(t.graph, s));
        } else {  // not capturable here: stay eager for this tile
            (void)cudaGetLastError();
            t.graph_failed = true;
            c->launches = l0;
            issue_all();
        }
    } else {
        issue_all();
    }
    ++t.chol_runs;
    // first failing column over all ranks (-1 as uint64 is the largest value)
    if (t.dist && t.dist->world > 1) dist_allreduce_min_u64(t.dist, dinfo, s);
    return read_info();
}

}  // namespace mpcr

namespace {

// Whole-matrix Matern fill in one launch (square tiles, nb % 32 == 0): each
// lower tile (i, j) is computed once and also written, transposed, to (j, i).
bool fill_matern_batched(Ctx* c, mp_tile_s& x, const double* dx, const double* dy, int64_t side, double nu,
                         double range, double variance, double nugget) {
    if (x.rows != x.cols || x.br != x.bc || x.br % 32) return false;
    const size_t isz = matern_item_bytes();
    std::vector<char> items;
    for (int64_t j = 0; j < x.tc; ++j)
        for (int64_t i = j; i < x.tr; ++i) {
            void* lo = x.has(i, j) ? x.ptr(i, j) : nullptr;
            void* up = (i != j && x.has(j, i)) ? x.ptr(j, i) : nullptr;
            if (!lo && !up) continue;
            if (!lo) {  // only the upper tile is stored here: generate it as the "lower" of (j, i)
                items.resize(items.size() + isz);
                matern_item_fill(items.data() + items.size() - isz, up, nullptr, x.p(j, i), 0, j * x.br,
                                 i * x.br);
                continue;
            }
            items.resize(items.size() + isz);
            matern_item_fill(items.data() + items.size() - isz, lo, up, x.p(i, j), up ? x.p(j, i) : 0,
                             i * x.br, j * x.br);
        }
    const int64_t count = static_cast<int64_t>(items.size() / isz);
    if (count == 0) return true;
    void* d = c->ensure_scratch(items.size(), 0);
    MP_CUDA(cudaMemcpyAsync(d, items.data(), items.size(), cudaMemcpyHostToDevice, c->stream));
    launch_matern_tiles(c, c->stream, d, count, x.br, dx, dy, side, nu, range, variance, nugget);
    return true;
}

// Gaussian negative log-likelihood of z under the covariance held in t
// (factored in place).  z may be host or device memory.
void tile_nll(Ctx* c, mp_tile_s& t, const double* host_z, double jitter, double max_jitter, double* nll,
              double* logdet, double* quad, double* jitter_used) {
    if (!c || !host_z) fail(MP_INVALID_PARAM, "null argument");
    if (t.rows != t.cols || t.br != t.bc) fail(MP_SHAPE_MISMATCH, "nll: square MPCRTile required");
    cudaStream_t s = c->stream;
    const int64_t n = t.rows, nb = t.br, NT = t.tr;
    // backup of the input for jitter escalation (workloads.cpp:63-67); the
    // buffers stay with the tile (a likelihood is usually evaluated many times)
    void** backup = t.backup;
    auto slab_bytes = [&](int q) {
        return static_cast<size_t>(t.nslot[q]) * t.tt() * elem_bytes((mp_precision)q);
    };
    if (jitter > 0.0)
        for (int q = 0; q < 3; ++q)
            if (t.nslot[q]) {
                if (!backup[q]) MP_CUDA(cudaMalloc(&backup[q], slab_bytes(q)));
                MP_CUDA(cudaMemcpyAsync(backup[q], t.slab[q], slab_bytes(q), cudaMemcpyDeviceToDevice, s));
            }
    double jit = jitter > 0.0 ? jitter : 0.0;
    for (;;) {
        if (jit > 0.0)
            for (int64_t d = 0; d < NT; ++d)
                if (t.has(d, d)) launch_add_diag(c, s, t.p(d, d), t.ptr(d, d), nb, static_cast<int>(nb), jit);
        const int64_t inf = tile_chol_inplace(c, t);
        if (inf < 0) break;
        if (jit <= 0.0 || jit * 10.0 > max_jitter)
            throw Error(MP_NOT_POSITIVE_DEFINITE,
                        "matrix is not positive definite at pivot column " + std::to_string(inf), inf);
        jit *= 10.0;
        for (int q = 0; q < 3; ++q)
            if (t.nslot[q])
                MP_CUDA(cudaMemcpyAsync(t.slab[q], backup[q], slab_bytes(q), cudaMemcpyDeviceToDevice, s));
    }
    static const bool dbg_nll = getenv("MPCR_DEBUG_NLL") != nullptr;  // phase timings (diagnostics)
    cudaEvent_t dbg_ev[3] = {nullptr, nullptr, nullptr};
    if (dbg_nll) {
        for (auto& e : dbg_ev) MP_CUDA(cudaEventCreate(&e));
        MP_CUDA(cudaEventRecord(dbg_ev[0], s));
    }
    // forward solve w = L^{-1} z, tile row by tile row.  Distributed: every
    // rank accumulates its own tiles' contributions to r (rank 0 starts from
    // z, the others from 0); segment i is summed over ranks just before the
    // owner of L_ii solves it, and w_i then travels back to every rank.
    Dist* D = (t.dist && t.dist->world > 1) ? t.dist : nullptr;
    double* r = static_cast<double*>(c->ensure_scratch((n + 64) * sizeof(double), 3));
    double* dsum = r + n;
    if (D && D->rank != 0)
        MP_CUDA(cudaMemsetAsync(r, 0, n * sizeof(double), s));
    else
        MP_CUDA(cudaMemcpyAsync(r, host_z, n * sizeof(double), cudaMemcpyDefault, s));
    std::vector<TrsvItem> items;
    std::vector<size_t> off(NT * 3 + 1, 0);
    std::vector<int64_t> cnt(NT * 3, 0);
    for (int64_t i = 0; i < NT; ++i)
        for (int q = 0; q < 3; ++q) {
            off[i * 3 + q] = items.size();
            for (int64_t j = i + 1; j < NT; ++j)
                if (t.has(j, i) && t.p(j, i) == q) items.push_back(TrsvItem{t.ptr(j, i), r + j * nb});
            cnt[i * 3 + q] = static_cast<int64_t>(items.size() - off[i * 3 + q]);
        }
    TrsvItem* ditems = nullptr;
    if (!items.empty()) {
        ditems = static_cast<TrsvItem*>(c->ensure_scratch(items.size() * sizeof(TrsvItem), 0));
        MP_CUDA(cudaMemcpyAsync(ditems, items.data(), items.size() * sizeof(TrsvItem),
                                cudaMemcpyHostToDevice, s));
    }
    for (int64_t i = 0; i < NT; ++i) {
        if (D) dist_allreduce_sum_f64(D, r + i * nb, nb, s);
        if (t.has(i, i)) launch_tile_trsv(c, s, t.p(i, i), t.ptr(i, i), nb, static_cast<int>(nb), r + i * nb);
        if (D) dist_bcast(D, r + i * nb, nb * sizeof(double), dist_owner(i, i, D->P, D->Q), DC_WORLD, s);
        for (int q = 0; q < 3; ++q)
            if (cnt[i * 3 + q])
                launch_tile_gemv(c, s, (mp_precision)q, ditems + off[i * 3 + q], cnt[i * 3 + q],
                                 static_cast<int>(nb), r + i * nb);
    }
    if (dbg_nll) MP_CUDA(cudaEventRecord(dbg_ev[1], s));
    launch_square_sum(c, s, r, n, dsum);
    MP_CUDA(cudaMemsetAsync(dsum + 1, 0, sizeof(double), s));
    for (int64_t d = 0; d < NT; ++d)
        if (t.has(d, d)) launch_logdiag_sum(c, s, t.p(d, d), t.ptr(d, d), nb, nb, dsum + 1);
    if (D) dist_allreduce_sum_f64(D, dsum + 1, 1, s);
    double h[2];
    MP_CUDA(cudaMemcpyAsync(h, dsum, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (dbg_nll) MP_CUDA(cudaEventRecord(dbg_ev[2], s));
    MP_CUDA(cudaStreamSynchronize(s));
    if (dbg_nll) {
        float a = 0, b = 0;
        MP_CUDA(cudaEventElapsedTime(&a, dbg_ev[0], dbg_ev[1]));
        MP_CUDA(cudaEventElapsedTime(&b, dbg_ev[1], dbg_ev[2]));
        std::fprintf(stderr, "[mpcr] nll: forward solve %.3f ms, sums %.3f ms\n", a, b);
        for (auto e : dbg_ev) cudaEventDestroy(e);
    }
    const double ld = 2.0 * h[1];
    if (quad) *quad = h[0];
    if (logdet) *logdet = ld;
    if (nll) *nll = 0.5 * h[0] + 0.5 * ld + 0.5 * static_cast<double>(n) * std::log(2.0 * M_PI);
    if (jitter_used) *jitter_used = jit;
}

// Shared by mp_tile_create / mp_tile_create_dist: with `dist`, only the
// lower-triangle tiles this rank owns get storage (slot -1 elsewhere).
mp_tile_s* tile_new(Ctx* ctx, mp_dist_s* dist, int64_t rows, int64_t cols, int64_t rpt, int64_t cpt,
                    const int* precisions) {
    if (rows < 1 || cols < 1 || rpt < 1 || cpt < 1)
        fail(MP_INVALID_PARAM, "MPCRTile: sizes must be >= 1");
    if (rows % rpt || cols % cpt)
        fail(MP_SHAPE_MISMATCH, "MPCRTile: tile size must divide the matrix size");
    auto* t = new mp_tile_s();
    t->ctx = ctx;
    t->dist = dist;
    t->rows = rows;
    t->cols = cols;
    t->br = rpt;
    t->bc = cpt;
    t->tr = rows / rpt;
    t->tc = cols / cpt;
    const int64_t nt = t->tr * t->tc;
    t->prec.resize(nt);
    t->slot.resize(nt);
    for (int64_t q = 0; q < nt; ++q) {
        if (precisions[q] < 0 || precisions[q] > 2) {
            delete t;
            fail(MP_INVALID_PARAM, "MPCRTile: unknown precision code");
        }
        t->prec[q] = static_cast<mp_precision>(precisions[q]);
        const int64_t i = q % t->tr, j = q / t->tr;
        const bool stored = !dist || (i >= j && dist_owner(i, j, dist->P, dist->Q) == dist->rank);
        t->slot[q] = stored ? t->nslot[precisions[q]]++ : -1;
    }
    try {
        for (int q = 0; q < 3; ++q)
            if (t->nslot[q]) {
                const size_t bytes = static_cast<size_t>(t->nslot[q]) * t->tt() * elem_bytes((mp_precision)q);
                MP_CUDA(cudaMalloc(&t->slab[q], bytes));
                MP_CUDA(cudaMemsetAsync(t->slab[q], 0, bytes, ctx->stream));
            }
    } catch (...) {
        delete t;
        throw;
    }
    return t;
}

}  // namespace

extern "C" {

mp_status mp_tile_create(mp_ctx ctx, int64_t rows, int64_t cols, int64_t rpt, int64_t cpt,
                         const int* precisions, mp_tile* out) {
    MP_API_BEGIN
    if (!ctx || !out || !precisions) fail(MP_INVALID_PARAM, "null argument");
    bind_device(ctx);
    *out = tile_new(ctx, nullptr, rows, cols, rpt, cpt, precisions);
    MP_API_END
}

// 2D block-cyclic MPCRTile: tile (i, j), i >= j, stored on rank
// (i mod P) * Q + (j mod Q) only.
mp_status mp_tile_create_dist(mp_ctx ctx, mp_dist dist, int64_t n, int64_t tile, const int* precisions,
                              mp_tile* out) {
    MP_API_BEGIN
    if (!ctx || !dist || !out || !precisions) fail(MP_INVALID_PARAM, "null argument");
    bind_device(ctx);
    if (dist->ctx != static_cast<Ctx*>(ctx)) fail(MP_INVALID_PARAM, "dist belongs to another context");
    *out = tile_new(ctx, dist, n, n, tile, tile, precisions);
    MP_API_END
}

int mp_tile_owns(mp_tile t, int64_t i, int64_t j) {
    if (!t || i < 0 || j < 0 || i >= t->tr || j >= t->tc) return 0;
    return t->has(i, j) ? 1 : 0;
}

mp_status mp_tile_destroy(mp_tile t) {
    MP_API_BEGIN
    if (t) delete t;  // cudaFree in the destructor synchronises the device
    MP_API_END
}

mp_status mp_tile_info(mp_tile t, int64_t* rows, int64_t* cols, int64_t* rpt, int64_t* cpt,
                       int64_t* tiles_r, int64_t* tiles_c) {
    MP_API_BEGIN
    mp_tile_s& x = T_(t);
    if (rows) *rows = x.rows;
    if (cols) *cols = x.cols;
    if (rpt) *rpt = x.br;
    if (cpt) *cpt = x.bc;
    if (tiles_r) *tiles_r = x.tr;
    if (tiles_c) *tiles_c = x.tc;
    MP_API_END
}

mp_status mp_tile_set_values_device(mp_tile t, const double* dev, int64_t ld) {
    MP_API_BEGIN
    mp_tile_s& x = T_(t);
    Ctx* c = x.ctx;
    for (int64_t j = 0; j < x.tc; ++j)
        for (int64_t i = 0; i < x.tr; ++i)
            if (x.has(i, j))
                launch_convert(c, c->stream, MP_DOUBLE, dev + (j * x.bc) * ld + i * x.br, ld, x.p(i, j),
                               x.ptr(i, j), x.br, x.br, x.bc);
    MP_API_END
}

mp_status mp_tile_set_values(mp_tile t, const double* host) {
    MP_API_BEGIN
    mp_tile_s& x = T_(t);
    Ctx* c = x.ctx;
    // one tile-column panel at a time (rows x bc doubles)
    const size_t panel = static_cast<size_t>(x.rows) * x.bc;
    double* tmp = static_cast<double*>(c->ensure_scratch(panel * sizeof(double), 1));
    for (int64_t j = 0; j < x.tc; ++j) {
        MP_CUDA(cudaMemcpyAsync(tmp, host + j * x.bc * x.rows, panel * sizeof(double),
                                cudaMemcpyHostToDevice, c->stream));
        for (int64_t i = 0; i < x.tr; ++i)
            if (x.has(i, j))
                launch_convert(c, c->stream, MP_DOUBLE, tmp + i * x.br, x.rows, x.p(i, j), x.ptr(i, j),
                               x.br, x.br, x.bc);
        MP_CUDA(cudaStreamSynchronize(c->stream));
    }
    MP_API_END
}

mp_status mp_tile_get_values(mp_tile t, double* host) {
    MP_API_BEGIN
    mp_tile_s& x = T_(t);
    Ctx* c = x.ctx;
    const size_t panel = static_cast<size_t>(x.rows) * x.bc;
    double* tmp = static_cast<double*>(c->ensure_scratch(panel * sizeof(double), 1));
    for (int64_t j = 0; j < x.tc; ++j) {
        // distributed tiles: tiles held by other ranks read as zeros
        if (x.dist) MP_CUDA(cudaMemsetAsync(tmp, 0, panel * sizeof(double), c->stream));
        for (int64_t i = 0; i < x.tr; ++i)
            if (x.has(i, j))
                launch_convert(c, c->stream, x.p(i, j), x.ptr(i, j), x.br, MP_DOUBLE, tmp + i * x.br,
                               x.rows, x.br, x.bc);
        MP_CUDA(cudaMemcpyAsync(host + j * x.bc * x.rows, tmp, panel * sizeof(double),
                                cudaMemcpyDeviceToHost, c->stream));
        MP_CUDA(cudaStreamSynchronize(c->stream));
    }
    MP_API_END
}

// Selected rows of the whole matrix, widened to double, row-major
// (count x cols, out[q * cols + c]); tiles this rank does not store read as
// zeros.  Used to check factors too large to download (sampled residuals).
mp_status mp_tile_get_rows(mp_tile t, const int64_t* rows, int64_t count, double* host) {
    MP_API_BEGIN
    mp_tile_s& x = T_(t);
    if (count < 0 || (count > 0 && (!rows || !host))) fail(MP_INVALID_PARAM, "get_rows: null argument");
    if (count == 0) return MP_OK;
    if (x.br != x.bc) fail(MP_SHAPE_MISMATCH, "get_rows: square tiles required");
    for (int64_t q = 0; q < count; ++q)
        if (rows[q] < 0 || rows[q] >= x.rows) fail(MP_INDEX_OUT_OF_RANGE, "get_rows: row index out of range");
    Ctx* c = x.ctx;
    const size_t out_bytes = static_cast<size_t>(count) * x.cols * sizeof(double);
    std::vector<RowItem> items;
    items.reserve(static_cast<size_t>(count) * x.tc);
    char* scr = static_cast<char*>(c->ensure_scratch(out_bytes + 256 + count * x.tc * sizeof(RowItem), 1));
    double* dout = reinterpret_cast<double*>(scr);
    RowItem* dit = reinterpret_cast<RowItem*>(scr + (out_bytes + 255) / 256 * 256);
    MP_CUDA(cudaMemsetAsync(dout, 0, out_bytes, c->stream));
    for (int64_t q = 0; q < count; ++q) {
        const int64_t i = rows[q] / x.br, r = rows[q] % x.br;
        for (int64_t j = 0; j < x.tc; ++j)
            if (x.has(i, j))
                items.push_back(RowItem{x.ptr(i, j), dout + q * x.cols + j * x.bc, static_cast<int32_t>(r),
                                        static_cast<int32_t>(x.p(i, j))});
    }
    if (!items.empty()) {
        MP_CUDA(cudaMemcpyAsync(dit, items.data(), items.size() * sizeof(RowItem), cudaMemcpyHostToDevice,
                                c->stream));
        launch_gather_rows(c, c->stream, dit, static_cast<int64_t>(items.size()), x.br, 1);
    }
    MP_CUDA(cudaMemcpyAsync(host, dout, out_bytes, cudaMemcpyDeviceToHost, c->stream));
    MP_CUDA(cudaStreamSynchronize(c->stream));
    MP_API_END
}

mp_status mp_tile_get_tile(mp_tile t, int64_t i, int64_t j, mp_array* view) {
    MP_API_BEGIN
    mp_tile_s& x = T_(t);
    if (i < 0 || j < 0 || i >= x.tr || j >= x.tc)
        fail(MP_INDEX_OUT_OF_RANGE, "GetTile: tile index out of range");
    if (!x.has(i, j)) fail(MP_INVALID_PARAM, "GetTile: tile is stored on another rank");
    return mp_array_wrap(static_cast<mp_ctx>(x.ctx), x.p(i, j), x.br, x.bc, x.br, x.ptr(i, j), view);
    MP_API_END
}

mp_status mp_tile_precision(mp_tile t, int64_t i, int64_t j, mp_precision* p) {
    MP_API_BEGIN
    mp_tile_s& x = T_(t);
    if (i < 0 || j < 0 || i >= x.tr || j >= x.tc)
        fail(MP_INDEX_OUT_OF_RANGE, "tile index out of range");
    *p = x.p(i, j);
    MP_API_END
}

mp_status mp_tile_chol(mp_ctx ctx, mp_tile a, int overwrite_input, mp_tile* out, int64_t* info) {
    MP_API_BEGIN
    mp_tile_s& x = T_(a);
    if (info) *info = -1;
    if (!ctx) fail(MP_INVALID_PARAM, "null context");
    if (x.rows != x.cols || x.br != x.bc)
        fail(MP_SHAPE_MISMATCH, "chol: MPCRTile must be square with square tiles");
    mp_tile_s* target = &x;
    if (!overwrite_input) {
        if (!out) fail(MP_INVALID_PARAM, "chol: out is required when overwrite_input is false");
        std::vector<int> pr(x.prec.begin(), x.prec.end());
        mp_tile nt = tile_new(ctx, x.dist, x.rows, x.cols, x.br, x.bc, pr.data());
        for (int q = 0; q < 3; ++q)
            if (x.nslot[q])
                MP_CUDA(cudaMemcpyAsync(nt->slab[q], x.slab[q],
                                        static_cast<size_t>(x.nslot[q]) * x.tt() * elem_bytes((mp_precision)q),
                                        cudaMemcpyDeviceToDevice, ctx->stream));
        target = nt;
        *out = nt;
    }
    const int64_t inf = tile_chol_inplace(ctx, *target);
    if (inf >= 0) {
        if (info) *info = inf;
        throw Error(MP_NOT_POSITIVE_DEFINITE,
                    "matrix is not positive definite at pivot column " + std::to_string(inf), inf);
    }
    MP_API_END
}

// MPCRTile.gemm: every tile product in C-tile precision,
// operands converted to it (oracle: ref_tile_gemm).
mp_status mp_tile_gemm(mp_ctx ctx, mp_tile a, mp_tile b, mp_tile cc, int ta, int tb, double alpha,
                       double beta) {
    MP_API_BEGIN
    mp_tile_s &A = T_(a), &B = T_(b), &C = T_(cc);
    Ctx* c = ctx;
    if (!c) fail(MP_INVALID_PARAM, "null context");
    if (A.dist || B.dist || C.dist) fail(MP_INVALID_PARAM, "tile gemm: distributed MPCRTile not supported");
    const int64_t kt = ta ? A.tr : A.tc, kb = tb ? B.tc : B.tr;
    const int64_t mt = ta ? A.tc : A.tr, ntl = tb ? B.tr : B.tc;
    const int64_t abr = ta ? A.bc : A.br, abk = ta ? A.br : A.bc;
    const int64_t bbk = tb ? B.bc : B.br, bbn = tb ? B.br : B.bc;
    if (kt != kb || mt != C.tr || ntl != C.tc || abk != bbk || abr != C.br || bbn != C.bc)
        fail(MP_SHAPE_MISMATCH, "tile gemm: incompatible tile grids");
    const size_t amax = static_cast<size_t>(A.tt()) * 8, bmax = static_cast<size_t>(B.tt()) * 8;
    char* scr = static_cast<char*>(c->ensure_scratch(amax + bmax + 256, 0));
    void* xa = scr;
    void* xb = scr + ((amax + 255) / 256) * 256;
    for (int64_t j = 0; j < C.tc; ++j)
        for (int64_t i = 0; i < C.tr; ++i) {
            const mp_precision pc = C.p(i, j);
            for (int64_t l = 0; l < kt; ++l) {
                const int64_t ai = ta ? l : i, aj = ta ? i : l;
                const int64_t bi = tb ? j : l, bj = tb ? l : j;
                const void* pa = A.ptr(ai, aj);
                const void* pb = B.ptr(bi, bj);
                if (A.p(ai, aj) != pc) {
                    launch_convert(c, c->stream, A.p(ai, aj), pa, A.br, pc, xa, A.br, A.br, A.bc);
                    pa = xa;
                }
                if (B.p(bi, bj) != pc) {
                    launch_convert(c, c->stream, B.p(bi, bj), pb, B.br, pc, xb, B.br, B.br, B.bc);
                    pb = xb;
                }
                GemmDesc g{pc, pc, pc, ta != 0, tb != 0, C.br, C.bc, abk, alpha, l == 0 ? beta : 1.0,
                           pa, A.br, pb, B.br, C.ptr(i, j), C.br};
                launch_gemm(c, c->stream, g);
            }
        }
    MP_API_END
}

// MPCRTile.trsm: tile substitution in B-tile precision
// (oracle: ref_tile_trsm).  All diagonal tiles are checked for exact zeros
// before B is touched.
mp_status mp_tile_trsm(mp_ctx ctx, mp_tile a, mp_tile b, mp_side side, int upper, int trans,
                       double alpha) {
    MP_API_BEGIN
    mp_tile_s &A = T_(a), &B = T_(b);
    Ctx* c = ctx;
    if (!c) fail(MP_INVALID_PARAM, "null context");
    if (A.dist || B.dist) fail(MP_INVALID_PARAM, "tile trsm: distributed MPCRTile not supported");
    if (A.rows != A.cols || A.br != A.bc) fail(MP_SHAPE_MISMATCH, "tile trsm: A must be square");
    const int64_t nt = A.tr, nb = A.br;
    const bool right = side == MP_RIGHT;
    if (!right && (B.tr != nt || B.br != nb)) fail(MP_SHAPE_MISMATCH, "tile trsm: B row tiling");
    if (right && (B.tc != nt || B.bc != nb)) fail(MP_SHAPE_MISMATCH, "tile trsm: B col tiling");
    for (int64_t d = 0; d < nt; ++d) {
        // zero check in the compute precision of every B tile that uses A_dd
        mp_precision worst = MP_DOUBLE;
        for (int64_t q = 0; q < (right ? B.tr : B.tc); ++q) {
            const mp_precision pb = right ? B.p(q, d) : B.p(d, q);
            worst = std::min(worst, compute_precision(pb));
        }
        if (find_zero_diag(c, c->stream, A.p(d, d), A.ptr(d, d), nb, nb, worst) >= 0)
            fail(MP_SINGULAR_MATRIX, "triangular solve: zero diagonal in tile " + std::to_string(d));
    }
    const bool eff_lower = (upper != 0) == (trans != 0);
    const size_t tmax = static_cast<size_t>(std::max(A.tt(), B.tt())) * 8;
    char* scr = static_cast<char*>(c->ensure_scratch(2 * tmax + 256, 0));
    void* xa = scr;
    void* xb = scr + ((tmax + 255) / 256) * 256;
    auto opA = [&](int64_t r, int64_t k, int64_t& si, int64_t& sj) {
        si = trans ? k : r;
        sj = trans ? r : k;
    };
    auto conv = [&](const mp_tile_s& T, int64_t i, int64_t j, mp_precision to, void* tmp) -> const void* {
        if (T.p(i, j) == to) return T.ptr(i, j);
        launch_convert(c, c->stream, T.p(i, j), T.ptr(i, j), T.br, to, tmp, T.br, T.br, T.bc);
        return tmp;
    };
    if (!right) {
        for (int64_t s = 0; s < nt; ++s) {
            const int64_t r = eff_lower ? s : nt - 1 - s;
            for (int64_t cidx = 0; cidx < B.tc; ++cidx) {
                const mp_precision pt = B.p(r, cidx);
                bool first = true;
                for (int64_t q = 0; q < s; ++q) {
                    const int64_t k = eff_lower ? q : nt - 1 - q;
                    int64_t si, sj;
                    opA(r, k, si, sj);
                    const void* pa = conv(A, si, sj, pt, xa);
                    const void* pbp = conv(B, k, cidx, pt, xb);
                    GemmDesc g{pt, pt, pt, trans != 0, false, nb, B.bc, nb, -1.0, first ? alpha : 1.0,
                               pa, nb, pbp, B.br, B.ptr(r, cidx), B.br};
                    launch_gemm(c, c->stream, g);
                    first = false;
                }
                const void* pd = conv(A, r, r, pt, xa);
                launch_tri_solve(c, c->stream, pt, pd, nb, nb, upper != 0, trans != 0, pt,
                                 B.ptr(r, cidx), B.br, B.bc, first ? alpha : 1.0, false, B.br);
            }
        }
    } else {
        for (int64_t s = 0; s < nt; ++s) {
            const int64_t cidx = eff_lower ? nt - 1 - s : s;
            for (int64_t r = 0; r < B.tr; ++r) {
                const mp_precision pt = B.p(r, cidx);
                bool first = true;
                for (int64_t q = 0; q < s; ++q) {
                    const int64_t k = eff_lower ? nt - 1 - q : q;
                    int64_t si, sj;
                    opA(k, cidx, si, sj);
                    const void* pbp = conv(B, r, k, pt, xb);
                    const void* pa = conv(A, si, sj, pt, xa);
                    GemmDesc g{pt, pt, pt, false, trans != 0, B.br, nb, nb, -1.0, first ? alpha : 1.0,
                               pbp, B.br, pa, nb, B.ptr(r, cidx), B.br};
                    launch_gemm(c, c->stream, g);
                    first = false;
                }
                const void* pd = conv(A, cidx, cidx, pt, xa);
                launch_tri_solve(c, c->stream, pt, pd, nb, nb, upper != 0, trans != 0, pt,
                                 B.ptr(r, cidx), B.br, B.bc, first ? alpha : 1.0, true, B.br);
            }
        }
    }
    MP_API_END
}

mp_status mp_tile_logdet(mp_ctx ctx, mp_tile l, double* logdet) {
    MP_API_BEGIN
    mp_tile_s& x = T_(l);
    Ctx* c = ctx;
    if (!c) fail(MP_INVALID_PARAM, "null context");
    if (x.rows != x.cols || x.br != x.bc) fail(MP_SHAPE_MISMATCH, "logdet: square MPCRTile required");
    double* acc = static_cast<double*>(c->ensure_scratch(64, 1));
    MP_CUDA(cudaMemsetAsync(acc, 0, sizeof(double), c->stream));
    for (int64_t d = 0; d < x.tr; ++d)
        if (x.has(d, d)) launch_logdiag_sum(c, c->stream, x.p(d, d), x.ptr(d, d), x.br, x.br, acc);
    if (x.dist) dist_allreduce_sum_f64(x.dist, acc, 1, c->stream);
    double h = 0;
    MP_CUDA(cudaMemcpyAsync(&h, acc, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    MP_CUDA(cudaStreamSynchronize(c->stream));
    *logdet = 2.0 * h;
    MP_API_END
}

mp_status mp_tile_fill_matern(mp_ctx ctx, mp_tile t, int64_t side, double nu, double range,
                              double variance) {
    MP_API_BEGIN
    mp_tile_s& x = T_(t);
    Ctx* c = ctx;
    if (!c) fail(MP_INVALID_PARAM, "null context");
    if (side < 2) fail(MP_INVALID_PARAM, "grid_locations: side length must be >= 2");
    if (side * side < x.rows || side * side < x.cols)
        fail(MP_INVALID_PARAM, "matern: grid has fewer points than the matrix");
    if (range <= 0.0 || variance <= 0.0)
        fail(MP_INVALID_PARAM, "matern_cov: range and variance must be positive");
    if (nu != 0.5 && nu != 1.5 && nu != 2.5) fail(MP_INVALID_PARAM, "matern_cov: nu must be 0.5, 1.5, or 2.5");
    if (!fill_matern_batched(c, x, nullptr, nullptr, side, nu, range, variance, 0.0))
        for (int64_t j = 0; j < x.tc; ++j)
            for (int64_t i = 0; i < x.tr; ++i)
                if (x.has(i, j))
                    launch_matern_tile(c, c->stream, x.p(i, j), x.ptr(i, j), x.br, i * x.br, j * x.bc,
                                       x.br, x.bc, side, nu, range, variance);
    MP_API_END
}

mp_status mp_tile_fill_matern_points(mp_ctx ctx, mp_tile t, const double* host_x,
                                     const double* host_y, int64_t n, double nu, double range,
                                     double variance, double nugget) {
    MP_API_BEGIN
    mp_tile_s& x = T_(t);
    Ctx* c = ctx;
    if (!c || !host_x || !host_y) fail(MP_INVALID_PARAM, "null argument");
    if (n != x.rows || n != x.cols) fail(MP_SHAPE_MISMATCH, "matern: n must equal rows = cols");
    if (range <= 0.0 || variance <= 0.0)
        fail(MP_INVALID_PARAM, "matern_cov: range and variance must be positive");
    if (nu != 0.5 && nu != 1.5 && nu != 2.5) fail(MP_INVALID_PARAM, "matern_cov: nu must be 0.5, 1.5, or 2.5");
    double* xy = static_cast<double*>(c->ensure_scratch(2 * n * sizeof(double), 1));
    MP_CUDA(cudaMemcpyAsync(xy, host_x, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    MP_CUDA(cudaMemcpyAsync(xy + n, host_y, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    if (!fill_matern_batched(c, x, xy, xy + n, 0, nu, range, variance, nugget))
        for (int64_t j = 0; j < x.tc; ++j)
            for (int64_t i = 0; i < x.tr; ++i)
                if (x.has(i, j))
                    launch_matern_points(c, c->stream, x.p(i, j), x.ptr(i, j), x.br, i * x.br, j * x.bc,
                                         x.br, x.bc, xy, xy + n, nu, range, variance, nugget);
    MP_API_END
}

mp_status mp_tile_gaussian_nll(mp_ctx ctx, mp_tile cov, const double* host_z, double jitter,
                               double max_jitter, double* nll, double* logdet, double* quad,
                               double* jitter_used) {
    MP_API_BEGIN
    tile_nll(ctx, T_(cov), host_z, jitter, max_jitter, nll, logdet, quad, jitter_used);
    MP_API_END
}

// matern_mle (workloads.cpp:89-110) with the likelihood on the device.  The
// simplex search restates stats::nelder_mead (optimize.cpp:9-95): start
// simplex x0 and x0 + 5 % (2.5e-4 for a zero coordinate) per axis, vertices
// kept sorted by value (stable), stop when the population standard deviation
// of the vertex values is below tol; reflection -1, expansion -2, outside /
// inside contraction -1/2 / +1/2 about the centroid of all but the worst,
// shrink 1/2 toward the best.  Every evaluation regenerates the Matern
// covariance for (range, sigma2) = exp(params) on the device and factors it.
mp_status mp_tile_matern_mle(mp_ctx ctx, mp_tile cov, const double* host_x, const double* host_y,
                             const double* host_z, int64_t n, double nu, double init_log_range,
                             double init_log_sigma2, int max_iter, double tol, double jitter,
                             double max_jitter, double* range_hat, double* sigma2_hat, double* nll,
                             int* iterations, int* converged) {
    MP_API_BEGIN
    mp_tile_s& t = T_(cov);
    Ctx* c = ctx;
    if (!c || !host_x || !host_y || !host_z) fail(MP_INVALID_PARAM, "null argument");
    if (n != t.rows || n != t.cols || t.br != t.bc) fail(MP_SHAPE_MISMATCH, "mle: n x n MPCRTile with square tiles");
    if (nu != 0.5 && nu != 1.5 && nu != 2.5) fail(MP_INVALID_PARAM, "matern_cov: nu must be 0.5, 1.5, or 2.5");
    if (max_iter < 0) fail(MP_INVALID_PARAM, "mle: max_iter must be >= 0");
    // points and observations stay on the device for the whole search
    double* d = nullptr;
    MP_CUDA(cudaMalloc(&d, 3 * n * sizeof(double)));
    struct Free {
        double* p;
        ~Free() {
            if (p) cudaFree(p);
        }
    } free_d{d};
    MP_CUDA(cudaMemcpyAsync(d, host_x, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    MP_CUDA(cudaMemcpyAsync(d + n, host_y, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    MP_CUDA(cudaMemcpyAsync(d + 2 * n, host_z, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    using Pt = std::array<double, 2>;
    auto objective = [&](const Pt& q) {
        const double range = std::exp(q[0]), sigma2 = std::exp(q[1]);
        if (!(range > 0.0) || !(sigma2 > 0.0) || !std::isfinite(range) || !std::isfinite(sigma2))
            fail(MP_INVALID_PARAM, "matern_cov: range and variance must be positive");
        if (!fill_matern_batched(c, t, d, d + n, 0, nu, range, sigma2, 0.0))
            for (int64_t j = 0; j < t.tc; ++j)
                for (int64_t i = 0; i < t.tr; ++i)
                    if (t.has(i, j))
                        launch_matern_points(c, c->stream, t.p(i, j), t.ptr(i, j), t.br, i * t.br, j * t.bc, t.br,
                                             t.bc, d, d + n, nu, range, sigma2, 0.0);
        double v = 0.0;
        tile_nll(c, t, d + 2 * n, jitter, max_jitter, &v, nullptr, nullptr, nullptr);
        return v;
    };
    constexpr int K = 2;
    std::array<Pt, K + 1> vx;
    std::array<double, K + 1> vf;
    const Pt x0 = {init_log_range, init_log_sigma2};
    for (int v = 0; v <= K; ++v) vx[v] = x0;
    for (int i = 0; i < K; ++i) vx[i + 1][i] += x0[i] != 0.0 ? 0.05 * x0[i] : 0.00025;
    for (int v = 0; v <= K; ++v) vf[v] = objective(vx[v]);
    auto spread = [&] {  // population standard deviation of the vertex values
        double mean = 0.0;
        for (double f : vf) mean += f;
        mean /= static_cast<double>(K + 1);
        double acc = 0.0;
        for (double f : vf) acc += (f - mean) * (f - mean);
        return std::sqrt(acc / static_cast<double>(K + 1));
    };
    int it = 0;
    bool done = false;
    for (; it < max_iter; ++it) {
        std::array<int, K + 1> ord;
        for (int v = 0; v <= K; ++v) ord[v] = v;
        std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return vf[a] < vf[b]; });
        const auto ox = vx;
        const auto of = vf;
        for (int v = 0; v <= K; ++v) {
            vx[v] = ox[ord[v]];
            vf[v] = of[ord[v]];
        }
        if (spread() < tol) {
            done = true;
            break;
        }
        Pt cen = {0.0, 0.0};
        for (int i = 0; i < K; ++i) {
            for (int v = 0; v < K; ++v) cen[i] += vx[v][i];
            cen[i] /= static_cast<double>(K);
        }
        auto along = [&](double coef) {
            Pt q;
            for (int i = 0; i < K; ++i) q[i] = cen[i] + coef * (vx[K][i] - cen[i]);
            return q;
        };
        const Pt xr = along(-1.0);
        const double fr = objective(xr);
        if (fr < vf[0]) {
            const Pt xe = along(-2.0);
            const double fe = objective(xe);
            if (fe < fr) {
                vx[K] = xe;
                vf[K] = fe;
            } else {
                vx[K] = xr;
                vf[K] = fr;
            }
        } else if (fr < vf[K - 1]) {
            vx[K] = xr;
            vf[K] = fr;
        } else {
            const bool outside = fr < vf[K];
            const Pt xc = along(outside ? -0.5 : 0.5);
            const double fc = objective(xc);
            if (fc < (outside ? fr : vf[K])) {
                vx[K] = xc;
                vf[K] = fc;
            } else {
                for (int v = 1; v <= K; ++v) {
                    for (int i = 0; i < K; ++i) vx[v][i] = vx[0][i] + 0.5 * (vx[v][i] - vx[0][i]);
                    vf[v] = objective(vx[v]);
                }
            }
        }
    }
    int best = 0;
    if (!done)
        for (int v = 1; v <= K; ++v)
            if (vf[v] < vf[best]) best = v;
    if (range_hat) *range_hat = std::exp(vx[best][0]);
    if (sigma2_hat) *sigma2_hat = std::exp(vx[best][1]);
    if (nll) *nll = vf[best];
    if (iterations) *iterations = it;
    if (converged) *converged = done ? 1 : 0;
    MP_API_END
}

// Tile-wise MPArray::converted (array.cpp:187-191): every tile of src
// converted into the precision dst holds for it (same grid and tiling).
mp_status mp_tile_convert(mp_ctx ctx, mp_tile dst, mp_tile src) {
    MP_API_BEGIN
    mp_tile_s &d = T_(dst), &s = T_(src);
    if (!ctx) fail(MP_INVALID_PARAM, "null context");
    if (d.rows != s.rows || d.cols != s.cols || d.br != s.br || d.bc != s.bc)
        fail(MP_SHAPE_MISMATCH, "tile convert: grids differ");
    for (int64_t j = 0; j < s.tc; ++j)
        for (int64_t i = 0; i < s.tr; ++i) {
            if (s.has(i, j) != d.has(i, j)) fail(MP_SHAPE_MISMATCH, "tile convert: tiles distributed differently");
            if (s.has(i, j))
                launch_convert(ctx, ctx->stream, s.p(i, j), s.ptr(i, j), s.br, d.p(i, j), d.ptr(i, j), d.br, s.br,
                               s.bc);
        }
    MP_API_END
}

mp_status mp_tile_copy(mp_ctx ctx, mp_tile dst, mp_tile src) {
    MP_API_BEGIN
    mp_tile_s &d = T_(dst), &s = T_(src);
    if (!ctx) fail(MP_INVALID_PARAM, "null context");
    if (d.rows != s.rows || d.cols != s.cols || d.br != s.br || d.bc != s.bc || d.prec != s.prec)
        fail(MP_SHAPE_MISMATCH, "tile copy: grids differ");
    if (d.slot != s.slot) fail(MP_SHAPE_MISMATCH, "tile copy: tiles distributed differently");
    for (int q = 0; q < 3; ++q)
        if (s.nslot[q])
            MP_CUDA(cudaMemcpyAsync(d.slab[q], s.slab[q],
                                    static_cast<size_t>(s.nslot[q]) * s.tt() * elem_bytes((mp_precision)q),
                                    cudaMemcpyDeviceToDevice, ctx->stream));
    MP_API_END
}

}  // extern "C"
