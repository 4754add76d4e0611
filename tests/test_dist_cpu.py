"""Multi-process (gloo, CPU) test of the distributed MPCRTile Cholesky plan.

The GPU executor (csrc/tile.cpp over csrc/dist.cpp) runs, on every rank, the
action list ``mp_dist_schedule`` returns for a P x Q 2D block-cyclic grid.
This test runs the SAME action lists on 2 or 4 CPU processes, with the tile
kernels taken from the oracle port (oracle/mpnum_oracle.c, the restatement
of the reference composition ref_tile_chol) and the NCCL
broadcasts replaced by gloo broadcasts on the same row / column groups the
GPU executor splits its communicator into (L_kk^-1 down process column
k mod Q; L_ik along process row i mod P, then down process column i mod Q).
The distributed result must equal the single-process oracle factor bit for
bit: the plan moves exactly the data every tile kernel needs, in the order
the sequential algorithm uses it.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp_

POTRF, BCAST_DIAG, TRSM, BCAST_PANEL, UPDATE = 1, 2, 3, 4, 5
WORLD, ROW, COL = 0, 1, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(n, nb, seed=7):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, n))
    A = X @ X.T / n + np.eye(n) * 2.0
    nt = n // nb
    i, j = np.indices((nt, nt))
    prec = np.where(i == j, 2, np.where(abs(i - j) <= 2, 1, 0)).astype(np.int32)
    return A, prec


def _worker(rank, world, P, Q, port, n, nb, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2406_02701_b200 as mp
        from oracle.oracle import Port, round_to

        port_ = Port()
        A, prec = _problem(n, nb)
        nt = n // nb
        tile = lambda M, i, j: np.array(M[i * nb:(i + 1) * nb, j * nb:(j + 1) * nb], order="F")
        # owned lower tiles, rounded to their precision (MPCRTile storage)
        mine = {}
        for j in range(nt):
            for i in range(j, nt):
                if mp.dist_owner(i, j, P, Q) == rank:
                    mine[(i, j)] = round_to(tile(A, i, j), int(prec[i, j]))
        sched = mp.dist_schedule(rank, P, Q, nt, prec)
        # the row / column communicators (every rank creates every group)
        rows = [dist.new_group([r * Q + c for c in range(Q)]) for r in range(P)]
        cols = [dist.new_group([r * Q + c for r in range(P)]) for c in range(Q)]
        group = {ROW: rows[rank // Q], COL: cols[rank % Q], WORLD: None}
        u = np.zeros((nb, nb), order="F")
        panel = {}
        for op, k, i, j, root, p, comm in sched.tolist():
            if op == POTRF:
                u = port_.chol(p, mine[(k, k)])           # U_kk (reads the upper triangle)
                mine[(k, k)] = np.asfortranarray(u.T)     # L_kk = U_kk^T
            elif op == BCAST_DIAG:
                assert comm == COL and root % Q == rank % Q
                t = torch.from_numpy(np.ascontiguousarray(u))
                dist.broadcast(t, src=root, group=group[comm])
                u = np.asfortranarray(t.numpy())
            elif op == TRSM:
                x = round_to(u, p)                        # U_kk.converted(p_ik)
                mine[(i, k)] = port_.trsm(p, p, x, mine[(i, k)], side_right=True, upper=True)
                panel[i] = mine[(i, k)]
            elif op == BCAST_PANEL:
                t = torch.from_numpy(np.ascontiguousarray(panel[i] if rank == root
                                                          else np.zeros((nb, nb))))
                dist.broadcast(t, src=root, group=group[comm])
                panel[i] = np.asfortranarray(t.numpy())
            elif op == UPDATE:
                x = round_to(panel[i], p)
                y = round_to(panel[j], p)
                mine[(i, j)] = port_.gemm(p, p, p, x, y, mine[(i, j)], ta=False, tb=True,
                                          alpha=-1.0, beta=1.0)
            else:
                raise AssertionError(op)
        np.savez(os.path.join(outdir, f"rank{rank}.npz"),
                 keys=np.array(list(mine.keys()), dtype=np.int64).reshape(-1, 2),
                 vals=np.stack(list(mine.values())) if mine else np.zeros((0, nb, nb)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P,Q", [(1, 2), (2, 1), (2, 2), (1, 3)])
def test_distributed_plan_matches_oracle(tmp_path, P, Q):
    n, nb = 256, 32
    world = P * Q
    mp_.spawn(_worker, args=(world, P, Q, _free_port(), n, nb, str(tmp_path)), nprocs=world,
              join=True)
    from oracle.oracle import Port

    A, prec = _problem(n, nb)
    L = Port().tile_chol(n, nb, prec, A)
    nt = n // nb
    seen = set()
    for r in range(world):
        z = np.load(tmp_path / f"rank{r}.npz")
        for (i, j), v in zip(z["keys"], z["vals"]):
            want = L[i * nb:(i + 1) * nb, j * nb:(j + 1) * nb]
            if i == j:
                v = np.tril(v)
            assert np.array_equal(v, want), (r, i, j, np.abs(v - want).max())
            seen.add((int(i), int(j)))
    assert seen == {(i, j) for j in range(nt) for i in range(j, nt)}


def test_schedule_partitions_work():
    """Every tile op of the sequential algorithm runs on exactly one rank, on
    the owner of its output tile; the broadcasts of each row / column
    communicator appear identically (same order, same root) on all of its
    members, so the collectives match up."""
    import paper_2406_02701_b200 as mp

    nt = 9
    for P, Q in [(1, 1), (1, 3), (3, 1), (2, 2), (2, 4), (4, 2)]:
        world = P * Q
        scheds = [mp.dist_schedule(r, P, Q, nt) for r in range(world)]
        ops = {}
        for r, s in enumerate(scheds):
            for op, k, i, j, root, p, comm in s.tolist():
                if op in (POTRF, TRSM, UPDATE):
                    key = (op, k, i, j)
                    assert key not in ops, key
                    ops[key] = r
                    assert mp.dist_owner(i, j, P, Q) == r
        want = set()
        for k in range(nt):
            want.add((POTRF, k, k, k))
            for i in range(k + 1, nt):
                want.add((TRSM, k, i, k))
            for j in range(k + 1, nt):
                for i in range(j, nt):
                    want.add((UPDATE, k, i, j))
        assert set(ops) == want
        # every communicator sees the same collectives in the same order on
        # all its members (row r: ranks r*Q..r*Q+Q-1; column c: c, c+Q, ...)
        for kind, members in ([(ROW, [r * Q + c for c in range(Q)]) for r in range(P)] +
                              [(COL, [r * Q + c for r in range(P)]) for c in range(Q)]):
            seqs = [[tuple(a) for a in scheds[m].tolist() if a[0] in (BCAST_DIAG, BCAST_PANEL) and a[6] == kind]
                    for m in members]
            assert all(q == seqs[0] for q in seqs)
        if world == 1:
            assert not any(a[0] in (BCAST_DIAG, BCAST_PANEL) for a in scheds[0].tolist())


@pytest.mark.parametrize("P,Q", [(2, 2), (2, 4), (4, 2), (1, 4), (3, 3)])
def test_row_column_broadcasts_move_only_needed_tiles(P, Q):
    """SURVEY §8e volume: each panel tile L_ik reaches exactly P + Q - 2 other
    ranks, all in process row i mod P or process column i mod Q; every tile a
    rank's updates read is owned or received; a received tile goes unused only
    at the matrix edge (i - k < Q for a row copy, NT - i < P for a column copy).
    L_kk^-1 reaches exactly the TRSM owners of tile column k."""
    import paper_2406_02701_b200 as mp

    nt = 11
    world = P * Q
    scheds = [mp.dist_schedule(r, P, Q, nt) for r in range(world)]
    own = lambda i, j: mp.dist_owner(i, j, P, Q)
    for k in range(nt - 1):
        for i in range(k + 1, nt):
            got = {}  # rank -> comms it received L_ik on
            for r in range(world):
                for op, kk, ii, jj, root, p, comm in scheds[r].tolist():
                    if op == BCAST_PANEL and kk == k and ii == i and r != root:
                        got.setdefault(r, []).append(comm)
            assert all(len(c) == 1 for c in got.values()), got
            assert len(got) == P + Q - 2, (k, i, got)
            for r, (comm,) in got.items():
                pr, pc = divmod(r, Q)
                assert (comm == ROW and pr == i % P) or (comm == COL and pc == i % Q)
                need_a = any(own(i, j) == r for j in range(k + 1, i + 1))
                need_b = any(own(m, i) == r for m in range(i, nt))
                if not (need_a or need_b):
                    assert (comm == ROW and i - k < Q) or (comm == COL and nt - i < P), (k, i, r)
            for r in range(world):  # every reader holds the tile
                reads = any(own(i, j) == r for j in range(k + 1, i + 1)) or any(own(m, i) == r for m in range(i, nt))
                if reads:
                    assert r == own(i, k) or r in got, (k, i, r)
        diag = {r for r in range(world) for op, kk, *_ in scheds[r].tolist() if op == BCAST_DIAG and kk == k}
        trsm = {own(i, k) for i in range(k + 1, nt)}
        if P > 1:
            assert trsm <= diag and diag == {r for r in range(world) if r % Q == k % Q}
        else:
            assert not diag and trsm == {own(k, k)}


def test_dist_owner_2x2():
    """Rank 3 of a 2 x 2 grid owns the lower tiles with odd row and column."""
    import paper_2406_02701_b200 as mp

    nt = 6
    own = {(i, j) for j in range(nt) for i in range(j, nt) if mp.dist_owner(i, j, 2, 2) == 3}
    assert own == {(i, j) for j in range(1, nt, 2) for i in range(j, nt) if i % 2 == 1}
