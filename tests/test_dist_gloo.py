"""Multi-process (world size 2, gloo, CPU) test of the frame-pair sharding protocol.

The device path (paper_1604_01093_b200.shard + libsfb's _begin/_end calls)
needs GPUs; this test drives the same protocol - ShardComm, ownership of
directed edges / filter candidates (d % world == rank), exchange buffers with
exactly one owner per entry - through a host-memory problem whose per-edge
sums come from the CPU oracle, and checks that every rank ends with the
unsharded result bit-for-bit.
"""

import os
import socket

import numpy as np
import pytest

from golden_io import GoldenScene
from oracle import scanfuse_oracle as O


def _sym_pack(H):
    return np.array([H[r, c] for r in range(6) for c in range(r, 6)])


class HostShardProblem:
    """Host mirror of the sharded device problem (exchange buffers 0 and 2)."""

    def __init__(self, scene, rank=0, world=1):
        self.s = scene
        self.poses = {f: O.pose_of(p) for f, p in scene.init.items()}
        self.rank, self.world = rank, world
        self.flags = np.zeros(0, dtype=np.uint8)
        self.edge_out = np.zeros((0, 32))

    def exchange_array(self, which):
        return {0: self.edge_out.reshape(-1), 2: self.flags}[which]

    def build_dense_edges(self, exchange):
        ids = self.s.ids
        cand = [(a, b) for a in range(len(ids)) for b in range(a + 1, len(ids))
                if O.view_angle_deg(self.poses[ids[a]], self.poses[ids[b]]) < 60.0]
        self.flags = np.zeros(len(cand), dtype=np.uint8)
        for c, (a, b) in enumerate(cand):
            if c % self.world != self.rank:
                continue
            i, j = ids[a], ids[b]
            ci, cj = self.s.caches[i], self.s.caches[j]
            if (O.frustum_overlap(ci, self.poses[i], cj, self.poses[j]) > 0.0
                    and O.frustum_overlap(cj, self.poses[j], ci, self.poses[i]) > 0.0):
                self.flags[c] = 1
        if exchange is not None:
            exchange(self, 2)
        self.edges = [(ids[a], ids[b]) for c, (a, b) in enumerate(cand) if self.flags[c]]
        return self.edges

    def linearize(self, w_dense, exchange):
        self.edge_out = np.zeros((len(self.edges), 32))
        for d, (i, j) in enumerate(self.edges):
            if d % self.world != self.rank:
                continue
            ci, cj = self.s.caches[i], self.s.caches[j]
            pts, ref = O.assoc_photo(self.poses, i, j, ci, cj)
            res, J = O.photo_lin(self.poses, i, j, pts, ref, cj)
            Jr, rr = J.reshape(-1, 6), res.reshape(-1)
            gp, gn, gt = O.assoc_geo(self.poses, i, j, ci, cj)
            r2, J2 = O.geo_lin(self.poses, i, j, gp, gn, gt)
            sp, sg = w_dense * self.s.weights["photo"], w_dense * self.s.weights["geo"]
            H = sp * (Jr.T @ Jr) + sg * (J2.T @ J2)
            self.edge_out[d, :21] = _sym_pack(H)
            self.edge_out[d, 21:27] = sp * (Jr.T @ rr) + sg * (J2.T @ r2)
            self.edge_out[d, 27] = float(np.sum(rr ** 2))
            self.edge_out[d, 28] = float(np.sum(r2 ** 2))
        if exchange is not None:
            exchange(self, 0)
        return self.edge_out


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1604_01093_b200.shard import ShardComm
        comm = ShardComm()
        scene = GoldenScene("cfg2")
        hp = HostShardProblem(scene, comm.rank, comm.world)
        edges = hp.build_dense_edges(comm)
        eo = hp.linearize(1.0, comm)
        out_q.put((rank, edges, eo.copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_protocol_matches_unsharded():
    import torch.multiprocessing as mp
    scene = GoldenScene("cfg2")
    ref = HostShardProblem(scene)
    ref_edges = ref.build_dense_edges(None)
    assert np.array_equal(np.array(ref_edges), scene.g["edges"])
    ref_eo = ref.linearize(1.0, None)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=280) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, edges, eo in results:
        assert edges == ref_edges                   # identical edge list on every rank
        assert np.array_equal(eo, ref_eo)           # per-edge sums bit-identical
    # the owner split really divided the work
    assert all(np.any(ref_eo[d::world]) for d in range(world))


def test_ownership_partition():
    from paper_1604_01093_b200.shard import owned_edges
    n, world = 103, 4
    parts = [owned_edges(n, r, world) for r in range(world)]
    assert sorted(np.concatenate(parts).tolist()) == list(range(n))


# ---------------------------------------------------------------------------
# Sharded-PCG protocol (ShardComm(pcg="sharded")): partial
# systems (own edges; the sparse sets on rank 0), one all-reduce of
# [g | diag] per linearisation and one of A.p per PCG iteration.


def _partial_system(scene, edge_out, edges, rank, world, with_sparse):
    """Dense n_vars^2 partial normal equations of one rank (host mirror of
    k_assemble over the rank's own directed edges, solver.py:615-628)."""
    ids = scene.ids
    var = {f: k - 1 for k, f in enumerate(ids)}
    nv = 6 * (len(ids) - 1)
    A = np.zeros((nv, nv))
    g = np.zeros(nv)
    for d, (i, j) in enumerate(edges):
        if d % world != rank:
            continue
        e = edge_out[d]
        H = np.zeros((6, 6))
        k = 0
        for r in range(6):
            for c in range(r, 6):
                H[r, c] = H[c, r] = e[k]
                k += 1
        ge = e[21:27]
        vi, vj = var[i], var[j]
        if vi >= 0:
            A[6 * vi:6 * vi + 6, 6 * vi:6 * vi + 6] += H
            g[6 * vi:6 * vi + 6] += ge
        if vj >= 0:
            A[6 * vj:6 * vj + 6, 6 * vj:6 * vj + 6] += H
            g[6 * vj:6 * vj + 6] -= ge
        if vi >= 0 and vj >= 0:
            A[6 * vi:6 * vi + 6, 6 * vj:6 * vj + 6] -= H
            A[6 * vj:6 * vj + 6, 6 * vi:6 * vi + 6] -= H
    if with_sparse:
        P = O.Problem(ids, {f: O.pose_of(p) for f, p in scene.init.items()}, scene.corr_sets, None)
        S_, _, _ = P.linearize(O.DEFAULT_W, 0.0, O.DEFAULT_CFG)
        S_.dense = np.zeros((nv, nv))
        A += np.stack([S_.apply(col) for col in np.eye(nv)], axis=1)
        g += S_.gradient
    return A, g


def pcg_sharded_host(A_r, g_r, allreduce, max_it=50, tol=1e-6, restart=20):
    """pcg_solve's recurrence (solver.py:463-508) over a partial system: the
    gradient / diagonal once and A.p every iteration are all-reduced."""
    gd = np.concatenate([g_r, np.diag(A_r).copy()])
    allreduce(gd)
    n = g_r.shape[0]
    b, diag = -gd[:n], gd[n:]
    inv = 1.0 / np.maximum(diag, 1e-12)
    x = np.zeros(n)
    r = b.copy()
    z = inv * r
    p = z.copy()
    rz = float(r @ z)
    nb = float(np.sqrt(b @ b))
    it, rel = 0, 1.0
    for k in range(1, max_it + 1):
        it = k
        q = A_r @ p
        allreduce(q)
        pAp = float(p @ q)
        if pAp <= 0.0:
            break
        alpha = rz / pAp
        x = x + alpha * p
        if k % restart == 0:
            q2 = A_r @ x
            allreduce(q2)
            r = b - q2
        else:
            r = r - alpha * q
        z = inv * r
        rel = float(np.sqrt(r @ r)) / nb
        if rel < tol:
            break
        rzn = float(r @ z)
        p = z + (rzn / rz) * p
        rz = rzn
    return x, it, rel


def _pcg_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1604_01093_b200.shard import ShardComm
        comm = ShardComm(pcg="sharded")
        scene = GoldenScene("cfg2")
        hp = HostShardProblem(scene, comm.rank, comm.world)
        edges = hp.build_dense_edges(comm)
        hp.edge_out = np.zeros((len(edges), 32))
        eo = hp.linearize(1.0, None)  # own edges only: no exchange of the per-edge sums
        A_r, g_r = _partial_system(scene, eo, edges, rank, world, with_sparse=rank == 0)
        x, it, rel = pcg_sharded_host(A_r, g_r, comm.pcg_allreduce(hp))
        out_q.put((rank, x, it, rel, int(np.count_nonzero(A_r))))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_pcg_protocol():
    import torch.multiprocessing as mp
    scene = GoldenScene("cfg2")
    full = HostShardProblem(scene)
    edges = full.build_dense_edges(None)
    eo = full.linearize(1.0, None)
    A, g = _partial_system(scene, eo, edges, 0, 1, with_sparse=True)
    x_ref, it_ref, rel_ref = pcg_sharded_host(A, g, lambda v: None)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pcg_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=280) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, x0, it0, rel0, nz0), (_, x1, it1, rel1, nz1) = res
    assert np.array_equal(x0, x1) and it0 == it1 and rel0 == rel1  # identical on every rank
    assert nz0 > 0 and nz1 > 0 and nz0 != nz1                       # really partial systems
    assert it0 == it_ref
    assert np.linalg.norm(x0 - x_ref) <= 1e-9 * np.linalg.norm(x_ref)
