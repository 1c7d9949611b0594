"""GPU test of the sharded solve: two ranks (processes) share one GPU and sum
their exchange buffers with gloo (NCCL refuses two ranks per device; the
protocol and the kernels are the same).  The sharded solve must reproduce the
single-process solve bit-for-bit: every exchange entry has one owner."""

import os
import socket

import numpy as np
import pytest

from golden_io import GoldenScene

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _solve(name, comm=None):
    from paper_1604_01093_b200 import solver as S
    sc = GoldenScene(name)
    p = S.AlignmentProblem(sc.ids, sc.init, sc.corr_sets, sc.caches, comm=comm)
    st = p.solve(sc.weights_obj(S), sc.config_obj(S), sc.max_iterations)
    R = np.stack([np.asarray(p.poses[f].rotation) for f in sc.ids])
    t = np.stack([np.asarray(p.poses[f].translation) for f in sc.ids])
    recs = [(r.energy_before, r.energy_after, r.pcg_iterations, r.accepted) for r in st.iterations]
    return R, t, recs, list(p.dense_edges)


def _worker(rank, world, port, name, q, p2p=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SFB_DEVICE="0")
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1604_01093_b200.shard import ShardComm
        q.put((rank, _solve(name, ShardComm(p2p=p2p))))
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("name,p2p", [("cfg2", False), ("cfg3", False), ("cfg2", True), ("cfg3", True)])
def test_sharded_solve_bit_identical(name, p2p):
    """p2p: the per-edge sums go from the edge-reduction kernel straight into
    the other rank's buffer (CUDA IPC; here two processes share one GPU)
    followed by the device-side flag barrier - no host collective for them."""
    import torch.multiprocessing as mp
    R1, t1, recs1, edges1 = _solve(name)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q, p2p)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    try:
        for _ in range(world):
            rank, res = q.get(timeout=300)
            out[rank] = res
            assert not isinstance(res, str), f"rank {rank}: {res}"
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for rank in range(world):
        res = out[rank]
        assert not isinstance(res, str), res
        R, t, recs, edges = res
        assert edges == edges1
        assert recs == recs1
        assert np.array_equal(R, R1) and np.array_equal(t, t1)


def _nccl_worker(port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SFB_DEVICE="0")
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_1604_01093_b200 import solver as S
        from paper_1604_01093_b200.shard import ShardComm
        comm = ShardComm()
        sc = GoldenScene(name)
        p = S.AlignmentProblem(sc.ids, sc.init, sc.corr_sets, sc.caches)
        # force the two-phase sharded protocol on a one-rank NCCL group: every
        # exchange buffer goes through ShardComm's device path (the solver's
        # stream as an ExternalStream, the libsfb buffer as a CUDA array view)
        p._xch = comm
        p._problem()
        p._dp.set_shard(0, 1)
        calls = []
        orig = comm.__call__

        def counted(dp, which):
            calls.append(which)
            return orig(dp, which)
        p._xch = counted
        counted.rank, counted.world = 0, 1
        st = p.solve(sc.weights_obj(S), sc.config_obj(S), sc.max_iterations)
        R = np.stack([np.asarray(p.poses[f].rotation) for f in sc.ids])
        t = np.stack([np.asarray(p.poses[f].translation) for f in sc.ids])
        recs = [(r.energy_before, r.energy_after, r.pcg_iterations, r.accepted) for r in st.iterations]
        q.put((R, t, recs, list(p.dense_edges), sorted(set(calls)), dist.get_backend()))
    except Exception as e:
        import traceback
        q.put(traceback.format_exc())
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_nccl_exchange_path_world1():
    """The NCCL branch of ShardComm (device buffers on the solver's stream)
    on a one-rank NCCL group: the sharded protocol must reproduce the plain
    solve bit-for-bit (all_reduce over one rank is the identity)."""
    import torch.multiprocessing as mp
    R1, t1, recs1, edges1 = _solve("cfg2")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    proc = ctx.Process(target=_nccl_worker, args=(_free_port(), "cfg2", q))
    proc.start()
    try:
        res = q.get(timeout=300)
    finally:
        proc.join(timeout=30)
        if proc.is_alive():
            proc.kill()
    assert not isinstance(res, str), res
    R, t, recs, edges, calls, backend = res
    assert backend == "nccl"
    assert set(calls) >= {0, 2}, calls  # per-edge sums and the filter flags were exchanged
    assert edges == edges1 and recs == recs1
    assert np.array_equal(R, R1) and np.array_equal(t, t1)


def _sharded_pcg_worker(rank, world, port, name, precond, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SFB_DEVICE="0")
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1604_01093_b200 import solver as S
        from paper_1604_01093_b200.shard import ShardComm
        sc = GoldenScene(name)
        p = S.AlignmentProblem(sc.ids, sc.init, sc.corr_sets, sc.caches, comm=ShardComm(pcg="sharded"))
        cfg = S.SolverConfig(**{**sc.config, "preconditioner": precond})
        st = p.solve(sc.weights_obj(S), cfg, sc.max_iterations)
        R = np.stack([np.asarray(p.poses[f].rotation) for f in sc.ids])
        t = np.stack([np.asarray(p.poses[f].translation) for f in sc.ids])
        recs = [(r.energy_before, r.energy_after, r.pcg_iterations, r.accepted, r.pcg_residual)
                for r in st.iterations]
        q.put((rank, (R, t, recs, [st.converged, st.aborted])))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("name,precond", [("cfg2", "jacobi"), ("cfg3", "jacobi"), ("cfg3", "block_jacobi")])
def test_sharded_pcg_mode(name, precond):
    """ShardComm(pcg="sharded"): partial systems per rank, one all-reduce of
    A.p per PCG iteration.  Ranks agree bit-for-bit with each other and with
    the single-process solve to rounding (the partial systems are summed in a
    different order): same PCG iteration counts and accept decisions."""
    import torch.multiprocessing as mp
    from paper_1604_01093_b200 import solver as S
    sc = GoldenScene(name)
    p1 = S.AlignmentProblem(sc.ids, sc.init, sc.corr_sets, sc.caches)
    st1 = p1.solve(sc.weights_obj(S), S.SolverConfig(**{**sc.config, "preconditioner": precond}),
                   sc.max_iterations)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_sharded_pcg_worker, args=(r, world, port, name, precond, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    out = {}
    try:
        for _ in range(world):
            rank, res = q.get(timeout=500)
            assert not isinstance(res, str), f"rank {rank}: {res}"
            out[rank] = res
    finally:
        for pr in procs:
            pr.join(timeout=30)
            if pr.is_alive():
                pr.kill()
    R0, t0, recs0, flags0 = out[0]
    R1, t1, recs1, flags1 = out[1]
    assert np.array_equal(R0, R1) and np.array_equal(t0, t1) and recs0 == recs1
    assert flags0 == [st1.converged, st1.aborted]
    assert [(r[2], r[3]) for r in recs0] == [(r.pcg_iterations, r.accepted) for r in st1.iterations]
    for r, ref in zip(recs0, st1.iterations):
        assert r[0] == pytest.approx(ref.energy_before, rel=1e-9)
        assert r[1] == pytest.approx(ref.energy_after, rel=1e-9)
    R = np.stack([np.asarray(p1.poses[f].rotation) for f in sc.ids])
    t = np.stack([np.asarray(p1.poses[f].translation) for f in sc.ids])
    assert np.abs(R0 - R).max() < 1e-8 and np.abs(t0 - t).max() < 1e-8
