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


def _worker(rank, world, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SFB_DEVICE="0")
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1604_01093_b200.shard import ShardComm
        q.put((rank, _solve(name, ShardComm())))
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_sharded_solve_bit_identical(name):
    import torch.multiprocessing as mp
    R1, t1, recs1, edges1 = _solve(name)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
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
