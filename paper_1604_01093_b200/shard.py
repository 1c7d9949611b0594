"""Data-parallel sharding of one solve over the GPUs of a node.

One process per GPU (torchrun).  Every rank holds the full frame store and
the full problem; rank r owns every world-th directed dense edge and every
world-th frame-pair filter candidate.  Two PCG modes:

* ``pcg="replicated"`` (default): the per-edge sums of each dense pass are
  all-gathered (each row has exactly one owning rank, which sends only its
  rows: an exact copy, half the bytes of an all-reduce), every rank
  assembles the bit-identical block system and runs the same PCG - no
  per-PCG-iteration communication.
* ``pcg="sharded"``: each rank keeps only its partial system
  (its edges; the correspondence sets on rank 0); one all-reduce of
  [gradient | Jacobi diagonal | dense energies] per linearisation and one of
  the partial A.p per PCG iteration; the PCG scalars are then computed
  redundantly on identical bits.  The summation order of the partial systems
  differs from a single GPU's, so results agree to rounding, not bitwise.

Usage:
    comm = ShardComm()                      # after dist.init_process_group
    problem = AlignmentProblem(ids, poses, sets, caches, comm=comm)
    problem.solve(weights, config)
"""

from __future__ import annotations

import numpy as np

# dtype of each exchange buffer (include/sfb.h: sfb_exchange_buffer)
EXCHANGE_DTYPES = {0: "f8", 1: "f8", 2: "u1", 3: "f8"}
# buffers 0-2 hold rows owned by exactly one rank (row d by rank d % world):
# they are all-GATHERED (each rank sends only its rows); buffer 3 (the
# sharded-PCG partial system) is a true sum
EXCHANGE_ROW = {0: 32, 1: 2, 2: 1}
PCG_MODES = ("replicated", "sharded")


class _CudaView:
    """__cuda_array_interface__ over a device pointer owned by libsfb."""

    def __init__(self, ptr: int, nbytes: int, typestr: str):
        item = int(typestr[-1])
        self.__cuda_array_interface__ = {
            "shape": (nbytes // item,), "typestr": "<" + typestr, "data": (ptr, False),
            "version": 3, "strides": None, "stream": None,
        }


class ShardComm:
    """Sums exchange buffers across the ranks of a torch.distributed group."""

    def __init__(self, group=None, pcg: str = "replicated", p2p: bool = False):
        import torch.distributed as dist
        if pcg not in PCG_MODES:
            raise ValueError(f"pcg must be one of {PCG_MODES}")
        self._dist = dist
        self.group = group
        self.pcg = pcg
        # replicated mode: the per-edge sums go peer-to-peer from the edge
        # reduction kernel into every rank's buffer (CUDA IPC, one node)
        self.p2p = bool(p2p) and pcg == "replicated"
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._p2p_handles = {}

    def p2p_setup(self, dp) -> None:
        """Exchange and map the IPC handles of every rank's per-edge buffer and
        flags (again whenever a rank's buffer was reallocated)."""
        mine = (dp.ipc_export(0), dp.ipc_export(1))
        allh = [None] * self.world
        self._dist.all_gather_object(allh, mine, group=self.group)
        key = id(dp)
        for which in (0, 1):
            hs = [h[which] for h in allh]
            if self._p2p_handles.get((key, which)) != hs:
                dp.ipc_attach(which, hs)
                self._p2p_handles[(key, which)] = hs
        dp.set_p2p(True)

    @property
    def active(self) -> bool:
        return self.world > 1

    def __call__(self, dp, which: int) -> None:
        import torch
        typestr = EXCHANGE_DTYPES[which]
        if hasattr(dp, "exchange_array"):  # host-memory problem (CPU / gloo)
            arr = dp.exchange_array(which)
            if arr.size == 0:
                return
            t = torch.from_numpy(arr)
            if which in EXCHANGE_ROW:
                self._gather_owned(t, EXCHANGE_ROW[which])
            else:
                self._dist.all_reduce(t, op=self._dist.ReduceOp.SUM, group=self.group)
            return
        ptr, nbytes = dp.exchange_buffer(which)
        if nbytes == 0:
            return
        if which not in EXCHANGE_ROW:
            self.allreduce_device(ptr, nbytes, typestr, dp.stream_ptr())
            return
        dev = torch.device("cuda", torch.cuda.current_device())
        t = torch.as_tensor(_CudaView(ptr, nbytes, typestr), device=dev)
        with torch.cuda.stream(torch.cuda.ExternalStream(dp.stream_ptr(), device=dev)):
            self._gather_owned(t, EXCHANGE_ROW[which])

    def _gather_owned(self, t, row_len: int) -> None:
        """In place: rows d of `t` (row_len elements each) are valid on rank
        d % world only; after the call every rank holds all of them.  One
        all-gather of each rank's rows (half the bytes of the equivalent
        all-reduce, and an exact copy of the owner's values)."""
        import torch
        rows = t.view(-1, row_len)
        n, world, rank = rows.shape[0], self.world, self.rank
        per = (n + world - 1) // world
        send = torch.zeros((per, row_len), dtype=t.dtype, device=t.device)
        mine = rows[rank::world]
        send[:mine.shape[0]] = mine
        recv = [torch.empty_like(send) for _ in range(world)]
        self._dist.all_gather(recv, send, group=self.group)
        for r in range(world):
            cnt = rows[r::world].shape[0]
            rows[r::world] = recv[r][:cnt]

    def allreduce_device(self, ptr: int, nbytes: int, typestr: str, stream: int) -> None:
        """In-place sum of a device buffer across ranks, ordered on `stream`."""
        import torch
        dev = torch.device("cuda", torch.cuda.current_device())
        t = torch.as_tensor(_CudaView(ptr, nbytes, typestr), device=dev)
        with torch.cuda.stream(torch.cuda.ExternalStream(stream, device=dev)):
            self._dist.all_reduce(t, op=self._dist.ReduceOp.SUM, group=self.group)

    def pcg_allreduce(self, dp):
        """The per-PCG-iteration collective of the sharded mode: A.p (n doubles)."""
        if hasattr(dp, "exchange_array"):  # host-memory problem (CPU / gloo): numpy in place
            import torch

            def host(arr) -> None:
                self._dist.all_reduce(torch.from_numpy(arr), op=self._dist.ReduceOp.SUM,
                                      group=self.group)
            return host

        def fn(ptr: int, n: int, stream: int) -> None:
            self.allreduce_device(ptr, 8 * n, "f8", stream)
        return fn


def owned_edges(n_directed: int, rank: int, world: int) -> np.ndarray:
    """Directed-edge ownership used by libsfb (rebuild_structure): d % world == rank."""
    return np.arange(n_directed)[np.arange(n_directed) % world == rank]
