"""Data-parallel sharding of one solve over the GPUs of a node.

One process per GPU (torchrun).  Every rank holds the full frame store and
the full problem; rank r owns every world-th directed dense edge and every
world-th frame-pair filter candidate.  The only collectives are the sums of
the per-edge exchange buffers after each dense pass (and of the filter pass
flags once per solve).  Each buffer entry has exactly one owning rank, so the
sum is exact: every rank ends with the bit-identical block system and runs
the same replicated PCG - no per-PCG-iteration communication and no
control-flow divergence between ranks.

Usage:
    comm = ShardComm()                      # after dist.init_process_group
    problem = AlignmentProblem(ids, poses, sets, caches, comm=comm)
    problem.solve(weights, config)
"""

from __future__ import annotations

import numpy as np

# dtype of each exchange buffer (include/sfb.h: sfb_exchange_buffer)
EXCHANGE_DTYPES = {0: "f8", 1: "f8", 2: "u1"}


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

    def __init__(self, group=None):
        import torch.distributed as dist
        self._dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

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
            self._dist.all_reduce(t, op=self._dist.ReduceOp.SUM, group=self.group)
            return
        ptr, nbytes = dp.exchange_buffer(which)
        if nbytes == 0:
            return
        dev = torch.device("cuda", torch.cuda.current_device())
        t = torch.as_tensor(_CudaView(ptr, nbytes, typestr), device=dev)
        # enqueue on the solver's stream so the collective orders with its kernels
        with torch.cuda.stream(torch.cuda.ExternalStream(dp.stream_ptr(), device=dev)):
            self._dist.all_reduce(t, op=self._dist.ReduceOp.SUM, group=self.group)


def owned_edges(n_directed: int, rank: int, world: int) -> np.ndarray:
    """Directed-edge ownership used by libsfb (rebuild_structure): d % world == rank."""
    return np.arange(n_directed)[np.arange(n_directed) % world == rank]
