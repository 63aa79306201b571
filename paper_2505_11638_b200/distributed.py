"""Point-sharded multi-GPU execution.

One process per GPU.  Collocation points are split into contiguous interior
and boundary ranges, balanced by channel cost (an interior point carries d+2
Taylor channels, a boundary point one).  theta, v, Omega and every p-vector
are replicated; the library all-reduces (NCCL, on the compute stream, inside
the C-ABI calls) the only cross-shard quantities:

  matvec  J^T(w o Jv)   -> ncclAllReduce(sum, p)
  sketch  Y = G Omega   -> ncclAllReduce(sum, p x ell)
  loss / candidate loss -> ncclAllReduce(sum, 1)
  gradient              -> ncclAllReduce(sum, p)

PCG vector work and the ell x ell factorizations are replicated and therefore
bitwise identical on every rank.  The NCCL unique id is exchanged through
torch.distributed (plumbing only).
"""

from __future__ import annotations

import ctypes

from . import _lib


def shard_range(n, rank, nranks):
    """Contiguous [lo, hi) of n items for rank (first n % nranks ranks get one extra)."""
    base, extra = divmod(n, nranks)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def shard_slices(n_int, n_bnd, channels, rank, nranks):
    """Interior and boundary slices of one rank.

    Interior points (cost ``channels`` each) and boundary points (cost 1) are
    both split contiguously and evenly, so every rank carries the same
    channel-point count to within one point of each kind."""
    if nranks < 1 or not 0 <= rank < nranks:
        raise ValueError("bad rank / world size")
    li, hi = shard_range(n_int, rank, nranks)
    lb, hb = shard_range(n_bnd, rank, nranks)
    return slice(li, hi), slice(lb, hb)


def shard_cost(n_int, n_bnd, channels, rank, nranks):
    si, sb = shard_slices(n_int, n_bnd, channels, rank, nranks)
    return (si.stop - si.start) * channels + (sb.stop - sb.start)


class NcclComm:
    """Binds libngd contexts to NCCL communicators created from a torch.distributed
    process group.  Every bound context gets its own communicator: rank 0 makes a
    fresh unique id per ``bind`` and broadcasts it (all ranks bind in the same order)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.group = group
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)

    def _unique_id(self):
        import torch.distributed as dist

        uid = bytes(128)
        if self.rank == 0:
            buf = (ctypes.c_char * 128)()
            _lib.check(_lib.load().ngd_nccl_unique_id(buf))
            uid = bytes(buf.raw)
        obj = [uid]
        dist.broadcast_object_list(obj, src=0, group=self.group)
        return obj[0]

    def bind(self, ctx):
        ctx.call("ngd_ctx_set_comm", self._unique_id(), self.rank, self.nranks)


def attach(problem, comm):
    """Make ``problem`` compute on this rank's shard with all-reduced results."""
    problem.shard = (comm.rank, comm.nranks)
    problem.comm = comm
    problem._ctxs = []
    return problem
