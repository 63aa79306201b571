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


def shard_range(n, rank, nranks, block=1):
    """Contiguous [lo, hi) of n items for rank, in whole blocks of ``block`` items (the first
    ranks get one extra block; the last rank takes the ragged tail)."""
    nblk = -(-n // block)
    base, extra = divmod(nblk, nranks)
    lo = min(n, (rank * base + min(rank, extra)) * block)
    hi = min(n, lo + (base + (1 if rank < extra else 0)) * block)
    return lo, hi


def shard_slices(n_int, n_bnd, rank, nranks, block=16):
    """Interior and boundary slices of one rank.

    Both point kinds are split contiguously into whole 16-point blocks (the
    kernels' point-block granularity, csrc/ngd_common.cuh: no padded point
    blocks inside a shard), evenly per kind, so every rank carries the same
    channel-point count -- interior points cost d+2 Taylor channels, boundary
    points one -- to within one block of each kind (``shard_cost``)."""
    if nranks < 1 or not 0 <= rank < nranks:
        raise ValueError("bad rank / world size")
    if -(-n_int // block) < nranks and -(-n_bnd // block) < nranks:
        block = 1  # too few blocks for every rank to get one: split point by point
    li, hi = shard_range(n_int, rank, nranks, block)
    lb, hb = shard_range(n_bnd, rank, nranks, block)
    return slice(li, hi), slice(lb, hb)


def shard_cost(n_int, n_bnd, channels, rank, nranks):
    """Channel-points of a rank's shard (interior points carry ``channels`` channels)."""
    si, sb = shard_slices(n_int, n_bnd, rank, nranks)
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
