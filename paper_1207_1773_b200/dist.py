"""Multi-GPU plumbing: one process per GPU.

All multi-GPU work happens inside libeigb200 (comm.cu): the collective
eig_solve_gen / eig_hotpath run the unsharded stages on rank 0, move the
factors by NCCL broadcast (lower triangles only) on a communication stream
overlapped with rank 0's later stages, scatter the tridiagonal eigenvectors by
column slice and back-transform each rank's contiguous columns
[floor(r m / P), floor((r+1) m / P)) (the back-transform acts on columns
independently).  torch.distributed only ships the 128-byte NCCL
unique id from rank 0 to the other ranks, which is all this module does.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from ._binding import Solver, column_slice, unique_id  # noqa: F401  (column_slice re-exported)


def ship_unique_id(group=None, device=None) -> bytes:
    """Rank 0 creates the NCCL unique id (eig_get_unique_id) and broadcasts its
    128 bytes over the torch.distributed group; every rank returns them."""
    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", device) if (backend == "nccl" and device is not None) else (
        torch.device("cuda") if backend == "nccl" else torch.device("cpu"))
    buf = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(unique_id()), dtype=torch.uint8))
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast(buf, src=src, group=group)
    return bytes(buf.cpu().numpy().tobytes())


def collective_solver(device: int, nb: int = 64, q2_group: int = 0, group=None, n_max: int = 0, flags: int = 0,
                      stream=None) -> Solver:
    """A collective Solver handle on every rank of `group` (eig_init with
    {rank, nranks, nccl_id}); must be called by all ranks."""
    uid = ship_unique_id(group, device)
    return Solver(device, nb=nb, q2_group=q2_group, stream=stream, rank=dist.get_rank(group),
                  nranks=dist.get_world_size(group), nccl_id=uid, n_max=n_max, flags=flags)
