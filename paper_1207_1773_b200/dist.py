"""Multi-GPU back-transform driver: one process per GPU,
eigenvector columns sharded in contiguous slices, he2hb on rank 0.

Every back-transform step acts on the columns of Z independently (S:L469,
"column-block parallelism"), so rank r owns columns
[floor(r m / P), floor((r+1) m / P)) and the only exchange is the broadcast of
the read-only factors from rank 0 (he2hb's A = band + V1 and T1, the bulge
chase reflectors V2/tau2, and L) over NCCL (NVLink / NVSwitch).  E stays
distributed (optionally gathered).  The compute is the single-GPU C-ABI path
(`Solver`); this module only does plumbing with torch.distributed.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def column_slice(m: int, rank: int, world: int):
    """Contiguous, balanced slice [lo, hi) of m columns owned by `rank`."""
    return (m * rank) // world, (m * (rank + 1)) // world


def _dense(t):
    """A contiguous alias of t (same storage): the column-major matrices of the
    C ABI are transposed views, which NCCL collectives reject as
    non-contiguous; their transpose is the contiguous row-major alias."""
    if t.is_contiguous():
        return t
    if t.dim() == 2 and t.t().is_contiguous():
        return t.t()
    raise ValueError("broadcast needs a dense (row- or column-major) tensor")


def broadcast_factors(tensors, src: int = 0, group=None):
    """Broadcast the read-only factors from `src` (in place, list order).
    One collective per tensor; NCCL pipelines them on its stream."""
    for t in tensors:
        dist.broadcast(_dense(t), src=src, group=group)


def hotpath_sharded(solver, A, tau1, T1, V2, tau2, L, Z_slice, E_slice, group=None):
    """One pass of the hot path with the back-transform sharded by columns.

    rank 0: he2hb(A) (a1..a5).  All ranks: receive A (band + V1), T1, V2, tau2,
    L from rank 0, then E_slice = L^-H Q1 Q2 complex(Z_slice) (a6..a8).
    `solver` is a paper_1207_1773_b200.Solver (or any object with the same
    methods, e.g. a CPU stand-in in the gloo tests).  Returns E_slice."""
    rank = dist.get_rank(group)
    if rank == 0:
        tau1_, T1_ = solver.he2hb(A)
        tau1.copy_(tau1_)
        T1.copy_(T1_)
    broadcast_factors([A, T1, V2, tau2, L], src=0, group=group)
    solver.apply_q2(V2, tau2, E_slice, Z=Z_slice)
    solver.apply_q1(A, T1, E_slice)
    solver.trsm_lh(L, E_slice)
    return E_slice


def solve_gen_sharded(solver, A, B, nb: int, group=None):
    """Algorithm 1 with the back-transform sharded by eigenvector columns
    (SURVEY.md §8(e), CS2): rank 0 runs potrf, hegst, he2hb, hb2st and stedc;
    A (band + V1), T1, V2/tau2, L (in B), w and the tridiagonal eigenvectors
    Z' are broadcast; every rank forms E = L^-H Q1 Q2 Z'[:, slice] for its
    contiguous column slice.  A, B (n x n column-major) must exist on every
    rank (contents only matter on rank 0).  Returns (w [n], E_slice, (lo, hi))."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    n = A.shape[0]
    dev = A.device
    K = 0 if n <= nb else (n - nb - 1) // nb + 1
    slots = 0
    j = 0
    while 1 + j * nb <= n - 1:
        slots += n - 1 - j * nb
        j += 1
    if rank == 0:
        info = solver.potrf(B)
        if info:
            raise RuntimeError(f"B not positive definite (info {info})")
        solver.hegst(A, B)
        tau1, T1 = solver.he2hb(A)
        d, e, V2, tau2 = solver.hb2st(A)
        w, Zr = solver.stedc(d, e)
        T1 = T1.contiguous()
        V2 = V2.contiguous()
        tau2 = tau2.contiguous()
        w = w.contiguous()
    else:
        T1 = torch.zeros(max(K * nb * nb, 1), dtype=torch.complex128, device=dev)
        V2 = torch.zeros((slots, nb), dtype=torch.complex128, device=dev)
        tau2 = torch.zeros(slots, dtype=torch.complex128, device=dev)
        w = torch.zeros(n, dtype=torch.float64, device=dev)
        Zr = torch.zeros((n, n), dtype=torch.float64, device=dev).t()
    broadcast_factors([A, T1, V2, tau2, B, w, Zr], src=0, group=group)
    lo, hi = column_slice(n, rank, world)
    E = torch.empty((hi - lo, n), dtype=torch.complex128, device=dev).t()
    solver.apply_q2(V2, tau2, E, Z=Zr[:, lo:hi])
    solver.apply_q1(A, T1, E)
    solver.trsm_lh(B, E)
    return w, E, (lo, hi)


def gather_columns(E_slice: torch.Tensor, m: int, group=None):
    """Gather the column slices to every rank (column-major n x m result)."""
    world = dist.get_world_size(group)
    n = E_slice.shape[0]
    parts = []
    for r in range(world):
        lo, hi = column_slice(m, r, world)
        parts.append(torch.empty((hi - lo, n), dtype=E_slice.dtype, device=E_slice.device))
    mine = E_slice.t().contiguous()
    # all_gather needs equal sizes: pad to the largest slice
    mx = max(p.shape[0] for p in parts)
    pad = torch.zeros((mx, n), dtype=E_slice.dtype, device=E_slice.device)
    pad[: mine.shape[0]] = mine
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    cols = [bufs[r][: parts[r].shape[0]] for r in range(world)]
    return torch.cat(cols, dim=0).t()
