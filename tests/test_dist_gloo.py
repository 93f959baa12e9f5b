"""Multi-process (world_size 2, gloo, CPU) test of the column-sharded
back-transform driver paper_1207_1773_b200/dist.py.

The driver's plumbing (column slicing, broadcast of the factors from rank 0,
per-rank back-transform, gather) is exercised with a CPU stand-in solver whose
arithmetic is the oracle's (test-only); the result must be bitwise equal to
the single-process composition, because every back-transform step acts on
columns independently."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

N, NB, M = 70, 8, 11


class OracleSolver:
    """CPU stand-in with the Solver interface (test-only; uses oracle/)."""

    def __init__(self, nb):
        self.nb = nb

    def he2hb(self, A):
        n = A.shape[0]
        A_o, tau = oracle.he2hb(oracle.full_hermitian(A.numpy()), self.nb)
        A.copy_(torch.from_numpy(np.asfortranarray(A_o)).t().contiguous().t())
        K = 0
        while K * self.nb + self.nb < n:
            K += 1
        T = np.zeros((K, self.nb, self.nb), complex)
        for k in range(K):
            r0 = (k + 1) * self.nb
            V = np.tril(A_o[r0:, k * self.nb:(k + 1) * self.nb], -1)
            for j in range(min(self.nb, n - r0)):
                V[j, j] = 1
            T[k] = oracle.larft(V, tau[k * self.nb:(k + 1) * self.nb])
        return torch.from_numpy(tau[:max(K * self.nb, 1)].copy()), torch.from_numpy(
            T.transpose(0, 2, 1).reshape(-1).copy() if K else np.zeros(1, complex))

    def apply_q2(self, V2, tau2, E, Z=None):
        src = Z.numpy().astype(complex) if Z is not None else E.numpy()
        E.copy_(torch.from_numpy(oracle.apply_q2(V2.numpy(), tau2.numpy(), self.nb, src)))

    def apply_q1(self, A, T, E):
        n = A.shape[0]
        K = T.numel() // (self.nb * self.nb)
        Tb = T.numpy()[:K * self.nb * self.nb].reshape(K, self.nb, self.nb)
        tau = np.zeros(max(n, 1), complex)
        for k in range(K):
            tau[k * self.nb:(k + 1) * self.nb] = np.diag(Tb[k])
        E.copy_(torch.from_numpy(oracle.apply_q1(A.numpy(), tau, self.nb, E.numpy())))

    def trsm_lh(self, L, E):
        E.copy_(torch.from_numpy(oracle.backsub_lh(np.tril(L.numpy()), E.numpy())))

    # front end / tridiagonal stages (for the sharded Algorithm 1)
    def potrf(self, B):
        L, info = oracle.potrf(oracle.full_hermitian(B.numpy()))
        B.copy_(_cm(L))
        return info

    def hegst(self, A, L):
        A.copy_(_cm(oracle.std_form(A.numpy(), np.tril(L.numpy()))))

    def hb2st(self, A):
        n = A.shape[0]
        Ao = A.numpy()
        r, c = np.indices((n, n))
        Bl = np.where((r - c >= 0) & (r - c <= self.nb), Ao, 0)
        Band = np.tril(Bl) + np.tril(Bl, -1).conj().T
        Band[np.diag_indices(n)] = Band.diagonal().real
        d, e, V2, tau2 = oracle.hb2st(Band, self.nb)
        return torch.from_numpy(d), torch.from_numpy(e.copy()), torch.from_numpy(V2.copy()), torch.from_numpy(tau2.copy())

    def stedc(self, d, e):
        w, Z, info = oracle.tql2(d.numpy(), e.numpy())
        assert info == 0
        return torch.from_numpy(w), _cm(Z)


def _cm(x):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x).T)).t()


def _inputs():
    A = synth.rand_hermitian(N, 4)
    V2, tau2 = synth.synthetic_v2(N, NB, 4)
    L = synth.unit_lower(N, 4)
    Z = synth.real_orthonormalish(N, M, 4)
    return A, V2, tau2, L, Z


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1207_1773_b200.dist import column_slice, gather_columns, hotpath_sharded
    A, V2, tau2, L, Z = _inputs()
    lo, hi = column_slice(M, rank, world)
    slots = V2.shape[0]
    K = (N - NB - 1) // NB + 1
    if rank == 0:
        tA, tV2, tt2, tL = _cm(A), torch.from_numpy(V2), torch.from_numpy(tau2), _cm(L)
    else:   # other ranks receive everything from rank 0
        tA = torch.zeros((N, N), dtype=torch.complex128).t().contiguous().t()
        tV2 = torch.zeros((slots, NB), dtype=torch.complex128)
        tt2 = torch.zeros(slots, dtype=torch.complex128)
        tL = torch.zeros((N, N), dtype=torch.complex128).t().contiguous().t()
    tau1 = torch.zeros(K * NB, dtype=torch.complex128)
    T1 = torch.zeros(K * NB * NB, dtype=torch.complex128)
    Zs = _cm(Z[:, lo:hi])
    Es = torch.zeros((hi - lo, N), dtype=torch.complex128).t()
    hotpath_sharded(OracleSolver(NB), tA, tau1, T1, tV2, tt2, tL, Zs, Es)
    Eall = gather_columns(Es, M)
    if rank == 0:
        out.put(Eall.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker_gen(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1207_1773_b200.dist import gather_columns, solve_gen_sharded
    A, B = synth.pencil_rand(N, seed=9, kappa=10.0)
    if rank == 0:
        tA, tB = _cm(A), _cm(B)
    else:
        tA = torch.zeros((N, N), dtype=torch.complex128).t().contiguous().t()
        tB = torch.zeros((N, N), dtype=torch.complex128).t().contiguous().t()
    w, Es, _ = solve_gen_sharded(OracleSolver(NB), tA, tB, NB)
    Eall = gather_columns(Es, N)
    if rank == 0:
        out.put((w.numpy().copy(), Eall.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_solve_gen_gloo_world2():
    """Algorithm 1 with the sharded back-transform (2 ranks): the gathered
    eigenvectors satisfy the residual / B-orthogonality gates and equal the
    single-process composition bitwise."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_gen, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    w, E = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    A, B = synth.pencil_rand(N, seed=9, kappa=10.0)
    R = A @ E - (B @ E) * w[None, :]
    assert np.linalg.norm(R, 1) / (N * np.linalg.norm(A, 1) * np.linalg.norm(E, 1)) < 1e-14
    assert np.linalg.norm(E.conj().T @ B @ E - np.eye(N), 1) / N < 1e-14
    # single process, same stand-in solver
    s = OracleSolver(NB)
    tA, tB = _cm(A), _cm(B)
    assert s.potrf(tB) == 0
    s.hegst(tA, tB)
    tau1, T1 = s.he2hb(tA)
    d, e, V2, tau2 = s.hb2st(tA)
    w1, Zr = s.stedc(d, e)
    E1 = torch.zeros((N, N), dtype=torch.complex128).t()
    s.apply_q2(V2, tau2, E1, Z=Zr)
    s.apply_q1(tA, T1, E1)
    s.trsm_lh(tB, E1)
    assert np.array_equal(E, E1.numpy()) and np.array_equal(w, w1.numpy())


def test_column_slices_partition():
    from paper_1207_1773_b200.dist import column_slice
    for m in (1, 7, 10000):
        for P in (1, 2, 4, 8):
            sl = [column_slice(m, r, P) for r in range(P)]
            assert sl[0][0] == 0 and sl[-1][1] == m
            assert all(sl[r][1] == sl[r + 1][0] for r in range(P - 1))
            assert max(b - a for a, b in sl) - min(b - a for a, b in sl) <= 1


def test_sharded_backtransform_gloo_world2_bitwise():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    E_dist = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    A, V2, tau2, L, Z = _inputs()
    A_o, tau_o = oracle.he2hb(A, NB)
    E_ref = oracle.backsub_lh(L, oracle.apply_q1(A_o, tau_o, NB, oracle.apply_q2(V2, tau2, NB, Z.astype(complex))))
    assert np.array_equal(E_dist, E_ref)
