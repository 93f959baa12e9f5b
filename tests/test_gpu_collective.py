"""The collective (multi-GPU) code path of the C ABI on ONE GPU (marker: gpu).

A handle created with an NCCL id and nranks = 1 runs the whole collective
protocol of comm.cu — packing of the lower triangles, ncclBroadcast of L / V1
/ T1 / V2 / tau2 / w, the grouped send/recv scatter of the eigenvector
slices, the status broadcasts, the per-rank back-transform — over a
one-rank communicator.  Its results must be bitwise those of the
single-GPU handle (same kernels on the same data); nothing here runs two
ranks on one GPU.  The N > 1 runs are the driver's scaling runs
(bench.py --gpus N)."""
import numpy as np
import pytest
import torch

import synth

gpu = pytest.mark.gpu


def _dev(x):
    from paper_1207_1773_b200 import colmajor
    return colmajor(x, torch.device("cuda:0"))


def _coll(nb=64, g=0, flags=0):
    from paper_1207_1773_b200 import Solver, unique_id
    return Solver(0, nb=nb, q2_group=g, rank=0, nranks=1, nccl_id=unique_id(), flags=flags)


@gpu
@pytest.mark.parametrize("n,nb,kw", [(300, 16, {}), (777, 64, {"fraction": 0.25}), (1000, 64, {"il": 101, "iu": 400})])
def test_collective_solve_gen_p1_bitwise_equals_single(n, nb, kw):
    from paper_1207_1773_b200 import EIG_GATHER_Z, Solver
    A, B = synth.pencil_rand(n, seed=n, kappa=1e2)
    s1 = Solver(0, nb=nb)
    w1, Z1 = s1.solve_gen(_dev(np.tril(A)), _dev(np.tril(B)), **kw)
    for flags in (0, EIG_GATHER_Z):
        sc = _coll(nb=nb, flags=flags)
        w, Z, st = sc.solve_gen(_dev(np.tril(A)), _dev(np.tril(B)), stats=True, **kw)
        torch.cuda.synchronize()
        assert torch.equal(w, w1) and torch.equal(Z, Z1)
        m = Z1.shape[1]
        assert st["m"] == m and st["cols"] == (0, m) and st["nranks"] == 1
        # factors really went through NCCL: lower triangles of L and A, T1, V2, tau2, w, status words
        assert st["bytes_comm"] >= 2 * n * (n + 1) // 2 * 16 + n * 8
        for k in ("potrf", "hegst", "he2hb", "hb2st", "stedc", "q2", "q1", "trsm", "bt", "total"):
            assert st["seconds"][k] > 0, k
        assert st["seconds"]["bt"] <= st["seconds"]["total"]
        assert st["flops"]["bt"] == pytest.approx(20.0 * n * n * m)
        sc.close()


@gpu
def test_collective_solve_gen_not_pd_error_on_every_rank():
    from paper_1207_1773_b200 import EigError
    A = synth.rand_hermitian(100, 1)
    B = synth.hpd_with_condition(100, 10.0, 1)
    B[40, 40] = -1.0
    sc = _coll()
    with pytest.raises(EigError, match="rc=141"):
        sc.solve_gen(_dev(np.tril(A)), _dev(np.tril(B)))


@gpu
@pytest.mark.parametrize("n,nb,g,m", [(600, 64, 32, 333), (513, 32, 16, 100)])
def test_collective_hotpath_p1_bitwise_equals_single(n, nb, g, m):
    from paper_1207_1773_b200 import Solver
    A = synth.rand_hermitian(n, 2)
    V2, tau2 = synth.synthetic_v2(n, nb, 2)
    L = synth.unit_lower(n, 2)
    Z = synth.real_orthonormalish(n, m, 2)
    dV2, dt2 = torch.from_numpy(V2).cuda(), torch.from_numpy(tau2).cuda()
    s1 = Solver(0, nb=nb, q2_group=g)
    E1, tau1, T1 = s1.hotpath(_dev(A), dV2, dt2, _dev(L), _dev(Z))
    sc = _coll(nb=nb, g=g)
    E, _, _ = sc.hotpath(_dev(A), dV2, dt2, _dev(L), _dev(Z))
    torch.cuda.synchronize()
    assert torch.equal(E, E1)
    st = sc.last_stats()
    assert st["seconds"]["he2hb"] > 0 and st["seconds"]["bt"] > 0
    assert st["bytes_comm"] >= 2 * n * (n + 1) // 2 * 16


@gpu
def test_collective_host_buffers_not_available():
    from paper_1207_1773_b200 import EIG_HOST_BUFFERS, EigError, lib
    import ctypes as C
    sc = _coll()
    rc = lib().eig_hotpath(sc.h, 10, None, 10, None, None, None, None, None, 10, None, 10, None, 10, 1,
                           EIG_HOST_BUFFERS)
    assert rc == -1005


@gpu
@pytest.mark.parametrize("n,nb", [(300, 16), (1000, 64)])
def test_collective_solve_gen_distributed_he2hb_p1(n, nb):
    """EIG_DIST_HE2HB on a one-rank communicator: the whole NEXT-4 path over
    NCCL (block scatter, per-step V/T broadcasts and W allreduce, band gather)
    gives the same eigenpairs as the single-GPU solver within the gates."""
    import math
    from paper_1207_1773_b200 import EIG_DIST_HE2HB, Solver
    A, B = synth.pencil_rand(n, seed=n + 5, kappa=1e2)
    w1, Z1 = Solver(0, nb=nb).solve_gen(_dev(np.tril(A)), _dev(np.tril(B)))
    sc = _coll(nb=nb, flags=EIG_DIST_HE2HB)
    w, Z, st = sc.solve_gen(_dev(np.tril(A)), _dev(np.tril(B)), stats=True)
    torch.cuda.synchronize()
    w, w1 = w.cpu().numpy(), w1.cpu().numpy()
    assert np.max(np.abs(w - w1)) / np.max(np.abs(w1)) < 1e-12
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    R = Ad @ Z - (Bd @ Z) * torch.from_numpy(w).cuda()[None, :]
    one = lambda M: torch.linalg.matrix_norm(M, ord=1).item()  # noqa: E731
    assert one(R) / (n * one(Ad) * one(Z)) < 1e-14
    assert one(Z.conj().T @ Bd @ Z - torch.eye(n, dtype=Z.dtype, device=Z.device)) / n < 1e-14
    assert st["seconds"]["he2hb"] > 0 and st["bytes_comm"] > 0


@gpu
@pytest.mark.parametrize("n,nb,g,m", [(600, 64, 32, 333), (513, 32, 16, 100)])
def test_collective_hotpath_distributed_he2hb_p1(n, nb, g, m):
    """EIG_DIST_HE2HB in the collective hot path (one-rank communicator): E
    agrees with the single-GPU hot path to the parity tolerance (the
    distributed reduction sums W by ranks and updates full columns, so it is
    not bitwise the one-GPU reduction)."""
    from paper_1207_1773_b200 import EIG_DIST_HE2HB, Solver
    A = synth.rand_hermitian(n, 4)
    V2, tau2 = synth.synthetic_v2(n, nb, 4)
    L = synth.unit_lower(n, 4)
    Z = synth.real_orthonormalish(n, m, 4)
    dV2, dt2 = torch.from_numpy(V2).cuda(), torch.from_numpy(tau2).cuda()
    E1, _, _ = Solver(0, nb=nb, q2_group=g).hotpath(_dev(A), dV2, dt2, _dev(L), _dev(Z))
    sc = _coll(nb=nb, g=g, flags=EIG_DIST_HE2HB)
    E, _, _ = sc.hotpath(_dev(A), dV2, dt2, _dev(L), _dev(Z))
    torch.cuda.synchronize()
    err = (E - E1).abs().max().item() / E1.abs().max().item()
    assert err < 1e-11, err
    st = sc.last_stats()
    assert st["seconds"]["he2hb"] > 0 and st["seconds"]["bt"] > 0
