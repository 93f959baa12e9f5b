"""NEXT-4: the 1D block-cyclic distributed he2hb (§6), its arithmetic
checked on one GPU with P virtual ranks (eig_he2hb_sim: per-rank panel /
partial W / allreduce / owned-column update, collectives as device copies and
a fixed-order sum) against the CPU oracle element by element, and against
the single-GPU reduction (marker: gpu).  The NCCL collectives of the real
multi-GPU run are the only part not exercised here."""
import numpy as np
import pytest
import torch

import oracle
import synth

gpu = pytest.mark.gpu
TOL = 1e-11


def _dev(x):
    from paper_1207_1773_b200 import colmajor
    return colmajor(x, torch.device("cuda:0"))


def _rel(a, b):
    return np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.max(np.abs(b)), 1e-300)


@gpu
@pytest.mark.parametrize("n,nb,P", [(300, 32, 1), (300, 32, 2), (517, 64, 3), (256, 16, 4), (640, 64, 8), (97, 8, 5)])
def test_he2hb_distributed_vs_oracle(n, nb, P):
    from paper_1207_1773_b200 import Solver, num_panels
    s = Solver(0, nb=nb)
    A = synth.rand_hermitian(n, 40 + P)
    dA = _dev(A)
    tau, T = s.he2hb_sim(dA, P)
    Ag = dA.cpu().numpy()
    A_o, tau_o = oracle.he2hb(A, nb)
    r, c = np.indices((n, n))
    low = r >= c
    assert _rel(Ag[low], A_o[low]) < TOL * max(1, n / 256)
    K = num_panels(n, nb)
    assert np.max(np.abs(tau.cpu().numpy()[:K * nb] - tau_o[:K * nb])) < TOL * max(1, n / 256)
    # T_k against the oracle's larft on the oracle's V_k
    Tg = T.cpu().numpy()[:K * nb * nb].reshape(K, nb, nb).transpose(0, 2, 1)
    for k in range(K):
        r0 = (k + 1) * nb
        V = np.tril(A_o[r0:, k * nb:(k + 1) * nb], -1)
        for j in range(min(nb, n - r0)):
            V[j, j] = 1
        assert _rel(Tg[k], oracle.larft(V, tau_o[k * nb:(k + 1) * nb])) < 1e-10


@gpu
def test_he2hb_distributed_matches_single_gpu_and_back_transform():
    """P = 4 virtual ranks at n = 1000: the reduction agrees with the
    single-GPU he2hb, and the back-transform on its output reproduces the
    oracle's (the V1 / T1 every rank keeps are what the sharded BT uses)."""
    from paper_1207_1773_b200 import EIG_SKIP_HE2HB, Solver
    n, nb, m = 1000, 64, 64
    s = Solver(0, nb=nb, q2_group=32)
    A = synth.rand_hermitian(n, 7)
    d1, d2 = _dev(A), _dev(A)
    tau1, T1 = s.he2hb(d1)
    tau2, T2 = s.he2hb_sim(d2, 4)
    r, c = np.indices((n, n))
    low = r >= c
    assert _rel(d2.cpu().numpy()[low], d1.cpu().numpy()[low]) < 1e-11
    V2, t2 = synth.synthetic_v2(n, nb, 7)
    L = synth.unit_lower(n, 7)
    Z = synth.real_orthonormalish(n, m, 7)
    E, _, _ = s.hotpath(d2, torch.from_numpy(V2).cuda(), torch.from_numpy(t2).cuda(), _dev(L), _dev(Z),
                        flags=EIG_SKIP_HE2HB, tau1=tau2, T1=T2)
    A_o, tau_o = oracle.he2hb(A, nb)
    E_o = oracle.backsub_lh(L, oracle.apply_q1(A_o, tau_o, nb, oracle.apply_q2(V2, t2, nb, Z.astype(complex))))
    assert _rel(E.cpu().numpy(), E_o) < 1e-11
