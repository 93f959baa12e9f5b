"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (nb = 64, g = 32, n = m = 10000), on sampled outputs the oracle can
compute one by one, plus properties that hold at any size (marker: gpu).

Also BASELINE configs[1] (n = 2000, m = 2000): the whole pass vs the oracle
chain on sampled columns.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

gpu = pytest.mark.gpu

N_FULL = 10000
NB = 64


def _solver(nb=NB, g=32):
    from paper_1207_1773_b200 import Solver
    return Solver(0, nb=nb, q2_group=g)


def _dev(x):
    from paper_1207_1773_b200 import colmajor
    return colmajor(x, torch.device("cuda:0"))


def _rel(a, b):
    return np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.max(np.abs(b)), 1e-300)


@pytest.fixture(scope="module")
def he2hb_full():
    n = N_FULL
    A = synth.rand_hermitian(n, 0)
    s = _solver()
    dA = _dev(A)
    tau, T = s.he2hb(dA)
    torch.cuda.synchronize()
    return A, dA, tau, T, s


@gpu
def test_full_he2hb_first_panel_vs_oracle(he2hb_full):
    """The first panel's reflectors, R block and taus (the first nb reflectors of
    the whole reduction) against the oracle run for exactly those reflectors."""
    A, dA, tau, T, s = he2hb_full
    n = A.shape[0]
    A_o, tau_o = oracle.he2hb_partial(A, NB, NB)
    cols = dA[:, :NB].cpu().numpy()
    low = np.tril(np.ones((n, NB), bool))          # rows >= column (lower part of the panel columns)
    assert _rel(cols[low], A_o[:, :NB][low]) < 1e-11
    assert np.max(np.abs(tau.cpu().numpy()[:NB] - tau_o[:NB])) < 1e-11


@gpu
def test_full_he2hb_invariants(he2hb_full):
    """Trace, Frobenius norm and A (Q1 x) = Q1 (Band x) at n = 10000."""
    A, dA, tau, T, s = he2hb_full
    n = A.shape[0]
    dev = dA.device
    Ag = torch.from_numpy(A).to(dev)
    Bl = torch.tril(dA)                              # lower part incl. V below the band
    r = torch.arange(n, device=dev)
    band_mask = (r[:, None] - r[None, :] <= NB) & (r[:, None] >= r[None, :])
    Bl = torch.where(band_mask, Bl, torch.zeros((), dtype=Bl.dtype, device=dev))
    Band = Bl + torch.tril(Bl, -1).conj().T
    Band.diagonal().imag.zero_()
    assert abs(torch.trace(Band).real.item() - np.trace(A).real) < 1e-9
    nA = torch.linalg.norm(Ag).item()
    assert abs(torch.linalg.norm(Band).item() - nA) / nA < 1e-13
    x = synth.cnormal(5, 5, (n, 2))
    from paper_1207_1773_b200 import colmajor
    qx = colmajor(x, dev)
    s.apply_q1(dA, T, qx)                           # Q1 x
    bx = colmajor((Band @ torch.from_numpy(x).to(dev)).cpu().numpy(), dev)
    s.apply_q1(dA, T, bx)                           # Q1 Band x
    lhs = Ag @ qx
    err = torch.linalg.norm(lhs - bx).item() / (nA * np.linalg.norm(x))
    assert err < 1e-14


@gpu
def test_full_q2_sampled_columns_vs_oracle():
    n, m = N_FULL, N_FULL
    s = _solver()
    V2, tau2 = synth.synthetic_v2(n, NB, 0)
    Z = synth.real_orthonormalish(n, m, 0)
    from paper_1207_1773_b200 import empty_colmajor
    dE = empty_colmajor(n, m)
    s.apply_q2(torch.from_numpy(V2).cuda(), torch.from_numpy(tau2).cuda(), dE, Z=_dev(Z))
    cols = [0, 1, 4567, m - 1]
    ref = oracle.apply_q2(V2, tau2, NB, Z[:, cols].astype(complex))
    got = dE[:, cols].cpu().numpy()
    assert _rel(got, ref) < 1e-11
    # unitarity on all columns: ||Q2 z|| = ||z||
    nrm = torch.linalg.norm(dE, dim=0).cpu().numpy()
    assert np.max(np.abs(nrm - np.linalg.norm(Z, axis=0))) < 1e-12


@gpu
def test_full_q1_sampled_columns_vs_oracle():
    """Q1 with random exactly-unitary reflectors in the he2hb layout (their T
    factors from the oracle's larft) at n = 10000, sampled columns."""
    n = N_FULL
    A1, tau1 = synth.synthetic_v1(n, NB, 1)
    from paper_1207_1773_b200 import num_panels
    K = num_panels(n, NB)
    Ts = np.zeros((K, NB, NB), complex)
    for k in range(K):
        r0 = (k + 1) * NB
        V = np.tril(A1[r0:, k * NB:(k + 1) * NB], -1)
        for j in range(min(NB, n - r0)):
            V[j, j] = 1
        Ts[k] = oracle.larft(V, tau1[k * NB:(k + 1) * NB])
    m = 300
    E0 = synth.cnormal(1, 7, (n, m))
    s = _solver()
    dE = _dev(E0)
    s.apply_q1(_dev(A1), torch.from_numpy(Ts.transpose(0, 2, 1).reshape(-1).copy()).cuda(), dE)
    cols = [0, 150, m - 1]
    ref = oracle.apply_q1(A1, tau1, NB, E0[:, cols])
    assert _rel(dE[:, cols].cpu().numpy(), ref) < 1e-11


@gpu
def test_full_trsm_sampled_columns_vs_oracle():
    n, m = N_FULL, 512
    L = synth.unit_lower(n, 2)
    E0 = synth.cnormal(2, 8, (n, m))
    s = _solver()
    dE = _dev(E0)
    s.trsm_lh(_dev(L), dE)
    cols = [0, 255, m - 1]
    ref = oracle.backsub_lh(L, E0[:, cols])
    assert _rel(dE[:, cols].cpu().numpy(), ref) < 1e-11


@gpu
def test_full_hotpath_bench_configuration_properties():
    """The exact bench step (n = m = 10000, nb = 64, g = 32): ||L^H E|| = ||Z||
    column by column (Q1 Q2 is unitary) and the Q2 part on sampled columns."""
    n, m = N_FULL, N_FULL
    s = _solver()
    A = synth.rand_hermitian(n, 0)
    V2, tau2 = synth.synthetic_v2(n, NB, 0)
    L = synth.unit_lower(n, 0)
    Z = synth.real_orthonormalish(n, m, 0)
    dL = _dev(L)
    E, tau1, T1 = s.hotpath(_dev(A), torch.from_numpy(V2).cuda(), torch.from_numpy(tau2).cuda(), dL, _dev(Z))
    LE = torch.tril(dL).conj().T @ E
    nrm = torch.linalg.norm(LE, dim=0).cpu().numpy()
    assert np.max(np.abs(nrm - np.linalg.norm(Z, axis=0))) < 1e-11
    assert torch.isfinite(E).all()


@gpu
def test_config1_n2000_whole_pass_sampled_vs_oracle():
    """BASELINE configs[1]: n = 2000, all 2000 eigenvector columns on the GPU;
    the oracle chain (he2hb, Q2, Q1, L^-H, one reflector at a time) on 16
    sampled columns."""
    n, m = 2000, 2000
    s = _solver()
    A = synth.rand_hermitian(n, 3)
    V2, tau2 = synth.synthetic_v2(n, NB, 3)
    L = synth.unit_lower(n, 3)
    Z = synth.real_orthonormalish(n, m, 3)
    E, tau1, T1 = s.hotpath(_dev(A), torch.from_numpy(V2).cuda(), torch.from_numpy(tau2).cuda(), _dev(L), _dev(Z))
    cols = list(range(0, m, m // 16))
    A_o, tau_o = oracle.he2hb(A, NB)
    E_o = oracle.backsub_lh(L, oracle.apply_q1(A_o, tau_o, NB,
                                                oracle.apply_q2(V2, tau2, NB, Z[:, cols].astype(complex))))
    assert _rel(E[:, cols].cpu().numpy(), E_o) < 1e-11
