"""NEXT-2 parity: device divide and conquer (eig_stedc) vs the oracle's
tridiagonal solvers (QL tql2, Sturm bisection) and closed forms (marker: gpu).
Eigenvalues are compared directly; eigenvectors through the residual and
orthogonality (they are unique only up to sign, reading R14/C12)."""
import numpy as np
import pytest
import torch

import oracle
import synth

gpu = pytest.mark.gpu


def _solve(d, e, il=1, iu=None):
    from paper_1207_1773_b200 import Solver
    s = Solver(0, nb=64)
    w, Z = s.stedc(torch.from_numpy(np.ascontiguousarray(d)).cuda(), torch.from_numpy(np.ascontiguousarray(e)).cuda(),
                   il, iu)
    return w.cpu().numpy(), Z.cpu().numpy()


def _check(d, e, il=1, iu=None, tol_res=None):
    n = d.shape[0]
    iu = n if iu is None else iu
    w, Z = _solve(d, e, il, iu)
    ws = oracle.sturm_values(d, e)
    Tn = max(np.max(np.abs(d)) + 2 * np.max(np.abs(e)) if n > 1 else abs(d[0]), 1e-300)
    assert np.max(np.abs(w - ws)) <= 100 * n * np.finfo(float).eps * Tn
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    m = iu - il + 1
    R = T @ Z - Z * w[il - 1:iu]
    assert np.linalg.norm(R) / (np.sqrt(m) * Tn) <= (tol_res or 100 * n * np.finfo(float).eps)
    assert np.linalg.norm(Z.T @ Z - np.eye(m)) <= 100 * n * np.finfo(float).eps
    return w, Z


@gpu
@pytest.mark.parametrize("n", [1, 2, 5, 32, 33, 64, 100, 257, 1000])
def test_stedc_random(n):
    d = synth.rnormal(n, 1, (n,))
    e = synth.rnormal(n, 2, (max(n - 1, 0),))
    _check(d, e)


@gpu
def test_stedc_closed_forms():
    # n = 2, d = (0, 0), e = (1) -> +-1
    w, Z = _solve(np.zeros(2), np.ones(1))
    assert np.allclose(w, [-1, 1], atol=1e-15)
    # d = 0, e = 1: 2 cos(k pi / (n+1))
    n = 300
    w, Z = _check(np.zeros(n), np.ones(n - 1))
    assert np.max(np.abs(w - np.sort(2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1))))) < 1e-13
    # diagonal (e = 0): everything deflates
    dd = synth.rnormal(3, 3, (200,))
    w, Z = _check(dd, np.zeros(199))
    assert np.array_equal(w, np.sort(dd))


@gpu
def test_stedc_clustered_and_glued():
    # Wilkinson-like glued matrix with tight clusters (heavy close-pole deflation)
    n = 400
    d = np.abs(np.arange(n) % 21 - 10).astype(float)
    e = np.ones(n - 1)
    e[20::21] = 1e-9
    _check(d, e, tol_res=1e-12)


@gpu
@pytest.mark.parametrize("il,iu", [(1, 100), (450, 550), (1000, 1000)])
def test_stedc_partial_last_merge(il, iu):
    n = 1000
    d = synth.rnormal(7, 1, (n,))
    e = synth.rnormal(7, 2, (n - 1,))
    w, Z = _check(d, e, il, iu)
    wf, Zf = _solve(d, e)
    # the selected columns equal the full solve's columns up to sign
    Zs = Zf[:, il - 1:iu]
    sgn = np.sign(np.sum(Z * Zs, axis=0))
    assert np.max(np.abs(Z - Zs * sgn)) < 1e-10


@gpu
def test_stedc_full_size():
    n = 10000
    d = synth.rnormal(9, 1, (n,))
    e = synth.rnormal(9, 2, (n - 1,))
    w, Z = _solve(d, e)
    idx = np.unique(np.linspace(1, n, 40).astype(int))
    ws = np.array([oracle.sturm_values(d, e, k, k)[0] for k in idx])
    Tn = np.max(np.abs(d)) + 2 * np.max(np.abs(e))
    assert np.max(np.abs(w[idx - 1] - ws)) <= 100 * n * np.finfo(float).eps * Tn
    cols = idx[:8] - 1
    T_Z = d[:, None] * Z[:, cols]
    T_Z[:-1] += e[:, None] * Z[1:, cols]
    T_Z[1:] += e[:, None] * Z[:-1, cols]
    assert np.linalg.norm(T_Z - Z[:, cols] * w[cols]) / (np.sqrt(len(cols)) * Tn) < 1e-12
    G = Z[:, cols].T @ Z
    G[np.arange(len(cols)), cols] -= 1.0
    assert np.max(np.abs(G)) < 1e-11
