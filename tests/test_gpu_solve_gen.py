"""NEXT-3 front end (potrf, hegst) parity and the whole generalized solver
(Algorithm 1, eig_solve_gen) against the oracle and the acceptance gates of
DESIGN.md readings R9/R10 (marker: gpu):
  eigenvalues  max|l - l_ref| / max|l_ref| <= min(1e-10, 1e-12 n kappa(B))
  residual     ||A Z - B Z L||_1 / (n ||A||_1 ||Z||_1) <= 1e-14
  B-orth       ||Z^H B Z - I||_1 / n <= 1e-14
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth

gpu = pytest.mark.gpu


def _solver(nb=64):
    from paper_1207_1773_b200 import Solver
    return Solver(0, nb=nb)


def _dev(x):
    from paper_1207_1773_b200 import colmajor
    return colmajor(x, torch.device("cuda:0"))


def gates(A, B, w_sel, Z):
    """R10 gates on the GPU with torch (test-side matmuls)."""
    A = torch.as_tensor(A).cuda() if not torch.is_tensor(A) else A
    B = torch.as_tensor(B).cuda() if not torch.is_tensor(B) else B
    Z = Z if torch.is_tensor(Z) else torch.as_tensor(Z).cuda()
    w_sel = torch.as_tensor(w_sel, device=Z.device)
    n = A.shape[0]
    R = A @ Z - (B @ Z) * w_sel[None, :]
    one = lambda M: torch.linalg.matrix_norm(M, ord=1).item()  # noqa: E731
    res = one(R) / (n * one(A) * one(Z))
    m = Z.shape[1]
    orth = one(Z.conj().T @ B @ Z - torch.eye(m, dtype=Z.dtype, device=Z.device)) / n
    return res, orth


# ------------------------------------------------------------------ potrf / hegst
@gpu
@pytest.mark.parametrize("n", [1, 64, 300, 517])
def test_potrf_parity(n):
    B = synth.hpd_with_condition(n, 1e3, 2) if n > 1 else np.array([[9.0 + 0j]])
    L_o, info = oracle.potrf(B)
    assert info == 0
    s = _solver()
    dB = _dev(B)
    assert s.potrf(dB) == 0
    Lg = np.tril(dB.cpu().numpy())
    assert np.max(np.abs(Lg - L_o)) < 1e-12 * np.max(np.abs(L_o))


@gpu
def test_potrf_not_positive_definite():
    s = _solver()
    assert s.potrf(_dev(np.array([[1, 2], [2, 1]], dtype=complex))) == 2 + 2   # S:L202 -> n + 2
    B = synth.hpd_with_condition(130, 10.0, 1)
    B[100, 100] = -5.0
    info = s.potrf(_dev(B))
    _, info_o = oracle.potrf(B)
    assert info == info_o and info > 130


@gpu
@pytest.mark.parametrize("n", [64, 300, 517])
def test_hegst_parity(n):
    A, B = synth.pencil_rand(n, seed=n, kappa=1e2)
    L = np.linalg.cholesky(B)
    C_o = oracle.std_form(A, L)
    s = _solver()
    dA = _dev(np.tril(A))
    s.hegst(dA, _dev(L))
    Cg = dA.cpu().numpy()
    low = np.tril(np.ones((n, n), bool))
    assert np.max(np.abs(Cg[low] - C_o[low])) < 1e-11 * np.max(np.abs(C_o))


# ------------------------------------------------------------------ whole solver
def _run(A, B, **kw):
    s = _solver(kw.pop("nb", 64))
    w, Z = s.solve_gen(_dev(np.tril(A)), _dev(np.tril(B)), **kw)
    return w.cpu().numpy(), Z


@gpu
@pytest.mark.parametrize("n,nb", [(256, 16), (300, 64), (2, 64), (65, 16)])
def test_solve_gen_vs_oracle(n, nb):
    A, B = synth.pencil_rand(n, seed=n + 1, kappa=1e2)
    w_o, Z_o, info, _ = oracle.solve_gen(A, B)
    assert info == 0
    w, Z = _run(A, B, nb=nb)
    assert np.max(np.abs(w - w_o)) / np.max(np.abs(w_o)) <= 1e-10
    res, orth = gates(A, B, w, Z)
    assert res <= 1e-14 and orth <= 1e-14


@gpu
def test_solve_gen_diagonal_and_2x2_pins():
    # P1: diag(2,4), diag(1,2) -> (2, 2)
    w, Z = _run(np.diag([2.0, 4.0]).astype(complex), np.diag([1.0, 2.0]).astype(complex))
    assert np.allclose(w, [2.0, 2.0], atol=1e-15)
    # P2 closed form (2 x 2)
    A = synth.rand_hermitian(2, 7)
    B = synth.hpd_with_condition(2, 10.0, 7, r=2)
    a11, a22, a21 = A[0, 0].real, A[1, 1].real, A[1, 0]
    b11, b22, b21 = B[0, 0].real, B[1, 1].real, B[1, 0]
    al = b11 * b22 - abs(b21) ** 2
    be = a11 * b22 + a22 * b11 - 2 * (np.conj(a21) * b21).real
    ga = a11 * a22 - abs(a21) ** 2
    disc = math.sqrt(be * be - 4 * al * ga)
    q = -0.5 * (-be - math.copysign(disc, -be))
    w, Z = _run(A, B)
    assert np.max(np.abs(w - np.sort([q / al, ga / q]))) < 1e-14


@gpu
@pytest.mark.parametrize("clustered", [False, True])
def test_solve_gen_known_spectrum_fraction(clustered):
    n = 500
    A, B, D = synth.pencil_known(n, seed=3, kappa=1e3, clustered=clustered)
    w, Z = _run(A, B, fraction=0.1)
    assert Z.shape[1] == 50
    assert np.max(np.abs(w - D)) / np.max(np.abs(D)) <= 1e-10
    res, orth = gates(A, B, w[:50], Z)
    assert res <= 1e-14 and orth <= 1e-14


@gpu
def test_solve_gen_not_pd():
    from paper_1207_1773_b200 import EigError
    A = synth.rand_hermitian(100, 1)
    B = synth.hpd_with_condition(100, 10.0, 1)
    B[40, 40] = -1.0
    with pytest.raises(EigError, match="rc=1"):
        _run(A, B)


@gpu
def test_config1_n2000_all_vectors():
    """BASELINE configs[1]: n = 2000, 100% eigenvectors; oracle eigenvalues + gates."""
    n = 2000
    A, B = synth.pencil_rand(n, seed=0, kappa=1e2)
    w_o, _, info, _ = oracle.solve_gen(A, B, 1, 1)
    assert info == 0
    w, Z = _run(A, B)
    assert np.max(np.abs(w - w_o)) / np.max(np.abs(w_o)) <= 1e-10
    res, orth = gates(A, B, w, Z)
    assert res <= 1e-14 and orth <= 1e-14


@gpu
@pytest.mark.parametrize("frac", [0.10, 0.25])
def test_config2_n5000_fraction(frac):
    """BASELINE configs[2]: n = 5000, 10% / 25% of the eigenvectors (known spectrum)."""
    n = 5000
    A, B, D = synth.pencil_known(n, seed=5, kappa=1e2, clustered=True)
    w, Z = _run(A, B, fraction=frac)
    m = int(math.ceil(frac * n))
    assert Z.shape[1] == m
    assert np.max(np.abs(w - D)) / np.max(np.abs(D)) <= 1e-10
    res, orth = gates(A, B, w[:m], Z)
    assert res <= 1e-14 and orth <= 1e-14


def _known_pencil_torch(n, seed, kappa=100.0):
    """Known-spectrum pencil built on the GPU (test-side): B = P P^H,
    A = P (W^H D W) P^H, P = U^H diag(sqrt s) U; lambda(A, B) = D, kappa(B) = kappa."""
    dev = torch.device("cuda:0")
    D = np.sort(synth.uniform(seed, 10, n) * 2.0 - 1.0)
    s = kappa ** (np.arange(n) / (n - 1))
    U = torch.from_numpy(synth.random_reflectors(n, 8, seed, 11)).to(dev)
    Wr = torch.from_numpy(synth.random_reflectors(n, 8, seed, 12)).to(dev)

    def congr(d, R):
        M = torch.diag(torch.as_tensor(d, dtype=torch.complex128, device=dev))
        for t in range(R.shape[1]):
            u = R[:, t:t + 1]
            M = M - 2.0 * u @ (u.conj().T @ M)
            M = M - 2.0 * (M @ u) @ u.conj().T
        return 0.5 * (M + M.conj().T)
    P = congr(np.sqrt(s), U)
    Cw = congr(D, Wr)
    A = P @ Cw @ P.conj().T
    A = 0.5 * (A + A.conj().T)
    B = P @ P.conj().T
    B = 0.5 * (B + B.conj().T)
    return A, B, D


@gpu
def test_config3_n10000_all_vectors_known_spectrum():
    """BASELINE configs[3] / the north-star target: n = 10000, 100% eigenvectors,
    all oracle tolerances (exact spectrum, residual, B-orthogonality)."""
    n = 10000
    A, B, D = _known_pencil_torch(n, 8)
    s = _solver()
    Ac = torch.tril(A).t().contiguous().t()
    Bc = torch.tril(B).t().contiguous().t()
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    w, Z = s.solve_gen(Ac, Bc)
    print(f"eig_solve_gen n={n} all vectors: {time.perf_counter() - t0:.3f} s")
    del Ac, Bc
    w = w.cpu().numpy()
    assert np.max(np.abs(w - D)) / np.max(np.abs(D)) <= 1e-10
    res, orth = gates(A, B, torch.from_numpy(w).cuda(), Z)
    assert res <= 1e-14 and orth <= 1e-14


@gpu
@pytest.mark.parametrize("frac", [0.10, 0.50, 1.00])
def test_config4_n20000_fraction_known_spectrum(frac):
    """BASELINE configs[4]: n = 20000, 10% / 50% / 100% of the eigenvectors
    (known spectrum, all gates).  Exercises the large-n paths: panel CTA count
    bound by shared memory, 106-CTA bulge chase, the widest Q2/Q1/trsm."""
    n = 20000
    A, B, D = _known_pencil_torch(n, 21)
    s = _solver()
    Ac = torch.tril(A).t().contiguous().t()
    Bc = torch.tril(B).t().contiguous().t()
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    w, Z = s.solve_gen(Ac, Bc, fraction=frac)
    print(f"eig_solve_gen n={n} {frac:.0%} vectors: {time.perf_counter() - t0:.3f} s")
    del Ac, Bc
    m = Z.shape[1]
    assert m == int(math.ceil(frac * n))
    w = w.cpu().numpy()
    assert np.max(np.abs(w - D)) / np.max(np.abs(D)) <= 1e-10
    res, orth = gates(A, B, torch.from_numpy(w[:m]).cuda(), Z)
    assert res <= 1e-14 and orth <= 1e-14


@gpu
def test_kappa1e4_n2000_vs_oracle():
    """SURVEY C9/G1 stress case: kappa(B) = 1e4 (potrf, hegst and trsm use
    explicit inverses of 64 x 64 diagonal blocks of L, whose error grows with
    kappa).  Eigenvalues vs the oracle, gates R9/R10 (eigenvalue bound
    min(1e-10, 1e-12 n kappa) = 1e-10)."""
    n = 2000
    A, B = synth.pencil_rand(n, seed=4, kappa=1e4)
    w_o, _, info, _ = oracle.solve_gen(A, B, 1, 1)
    assert info == 0
    w, Z = _run(A, B)
    err = np.max(np.abs(w - w_o)) / np.max(np.abs(w_o))
    res, orth = gates(A, B, w, Z)
    print(f"kappa 1e4 n={n}: eig {err:.2e} res {res:.2e} orth {orth:.2e}")
    assert err <= 1e-10
    assert res <= 1e-14 and orth <= 1e-14


@gpu
def test_kappa1e4_n10000_known_spectrum():
    """kappa(B) = 1e4 at the headline size n = 10000, all eigenvectors."""
    n = 10000
    A, B, D = _known_pencil_torch(n, 9, kappa=1e4)
    s = _solver()
    Ac = torch.tril(A).t().contiguous().t()
    Bc = torch.tril(B).t().contiguous().t()
    w, Z = s.solve_gen(Ac, Bc)
    del Ac, Bc
    w = w.cpu().numpy()
    err = np.max(np.abs(w - D)) / np.max(np.abs(D))
    res, orth = gates(A, B, torch.from_numpy(w).cuda(), Z)
    print(f"kappa 1e4 n={n}: eig {err:.2e} res {res:.2e} orth {orth:.2e}")
    assert err <= 1e-10
    assert res <= 1e-14 and orth <= 1e-14


@gpu
@pytest.mark.parametrize("il,iu", [(101, 160), (1, 1), (500, 500), (250, 251)])
def test_solve_gen_index_range(il, iu):
    """EIG_RANGE_INDEX (S:L57-L65 index-range il..iu): all eigenvalues, eigenvectors of
    the il-th .. iu-th only, which must pass the gates on their own."""
    n = 500
    A, B, D = synth.pencil_known(n, seed=12, kappa=1e2, clustered=False)
    w, Z = _run(A, B, il=il, iu=iu)
    assert Z.shape[1] == iu - il + 1
    assert np.max(np.abs(w - D)) / np.max(np.abs(D)) <= 1e-10
    res, orth = gates(A, B, w[il - 1:iu], Z)
    assert res <= 1e-14 and orth <= 1e-14


@gpu
def test_solve_gen_tiny_fraction():
    """fraction -> il = 1, iu = ceil(f n) = 1: one eigenvector, the lowest."""
    n = 300
    A, B, D = synth.pencil_known(n, seed=13, kappa=10.0, clustered=True)
    w, Z = _run(A, B, fraction=0.001)
    assert Z.shape[1] == 1
    assert np.max(np.abs(w - D)) / np.max(np.abs(D)) <= 1e-10
    res, orth = gates(A, B, w[:1], Z)
    assert res <= 1e-14 and orth <= 1e-14
