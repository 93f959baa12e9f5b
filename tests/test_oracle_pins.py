"""Pins for the CPU oracle (tests/ -m "not gpu").

Each test checks the oracle against something other than itself: closed
forms, brute force, invariants, or a library routine (scipy/LAPACK), chosen so
that a dropped term, a wrong sign/index or a transposed operand fails at least
one of them.  Pin ids (P1..P12) follow DESIGN.md "Oracle pins".
"""
import itertools
import math

import numpy as np
import pytest
import scipy.linalg as sla

import oracle
import synth

EPS = np.finfo(float).eps


def rel_eig_err(w, w_ref):
    w = np.sort(np.asarray(w))
    w_ref = np.sort(np.asarray(w_ref))
    return np.max(np.abs(w - w_ref)) / max(np.max(np.abs(w_ref)), 1e-300)


def residual_1(A, B, Z, w):
    """C9 reading: ||A Z - B Z diag(w)||_1 / (n ||A||_1 ||Z||_1)."""
    n = A.shape[0]
    R = A @ Z - (B @ Z) * w[None, :]
    return np.linalg.norm(R, 1) / (n * np.linalg.norm(A, 1) * np.linalg.norm(Z, 1))


def borth_1(B, Z):
    m = Z.shape[1]
    return np.linalg.norm(Z.conj().T @ B @ Z - np.eye(m), 1) / Z.shape[0]


# --------------------------------------------------------------- P1 diagonal
def test_p1_diagonal_pencil_spec_example():
    # A = diag(2,4), B = diag(1,2) -> lambda = (2, 2)
    A = np.diag([2.0, 4.0]).astype(complex)
    B = np.diag([1.0, 2.0]).astype(complex)
    w, Z, info, _ = oracle.solve_gen(A, B)
    assert info == 0
    assert np.allclose(w, [2.0, 2.0], atol=1e-15)
    assert borth_1(B, Z) < 1e-15


def test_p1_diagonal_pencil_random():
    n = 37
    a = synth.uniform(3, 1, n) * 4 - 2
    b = synth.uniform(3, 2, n) + 0.5
    w, Z, info, _ = oracle.solve_gen(np.diag(a).astype(complex), np.diag(b).astype(complex))
    assert info == 0
    assert np.allclose(w, np.sort(a / b), rtol=0, atol=4 * EPS * 4)
    # x_i = e_i / sqrt(b_ii) up to a unit phase
    order = np.argsort(a / b, kind="stable")
    for c, i in enumerate(order):
        assert abs(abs(Z[i, c]) - 1 / math.sqrt(b[i])) < 1e-14


# --------------------------------------------------------------- P2 2x2
def test_p2_two_by_two_closed_form():
    for seed in range(20):
        A = synth.rand_hermitian(2, seed)
        B = synth.hpd_with_condition(2, 10.0, seed, r=2)
        a11, a22, a21 = A[0, 0].real, A[1, 1].real, A[1, 0]
        b11, b22, b21 = B[0, 0].real, B[1, 1].real, B[1, 0]
        al = b11 * b22 - abs(b21) ** 2
        be = a11 * b22 + a22 * b11 - 2 * (np.conj(a21) * b21).real
        ga = a11 * a22 - abs(a21) ** 2
        disc = math.sqrt(be * be - 4 * al * ga)
        q = -0.5 * (-be - math.copysign(disc, -be))
        roots = np.sort([q / al, ga / q])
        w, Z, info, _ = oracle.solve_gen(A, B)
        assert info == 0
        assert np.max(np.abs(w - roots)) <= 1e-14 * max(1, np.max(np.abs(roots)))


# --------------------------------------------------------------- P3 brute force
def _charpoly_det(A, B):
    """det(A - lam B) by Leibniz expansion -> real polynomial coefficients
    (highest degree first)."""
    n = A.shape[0]
    total = np.zeros(n + 1, dtype=complex)
    for perm in itertools.permutations(range(n)):
        inv = sum(1 for i in range(n) for j in range(i + 1, n) if perm[i] > perm[j])
        poly = np.array([1.0 + 0j])
        for i in range(n):
            poly = np.polymul(poly, np.array([-B[i, perm[i]], A[i, perm[i]]]))
        total = total + (-1) ** inv * poly
    return total.real


def _polish(p, x):
    dp = np.polyder(p)
    for _ in range(50):
        f, d = np.polyval(p, x), np.polyval(dp, x)
        if d == 0:
            break
        step = f / d
        x = x - step
        if abs(step) <= 1e-17 * max(1, abs(x)):
            break
    return x


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_p3_brute_force_small(n):
    for seed in range(5):
        A = synth.rand_hermitian(n, seed + 100)
        B = synth.hpd_with_condition(n, 5.0, seed + 100, r=n)
        p = _charpoly_det(A, B)
        roots = np.sort([_polish(p, r.real) for r in np.roots(p)])
        w, Z, info, _ = oracle.solve_gen(A, B)
        assert info == 0
        assert np.max(np.abs(w - roots)) <= 1e-11 * max(1, np.max(np.abs(roots)))
        assert residual_1(A, B, Z, w) < 1e-15


# --------------------------------------------------------------- P4 Kronecker
def test_p4_kronecker_sum_and_product():
    n1, n2 = 6, 7
    K1, M1, l1 = synth.fem_pencil(n1, 1)
    K2, M2, l2 = synth.fem_pencil(n2, 2)
    A = np.kron(K1, M2) + np.kron(M1, K2)
    B = np.kron(M1, M2)
    w, Z, info, _ = oracle.solve_gen(A, B)
    assert info == 0
    exact = np.sort((l1[:, None] + l2[None, :]).ravel())
    assert rel_eig_err(w, exact) < 1e-13
    A2 = np.kron(K1, K2)
    w2, _, info, _ = oracle.solve_gen(A2, B)
    assert info == 0
    exact2 = np.sort((l1[:, None] * l2[None, :]).ravel())
    assert rel_eig_err(w2, exact2) < 1e-13


# --------------------------------------------------------------- P5 known spectrum
@pytest.mark.parametrize("clustered", [False, True])
def test_p5_known_spectrum(clustered):
    n = 96
    A, B, D = synth.pencil_known(n, seed=4, kappa=1e3, clustered=clustered)
    w, Z, info, _ = oracle.solve_gen(A, B)
    assert info == 0
    assert rel_eig_err(w, D) < 1e-12
    assert residual_1(A, B, Z, w) < 1e-14
    assert borth_1(B, Z) < 1e-14


# --------------------------------------------------------------- P6 FEM closed form
def test_p6_fem_closed_form():
    n = 120
    A, B, lam = synth.fem_pencil(n, 7)
    w, Z, info, _ = oracle.solve_gen(A, B)
    assert info == 0
    assert rel_eig_err(w, lam) < 1e-13


# --------------------------------------------------------------- P7 invariances
def test_p7_shift_scale_congruence():
    n = 40
    A, B = synth.pencil_rand(n, seed=5, kappa=1e2)
    w, _, _, _ = oracle.solve_gen(A, B)
    sig = 0.75
    ws, _, _, _ = oracle.solve_gen(A + sig * B, B)
    assert np.max(np.abs(ws - (w + sig))) < 1e-13
    wc, _, _, _ = oracle.solve_gen(3.0 * A, B)
    assert np.max(np.abs(wc - 3.0 * w)) < 1e-13
    wb, _, _, _ = oracle.solve_gen(A, 2.0 * B)
    assert np.max(np.abs(wb - 0.5 * w)) < 1e-13
    # nonsingular congruence P^H A P, P^H B P
    P = np.eye(n) + 0.3 * synth.cnormal(9, 1, (n, n)) / np.sqrt(n)
    wp, _, _, _ = oracle.solve_gen(synth.hermitian_full(P.conj().T @ A @ P), synth.hermitian_full(P.conj().T @ B @ P))
    assert rel_eig_err(wp, w) < 1e-12


def test_p7_identity_B_is_standard_problem():
    n = 50
    A = synth.rand_hermitian(n, 6)
    w, Z, info, L = oracle.solve_gen(A, np.eye(n, dtype=complex))
    assert info == 0
    assert np.allclose(np.tril(L), np.eye(n))
    wj, _ = oracle.jacobi(A)
    assert np.max(np.abs(w - wj)) < 10 * n * EPS * 2


# --------------------------------------------------------------- P8 library routine
@pytest.mark.parametrize("n,kappa", [(64, 1e2), (200, 1e3)])
def test_p8_lapack_cross_check(n, kappa):
    A, B = synth.pencil_rand(n, seed=n, kappa=kappa)
    w, Z, info, _ = oracle.solve_gen(A, B)
    assert info == 0
    wl = sla.eigh(A, B, eigvals_only=True, driver="gvd")
    assert rel_eig_err(w, wl) < 1e-12


# --------------------------------------------------------------- P9 invariants
def test_p9_residual_and_borth_gates_partial():
    n = 256
    A, B = synth.pencil_rand(n, seed=1, kappa=1e2)
    il, iu = 1, 26
    w, Z, info, _ = oracle.solve_gen(A, B, il, iu)
    assert info == 0 and Z.shape == (n, iu - il + 1)
    assert residual_1(A, B, Z, w[il - 1:iu]) < 1e-14
    assert borth_1(B, Z) < 1e-14


# --------------------------------------------------------------- Cholesky / transforms
def test_potrf_spec_examples():
    L, info = oracle.potrf(np.eye(4, dtype=complex))
    assert info == 0 and np.allclose(L, np.eye(4), atol=0)
    L, info = oracle.potrf(np.diag([4.0, 9.0]).astype(complex))
    assert info == 0 and np.allclose(L, np.diag([2.0, 3.0]), atol=0)
    # [[1,2],[2,1]] not PD at the second pivot -> info = n + 2
    _, info = oracle.potrf(np.array([[1, 2], [2, 1]], dtype=complex))
    assert info == 2 + 2


def test_potrf_reconstruction_and_lapack():
    n = 120
    B = synth.hpd_with_condition(n, 1e3, 3)
    L, info = oracle.potrf(B)
    assert info == 0
    assert np.linalg.norm(L @ L.conj().T - B) <= 10 * n * EPS * np.linalg.norm(B)
    assert np.allclose(L, np.linalg.cholesky(B), atol=1e-12)
    assert np.all(np.diag(L).real > 0) and np.all(np.diag(L).imag == 0)


def test_std_form_examples_and_congruence():
    n = 30
    A = synth.rand_hermitian(n, 2)
    C = oracle.std_form(A, np.eye(n, dtype=complex))
    assert np.allclose(C, A, atol=1e-15)
    C = oracle.std_form(np.eye(n, dtype=complex), 2 * np.eye(n, dtype=complex))
    assert np.allclose(C, np.eye(n) / 4, atol=1e-16)
    B = synth.hpd_with_condition(n, 1e2, 2)
    L = np.linalg.cholesky(B)
    C = oracle.std_form(A, L)
    X = sla.solve_triangular(L, sla.solve_triangular(L, A, lower=True).conj().T, lower=True).conj().T
    assert np.linalg.norm(C - X) <= 50 * n * EPS * np.linalg.norm(A) * 1e2
    assert np.allclose(C, C.conj().T, atol=0)


def test_backsub_lh_vs_library():
    n, m = 50, 7
    L = synth.unit_lower(n, 3)
    Y = synth.cnormal(3, 5, (n, m))
    X = oracle.backsub_lh(L, Y)
    ref = sla.solve_triangular(L.conj().T, Y, lower=False)
    assert np.allclose(X, ref, rtol=1e-13, atol=1e-14)
    assert np.linalg.norm(L.conj().T @ X - Y) < 1e-13


# --------------------------------------------------------------- P12 tridiagonal
def test_p12_tridiagonal_closed_form_all_paths():
    n = 60
    d = np.zeros(n)
    e = np.ones(n - 1)
    exact = np.sort(2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1)))
    w, Zt, info = oracle.tql2(d, e)
    assert info == 0 and np.max(np.abs(w - exact)) < 1e-14
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    assert np.linalg.norm(T @ Zt - Zt * w) < 1e-13
    assert np.linalg.norm(Zt.T @ Zt - np.eye(n)) < 1e-13
    ws = oracle.sturm_values(d, e)
    assert np.max(np.abs(ws - exact)) < 1e-14
    # n=2, d=(0,0), e=(1) -> +-1
    w2, _, _ = oracle.tql2(np.zeros(2), np.ones(1))
    assert np.allclose(w2, [-1, 1], atol=1e-16)


def test_hetd2_reconstruction_and_flop_free_invariants():
    n = 48
    A = synth.rand_hermitian(n, 8)
    d, e, Cref, tau = oracle.hetd2(A)
    # explicit Q from the stored reflectors (dense products; independent path)
    Q = np.eye(n, dtype=complex)
    for k in range(n - 1):
        v = np.zeros(n, dtype=complex)
        v[k + 1] = 1
        v[k + 2:] = Cref[k + 2:, k]
        Q = Q @ (np.eye(n) - tau[k] * np.outer(v, v.conj()))
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    assert np.linalg.norm(Q.conj().T @ A @ Q - T) <= 50 * n * EPS * np.linalg.norm(A)
    assert np.linalg.norm(Q.conj().T @ Q - np.eye(n)) <= 50 * n * EPS
    assert rel_eig_err(np.linalg.eigvalsh(T), np.linalg.eigvalsh(A)) < 1e-13


def test_jacobi_vs_lapack():
    n = 64
    A = synth.rand_hermitian(n, 9)
    w, V = oracle.jacobi(A)
    assert np.max(np.abs(w - np.linalg.eigvalsh(A))) < 10 * n * EPS
    assert np.linalg.norm(A @ V - V * w) < 1e-13


# --------------------------------------------------------------- larfg (R1)
def test_larfg_convention():
    rng_x = synth.cnormal(1, 1, (7,))
    alpha = 0.3 - 0.8j
    beta, tau, v = oracle.larfg(alpha, rng_x)
    x = np.concatenate([[alpha], rng_x])
    H = np.eye(8) - tau * np.outer(v, v.conj())
    y = H.conj().T @ x
    # |beta| ~ 3: a few ulps (the scaled dznrm2/dlapy3 norms of reading R1
    # round differently from a plain sum of squares)
    assert abs(y[0] - beta) < 4 * EPS * abs(beta) and np.max(np.abs(y[1:])) < 4 * EPS * abs(beta)
    assert np.linalg.norm(H.conj().T @ H - np.eye(8)) < 1e-14
    assert beta == pytest.approx(-math.copysign(np.linalg.norm(x), alpha.real), rel=2 * EPS)
    assert v[0] == 1
    # zero x, real alpha -> tau = 0 (H = I); zero x, complex alpha -> real beta
    b0, t0, _ = oracle.larfg(2.5 + 0j, np.zeros(3))
    assert t0 == 0 and b0 == 2.5
    b1, t1, _ = oracle.larfg(1.0 + 1.0j, np.zeros(1))
    assert t1 != 0 and abs(b1 + math.sqrt(2)) < 1e-15


@pytest.mark.parametrize("s", [1e-300, 1e-310, 1e-320, 1e200, 1e300])
def test_larfg_extreme_scales(s):
    """Reading R1: LAPACK zlarfg forms ||x|| with the scaled dznrm2 and
    ||(alpha, x)|| with dlapy3, and rescales by 1/safmin while |beta| <
    safmin, so H is scale invariant: larfg(s alpha, s x) = (s beta, tau, v)
    wherever s beta is representable.  A plain sum of |x_i|^2 overflows at
    s = 1e200 (1e400) and underflows to 0 at s = 1e-300 (tau would become 0
    or v would be inf), so each case fails a naive norm.  The expected beta
    is formed independently: s * -copysign(||(alpha, x)||, Re alpha) with
    numpy's norm on the unscaled vector."""
    x = synth.cnormal(7, 1, (9,))
    alpha = -0.4 + 0.7j
    beta1, tau1, v1 = oracle.larfg(alpha, x)
    ref_beta = -math.copysign(np.linalg.norm(np.concatenate([[alpha], x])), alpha.real)
    assert abs(beta1 - ref_beta) <= 4 * EPS * abs(ref_beta)
    with np.errstate(all="ignore"):
        beta, tau, v = oracle.larfg(alpha * s, x * s)
    # subnormal inputs (s <= 1e-310) carry fewer significant bits: the
    # tolerance is relative to the precision the inputs still have
    prec = max(EPS, 2.0 ** -1074 / (s * np.min(np.abs(np.concatenate([[alpha], x])))))
    assert np.isfinite(beta) and np.isfinite(tau) and np.all(np.isfinite(v))
    assert abs(beta - s * ref_beta) <= 8 * prec * abs(s * ref_beta)
    assert abs(tau - tau1) <= 8 * prec
    assert np.max(np.abs(v - v1)) <= 8 * prec * np.max(np.abs(v1))
    # H^H (alpha; x) = (beta; 0) at the scaled values, relative to s
    xs = np.concatenate([[alpha], x]) * s
    y = xs - np.conj(tau) * v * (v.conj() @ xs)
    assert abs(y[0] - beta) <= 16 * prec * abs(beta)
    assert np.max(np.abs(y[1:])) <= 16 * prec * abs(beta)


def test_larfg_zero_tail_complex_alpha():
    """x = 0 with complex alpha: tau != 0, beta = -sign(Re alpha)|alpha| real,
    and H^H maps alpha to beta (the phase-fixing reflector of reading R1)."""
    for alpha in (0.3 + 0.4j, -2.0 - 1e-3j, 1e-305 + 1e-305j, 1e250 - 3e250j):
        beta, tau, v = oracle.larfg(alpha, np.zeros(5))
        assert beta == pytest.approx(-math.copysign(abs(alpha), alpha.real), rel=4 * EPS)
        assert np.all(v[1:] == 0)
        assert abs((1 - np.conj(tau)) * alpha - beta) <= 8 * EPS * abs(beta)


# --------------------------------------------------------------- he2hb (R3, R6)
def _q1_explicit(A_out, tau, nb):
    n = A_out.shape[0]
    Q = np.eye(n, dtype=complex)
    i = 0
    while i + nb < n:
        for j in range(nb):
            r0 = i + nb + j
            if r0 >= n:
                continue
            v = np.zeros(n, dtype=complex)
            v[r0] = 1
            v[r0 + 1:] = A_out[r0 + 1:, i + j]
            Q = Q @ (np.eye(n) - tau[i + j] * np.outer(v, v.conj()))
        i += nb
    return Q


def _band_of(A_out, nb):
    n = A_out.shape[0]
    r, c = np.indices((n, n))
    Bl = np.where((r - c >= 0) & (r - c <= nb), A_out, 0)
    return synth.hermitian_full(np.tril(Bl) + np.tril(Bl, -1).conj().T)


@pytest.mark.parametrize("n,nb", [(48, 8), (50, 7), (33, 16), (17, 16), (16, 16), (64, 16)])
def test_he2hb_oracle_unitary_reconstruction(n, nb):
    A = synth.rand_hermitian(n, n + nb)
    A_out, tau = oracle.he2hb(A, nb)
    Band = _band_of(A_out, nb)
    Q = _q1_explicit(A_out, tau, nb)
    assert np.linalg.norm(Q.conj().T @ Q - np.eye(n)) <= 50 * n * EPS
    assert np.linalg.norm(Q.conj().T @ A @ Q - Band) <= 50 * n * EPS * np.linalg.norm(A)
    assert rel_eig_err(np.linalg.eigvalsh(Band), np.linalg.eigvalsh(A)) < 1e-13
    # outermost band entries produced by panels are real (diag(R) = beta)
    i = 0
    while i + nb < n:
        for j in range(min(nb, n - i - nb)):
            assert A_out[i + nb + j, i + j].imag == 0
        i += nb


def _reflector_order(n, nb):
    """(panel column c, unit-head row r0) of every he2hb reflector in the
    order orc_he2hb generates them (reading R3)."""
    out = []
    i = 0
    while i + nb < n:
        for j in range(min(nb, n - i - nb)):
            out.append((i + j, i + nb + j))
        i += nb
    return out


@pytest.mark.parametrize("n,nb", [(40, 8), (37, 6)])
def test_he2hb_partial_oracle_is_prefix_two_sided_similarity(n, nb):
    """Pin of orc_he2hb_partial (bench cpu_baseline sample and reference of
    the full-size first-panel GPU test): after r reflectors the stored state
    M_r (lower triangle, processed reflector tails zeroed, Hermitian
    completion) equals Q_r^H A Q_r with Q_r = H_1 ... H_r built explicitly
    from the stored (v, tau); columns processed so far are in band form; no
    tau beyond r is set; and r = K*nb (all reflectors) reproduces orc_he2hb."""
    A = synth.rand_hermitian(n, 11 * n + nb)
    order = _reflector_order(n, nb)
    for r in sorted({0, 1, 3, nb - 1, nb, nb + 2, 2 * nb + 1, len(order)}):
        r = min(r, len(order))
        Ar, tau = oracle.he2hb_partial(A, nb, r)
        Q = np.eye(n, dtype=complex)
        M = np.tril(Ar).copy()
        for (c, r0) in order[:r]:
            v = np.zeros(n, dtype=complex)
            v[r0] = 1
            v[r0 + 1:] = Ar[r0 + 1:, c]
            t = tau[(c // nb) * nb + c % nb]
            Q = Q @ (np.eye(n) - t * np.outer(v, v.conj()))
            M[r0 + 1:, c] = 0
            assert Ar[r0, c].imag == 0          # diag(R) = beta is real
        M = M + np.tril(M, -1).conj().T
        M[np.diag_indices(n)] = M[np.diag_indices(n)].real
        assert np.linalg.norm(Q.conj().T @ Q - np.eye(n)) <= 50 * n * EPS
        assert np.linalg.norm(Q.conj().T @ A @ Q - M) <= 50 * n * EPS * np.linalg.norm(A)
        done = {(c // nb) * nb + c % nb for (c, _) in order[:r]}
        assert all(tau[k] == 0 for k in range(len(tau)) if k not in done)
    Af, tauf = oracle.he2hb(A, nb)
    Ap, taup = oracle.he2hb_partial(A, nb, len(order))
    assert np.array_equal(Af, Ap) and np.array_equal(tauf, taup)


def test_he2hb_oracle_scale_invariance_extreme():
    """Reading R1 + R6: he2hb is homogeneous, he2hb(s A) = (s Band, V, tau),
    with s = 2^k exactly representable, so every stage except beta's norm is
    bitwise scaled; with LAPACK's scaled norms the result holds at s = 2^-1000
    (entries ~1e-302, |x|^2 underflows) and s = 2^700 (|x|^2 overflows)."""
    n, nb = 40, 6
    A = synth.rand_hermitian(n, 5)
    A1, t1 = oracle.he2hb(A, nb)
    r, c = np.indices((n, n))
    band = (r - c >= 0) & (r - c <= nb)
    below = r - c > nb
    for k in (-1000, 700):
        s = 2.0 ** k
        As, ts = oracle.he2hb(A * s, nb)
        assert np.all(np.isfinite(As))
        assert np.max(np.abs(ts - t1)) <= 64 * EPS
        assert np.max(np.abs(As[below] - A1[below])) <= 64 * n * EPS * np.max(np.abs(A1[below]))
        assert np.max(np.abs(As[band] / s - A1[band])) <= 64 * n * EPS * np.max(np.abs(A1[band]))


def test_he2hb_oracle_degenerate_cases():
    # n=4, b=3 -> unchanged up to the phase of A[3,0] (reading R3)
    A = synth.rand_hermitian(4, 1)
    A_out, tau = oracle.he2hb(A, 3)
    assert np.allclose(np.diag(A_out), np.diag(A))
    assert abs(abs(A_out[3, 0]) - abs(A[3, 0])) < 1e-15
    # real entries: the 1-row panel's reflector is H = I or a sign flip
    # (zlarfg: tau = 0 iff Im(alpha) = 0 and x = 0), so the band is unchanged
    # up to the sign of A[3,0]
    Ar = A.real.astype(complex)
    A_out, tau = oracle.he2hb(Ar, 3)
    assert np.all(tau == 0)
    assert np.array_equal(np.tril(A_out), np.tril(Ar))
    # diagonal input -> unchanged, all tau = 0 (zero column -> tau = 0)
    D = np.diag(synth.uniform(2, 2, 20)).astype(complex)
    A_out, tau = oracle.he2hb(D, 4)
    assert np.allclose(A_out, D, atol=0) and np.all(tau == 0)


def test_larft_matches_reflector_product():
    m, k = 30, 8
    V = np.tril(synth.cnormal(2, 3, (m, k)), -1)
    for j in range(k):
        V[j, j] = 1
    tau = np.array([oracle.larfg(1.0 + 0.2j * t, synth.cnormal(5, t, (3,)))[1] for t in range(k)])
    T = oracle.larft(V, tau)
    P = np.eye(m, dtype=complex)
    for j in range(k):
        P = P @ (np.eye(m) - tau[j] * np.outer(V[:, j], V[:, j].conj()))
    assert np.linalg.norm(P - (np.eye(m) - V @ T @ V.conj().T)) < 1e-13 * np.linalg.norm(P)
    assert np.allclose(np.tril(T, -1), 0) and np.allclose(np.diag(T), tau)


def test_apply_q1_matches_explicit_q():
    n, nb, m = 40, 6, 5
    A = synth.rand_hermitian(n, 11)
    A_out, tau = oracle.he2hb(A, nb)
    Q = _q1_explicit(A_out, tau, nb)
    E = synth.cnormal(1, 2, (n, m))
    assert np.linalg.norm(oracle.apply_q1(A_out, tau, nb, E) - Q @ E) < 1e-13


# --------------------------------------------------------------- hb2st (R5) and Q2
def _q2_explicit(V2, tau2, n, nb):
    offs, _ = synth.v2_layout(n, nb)
    Q = np.eye(n, dtype=complex)
    for i in range(n - 1):
        j = 0
        while 1 + i + j * nb <= n - 1:
            r0 = i + 1 + j * nb
            slot = offs[j] + i
            r1 = min(i + (j + 1) * nb, n - 1)
            v = np.zeros(n, dtype=complex)
            v[r0:r1 + 1] = V2[slot, :r1 - r0 + 1]
            Q = Q @ (np.eye(n) - tau2[slot] * np.outer(v, v.conj()))
            j += 1
    return Q


@pytest.mark.parametrize("n,nb", [(40, 4), (45, 6), (30, 1), (24, 8)])
def test_hb2st_oracle_tridiagonal_and_unitary(n, nb):
    A = synth.rand_hermitian(n, 3 * n + nb)
    A_out, _ = oracle.he2hb(A, nb)
    Band = _band_of(A_out, nb)
    d, e, V2, tau2 = oracle.hb2st(Band, nb)
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    Q2 = _q2_explicit(V2, tau2, n, nb)
    assert np.linalg.norm(Q2.conj().T @ Q2 - np.eye(n)) <= 50 * n * EPS
    assert np.linalg.norm(Q2.conj().T @ Band @ Q2 - T) <= 50 * n * EPS * np.linalg.norm(Band)
    assert rel_eig_err(oracle.sturm_values(d, e), np.linalg.eigvalsh(A)) < 1e-13


def test_apply_q2_matches_explicit_and_order_matters():
    n, nb, m = 37, 5, 4
    V2, tau2 = synth.synthetic_v2(n, nb, 3)
    E = synth.cnormal(3, 9, (n, m))
    Q2 = _q2_explicit(V2, tau2, n, nb)
    assert np.linalg.norm(Q2.conj().T @ Q2 - np.eye(n)) < 1e-12
    assert np.linalg.norm(oracle.apply_q2(V2, tau2, nb, E) - Q2 @ E) < 1e-12
    # negative: the reverse product (first reflector applied first) differs
    offs, _ = synth.v2_layout(n, nb)
    Er = E.copy()
    for i in range(n - 1):                 # wrong order: H_{0,0} applied first
        j = 0
        while 1 + i + j * nb <= n - 1:
            r0, r1 = i + 1 + j * nb, min(i + (j + 1) * nb, n - 1)
            s = offs[j] + i
            v = V2[s, :r1 - r0 + 1]
            Er[r0:r1 + 1] -= tau2[s] * np.outer(v, v.conj() @ Er[r0:r1 + 1])
            j += 1
    assert np.linalg.norm(Er - Q2 @ E) > 1e-3


def test_two_stage_oracle_pipeline_eigenvectors():
    """he2hb -> hb2st -> tql2 -> Q2 -> Q1: eigenvectors of A (standard problem)."""
    n, nb = 36, 5
    A = synth.rand_hermitian(n, 77)
    A_out, tau = oracle.he2hb(A, nb)
    d, e, V2, tau2 = oracle.hb2st(_band_of(A_out, nb), nb)
    w, Y, info = oracle.tql2(d, e)
    assert info == 0
    E = oracle.apply_q1(A_out, tau, nb, oracle.apply_q2(V2, tau2, nb, Y.astype(complex)))
    assert np.linalg.norm(A @ E - E * w) < 1e-12 * np.linalg.norm(A)
    assert np.linalg.norm(E.conj().T @ E - np.eye(n)) < 1e-12
    assert np.max(np.abs(w - np.linalg.eigvalsh(A))) < 1e-13
