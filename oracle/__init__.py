"""CPU oracle for arXiv 1207.1773 — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_1207_1773_b200``) never imports it and shares no code
with it.  The arithmetic lives in ``oracle/oracle.c`` (plain C99 complex,
binary64); this module only loads the shared library with ctypes and
marshals numpy arrays (complex128 / float64, Fortran order).

Every function cites the PAPER.md passage it follows (see oracle.c's header).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

CFLAGS = ["-O2", "-std=gnu11", "-fPIC", "-shared", "-fopenmp", "-fno-fast-math", "-ffp-contract=off"]


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so with gcc (plain -O2, no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        P, I = C.c_void_p, C.c_int64
        sig = {
            "orc_potrf": (I, [I, P, I]),
            "orc_backsub_lh": (None, [I, I, P, I, P, I]),
            "orc_std_form": (None, [I, P, I, P, I, P, I]),
            "orc_hetd2": (None, [I, P, I, P, P, P]),
            "orc_apply_hetd2_q": (None, [I, I, P, I, P, P, I]),
            "orc_tql2": (I, [I, P, P, P, I]),
            "orc_sturm_values": (None, [I, P, P, I, I, P]),
            "orc_jacobi": (I, [I, P, I, P, P, I]),
            "orc_solve_gen": (I, [I, P, I, P, I, I, I, P, P, I]),
            "orc_he2hb": (None, [I, I, P, I, P]),
            "orc_he2hb_partial": (None, [I, I, P, I, P, I]),
            "orc_larft": (None, [I, I, P, I, P, P, I]),
            "orc_apply_q1": (None, [I, I, I, P, I, P, P, I]),
            "orc_v2_slots": (I, [I, I]),
            "orc_hb2st": (None, [I, I, P, I, P, P, P, P]),
            "orc_apply_q2": (None, [I, I, I, P, P, P, I]),
            "orc_larfg": (None, [I, P, P, I, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _z(a):
    a = np.asfortranarray(np.asarray(a, dtype=np.complex128))
    return a


def _d(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def full_hermitian(A_lower):
    """Full Hermitian matrix from the lower triangle (imag(diag) ignored)."""
    A = np.tril(np.asarray(A_lower, dtype=np.complex128))
    A = A + np.tril(A, -1).conj().T
    A[np.diag_indices_from(A)] = A.diagonal().real
    return A


# ---------------------------------------------------------------- Algorithm 1
def potrf(B):
    """Step 1: returns (L, info). info = n+j+1 if minor j+1 not PD."""
    L = _z(B).copy(order="F")
    n = L.shape[0]
    info = lib().orc_potrf(n, _p(L), n)
    return L, int(info)


def std_form(A, L):
    """Step 2: C = L^-1 A L^-H by explicit solves (reading R2)."""
    A = _z(A)
    L = _z(L)
    n = A.shape[0]
    Cm = np.zeros((n, n), dtype=np.complex128, order="F")
    lib().orc_std_form(n, _p(A), n, _p(L), n, _p(Cm), n)
    return Cm


def backsub_lh(L, X):
    """Step 4: X <- L^-H X."""
    L = _z(L)
    X = _z(X).copy(order="F")
    n, m = X.shape
    lib().orc_backsub_lh(n, m, _p(L), n, _p(X), n)
    return X


def hetd2(Cm):
    """Algorithm 2 step 1, one stage: returns (d, e, Cref, tau)."""
    Cm = _z(Cm).copy(order="F")
    n = Cm.shape[0]
    d = np.zeros(n)
    e = np.zeros(max(n, 1))
    tau = np.zeros(max(n, 1), dtype=np.complex128)
    lib().orc_hetd2(n, _p(Cm), n, _p(d), _p(e), _p(tau))
    return d, e[: max(n - 1, 0)].copy(), Cm, tau


def apply_hetd2_q(Cref, tau, Y):
    """Algorithm 2 step 3, one stage: Y <- Q Y."""
    Y = _z(Y).copy(order="F")
    n, m = Y.shape
    lib().orc_apply_hetd2_q(n, m, _p(_z(Cref)), n, _p(_z(tau)), _p(Y), n)
    return Y


def tql2(d, e, Z=None):
    """Algorithm 2 step 2: QL with implicit shifts.  Returns (w, Z, info)."""
    d = _d(d).copy()
    n = d.shape[0]
    ee = np.zeros(max(n, 1))
    ee[: n - 1] = e[: n - 1]
    Z = np.eye(n, order="F") if Z is None else np.asfortranarray(np.asarray(Z, dtype=np.float64)).copy(order="F")
    info = lib().orc_tql2(n, _p(d), _p(ee), _p(Z), n)
    return d, Z, int(info)


def sturm_values(d, e, il=1, iu=None):
    """Eigenvalues il..iu (1-based) of tridiagonal (d, e) by Sturm bisection."""
    d = _d(d)
    n = d.shape[0]
    iu = n if iu is None else iu
    ee = np.zeros(max(n, 1))
    ee[: n - 1] = e[: n - 1]
    w = np.zeros(iu - il + 1)
    lib().orc_sturm_values(n, _p(d), _p(ee), il, iu, _p(w))
    return w


def jacobi(A):
    """Cyclic complex Jacobi on full Hermitian A (n <= 512).  Returns (w, V)."""
    A = _z(A).copy(order="F")
    n = A.shape[0]
    w = np.zeros(n)
    V = np.zeros((n, n), dtype=np.complex128, order="F")
    sweeps = lib().orc_jacobi(n, _p(A), n, _p(w), _p(V), n)
    if sweeps < 0:
        raise RuntimeError("jacobi did not converge")
    return w, V


def solve_gen(A, B, il=1, iu=None):
    """Algorithm 1 + one-stage Algorithm 2.

    A, B: lower triangles read.  Returns (w_all, Z, info, L)."""
    A = _z(A)
    L = _z(B).copy(order="F")
    n = A.shape[0]
    iu = n if iu is None else iu
    m = iu - il + 1
    w = np.zeros(n)
    Z = np.zeros((n, m), dtype=np.complex128, order="F")
    info = lib().orc_solve_gen(n, _p(A), n, _p(L), n, il, iu, _p(w), _p(Z), n)
    return w, Z, int(info), L


# ------------------------------------------------------- two-stage references
def larfg(alpha, x):
    """LAPACK zlarfg convention (reading R1).  Returns (beta, tau, v)."""
    x = _z(np.atleast_1d(x)).copy()
    a = np.array([alpha], dtype=np.complex128)
    t = np.zeros(1, dtype=np.complex128)
    m = x.shape[0] + 1
    lib().orc_larfg(m, _p(a), _p(x), 1, _p(t))
    return a[0].real, t[0], np.concatenate([[1.0 + 0j], x])


def he2hb(A_full, nb):
    """Reduction to band, one reflector at a time.

    A_full: full Hermitian n x n.  Returns (A_out, tau) in the he2hb layout
    (band in 0 <= r-c <= nb, V below it, tau[k*nb + j])."""
    A = _z(A_full).copy(order="F")
    n = A.shape[0]
    tau = np.zeros(max(n, 1), dtype=np.complex128)
    lib().orc_he2hb(n, nb, _p(A), n, _p(tau))
    return A, tau


def he2hb_partial(A_full, nb, max_reflectors):
    """orc_he2hb stopped after max_reflectors reflectors (bench CPU sample)."""
    A = _z(A_full).copy(order="F")
    n = A.shape[0]
    tau = np.zeros(max(n, 1), dtype=np.complex128)
    lib().orc_he2hb_partial(n, nb, _p(A), n, _p(tau), max_reflectors)
    return A, tau


def larft(V, tau):
    """T with H_0...H_{k-1} = I - V T V^H (forward, columnwise)."""
    V = _z(V)
    m, k = V.shape
    T = np.zeros((k, k), dtype=np.complex128, order="F")
    lib().orc_larft(m, k, _p(V), m, _p(_z(tau)), _p(T), k)
    return T


def apply_q1(A_he2hb, tau, nb, E):
    """E <- Q1 E, one reflector at a time."""
    E = _z(E).copy(order="F")
    n, m = E.shape
    lib().orc_apply_q1(n, nb, m, _p(_z(A_he2hb)), n, _p(_z(tau)), _p(E), n)
    return E


def v2_slots(n, nb):
    return int(lib().orc_v2_slots(n, nb))


def hb2st(Band_full, nb):
    """Column-wise bulge chase on a dense copy.  Returns (d, e, V2, tau2)."""
    M = _z(Band_full).copy(order="F")
    n = M.shape[0]
    slots = v2_slots(n, nb)
    d = np.zeros(n)
    e = np.zeros(max(n - 1, 1))
    V2 = np.zeros(max(slots, 1) * nb, dtype=np.complex128)
    tau2 = np.zeros(max(slots, 1), dtype=np.complex128)
    lib().orc_hb2st(n, nb, _p(M), n, _p(d), _p(e), _p(V2), _p(tau2))
    return d, e[: max(n - 1, 0)], V2[: slots * nb].reshape(slots, nb), tau2[:slots]


def apply_q2(V2, tau2, nb, E):
    """E <- Q2 E, one reflector at a time, last first."""
    E = _z(E).copy(order="F")
    n, m = E.shape
    V2 = np.ascontiguousarray(np.asarray(V2, dtype=np.complex128))
    lib().orc_apply_q2(n, nb, m, _p(V2), _p(_z(tau2)), _p(E), n)
    return E
