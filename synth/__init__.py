"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and
bench.py.  Holds none of the method's arithmetic (no Cholesky, no reduction,
no back-transform): only a counter-based RNG and the pencil / reflector-set
recipes stated in DESIGN.md "Input recipe".

RNG: SplitMix64 over a 64-bit counter keyed by (seed, stream); the value at
counter c is independent of how many values were drawn before, so any slice
can be regenerated exactly.
"""
from __future__ import annotations

import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_G = np.uint64(0x9E3779B97F4A7C15)


def _mix(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * _M1
    z = z ^ (z >> np.uint64(27))
    z = z * _M2
    return z ^ (z >> np.uint64(31))


def _key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        k = _mix(np.array([(seed * 0x632BE59BD9B4E019 + stream * 0x8CB92BA72F3D8DD7 + 1) & 0xFFFFFFFFFFFFFFFF],
                          dtype=np.uint64))[0]
    return k


def uniform(seed: int, stream: int, count: int, start: int = 0) -> np.ndarray:
    """count uniforms in (0, 1] from counter start.. of (seed, stream)."""
    with np.errstate(over="ignore"):
        c = np.arange(start, start + count, dtype=np.uint64)
        z = _mix(_key(seed, stream) + c * _G)
    return ((z >> np.uint64(11)).astype(np.float64) + 1.0) * (1.0 / 9007199254740992.0)


def cnormal(seed: int, stream: int, shape, chunk: int = 1 << 24, start: int = 0) -> np.ndarray:
    """Complex N(0, 1/2) + i N(0, 1/2) entries, Fortran order (Box-Muller).
    `start` offsets the element counter (a column slice of a larger matrix)."""
    count = int(np.prod(shape))
    out = np.empty(count, dtype=np.complex128)
    for s in range(0, count, chunk):
        k = min(chunk, count - s)
        u = uniform(seed, stream, 2 * k, 2 * (s + start))
        r = np.sqrt(-np.log(u[0::2]))
        th = 2.0 * np.pi * u[1::2]
        out[s:s + k] = r * np.cos(th) + 1j * (r * np.sin(th))
    return out.reshape(shape, order="F")


def rnormal(seed: int, stream: int, shape, start: int = 0) -> np.ndarray:
    """Real N(0,1) entries, Fortran order."""
    return np.sqrt(2.0) * cnormal(seed, stream, shape, start=start).real


def hermitian_full(M: np.ndarray) -> np.ndarray:
    H = 0.5 * (M + M.conj().T)
    H[np.diag_indices_from(H)] = H.diagonal().real
    return np.asfortranarray(H)


# ------------------------------------------------------------------ pencils
def rand_hermitian(n: int, seed: int = 0, stream: int = 1) -> np.ndarray:
    """G1 A: (G + G^H) / (2 sqrt n): semicircle spectrum on [-sqrt2, sqrt2]."""
    G = cnormal(seed, stream, (n, n))
    A = (G + G.conj().T) / (2.0 * np.sqrt(n))
    A[np.diag_indices_from(A)] = A.diagonal().real
    return np.asfortranarray(A)


def random_reflectors(n: int, r: int, seed: int, stream: int):
    """r random Householder reflectors H = I - 2 u u^H (unit u)."""
    U = cnormal(seed, stream, (n, r))
    U /= np.linalg.norm(U, axis=0, keepdims=True)
    return U


def apply_reflectors_congruence(M: np.ndarray, U: np.ndarray) -> np.ndarray:
    """M <- H_r^H ... H_1^H M H_1 ... H_r with H_t = I - 2 u_t u_t^H."""
    M = np.array(M, dtype=np.complex128, order="F")
    for t in range(U.shape[1]):
        u = U[:, t:t + 1]
        M -= 2.0 * u @ (u.conj().T @ M)
        M -= 2.0 * (M @ u) @ u.conj().T
    return hermitian_full(M)


def hpd_with_condition(n: int, kappa: float, seed: int = 0, stream: int = 2, r: int | None = None) -> np.ndarray:
    """G1 B = U^H diag(kappa^(k/(n-1))) U, exact kappa_2(B) = kappa."""
    r = r if r is not None else min(n, 32)
    d = kappa ** (np.arange(n) / max(n - 1, 1))
    U = random_reflectors(n, r, seed, stream)
    return apply_reflectors_congruence(np.diag(d).astype(np.complex128), U)


def pencil_rand(n: int, seed: int = 0, kappa: float = 1e2):
    """G1 'rand' pencil (A, B), full Hermitian matrices."""
    return rand_hermitian(n, seed, 1), hpd_with_condition(n, kappa, seed, 2)


def pencil_known(n: int, seed: int = 0, kappa: float = 1e2, clustered: bool = True):
    """G2 'known spectrum' (pin P5): B = P P^H, A = P W^H D W P^H with
    P = U^H diag(sqrt s) U, so lambda(A, B) = D exactly.  Returns (A, B, D)."""
    if clustered:
        k = max(1, n // 5)
        base = np.sort(uniform(seed, 10, n)) * 2.0 - 1.0
        D = base.copy()
        # lowest 20%: clusters of 1-4 near-degenerate values spaced 1e-8
        i = 0
        while i < k:
            size = 1 + (i % 4)
            for t in range(size):
                if i + t < k:
                    D[i + t] = D[i] + 1e-8 * t
            i += size
        D = np.sort(D)
    else:
        D = np.sort(uniform(seed, 10, n) * 2.0 - 1.0)
    U = random_reflectors(n, min(n, 32), seed, 11)
    W = random_reflectors(n, min(n, 32), seed, 12)
    s = kappa ** (np.arange(n) / max(n - 1, 1))
    # P = U^H diag(sqrt s) U  (Hermitian PD)
    P = apply_reflectors_congruence(np.diag(np.sqrt(s)).astype(np.complex128), U)
    Cw = apply_reflectors_congruence(np.diag(D).astype(np.complex128), W)   # W^H D W
    A = hermitian_full(P @ Cw @ P.conj().T)
    B = hermitian_full(P @ P.conj().T)
    return A, B, D


def known_hermitian(n: int, seed: int = 0, r: int = 8):
    """Standard Hermitian matrix with an exactly known spectrum:
    A = W^H diag(D) W, W a product of r random reflectors, D sorted U(-1, 1)
    with 10% of the values in near-degenerate pairs (spacing 1e-9).
    Returns (A full, D ascending)."""
    D = np.sort(uniform(seed, 70, n) * 2.0 - 1.0)
    k = n // 10
    D[1:2 * k:2] = D[0:2 * k - 1:2] + 1e-9
    D = np.sort(D)
    W = random_reflectors(n, min(n, r), seed, 71)
    return apply_reflectors_congruence(np.diag(D).astype(np.complex128), W), D


def fem_pencil(n: int, seed: int = 0):
    """G4 (pin P6): K = tridiag(-1,2,-1), M = tridiag(1/6,2/3,1/6) under a
    unitary congruence; lambda_k = 6(1-cos t_k)/(2+cos t_k), t_k = k pi/(n+1)."""
    K = np.diag(np.full(n, 2.0)) - np.diag(np.ones(n - 1), 1) - np.diag(np.ones(n - 1), -1)
    M = np.diag(np.full(n, 2.0 / 3.0)) + np.diag(np.full(n - 1, 1 / 6.0), 1) + np.diag(np.full(n - 1, 1 / 6.0), -1)
    U = random_reflectors(n, min(n, 16), seed, 20)
    A = apply_reflectors_congruence(K.astype(np.complex128), U)
    B = apply_reflectors_congruence(M.astype(np.complex128), U)
    th = np.arange(1, n + 1) * np.pi / (n + 1)
    lam = 6.0 * (1.0 - np.cos(th)) / (2.0 + np.cos(th))
    return A, B, np.sort(lam)


# ------------------------------------------------- hot-path synthetic inputs
def unit_lower(n: int, seed: int = 0, stream: int = 30, offscale: float = 0.5) -> np.ndarray:
    """Well-conditioned lower-triangular L with real positive diagonal in
    [1, 2] and strictly-lower entries N(0, offscale^2/n) (bench / trsm input)."""
    L = np.tril(cnormal(seed, stream, (n, n)) * (offscale / np.sqrt(n)), -1)
    L[np.diag_indices(n)] = 1.0 + uniform(seed, stream + 1, n)
    return np.asfortranarray(L)


def real_orthonormalish(n: int, m: int, seed: int = 0, stream: int = 40, col0: int = 0) -> np.ndarray:
    """Real n x m matrix with N(0, 1/n) entries (stand-in for tridiagonal
    eigenvectors Z in the timed step; columns have norm ~1).  col0 selects
    columns col0..col0+m-1 of the same global matrix (column slices)."""
    return np.asfortranarray(rnormal(seed, stream, (n, m), start=col0 * n) / np.sqrt(n))


def synthetic_v1(n: int, nb: int, seed: int = 0, stream: int = 60):
    """Random exactly-unitary reflectors in the he2hb layout (band entries
    untouched, v tails below the band, tau = (1+e^{i theta})/|v|^2): the shape
    of the Q1 workload for the CPU baseline sample.  Returns (A, tau)."""
    A = np.asfortranarray(cnormal(seed, stream, (n, n)) / np.sqrt(n))
    tau = np.zeros(max(n, 1), dtype=np.complex128)
    th = 2.0 * np.pi * uniform(seed, stream + 1, n)
    i = 0
    while i + nb < n:
        for j in range(min(nb, n - i - nb)):
            r0 = i + nb + j
            nrm2 = 1.0 + np.sum(np.abs(A[r0 + 1:, i + j]) ** 2)
            tau[i + j] = (1.0 + np.exp(1j * th[i + j])) / nrm2
        i += nb
    return A, tau


def v2_layout(n: int, nb: int):
    """Slot table of the Q2 reflector layout (include/eig.h, EIG V2 layout):
    returns (offsets[j], lengths per slot) for steps j with n-1-j*nb > 0."""
    offs = []
    off = 0
    j = 0
    while 1 + j * nb <= n - 1:
        offs.append(off)
        off += n - 1 - j * nb
        j += 1
    return np.array(offs, dtype=np.int64), off


def synthetic_v2(n: int, nb: int, seed: int = 0, stream: int = 50):
    """Random unitary reflectors in the V2 layout: slot (j, i) acts on rows
    i+1+j*nb .. min(i+(j+1)*nb, n-1); v[0] = 1, v[1:len] ~ N(0, 1/len),
    zero padding to nb; tau = (1 + e^{i theta}) / |v|^2 (H exactly unitary).
    Returns (V2 [slots, nb] complex, tau2 [slots] complex)."""
    offs, slots = v2_layout(n, nb)
    V2 = np.zeros((slots, nb), dtype=np.complex128)
    tau2 = np.zeros(slots, dtype=np.complex128)
    R = cnormal(seed, stream, (slots, nb), chunk=1 << 22)
    th = 2.0 * np.pi * uniform(seed, stream + 1, slots)
    for j, off in enumerate(offs):
        cnt = n - 1 - j * nb
        i = np.arange(cnt)
        r0 = i + 1 + j * nb
        r1 = np.minimum(i + (j + 1) * nb, n - 1)
        ln = r1 - r0 + 1
        block = R[off:off + cnt]
        mask = np.arange(nb)[None, :] < ln[:, None]
        block = np.where(mask, block / np.sqrt(np.maximum(ln, 1))[:, None], 0)
        block[:, 0] = 1.0
        V2[off:off + cnt] = block
        nrm2 = np.sum(np.abs(block) ** 2, axis=1)
        tau2[off:off + cnt] = (1.0 + np.exp(1j * th[off:off + cnt])) / nrm2
    return V2, tau2
