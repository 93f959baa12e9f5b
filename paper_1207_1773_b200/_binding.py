"""Thin ctypes binding of include/eig.h (argument marshalling only).

Every step of the hot path runs in libeigb200.so's CUDA kernels; this module
only converts torch tensors to (pointer, leading dimension) pairs.  torch is
used for device memory and streams.  There is no CPU fallback: if the
extension or the GPU is missing, every call raises.

Matrices are column-major: a math m x n matrix is a torch tensor of shape
(m, n) with strides (1, ld), ld >= m (see ``colmajor`` / ``empty_colmajor``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# EIG_LIB overrides the library path (A/B profiling of two builds only)
_SO = os.environ.get("EIG_LIB") or os.path.join(_HERE, "libeigb200.so")

EIG_RANGE_ALL, EIG_RANGE_FRACTION, EIG_RANGE_INDEX = 0, 1, 2
EIG_HOST_BUFFERS = 1
EIG_SKIP_HE2HB = 2
EIG_SKIP_BT = 4
EIG_GATHER_Z = 1          # eig_config.flags
EIG_USE_3M = 2
EIG_NO_3M = 4
EIG_DIST_HE2HB = 8
STAGES = ["potrf", "hegst", "he2hb", "hb2st", "stedc", "wait", "q2", "q1", "trsm", "bt", "gather", "total"]

_lib = None


class EigError(RuntimeError):
    pass


class _Config(C.Structure):
    _fields_ = [("device", C.c_int), ("nb", C.c_int), ("q2_group", C.c_int), ("stream", C.c_void_p),
                ("rank", C.c_int), ("nranks", C.c_int), ("nccl_id", C.c_void_p), ("n_max", C.c_int64),
                ("flags", C.c_uint)]


class _Stats(C.Structure):
    _fields_ = [("seconds", C.c_double * len(STAGES)), ("flops", C.c_double * len(STAGES)), ("m", C.c_int64),
                ("col_lo", C.c_int64), ("col_hi", C.c_int64), ("bytes_comm", C.c_int64), ("rank", C.c_int),
                ("nranks", C.c_int)]

    def to_dict(self):
        return {"seconds": {k: self.seconds[i] for i, k in enumerate(STAGES)},
                "flops": {k: self.flops[i] for i, k in enumerate(STAGES)}, "m": self.m,
                "cols": (self.col_lo, self.col_hi), "bytes_comm": self.bytes_comm, "rank": self.rank,
                "nranks": self.nranks}


def lib():
    """Load libeigb200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise EigError(f"{_SO} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(_SO)
        P, I, D, U = C.c_void_p, C.c_int64, C.c_double, C.c_uint
        h = C.c_void_p
        sig = {
            "eig_init": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(_Config)]),
            "eig_finalize": (C.c_int, [h]),
            "eig_strerror": (C.c_char_p, [C.c_int]),
            "eig_last_cuda_error": (C.c_char_p, [h]),
            "eig_launch_count": (I, [h]),
            "eig_sync": (C.c_int, [h]),
            "eig_num_panels": (I, [I, C.c_int]),
            "eig_v2_slots": (I, [I, C.c_int]),
            "eig_he2hb": (C.c_int, [h, I, P, I, P, P]),
            "eig_apply_q1": (C.c_int, [h, I, P, I, P, P, I, I]),
            "eig_apply_q2": (C.c_int, [h, I, P, P, P, I, P, I, I]),
            "eig_trsm_lh": (C.c_int, [h, I, P, I, P, I, I]),
            "eig_hotpath": (C.c_int, [h, I, P, I, P, P, P, P, P, I, P, I, P, I, I, U]),
            "eig_zgemm": (C.c_int, [h, C.c_char, C.c_char, I, I, I, D, P, I, P, I, D, P, I, C.c_int, C.c_int]),
            "eig_solve_gen": (C.c_int, [h, I, P, I, P, I, C.c_int, D, I, I, P, P, I, P, P]),
            "eig_get_unique_id": (C.c_int, [P]),
            "eig_he2hb_sim": (C.c_int, [h, I, C.c_int, P, I, P, P]),
            "eig_column_slice": (C.c_int, [I, C.c_int, C.c_int, C.POINTER(I), C.POINTER(I)]),
            "eig_resolve_range": (C.c_int, [I, C.c_int, D, I, I, C.POINTER(I), C.POINTER(I), C.POINTER(I)]),
            "eig_last_stats": (C.c_int, [h, P]),
            "eig_debug_q2_profile": (C.c_int, [h, P]),
            "eig_hb2st": (C.c_int, [h, I, P, I, P, P, P, P]),
            "eig_stedc": (C.c_int, [h, I, P, P, I, I, P, P, I]),
            "eig_potrf": (C.c_int, [h, I, P, I]),
            "eig_hegst": (C.c_int, [h, I, P, I, P, I]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return ["eig_init", "eig_finalize", "eig_strerror", "eig_last_cuda_error", "eig_launch_count", "eig_sync",
            "eig_num_panels", "eig_v2_slots", "eig_he2hb", "eig_apply_q1", "eig_apply_q2", "eig_trsm_lh",
            "eig_hotpath", "eig_zgemm", "eig_solve_gen", "eig_debug_q2_profile", "eig_hb2st", "eig_stedc", "eig_potrf",
            "eig_hegst", "eig_get_unique_id", "eig_column_slice", "eig_resolve_range", "eig_last_stats",
            "eig_he2hb_sim"]


def unique_id() -> bytes:
    """128-byte NCCL unique id (eig_get_unique_id; host-only, call on rank 0)."""
    buf = C.create_string_buffer(128)
    rc = lib().eig_get_unique_id(C.cast(buf, C.c_void_p))
    if rc:
        raise EigError(f"eig_get_unique_id rc={rc}: {lib().eig_strerror(rc).decode()}")
    return buf.raw


def column_slice(m: int, rank: int, nranks: int):
    """Columns [lo, hi) of m owned by `rank` in the collective calls (eig_column_slice)."""
    lo, hi = C.c_int64(0), C.c_int64(0)
    rc = lib().eig_column_slice(m, rank, nranks, C.byref(lo), C.byref(hi))
    if rc:
        raise EigError(f"eig_column_slice rc={rc}")
    return lo.value, hi.value


def resolve_range(n: int, fraction=None, il=None, iu=None):
    """(il, iu, m) exactly as eig_solve_gen selects them (eig_resolve_range)."""
    rng, f, a, b = _range_args(fraction, il, iu)
    o = [C.c_int64(0) for _ in range(3)]
    rc = lib().eig_resolve_range(n, rng, f, a, b, *[C.byref(x) for x in o])
    if rc:
        raise EigError(f"eig_resolve_range rc={rc}")
    return tuple(x.value for x in o)


def _range_args(fraction, il, iu):
    if fraction is not None:
        return EIG_RANGE_FRACTION, float(fraction), 0, 0
    if il is not None:
        return EIG_RANGE_INDEX, 0.0, int(il), int(iu)
    return EIG_RANGE_ALL, 0.0, 0, 0


def num_panels(n: int, nb: int) -> int:
    return int(lib().eig_num_panels(n, nb))


def v2_slots(n: int, nb: int) -> int:
    return int(lib().eig_v2_slots(n, nb))


# ------------------------------------------------------------ layout helpers
def empty_colmajor(rows, cols, dtype=torch.complex128, device="cuda", ld=None):
    ld = rows if ld is None else ld
    return torch.empty((cols, ld), dtype=dtype, device=device).t()[:rows]


def colmajor(x: torch.Tensor, device=None) -> torch.Tensor:
    """Column-major (Fortran) copy of a 2-D tensor or numpy array."""
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    if x.dim() == 1:
        x = x[:, None]
    y = x.t().contiguous().t()
    return y.to(device) if device is not None else y


def _ld(x: torch.Tensor) -> int:
    if x.dim() != 2:
        raise EigError("expected a 2-D column-major tensor")
    if x.stride(0) != 1 and x.numel() > 1:
        raise EigError("tensor is not column-major (stride(0) must be 1); use colmajor()")
    return max(x.stride(1) if x.shape[1] > 1 else x.shape[0], 1)


def _ptr(x):
    return None if x is None else C.c_void_p(x.data_ptr())


class Solver:
    """One library handle (eig_init) bound to a CUDA device and stream."""

    def __init__(self, device: int = 0, nb: int = 64, q2_group: int = 0, stream=None, rank: int = 0,
                 nranks: int = 1, nccl_id: bytes | None = None, n_max: int = 0, flags: int = 0):
        """nccl_id (128 bytes from unique_id() on rank 0, same on every rank)
        makes the handle collective: eig_init, solve_gen and hotpath must
        then be called by all `nranks` processes (one per GPU)."""
        if not torch.cuda.is_available():
            raise EigError("no CUDA device: the B200 path has no CPU fallback")
        self.device = device
        self.nb = nb
        self.q2_group = q2_group
        self.rank, self.nranks = rank, max(1, nranks)
        self.collective = nccl_id is not None
        self.flags = flags
        torch.cuda.set_device(device)
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        self._id = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        cfg = _Config(device, nb, q2_group, C.c_void_p(stream.cuda_stream), rank, nranks,
                      C.cast(self._id, C.c_void_p) if self._id is not None else None, n_max, flags)
        h = C.c_void_p()
        self._check(lib().eig_init(C.byref(h), C.byref(cfg)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().eig_finalize(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _dv(self, x, dtype, name, min_numel=0):
        """Argument check before a pointer crosses the ABI: a device tensor of
        this handle's GPU, the dtype the C ABI expects, at least min_numel
        elements (the ABI reads raw memory and cannot check any of this)."""
        if not isinstance(x, torch.Tensor):
            raise EigError(f"{name}: expected a torch.Tensor")
        if x.device.type != "cuda" or (x.device.index or 0) != self.device:
            raise EigError(f"{name}: expected a tensor on cuda:{self.device}, got {x.device}")
        if x.dtype != dtype:
            raise EigError(f"{name}: expected {dtype}, got {x.dtype}")
        if x.numel() < min_numel:
            raise EigError(f"{name}: needs at least {min_numel} elements, has {x.numel()}")
        return x

    def _mat(self, x, name, rows, cols, dtype=torch.complex128):
        self._dv(x, dtype, name)
        if x.dim() != 2 or x.shape[0] < rows or x.shape[1] < cols:
            raise EigError(f"{name}: expected at least {rows} x {cols}, got {tuple(x.shape)}")
        return x

    def _check(self, rc):
        if rc != 0:
            msg = lib().eig_strerror(rc).decode()
            extra = ""
            if getattr(self, "h", None):
                extra = lib().eig_last_cuda_error(self.h).decode()
            raise EigError(f"eig rc={rc}: {msg} {extra}".strip())

    @property
    def launches(self) -> int:
        return int(lib().eig_launch_count(self.h))

    def q2_profile(self):
        """Cycles of CTA 0: apply_q2 phases [0:5], panel_qr phases [8:14]; needs EIG_Q2_PROFILE."""
        out = (C.c_ulonglong * 32)()
        self._check(lib().eig_debug_q2_profile(self.h, C.cast(out, C.c_void_p)))
        return list(out)

    def sync(self):
        self._check(lib().eig_sync(self.h))

    # ------------------------------------------------------------ stages
    def he2hb(self, A: torch.Tensor):
        """a1..a5: A (n x n column-major complex128, lower) -> band + V in place.
        Returns (tau [K*nb], T [K, nb, nb] column-major blocks as (K, nb*nb))."""
        n = A.shape[0]
        self._mat(A, "A", n, n)
        K = num_panels(n, self.nb)
        tau = torch.zeros(max(K * self.nb, 1), dtype=torch.complex128, device=A.device)
        T = torch.zeros(max(K * self.nb * self.nb, 1), dtype=torch.complex128, device=A.device)
        self._check(lib().eig_he2hb(self.h, n, _ptr(A), _ld(A), _ptr(tau), _ptr(T)))
        return tau, T

    def he2hb_sim(self, A: torch.Tensor, nranks: int):
        """NEXT-4: he2hb by the 1D block-cyclic distributed algorithm with
        `nranks` virtual ranks on this GPU (same outputs as he2hb)."""
        n = A.shape[0]
        self._mat(A, "A", n, n)
        K = num_panels(n, self.nb)
        tau = torch.zeros(max(K * self.nb, 1), dtype=torch.complex128, device=A.device)
        T = torch.zeros(max(K * self.nb * self.nb, 1), dtype=torch.complex128, device=A.device)
        self._check(lib().eig_he2hb_sim(self.h, n, nranks, _ptr(A), _ld(A), _ptr(tau), _ptr(T)))
        return tau, T

    def hb2st(self, A):
        """NEXT-1: band (he2hb output A) -> (d, e, V2 [slots, nb], tau2 [slots])."""
        n = A.shape[0]
        self._mat(A, "A", n, n)
        slots = v2_slots(n, self.nb)
        d = torch.zeros(max(n, 1), dtype=torch.float64, device=A.device)
        e = torch.zeros(max(n, 1), dtype=torch.float64, device=A.device)
        V2 = torch.zeros((max(slots, 1), self.nb), dtype=torch.complex128, device=A.device)
        tau2 = torch.zeros(max(slots, 1), dtype=torch.complex128, device=A.device)
        self._check(lib().eig_hb2st(self.h, n, _ptr(A), _ld(A), _ptr(d), _ptr(e), _ptr(V2), _ptr(tau2)))
        return d[:n], e[:max(n - 1, 0)], V2[:slots], tau2[:slots]

    def stedc(self, d, e, il=1, iu=None):
        """NEXT-2: tridiagonal D&C.  Returns (w [n] all eigenvalues, Z [n, iu-il+1] real)."""
        n = d.shape[0]
        self._dv(d, torch.float64, "d", n)
        self._dv(e, torch.float64, "e", max(n - 1, 0))
        iu = n if iu is None else iu
        w = torch.zeros(max(n, 1), dtype=torch.float64, device=d.device)
        Z = empty_colmajor(n, iu - il + 1, dtype=torch.float64, device=d.device)
        e_ = e if e.numel() > 0 else torch.zeros(1, dtype=torch.float64, device=d.device)
        self._check(lib().eig_stedc(self.h, n, _ptr(d), _ptr(e_), il, iu, _ptr(w), _ptr(Z), _ld(Z)))
        return w[:n], Z

    def potrf(self, B):
        """NEXT-3: B <- L (lower) in place.  Returns LAPACK-style info (0 or n + j)."""
        n = B.shape[0]
        self._mat(B, "B", n, n)
        rc = lib().eig_potrf(self.h, n, _ptr(B), _ld(B))
        if rc < 0:
            self._check(rc)
        return rc

    def hegst(self, A, L):
        """NEXT-3: A <- L^-1 A L^-H (full Hermitian storage)."""
        n = A.shape[0]
        self._mat(A, "A", n, n)
        self._mat(L, "L", n, n)
        self._check(lib().eig_hegst(self.h, n, _ptr(A), _ld(A), _ptr(L), _ld(L)))
        return A

    def solve_gen(self, A, B, fraction=None, il=None, iu=None, n=None, stats=False):
        """Algorithm 1: A x = lambda B x.  A, B device column-major complex128
        (lower read; both destroyed, B <- L).  Returns (w [n], Z [n, m]) (and
        the per-stage statistics dict if stats=True).  Raises EigError on
        failure (info n + j: B not positive definite).
        Collective handle: every rank calls it; ranks > 0 may pass A = B =
        None (then give n); Z is this rank's column slice (rank 0: all m
        columns with EIG_GATHER_Z)."""
        if n is None:
            n = A.shape[0]
        if A is not None or not self.collective or self.rank == 0:
            self._mat(A, "A", n, n)
            self._mat(B, "B", n, n)
        il_, iu_, m = resolve_range(n, fraction, il, iu)
        rng, f, a, b = _range_args(fraction, il, iu)
        lo, hi = (0, m) if not self.collective else column_slice(m, self.rank, self.nranks)
        if self.collective and self.rank == 0 and (self.flags & EIG_GATHER_Z):
            lo, hi = 0, m
        w = torch.zeros(max(n, 1), dtype=torch.float64, device=torch.device("cuda", self.device))
        Z = empty_colmajor(n, max(hi - lo, 1), device=torch.device("cuda", self.device))
        mo = C.c_int64(0)
        st = _Stats()
        rc = lib().eig_solve_gen(self.h, n, _ptr(A), _ld(A) if A is not None else n, _ptr(B),
                                 _ld(B) if B is not None else n, rng, f, a, b, _ptr(w), _ptr(Z), _ld(Z), C.byref(mo),
                                 C.byref(st))
        self._check(rc)
        out = (w[:n], Z[:, :hi - lo])
        return (*out, st.to_dict()) if stats else out

    def last_stats(self):
        """Per-stage seconds / flops of the last hotpath or solve_gen call (eig_last_stats)."""
        st = _Stats()
        self._check(lib().eig_last_stats(self.h, C.byref(st)))
        return st.to_dict()

    def apply_q1(self, A, T, E):
        n, m = E.shape
        self._mat(A, "A", n, n)
        self._mat(E, "E", n, m)
        self._dv(T, torch.complex128, "T", num_panels(n, self.nb) * self.nb * self.nb)
        self._check(lib().eig_apply_q1(self.h, n, _ptr(A), _ld(A), _ptr(T), _ptr(E), _ld(E), m))
        return E

    def apply_q2(self, V2, tau2, E, Z=None):
        n, m = E.shape
        self._mat(E, "E", n, m)
        slots = v2_slots(n, self.nb)
        self._dv(V2, torch.complex128, "V2", slots * self.nb)
        self._dv(tau2, torch.complex128, "tau2", slots)
        if Z is not None:
            self._mat(Z, "Z", n, m, torch.float64)
        ldz = _ld(Z) if Z is not None else n
        self._check(lib().eig_apply_q2(self.h, n, _ptr(V2), _ptr(tau2), _ptr(Z), ldz, _ptr(E), _ld(E), m))
        return E

    def trsm_lh(self, L, E):
        n, m = E.shape
        self._mat(L, "L", n, n)
        self._mat(E, "E", n, m)
        self._check(lib().eig_trsm_lh(self.h, n, _ptr(L), _ld(L), _ptr(E), _ld(E), m))
        return E

    def zgemm(self, opa, opb, A, B, Cm, alpha=1.0, beta=0.0, herm_a=False, lower_c=False, K=None):
        M, N = Cm.shape
        if K is None:
            K = A.shape[1] if opa == "N" else A.shape[0]
        self._mat(Cm, "C", M, N)
        self._mat(A, "A", *((M, K) if opa == "N" else (K, M)))
        self._mat(B, "B", *((K, N) if opb == "N" else (N, K)))
        self._check(lib().eig_zgemm(self.h, opa.encode(), opb.encode(), M, N, K, alpha, _ptr(A), _ld(A), _ptr(B),
                                    _ld(B), beta, _ptr(Cm), _ld(Cm), int(herm_a), int(lower_c)))
        return Cm

    def hotpath(self, A, V2, tau2, L, Z, E=None, flags=0, tau1=None, T1=None):
        """One pass of the whole hot path on device tensors:
        he2hb(A) -> E = complex(Z) -> Q2 -> Q1 -> L^-H.  Returns (E, tau1, T1).
        Collective handle: ranks > 0 pass A = V2 = tau2 = L = None; Z / E are
        every rank's own column slice."""
        n = Z.shape[0]
        m = Z.shape[1]
        self._mat(Z, "Z", n, m, torch.float64)
        slots = v2_slots(n, self.nb)
        K = num_panels(n, self.nb)
        if self.collective and self.rank != 0 and A is None:
            if E is None:
                E = empty_colmajor(n, m, device=Z.device)
            self._mat(E, "E", n, m)
            self._check(lib().eig_hotpath(self.h, n, None, n, None, None, None, None, None, n, _ptr(Z), _ld(Z),
                                          _ptr(E), _ld(E), m, flags))
            return E, None, None
        self._mat(A, "A", n, n)
        self._mat(L, "L", n, n)
        self._dv(V2, torch.complex128, "V2", slots * self.nb)
        self._dv(tau2, torch.complex128, "tau2", slots)
        if tau1 is None:
            tau1 = torch.zeros(max(K * self.nb, 1), dtype=torch.complex128, device=A.device)
        if T1 is None:
            T1 = torch.zeros(max(K * self.nb * self.nb, 1), dtype=torch.complex128, device=A.device)
        if E is None:
            E = empty_colmajor(n, m, device=A.device)
        self._mat(E, "E", n, m)
        self._dv(tau1, torch.complex128, "tau1", K * self.nb)
        self._dv(T1, torch.complex128, "T1", K * self.nb * self.nb)
        self._check(lib().eig_hotpath(self.h, n, _ptr(A), _ld(A), _ptr(tau1), _ptr(T1), _ptr(V2), _ptr(tau2),
                                      _ptr(L), _ld(L), _ptr(Z), _ld(Z), _ptr(E), _ld(E), m, flags))
        return E, tau1, T1

    def hotpath_host(self, A: np.ndarray, V2: np.ndarray, tau2: np.ndarray, L: np.ndarray, Z: np.ndarray,
                     E: np.ndarray):
        """Same pass through the C ABI with HOST buffers (EIG_HOST_BUFFERS):
        copies in, runs, copies E out, synchronously.  Arrays must be
        Fortran-ordered (column-major); pinned memory is recommended."""
        n = A.shape[0]
        m = Z.shape[1]
        for name, x, dt in (("A", A, np.complex128), ("L", L, np.complex128), ("Z", Z, np.float64),
                            ("E", E, np.complex128), ("V2", V2, np.complex128), ("tau2", tau2, np.complex128)):
            if x.dtype != dt:
                raise EigError(f"{name} must be {np.dtype(dt).name}, got {x.dtype}")
            if x.ndim == 2 and not x.flags.f_contiguous and x.shape[1] > 1 and name != "V2":
                raise EigError(f"{name} must be Fortran-ordered")
        slots = v2_slots(n, self.nb)
        if V2.size < slots * self.nb or tau2.size < slots or not V2.flags.c_contiguous:
            raise EigError("V2 / tau2 too small or not contiguous")
        if A.shape != (n, n) or L.shape != (n, n) or Z.shape[0] != n or E.shape != (n, m):
            raise EigError("host buffer shapes do not match n, m")

        def hp(x):
            return C.c_void_p(x.ctypes.data)

        self._check(lib().eig_hotpath(self.h, n, hp(A), n, None, None, hp(V2), hp(tau2), hp(L), n, hp(Z), n,
                                      hp(E), n, m, EIG_HOST_BUFFERS))
        return E
