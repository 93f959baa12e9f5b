"""B200-native (sm_100a) hot path of the two-stage Hermitian generalized
eigensolver of arXiv 1207.1773: he2hb (panel QR, T factor, two-sided update)
and the eigenvector back-transform E = L^-H Q1 (Q2 Z).

All compute runs in ``libeigb200.so`` (hand-written CUDA, FP64 DMMA).  This
package is the C-ABI binding (``include/eig.h``) plus torch plumbing.  It
never imports ``oracle/`` and has no CPU fallback.
"""
from ._binding import (EIG_DIST_HE2HB, EIG_GATHER_Z, EIG_HOST_BUFFERS, EIG_NO_3M, EIG_USE_3M, EIG_SKIP_BT, EIG_SKIP_HE2HB, STAGES, EigError,  # noqa: F401
                       Solver, colmajor, column_slice, empty_colmajor, exported_symbols, lib, num_panels,
                       resolve_range, unique_id, v2_slots)

__all__ = ["Solver", "EigError", "colmajor", "empty_colmajor", "lib", "num_panels", "v2_slots", "exported_symbols",
           "unique_id", "column_slice", "resolve_range", "STAGES", "EIG_HOST_BUFFERS", "EIG_SKIP_BT",
           "EIG_SKIP_HE2HB", "EIG_GATHER_Z", "EIG_USE_3M", "EIG_NO_3M", "EIG_DIST_HE2HB"]
