#!/usr/bin/env python
"""Small invocations of every spin-wait / grid-sync / shared-memory-heavy kernel
for compute-sanitizer (memcheck, racecheck, synccheck), one tool per run:

    compute-sanitizer --tool memcheck  --error-exitcode 1 python tools/sanitize.py
    compute-sanitizer --tool racecheck --error-exitcode 1 python tools/sanitize.py
    compute-sanitizer --tool synccheck --error-exitcode 1 python tools/sanitize.py

Covers panel_qr_kernel (cooperative, arrival counter), hb2st_kernel (release /
acquire wavefront), apply_q2wave_kernel (cooperative grid.sync wavefront),
apply_q2_kernel (generic grouped Q2), the zgemm engine (4M and 3M), stedc and
the potrf / hegst front end at n = 256 / nb = 16 and n = 600 / nb = 64.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_1207_1773_b200 import EIG_NO_3M, EIG_USE_3M, Solver, colmajor  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    for n, nb, g in [(256, 16, 8), (600, 64, 32)]:
        for flags in (EIG_NO_3M, EIG_USE_3M):
            s = Solver(0, nb=nb, q2_group=g, flags=flags)
            A = colmajor(synth.rand_hermitian(n, 1), dev)
            V2, tau2 = synth.synthetic_v2(n, nb, 1)
            L = colmajor(synth.unit_lower(n, 1), dev)
            Z = colmajor(synth.real_orthonormalish(n, min(n, 100), 1), dev)
            E, tau1, T1 = s.hotpath(A, torch.from_numpy(V2).to(dev), torch.from_numpy(tau2).to(dev), L, Z)
            d, e, V2d, tau2d = s.hb2st(A)
            w, Zr = s.stedc(d, e)
            A2, B2 = synth.pencil_rand(n, seed=2, kappa=1e2)
            w2, Z2 = s.solve_gen(colmajor(np.tril(A2), dev), colmajor(np.tril(B2), dev))
            torch.cuda.synchronize()
            assert torch.isfinite(E).all() and torch.isfinite(Z2).all()
            s.close()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
