#!/usr/bin/env python
"""eig_solve_gen timings on the BASELINE configs (synthetic known-spectrum
pencils built on the device, kappa(B) = 100): one warm-up call, then the
median of three timed calls (CUDA events on the solver's stream), with the
accuracy gates of DESIGN.md R9/R10 checked on the result."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from test_gpu_solve_gen import _known_pencil_torch, gates  # noqa: E402
from paper_1207_1773_b200 import Solver  # noqa: E402


def run(n, frac):
    A, B, D = _known_pencil_torch(n, 3)
    s = Solver(0, nb=64)
    ts = []
    for r in range(4):
        Ac = torch.tril(A).t().contiguous().t()
        Bc = torch.tril(B).t().contiguous().t()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s.stream)
        w, Z = s.solve_gen(Ac, Bc, fraction=frac)
        e1.record(s.stream)
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1) * 1e-3)
    w = w.cpu().numpy()
    m = Z.shape[1]
    ev = np.max(np.abs(w - D)) / np.max(np.abs(D))
    res, orth = gates(A, B, torch.from_numpy(w[:m]).cuda(), Z)
    print(f"n={n:6d} fraction={frac:4.2f} m={m:6d}: {np.median(ts):.3f} s  eig rel {ev:.1e}  residual {res:.1e}  B-orth {orth:.1e}",
          flush=True)


if __name__ == "__main__":
    for n, fr in [(2000, 1.0), (5000, 0.10), (5000, 0.25), (10000, 1.0), (10000, 0.10), (20000, 0.10), (20000, 0.5), (20000, 1.0)]:
        run(n, fr)
