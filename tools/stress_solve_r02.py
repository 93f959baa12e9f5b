#!/usr/bin/env python
"""Repeated eig_solve_gen on random sizes / fractions against the known
spectrum and the R9/R10 gates (end-to-end race check of every kernel)."""
import argparse
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import synth  # noqa: E402
from test_gpu_solve_gen import _run, gates  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--iters", type=int, default=12)
    a = p.parse_args()
    rng = np.random.default_rng(99)
    for it in range(a.iters):
        n = int(rng.integers(300, 2600))
        frac = float(rng.choice([0.1, 0.3, 1.0]))
        A, B, D = synth.pencil_known(n, seed=int(rng.integers(1, 10 ** 6)), kappa=1e2, clustered=bool(it % 2))
        w, Z = _run(A, B, fraction=frac)
        m = int(math.ceil(frac * n))
        ev = np.max(np.abs(w - D)) / np.max(np.abs(D))
        res, orth = gates(A, B, w[:m], Z)
        print(f"it {it}: n={n} frac={frac}: eig {ev:.2e} res {res:.2e} orth {orth:.2e}", flush=True)
        assert ev <= 1e-10 and res <= 1e-14 and orth <= 1e-14, (n, frac)
    print("all ok")


if __name__ == "__main__":
    main()
