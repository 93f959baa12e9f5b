"""Gate values (eigenvalue error, residual, B-orthogonality) of the n = 5000
clustered known-spectrum pencils (test_config2) for the current settings."""
import math
import sys
import os
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from test_gpu_solve_gen import _run, gates  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
A, B, D = synth.pencil_known(n, seed=5, kappa=1e2, clustered=True)
for frac in (0.10, 0.25, 1.0):
    w, Z = _run(A, B, fraction=frac)
    m = int(math.ceil(frac * n))
    res, orth = gates(A, B, w[:m], Z)
    print(f"n={n} frac={frac}: eig {np.max(np.abs(w - D)) / np.max(np.abs(D)):.3e} res {res:.3e} orth {orth:.3e}",
          flush=True)
