"""Column slicing of the back-transform is exact:
the multi-GPU path gives each rank a contiguous slice of the eigenvector
columns, so E = L^-H Q1 Q2 Z computed slice by slice must be BITWISE equal to
the unsliced E.  Every back-transform kernel treats columns independently
and the zgemm split-K factor of the back-transform GEMMs does not depend on
the column count (kBtSplitN), so the summation order of a column is the same
in both runs.  Runs on one GPU: P slices in sequence (marker: gpu)."""
import numpy as np
import pytest
import torch

import synth

gpu = pytest.mark.gpu


def _slices(m, P):
    return [(r * m // P, (r + 1) * m // P) for r in range(P)]


@gpu
@pytest.mark.parametrize("n,nb,g,m", [(1000, 64, 32, 1000), (777, 32, 16, 333), (2000, 64, 32, 1250)])
def test_backtransform_column_slices_bitwise(n, nb, g, m):
    from paper_1207_1773_b200 import EIG_SKIP_HE2HB, Solver, colmajor, empty_colmajor
    dev = torch.device("cuda:0")
    s = Solver(0, nb=nb, q2_group=g)
    A = colmajor(synth.rand_hermitian(n, 3), dev)
    tau1, T1 = s.he2hb(A)
    V2, tau2 = synth.synthetic_v2(n, nb, 3)
    V2 = torch.from_numpy(V2).to(dev)
    tau2 = torch.from_numpy(tau2).to(dev)
    L = colmajor(synth.unit_lower(n, 3), dev)
    Z = colmajor(synth.real_orthonormalish(n, m, 3), dev)
    E_full, _, _ = s.hotpath(A, V2, tau2, L, Z, flags=EIG_SKIP_HE2HB, tau1=tau1, T1=T1)
    torch.cuda.synchronize()
    for P in (2, 3, 4, 8):
        E = empty_colmajor(n, m, device=dev)
        for (a, b) in _slices(m, P):
            if b > a:
                s.hotpath(A, V2, tau2, L, Z[:, a:b], E=E[:, a:b], flags=EIG_SKIP_HE2HB, tau1=tau1, T1=T1)
        torch.cuda.synchronize()
        assert torch.equal(E, E_full), f"P={P}: max diff {(E - E_full).abs().max().item():.3e}"
