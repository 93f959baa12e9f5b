#!/usr/bin/env python
"""Repeated oracle comparisons of the kernels with cross-CTA protocols (the
position-stationary bulge chase, the dataflow Q2 wavefront, the panel's
messenger warp) on varied sizes and seeds, to catch rare ordering bugs.
    python tools/stress_r02.py [--iters 20]"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1207_1773_b200 import Solver, colmajor, empty_colmajor  # noqa: E402
from test_gpu_hb2st import _band_full  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--iters", type=int, default=20)
    a = p.parse_args()
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(1234)
    worst = {"hb2st": 0.0, "q2": 0.0, "he2hb": 0.0}
    for it in range(a.iters):
        n = int(rng.integers(200, 900))
        nb = int(rng.choice([16, 32, 64]))
        seed = int(rng.integers(1, 10 ** 6))
        s = Solver(0, nb=nb)
        A = synth.rand_hermitian(n, seed)
        # he2hb (panel) vs oracle
        dA = colmajor(A, dev)
        s.he2hb(dA)
        A_o, _ = oracle.he2hb(A, nb)
        r, c = np.indices((n, n))
        low = r >= c
        e1 = np.max(np.abs(dA.cpu().numpy()[low] - A_o[low])) / np.max(np.abs(A_o))
        # hb2st on the oracle's band
        d, e, V2, tau2 = s.hb2st(colmajor(A_o, dev))
        d_o, e_o, V2_o, tau2_o = oracle.hb2st(_band_full(A_o, nb), nb)
        e2 = max(np.max(np.abs(d.cpu().numpy() - d_o)), np.max(np.abs(e.cpu().numpy() - e_o))) / np.max(np.abs(A))
        e2 = max(e2, np.max(np.abs(V2.cpu().numpy() - V2_o)))
        # Q2 (nb = 64, g = 32 runs the 3M dataflow wavefront)
        s64 = Solver(0, nb=64, q2_group=32)
        m = int(rng.integers(8, 400))
        V2s, t2s = synth.synthetic_v2(n, 64, seed)
        Z = synth.real_orthonormalish(n, m, seed)
        dE = empty_colmajor(n, m)
        s64.apply_q2(torch.from_numpy(V2s).to(dev), torch.from_numpy(t2s).to(dev), dE, Z=colmajor(Z, dev))
        ref = oracle.apply_q2(V2s, t2s, 64, Z.astype(complex))
        e3 = np.max(np.abs(dE.cpu().numpy() - ref)) / np.max(np.abs(ref))
        worst["he2hb"] = max(worst["he2hb"], e1)
        worst["hb2st"] = max(worst["hb2st"], e2)
        worst["q2"] = max(worst["q2"], e3)
        print(f"it {it}: n={n} nb={nb} m={m} he2hb {e1:.2e} hb2st {e2:.2e} q2 {e3:.2e}", flush=True)
        assert e1 < 1e-11 and e2 < 1e-9 and e3 < 1e-11, (n, nb, m, seed)
        s.close()
        s64.close()
    print("worst", worst)


if __name__ == "__main__":
    main()
