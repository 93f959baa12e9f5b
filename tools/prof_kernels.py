#!/usr/bin/env python
"""Per-kernel timing probes (CUDA events) for the hot-path kernels; used
standalone and under ncu.  Modes:
  gemm  : zgemm engine on square / he2hb-shaped products
  q2    : apply_q2 at (n, m) with synthetic reflectors
  he2hb : he2hb alone at n
  hb2st : bulge chasing alone at n
  stedc : tridiagonal divide and conquer at n (random d, e)
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_1207_1773_b200 import Solver, colmajor, empty_colmajor  # noqa: E402


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    p = argparse.ArgumentParser()
    p.add_argument("mode")
    p.add_argument("--n", type=int, default=8192)
    p.add_argument("--m", type=int, default=None)
    p.add_argument("--k", type=int, default=None)
    p.add_argument("--nb", type=int, default=64)
    p.add_argument("--g", type=int, default=0)
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--m3", action="store_true", help="complex GEMMs as three real products (EIG_USE_3M)")
    p.add_argument("--kw", type=int, default=0, help="gemm mode: panel width of the V^H E / E -= V Y shapes (default nb)")
    a = p.parse_args()
    dev = torch.device("cuda:0")
    from paper_1207_1773_b200 import EIG_NO_3M, EIG_USE_3M
    s = Solver(0, nb=a.nb, q2_group=a.g, flags=EIG_USE_3M if a.m3 else EIG_NO_3M)
    n = a.n
    m = a.m or n
    if a.mode == "gemm":
        k = a.k or n
        A = torch.randn(k, n, dtype=torch.complex128, device=dev).t()   # n x k col-major
        B = torch.randn(m, k, dtype=torch.complex128, device=dev).t()   # k x m
        C = torch.zeros(m, n, dtype=torch.complex128, device=dev).t()   # n x m
        ms = timeit(lambda: s.zgemm("N", "N", A, B, C), a.reps)
        print(f"zgemm NN {n}x{m}x{k}: {ms:.3f} ms  {8.0 * n * m * k / ms / 1e9:.2f} TFLOP/s")
        H = torch.randn(n, n, dtype=torch.complex128, device=dev).t()
        V = torch.randn(a.nb, n, dtype=torch.complex128, device=dev).t()
        W = torch.zeros(a.nb, n, dtype=torch.complex128, device=dev).t()
        ms = timeit(lambda: s.zgemm("N", "N", H, V, W, herm_a=True), a.reps)
        print(f"hemm {n}x{a.nb}: {ms:.3f} ms  {8.0 * n * n * a.nb / ms / 1e9:.2f} TFLOP/s")
        VX = torch.randn(2 * a.nb, n, dtype=torch.complex128, device=dev).t()
        ms = timeit(lambda: s.zgemm("N", "C", VX, VX, H, alpha=-1.0, beta=1.0, lower_c=True), a.reps)
        print(f"her2k {n} k={2 * a.nb}: {ms:.3f} ms  {8.0 * n * n * a.nb / ms / 1e9:.2f} TFLOP/s (nominal 8 s^2 nb)")
        kw = a.kw or a.nb
        V = torch.randn(kw, n, dtype=torch.complex128, device=dev).t()
        Y = torch.zeros(m, kw, dtype=torch.complex128, device=dev).t()
        E = torch.randn(m, n, dtype=torch.complex128, device=dev).t()
        ms = timeit(lambda: s.zgemm("C", "N", V, E, Y), a.reps)
        print(f"V^H E {kw}x{m} K={n}: {ms:.3f} ms  {8.0 * n * m * kw / ms / 1e9:.2f} TFLOP/s")
        Y2 = torch.randn(m, kw, dtype=torch.complex128, device=dev).t()
        ms = timeit(lambda: s.zgemm("N", "N", V, Y2, E, alpha=-1.0, beta=1.0), a.reps)
        print(f"E -= V Y {n}x{m} K={kw}: {ms:.3f} ms  {8.0 * n * m * kw / ms / 1e9:.2f} TFLOP/s")
    elif a.mode == "q2":
        V2, tau2 = synth.synthetic_v2(n, a.nb, 0)
        V2d, t2d = torch.from_numpy(V2).to(dev), torch.from_numpy(tau2).to(dev)
        E = empty_colmajor(n, m, device=dev)
        E.copy_(torch.randn(m, n, dtype=torch.complex128, device=dev).t())
        ms = timeit(lambda: s.apply_q2(V2d, t2d, E), a.reps)
        print(f"apply_q2 n={n} m={m} nb={a.nb} g={s.q2_group}: {ms:.3f} ms  {8.0 * n * n * m / ms / 1e9:.2f} TFLOP/s")
        if os.environ.get("EIG_Q2_PROFILE"):
            pr = s.q2_profile()[:5]
            tot = max(sum(pr), 1)
            print("  CTA0 phase cycles (load, A, B, C, commit):", [f"{x / tot * 100:.1f}%" for x in pr], tot)
            pw = s.q2_profile()[24:29]
            tw = max(sum(pw), 1)
            print("  q2w CTA0 warp0 (wait, A, B, C, release) / q2s (V/T wait, E wait, group barrier, block, release):",
                  [f"{x / tw * 100:.1f}%" for x in pw], tw)
    elif a.mode == "hb2st":
        A0 = colmajor(synth.rand_hermitian(n, 0), dev)
        s.he2hb(A0)
        ms = timeit(lambda: s.hb2st(A0), a.reps)
        print(f"hb2st n={n} nb={a.nb}: {ms:.3f} ms  band bytes {n * (2 * a.nb + 2) * 16 / 1e6:.1f} MB")
        if os.environ.get("EIG_Q2_PROFILE"):
            pr = s.q2_profile()[16:22]
            tot = sum(pr)
            print("  hb2st CTA0 (wait, load, refl, update, -, flag):", [f"{x / tot * 100:.1f}%" for x in pr], tot)
    elif a.mode == "stedc":
        rng = np.random.default_rng(0)
        d = torch.from_numpy(rng.standard_normal(n)).to(dev)
        e = torch.from_numpy(rng.standard_normal(n - 1)).to(dev)
        ms = timeit(lambda: s.stedc(d, e), a.reps)
        print(f"stedc n={n}: {ms:.3f} ms")
    elif a.mode == "he2hb":
        A0 = colmajor(synth.rand_hermitian(n, 0), dev)
        A = A0.clone()

        def run():
            A.copy_(A0)
            s.he2hb(A)
        ms = timeit(run, a.reps)
        print(f"he2hb n={n} nb={a.nb}: {ms:.3f} ms  {16.0 / 3.0 * n ** 3 / ms / 1e9:.2f} TFLOP/s")
        if os.environ.get("EIG_Q2_PROFILE"):
            pr = s.q2_profile()[8:14]
            tot = sum(pr)
            print("  panel CTA0 cycles (wait, reduce, beta, lookahead-col, publish, bulk+T):",
                  [f"{x / tot * 100:.1f}%" for x in pr], f"{tot / 1.965e6 / (a.reps + 1):.1f} ms/run")
    s.close()


if __name__ == "__main__":
    main()
