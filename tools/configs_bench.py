#!/usr/bin/env python
"""Per-config table of the BASELINE configs, one JSON
object per (n, fraction) on stdout (and in --out):

  * zhegv seconds of eig_solve_gen (median of --reps calls after a warm-up) on
    a known-spectrum pencil built on the device (kappa(B) = 100), with the
    R9/R10 gates checked on the last call's result;
  * he2hb + back-transform TFLOP/s from the SAME calls' eig_stats stage times:
    (16/3 n^3 + 20 n^2 m) / (t_he2hb + t_BT), and its fraction of the measured
    DMMA peak (37.1 TFLOP/s, profiles/fp64_peak_r01.json);
  * the CPU oracle (as it stands) on a bounded sample of the same n (the first
    r he2hb reflectors and c eigenvector columns through Q2, Q1, L^-H), with
    the core count and CPU model.

    python tools/configs_bench.py [--reps 3] [--out profiles/configs_r02.json]
"""
import argparse
import functools
import json
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

CONFIGS = [(256, 1.0, 16), (2000, 1.0, 64), (5000, 0.10, 64), (5000, 0.25, 64), (10000, 1.0, 64),
           (20000, 0.10, 64), (20000, 0.50, 64), (20000, 1.0, 64)]


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


@functools.lru_cache(maxsize=None)
def oracle_sample(n, nb, budget_refl, cols):
    """Oracle TFLOP/s on the first r he2hb reflectors + c columns through the BT (bench.py's recipe)."""
    import oracle
    import synth
    oracle.build()
    A = oracle.full_hermitian(synth.rand_hermitian(n, 0))
    t0 = time.perf_counter()
    oracle.he2hb_partial(A, nb, budget_refl)
    t_he = time.perf_counter() - t0
    fl_he = sum(16.0 * (n - nb - j) ** 2 for j in range(budget_refl))
    V2, tau2 = synth.synthetic_v2(n, nb, 0)
    A1, tau1 = synth.synthetic_v1(n, nb, 0)
    L = synth.unit_lower(n, 0)
    Z = synth.real_orthonormalish(n, cols, 0).astype(complex)
    t0 = time.perf_counter()
    E = oracle.backsub_lh(L, oracle.apply_q1(A1, tau1, nb, oracle.apply_q2(V2, tau2, nb, Z)))
    t_bt = time.perf_counter() - t0
    assert np.all(np.isfinite(E))
    return {"value": (fl_he + 20.0 * n * n * cols) / (t_he + t_bt) / 1e12, "unit": "TFLOP/s",
            "cores": len(os.sched_getaffinity(0)), "cpu": cpu_model(), "kind": "oracle",
            "sample": f"first {budget_refl} he2hb reflectors ({t_he:.1f} s) + {cols} eigenvector columns through "
                      f"Q2, Q1, L^-H ({t_bt:.1f} s)"}


def run(n, frac, nb, reps, peak, with_cpu):
    A, B, D = _known_pencil_torch(n, 3)
    s = Solver(0, nb=nb)
    secs, st_all = [], []
    for r in range(reps + 1):
        Ac = torch.tril(A).t().contiguous().t()
        Bc = torch.tril(B).t().contiguous().t()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s.stream)
        w, Z, st = s.solve_gen(Ac, Bc, fraction=frac, stats=True)
        e1.record(s.stream)
        torch.cuda.synchronize()
        del Ac, Bc
        if r:
            secs.append(e0.elapsed_time(e1) * 1e-3)
            st_all.append(st)
    m = Z.shape[1]
    w = w.cpu().numpy()
    ev = float(np.max(np.abs(w - D)) / np.max(np.abs(D)))
    res, orth = gates(A, B, torch.from_numpy(w[:m]).cuda(), Z)
    med = int(np.argsort(secs)[len(secs) // 2])
    st = st_all[med]
    t_hb = st["seconds"]["he2hb"] + st["seconds"]["bt"]
    flops = 16.0 / 3.0 * n ** 3 + 20.0 * n * n * m
    out = {"n": n, "fraction": frac, "m": m, "nb": nb, "zhegv_s": secs[med],
           "zhegv_s_min_max": [min(secs), max(secs)],
           "stages_ms": {k: v * 1e3 for k, v in st["seconds"].items() if v > 0},
           "he2hb_bt_tflops": flops / t_hb / 1e12, "he2hb_bt_frac_of_dmma_peak": flops / t_hb / 1e12 / peak,
           "gates": {"eig_rel": ev, "residual": res, "b_orth": orth,
                     "pass": bool(ev <= 1e-10 and res <= 1e-14 and orth <= 1e-14)}}
    del A, B, Z
    torch.cuda.empty_cache()
    if with_cpu:
        r, c = (8, 16) if n <= 10000 else (4, 4)
        out["cpu_baseline"] = oracle_sample(n, nb, min(r, max(1, n - nb - 1)), c)
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--out", default=None)
    p.add_argument("--no-cpu", action="store_true")
    a = p.parse_args()
    try:
        peak = float(json.load(open(os.path.join(ROOT, "profiles", "fp64_peak_r01.json")))["dmma_tflops_sustained"])
    except Exception:
        peak = 37.1
    rows = []
    for n, frac, nb in CONFIGS:
        row = run(n, frac, nb, a.reps, peak, not a.no_cpu)
        print(json.dumps(row), flush=True)
        rows.append(row)
    if a.out:
        json.dump({"configs": rows, "dmma_peak_tflops": peak, "gemm": "3M (default)",
                   "note": "known-spectrum pencils built on the device, kappa(B) = 100; he2hb+BT TFLOP/s from the "
                           "eig_stats stage times of the timed solve"}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
