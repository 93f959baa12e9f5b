#!/usr/bin/env python
"""Benchmark of the B200 hot path: one step = he2hb of the
standard-form matrix + complexify + Q2 + Q1 + L^-H on the m eigenvector columns.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Metric (BASELINE.json): FP64 TFLOP/s of he2hb + back-transform, nominal flops
16/3 n^3 + 20 n^2 m (8 real flops per complex multiply-add), workload n = 10000,
m = 10000 (configs[3]).  N > 1 (torchrun, one process per GPU): the
collective C-ABI call eig_hotpath runs he2hb 1D block-cyclically over the
ranks (EIG_DIST_HE2HB, NEXT-4; --no-dist-he2hb: on rank 0 with the factors
broadcast as lower triangles), sends V2 / L over NCCL from inside libeigb200
and back-transforms each rank's eigenvector column slice (strong scaling); the
line adds t_BT(P) (max over ranks) and t_BT(1) / t_BT(P), and the zhegv
seconds with both he2hb placements.
Inputs (1.6 GB each) exceed L2 (126 MB), so no explicit L2 flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 TFLOP/s he2hb+back-transform; zhegv seconds n=10k at 1/2/4/8 B200"
DMMA_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peak_r01.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "traffic_r02.json")


def ncu_traffic(kernel, n, m, nb, g):
    """dram read+write bytes per launch of `kernel` from the committed ncu capture
    (only if it was taken on this exact workload)."""
    try:
        d = json.load(open(TRAFFIC_FILE))
        if d["workload"] != {"n": n, "m": m, "nb": nb, "g": g}:
            return None
        k = d[kernel]
        return k["dram_bytes_read"] + k["dram_bytes_write"]
    except Exception:
        return None


def nominal_flops(n, m):
    return 16.0 / 3.0 * n ** 3 + 20.0 * n * n * m


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--n", type=int, default=10000)
    p.add_argument("--m", type=int, default=None)
    p.add_argument("--nb", type=int, default=64)
    p.add_argument("--g", type=int, default=32)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-zhegv", action="store_true", help="skip the end-to-end generalized solve timing")
    p.add_argument("--no-dist-he2hb", action="store_true",
                   help="N > 1: he2hb on rank 0 instead of 1D block-cyclic over the ranks (EIG_DIST_HE2HB)")
    p.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of oracle work for cpu_baseline")
    p.add_argument("--gemm", default="3m", choices=["3m", "4m"],
                   help="complex GEMMs (he2hb updates, Q1, L^-H, front end) as 3 real DMMA products (3M) or 4 (4M)")
    a = p.parse_args()
    if a.m is None:
        a.m = a.n
    return a


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for k, nm in enumerate(names):
                    if r[5 + k].strip() == "Active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dmma_peak():
    try:
        d = json.load(open(DMMA_PEAK_FILE))
        return float(d["dmma_tflops_sustained"]), "measured DMMA (profiles/fp64_peak_r01.json)"
    except Exception:
        return 37.0, "fallback datasheet FP64 tensor"


# ------------------------------------------------------------------ CPU oracle sample
def cpu_sample(n, nb, seed, budget, pre=None):
    """The oracle as it stands, on a bounded sample of the same workload:
    the first r he2hb reflectors of A' (n x n) and c eigenvector columns through
    Q2, Q1, L^-H.  Returns (TFLOP/s, cores, description).  `pre` may hold the
    already generated (A, V2, tau2, L) of the same seed."""
    import oracle
    import synth
    oracle.build()
    cores = len(os.sched_getaffinity(0))
    A = pre[0] if pre else synth.rand_hermitian(n, seed)
    Ah = oracle.full_hermitian(A)
    # he2hb sample
    r = 8
    t0 = time.perf_counter()
    oracle.he2hb_partial(Ah, nb, r)
    t_he = time.perf_counter() - t0
    fl_he = sum(16.0 * (n - nb - j) ** 2 for j in range(r))
    # BT sample
    c = max(1, min(cores, 16))
    V2, tau2 = (pre[1], pre[2]) if pre else synth.synthetic_v2(n, nb, seed)
    A1, tau1 = synth.synthetic_v1(n, nb, seed)
    L = pre[3] if pre else synth.unit_lower(n, seed)
    Z = synth.real_orthonormalish(n, c, seed).astype(complex)
    t0 = time.perf_counter()
    E = oracle.apply_q2(V2, tau2, nb, Z)
    E = oracle.apply_q1(A1, tau1, nb, E)
    E = oracle.backsub_lh(L, E)
    t_bt = time.perf_counter() - t0
    fl_bt = 20.0 * n * n * c
    value = (fl_he + fl_bt) / (t_he + t_bt) / 1e12
    desc = (f"oracle on n={n}: first {r} he2hb reflectors ({t_he:.1f} s) + {c} eigenvector columns through "
            f"Q2,Q1,L^-H ({t_bt:.1f} s); nominal flops of the sample / time")
    cpu_sample.parts = {"he2hb_tflops": fl_he / t_he / 1e12, "bt_tflops": fl_bt / t_bt / 1e12,
                        "he2hb_s": t_he, "bt_s": t_bt, "reflectors": r, "columns": c}
    return value, cores, desc, t_he + t_bt


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_sample_threads(n, nb, threads):
    """The same oracle sample at order n in a child process with OMP_NUM_THREADS = threads."""
    code = ("import sys, json; sys.path.insert(0, %r); import bench; "
            "v, c, d, t = bench.cpu_sample(%d, %d, 0, 0.0); "
            "print(json.dumps({'value': v, 'desc': d, 'parts': bench.cpu_sample.parts}))" % (ROOT, n, nb))
    env = dict(os.environ, OMP_NUM_THREADS=str(threads))
    try:
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        return json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as e:   # reported, not fatal
        return {"error": str(e)[:200]}


def run_reference(a, rank, world):
    """--impl reference: the oracle (as it stands) on this arm's workload, each
    step a bounded sample (first he2hb reflectors + a few eigenvector columns
    through Q2, Q1, L^-H).  Rank 0 only; other ranks exit without work."""
    if rank != 0:
        return 0
    import synth
    pre = (synth.rand_hermitian(a.n, a.seed), *synth.synthetic_v2(a.n, a.nb, a.seed), synth.unit_lower(a.n, a.seed))
    vals = []
    cores, desc = 0, ""
    for i in range(a.warmup + a.steps):
        v, cores, desc, _ = cpu_sample(a.n, a.nb, a.seed, a.cpu_budget, pre=pre)
        if i >= a.warmup:
            vals.append(v)
    v = statistics.mean(vals)
    line = {"metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "higher_is_better": True, "impl": "reference", "dtype": "f64",
            "data": "synthetic", "scaling": "weak", "vs_baseline": None,
            "config": {"workload": f"he2hb+BT n={a.n} m={a.m} nb={a.nb} g={a.g}", "n": a.n, "m": a.m, "nb": a.nb,
                       "q2_group": a.g},
            "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ zhegv (Algorithm 1 end to end)
def hpd_on_device(n, kappa, seed, dev, r=8):
    """G1 B = U^H diag(kappa^(k/(n-1))) U built with torch on the device from
    synth's seeded reflectors (same recipe as synth.hpd_with_condition)."""
    import torch

    import synth
    U = torch.from_numpy(synth.random_reflectors(n, r, seed, 2)).to(dev)
    d = torch.as_tensor(kappa ** (np.arange(n) / max(n - 1, 1)), dtype=torch.complex128, device=dev)
    M = torch.diag(d)
    for t in range(r):
        u = U[:, t:t + 1]
        M = M - 2.0 * u @ (u.conj().T @ M)
        M = M - 2.0 * (M @ u) @ u.conj().T
    M = 0.5 * (M + M.conj().T)
    return M.t().contiguous().t()


def zhegv_timing(solver, A0, B0, stream):
    """Seconds of one eig_solve_gen (all eigenvectors) after a warm-up call, plus
    a per-stage breakdown from the stage entry points (CUDA events)."""
    import torch
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    A, B = A0.clone(), B0.clone()
    solver.solve_gen(A, B)
    A.copy_(A0)
    B.copy_(B0)
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record(stream)
    w, Z = solver.solve_gen(A, B)
    e1.record(stream)
    torch.cuda.synchronize()
    total = e0.elapsed_time(e1) * 1e-3
    # stage breakdown (same work through the stage entry points); the second of
    # two passes is timed, so the stages' output tensors come from the
    # allocator's cache instead of a cudaMalloc inside a stage
    for rep in range(2):
        A.copy_(A0)
        B.copy_(B0)
        torch.cuda.synchronize()
        evs = [ev() for _ in range(7)]
        evs[0].record(stream)
        solver.potrf(B)
        evs[1].record(stream)
        solver.hegst(A, B)
        evs[2].record(stream)
        tau1, T1 = solver.he2hb(A)
        evs[3].record(stream)
        d, e, V2, tau2 = solver.hb2st(A)
        evs[4].record(stream)
        w2, Zr = solver.stedc(d, e)
        evs[5].record(stream)
        solver.apply_q2(V2, tau2, Z, Z=Zr)
        solver.apply_q1(A, T1, Z)
        solver.trsm_lh(B, Z)
        evs[6].record(stream)
        torch.cuda.synchronize()
        del tau1, T1, d, e, V2, tau2, w2, Zr
    names = ["potrf", "hegst", "he2hb", "hb2st", "stedc", "backtransform"]
    stages = {nm: evs[i].elapsed_time(evs[i + 1]) for i, nm in enumerate(names)}
    return total, stages


# ------------------------------------------------------------------ B200 arm
def run_b200(a, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import synth
    from paper_1207_1773_b200 import Solver, colmajor, column_slice, empty_colmajor, num_panels, v2_slots
    from paper_1207_1773_b200.dist import collective_solver

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    n, m, nb = a.n, a.m, a.nb
    K = num_panels(n, nb)
    slots = v2_slots(n, nb)
    lo, hi = column_slice(m, rank, world)
    ml = hi - lo

    t_gen = time.perf_counter()
    if rank == 0:
        A_h = synth.rand_hermitian(n, a.seed)
        V2_h, tau2_h = synth.synthetic_v2(n, nb, a.seed)
        L_h = synth.unit_lower(n, a.seed)
        A0 = colmajor(A_h, dev)
        V2 = torch.from_numpy(V2_h).to(dev)
        tau2 = torch.from_numpy(tau2_h).to(dev)
        L = colmajor(L_h, dev)
        A = empty_colmajor(n, n, device=dev)
    else:   # ranks > 0 receive the factors inside the collective call
        A_h = V2_h = tau2_h = L_h = None
        A0 = V2 = tau2 = L = A = None
    Z_h = synth.real_orthonormalish(n, ml, a.seed, col0=lo)
    Z = colmajor(Z_h, dev)
    E = empty_colmajor(n, ml, device=dev)
    t_gen = time.perf_counter() - t_gen

    from paper_1207_1773_b200 import EIG_NO_3M, EIG_USE_3M
    gflags = EIG_USE_3M if a.gemm == "3m" else EIG_NO_3M
    from paper_1207_1773_b200 import EIG_DIST_HE2HB
    dflag = 0 if a.no_dist_he2hb else EIG_DIST_HE2HB   # N > 1: he2hb 1D block-cyclic over the ranks (NEXT-4)
    solver = (Solver(local_rank, nb=nb, q2_group=a.g, flags=gflags) if world == 1
              else collective_solver(local_rank, nb, a.g, flags=gflags | dflag))
    stream = solver.stream
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    stage_names = ["he2hb", "q2", "q1", "trsm"]

    def step(events=None):
        if world == 1:
            if events:
                events[0].record(stream)
            A.copy_(A0)
            tau_, T_ = solver.he2hb(A)
            if events:
                events[1].record(stream)
            solver.apply_q2(V2, tau2, E, Z=Z)
            if events:
                events[2].record(stream)
            solver.apply_q1(A, T_, E)
            if events:
                events[3].record(stream)
            solver.trsm_lh(L, E)
            if events:
                events[4].record(stream)
        else:   # collective C-ABI call: he2hb on rank 0, NCCL broadcast, sharded back-transform
            if events:
                events[0].record(stream)
            if rank == 0:
                A.copy_(A0)
            solver.hotpath(A, V2, tau2, L, Z, E=E)
            if events:
                events[4].record(stream)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    launches0 = solver.launches
    t_start, t_end = ev(), ev()
    step_events = [[ev() for _ in range(5)] for _ in range(a.steps)]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_start.record(stream)
    for s in range(a.steps):
        step(step_events[s])
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = solver.launches - launches0
    clk = clocks.stop()
    ms_total = t_start.elapsed_time(t_end)
    bt_scaling = None
    if world > 1:
        tt = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_total = float(tt.item())
        # t_BT(P): this rank's back-transform of the last step (eig_last_stats), max over ranks
        st = solver.last_stats()
        tb = torch.tensor([st["seconds"]["bt"], st["seconds"]["wait"]], dtype=torch.float64, device=dev)
        dist.all_reduce(tb, op=dist.ReduceOp.MAX)
        t_bt_p = float(tb[0].item())
        t_bt_1 = None
        if rank == 0:   # t_BT(1): the same back-transform of all m columns on one GPU (rank 0's factors)
            s1 = Solver(local_rank, nb=nb, q2_group=a.g, flags=gflags)
            from paper_1207_1773_b200 import EIG_SKIP_HE2HB
            Zall = colmajor(synth.real_orthonormalish(n, m, a.seed), dev)
            Eall = empty_colmajor(n, m, device=dev)
            A.copy_(A0)
            tau_1, T_1 = s1.he2hb(A)
            for _ in range(2):
                s1.hotpath(A, V2, tau2, L, Zall, E=Eall, flags=EIG_SKIP_HE2HB, tau1=tau_1, T1=T_1)
            t_bt_1 = s1.last_stats()["seconds"]["bt"]
            s1.close()
            del Zall, Eall
        bt_scaling = {"t_bt_P_s": t_bt_p, "t_bt_1_s": t_bt_1, "bt_scaling": (t_bt_1 / t_bt_p) if t_bt_1 else None,
                      "wait_max_s": float(tb[1].item()), "bytes_comm_rank": st["bytes_comm"],
                      "note": "t_BT = complexify+Q2+Q1+L^-H of this rank's column slice (CUDA events, eig_last_stats), "
                              "max over ranks; t_BT(1) = all m columns on rank 0's GPU alone"}
    ms_step = ms_total / a.steps
    stages = {}
    if world == 1:
        for k, nm in enumerate(stage_names):
            stages[nm] = statistics.mean(step_events[s][k].elapsed_time(step_events[s][k + 1])
                                         for s in range(a.steps))
    flops = nominal_flops(n, m)
    value = flops / (ms_step * 1e-3) / 1e12

    # roofline of the dominant kernel (per-stage events; Q2 is one kernel launch)
    peak, peak_src = dmma_peak()
    roof = None
    if stages:
        stage_flops = {"he2hb": 16.0 / 3.0 * n ** 3, "q2": 8.0 * n * n * m, "q1": 8.0 * n * n * m,
                       "trsm": 4.0 * n * n * m}
        q2_3m = os.environ.get("EIG_Q2_3M", "1") != "0"
        q2k = (("apply_q2wave3_kernel" if q2_3m else "apply_q2wave_kernel") if (nb == 64 and a.g == 32)
               else "apply_q2_kernel")
        kern = {"he2hb": "zgemm_kernel (hemm+her2k) + panel_qr_kernel", "q2": q2k,
                "q1": "zgemm_kernel", "trsm": "zgemm_kernel"}
        dom = max(stages, key=stages.get)
        ach = stage_flops[dom] / (stages[dom] * 1e-3) / 1e12
        traffic = ncu_traffic(q2k, n, m, nb, a.g) if dom == "q2" else None
        roof = {"bound": "tensor", "kernel": kern[dom], "stage": dom, "achieved": ach, "peak": peak,
                "unit": "TFLOP/s", "frac": ach / peak, "traffic": traffic,
                "traffic_note": "dram read+write bytes per launch (ncu --set full, profiles/traffic_r02.json); "
                                "algorithmic E traffic n^2/(2g) m 16 B each way = 2 x 250 GB (the wavefront kernel moves whole 95-row windows: 786 GB measured, 1.6x); compute-bound",
                "peak_source": peak_src,
                "stage_tflops": {k: stage_flops[k] / (stages[k] * 1e-3) / 1e12 for k in stages},
                # tensor-pipe work: 3M issues 6 real flops per complex MAC (he2hb updates, Q1, trsm and, by
                # default, Q2), the real embedding 8 (Q2's 492/384 or 616/512 parallelogram overhead not counted)
                "gemm_mode": a.gemm.upper(),
                "stage_pipe_frac": {k: stage_flops[k] * (0.75 if ((a.gemm == "3m" and k != "q2") or (k == "q2" and q2_3m))
                                                         else 1.0)
                                    / (stages[k] * 1e-3) / 1e12 / peak for k in stages}}

    # e2e through the C ABI with HOST buffers (pinned), N = 1
    e2e = None
    if rank == 0 and world == 1 and not a.no_e2e:
        def pinned(shape_cols, ld, dtype):
            return torch.empty((shape_cols, ld), dtype=dtype, pin_memory=True)

        Ap = pinned(n, n, torch.complex128)
        Ap.numpy()[:] = A_h.T
        Lp = pinned(n, n, torch.complex128)
        Lp.numpy()[:] = L_h.T
        Zp = pinned(m, n, torch.float64)
        Zp.numpy()[:] = Z_h.T
        V2p = torch.from_numpy(V2_h).pin_memory()
        t2p = torch.from_numpy(tau2_h).pin_memory()
        Ep = pinned(m, n, torch.complex128)
        e_steps = max(1, min(a.steps, 3))
        solver.hotpath_host(Ap.numpy().T, V2p.numpy(), t2p.numpy(), Lp.numpy().T, Zp.numpy().T, Ep.numpy().T)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            solver.hotpath_host(Ap.numpy().T, V2p.numpy(), t2p.numpy(), Lp.numpy().T, Zp.numpy().T, Ep.numpy().T)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / e_steps
        lower = sum((n - j0) * min(256, n - j0) for j0 in range(0, n, 256)) * 16   # A, L: lower 256-col blocks
        h2d = 2 * lower + slots * nb * 16 + slots * 16 + n * m * 8
        d2h = n * m * 16
        e2e = {"value": flops / dt / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": dt * 1e3, "steps": e_steps}

    zhegv = None
    if world > 1 and not a.no_zhegv:
        del E
        torch.cuda.empty_cache()
        B0 = hpd_on_device(n, 1e2, a.seed, dev) if rank == 0 else None
        Aw, Bw = (A0.clone(), B0.clone()) if rank == 0 else (None, None)
        solver.solve_gen(Aw, Bw, n=n)                  # warm-up (collective)
        if rank == 0:
            Aw.copy_(A0)
            Bw.copy_(B0)
        torch.cuda.synchronize()
        dist.barrier()
        z0, z1 = ev(), ev()
        z0.record(stream)
        w_, Z_, zst = solver.solve_gen(Aw, Bw, n=n, stats=True)
        z1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        tt = torch.tensor([z0.elapsed_time(z1) * 1e-3, zst["seconds"]["bt"]], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        zhegv = {"seconds": float(tt[0].item()), "t_bt_max_s": float(tt[1].item()), "n": n, "m": n, "kappa_B": 1e2,
                 "ranks": world, "stages_ms_rank0": {k: v * 1e3 for k, v in zst["seconds"].items()} if rank == 0 else None,
                 "note": "collective eig_solve_gen: rank 0 potrf, hegst, he2hb, hb2st, stedc; NCCL broadcast of "
                         "L / V1 / T1 (during hb2st) and V2 (during stedc), scatter of the eigenvector slices; "
                         "back-transform sharded by eigenvector columns; max over ranks"}
        zhegv["dist_he2hb"] = bool(dflag)
        if True:   # the same solve with the other he2hb placement, for comparison
            sd = collective_solver(local_rank, nb, a.g, flags=gflags | (EIG_DIST_HE2HB ^ dflag))
            if rank == 0:
                Aw.copy_(A0)
                Bw.copy_(B0)
            sd.solve_gen(Aw, Bw, n=n)                   # warm-up
            if rank == 0:
                Aw.copy_(A0)
                Bw.copy_(B0)
            torch.cuda.synchronize()
            dist.barrier()
            w_, Z_, dst = sd.solve_gen(Aw, Bw, n=n, stats=True)
            torch.cuda.synchronize()
            dist.barrier()
            td = torch.tensor([dst["seconds"]["total"], dst["seconds"]["he2hb"]], dtype=torch.float64, device=dev)
            dist.all_reduce(td, op=dist.ReduceOp.MAX)
            zhegv["other_he2hb_placement"] = {"dist_he2hb": not dflag, "seconds": float(td[0].item()),
                                              "he2hb_s_max": float(td[1].item())}
            sd.close()
        del Aw, Bw, B0, w_, Z_
    if rank == 0 and world == 1 and not a.no_zhegv:
        del E
        torch.cuda.empty_cache()
        B0 = hpd_on_device(n, 1e2, a.seed, dev)
        zs, zst = zhegv_timing(solver, A0, B0, stream)
        zhegv = {"seconds": zs, "stages_ms": zst, "n": n, "m": n, "kappa_B": 1e2,
                 "note": "eig_solve_gen (potrf, hegst, he2hb, hb2st, stedc, Q2, Q1, L^-H), all eigenvectors, "
                         "one call after a warm-up; stage breakdown from the stage entry points"}
        del B0

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        v, cores, desc, secs = cpu_sample(n, nb, a.seed, a.cpu_budget, pre=(A_h, V2_h, tau2_h, L_h))
        cpu = {"value": v, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": desc, "cpu": cpu_model(),
               "parts": cpu_sample.parts,
               "one_thread_n2000": cpu_sample_threads(2000, nb, 1),
               "note": "per-part TFLOP/s beside the GPU stage_tflops (he2hb vs q2+q1+trsm); the oracle's "
                       "reflector updates and column loops are OpenMP-parallel over `cores` threads"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded SplitMix64; G1 Hermitian A', random unitary V2, well-conditioned L, real Z)",
                "config": {"workload": f"he2hb+BT n={n} m={m} nb={nb} g={a.g}", "n": n, "m": m, "nb": nb,
                           "q2_group": a.g,
                           "parallelism": (f"bt-columns{world}" + ("+he2hb-1d-cyclic" if dflag else "")) if world > 1
                           else "single",
                           "gemm": a.gemm.upper(),
                           "zhegv_seconds_hotpath": ms_step * 1e-3,
                           "l2": "inputs (1.6 GB each) exceed L2; no flush needed",
                           "input_gen_s": round(t_gen, 1)},
                "stages_ms": stages, "gpu_launches": launches,
                "gpu_launches_per_step": launches / max(a.steps, 1), "roofline": roof, "clocks": clk,
                "e2e": e2e, "cpu_baseline": cpu, "zhegv": zhegv, "bt_scaling": bt_scaling}
        print(json.dumps(line), flush=True)
    solver.close()
    return 0


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        return run_reference(a, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    rc = run_b200(a, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
