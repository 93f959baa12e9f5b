"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU plumbing
(DESIGN.md §8).

The collective work itself (NCCL broadcast of the factors, scatter of the
eigenvector slices, per-rank back-transform) lives in libeigb200 (comm.cu)
and needs GPUs; what runs here is everything around it that does not:

* the C ABI's rank and argument logic: eig_get_unique_id on rank 0 shipped
  to the other rank over torch.distributed (paper_1207_1773_b200.dist),
  eig_column_slice / eig_resolve_range agreeing on every rank, and eig_init
  rejecting bad {rank, nranks, nccl_id} before touching a device;
* the property the sharding rests on: the back-transform of a column
  slice does not depend on the other columns, so per-rank slices computed
  with the CPU oracle and gathered are bitwise the unsliced result.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

N, NB, M = 70, 8, 11


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(target, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    return res


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


# ------------------------------------------------------------------ ABI rank / argument logic
def _worker_abi(rank, world, port, out):
    _init(rank, world, port)
    from paper_1207_1773_b200 import column_slice, lib, resolve_range
    from paper_1207_1773_b200._binding import _Config
    from paper_1207_1773_b200.dist import ship_unique_id
    uid = ship_unique_id()                              # rank 0: eig_get_unique_id, gloo broadcast
    ids = [None] * world
    dist.all_gather_object(ids, uid)
    slices = {m: column_slice(m, rank, world) for m in (0, 1, 7, 1250, 10000)}
    allsl = [None] * world
    dist.all_gather_object(allsl, slices)
    rng = [resolve_range(5000, fraction=f) for f in (0.1, 0.25, 1e-9, 1.0)] + [resolve_range(300, il=5, iu=9)]
    allrng = [None] * world
    dist.all_gather_object(allrng, rng)
    # eig_init validates {rank, nranks, nccl_id} before any device call
    idbuf = C.create_string_buffer(uid, 128)
    h = C.c_void_p()

    def init(rk, nr, with_id):
        cfg = _Config(0, 64, 0, None, rk, nr, C.cast(idbuf, C.c_void_p) if with_id else None, 0, 0)
        return lib().eig_init(C.byref(h), C.byref(cfg))
    codes = {"bad_rank": init(world + 3, world, True), "neg_rank": init(-1, world, True),
             "no_id": init(rank, world, False)}
    if not torch.cuda.is_available():
        codes["valid_no_gpu"] = init(rank, world, True)  # passes validation, then no device: EIG_ERR_CUDA
    lo, hi = C.c_int64(), C.c_int64()
    codes["slice_bad_rank"] = lib().eig_column_slice(10, world, world, C.byref(lo), C.byref(hi))
    codes["slice_bad_m"] = lib().eig_column_slice(-1, 0, world, C.byref(lo), C.byref(hi))
    if rank == 0:
        out.put((ids, allsl, allrng, codes))
    dist.barrier()
    dist.destroy_process_group()


def test_abi_rank_and_argument_logic_gloo_world2():
    ids, allsl, allrng, codes = _spawn(_worker_abi)
    assert len(ids[0]) == 128 and ids[0] == ids[1] and any(ids[0])
    for m in (0, 1, 7, 1250, 10000):
        sl = [allsl[r][m] for r in range(2)]
        assert sl == [(0, m // 2), (m // 2, m)]           # floor(r m / P): contiguous, balanced, ordered
    assert allrng[0] == allrng[1]
    assert allrng[0][0] == (1, 500, 500) and allrng[0][1] == (1, 1250, 1250)
    assert allrng[0][2] == (1, 1, 1) and allrng[0][3] == (1, 5000, 5000) and allrng[0][4] == (5, 9, 5)
    assert codes["bad_rank"] == -2 and codes["neg_rank"] == -2 and codes["no_id"] == -2
    if "valid_no_gpu" in codes:
        assert codes["valid_no_gpu"] == -1001             # EIG_ERR_CUDA: validation passed
    assert codes["slice_bad_rank"] == -2 and codes["slice_bad_m"] == -1


def test_column_slices_partition():
    from paper_1207_1773_b200 import column_slice
    for m in (0, 1, 7, 10000):
        for P in (1, 2, 3, 4, 8):
            sl = [column_slice(m, r, P) for r in range(P)]
            assert sl[0][0] == 0 and sl[-1][1] == m
            assert all(sl[r][1] == sl[r + 1][0] for r in range(P - 1))
            assert max(b - a for a, b in sl) - min(b - a for a, b in sl) <= 1


def test_resolve_range_matches_reading_r12():
    from paper_1207_1773_b200 import EigError, resolve_range
    assert resolve_range(10000) == (1, 10000, 10000)
    assert resolve_range(5000, fraction=0.1) == (1, 500, 500)       # lowest ceil(f n) (R12)
    assert resolve_range(7, fraction=0.5) == (1, 4, 4)
    with pytest.raises(EigError):
        resolve_range(10, fraction=0.0)
    with pytest.raises(EigError):
        resolve_range(10, il=4, iu=3)


# ------------------------------------------------------------------ slice independence (oracle)
def _inputs():
    A = synth.rand_hermitian(N, 4)
    V2, tau2 = synth.synthetic_v2(N, NB, 4)
    L = synth.unit_lower(N, 4)
    Z = synth.real_orthonormalish(N, M, 4)
    return A, V2, tau2, L, Z


def _bt_oracle(A_o, tau_o, V2, tau2, L, Z):
    return oracle.backsub_lh(L, oracle.apply_q1(A_o, tau_o, NB, oracle.apply_q2(V2, tau2, NB, Z.astype(complex))))


def _worker_bt(rank, world, port, out):
    _init(rank, world, port)
    from paper_1207_1773_b200 import column_slice
    A, V2, tau2, L, Z = _inputs()
    A_o, tau_o = oracle.he2hb(A, NB)
    lo, hi = column_slice(M, rank, world)
    E = _bt_oracle(A_o, tau_o, V2, tau2, L, Z[:, lo:hi])
    parts = [None] * world
    dist.all_gather_object(parts, (lo, E))
    if rank == 0:
        out.put(np.concatenate([p[1] for p in sorted(parts, key=lambda t: t[0])], axis=1))
    dist.barrier()
    dist.destroy_process_group()


def test_sliced_backtransform_gloo_world2_bitwise():
    E_dist = _spawn(_worker_bt)
    A, V2, tau2, L, Z = _inputs()
    A_o, tau_o = oracle.he2hb(A, NB)
    assert np.array_equal(E_dist, _bt_oracle(A_o, tau_o, V2, tau2, L, Z))
