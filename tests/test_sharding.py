"""Sharded (multi-GPU) FETI-DP path, SURVEY.md §8e.

CPU (`not gpu`): the per-rank layout built by the C++ host core (fetigpu_rank_info) tiles the
global multipliers, free dofs and subdomains, and neighbouring ranks agree on every halo size,
checked both in-process and across a world_size-2 gloo process group (each process builds its
own rank's layout, exactly as one process per GPU does under NCCL).

GPU: the sharded solve with W ranks emulated by host threads on one device (device-to-device
copies standing in for NCCL, ThreadComm in csrc/comm.hpp) reproduces the single-GPU solve.
"""
import os
import socket

import numpy as np
import pytest

CASES = [  # (n_x, n_y, physics, s_x, s_y, worlds)
    (64, 64, 0, 4, 4, (2, 4)),
    (256, 256, 0, 8, 8, (2, 4, 8)),
    (1024, 1024, 0, 32, 32, (2, 4, 8)),
    (48, 32, 1, 6, 4, (2, 4)),
]


def _problem(F, n_x, n_y, physics):
    if physics == 1:
        return F.make_problem(n_x, n_y, 1e-4, physics=1, len_x=1.5, len_y=1.0, young=1.0, poisson=0.3)
    return F.make_problem(n_x, n_y, 1e-4)


def check_layout(infos, part):
    world = len(infos)
    assert sum(i["n_owned"] for i in infos) == part["n_lambda"]
    assert sum(i["free_count"] for i in infos) == part["n"]
    assert sum(i["n_sub_local"] for i in infos) == part["n_subdomains"]
    own_first = 0
    free_first = 0
    for r, i in enumerate(infos):
        assert i["free_first"] == free_first
        free_first += i["free_count"]
        # local numbering: [ghost rows = top cut of rank r-1][owned rows incl. own top cut]
        assert i["lam_base"] + i["n_ghost"] == own_first
        assert i["n_lambda_local"] == i["n_ghost"] + i["n_owned"]
        own_first += i["n_owned"]
        if r == 0:
            assert i["n_ghost"] == 0 and i["halo_down"] == 0
        else:
            assert i["n_ghost"] == infos[r - 1]["n_top_cut"]
            assert i["halo_down"] == infos[r - 1]["halo_up"]
        if r == world - 1:
            assert i["n_top_cut"] == 0 and i["halo_up"] == 0
        else:
            assert i["n_top_cut"] > 0 and i["halo_up"] > 0


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}x{c[1]}-p{c[2]}-{c[3]}x{c[4]}")
def test_rank_layout_tiles(fetigpu, case):
    n_x, n_y, physics, s_x, s_y, worlds = case
    p = _problem(fetigpu, n_x, n_y, physics)
    part = fetigpu.partition_info(p, s_x, s_y)
    for world in worlds:
        infos = [fetigpu.rank_info(p, s_x, s_y, r, world) for r in range(world)]
        check_layout(infos, part)


def test_rank_layout_rejects_bad_world(fetigpu):
    p = fetigpu.make_problem(64, 64, 1e-4)
    with pytest.raises(fetigpu.ContractError):
        fetigpu.rank_info(p, 4, 4, 0, 3)  # s_y % world != 0
    with pytest.raises(fetigpu.ContractError):
        fetigpu.rank_info(p, 4, 4, 2, 2)  # rank out of range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1312_5653_b200 as F
        p = F.make_problem(256, 256, 1e-4)
        mine = F.rank_info(p, 8, 8, rank, world)
        infos = [None] * world
        dist.all_gather_object(infos, mine)
        part = F.partition_info(p, 8, 8)
        check_layout(infos, part)
        # allgatherv of the primal solution: each rank contributes its owned free dofs of a
        # known vector; the sum over ranks (zero elsewhere) reassembles it exactly
        x = np.arange(part["n"], dtype=np.float64) * 0.5 + 1.0
        mine_x = np.zeros_like(x)
        sl = slice(mine["free_first"], mine["free_first"] + mine["free_count"])
        mine_x[sl] = x[sl]
        t = torch.from_numpy(mine_x)
        dist.all_reduce(t)
        assert np.array_equal(t.numpy(), x)
        # the replicated Krylov scalars: an allreduce of owned-row partial dots equals the
        # global dot product (owned rows tile the multipliers)
        v = np.sin(np.arange(part["n_lambda"], dtype=np.float64))
        lo = mine["lam_base"] + mine["n_ghost"]
        d = torch.tensor([float(np.dot(v[lo:lo + mine["n_owned"]], v[lo:lo + mine["n_owned"]]))],
                         dtype=torch.float64)
        dist.all_reduce(d)
        assert abs(d.item() - float(np.dot(v, v))) <= 1e-12 * float(np.dot(v, v))
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_rank_layout():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


GPU_CASES = [  # (n_x, n_y, physics, s_x, s_y, world)
    (64, 64, 0, 4, 4, 2),
    (64, 64, 0, 4, 4, 4),
    (256, 256, 0, 8, 8, 2),
    (256, 256, 0, 8, 8, 8),
    (48, 32, 1, 6, 4, 2),
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", GPU_CASES, ids=lambda c: f"{c[0]}x{c[1]}-p{c[2]}-{c[3]}x{c[4]}-w{c[5]}")
def test_emulated_sharded_solve_matches_single_gpu(fetigpu, case):
    n_x, n_y, physics, s_x, s_y, world = case
    p = _problem(fetigpu, n_x, n_y, physics)
    solver = fetigpu.SchurSolver(p, s_x, s_y, tol=1e-10, max_iter=1000)
    ref = solver.solve()
    solver.close()
    out = fetigpu.emulated_schur_solve(p, world, s_x, s_y, tol=1e-10, max_iter=1000)
    assert out["converged"] and ref["converged"]
    for k in ("y", "u", "lambda"):
        assert rel(out[k], ref[k]) <= 1e-8, k
    for side in ("plus_stats", "minus_stats"):
        assert abs(out[side]["iterations"] - ref[side]["iterations"]) <= 2


@pytest.mark.gpu
def test_emulated_sharded_full_coarse_inverse(fetigpu, monkeypatch):
    """Each rank keeps only the C^-1 rows of the corners its subdomains (and phantom
    neighbours) touch; FETIGPU_FULL_COARSE=1 keeps the whole inverse on every rank.  Same
    iterations, results equal to rounding."""
    p = _problem(fetigpu, 256, 256, 0)
    a = fetigpu.emulated_schur_solve(p, 4, 8, 8, tol=1e-10, max_iter=1000)
    monkeypatch.setenv("FETIGPU_FULL_COARSE", "1")
    b = fetigpu.emulated_schur_solve(p, 4, 8, 8, tol=1e-10, max_iter=1000)
    for side in ("plus_stats", "minus_stats"):
        assert a[side]["iterations"] == b[side]["iterations"]
    for k in ("y", "u", "lambda"):
        assert rel(a[k], b[k]) <= 1e-11, k


@pytest.mark.gpu
def test_nccl_plumbing_one_rank(fetigpu):
    """The NCCL communicator of the sharded paths initialises and runs its collectives on
    the box (one rank: the results equal the inputs).  Multi-rank NCCL needs several GPUs."""
    import ctypes as C

    from paper_1312_5653_b200 import _native

    uid = fetigpu.nccl_unique_id()
    out = np.zeros(4)
    rc = _native.lib().fetigpu_nccl_selftest(bytes(uid), 0, 1, 0, out.ctypes.data_as(C.POINTER(C.c_double)))
    assert rc == 0, _native.lib().fetigpu_last_error()
    assert out.tolist() == [1.0, 2.0, -1.0, 0.0]
