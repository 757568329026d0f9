"""Sharded 3D path (SURVEY.md §8e for BASELINE configs 4-5): contiguous subdomain ranges per
rank (whole z-layers when the ranks divide s_z, else y-row blocks of a layer: config 5's
4x4x4 grid on 8 ranks),
replicated dual/primal vectors, one allreduce completing every jump gather.

CPU (`not gpu`): the per-rank views built by the C++ host core (fetigpu3d_rank_info) tile the
subdomains, every multiplier row has its two owners somewhere among the ranks, corner slots
are partitioned — in-process and across a world_size-2 gloo process group (each process
builds its own rank's view, as one process per GPU does under NCCL), where an allreduce of
per-rank partial jumps of a known interface field reproduces the global jump exactly.
GPU: W ranks emulated by host threads on one device (ThreadComm) reproduce the single-GPU
solve (relative 1e-12: the partial sums are exact, only the primal assembly of multiplicity-4
dofs may round differently).
"""
import os
import socket

import numpy as np
import pytest


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


LAYOUT_CASES = [  # n, physics, s, worlds
    (8, 0, 2, (2,)),
    (12, 0, 3, (3,)),
    (32, 0, 4, (2, 4)),
    (128, 0, 8, (2, 4, 8)),
    (64, 1, 4, (2, 4, 8)),    # BASELINE config 5 on 8 ranks: 2 y-rows of one z-layer each
    (12, 0, 3, (9, 27)),       # ranks not dividing s_z: partial layers
]


def check_layout(F, box, p, s, world):
    info = box.box_partition_info(p, s)
    infos = [box.rank_info_3d(p, s, r, world) for r in range(world)]
    assert sum(i["n_sub_local"] for i in infos) == info["n_subdomains"]
    firsts = [i["sub_first"] for i in infos]
    assert firsts == sorted(firsts) and firsts[0] == 0
    for a, b in zip(infos, infos[1:]):
        assert a["sub_first"] + a["n_sub_local"] == b["sub_first"]
    assert sum(i["row_owners"] for i in infos) == 2 * info["n_lambda"]
    return infos


@pytest.mark.parametrize("case", LAYOUT_CASES, ids=lambda c: f"n{c[0]}-p{c[1]}-s{c[2]}")
def test_rank_layout3d_tiles(fetigpu, case):
    from paper_1312_5653_b200 import box

    n, physics, s, worlds = case
    p = box.make_box_problem(n, phi=1e-4, physics=physics, young=1.0, poisson=0.3)
    single = box.rank_info_3d(p, s, 0, 1)
    for world in worlds:
        infos = check_layout(fetigpu, box, p, s, world)
        # rows split across a cut have one owner on each side: fewer rows with both owners local
        assert sum(i["rows_both_local"] for i in infos) < single["rows_both_local"]
        assert sum(i["corner_slots"] for i in infos) == single["corner_slots"]


def test_rank_layout3d_rejects_bad_world(fetigpu):
    from paper_1312_5653_b200 import ContractError, box

    p = box.make_box_problem(12, phi=1e-4)
    with pytest.raises(ContractError):
        box.rank_info_3d(p, 3, 0, 2)  # 27 subdomains over 2 ranks


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1312_5653_b200 import box
        p = box.make_box_problem(32, phi=1e-4)
        mine = box.rank_info_3d(p, 4, rank, world)
        infos = [None] * world
        dist.all_gather_object(infos, mine)
        info = box.box_partition_info(p, 4)
        assert sum(i["n_sub_local"] for i in infos) == info["n_subdomains"]
        assert sum(i["row_owners"] for i in infos) == 2 * info["n_lambda"]
        # replicated dual vectors: each rank's partial row values (owned owners only) sum to
        # the global value; with +a on the lower and -b on the higher owner the allreduce of
        # the partials equals a - b bitwise (two nonzero terms per row)
        n_l = info["n_lambda"]
        a = np.cos(np.arange(n_l, dtype=np.float64))
        b = np.sin(np.arange(n_l, dtype=np.float64) * 0.37)
        both = mine["rows_both_local"]
        t = torch.tensor([float(mine["row_owners"]), float(both)], dtype=torch.float64)
        dist.all_reduce(t)
        assert int(t[0].item()) == 2 * n_l
        full = torch.from_numpy(a - b)
        part = torch.from_numpy(np.where(np.arange(n_l) % world == rank, a, 0.0) -
                                np.where(np.arange(n_l) % world != rank, b, 0.0))
        dist.all_reduce(part)
        assert torch.equal(part, full)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_rank_layout3d():
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


GPU_CASES = [  # n, physics, s, world
    (12, 0, 3, 3),
    (16, 0, 2, 2),
    (32, 0, 4, 4),
    (8, 1, 2, 2),
    (16, 1, 4, 2),
    (16, 1, 4, 8),   # config 5's 4x4x4 grid (at 16^3) on 8 ranks: partial z-layers
    (16, 0, 2, 4),   # 2x2x2 on 4 ranks: one y-row of a layer per rank
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", GPU_CASES, ids=lambda c: f"n{c[0]}-p{c[1]}-s{c[2]}-w{c[3]}")
def test_emulated_sharded3d_matches_single_gpu(fetigpu, case):
    from paper_1312_5653_b200 import box

    n, physics, s, world = case
    p = box.make_box_problem(n, phi=1e-4, physics=physics, young=1.0, poisson=0.3, seed=5)
    ref = box.solve_range_space_3d(p, s, tol=1e-10, max_iter=1000)
    out = box.emulated_schur_solve_3d(p, s, world, tol=1e-10, max_iter=1000)
    assert out["converged"] and ref["converged"]
    for k in ("y", "u", "lambda"):
        assert rel(out[k], ref[k]) <= 1e-12, k
    for side in ("plus_stats", "minus_stats"):
        assert out[side]["iterations"] == ref[side]["iterations"]
