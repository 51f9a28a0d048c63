"""World-size-2 gloo test of the multi-GPU host path (CPU only).

Two ranks each own half of the runs (runs.shard), produce their per-run
snapshot sums (here with the oracle, since there is no GPU), exchange them
with runs.gather_run_sums, and rank 0 forms the ensemble.  It must equal the
single-process ensemble over all runs bit for bit (same fold order, R18), and
the job time / particle-step reductions must be max / sum over ranks.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_path):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle import oracle
    from paper_cs_9902024_b200 import runs
    from workloads import configs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    job = configs.get("c2_small", n_runs=4, n_steps=20)
    mine = runs.shard(job, rank, world, runs_per_rank=2)
    assert mine["run_id0"] == 2 * rank and mine["n_runs"] == 2
    sums = []
    for r in range(mine["run_id0"], mine["run_id0"] + mine["n_runs"]):
        o = oracle.OracleRun(mine, r)
        o.fill()
        o.step(20)
        sums.append(o.get_snap(0))
    local = torch.from_numpy(np.array(sums).transpose(1, 0, 2).copy())   # [5][n_local][Nc]
    full = runs.gather_run_sums(local)
    t = runs.max_over_ranks(1.0 + rank)
    n = runs.sum_over_ranks(10.0 * (rank + 1))
    if rank == 0:
        ens = oracle.ensemble(full.numpy().transpose(1, 0, 2), job["fnum_vc"])
        np.savez(out_path, ens=ens, t=t, n=n)
    dist.barrier()
    dist.destroy_process_group()


def _worker_slot_layout(rank, world, port, out_path, sub=1):
    """The exchange in the product's layout: each rank's slot sums as dsmc_read_sums /
    Simulation.slot_sums_device lay them out, [5][n_local*Nc], gathered into
    [world][5][n_local*Nc] by runs.gather_slot_sums (the input of
    dsmc_read_macros_gathered).  sub > 1: the rank holds its runs in `sub`
    sub-batch contexts (bench.py's e2e leg), their slot sums stacked
    [sub][5][n_local/sub*Nc] before the gather and the result read as
    world*sub blocks."""
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle import oracle
    from paper_cs_9902024_b200 import runs
    from workloads import configs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    job = configs.get("c2_small", n_runs=6, n_steps=20)
    mine = runs.shard(job, rank, world, runs_per_rank=3)
    Nc = configs.n_cells(job)
    snaps = []
    for r in range(mine["run_id0"], mine["run_id0"] + mine["n_runs"]):
        o = oracle.OracleRun(mine, r)
        o.fill()
        o.step(20)
        snaps.append(o.get_snap(0))                                    # [5][Nc]
    m = 3 // sub
    blocks = [np.array(snaps[b * m:(b + 1) * m]).transpose(1, 0, 2).reshape(5, m * Nc) for b in range(sub)]
    local = torch.from_numpy(np.array(blocks[0] if sub == 1 else blocks).copy())
    g = runs.gather_slot_sums(local)
    assert tuple(g.shape) == ((world, 5, 3 * Nc) if sub == 1 else (world, sub, 5, m * Nc))
    g = g.reshape(-1, 5, m * Nc)                                       # world*sub blocks in run order
    if rank == 0:
        per_run = g.numpy().reshape(world * sub, 5, m, Nc).transpose(0, 2, 1, 3).reshape(world * 3, 5, Nc)
        np.savez(out_path, ens=oracle.ensemble(per_run, job["fnum_vc"]), per_run=per_run)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("sub", [1, 3])
def test_two_rank_gather_in_product_layout(tmp_path, oracle_mod, sub):
    """runs.gather_slot_sums over gloo, world size 2: block k of the gathered tensor is
    rank k's slot, so the runs come out in ascending global id and the ensemble of
    the gathered sums equals the single-process ensemble over all 6 runs bit for bit
    (sub = 3: each rank's runs in three sub-batch contexts, as bench.py's e2e leg)."""
    from workloads import configs
    out = str(tmp_path / "g0.npz")
    mp.spawn(_worker_slot_layout, args=(2, _free_port(), out, sub), nprocs=2, join=True)
    got = np.load(out)
    job = configs.get("c2_small", n_runs=6, n_steps=20)
    sums = []
    for r in range(6):
        o = oracle_mod.OracleRun(job, r)
        o.fill()
        o.step(20)
        sums.append(o.get_snap(0))
    sums = np.array(sums)
    assert np.array_equal(got["per_run"], sums)
    want = oracle_mod.ensemble(sums, job["fnum_vc"])
    assert np.array_equal(np.nan_to_num(got["ens"], nan=-7.0), np.nan_to_num(want, nan=-7.0))


def test_two_rank_ensemble_equals_single(tmp_path, oracle_mod):
    from workloads import configs
    out = str(tmp_path / "r0.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    assert got["t"] == 2.0 and got["n"] == 30.0
    job = configs.get("c2_small", n_runs=4, n_steps=20)
    sums = []
    for r in range(4):
        o = oracle_mod.OracleRun(job, r)
        o.fill()
        o.step(20)
        sums.append(o.get_snap(0))
    want = oracle_mod.ensemble(np.array(sums), job["fnum_vc"])
    assert np.array_equal(np.nan_to_num(got["ens"], nan=-7.0), np.nan_to_num(want, nan=-7.0))


def test_shard_offsets():
    sys.path.insert(0, ROOT)
    from paper_cs_9902024_b200 import runs
    from workloads import configs
    p = configs.get("c4_small", n_runs=3)
    shards = [runs.shard(p, k, 4) for k in range(4)]
    ids = [i for q in shards for i in range(q["run_id0"], q["run_id0"] + q["n_runs"])]
    assert ids == list(range(12))
