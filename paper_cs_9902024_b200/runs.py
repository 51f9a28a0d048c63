"""Multi-GPU host logic: the paper's first level (PSIR).

Runs are statistically independent, so N GPUs split the
runs: rank k owns runs [k*n, (k+1)*n) of the job (Philox key run id =
run_id0 + r, R4), with no collective on the data path.  The one exchange the
paper has -- "the data exchange between processors goes after all
calculation are finished. Only one processor sequentially analyzes the
results" -- is `gather_run_sums`: the per-run snapshot
sums of every rank are gathered in ascending run id, after which one rank
forms the ensemble (dsmc_read_macros semantics, R18).  Timing of a multi-GPU
job is the maximum over ranks (`max_over_ranks`).
"""
from __future__ import annotations

import copy


def shard(p, rank, world, runs_per_rank=None):
    """Problem dict of `rank`: n runs per rank (weak scaling), ids offset by rank*n."""
    q = copy.deepcopy(p)
    n = runs_per_rank if runs_per_rank is not None else p["n_runs"]
    q["n_runs"] = n
    q["run_id0"] = p.get("run_id0", 0) + rank * n
    return q


def max_over_ranks(value, group=None):
    """Max of a float over ranks (a job's time is its slowest rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(value, group=None):
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())


def gather_slot_sums(local, group=None):
    """The one exchange, in the product's layout: `local` is this
    rank's slot sums [5][n_local*Nc] fp64 (Simulation.slot_sums_device on a GPU, or
    any tensor of that layout); returns [world][5][n_local*Nc] with block k = rank
    k's, i.e. runs in ascending global run id when rank k owns runs [k*n, (k+1)*n)
    (shard).  One all-gather over NCCL (NVLink) for device tensors, gloo for host
    ones; feed the result to Simulation.read_macros_gathered."""
    import torch
    import torch.distributed as dist
    local = local.contiguous()
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return local.reshape(1, *local.shape)
    world = dist.get_world_size(group)
    out = torch.empty((world, *local.shape), dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, local, group=group)      # one NCCL all-gather into the block layout
    else:                                                          # gloo: no _allgather_base
        dist.all_gather(list(out.unbind(0)), local, group=group)
    return out


def ensemble_over_ranks(sim, slot, group=None):
    """Ensemble macros of `slot` over the runs of every rank (bit-identical to one GPU
    holding all of them): gather the slot sums, then dsmc_read_macros_gathered."""
    g = gather_slot_sums(sim.slot_sums_device(slot), group)
    return sim.read_macros_gathered(slot, g, g.shape[0])


def gather_run_sums(local, group=None):
    """local: tensor [5][n_local][Nc] (float64) of this rank's runs (ascending
    run id).  Returns [5][n_local*world][Nc] on every rank, runs ordered by
    (rank, local run) = ascending global run id -- the fold order of R18."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return local
    world = dist.get_world_size(group)
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local.contiguous(), group=group)
    return torch.cat(parts, dim=1)
