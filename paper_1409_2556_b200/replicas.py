"""Multi-GPU plumbing for bench.py (one process per GPU, torch.distributed).

The hot path does not need a data-path collective for the benchmark workload: every rank
builds the Jacobian of its own field realisation (independent replicas of the per-GPU
workload, "weak" scaling).  The only collective is the max-over-ranks reduction of the
device-timed step durations (and a barrier around the timed region).
"""
from __future__ import annotations

import copy

REPLICA_SEED_STRIDE = 1000


def replica_config(cfg, rank: int):
    """Same statistics, distinct seeded realisation per rank (rank 0 = the BASELINE input)."""
    out = copy.deepcopy(cfg)
    if rank > 0:
        out.log_kappa = {**cfg.log_kappa, "seed": cfg.log_kappa["seed"] + REPLICA_SEED_STRIDE * rank}
        if "seed" in cfg.log_storativity:
            out.log_storativity = {**cfg.log_storativity,
                                   "seed": cfg.log_storativity["seed"] + REPLICA_SEED_STRIDE * rank}
    return out


def max_over_ranks(values, device=None):
    """Elementwise max of a list of floats over all ranks (identity when not distributed)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [float(v) for v in values]
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def barrier(device=None):
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
