"""Data-parallel plumbing: one process per GPU, a full
compressed-feature + CSR replica per GPU, seed ids sharded across ranks, one
all-reduce of the flat fp32 gradient per step.

Sharding: train ids are made unique and sorted (pipeline.py:194), rank r of
W takes ids[r::W] and runs the reference sampler semantics on its shard with
the integer seed ``(seed + epoch) * W + r`` — so each rank's batches are
exactly ``sample_batches(g, shard_r, SamplerConfig(f, bs, seed_r))`` of the
reference and can be checked against the CPU oracle per rank.  Ranks agree
on the minimum batch count so the all-reduces line up.
"""

from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist


def shard_ids(train_ids, rank: int, world: int) -> np.ndarray:
    ids = np.unique(np.asarray(train_ids, dtype=np.int64))
    return ids[rank::world]


def rank_seed(seed: int, epoch: int, rank: int, world: int) -> int:
    return (seed + epoch) * world + rank


def agree_num_batches(nb: int, group=None, device=None) -> int:
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return nb
    t = torch.tensor([nb], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return int(t.item())


def average_flat_(flat: torch.Tensor, group=None) -> torch.Tensor:
    """In-place mean over ranks of a flat gradient buffer (one collective)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(flat, group=group)
        flat.div_(dist.get_world_size(group))
    return flat


def init_from_env(backend: str = "nccl"):
    """torchrun-style init (RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend, rank=rank, world_size=world,
                                device_id=torch.device("cuda", local) if backend == "nccl" else None)
    return rank, world, local


def max_over_ranks(value: float, device=None) -> float:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
