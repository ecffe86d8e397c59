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

from .graph import sorted_unique_ids


def shard_ids(train_ids, rank: int, world: int) -> np.ndarray:
    ids = sorted_unique_ids(train_ids)
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
        if dist.get_backend(group) == "nccl":
            dist.all_reduce(flat, op=dist.ReduceOp.AVG, group=group)  # one NCCL kernel
        else:
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


# -- sharded preprocessing (SURVEY.md §8e "Preprocessing"): each rank encodes
# a contiguous row block of the codec, one all-gather assembles the replica;
# VQ parts are fitted round-robin and their codebooks broadcast by the owner.

def world_of(group=None) -> tuple[int, int]:
    if not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def row_block(n: int, rank: int, world: int) -> tuple[int, int, int]:
    """Rows [r0, r1) encoded by ``rank``; every block is ``chunk`` rows long
    except the tail (the gather buffer is padded to world*chunk rows)."""
    chunk = -(-n // world) if n else 0
    r0 = min(rank * chunk, n)
    return r0, min(r0 + chunk, n), chunk


def padded_rows(n: int, stride: int, world: int, device) -> torch.Tensor:
    """Row buffer with room for world equal blocks; the codec uses [:n]."""
    _, _, chunk = row_block(n, 0, world)
    return torch.zeros((max(chunk * world, n), stride), dtype=torch.uint8, device=device)


def allgather_rows_(buf: torch.Tensor, n: int, group=None) -> torch.Tensor:
    """Every rank filled its own block of ``buf`` (padded_rows); afterwards
    every rank holds all n rows.  NCCL gathers over NVLink; gloo (CPU
    tests, several ranks on one device) stages through host memory."""
    rank, world = world_of(group)
    if world == 1:
        return buf
    _, _, chunk = row_block(n, rank, world)
    if chunk == 0:
        return buf
    if dist.get_backend(group) == "nccl":
        # the local block as a separate input (no aliasing of the output)
        mine = buf[rank * chunk:(rank + 1) * chunk].clone()
        dist.all_gather_into_tensor(buf[:chunk * world], mine, group=group)
        return buf
    host = buf[:chunk * world].cpu()
    outs = list(host.view(world, chunk, -1).unbind(0))
    dist.all_gather(outs, host[rank * chunk:(rank + 1) * chunk].clone(), group=group)
    buf[:chunk * world].copy_(host)
    return buf


def part_owner(part: int, world: int) -> int:
    return part % world


def share_parts(books: list, stats: list, group=None) -> None:
    """Owner of part p (p % W) broadcasts its fitted codebook and stats."""
    rank, world = world_of(group)
    if world == 1:
        return
    for p in range(len(books)):
        obj = [(books[p], stats[p]) if part_owner(p, world) == rank else None]
        src = part_owner(p, world)
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, src) if group else src,
                                   group=group)
        books[p], stats[p] = obj[0]
