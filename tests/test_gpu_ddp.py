"""Data-parallel trainer with two ranks on one GPU (gloo, eager steps): the
flat-gradient all-reduce keeps the replicas identical, each rank trains on
its own shard, and each rank's batches are the reference sampler's batches
for (shard_r, seed (seed+epoch)*W + r)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2207_14696_b200 import ddp
    from paper_2207_14696_b200.sage import SageTrainer, TrainConfig
    from paper_2207_14696_b200.synth import build_sq_codec, generate_graph, split_ids
    from oracle.sampler import sample_batches_oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        n, d, C = 12_000, 32, 6
        dg, labels = generate_graph(n, 12.0, C, seed=1)
        dc = build_sq_codec(n, d, 8, labels=labels, num_classes=C, seed=1)
        train, _ = split_ids(n, n // 4, n // 10, 1)
        fans = (10, 5)
        t = SageTrainer(dg, dc, labels, C, TrainConfig(fanouts=fans, batch_size=256, hidden=64),
                        process_group=dist.group.WORLD)
        nb = t.begin_epoch(train, 0)
        # this rank's first batch vs the oracle sampler on its shard
        t.prepare(0)
        sb = t.samplers[0].batch_view()
        host = dg.to_host()
        shard = ddp.shard_ids(train, rank, world)
        ref, _ = sample_batches_oracle(host.row_offsets, host.col_indices, shard, fans, 256,
                                       ddp.rank_seed(0, 0, rank, world), max_batches=1)
        npk = int(sb.n_picks[0].item())
        same_batch = bool(np.array_equal(sb.picks[0][:npk].cpu().numpy(), ref[0].layers[0].picks))
        for b in range(3):
            t.replay(b) if b == 0 else t.step(b)
        torch.cuda.synchronize()
        params = t.flat_param.detach().cpu()
        gathered = [torch.zeros_like(params) for _ in range(world)]
        dist.all_gather(gathered, params)
        q.put((rank, nb, same_batch, all(torch.equal(gathered[0], g) for g in gathered),
               float(t.loss_buf.item())))
    finally:
        dist.destroy_process_group()


def test_two_rank_trainer_stays_in_sync():
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(120)
    assert out[0][1] == out[1][1]            # agreed batch count
    assert out[0][2] and out[1][2]           # per-rank batches = reference sampler
    assert out[0][3] and out[1][3]           # identical parameters after 3 steps
    assert np.isfinite([o[4] for o in out]).all() and out[0][4] != out[1][4]  # own shards


def _prep_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2207_14696_b200.synth import build_sq_codec, build_vq_codec, generate_graph
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        n, C = 7_001, 5
        _, labels = generate_graph(n, 8.0, C, seed=2)
        out = {}
        for g in (None, dist.group.WORLD):
            sq = build_sq_codec(n, 40, 4, labels=labels, num_classes=C, seed=2,
                                chunk_rows=1000, group=g)
            vq, host = build_vq_codec(n, 24, 4, 16, labels=labels, num_classes=C, seed=2,
                                      chunk_rows=1000, max_iters=8, restarts=2, group=g)
            out[g is None] = (sq.rows.cpu().numpy().copy(), sq.params,
                              vq.rows.cpu().numpy().copy(), [b.copy() for b in host.codebooks])
        a, b = out[True], out[False]
        q.put((rank, np.array_equal(a[0], b[0]) and a[1] == b[1],
               np.array_equal(a[2], b[2]) and all(np.array_equal(x, y) for x, y in zip(a[3], b[3]))))
    finally:
        dist.destroy_process_group()


def test_sharded_preprocessing_matches_single_process():
    """Row-block encode + all-gather and round-robin VQ part fitting give the
    single-process codec bit for bit (SURVEY.md §8e preprocessing)."""
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_prep_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(120)
    assert all(o[1] for o in out), "SQ rows differ"
    assert all(o[2] for o in out), "VQ rows/codebooks differ"


def test_bench_two_ranks_prints_one_line():
    """``bench.py --gpus 2`` relaunches itself under torch.distributed.run;
    both ranks build the world, train (gloo here: the sandbox has one GPU,
    so the ranks share it and the steps stay eager -- with NCCL the
    all-reduce is captured in the step graph), and rank 0 alone prints one
    line with n_gpus 2 and the max-over-ranks timing."""
    import json
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FG_DIST_BACKEND="gloo")
    cmd = [sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2", "--config", "products",
           "--scale", "0.2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-epoch"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=repo)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "dp2"
    assert d["config"]["global_batch"] == 2048 and d["value"] > 0 and d["e2e"]["value"] > 0
