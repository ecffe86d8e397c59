"""Benchmark: GraphSAGE train seeds/sec on compressed features (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config products|arxiv|papers100m|mag240m]

Default workload (N=1): BASELINE configs[1] — synthetic ogbn-products-shape
graph (2,449,029 nodes, avg degree ~50, 100-dim class-conditional features),
3-layer GraphSAGE, fanouts [15,10,5], batch 1024, VQ codebooks of 256 entries
(width 4, cosine, CR 16).  A step = one full training step on one batch of
seeds: sample (device PCG64) -> fused gather-dequant-mean -> bf16 SAGE
fwd/bwd -> all-reduce (N>1) -> Adam, replayed from one CUDA graph.

Prints ONE JSON line (rank 0).  ``value`` is device-timed with CUDA events,
seeds already resident in HBM, L2 flushed between steps; ``e2e`` is the same
step through the public API with the seed ids copied from pinned host memory
and the loss read back every step.  ``--impl reference`` times the CPU oracle
port of the reference path (numpy sampler + decoder restating pipeline.py /
vq.py / sq.py, plus a CPU fp32 PyTorch SAGE step) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIGS = {
    # name: (shape, codec, fanouts, batch, hidden)
    "products": ("products", ("vq", 4, 256), (15, 10, 5), 1024, 256),
    "arxiv": ("arxiv", ("sq", 8), (10, 5), 1024, 256),
    "papers100m": ("papers100m", ("sq", 4), (15, 10, 5), 1024, 256),
    "mag240m": ("mag240m", ("vq", 8, 256), (15, 10, 5), 1024, 256),
    # BASELINE config E: aggregator variants through the fused gather path
    "products-gcn": ("products", ("sq", 8), (15, 10, 5), 1024, 256, "gcn"),
    "products-sq8": ("products", ("sq", 8), (15, 10, 5), 1024, 256),
    "products-gat": ("products", ("sq", 8), (15, 10, 5), 1024, 256, "gat"),
}


def aggregator_of(cfg_name):
    spec = CONFIGS[cfg_name]
    return spec[5] if len(spec) > 5 else "mean"


def committed_traffic(config):
    """dram bytes per launch of the fused kernel from the committed ncu
    capture of this workload (profiles/<round>/fused_<config>_summary.json,
    written by tools/summarize_profiles.py), or None."""
    import glob
    best = None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for f in sorted(glob.glob(os.path.join(REPO, "profiles", "*", f"fused_{config}_summary.json"))):
        try:
            k = json.load(open(f))["kernels"][0]
            rd = float(k["dram__bytes_read.sum"][0].replace(",", ""))
            wr = float(k["dram__bytes_write.sum"][0].replace(",", ""))
            best = int(rd * scale[k["dram__bytes_read.sum"][1]] +
                       wr * scale[k["dram__bytes_write.sum"][1]])
        except Exception:
            continue
    return best


def gather_ceiling(row_bytes):
    """Measured random-row gather throughput (rows + 8 B index per row) for
    the nearest probed row size, 7 GB table (tools/gather_probe.py,
    profiles/*/gather_probe.json), or None.  A uniformly random gather of
    small rows is bounded by DRAM sector/activation rate, far below the
    sequential copy peak; this is the practical ceiling for the fused kernel."""
    import glob
    fs = sorted(glob.glob(os.path.join(REPO, "profiles", "*", "gather_probe.json")))
    if not fs:
        return None
    d = json.load(open(fs[-1]))
    sizes = [32, 64, 128, 256, 512]
    best = min(sizes, key=lambda r: (r < row_bytes, abs(r - row_bytes)))
    e = d.get(f"7GB_row{best}")
    return None if e is None else {"row_bytes_probed": best, "GBps": e["GBps_rows_and_idx"]}


def load_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi style clock / throttle sampling during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks"}

    def __init__(self, index=0, period=0.05):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.pynvml = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass
        self.period = period
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.pynvml.nvmlDeviceGetClockInfo(self.h,
                                                                       self.pynvml.NVML_CLOCK_SM))
                r = self.pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.ok:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join(2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons)}


# ------------------------------------------------------------------ setup

def build_workload(cfg_name, device, seed=0, scale=1.0):
    import torch
    from paper_2207_14696_b200.synth import SHAPES, build_sq_codec, build_vq_codec, make_shape
    shape, codec_spec, fanouts, bs, hidden = CONFIGS[cfg_name][:5]
    t0 = time.perf_counter()
    sg = make_shape(shape, seed=seed, scale=scale, device=device)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    n, d = sg.graph.n, SHAPES[shape]["d"]
    import torch.distributed as dist
    # N>1: rows encoded per rank block + one all-gather, VQ parts fitted round-robin
    group = dist.group.WORLD if dist.is_initialized() and dist.get_world_size() > 1 else None
    if codec_spec[0] == "vq":
        dc, host_codec = build_vq_codec(n, d, codec_spec[1], codec_spec[2], labels=sg.labels,
                                        num_classes=sg.num_classes, seed=seed, group=group)
        codec_desc = f"vq width {codec_spec[1]} length {codec_spec[2]} cosine (CR {32 * codec_spec[1] / math.log2(codec_spec[2]):.0f})"
    else:
        dc = build_sq_codec(n, d, codec_spec[1], labels=sg.labels, num_classes=sg.num_classes,
                            seed=seed, group=group)
        codec_desc = f"sq k={codec_spec[1]} (CR {32 / codec_spec[1]:.0f})"
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"[bench] {cfg_name}: graph n={sg.graph.n} nnz={sg.graph.nnz} built in {t1 - t0:.1f} s, "
          f"codec ({codec_desc}) in {t2 - t1:.1f} s, "
          f"{torch.cuda.max_memory_allocated(device) / 2**30:.1f} GiB peak", file=sys.stderr,
          flush=True)
    return sg, dc, codec_desc, fanouts, bs, hidden


def flush_l2(buf):
    buf.add_(1)  # 512 MB write > 126 MB L2


# ------------------------------------------------------------- our arm

def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist
    from paper_2207_14696_b200 import _native as N
    from paper_2207_14696_b200 import ddp
    from paper_2207_14696_b200.aggregate import gather_dequant_mean
    from paper_2207_14696_b200.sage import SageTrainer, TrainConfig

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    sg, dc, codec_desc, fanouts, bs, hidden = build_workload(args.config, dev, scale=args.scale)
    pg = dist.group.WORLD if world > 1 else None
    agg_kind = aggregator_of(args.config)
    if agg_kind == "gat":
        from paper_2207_14696_b200.gat import GatConfig, GatTrainer
        tr = GatTrainer(sg.graph, dc, sg.labels, sg.num_classes,
                        GatConfig(fanouts=fanouts, batch_size=bs, hidden=hidden, lr=3e-3),
                        process_group=pg)
    else:
        cfg = TrainConfig(fanouts=fanouts, batch_size=bs, hidden=hidden, lr=3e-3, seed=0,
                          aggregator=agg_kind)
        tr = SageTrainer(sg.graph, dc, sg.labels, sg.num_classes, cfg, process_group=pg)
    nb = tr.begin_epoch(sg.train_ids, 0)
    need = args.warmup + 2 * args.steps + 3
    if nb < need:
        raise SystemExit(f"epoch has {nb} batches per rank, need {need}")
    tr.capture(warmup_batches=max(3, args.warmup))
    flush = torch.zeros(128 * 1024 * 1024, dtype=torch.float32, device=dev)
    # warm-up replays
    for b in range(args.warmup):
        tr.step(b)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # ---- timed: K steps, seeds resident, L2 flushed between steps
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    l0 = N.lib().fg_launch_count()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            b = args.warmup + i
            flush_l2(flush)
            tr.prepare(b)  # stage seeds (device copy), outside the timed region
            evs[i][0].record()
            tr.replay(b)
            evs[i][1].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_ms = sum(s.elapsed_time(e) for s, e in evs)
    t_ms = ddp.max_over_ranks(t_ms, dev)
    # launches per step: one eager step counted by the library's counter
    b = args.warmup + args.steps
    tr.prepare(b)
    torch.cuda.synchronize()
    c0 = N.lib().fg_launch_count()
    tr._body(b % len(tr.samplers))
    torch.cuda.synchronize()
    launches_per_step = N.lib().fg_launch_count() - c0
    # ---- e2e: public API, seeds from pinned host, loss read back each step
    # step b's host input: the seeds of the batch it samples (b+1 when the
    # trainer pipelines sampling one batch ahead, else b)
    perm = tr.sampler.perm_host
    b0 = args.warmup + args.steps + 1
    ahead = 1 if tr.pipeline else 0
    pinned = [torch.from_numpy(perm[(b0 + i + ahead) * bs:(b0 + i + ahead + 1) * bs].copy())
              .pin_memory() for i in range(args.steps)]
    loss_host = torch.zeros((), dtype=torch.float32).pin_memory()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e_ms = 0.0
    for i in range(args.steps):
        flush_l2(flush)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        loss = tr.step(b0 + i, seeds_host=pinned[i])
        loss_host.copy_(loss, non_blocking=True)
        e.record()
        e.synchronize()
        e2e_ms += s.elapsed_time(e)
    e2e_ms = ddp.max_over_ranks(e2e_ms, dev)
    # ---- roofline: the fused gather-dequant-mean kernel, timed alone
    L = len(fanouts)
    row_bytes = dc.num_parts * dc.bits / 8 if hasattr(dc, "num_parts") else dc.d * dc.params.k / 8
    kt, kbytes = [], []
    for i in range(args.steps):
        tr.sampler.load_seeds(args.warmup + i)
        sb = tr.sampler.sample_loaded()
        torch.cuda.synchronize()
        E = int(sb.n_picks[L - 1].item())
        nd = int(sb.n_nodes[L - 1].item())
        flush_l2(flush)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # (the 512 MB flush still running on the device covers the host-side
        # enqueue, so the event pair brackets the kernel alone)
        s.record()
        if agg_kind == "gat":  # GAT decodes one row per pick (attention needs each source)
            dc.gather(sb.picks[L - 1], out_dtype=torch.bfloat16, check=False)
        else:
            gather_dequant_mean(dc, sb.indptr[L - 1], sb.picks[L - 1], sb.n_nodes[L - 1],
                                tr.caps[L - 1], out=tr.agg,
                                edge_w=sb.ew[L - 1] if sb.ew else None)
        e.record()
        e.synchronize()
        kt.append(s.elapsed_time(e))
        if agg_kind == "gat":  # E code rows + int32 ids in, E bf16 rows out
            kbytes.append(E * (row_bytes + 4) + E * dc.d * 2)
            continue
        out_b = tr.agg.element_size()
        # algorithmic bytes: E code rows + int32 source ids, N_dst indptr
        # entries + output rows (the padded rows past N_dst are zero-filled
        # but not counted)
        # (+4 B edge weight per pick for the weighted aggregators)
        wb = 4 if agg_kind != "mean" else 0
        kbytes.append(E * (row_bytes + 4 + wb) + nd * (4 + dc.d * out_b))
    avg_ms = sum(kt) / len(kt)
    ceiling = gather_ceiling(row_bytes)
    avg_bytes = sum(kbytes) / len(kbytes)
    peak, peak_kind = load_peaks()
    achieved = avg_bytes / (avg_ms * 1e-3) / 1e9
    seeds_per_step = bs * world
    value = seeds_per_step * args.steps / (t_ms * 1e-3)
    e2e = seeds_per_step * args.steps / (e2e_ms * 1e-3)
    result = {
        "metric": "GraphSAGE train seeds/sec",
        "value": round(value, 1),
        "unit": "seeds/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(t_ms / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (planted-partition power-law graph, class-conditional features)",
        "config": {"workload": f"{args.config}-shape "
                               f"{dict(gcn='GCN', gat='GAT').get(agg_kind, 'GraphSAGE')} "
                               f"{len(fanouts)}-layer "
                               f"fanout {list(fanouts)}, {codec_desc}",
                   "nodes": sg.graph.n, "edges_stored": sg.graph.nnz, "feature_dim": dc.d,
                   "global_batch": seeds_per_step, "per_rank_batch": bs, "hidden": hidden,
                   "parallelism": f"dp{world}", "l2": "flushed between steps (512 MB write)",
                   "graph": "one CUDA graph per step"},
        "e2e": {"value": round(e2e, 1), "unit": "seeds/s",
                "h2d_bytes_per_step": bs * 8, "d2h_bytes_per_step": 4},
        "gpu_launches": int(launches_per_step * args.steps),
        "roofline": {"kernel": ("fg_sq_gather_dequant / fg_vq_gather_decode" if agg_kind == "gat"
                               else "fg_gather_dequant_mean (k_vq_mean8_fast / k_sq_mean)"),
                     "bound": "hbm",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                     "traffic": committed_traffic(args.config),
                     "avg_launch_us": round(avg_ms * 1e3, 2),
                     "alg_bytes_per_launch": int(avg_bytes),
                     "random_gather_ceiling": ceiling,
                     "frac_of_gather_ceiling": (round(achieved / ceiling["GBps"], 4)
                                                if ceiling else None)},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(sg, dc, fanouts, hidden, budget_s=args.cpu_budget,
                                              aggregator=agg_kind)
    if rank == 0:
        print(json.dumps(result), flush=True)


# ------------------------------------------------------- CPU baseline

def _host_world(sg, dc):
    """Host copies for the CPU oracle: CSR, labels, decoder over codes."""
    host = sg.graph.to_host()
    labels = sg.labels.cpu().numpy()
    from oracle import codecs as oc
    from paper_2207_14696_b200.vq import DeviceVqCodec
    if isinstance(dc, DeviceVqCodec):
        import torch
        codes = torch.empty((dc.n, dc.num_parts), dtype=torch.int32, device=dc.rows.device)
        # codes come back from the device rows via the reference layout
        rows = dc.rows.cpu().numpy()
        b = dc.bits
        assert b == 8, "CPU baseline decoder supports 8-bit VQ codes"
        codes = rows[:, :dc.num_parts].astype(np.int32)
        books = dc.books_host
        w = dc.params.width

        def decode(r):
            return oc.vq_decode(codes, books, dc.d, w, r)
    else:
        c = dc.to_codec()
        p = c.params

        def decode(r):
            return oc.sq_dequant_rows(c.payload, c.n, c.d, p.k, p.e_min, p.e_max, r)
    return host, labels, decode


def oracle_model(ot, d, hidden, num_classes, fanouts, aggregator):
    """CPU fp32 oracle model + one-batch train function for the aggregator."""
    if aggregator == "gat":
        def step(model, opt, host, labels, ids, fanouts, batch, seed, decode):
            ot.gat_train_epoch(model, opt, host.row_offsets, host.col_indices, labels, ids,
                               fanouts, batch, seed, decode)
        return ot.OracleGat(d, hidden, num_classes, len(fanouts)), step

    def step(model, opt, host, labels, ids, fanouts, batch, seed, decode):
        ot.train_epoch(model, opt, host.row_offsets, host.col_indices, labels, ids, fanouts,
                       batch, seed, decode, aggregator=aggregator)
    return ot.OracleSage(d, hidden, num_classes, len(fanouts)), step


# ------------------------------------------- shard-parallel CPU baseline
# The reference is single-threaded numpy; its best case on a multi-core host
# is P independent processes over disjoint batches.
# Workers are SPAWNED (a forked child of a process that already ran torch /
# OpenMP can deadlock) and map the host world from .npy files (mmap, shared).

def save_host_world(host, labels, train, dc, path):
    """Host CSR, labels, train ids and the codec's host form as .npy files."""
    from paper_2207_14696_b200.vq import DeviceVqCodec
    meta = {"n": int(host.n), "d": int(dc.d)}
    np.save(os.path.join(path, "off.npy"), np.asarray(host.row_offsets))
    np.save(os.path.join(path, "col.npy"), np.asarray(host.col_indices))
    np.save(os.path.join(path, "labels.npy"), np.asarray(labels))
    np.save(os.path.join(path, "train.npy"), np.asarray(train))
    if isinstance(dc, DeviceVqCodec):
        rows = dc.rows.cpu().numpy()
        np.save(os.path.join(path, "codes.npy"), rows[:, :dc.num_parts].astype(np.int32))
        for p_, b in enumerate(dc.books_host):
            np.save(os.path.join(path, f"book{p_}.npy"), np.asarray(b))
        meta.update(kind="vq", width=int(dc.params.width), parts=int(dc.num_parts))
    else:
        c = dc.to_codec()
        np.save(os.path.join(path, "payload.npy"), np.frombuffer(c.payload, np.uint8))
        meta.update(kind="sq", k=int(c.params.k), e_min=float(c.params.e_min),
                    e_max=float(c.params.e_max))
    return meta


def _load_world(path, meta):
    from oracle import codecs as oc
    ld = lambda f: np.load(os.path.join(path, f), mmap_mode="r")  # noqa: E731
    w = {"off": ld("off.npy"), "col": ld("col.npy"), "labels": ld("labels.npy"),
         "train": ld("train.npy")}
    if meta["kind"] == "vq":
        codes = ld("codes.npy")
        books = tuple(np.load(os.path.join(path, f"book{p}.npy")) for p in range(meta["parts"]))
        w["decode"] = lambda r: oc.vq_decode(codes, books, meta["d"], meta["width"], r)
    else:
        payload = ld("payload.npy")
        w["decode"] = lambda r: oc.sq_dequant_rows(payload, meta["n"], meta["d"], meta["k"],
                                                   meta["e_min"], meta["e_max"], r)
    return w


def _spawn_worker(path, meta, cfg, wid, nsteps, warm, barrier, q):
    import torch
    from oracle import trainer as ot
    torch.set_num_threads(1)
    w = _load_world(path, meta)
    model, step = oracle_model(ot, meta["d"], cfg["hidden"], cfg["classes"], cfg["fanouts"],
                               cfg["agg"])
    opt = torch.optim.Adam(model.parameters(), lr=3e-3)

    class H:  # what the oracle train functions read
        row_offsets, col_indices = w["off"], w["col"]
    batch, train = cfg["batch"], w["train"]
    nb = max(1, train.size // batch)

    def one(b):
        step(model, opt, H, w["labels"], np.asarray(train[b * batch:(b + 1) * batch]),
             cfg["fanouts"], batch, b, w["decode"])
    for i in range(warm):
        one((wid * (nsteps + warm) + nsteps + i) % nb)
    barrier.wait()
    t0 = time.perf_counter()
    for i in range(nsteps):
        one((wid * (nsteps + warm) + i) % nb)
    q.put((wid, time.perf_counter() - t0))


def cpu_parallel_from_dir(path, meta, cfg, nsteps, warm=0, workers=None, timeout=600.0):
    """Run `workers` spawned oracle processes, each `nsteps` batches; returns
    (seeds, wall seconds, workers) or None if they do not finish in time."""
    import multiprocessing as mp
    workers = workers or os.cpu_count() or 1
    ctx = mp.get_context("spawn")
    barrier, q = ctx.Barrier(workers + 1), ctx.Queue()
    procs = [ctx.Process(target=_spawn_worker,
                         args=(path, meta, cfg, w, nsteps, warm, barrier, q), daemon=True)
             for w in range(workers)]
    for pr in procs:
        pr.start()
    try:
        barrier.wait(timeout=timeout)
        t0 = time.perf_counter()
        done = [q.get(timeout=timeout) for _ in range(workers)]
        wall = time.perf_counter() - t0
    except Exception:
        for pr in procs:
            pr.kill()
        return None
    for pr in procs:
        pr.join(30)
    return workers * nsteps * cfg["batch"], max(wall, max(t for _, t in done)), workers


def cpu_parallel(sg, dc, fanouts, hidden, aggregator, batch, nsteps, warm=0):
    """None when the pool cannot run (no space for the world files, spawn
    failure, timeout): callers fall back to the single-process timing."""
    import shutil
    import tempfile
    host = sg.graph.to_host()
    for base in ("/dev/shm", None):  # tmpfs first; /dev/shm may be small in containers
        if base and not os.path.isdir(base):
            continue
        path = tempfile.mkdtemp(prefix="fgb_cpu_", dir=base)
        try:
            meta = save_host_world(host, sg.labels.cpu().numpy(), sg.train_ids, dc, path)
            cfg = {"hidden": hidden, "classes": sg.num_classes, "fanouts": tuple(fanouts),
                   "agg": aggregator, "batch": batch}
            return cpu_parallel_from_dir(path, meta, cfg, nsteps, warm)
        except Exception as e:  # noqa: BLE001 - any failure -> next base / fallback
            print(f"[bench] shard-parallel CPU baseline unavailable under {base or 'tmp'}: "
                  f"{e}", file=sys.stderr)
        finally:
            shutil.rmtree(path, ignore_errors=True)
    return None


def cpu_baseline(sg, dc, fanouts, hidden, budget_s=20.0, batch=128, aggregator="mean"):
    """Oracle port of the reference path on the host cores: numpy sampler
    (pipeline.py:185-222 restated) + numpy decoder + CPU fp32 SAGE step."""
    import torch
    from oracle import trainer as ot
    host, labels, decode = _host_world(sg, dc)
    model, train_step = oracle_model(ot, dc.d, hidden, sg.num_classes, fanouts, aggregator)
    opt = torch.optim.Adam(model.parameters(), lr=3e-3)
    # size the shard-parallel run from one single-threaded batch (~budget_s)
    nt = torch.get_num_threads()
    torch.set_num_threads(1)
    t0 = time.perf_counter()
    train_step(model, opt, host, labels, sg.train_ids[:batch], fanouts, batch, 0, decode)
    per = time.perf_counter() - t0
    torch.set_num_threads(nt)
    par = cpu_parallel(sg, dc, fanouts, hidden, aggregator, batch,
                       max(1, int(budget_s / max(per, 1e-3))), warm=1)
    if par is not None:
        seeds, wall, workers = par
        return {"value": round(seeds / wall, 2), "unit": "seeds/s", "cores": workers,
                "kind": "port",
                "sample": f"{workers} spawned processes x {seeds // workers // batch} "
                          f"mini-batches of {batch} seeds, fanouts {list(fanouts)}, "
                          f"{wall:.1f} s wall (oracle port, one thread each, disjoint batches)"}
    seeds_done, t0, steps = 0, time.perf_counter(), 0
    train = sg.train_ids
    while True:
        train_step(model, opt, host, labels, train[steps * batch:(steps + 1) * batch], fanouts,
                   batch, steps, decode)
        steps += 1
        seeds_done += batch
        if time.perf_counter() - t0 >= budget_s or steps * batch >= train.size:
            break
    dt = time.perf_counter() - t0
    return {"value": round(seeds_done / dt, 2), "unit": "seeds/s",
            "cores": torch.get_num_threads(), "kind": "port",
            "sample": f"{steps} mini-batches of {batch} seeds, fanouts {list(fanouts)}, "
                      f"{dt:.1f} s (numpy sampler/decoder single-threaded, torch CPU "
                      f"fp32 SAGE step on {torch.get_num_threads()} threads)"}


def run_reference(args, rank, world, local):
    """The reference arm: CPU oracle port, rank 0 only."""
    if rank != 0:
        return
    import torch
    from oracle import trainer as ot
    dev = torch.device("cuda", local) if torch.cuda.is_available() else torch.device("cpu")
    if dev.type == "cuda":
        torch.cuda.set_device(dev)
    sg, dc, codec_desc, fanouts, bs, hidden = build_workload(args.config, dev, scale=args.scale)
    agg = aggregator_of(args.config)
    par = cpu_parallel(sg, dc, fanouts, hidden, agg, args.ref_batch, args.steps,
                       warm=args.warmup)
    if par is not None:  # every host core: one process per core over disjoint batches
        seeds, dt, workers = par
        v = seeds / dt
        line = {"impl": "reference", "metric": "GraphSAGE train seeds/sec",
                "value": round(v, 2), "unit": "seeds/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(dt * 1e3 / args.steps, 2),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic",
                "config": {"workload": f"{args.config}-shape "
                                       f"{dict(gcn='GCN', gat='GAT').get(agg, 'GraphSAGE')} "
                                       f"{len(fanouts)}-layer fanout {list(fanouts)}, "
                                       f"{codec_desc}",
                           "per_step_seeds": args.ref_batch * workers,
                           "parallelism": f"cpu x{workers} processes"},
                "cpu_baseline": {"value": round(v, 2), "unit": "seeds/s", "cores": workers,
                                 "kind": "port",
                                 "sample": f"{args.steps} steps x {workers} processes x "
                                           f"{args.ref_batch} seeds (oracle port, one thread "
                                           f"per process)"},
                "e2e": {"value": round(v, 2), "unit": "seeds/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    host, labels, decode = _host_world(sg, dc)  # fallback: one process, all torch threads
    torch.set_num_threads(os.cpu_count() or 1)
    model, train_step = oracle_model(ot, dc.d, hidden, sg.num_classes, fanouts,
                                     aggregator_of(args.config))
    opt = torch.optim.Adam(model.parameters(), lr=3e-3)
    batch = args.ref_batch
    train = sg.train_ids

    def one(i):
        train_step(model, opt, host, labels, train[i * batch:(i + 1) * batch], fanouts, batch,
                   i, decode)

    for i in range(args.warmup):
        one(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        one(args.warmup + i)
    dt = time.perf_counter() - t0
    v = batch * args.steps / dt
    line = {"impl": "reference", "metric": "GraphSAGE train seeds/sec", "value": round(v, 2),
            "unit": "seeds/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt * 1e3 / args.steps, 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.config}-shape GraphSAGE {len(fanouts)}-layer fanout "
                                   f"{list(fanouts)}, {codec_desc}",
                       "per_step_seeds": batch, "parallelism": "cpu"},
            "cpu_baseline": {"value": round(v, 2), "unit": "seeds/s",
                             "cores": torch.get_num_threads(), "kind": "port",
                             "sample": f"{args.steps} steps x {batch} seeds"},
            "e2e": {"value": round(v, 2), "unit": "seeds/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="products")
    ap.add_argument("--scale", type=float, default=1.0, help="node-count scale (tests only)")
    ap.add_argument("--ref-batch", type=int, default=128)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    from paper_2207_14696_b200 import ddp
    backend = "nccl" if args.impl == "ours" else "gloo"
    rank, world, local = ddp.init_from_env(backend)
    try:
        if args.impl == "reference":
            run_reference(args, rank, world, local)
        else:
            run_ours(args, rank, world, local)
    finally:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
