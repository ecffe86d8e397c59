"""Benchmark: GraphSAGE train seeds/sec on compressed features (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config papers100m|products|arxiv|mag240m|products-gcn|...]

Default workload: BASELINE config C, the one the metric's "seeds/sec at
1/2/4/8 B200" is quoted on -- a synthetic ogbn-papers100M-shape graph
(111,059,956 nodes, ~3.2e9 stored entries, 128-dim class-conditional
features, 4-bit SQ), 3-layer GraphSAGE, fanouts [15,10,5], 1024 seeds per
rank per step.  A step = one full training step on one batch: sample (device
PCG64) -> fused gather-dequant-mean -> bf16 SAGE fwd/bwd -> all-reduce (N>1)
-> Adam, replayed from one CUDA graph.

Prints ONE JSON line (rank 0).  ``value``: K steps device-timed with CUDA
events, seeds resident in HBM, L2 flushed between steps, max over ranks;
``e2e``: the same steps through the public API with the seed ids copied from
pinned host memory and the loss read back every step; ``epoch``: one whole
epoch (begin_epoch's host permutation + upload included) on the wall clock.

``--gpus N`` (N > 1) without a torchrun environment re-launches itself under
``torch.distributed.run`` with N ranks (NCCL, one GPU each).

``--impl reference`` times the reference's own CPU implementation of the path
(SURVEY.md §8(d)): the unmodified ``featgrind`` from ``baseline/_ref``
(sample_batches + dequantize_sq of each batch's frontier, loader-only: the
reference has no trainer) on every host core, over the SAME world -- graph,
labels, split and SQ payload rebuilt bit-identically on the CPU by
oracle/world.py (this process never loads the product library).
"""

from __future__ import annotations

import argparse
import json
import os
import shutil
import socket
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# BASELINE.json configs.  Shapes (nodes, dim, avg degree, classes, train
# split) mirror paper_2207_14696_b200/synth.py SHAPES (tests check they are
# equal); kept here so the reference arm needs no product import.
SHAPES = {
    "arxiv": dict(n=169_343, d=128, avg_deg=13.7, classes=40, train=90_941),
    "products": dict(n=2_449_029, d=100, avg_deg=50.5, classes=47, train=196_615),
    "papers100m": dict(n=111_059_956, d=128, avg_deg=29.1, classes=172, train=1_207_179),
    "mag240m": dict(n=244_160_499, d=768, avg_deg=27.9, classes=153, train=1_112_392),
}
CONFIGS = {
    # name: (shape, codec, fanouts, batch, hidden[, aggregator])
    "papers100m": ("papers100m", ("sq", 4), (15, 10, 5), 1024, 256),
    "products": ("products", ("vq", 4, 256), (15, 10, 5), 1024, 256),
    "arxiv": ("arxiv", ("sq", 8), (10, 5), 1024, 256),
    "mag240m": ("mag240m", ("vq", 8, 256), (15, 10, 5), 1024, 256),
    # BASELINE config E: aggregator variants through the fused gather path
    "products-gcn": ("products", ("sq", 8), (15, 10, 5), 1024, 256, "gcn"),
    "products-sq8": ("products", ("sq", 8), (15, 10, 5), 1024, 256),
    "products-gat": ("products", ("sq", 8), (15, 10, 5), 1024, 256, "gat"),
}
DEFAULT_CONFIG = "papers100m"
METRIC = "GraphSAGE train seeds/sec"


def aggregator_of(cfg_name):
    spec = CONFIGS[cfg_name]
    return spec[5] if len(spec) > 5 else "mean"


def shape_of(cfg_name, scale=1.0):
    s = dict(SHAPES[CONFIGS[cfg_name][0]])
    s["n"] = max(1000, int(s["n"] * scale))
    s["train"] = max(1, int(s["train"] * scale))
    return s


def codec_desc(cfg_name):
    c = CONFIGS[cfg_name][1]
    if c[0] == "vq":
        import math
        return f"vq width {c[1]} length {c[2]} cosine (CR {32 * c[1] / math.log2(c[2]):.0f})"
    return f"sq k={c[1]} (CR {32 // c[1]})"


def workload_config(cfg_name, nnz, world, scale=1.0):
    """The ``config`` object of the JSON line -- built the same way by both
    arms from the workload alone."""
    shape, _, fanouts, bs, hidden = CONFIGS[cfg_name][:5]
    s = shape_of(cfg_name, scale)
    agg = aggregator_of(cfg_name)
    return {"workload": f"{shape}-shape {dict(gcn='GCN', gat='GAT').get(agg, 'GraphSAGE')} "
                        f"{len(fanouts)}-layer fanout {list(fanouts)}, {codec_desc(cfg_name)}",
            "nodes": s["n"], "edges_stored": int(nnz), "feature_dim": s["d"],
            "fanouts": list(fanouts), "global_batch": bs * world, "per_rank_batch": bs,
            "hidden": hidden, "train_ids": s["train"], "parallelism": f"dp{world}"}


def committed_traffic(config):
    """dram bytes per launch of the fused kernel from the newest committed ncu
    --set full capture of this workload (profiles/<round>/fused_<config>_
    summary.json, tools/summarize_profiles.py), and its file, or (None, None)."""
    import glob
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    best = (None, None)
    for f in sorted(glob.glob(os.path.join(REPO, "profiles", "*", f"fused_{config}_summary.json"))):
        try:
            k = json.load(open(f))["kernels"][0]
            rd = float(k["dram__bytes_read.sum"][0].replace(",", ""))
            wr = float(k["dram__bytes_write.sum"][0].replace(",", ""))
            best = (int(rd * scale[k["dram__bytes_read.sum"][1]] +
                        wr * scale[k["dram__bytes_write.sum"][1]]), os.path.relpath(f, REPO))
        except Exception:
            continue
    return best


def gather_ceiling(row_bytes):
    """Measured random-row gather throughput (rows + 8 B index per row) for
    the nearest probed row size, 7 GB table (tools/gather_probe.py,
    profiles/*/gather_probe.json), or None: a uniformly random gather of
    small rows is bounded by the DRAM sector/activation rate, far below the
    sequential copy peak."""
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
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


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


def world_dir(prefix):
    """A scratch directory for a host world, on tmpfs when it has room."""
    for base in ("/dev/shm", None):
        if base and not os.path.isdir(base):
            continue
        try:
            return tempfile.mkdtemp(prefix=prefix, dir=base)
        except OSError:
            continue
    raise RuntimeError("no scratch directory for the host world")


# ------------------------------------------------------------------ setup

def build_workload(cfg_name, device, seed=0, scale=1.0):
    import torch
    from paper_2207_14696_b200.synth import build_sq_codec, build_vq_codec, make_shape
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
        dc, _ = build_vq_codec(n, d, codec_spec[1], codec_spec[2], labels=sg.labels,
                               num_classes=sg.num_classes, seed=seed, group=group)
    else:
        dc = build_sq_codec(n, d, codec_spec[1], labels=sg.labels, num_classes=sg.num_classes,
                            seed=seed, group=group)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"[bench] {cfg_name}: graph n={sg.graph.n} nnz={sg.graph.nnz} built in {t1 - t0:.1f} s, "
          f"codec ({codec_desc(cfg_name)}) in {t2 - t1:.1f} s, "
          f"{torch.cuda.max_memory_allocated(device) / 2**30:.1f} GiB peak", file=sys.stderr,
          flush=True)
    return sg, dc, codec_desc(cfg_name), fanouts, bs, hidden


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
    sg, dc, _, fanouts, bs, hidden = build_workload(args.config, dev, scale=args.scale)
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
    need = 2 * args.warmup + 2 * args.steps + 3
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
    # (each batch's slice of perm_host is already its sorted seed list)
    wu = args.warmup
    pinned = [torch.from_numpy(perm[(b0 + i + ahead) * bs:(b0 + i + ahead + 1) * bs]
                               .astype(np.int32)).pin_memory() for i in range(wu + args.steps)]
    # every step's loss lands in its own pinned host slot (a D2H copy per
    # step inside the timed region); the host does not block per step -- it
    # enqueues steps back to back like a training loop and synchronises once
    loss_host = torch.zeros(wu + args.steps, dtype=torch.float32).pin_memory()
    for i in range(wu):  # untimed e2e warm-up (first use of the pinned buffers)
        flush_l2(flush)
        loss = tr.step(b0 + i, seeds_host=pinned[i])
        loss_host[i].copy_(loss, non_blocking=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e_ms = 0.0
    for i in range(args.steps):
        flush_l2(flush)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        loss = tr.step(b0 + wu + i, seeds_host=pinned[wu + i])
        loss_host[wu + i].copy_(loss, non_blocking=True)
        e.record()
        evs[i] = (s, e)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(loss_host).all()), "non-finite loss read back"
    e2e_ms = sum(s.elapsed_time(e) for s, e in evs)
    e2e_ms = ddp.max_over_ranks(e2e_ms, dev)
    # ---- one whole epoch on the wall clock (epoch 1: new permutation)
    epoch = None
    if not args.no_epoch:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        nb1 = tr.begin_epoch(sg.train_ids, 1)
        t1 = time.perf_counter()
        for b in range(nb1):
            tr.step(b)
        t2 = time.perf_counter()
        torch.cuda.synchronize()
        ep_s = ddp.max_over_ranks(time.perf_counter() - t0, dev)
        epoch = {"seeds_per_s": round(nb1 * bs * world / ep_s, 1), "wall_s": round(ep_s, 4),
                 "begin_epoch_s": round(t1 - t0, 4), "enqueue_s": round(t2 - t1, 4),
                 "begin_epoch_parts_s": {k: round(v, 4) for k, v in
                                         {**getattr(tr, "begin_epoch_timing", {}),
                                          **getattr(tr.sampler, "begin_epoch_timing",
                                                    {})}.items()},
                 "batches_per_rank": nb1, "includes": "begin_epoch (host permutation + "
                 "upload) + every batch of the epoch, wall clock, max over ranks"}
    # ---- roofline: the fused gather-dequant-mean kernel, timed alone
    L = len(fanouts)
    row_bytes = dc.num_parts * dc.bits / 8 if hasattr(dc, "num_parts") else dc.d * dc.params.k / 8
    kt, kbytes = [], []
    # the sampler alone (sampler edges/s), replayed from a CUDA
    # graph as in the training step (eager, its ~40 small launches would be
    # host-bound); eager if the capture is refused
    st_ms, st_edges = [], []
    samp_graph = None
    try:
        tr.sampler.load_seeds(args.warmup)
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            tr.sampler.sample_loaded()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        samp_graph = torch.cuda.CUDAGraph()
        tr.sampler.load_seeds(args.warmup)
        with torch.cuda.graph(samp_graph):
            tr.sampler.sample_loaded()
        for w in range(2):  # untimed replays (the first one uploads the graph)
            tr.sampler.load_seeds(args.warmup + w)
            samp_graph.replay()
        torch.cuda.synchronize()
    except Exception as ex:  # noqa: BLE001 -- diagnostic leg only
        print(f"[bench] sampler graph capture refused ({ex}); timing it eagerly", file=sys.stderr)
        samp_graph = None
        torch.cuda.synchronize()
    for i in range(args.steps):
        tr.sampler.load_seeds(args.warmup + i)
        flush_l2(flush)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        if samp_graph is not None:
            samp_graph.replay()
            sb = tr.sampler.batch_view()
        else:
            sb = tr.sampler.sample_loaded()
        s1.record()
        torch.cuda.synchronize()
        st_ms.append(s0.elapsed_time(s1))
        st_edges.append(sum(int(x.item()) for x in sb.n_picks))
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
        # entries + output rows (+4 B edge weight per pick when weighted)
        wb = 4 if agg_kind != "mean" else 0
        kbytes.append(E * (row_bytes + 4 + wb) + nd * (4 + dc.d * out_b))
    avg_ms = sum(kt) / len(kt)
    ceiling = gather_ceiling(row_bytes)
    avg_bytes = sum(kbytes) / len(kbytes)
    peak, peak_kind = load_peaks()
    achieved = avg_bytes / (avg_ms * 1e-3) / 1e9
    traffic, traffic_src = committed_traffic(args.config)
    seeds_per_step = bs * world
    value = seeds_per_step * args.steps / (t_ms * 1e-3)
    e2e = seeds_per_step * args.steps / (e2e_ms * 1e-3)
    result = {
        "metric": METRIC,
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
        "config": workload_config(args.config, sg.graph.nnz, world, args.scale),
        "timing": {"l2": "flushed between steps (512 MB write)",
                   "graph": "one CUDA graph per step", "clock": "CUDA events, max over ranks"},
        "e2e": {"value": round(e2e, 1), "unit": "seeds/s",
                "h2d_bytes_per_step": bs * 4, "d2h_bytes_per_step": 4,
                "method": "public API (trainer.step with pinned host seeds, loss copied to a "
                          "pinned host slot every step), W untimed e2e warm-up steps, then K "
                          "steps enqueued back to back, CUDA events around each step, one "
                          "host sync after the K steps"},
        "epoch": epoch,
        "sampler": {"edges_per_s": round(sum(st_edges) / (sum(st_ms) * 1e-3), 1),
                    "us_per_batch": round(sum(st_ms) / len(st_ms) * 1e3, 2),
                    "edges_per_batch": int(sum(st_edges) / len(st_edges)),
                    "graphed": samp_graph is not None,
                    "method": "one batch's sampling alone (all layers: prefix, sample, fix-up, "
                              "unique, transposes) replayed from a CUDA graph, L2 flushed "
                              "before, CUDA events; in the training step it runs overlapped "
                              "on a side stream"},
        "gpu_launches": int(launches_per_step * args.steps),
        "roofline": {"kernel": ("fg_sq_gather_dequant / fg_vq_gather_decode" if agg_kind == "gat"
                               else "fg_gather_dequant_mean"),
                     "bound": "hbm",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "avg_launch_us": round(avg_ms * 1e3, 2),
                     "alg_bytes_per_launch": int(avg_bytes),
                     "random_gather_ceiling": ceiling,
                     "frac_of_gather_ceiling": (round(achieved / ceiling["GBps"], 4)
                                                if ceiling else None)},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            result["cpu_baseline"] = cpu_baseline(args, sg, dc, fanouts, bs)
        except Exception as e:  # noqa: BLE001 - reported, never fatal to the GPU line
            result["cpu_baseline"] = {"value": None, "unavailable": repr(e)[:300]}
    if rank == 0:
        print(json.dumps(result), flush=True)


# ------------------------------------------------------- CPU baseline

def export_device_world(sg, dc, path):
    """Our arm's device world as oracle/world.py files (CSR, labels, train
    ids, the reference's continuous SQ payload): the CPU leg then times the
    reference loader on exactly the data the GPU trained on."""
    from paper_2207_14696_b200.sq import DeviceSqCodec
    if not isinstance(dc, DeviceSqCodec):
        raise RuntimeError("the reference loader baseline covers SQ workloads "
                           "(dequantize_sq); VQ configs report no cpu_baseline")
    host = sg.graph
    host.row_offsets.cpu().numpy().tofile(os.path.join(path, "off.bin"))
    host.col_indices.cpu().numpy().tofile(os.path.join(path, "col.bin"))
    sg.labels.cpu().numpy().astype(np.int32).tofile(os.path.join(path, "labels.bin"))
    np.asarray(sg.train_ids, np.int64).tofile(os.path.join(path, "train.bin"))
    c = dc.to_codec()
    np.frombuffer(c.payload, np.uint8).tofile(os.path.join(path, "payload.bin"))
    meta = {"n": int(dc.n), "nnz": int(host.nnz), "d": int(dc.d), "k": int(c.params.k),
            "e_min": float(c.params.e_min), "e_max": float(c.params.e_max),
            "train": int(np.asarray(sg.train_ids).size), "seed": 0}
    with open(os.path.join(path, "meta.json"), "w") as fh:
        json.dump(meta, fh)
    return meta


def cpu_baseline(args, sg, dc, fanouts, bs):
    """The reference loader (featgrind.sample_batches + dequantize_sq of the
    frontier) on every host core over our own world, bounded to ~cpu_budget
    seconds of work."""
    from oracle import loader as OL
    path = world_dir("fgb_cpu_")
    try:
        export_device_world(sg, dc, path)
        probe = OL.run_pool(path, fanouts, bs, steps=1, warm=0, workers=1)
        per = probe["wall_s"]
        steps = max(1, int(args.cpu_budget / max(per, 1e-3)))
        r = OL.run_pool(path, fanouts, bs, steps=steps, warm=1)
    finally:
        shutil.rmtree(path, ignore_errors=True)
    info = OL.host_info()
    return {"value": round(r["seeds_per_s"], 2), "unit": "seeds/s", "cores": r["workers"],
            "kind": r["kind"],
            "sample": f"{r['workers']} spawned processes x {r['steps']} batches of {bs} seeds "
                      f"(featgrind.sample_batches {list(fanouts)} + dequantize_sq of the "
                      f"frontier; loader only: the reference has no trainer), "
                      f"{r['wall_s']:.1f} s wall, one thread each, over this run's world",
            "host": info}


# ------------------------------------------------------- reference arm

def run_reference(args, rank, world, local):
    """The reference arm: the reference's CPU loader on every host core over
    the same world, rebuilt on the CPU (oracle/world.py) -- this process never
    imports the product package or loads its library.  Rank 0 only."""
    if rank != 0:
        return
    from oracle import loader as OL
    from oracle import world as W
    codec = CONFIGS[args.config][1]
    _, _, fanouts, bs, _ = CONFIGS[args.config][:5]
    if codec[0] != "sq":
        print(json.dumps({"impl": "reference", "metric": METRIC,
                          "unavailable": "the CPU reference world covers the SQ configs "
                                         "(papers100m, arxiv, products-sq8/gcn); VQ fitting "
                                         "the 1e6-row sample on the CPU takes hours"}),
              flush=True)
        return
    s = shape_of(args.config, args.scale)
    path = world_dir("fgb_ref_")
    try:
        t0 = time.perf_counter()
        meta = W.build_world(path, n=s["n"], avg_deg=s["avg_deg"], classes=s["classes"],
                             d=s["d"], train=s["train"], sq_k=codec[1], seed=0,
                             log=lambda m: print(f"[bench/ref] {m}", file=sys.stderr, flush=True))
        build_s = time.perf_counter() - t0
        r = OL.run_pool(path, fanouts, bs, steps=args.steps, warm=args.warmup,
                        workers=args.ref_workers or None)
    finally:
        shutil.rmtree(path, ignore_errors=True)
    v = r["seeds_per_s"]
    info = OL.host_info()
    sample = (f"{args.steps} steps x {r['workers']} spawned processes x {bs} seeds "
              f"(+{args.warmup} warm-up batches each): featgrind.sample_batches "
              f"{list(fanouts)} + dequantize_sq of each batch's frontier "
              f"({'unmodified featgrind from baseline/_ref' if r['kind'] == 'reference' else 'numpy port in oracle/'}); "
              f"loader only (the reference has no trainer); one thread per process")
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 2), "unit": "seeds/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(r["wall_s"] * 1e3 / args.steps, 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64/f32 (numpy)",
            "data": "synthetic (planted-partition power-law graph, class-conditional features)"
                    " -- the GPU arm's world rebuilt bit-identically on the CPU",
            "config": workload_config(args.config, meta["nnz"], world, args.scale),
            "cpu_baseline": {"value": round(v, 2), "unit": "seeds/s", "cores": r["workers"],
                             "kind": r["kind"], "sample": sample, "host": info},
            "e2e": {"value": round(v, 2), "unit": "seeds/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "world_build_s": round(build_s, 1),
            "work": {"frontier_rows": r["frontier_rows"], "edges_touched": r["edges_touched"]}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- launcher

def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_distributed(n):
    """Re-run this command under torch.distributed.run with n ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def init_dist(backend):
    """torchrun environment -> (rank, world, local rank); the process group
    is created only for world > 1."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", rank=rank, world_size=world,
                                    device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo", rank=rank, world_size=world)
    return rank, world, local


def rank_device(local):
    """GPU of a local rank.  With FG_DIST_BACKEND=gloo (tests: several ranks
    sharing the sandbox's one GPU) local ranks wrap around the visible
    devices; NCCL needs one GPU per rank."""
    import torch
    if os.environ.get("FG_DIST_BACKEND", "nccl") == "gloo":
        return local % max(1, torch.cuda.device_count())
    return local


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default=DEFAULT_CONFIG)
    ap.add_argument("--scale", type=float, default=1.0, help="node-count scale (tests only)")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-workers", type=int, default=0, help="reference-arm processes "
                    "(default: every host core)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-epoch", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args.gpus))
    if args.impl == "reference":
        # rank 0 alone runs the CPU arm; no process group is needed
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        run_reference(args, rank, world, int(os.environ.get("LOCAL_RANK", "0")))
        return
    rank, world, local = init_dist(os.environ.get("FG_DIST_BACKEND", "nccl"))
    try:
        run_ours(args, rank, world, rank_device(local))
    finally:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
