"""Measured epoch breakdown — the reference's loading simulator re-expressed
with B200 stage times.

The reference prices an epoch with a cost model (pipeline.py:224-394:
``SimReport``, ``simulate_epoch``, ``compare_reports``, ``render_text``):
sample + PCIe load + dequantize + compute, never executed on a device.  Here
the same report is filled with MEASURED device times of the trainer's own
kernels on a batch sample of the epoch:

  sample_s   device sampler chain (CUDA graph of one batch's sampling)
  load_s     host->device copy of the batch's seed ids (features and graph
             are HBM-resident: the PCIe feature stage of the reference does
             not exist; bytes_transferred counts the seed ids)
  dequant_s  fused gather-dequantize-aggregate kernel
  compute_s  the rest of the training step (SAGE layers fwd/bwd, loss, Adam)

each scaled from the measured batches to the epoch's batch count.
``epoch_s`` is the stage sum, as the reference validates; the pipelined
trainer overlaps sampling with compute, so ``overlapped_epoch_s`` in the
workload block records the measured pipelined step time x batches too.
Cache fields: every row is resident (hit rate 1.0, budget = resident codec
bytes).
"""

from __future__ import annotations

import statistics
from dataclasses import dataclass, field, replace

import torch

from .errors import DataError


@dataclass(frozen=True)
class SimReport:
    """pipeline.py:224-275 (same fields, validation and dict form)."""

    label: str
    sample_s: float
    load_s: float
    dequant_s: float
    compute_s: float
    epoch_s: float
    bytes_transferred: float
    cache_hit_rate: float
    cache_budget_bytes: int
    bytes_per_row: float
    workload: dict = field(repr=False)
    speedup_vs_baseline: float | None = None

    def __post_init__(self) -> None:
        total = self.sample_s + self.load_s + self.dequant_s + self.compute_s
        if abs(total - self.epoch_s) > 1e-9 * max(total, 1.0):
            raise DataError("epoch_s must equal the stage sum")

    def to_dict(self) -> dict:
        return {"label": self.label, "sample_s": self.sample_s, "load_s": self.load_s,
                "dequant_s": self.dequant_s, "compute_s": self.compute_s,
                "epoch_s": self.epoch_s, "bytes_transferred": self.bytes_transferred,
                "cache_hit_rate": self.cache_hit_rate,
                "cache_budget_bytes": self.cache_budget_bytes,
                "bytes_per_row": self.bytes_per_row, "workload": dict(self.workload),
                "speedup_vs_baseline": self.speedup_vs_baseline}

    @classmethod
    def from_dict(cls, d: dict) -> "SimReport":
        try:
            return cls(str(d["label"]), float(d["sample_s"]), float(d["load_s"]),
                       float(d["dequant_s"]), float(d["compute_s"]), float(d["epoch_s"]),
                       float(d["bytes_transferred"]), float(d["cache_hit_rate"]),
                       int(d["cache_budget_bytes"]), float(d["bytes_per_row"]),
                       dict(d["workload"]), d.get("speedup_vs_baseline"))
        except KeyError as e:
            raise DataError(f"simulator report missing key {e.args[0]!r}") from e


def compare_reports(baseline: SimReport, variants: list[SimReport]) -> list[SimReport]:
    """pipeline.py:340-350: speedups vs the baseline; workloads must match
    (the measured-timing keys are excluded from the comparison)."""
    def key(r):
        return {k: v for k, v in r.workload.items() if not k.startswith("measured_")
                and k != "overlapped_epoch_s"}
    out = [replace(baseline, speedup_vs_baseline=1.0)]
    for v in variants:
        if key(v) != key(baseline):
            raise DataError(f"workload mismatch between {baseline.label!r} and {v.label!r}; "
                            "reports must come from the same sampling plan")
        out.append(replace(v, speedup_vs_baseline=baseline.epoch_s / v.epoch_s))
    return out


def render_text(reports: list[SimReport]) -> str:
    """pipeline.py:364-383 fixed-width table."""
    cols = ["label", "epoch_s", "sample_s", "load_s", "dequant_s", "compute_s", "load_frac",
            "hit_rate", "GB_moved", "speedup"]
    rows = [[r.label, f"{r.epoch_s:.4g}", f"{r.sample_s:.4g}", f"{r.load_s:.4g}",
             f"{r.dequant_s:.4g}", f"{r.compute_s:.4g}",
             f"{r.load_s / r.epoch_s:.3f}" if r.epoch_s > 0 else "n/a",
             f"{r.cache_hit_rate:.3f}", f"{r.bytes_transferred / 1e9:.4g}",
             f"{r.speedup_vs_baseline:.2f}" if r.speedup_vs_baseline else "-"] for r in reports]
    widths = [max(len(c), *(len(row[i]) for row in rows)) for i, c in enumerate(cols)]
    lines = ["  ".join(c.ljust(w) for c, w in zip(cols, widths)),
             "  ".join("-" * w for w in widths)]
    lines += ["  ".join(c.ljust(w) for c, w in zip(row, widths)) for row in rows]
    return "\n".join(lines)


def _median_us(fn, reps: int) -> float:
    evs = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        evs.append((s, e))
    torch.cuda.synchronize()
    return statistics.median(s.elapsed_time(e) for s, e in evs) * 1e3


def measure_epoch(trainer, train_ids, label: str, batches: int = 20, epoch: int = 0) -> SimReport:
    """Measured stage breakdown of one epoch of ``trainer`` (a SageTrainer
    with pipelined sampling) over ``train_ids``; ``batches`` batches are
    timed and the per-batch medians scaled to the epoch's batch count."""
    from .aggregate import gather_dequant_mean
    nb = trainer.begin_epoch(train_ids, epoch)
    L = len(trainer.cfg.fanouts)
    if trainer.graph is None and not trainer.graphs:
        trainer.capture(3)
    for b in range(3):
        trainer.step(b)
    torch.cuda.synchronize()
    smp = trainer.samplers[-1]
    sb = trainer.samplers[0].batch_view()
    g_sample, g_train, g_gather = (torch.cuda.CUDAGraph() for _ in range(3))
    with torch.cuda.graph(g_sample):
        smp.sample_loaded()
    with torch.cuda.graph(g_train):
        trainer._train(sb)
    with torch.cuda.graph(g_gather):
        gather_dequant_mean(trainer.codec, sb.indptr[L - 1], sb.picks[L - 1], sb.n_nodes[L - 1],
                            trainer.caps[L - 1], out=trainer.agg,
                            edge_w=sb.ew[L - 1] if sb.ew else None)
    torch.cuda.synchronize()
    reps = max(5, batches)
    t_sample = _median_us(g_sample.replay, reps)
    t_train = _median_us(g_train.replay, reps)
    t_gather = _median_us(g_gather.replay, reps)
    seeds = torch.from_numpy(smp.owner.perm_host[:trainer.cfg.batch_size].copy()).pin_memory()
    dst = torch.empty_like(seeds, device=trainer.device)
    t_load = _median_us(lambda: dst.copy_(seeds, non_blocking=True), reps)
    bb = [4 + reps]

    def step():
        trainer.step(bb[0] % nb)
        bb[0] += 1
    t_step = _median_us(step, reps)
    codec = trainer.codec
    row_bytes = (codec.num_parts * codec.bits / 8 if hasattr(codec, "num_parts")
                 else codec.d * codec.params.k / 8)
    resident = int(codec.rows.numel() * codec.rows.element_size())
    sample_s, load_s = t_sample * 1e-6 * nb, t_load * 1e-6 * nb
    dequant_s, compute_s = t_gather * 1e-6 * nb, max(t_train - t_gather, 0.0) * 1e-6 * nb
    workload = {"graph_n": trainer.sampler.g.n, "num_batches": nb,
                "fanouts": list(trainer.cfg.fanouts), "batch_size": trainer.cfg.batch_size,
                "seed": trainer.cfg.seed, "aggregator": trainer.cfg.aggregator,
                "measured_batches": reps, "measured_step_us": round(t_step, 2),
                "overlapped_epoch_s": t_step * 1e-6 * nb}
    return SimReport(label, sample_s, load_s, dequant_s, compute_s,
                     sample_s + load_s + dequant_s + compute_s,
                     float(8 * trainer.cfg.batch_size * nb), 1.0, resident, float(row_bytes),
                     workload)
