"""The reference's CPU mini-batch loader, timed on the host cores — TEST / BASELINE
INFRASTRUCTURE ONLY (bench.py --impl reference and the cpu_baseline leg).

One step of the reference path for one batch of seeds is exactly what the
reference package does on its hot path (SURVEY.md §8(d) "CPU baseline"):

    plan = featgrind.sample_batches(g, seeds, SamplerConfig(fanouts, bs, seed))
                                                       # pipeline.py:185-222
    x    = featgrind.dequantize_sq(codec, plan.batches[0].frontier)
                                                       # sq.py:132-153

run on the unmodified ``featgrind`` installed in ``baseline/_ref`` (or, when
that install is absent, the numpy restatement in oracle/sampler.py +
oracle/codecs.py, reported as kind "port").  The reference has no trainer, so
this is loader-only.  numpy is single-threaded here, so the best case on a
multi-core host is one process per core over disjoint batches (SURVEY.md
§8(d) (ii)): workers are SPAWNED (never forked from a CUDA/torch parent) and
map the world files written by oracle/world.py read-only.

The graph is handed to ``sample_batches`` as a ``CsrGraph`` built without
re-running its constructor validation (graphstore.py:94-127 lexsorts every
stored entry: minutes at papers100M scale); the world is valid by
construction (tests/test_world.py checks the constructor accepts it).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PATH = os.path.join(REPO, "baseline", "_ref")


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_PATH, "featgrind"))


def _import_featgrind():
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    import featgrind
    return featgrind


def host_info() -> dict:
    """CPU model, core count, numpy / BLAS versions of this host."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        cfg = np.show_config(mode="dicts")
        b = cfg.get("Build Dependencies", {}).get("blas", {})
        blas = f"{b.get('name')} {b.get('version')}"
    except Exception:  # noqa: BLE001 - informational only
        pass
    return {"cpu": model, "nproc": os.cpu_count(), "numpy": np.__version__, "blas": blas,
            "python": sys.version.split()[0]}


class Loader:
    """One worker's view of a world directory: the reference (or port)
    sampler + decoder over the mapped files."""

    def __init__(self, path: str, fanouts, batch: int, use_reference: bool = True):
        from . import world as W
        w = W.open_world(path)
        self.meta = w["meta"]
        self.fanouts = tuple(int(f) for f in fanouts)
        self.batch = batch
        self.use_ref = use_reference and reference_available()
        n = self.meta["n"]
        if self.use_ref:
            fgr = _import_featgrind()
            self.fgr = fgr
            g = object.__new__(fgr.CsrGraph)
            object.__setattr__(g, "n", n)
            object.__setattr__(g, "row_offsets", w["off"])
            object.__setattr__(g, "col_indices", w["col"])
            object.__setattr__(g, "has_self_loops", True)
            self.g = g
            p = fgr.SqParams(self.meta["k"], self.meta["e_min"], self.meta["e_max"])
            self.codec = fgr.SqCodec(p, n, self.meta["d"], w["payload"])
        else:
            self.off, self.col, self.payload = w["off"], w["col"], w["payload"]
        self.train = w["train"]

    def step(self, seeds: np.ndarray, seed: int) -> tuple[int, int]:
        """One batch: sample its blocks, decode its frontier.  Returns
        (frontier rows, edges touched)."""
        if self.use_ref:
            fgr = self.fgr
            plan = fgr.sample_batches(self.g, seeds,
                                      fgr.SamplerConfig(self.fanouts, self.batch, seed))
            b = plan.batches[0]
            x = fgr.dequantize_sq(self.codec, b.frontier)
            return int(x.values.shape[0]), int(b.edges_touched)
        from . import codecs as oc
        from .sampler import sample_batches_oracle
        ref, _ = sample_batches_oracle(self.off, self.col, seeds, self.fanouts, self.batch,
                                       seed, max_batches=1)
        m = self.meta
        x = oc.sq_dequant_rows(self.payload, m["n"], m["d"], m["k"], m["e_min"], m["e_max"],
                               ref[0].frontier)
        return int(x.shape[0]), int(sum(L.picks.size for L in ref[0].layers))


def _worker(path, fanouts, batch, use_ref, batches, warm, barrier, q):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    try:
        ld = Loader(path, fanouts, batch, use_ref)
        for b in batches[:warm]:
            ld.step(b, 0)
        barrier.wait()
        t0 = time.perf_counter()
        rows = edges = 0
        for b in batches[warm:]:
            r, e = ld.step(b, 0)
            rows += r
            edges += e
        q.put(("ok", time.perf_counter() - t0, rows, edges, ld.use_ref))
    except Exception as e:  # noqa: BLE001 - reported to the parent
        try:
            barrier.abort()
        except Exception:  # noqa: BLE001
            pass
        q.put(("err", repr(e), 0, 0, False))


def run_pool(path: str, fanouts, batch: int, steps: int, warm: int = 1, workers=None,
             use_reference: bool = True, timeout: float = 1800.0, seed: int = 0) -> dict:
    """``workers`` spawned processes (default: every host core), each running
    ``warm`` untimed then ``steps`` timed batches of ``batch`` seeds, disjoint
    across workers (consecutive slices of one permutation of the train ids).
    Returns throughput and what was run."""
    import multiprocessing as mp
    from . import world as W
    workers = workers or os.cpu_count() or 1
    train = W.open_world(path)["train"]
    perm = np.random.default_rng(seed).permutation(train)
    need = workers * (steps + warm) * batch
    reps = -(-need // perm.size)
    perm = np.tile(perm, reps)[:need]
    per = [[np.sort(perm[(w * (steps + warm) + i) * batch:(w * (steps + warm) + i + 1) * batch])
            for i in range(steps + warm)] for w in range(workers)]
    ctx = mp.get_context("spawn")
    barrier, q = ctx.Barrier(workers + 1), ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(path, tuple(fanouts), batch, use_reference,
                                               per[w], warm, barrier, q), daemon=True)
             for w in range(workers)]
    for p in procs:
        p.start()
    try:
        barrier.wait(timeout=timeout)
        t0 = time.perf_counter()
        res = [q.get(timeout=timeout) for _ in range(workers)]
        wall = time.perf_counter() - t0
    except Exception as e:  # noqa: BLE001
        errs = []
        while not q.empty():
            errs.append(q.get_nowait())
        for p in procs:
            p.kill()
        raise RuntimeError(f"loader pool failed: {e!r} {errs}") from None
    for p in procs:
        p.join(60)
    bad = [r for r in res if r[0] != "ok"]
    if bad:
        raise RuntimeError(f"loader worker failed: {bad[0][1]}")
    wall = max(wall, max(r[1] for r in res))
    seeds = workers * steps * batch
    return {"seeds_per_s": seeds / wall, "wall_s": wall, "workers": workers, "steps": steps,
            "batch": batch, "seeds": seeds, "frontier_rows": sum(r[2] for r in res),
            "edges_touched": sum(r[3] for r in res),
            "kind": "reference" if all(r[4] for r in res) else "port"}


def save_world_meta(path: str, meta: dict) -> None:
    with open(os.path.join(path, "meta.json"), "w") as fh:
        json.dump(meta, fh)
