"""Mini-batch neighbour sampling on the device (drop-in for the sampler half
of pkg/src/featgrind/pipeline.py: SamplerConfig 34-47, MiniBatchSample /
BatchPlan 165-182, sample_batches 185-222).

Semantics are the reference's, draw for draw:
  ids = unique(train_ids); rng = default_rng(seed); perm = rng.permutation(ids)
  per batch: seeds = sort(perm[lo:lo+bs]); for each fanout f (fanouts[0] at
  the seeds): every node of the current sorted layer picks min(f, deg) stored
  neighbours without replacement via rng.choice on the one serial stream;
  next layer = unique(picks); frontier = unique(seeds ∪ all layers);
  edges_touched = total picks.
The epoch permutation runs on the host (inherently serial; the C ABI's
``fg_rng_permutation_host``), everything per batch runs in sm_100a kernels
with the PCG64 stream state resident in HBM (``fg_sample_layer``), so a batch
needs no host synchronisation and can be captured in a CUDA graph.

Beyond the reference, ``DeviceSampler`` keeps the per-layer blocks (indptr +
picks in choice order + local source indices), which the trainer consumes.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .aggregate import AGGREGATORS
from .errors import DataError
from .graph import CsrGraph, DeviceGraph, sorted_unique_ids

__all__ = ["SamplerConfig", "MiniBatchSample", "BatchPlan", "sample_batches",
           "DeviceSampler", "SampledBatch", "rng_block_from_numpy"]


@dataclass(frozen=True)
class SamplerConfig:
    """Per-layer fanouts (outermost first), batch size, shuffle seed."""

    fanouts: tuple
    batch_size: int
    seed: int = 0

    def __post_init__(self) -> None:
        object.__setattr__(self, "fanouts", tuple(int(f) for f in self.fanouts))
        if any(f < 1 for f in self.fanouts):
            raise DataError("fanouts must be >= 1")
        if self.batch_size < 1:
            raise DataError("batch_size must be >= 1")


@dataclass(frozen=True)
class MiniBatchSample:
    seeds: np.ndarray
    frontier: np.ndarray
    edges_touched: int


@dataclass(frozen=True)
class BatchPlan:
    graph: CsrGraph
    config: SamplerConfig
    batches: tuple

    def num_batches(self) -> int:
        return len(self.batches)


def rng_block_from_numpy(state: dict) -> np.ndarray:
    """FG_RNG_WORDS-word block from ``Generator.bit_generator.state``."""
    blk = np.zeros(N.RNG_WORDS, dtype=np.uint64)
    st, inc = int(state["state"]["state"]), int(state["state"]["inc"])
    m64 = (1 << 64) - 1
    N.call("fg_rng_init", blk.ctypes.data, st >> 64, st & m64, inc >> 64, inc & m64,
           int(state["has_uint32"]), int(state["uinteger"]) & 0xFFFFFFFF)
    return blk


def rng_block_to_numpy(blk: np.ndarray, inc: int) -> dict:
    import ctypes
    hi, lo = ctypes.c_uint64(), ctypes.c_uint64()
    has, buf = ctypes.c_int(), ctypes.c_uint32()
    N.call("fg_rng_read", blk.ctypes.data, ctypes.byref(hi), ctypes.byref(lo),
           ctypes.byref(has), ctypes.byref(buf))
    return {"bit_generator": "PCG64", "state": {"state": (hi.value << 64) | lo.value, "inc": inc},
            "has_uint32": has.value, "uinteger": buf.value}


@dataclass
class SampledBatch:
    """Device-resident sample of one batch (static-capacity buffers).

    layer l (0 = seeds side) expands ``nodes[l]`` (sorted, count
    ``n_nodes[l]``) into ``picks[l]`` with CSR ``indptr[l]``; ``local[l]``
    maps each pick to its row in ``nodes[l+1]``.  Counts are device int64
    scalars so no host sync is needed."""

    nodes: list
    n_nodes: list
    indptr: list
    picks: list
    n_picks: list
    local: list
    frontier: object = None
    n_frontier: object = None
    trans: list = None   # per block (t_indptr, t_dst) or None
    t_eid: list = None   # per block transpose entry -> edge id (need_eid) or None
    ew: list = None      # per block edge weights (aggregator variants) or None


class DeviceSampler:
    """Batch sampler bound to one HBM-resident graph replica."""

    def __init__(self, graph: DeviceGraph, fanouts, batch_size: int, *,
                 need_local: bool = True, want_frontier: bool = False,
                 unique_last: bool = False, need_transpose: bool = False,
                 transpose_layers=None, share: "DeviceSampler | None" = None,
                 need_eid: bool = False,
                 aggregator: str = "mean"):
        """``share``: a second buffer set (slot) for pipelined training that
        continues ``share``'s PCG64 stream, permutation and scratch (only the
        per-batch outputs are its own), so batch b+1 can be sampled into one
        slot while batch b trains from the other.  ``aggregator`` 'gcn' also
        emits per-edge weights for every block (fg_block_edge_weights); the
        transposes then carry them for the backward."""
        import torch
        N.require_cuda()
        self.g = graph
        self.fanouts = tuple(int(f) for f in fanouts)
        self.bs = int(batch_size)
        self.want_frontier = want_frontier
        self.need_local = need_local
        self.unique_last = unique_last or want_frontier
        dev = graph.row_offsets.device
        self.device = dev
        L = len(self.fanouts)
        n = graph.n
        caps = [min(self.bs, n)]
        pcaps = []
        for f in self.fanouts:
            pcaps.append(caps[-1] * f)
            caps.append(min(n, pcaps[-1]))
        self.caps, self.pcaps = caps, pcaps
        i32, i64 = torch.int32, torch.int64
        z = lambda *s, dt=i32: torch.zeros(*s, dtype=dt, device=dev)  # noqa: E731
        self.nodes = [z(c) for c in caps]
        self.n_nodes = [z(1, dt=i64) for _ in caps]
        self.indptr = [z(caps[l] + 1) for l in range(L)]
        self.picks = [z(pcaps[l]) for l in range(L)]
        self.n_picks = [z(1, dt=i64) for _ in range(L)]
        self.local = [z(pcaps[l]) if (need_local and l < L - 1) else None for l in range(L)]
        self.aggregator = aggregator
        self.ew = ([z(pcaps[l], dt=torch.float32) for l in range(L)]
                   if aggregator != "mean" else None)
        # per hidden block: transpose (source rank -> edges) for the gather bwd
        # (``transpose_layers`` limits it to some hidden blocks; default all)
        self.need_transpose = need_transpose and need_local
        self.t_layers = set(range(L - 1) if transpose_layers is None else transpose_layers)
        self.t_indptr, self.t_dst, self.t_w, self.t_eid = [], [], [], []
        if self.need_transpose:
            for l in range(L - 1):
                on = l in self.t_layers
                self.t_indptr.append(z(caps[l + 1] + 1) if on else None)
                self.t_dst.append(z(pcaps[l]) if on else None)
                self.t_w.append(z(pcaps[l], dt=torch.float32) if on else None)
                self.t_eid.append(z(pcaps[l]) if on and need_eid else None)
            if share is None:
                self._alloc_t_scratch()
        self.owner = share or self
        if share is not None:  # shared stream state + scratch
            assert share.fanouts == self.fanouts and share.bs == self.bs and share.g is graph
            self.bitmap, self.wprefix = share.bitmap, share.wprefix
            self.ws_bm, self.ws_layer, self.err = share.ws_bm, share.ws_layer, share.err
            self.rng = share.rng
            if self.need_transpose:
                if not hasattr(share, "t_scratch"):
                    share._alloc_t_scratch()
                self.t_scratch = share.t_scratch
            self.want_frontier = False
            return
        words = N.lib().fg_bitmap_words(n)  # two-level: node bits + non-empty-word bits
        self.bitmap = torch.zeros(words, dtype=torch.int32, device=dev)
        self.wprefix = torch.zeros(words, dtype=torch.int32, device=dev)
        self.ws_bm = torch.zeros(max(N.lib().fg_bitmap_workspace_bytes(n), 256),
                                 dtype=torch.uint8, device=dev)
        self.ws_layer = torch.zeros(max(N.lib().fg_sample_workspace_bytes(max(caps)), 256),
                                    dtype=torch.uint8, device=dev)
        self.err = z(1)
        if want_frontier:
            self.fbitmap = torch.zeros(words, dtype=torch.int32, device=dev)
            self.fcap = min(n, sum(caps))
            self.frontier = z(self.fcap)
            self.n_frontier = z(1, dt=i64)
            self.ws_fbm = torch.zeros_like(self.ws_bm)
        self.rng = torch.zeros(N.RNG_WORDS, dtype=torch.int64, device=dev)
        self._inc = 0
        self.perm = None

    def _alloc_t_scratch(self) -> None:
        import torch
        nbytes = N.lib().fg_block_transpose_scratch_bytes(max(self.caps[1:]))
        self.t_scratch = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)

    # ------------------------------------------------------------- epoch
    def begin_epoch(self, train_ids, seed: int) -> int:
        """unique -> default_rng(seed) -> permutation (pipeline.py:194-200).
        Uploads the permutation and the post-permutation stream state;
        returns the number of batches."""
        import time

        import torch
        t0 = time.perf_counter()
        ids = sorted_unique_ids(train_ids)
        if ids.size == 0:
            raise DataError("train_ids must be non-empty")
        if ids.min() < 0 or ids.max() >= self.g.n:
            raise DataError("train id out of range")
        state = np.random.default_rng(seed).bit_generator.state
        self._inc = int(state["state"]["inc"])
        blk = rng_block_from_numpy(state)
        perm = np.ascontiguousarray(ids)
        t1 = time.perf_counter()
        N.call("fg_rng_permutation_host", blk.ctypes.data, perm.ctypes.data, perm.size)
        t2 = time.perf_counter()
        # each batch's seeds are np.sort(perm[lo:lo + bs]) (pipeline.py:203):
        # sort the slices once here, so a batch's seeds are one copy into the
        # sorted seed layer (no sort kernel in the sampling chain)
        full = perm.size // self.bs
        if full:
            perm[:full * self.bs].reshape(full, self.bs).sort(axis=1)
        perm[full * self.bs:].sort()
        self.perm_host = perm
        t3 = time.perf_counter()
        self.perm = torch.from_numpy(perm.astype(np.int32)).to(self.device)
        self.rng.copy_(torch.from_numpy(blk.view(np.int64)))
        # host-side cost breakdown of the last begin_epoch (bench.py reports it)
        self.begin_epoch_timing = {"unique_s": t1 - t0, "permutation_s": t2 - t1,
                                   "batch_sort_s": t3 - t2,
                                   "upload_s": time.perf_counter() - t3}
        return (perm.size + self.bs - 1) // self.bs

    def set_stream_state(self, state: dict) -> None:
        import torch
        self._inc = int(state["state"]["inc"])
        self.rng.copy_(torch.from_numpy(rng_block_from_numpy(state).view(np.int64)))

    def stream_state(self) -> dict:
        return rng_block_to_numpy(self.rng.cpu().numpy().view(np.uint64), self._inc)

    def load_seeds(self, b: int) -> None:
        """Batch b's seeds (its sorted slice of the permutation) into the seed
        layer, a device copy (the device-resident timed path)."""
        perm = self.owner.perm
        lo = b * self.bs
        cnt = min(self.bs, perm.numel() - lo)
        self.nodes[0][:cnt].copy_(perm[lo:lo + cnt])
        self.n_nodes[0].fill_(cnt)

    def load_seeds_host(self, seeds) -> None:
        """Seeds from a host tensor: the end-to-end input copy.  The seed
        layer holds the batch's ids in ascending order (np.sort of the
        permutation slice, pipeline.py:203): unsorted seeds are sorted on the
        host first.  A sorted pinned int32 tensor copies asynchronously."""
        import torch
        if seeds.numel() > 1 and not bool((seeds[1:] >= seeds[:-1]).all()):
            seeds = torch.sort(seeds.to(torch.int64)).values
        if seeds.dtype != torch.int32:
            seeds = seeds.to(torch.int32)
        cnt = seeds.numel()
        if cnt > self.bs:
            raise DataError("more seeds than the batch size")
        self.nodes[0][:cnt].copy_(seeds, non_blocking=True)
        self.n_nodes[0].fill_(cnt)

    def batch_view(self) -> SampledBatch:
        """The SampledBatch over this slot's static output buffers (what
        ``sample_loaded`` returns, without sampling)."""
        L = len(self.fanouts)
        out = SampledBatch(self.nodes, self.n_nodes, self.indptr, self.picks, self.n_picks,
                           self.local)
        if self.need_transpose:
            out.trans = [(self.t_indptr[l], self.t_dst[l], self.t_w[l], self.n_nodes[l + 1])
                         if l in self.t_layers else None for l in range(L - 1)] + [None]
            out.t_eid = self.t_eid + [None]
        out.ew = self.ew
        return out

    # ------------------------------------------------------------ sample
    def sample_loaded(self) -> SampledBatch:
        """Sample the batch whose seeds load_seeds[_host] put in the seed layer
        (``nodes[0]``; capture-safe)."""
        s = N.stream_handle()
        L = len(self.fanouts)
        n = self.g.n
        bm, wp = N.ptr(self.bitmap), N.ptr(self.wprefix)
        # the seed layer (sorted batch ids) was written by load_seeds[_host]
        if self.want_frontier:
            N.call("fg_bitmap_mark", N.ptr(self.nodes[0]), N.ptr(self.n_nodes[0]), self.caps[0],
                   N.ptr(self.fbitmap), n, s)
        for l, f in enumerate(self.fanouts):
            last = l == L - 1
            expand = (not last) or self.unique_last
            N.call("fg_sample_layer", N.ptr(self.g.row_offsets), N.ptr(self.g.col_indices), n,
                   N.ptr(self.nodes[l]), N.ptr(self.n_nodes[l]), self.caps[l], f,
                   N.ptr(self.rng), N.ptr(self.indptr[l]), N.ptr(self.picks[l]), self.pcaps[l],
                   N.ptr(self.n_picks[l]), bm if expand else None, N.ptr(self.ws_layer),
                   self.ws_layer.numel(), N.ptr(self.err), s)
            if self.ew is not None:
                N.call("fg_block_edge_weights", AGGREGATORS.index(self.aggregator),
                       N.ptr(self.g.row_offsets), N.ptr(self.nodes[l]), N.ptr(self.indptr[l]),
                       N.ptr(self.picks[l]), N.ptr(self.n_nodes[l]), self.caps[l],
                       N.ptr(self.ew[l]), s)
            if self.want_frontier:
                N.call("fg_bitmap_mark", N.ptr(self.picks[l]), N.ptr(self.n_picks[l]),
                       self.pcaps[l], N.ptr(self.fbitmap), n, s)
            if expand:
                N.call("fg_bitmap_compact", bm, n, N.ptr(self.nodes[l + 1]), self.caps[l + 1],
                       N.ptr(self.n_nodes[l + 1]), wp, N.ptr(self.ws_bm), self.ws_bm.numel(), s)
                if self.local[l] is not None:
                    N.call("fg_bitmap_rank", N.ptr(self.picks[l]), N.ptr(self.n_picks[l]),
                           self.pcaps[l], bm, wp, N.ptr(self.local[l]), s)
                    if self.need_transpose and l in self.t_layers:
                        self._transpose(l, s)
                N.call("fg_bitmap_clear", N.ptr(self.nodes[l + 1]), N.ptr(self.n_nodes[l + 1]),
                       self.caps[l + 1], bm, n, s)
        out = self.batch_view()
        if self.want_frontier:
            N.call("fg_bitmap_compact", N.ptr(self.fbitmap), n, N.ptr(self.frontier), self.fcap,
                   N.ptr(self.n_frontier), None, N.ptr(self.ws_fbm), self.ws_fbm.numel(), s)
            N.call("fg_bitmap_clear", N.ptr(self.frontier), N.ptr(self.n_frontier), self.fcap,
                   N.ptr(self.fbitmap), n, s)
            out.frontier, out.n_frontier = self.frontier, self.n_frontier
        return out

    def _transpose_on(self, l: int) -> None:
        """Allocate block l's transpose buffers (for a sampler built without
        them; tests use this to run both backward forms on one batch)."""
        import torch
        if self.t_indptr[l] is None:
            dev = self.device
            self.t_indptr[l] = torch.zeros(self.caps[l + 1] + 1, dtype=torch.int32, device=dev)
            self.t_dst[l] = torch.zeros(self.pcaps[l], dtype=torch.int32, device=dev)
            self.t_w[l] = torch.zeros(self.pcaps[l], dtype=torch.float32, device=dev)
            if not hasattr(self, "t_scratch"):
                nbytes = N.lib().fg_block_transpose_scratch_bytes(max(self.caps[1:]))
                self.t_scratch = torch.zeros(nbytes, dtype=torch.uint8, device=dev)

    def block_trans(self, l: int):
        return (self.t_indptr[l], self.t_dst[l], self.t_w[l], self.n_nodes[l + 1])

    def _transpose(self, l: int, s) -> None:
        """Block l's transpose (source rank -> dst of each incoming edge) for
        the gather-form backward of the hidden block mean."""
        N.call("fg_block_transpose_ex", N.ptr(self.local[l]), N.ptr(self.n_picks[l]),
               self.pcaps[l], N.ptr(self.indptr[l]), N.ptr(self.n_nodes[l]), self.caps[l],
               self.fanouts[l], self.caps[l + 1], N.ptr(self.t_indptr[l]), N.ptr(self.t_dst[l]),
               N.ptr(self.t_w[l]), N.ptr(self.t_eid[l]) if self.t_eid else None,
               N.ptr(self.ew[l]) if self.ew is not None else None, N.ptr(self.t_scratch),
               self.t_scratch.numel(), s)

    def sample(self, b: int) -> SampledBatch:
        self.load_seeds(b)
        return self.sample_loaded()

    def check_errors(self) -> None:
        v = int(self.err.item())
        if v:
            self.err.zero_()
            raise DataError("sampler capacity or fanout limit exceeded" if v == N.FG_EUSAGE
                            else "sampler data error")


def sample_batches(g: CsrGraph, train_ids, cfg: SamplerConfig) -> BatchPlan:
    """pipeline.py:185-222 on the device; identical seeds/frontier/edges."""
    ids = sorted_unique_ids(train_ids)  # checked before any launch
    if ids.size == 0:
        raise DataError("train_ids must be non-empty")
    if ids.min() < 0 or ids.max() >= g.n:
        raise DataError("train id out of range")
    dg = g.to_device()
    smp = DeviceSampler(dg, cfg.fanouts, cfg.batch_size, need_local=False, want_frontier=True)
    nb = smp.begin_epoch(train_ids, cfg.seed)
    out = []
    for b in range(nb):
        sb = smp.sample(b)
        ns = int(sb.n_nodes[0].item())
        nf = int(sb.n_frontier.item())
        edges = int(sum(int(x.item()) for x in sb.n_picks))
        out.append(MiniBatchSample(sb.nodes[0][:ns].long().cpu().numpy(),
                                   sb.frontier[:nf].long().cpu().numpy(), edges))
    smp.check_errors()
    return BatchPlan(g, cfg, tuple(out))
