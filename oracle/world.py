"""The synthetic BASELINE worlds built on the host cores — TEST INFRASTRUCTURE.

ctypes front end of ``oracle/_build/libfgoracle.so`` (fgoracle.c), the C
restatement of the device generators in paper_2207_14696_b200/csrc/fg_data.cu
and synth.py.  It lets the CPU reference arm of ``bench.py`` build exactly the
graph, labels, split and SQ payload the GPU arm trains on without loading the
product library, and lets tests prove the two worlds bit-identical.

What is restated (and where):
  * graph      synth.generate_graph (synth.py:54-103): E = round(n*avg_deg/2)
               counter-based edges, symmetric, self-loops, sorted unique rows;
  * labels     fg_graph_labels (fg_data.cu: k_node_labels);
  * split      synth.split_ids (default_rng(seed + 1).permutation);
  * features   fg_synth_features (kind 3, class-conditional);
  * fit_sq     the reference's fit_sq (sq.py:84-111): nonzero count, the
               linspace-strided 10^7 sample, log2 + np.quantile on the host;
  * payload    quantize_sq (sq.py:114-129) through the reference's bucket
               thresholds (oracle.codecs.sq_codes bisected per bucket) and
               the MSB-first continuous stream of bitpack.py:17-36.

The world lives in plain binary files (``off.bin`` int64, ``col.bin`` int32,
``labels.bin`` int32, ``train.bin`` int64, ``payload.bin`` uint8 + a
``meta.json``) so several spawned worker processes can map it read-only.
"""

from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

from . import codecs as oc

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libfgoracle.so")
LIB_V4 = os.path.join(HERE, "_build", "libfgoracle_v4.so")  # AVX-512 build

_lib = None


def build_lib() -> str:
    """make -C oracle (gcc; no CUDA)."""
    r = subprocess.run(["make", "-s", "-C", HERE], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle C build failed:\n{r.stderr}")
    return LIB


def _has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("flags"):
                    f = set(line.split())
                    return {"avx512f", "avx512dq", "avx512vl", "avx512bw"} <= f
    except OSError:
        pass
    return False


def lib():
    global _lib
    if _lib is None:
        if not (os.path.exists(LIB) and os.path.exists(LIB_V4)):
            build_lib()
        h = C.CDLL(LIB_V4 if _has_avx512() else LIB)
        vp, i64, u64, ci, dbl = C.c_void_p, C.c_int64, C.c_uint64, C.c_int, C.c_double
        sig = {
            "fgo_synth_features": (ci, [ci, u64, i64, vp, i64, i64, vp, i64, vp]),
            "fgo_find_zeros": (i64, [ci, u64, i64, i64, vp, i64, vp, i64]),
            "fgo_values_at": (ci, [ci, u64, i64, vp, i64, vp, i64, vp]),
            "fgo_sq_encode_stream": (i64, [ci, u64, i64, i64, vp, i64, ci, vp, vp]),
            "fgo_graph_open": (vp, [u64, i64, i64, dbl, dbl]),
            "fgo_graph_close": (None, [vp]),
            "fgo_graph_degrees": (i64, [vp, i64, vp]),
            "fgo_graph_build": (i64, [vp, i64, vp, vp, vp]),
            "fgo_graph_labels": (ci, [vp, vp]),
            "fgo_num_threads": (ci, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(h, name)
            fn.restype, fn.argtypes = res, args
        _lib = h
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def num_threads() -> int:
    return int(lib().fgo_num_threads())


# ------------------------------------------------------------------ graph

def num_edges(n: int, avg_deg: float) -> int:
    return int(round(n * avg_deg / 2))      # synth.py:63


class _Gen:
    """Generator handle (the position -> node Feistel table, built once)."""

    def __init__(self, n, classes, seed, alpha=0.8, homophily=0.75):
        self.h = lib().fgo_graph_open(seed, n, classes, alpha, homophily)
        if not self.h:
            raise MemoryError("fgo_graph_open")
        self.n = n

    def __enter__(self):
        return self

    def __exit__(self, *a):
        lib().fgo_graph_close(self.h)


def graph(n: int, avg_deg: float, classes: int, seed: int = 0, alpha: float = 0.8,
          homophily: float = 0.75, with_labels: bool = False, col_alloc=None):
    """(row_offsets int64 [n+1], col_indices int32 [nnz][, labels]) of
    synth.generate_graph (+ fg_graph_labels).  ``col_alloc(raw)`` may supply
    the column buffer (e.g. a memmap) of the raw entry count."""
    E = num_edges(n, avg_deg)
    with _Gen(n, classes, seed, alpha, homophily) as g:
        deg = np.empty(n, np.uint32)
        raw = int(lib().fgo_graph_degrees(g.h, E, _p(deg)))
        off = np.empty(n + 1, np.int64)
        col = col_alloc(raw) if col_alloc else np.empty(raw, np.int32)
        nnz = int(lib().fgo_graph_build(g.h, E, _p(deg), _p(off), _p(col)))
        if nnz < 0:
            raise MemoryError("fgo_graph_build")
        lab = None
        if with_labels:
            lab = np.empty(n, np.int32)
            lib().fgo_graph_labels(g.h, _p(lab))
    return (off, col[:nnz], lab) if with_labels else (off, col[:nnz])


def labels(n: int, classes: int, seed: int = 0) -> np.ndarray:
    out = np.empty(n, np.int32)
    with _Gen(n, classes, seed, 0.5, 0.0) as g:   # fg_graph_labels' generator
        lib().fgo_graph_labels(g.h, _p(out))
    return out


def split_ids(n: int, train: int, val: int, seed: int = 0):
    """synth.split_ids: default_rng(seed + 1).permutation(n)."""
    r = np.random.default_rng(seed + 1)
    perm = r.permutation(n)
    return np.sort(perm[:train]), np.sort(perm[train:train + val])


# --------------------------------------------------------------- features

def _classes(labels) -> int:
    return int(labels.max()) + 1 if labels is not None and labels.size else 1


def features(rows, d: int, *, row0: int = 0, kind: int = 3, seed: int = 0, labels=None):
    """Rows [row0, row0+rows) (int) or the listed row ids (array) of the
    row-addressable matrix of fg_synth_features."""
    ids = None
    if not isinstance(rows, (int, np.integer)):
        ids = np.ascontiguousarray(rows, dtype=np.int64)
        rows = ids.size
    out = np.empty((int(rows), d), np.float32)
    lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.int32)
    rc = lib().fgo_synth_features(kind, seed, row0, _p(ids), int(rows), d, _p(lab),
                                  _classes(lab), _p(out))
    if rc:
        raise ValueError("fgo_synth_features: bad arguments")
    return out


def _quantiles(vals, clip):
    logs = np.log2(np.abs(vals.astype(np.float64)))                           # sq.py:107
    e_min, e_max = np.quantile(logs, [clip, 1.0 - clip])                       # sq.py:108
    return float(e_min), float(e_max)


def _sample_ranks(nnz: int) -> np.ndarray:
    if nnz > oc.FIT_SAMPLE_CAP:
        return np.linspace(0, nnz - 1, oc.FIT_SAMPLE_CAP).astype(np.int64)   # sq.py:105
    return np.arange(nnz, dtype=np.int64)


def find_zeros(n: int, d: int, *, kind: int = 3, seed: int = 0, labels=None) -> np.ndarray:
    """Sorted flat positions of the matrix's zero elements (one generation
    pass; a class-conditional matrix holds ~1 exact zero per 1.6e7 values,
    from 0.6 m + 0.8 z cancelling in float32)."""
    lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.int32)
    cap = 1 << 16
    while True:
        pos = np.empty(cap, np.int64)
        cnt = int(lib().fgo_find_zeros(kind, seed, n, d, _p(lab), _classes(lab), _p(pos), cap))
        if cnt < 0:
            raise ValueError("fgo_find_zeros: bad arguments")
        if cnt <= cap:
            return np.sort(pos[:cnt])
        cap = cnt


def fit_sq(n: int, d: int, k: int, *, kind: int = 3, seed: int = 0, labels=None,
           clip: float = 0.005) -> tuple[float, float]:
    """The reference's fit_sq (sq.py:84-111) over the n x d synthetic matrix,
    which never exists whole: one pass finds the zeros, then only the values
    at the linspace-strided nonzero ranks (sq.py:104-106) are regenerated."""
    lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.int32)
    zpos = find_zeros(n, d, kind=kind, seed=seed, labels=lab)
    nnz = n * d - zpos.size
    if nnz == 0:
        if k == 1:
            return 0.0, 0.0
        raise ValueError("cannot fit an exponent range on an all-zero matrix")
    ranks = _sample_ranks(nnz)
    # nonzero rank r sits at position r + #{zeros z_i with z_i - i <= r}
    pos = ranks + np.searchsorted(zpos - np.arange(zpos.size), ranks, side="right")
    vals = np.empty(pos.size, np.float32)
    lib().fgo_values_at(kind, seed, d, _p(lab), _classes(lab), _p(pos), pos.size, _p(vals))
    return _quantiles(vals, clip)


def sq_thresholds(k: int, e_min: float, e_max: float) -> np.ndarray:
    """t_j = the smallest float32 |x| whose reference code offset
    (sq.py:120-127 via oracle.codecs.sq_codes) reaches j, j = 1 .. 2^(k-1)-1
    (+inf if none): bisection over the float32 bit patterns."""
    half = 1 << (k - 1)
    out = np.full(max(half - 1, 0), np.inf, np.float32)
    for j in range(1, half):
        lo, hi = 0, 0x7F800000  # [+0, +inf)
        while lo < hi:
            mid = (lo + hi) // 2
            v = np.array([mid], np.uint32).view(np.float32)
            off = int(oc.sq_codes(v.reshape(1, 1), k, e_min, e_max)[0, 0]) - half
            if off >= j:
                hi = mid
            else:
                lo = mid + 1
        if lo < 0x7F800000:
            out[j - 1] = np.array([lo], np.uint32).view(np.float32)[0]
    return out


def sq_payload(n: int, d: int, k: int, e_min: float, e_max: float, *, kind: int = 3,
               seed: int = 0, labels=None, out=None, return_zeros: bool = False):
    """quantize_sq(features, SqParams(k, e_min, e_max)).payload as uint8
    (and the number of zero elements met)."""
    total = (n * d * k + 7) // 8
    buf = out if out is not None else np.empty(total, np.uint8)
    assert buf.size == total
    thr = np.ascontiguousarray(sq_thresholds(k, e_min, e_max), dtype=np.float32)
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    zeros = int(lib().fgo_sq_encode_stream(kind, seed, n, d, _p(lab), _classes(lab), k,
                                           _p(thr) if thr.size else None, _p(buf)))
    if zeros < 0:
        raise ValueError("fgo_sq_encode_stream: bad arguments")
    return (buf, zeros) if return_zeros else buf


# ------------------------------------------------------------------ world

def build_world(path: str, *, n: int, avg_deg: float, classes: int, d: int, train: int,
                sq_k: int, seed: int = 0, log=None) -> dict:
    """The SQ BASELINE world of synth.make_shape + build_sq_codec in files
    under ``path``; returns its meta dict (also written to meta.json)."""
    import time
    os.makedirs(path, exist_ok=True)
    say = log or (lambda *_: None)
    t0 = time.perf_counter()
    cpath = os.path.join(path, "col.bin")
    off, col, lab = graph(n, avg_deg, classes, seed, with_labels=True,
                          col_alloc=lambda raw: np.memmap(cpath, np.int32, "w+", shape=(raw,)))
    nnz = int(col.size)
    off.tofile(os.path.join(path, "off.bin"))
    lab.tofile(os.path.join(path, "labels.bin"))
    col._mmap.flush() if hasattr(col, "_mmap") and col._mmap else None
    del off, col
    os.truncate(cpath, nnz * 4)
    t1 = time.perf_counter()
    say(f"graph n={n} nnz={nnz} + labels in {t1 - t0:.1f} s")
    tr = max(1, train)
    va = max(1, min(n - tr, tr // 5))
    train_ids, _ = split_ids(n, tr, va, seed)
    train_ids.astype(np.int64).tofile(os.path.join(path, "train.bin"))
    e_min, e_max = fit_sq(n, d, sq_k, seed=seed, labels=lab)
    t2 = time.perf_counter()
    say(f"fit_sq e_min={e_min:.17g} e_max={e_max:.17g} in {t2 - t1:.1f} s")
    ppath = os.path.join(path, "payload.bin")
    pay = np.memmap(ppath, np.uint8, "w+", shape=((n * d * sq_k + 7) // 8,))
    sq_payload(n, d, sq_k, e_min, e_max, seed=seed, labels=lab, out=pay)
    pay.flush()
    del pay, lab
    t3 = time.perf_counter()
    say(f"sq payload {(n * d * sq_k + 7) // 8 / 1e9:.2f} GB in {t3 - t2:.1f} s")
    meta = {"n": n, "nnz": nnz, "d": d, "classes": classes, "k": sq_k, "e_min": e_min,
            "e_max": e_max, "train": int(train_ids.size), "seed": seed,
            "build_s": round(t3 - t0, 1), "threads": num_threads()}
    with open(os.path.join(path, "meta.json"), "w") as fh:
        json.dump(meta, fh)
    return meta


def open_world(path: str) -> dict:
    """Read-only maps of a world written by ``build_world``."""
    with open(os.path.join(path, "meta.json")) as fh:
        meta = json.load(fh)
    n, nnz = meta["n"], meta["nnz"]
    m = lambda f, dt, shape: np.memmap(os.path.join(path, f), dt, "r", shape=shape)  # noqa: E731
    return dict(meta=meta, off=m("off.bin", np.int64, (n + 1,)),
                col=m("col.bin", np.int32, (nnz,)) if nnz else np.zeros(0, np.int32),
                labels=m("labels.bin", np.int32, (n,)),
                train=np.fromfile(os.path.join(path, "train.bin"), np.int64),
                payload=m("payload.bin", np.uint8, ((n * meta["d"] * meta["k"] + 7) // 8,)))
