"""The CPU-built synthetic world (oracle/world.py + fgoracle.c) and the
reference loader pool behind bench.py's reference arm -- CPU tests.

* the graph passes the reference's own CsrGraph validation
  (graphstore.py:94-127: sorted, duplicate-free, symmetric, self-loops);
* fit_sq / the SQ payload equal the reference's fit_sq / quantize_sq
  (sq.py:84-129, imported from baseline/_ref or /root/reference) on the
  generated features, including the >1e7-nonzero strided-sample path;
* the loader pool runs the unmodified reference sampler + decoder;
* bench.py's reference arm prints one line, also relaunched with --gpus 2.
The device side of the bit-identity is tests/test_gpu_world.py.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from oracle import loader as OL  # noqa: E402
from oracle import world as W  # noqa: E402


def _featgrind():
    for p in (os.path.join(REPO, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "featgrind")):
            if p not in sys.path:
                sys.path.insert(0, p)
            import featgrind
            return featgrind
    pytest.skip("reference package not available (baseline/_ref or /root/reference)")


def test_graph_is_a_valid_reference_csr():
    fgr = _featgrind()
    off, col, lab = W.graph(30_000, 12.0, 9, seed=5, with_labels=True)
    g = fgr.CsrGraph(30_000, off, col)          # the reference's full validation
    assert g.has_self_loops
    assert np.bincount(lab).min() >= 30_000 // 9
    assert np.array_equal(lab, W.labels(30_000, 9, seed=5))


@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_sq_world_matches_reference_fit_and_quantize(k):
    fgr = _featgrind()
    n, d = 6000, 24
    lab = W.labels(n, 7, seed=2)
    x = W.features(n, d, seed=2, labels=lab)
    fm = fgr.FeatureMatrix(x)
    p = fgr.fit_sq(fm, k)
    assert W.fit_sq(n, d, k, seed=2, labels=lab) == (p.e_min, p.e_max)
    pay, zeros = W.sq_payload(n, d, k, p.e_min, p.e_max, seed=2, labels=lab, return_zeros=True)
    assert zeros == int((x == 0).sum())
    assert bytes(pay) == fgr.quantize_sq(fm, p).payload


def test_sq_world_strided_fit_sample():
    """> 1e7 nonzeros: the reference's linspace-strided sample (sq.py:104-106)."""
    fgr = _featgrind()
    n, d = 90_000, 128
    lab = W.labels(n, 11, seed=0)
    x = W.features(n, d, seed=0, labels=lab)
    p = fgr.fit_sq(fgr.FeatureMatrix(x), 4)
    assert W.fit_sq(n, d, 4, seed=0, labels=lab) == (p.e_min, p.e_max)


def test_sq_world_fit_with_exact_zeros():
    """The class-conditional matrix holds rare exact zeros (0.6 m + 0.8 z
    cancelling in float32): the fit's nonzero-rank -> position mapping must
    skip them exactly like the reference's flat[flat != 0] (sq.py:99)."""
    from oracle import codecs as oc
    n, d = 300_000, 100
    lab = W.labels(n, 47, seed=0)
    x = W.features(n, d, seed=0, labels=lab)
    zeros = np.flatnonzero(x.reshape(-1) == 0)
    assert zeros.size >= 1                       # this seed/shape has one
    assert np.array_equal(W.find_zeros(n, d, seed=0, labels=lab), zeros)
    assert W.fit_sq(n, d, 8, seed=0, labels=lab) == oc.sq_fit(x, 8)


def test_feature_rows_are_row_addressable():
    lab = W.labels(5000, 4, seed=1)
    full = W.features(5000, 33, seed=1, labels=lab)
    ids = np.array([4999, 0, 17, 17, 2500])
    assert np.array_equal(W.features(ids, 33, seed=1, labels=lab), full[ids])
    for kind in (0, 1, 2):
        a = W.features(40, 9, row0=100, kind=kind, seed=3)
        b = W.features(np.arange(100, 140), 9, kind=kind, seed=3)
        assert np.array_equal(a, b) and np.isfinite(a).all()


def test_loader_pool_runs_the_reference(tmp_path):
    _featgrind()
    meta = W.build_world(str(tmp_path), n=20_000, avg_deg=10.0, classes=5, d=16, train=4000,
                         sq_k=4, seed=0)
    assert meta["nnz"] > 20_000
    r = OL.run_pool(str(tmp_path), (5, 3), 64, steps=2, warm=1, workers=2, timeout=300)
    # "reference" when baseline/_ref holds the pip-installed featgrind (the
    # reference arm's install), else the numpy port
    assert r["kind"] == ("reference" if OL.reference_available() else "port")
    assert r["seeds"] == 2 * 2 * 64 and r["seeds_per_s"] > 0
    # the numpy port does the same work on the same batches
    p = OL.run_pool(str(tmp_path), (5, 3), 64, steps=2, warm=1, workers=2, timeout=300,
                    use_reference=False)
    assert p["kind"] == "port"
    assert (p["frontier_rows"], p["edges_touched"]) == (r["frontier_rows"], r["edges_touched"])


def test_bench_shapes_match_synth():
    import bench
    from paper_2207_14696_b200.synth import SHAPES
    assert bench.SHAPES == SHAPES


@pytest.mark.parametrize("gpus", [1, 2])
def test_bench_reference_arm_line(gpus):
    """The reference arm end to end on CPU; --gpus 2 relaunches under
    torch.distributed.run, rank 0 alone prints."""
    _featgrind()
    cmd = [sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--config",
           "arxiv", "--scale", "0.05", "--steps", "2", "--warmup", "3", "--ref-workers", "2",
           "--gpus", str(gpus)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=REPO)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == gpus and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference"
    assert d["config"]["per_rank_batch"] == 1024 and d["config"]["nodes"] == 8467
    assert d["e2e"]["h2d_bytes_per_step"] == 0
