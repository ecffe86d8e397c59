"""Generate golden fixtures by running the REFERENCE itself (featgrind).

Run in the build container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The outputs (*.npz, *.bin) are committed; tests never read /root/reference.
Each fixture records the numpy version that produced it.
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import featgrind as fg  # noqa: E402  (the reference)
from oracle.sampler import sample_batches_oracle  # noqa: E402


def lognormal(seed, n, d, sigma=1.0, zeros=0.0):
    r = np.random.default_rng(seed)
    x = np.exp(r.normal(0.0, sigma, size=(n, d))) * (r.integers(0, 2, size=(n, d)) * 2 - 1)
    if zeros:
        x[r.random((n, d)) < zeros] = 0.0
    return x.astype(np.float32)


def make_sq():
    cases = {}
    mats = {
        "conftest": (lognormal(0xFEA7, 200, 16, 2.0), (1, 2, 3, 4, 5, 8)),
        "odd": (lognormal(11, 61, 7, 1.0, zeros=0.05), (1, 3, 5, 7)),
        "arxivlike": (lognormal(12, 300, 128, 1.0), (4, 8)),
        "products": (lognormal(13, 257, 100, 1.5, zeros=0.01), (8,)),
    }
    specials = np.array([[0.25, -0.5, 0.0, -0.0, 1.0, -1.0, 2.0 ** -9, -2.0 ** -9, 4.0]],
                        np.float32)
    out = {"numpy_version": np.array(np.__version__)}
    rows_r = np.random.default_rng(5)
    for name, (x, ks) in mats.items():
        out[f"{name}/x"] = x
        for k in ks:
            p = fg.fit_sq(fg.FeatureMatrix(x), k)
            c = fg.quantize_sq(fg.FeatureMatrix(x), p)
            rows = rows_r.integers(0, x.shape[0], size=37)
            key = f"{name}/k{k}"
            out[f"{key}/emin_emax"] = np.array([p.e_min, p.e_max])
            out[f"{key}/payload"] = np.frombuffer(c.payload, np.uint8)
            out[f"{key}/decoded"] = fg.dequantize_sq(c).values
            out[f"{key}/rows"] = rows
            out[f"{key}/gathered"] = fg.dequantize_sq(c, rows).values
            with tempfile.TemporaryDirectory() as t:
                fg.save_sq(c, os.path.join(t, "a.sqf"))
                out[f"{key}/sqf1"] = np.fromfile(os.path.join(t, "a.sqf"), np.uint8)
            cases[key] = True
    # frozen reference vector (test_sq.py frozen codes, k=3 over [-4, 0])
    p = fg.SqParams(3, -4.0, 0.0)
    c = fg.quantize_sq(fg.FeatureMatrix(specials), p)
    out["specials/x"] = specials
    out["specials/payload"] = np.frombuffer(c.payload, np.uint8)
    out["specials/decoded"] = fg.dequantize_sq(c).values
    np.savez_compressed(os.path.join(HERE, "sq_golden.npz"), **out)
    print("sq cases", len(cases))


def correlated(seed, n, d, w=0.9):
    r = np.random.default_rng(seed)
    s = r.standard_normal(d)
    return (np.sqrt(w) * s[None, :] + np.sqrt(1 - w) * r.standard_normal((n, d))).astype(np.float32)


def make_vq():
    out = {"numpy_version": np.array(np.__version__)}
    specs = [
        ("cos_w4_L16", correlated(21, 400, 16), dict(width=4, length=16, metric="cosine")),
        ("euc_w4_L16", correlated(22, 400, 16), dict(width=4, length=16, metric="euclidean")),
        ("cos_narrow", correlated(23, 300, 10), dict(width=4, length=8, metric="cosine",
                                                     code_layout="byte_aligned")),
        ("euc_narrow", correlated(24, 300, 10), dict(width=4, length=8, metric="euclidean")),
        ("cos_zeros", None, dict(width=2, length=8, metric="cosine")),
        ("cos_w4_L256", correlated(25, 3000, 100), dict(width=4, length=256, metric="cosine",
                                                        kmeans_max_iters=8, restarts=1)),
        ("euc_w8_L256", correlated(26, 2000, 64), dict(width=8, length=256, metric="euclidean",
                                                       kmeans_max_iters=8, restarts=1)),
        ("lossless", np.eye(6, dtype=np.float32)[np.arange(40) % 6], dict(width=3, length=8,
                                                                          metric="cosine")),
    ]
    for name, x, kw in specs:
        if x is None:
            x = correlated(27, 200, 6)
            x[::7, 0:2] = 0.0
            x[::11, 4:6] = 0.0
        f = fg.FeatureMatrix(x)
        p = fg.VqParams(**kw)
        c = fg.encode_vq(f, fg.fit_vq(f, p))
        # assignment stress set: fresh rows encoded against the fitted books
        probe = (x[np.random.default_rng(3).integers(0, x.shape[0], 500)]
                 + 0.05 * np.random.default_rng(4).standard_normal((500, x.shape[1]))
                 ).astype(np.float32)
        pc = fg.encode_vq(fg.FeatureMatrix(probe), c)
        out[f"{name}/x"] = x
        out[f"{name}/params"] = np.array([p.width, p.length, fg.vq.METRICS.index(p.metric),
                                          fg.vq.CODE_LAYOUTS.index(p.code_layout),
                                          p.kmeans_max_iters, p.restarts])
        out[f"{name}/entries"] = np.array([cb.shape[0] for cb in c.codebooks])
        out[f"{name}/books"] = np.concatenate([cb.reshape(-1) for cb in c.codebooks])
        out[f"{name}/codes"] = c.codes
        out[f"{name}/decoded"] = fg.decode_vq(c).values
        out[f"{name}/probe"] = probe
        out[f"{name}/probe_codes"] = pc.codes
        out[f"{name}/objective"] = np.array([s["objective"] for s in c.fit_stats])
        with tempfile.TemporaryDirectory() as t:
            fg.save_vq(c, os.path.join(t, "a.vqf"))
            out[f"{name}/vqf1"] = np.fromfile(os.path.join(t, "a.vqf"), np.uint8)
    np.savez_compressed(os.path.join(HERE, "vq_golden.npz"), **out)
    print("vq cases", len(specs))


def make_sampler():
    out = {"numpy_version": np.array(np.__version__)}
    graphs = {
        "pa2000": fg.generate_graph("preferential_attachment", 2000, seed=0, m=4, self_loops=True),
        "pa600_noloop": fg.generate_graph("preferential_attachment", 600, seed=1, m=3),
        "star5": fg.generate_graph("star", 5, self_loops=True),
        "complete30": fg.generate_graph("complete", 30, self_loops=True),
        "path10": fg.generate_graph("path", 10, self_loops=True),
        "er500": fg.generate_graph("erdos_renyi", 500, seed=2, p=0.03, self_loops=True),
    }
    configs = [
        ("pa2000", (4, 4), 32, 0, np.arange(200)),
        ("pa2000", (5, 10), 1000, 0, np.arange(1000)),
        ("pa2000", (10, 5), 64, 7, np.arange(0, 2000, 3)),
        ("pa2000", (15, 10, 5), 128, 3, np.arange(300, 700)),
        ("pa600_noloop", (3, 2), 50, 5, np.arange(600)),
        ("star5", (2,), 1, 3, np.array([0])),
        ("complete30", (30,), 1, 0, np.array([0])),
        ("path10", (2, 2), 4, 1, np.arange(10)),
        ("er500", (6, 3), 100, 9, np.arange(500)),
    ]
    for gname, g in graphs.items():
        out[f"graph/{gname}/row_offsets"] = g.row_offsets
        out[f"graph/{gname}/col_indices"] = g.col_indices
    for ci, (gname, fans, bs, seed, train) in enumerate(configs):
        g = graphs[gname]
        cfg = fg.SamplerConfig(fans, bs, seed)
        plan = fg.sample_batches(g, train, cfg)
        mine, _ = sample_batches_oracle(g.row_offsets, g.col_indices, train, fans, bs, seed)
        assert len(mine) == plan.num_batches()
        key = f"cfg{ci}"
        out[f"{key}/meta"] = np.array([ci, bs, seed, len(fans)] + list(fans))
        out[f"{key}/graph"] = np.array(gname)
        out[f"{key}/train"] = train
        for bi, (ref, ob) in enumerate(zip(plan.batches, mine)):
            assert np.array_equal(ref.seeds, ob.seeds)
            assert np.array_equal(ref.frontier, ob.frontier)
            assert ref.edges_touched == ob.edges_touched
            out[f"{key}/b{bi}/seeds"] = ref.seeds
            out[f"{key}/b{bi}/frontier"] = ref.frontier
            out[f"{key}/b{bi}/edges"] = np.array(ref.edges_touched)
            if bi < 3:  # blocks (per-node picks) for the first batches
                for li, L in enumerate(ob.layers):
                    out[f"{key}/b{bi}/l{li}/counts"] = L.counts
                    out[f"{key}/b{bi}/l{li}/picks"] = L.picks.astype(np.int32)
        out[f"{key}/nbatches"] = np.array(plan.num_batches())
    np.savez_compressed(os.path.join(HERE, "sampler_golden.npz"), **out)
    print("sampler configs", len(configs))


def make_formats():
    """FMAT1/CSRG1 byte images from the reference writers."""
    out = {}
    x = lognormal(31, 5, 3)
    g = fg.generate_graph("path", 6, self_loops=True)
    with tempfile.TemporaryDirectory() as t:
        fg.save_features(fg.FeatureMatrix(x), os.path.join(t, "f"))
        fg.save_graph(g, os.path.join(t, "g"))
        out["fmat1"] = np.fromfile(os.path.join(t, "f"), np.uint8)
        out["csrg1"] = np.fromfile(os.path.join(t, "g"), np.uint8)
    out["x"] = x
    out["row_offsets"] = g.row_offsets
    out["col_indices"] = g.col_indices
    np.savez_compressed(os.path.join(HERE, "formats_golden.npz"), **out)


if __name__ == "__main__":
    make_sq()
    make_vq()
    make_sampler()
    make_formats()
