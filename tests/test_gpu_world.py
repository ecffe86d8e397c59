"""The device world (synth.py / fg_data.cu) is bit-identical to the CPU world
(oracle/world.py / fgoracle.c) that bench.py's reference arm loads from --
graph, labels, split, features and the SQ payload -- at the
BASELINE shapes the benches run (products-shape and papers100M-shape)."""

import numpy as np
import pytest
import torch

from oracle import world as W
from paper_2207_14696_b200.synth import (SHAPES, build_sq_codec, generate_graph, make_shape,
                                         synth_feature_rows, synth_features)

pytestmark = pytest.mark.gpu


def _same_graph(dg, off, col):
    assert dg.nnz == col.size
    assert torch.equal(dg.row_offsets.cpu(), torch.from_numpy(off))
    # compare the columns in 1 G-entry chunks (papers100M: 3.2e9 entries)
    step = 1 << 30
    for i in range(0, col.size, step):
        assert torch.equal(dg.col_indices[i:i + step].cpu(), torch.from_numpy(col[i:i + step])), i


@pytest.mark.parametrize("n,avg,classes,seed", [(50_000, 9.0, 5, 1), (300_001, 31.0, 13, 7)])
def test_graph_labels_features_bit_identical(n, avg, classes, seed):
    dg, lab = generate_graph(n, avg, classes, seed=seed)
    off, col, lab_h = W.graph(n, avg, classes, seed=seed, with_labels=True)
    _same_graph(dg, off, col)
    assert np.array_equal(lab.cpu().numpy(), lab_h)
    for kind in (0, 1, 2, 3):
        x = synth_features(777, 48, row0=n - 777, kind=kind, seed=seed,
                           labels=lab if kind == 3 else None, num_classes=classes)
        h = W.features(777, 48, row0=n - 777, kind=kind, seed=seed,
                       labels=lab_h if kind == 3 else None)
        assert np.array_equal(x.cpu().numpy().view(np.uint32), h.view(np.uint32)), kind
    ids = torch.randint(0, n, (5000,), device="cuda")
    x = synth_feature_rows(ids, 100, seed=seed, labels=lab, num_classes=classes)
    h = W.features(ids.cpu().numpy(), 100, seed=seed, labels=lab_h)
    assert np.array_equal(x.cpu().numpy().view(np.uint32), h.view(np.uint32))


@pytest.mark.parametrize("shape,k", [("products", 8), ("papers100m", 4)])
def test_benchmark_world_bit_identical(shape, k):
    """The full BASELINE world of bench.py --config {products-sq8, papers100m}:
    CSR (papers100M: 3.2e9 stored entries), labels, train split and the
    reference-layout SQ payload (7.1 GB at papers100M) equal the CPU world."""
    s = SHAPES[shape]
    sg = make_shape(shape, seed=0)
    off, col, lab = W.graph(s["n"], s["avg_deg"], s["classes"], seed=0, with_labels=True)
    _same_graph(sg.graph, off, col)
    del off, col
    assert np.array_equal(sg.labels.cpu().numpy(), lab)
    tr, _ = W.split_ids(s["n"], s["train"], max(1, min(s["n"] - s["train"], s["train"] // 5)))
    assert np.array_equal(sg.train_ids, tr)
    dc = build_sq_codec(s["n"], s["d"], k, labels=sg.labels, num_classes=sg.num_classes, seed=0)
    e = W.fit_sq(s["n"], s["d"], k, seed=0, labels=lab)
    assert (dc.params.e_min, dc.params.e_max) == e
    pay = W.sq_payload(s["n"], s["d"], k, *e, seed=0, labels=lab)
    got = dc.to_codec().payload
    assert len(got) == pay.size
    assert np.array_equal(np.frombuffer(got, np.uint8), pay)
