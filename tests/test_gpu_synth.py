"""Scalable synthetic workload builders."""

import numpy as np
import pytest
import torch

import paper_2207_14696_b200 as fg
from paper_2207_14696_b200.sq import fit_sq_device, fit_sq_stream
from paper_2207_14696_b200.synth import (generate_graph, synth_feature_rows, synth_features)
from oracle import codecs as oc

pytestmark = pytest.mark.gpu


def test_generated_graph_is_valid_csr_and_chunk_invariant():
    g1, l1 = generate_graph(40_000, 14.0, 7, seed=3)
    g2, l2 = generate_graph(40_000, 14.0, 7, seed=3, chunk_entries=50_000)
    assert torch.equal(g1.row_offsets, g2.row_offsets)
    assert torch.equal(g1.col_indices, g2.col_indices)
    assert torch.equal(l1, l2)
    host = g1.to_host()
    checked = fg.CsrGraph(host.n, host.row_offsets, host.col_indices)  # full validation
    assert checked.has_self_loops
    lab = l1.cpu().numpy()
    assert lab.min() == 0 and lab.max() == 6
    avg = (host.nnz - host.n) / host.n
    assert 10.0 < avg < 14.5
    # homophily: most stored edges stay within a class
    rows = np.repeat(np.arange(host.n), np.diff(host.row_offsets))
    same = (lab[rows] == lab[host.col_indices]).mean()
    assert same > 0.6


def test_feature_rows_match_ranges():
    labels = torch.randint(0, 5, (10_000,), device="cuda", dtype=torch.int32)
    full = synth_features(10_000, 48, kind=3, seed=9, labels=labels, num_classes=5)
    ids = torch.tensor([5, 9999, 0, 5, 1234], device="cuda")
    rows = synth_feature_rows(ids, 48, kind=3, seed=9, labels=labels, num_classes=5)
    assert torch.equal(rows, full[ids])
    part = synth_features(100, 48, row0=700, kind=3, seed=9, labels=labels, num_classes=5)
    assert torch.equal(part, full[700:800])


def test_streaming_fit_sq_equals_whole_matrix_fit():
    r = np.random.default_rng(0)
    x = (np.exp(r.normal(0, 1.3, (90_000, 128))) * r.choice([-1, 1], (90_000, 128)))
    x[r.random(x.shape) < 0.03] = 0
    x = x.astype(np.float32)
    xt = torch.from_numpy(x).cuda()

    def chunks():
        for r0 in range(0, x.shape[0], 7_777):
            yield xt[r0:r0 + 7_777]

    for k in (3, 8):
        a = fit_sq_stream(chunks, k)
        b = fit_sq_device(xt.reshape(-1), k)
        assert (a.e_min, a.e_max) == (b.e_min, b.e_max) == oc.sq_fit(x, k)
