"""End-to-end GraphSAGE training on compressed features (GPU) and accuracy
parity against the CPU fp32 oracle trainer fed by the restated reference
sampler and decoder (north star: within 0.5 points)."""

import copy

import numpy as np
import pytest
import torch

from paper_2207_14696_b200.sage import SageTrainer, TrainConfig
from paper_2207_14696_b200.synth import build_sq_codec, build_vq_codec, generate_graph, split_ids
from oracle import codecs as oc
from oracle import trainer as ot

pytestmark = pytest.mark.gpu


def _small_world(n=20_000, d=64, classes=8, seed=0, vq=False):
    dg, labels = generate_graph(n, 12.0, classes, seed=seed)
    if vq:
        dc, _ = build_vq_codec(n, d, 4, 64, labels=labels, num_classes=classes, seed=seed,
                               max_iters=10, restarts=1)
    else:
        dc = build_sq_codec(n, d, 8, labels=labels, num_classes=classes, seed=seed)
    train, val = split_ids(n, n // 4, n // 10, seed)
    return dg, labels, dc, train, val


def test_graphed_training_learns():
    dg, labels, dc, train, val = _small_world()
    cfg = TrainConfig(fanouts=(10, 5), batch_size=512, hidden=64, lr=3e-3)
    t = SageTrainer(dg, dc, labels, 8, cfg)
    losses = []
    for e in range(3):
        nb = t.begin_epoch(train, e)
        if t.graph is None:
            t.capture(warmup_batches=2)
        for b in range(nb):
            losses.append(float(t.step(b).item()))
    assert losses[-1] < losses[0]
    acc = t.evaluate(val)
    assert acc > 0.3, acc
    t.sampler.check_errors()


def test_accuracy_parity_with_cpu_oracle_trainer():
    n, d, C = 12_000, 32, 6
    dg, labels, dc, train, val = _small_world(n=n, d=d, classes=C, seed=1)
    fans, bs, hidden, lr, epochs = (10, 5), 512, 64, 5e-3, 4
    cfg = TrainConfig(fanouts=fans, batch_size=bs, hidden=hidden, lr=lr, seed=0)
    gpu = SageTrainer(dg, dc, labels, C, cfg)
    cpu_model = ot.OracleSage(d, hidden, C, len(fans))
    cpu_model.load_state_dict(gpu.model.reference_state())
    opt = torch.optim.Adam(cpu_model.parameters(), lr=lr)
    host = dg.to_host()
    lab = labels.cpu().numpy()
    codec = dc.to_codec()
    p = codec.params

    def decode_rows(rows):
        return oc.sq_dequant_rows(codec.payload, n, d, 8, p.e_min, p.e_max, rows)

    for e in range(epochs):
        nb = gpu.begin_epoch(train, e)
        for b in range(nb):
            gpu.step(b)
        ot.train_epoch(cpu_model, opt, host.row_offsets, host.col_indices, lab, train, fans, bs,
                       e, decode_rows)
    acc_gpu = gpu.evaluate(val, seed=777)
    acc_cpu = ot.evaluate(cpu_model, host.row_offsets, host.col_indices, lab, val, fans, bs,
                          777, decode_rows)
    assert acc_cpu > 0.3
    assert abs(acc_gpu - acc_cpu) <= 0.005 + 1e-12, (acc_gpu, acc_cpu)


def test_vq_three_layer_training_runs():
    dg, labels, dc, train, val = _small_world(vq=True)
    cfg = TrainConfig(fanouts=(15, 10, 5), batch_size=256, hidden=64)
    t = SageTrainer(dg, dc, labels, 8, cfg)
    nb = t.begin_epoch(train, 0)
    t.capture(warmup_batches=2)
    first = float(t.step(0).item())
    for b in range(1, nb):
        t.step(b)
    last = float(t.loss_buf.item())
    assert np.isfinite(last) and last < first
    t.sampler.check_errors()
