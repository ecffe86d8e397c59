"""GAT (BASELINE config E): edge kernels against a torch reference of the same
math, and accuracy parity of the GPU trainer with the CPU fp32 oracle GAT fed
by the restated reference sampler and decoder."""

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from paper_2207_14696_b200.gat import GatAggregate, GatAttention, GatConfig, GatTrainer
from paper_2207_14696_b200.synth import build_sq_codec, generate_graph, split_ids
from oracle import codecs as oc
from oracle import trainer as ot

pytestmark = pytest.mark.gpu


def _torch_gat(z, el, er, counts, local, heads, slope=0.2):
    nd = counts.numel()
    seg = torch.repeat_interleave(torch.arange(nd, device=z.device), counts)
    cnt = counts.clamp_min(1).float()[:, None]
    q = torch.zeros(nd, heads, device=z.device).index_add_(0, seg, er[local]) / cnt
    s = F.leaky_relu(el[local] + q[seg], slope)
    mx = torch.full((nd, heads), -float("inf"), device=z.device).index_reduce_(0, seg, s, "amax")
    p = torch.exp(s - mx[seg])
    den = torch.zeros(nd, heads, device=z.device).index_add_(0, seg, p)
    alpha = p / den[seg]
    f = z.shape[1] // heads
    msg = (alpha[:, :, None] * z[local].view(-1, heads, f)).reshape(-1, z.shape[1])
    return alpha, torch.zeros(nd, z.shape[1], device=z.device).index_add_(0, seg, msg)


@pytest.mark.parametrize("heads,hf,with_local", [(4, 256, True), (1, 48, True), (2, 32, False)])
def test_gat_edge_kernels_match_torch(heads, hf, with_local):
    rng = np.random.default_rng(heads * hf)
    n_src, n_dst, max_dst, fan = 3000, 700, 760, 9
    counts = rng.integers(1, fan + 1, n_dst)
    counts[rng.random(n_dst) < 0.05] = 0
    E = int(counts.sum())
    indptr = np.zeros(max_dst + 1, np.int32)
    indptr[1:n_dst + 1] = np.cumsum(counts)
    indptr[n_dst + 1:] = E
    local = rng.integers(0, n_src, E).astype(np.int32) if with_local else np.arange(E, dtype=np.int32)
    rows = n_src if with_local else E
    dev = "cuda"
    z = torch.randn(rows, hf, device=dev).to(torch.bfloat16).float().requires_grad_(True)
    el = torch.randn(rows, heads, device=dev).requires_grad_(True)
    er = torch.randn(rows, heads, device=dev).requires_grad_(True)
    ip = torch.from_numpy(indptr).to(dev)
    lc = torch.from_numpy(local).to(dev)
    nd = torch.tensor([n_dst], device=dev)
    alpha = GatAttention.apply(el, er, ip, lc if with_local else None, nd, max_dst, E + 10, 0.2)
    out = GatAggregate.apply(z, alpha, ip, lc if with_local else None, nd, max_dst)
    ct = torch.from_numpy(counts).to(dev)
    z2, el2, er2 = (t.detach().clone().requires_grad_(True) for t in (z, el, er))
    a_ref, o_ref = _torch_gat(z2, el2, er2, ct, lc.long(), heads)
    assert torch.allclose(alpha[:E], a_ref, atol=1e-6, rtol=1e-5)
    assert (alpha[E:] == 0).all()
    assert torch.allclose(out[:n_dst], o_ref, atol=1e-5, rtol=1e-4)
    assert (out[n_dst:] == 0).all()
    g = torch.randn_like(out)
    out.backward(g)
    o_ref.backward(g[:n_dst])
    for got, want in ((z.grad, z2.grad), (el.grad, el2.grad), (er.grad, er2.grad)):
        assert torch.allclose(got, want, atol=1e-4, rtol=1e-3), (got - want).abs().max()


def _small_world(n=12_000, d=32, classes=6, seed=1):
    dg, labels = generate_graph(n, 12.0, classes, seed=seed)
    dc = build_sq_codec(n, d, 8, labels=labels, num_classes=classes, seed=seed)
    train, val = split_ids(n, n // 4, n // 10, seed)
    return dg, labels, dc, train, val


def test_gat_accuracy_parity_with_cpu_oracle():
    """Same init, same reference-sampler batches, same decoded features: GPU
    (bf16 autocast) and CPU fp32 oracle accuracies within 0.5 pt."""
    n, d, C = 12_000, 32, 6
    dg, labels, dc, train, val = _small_world(n=n, d=d, classes=C)
    fans, bs, hidden, lr, epochs = (10, 5), 512, 64, 5e-3, 4
    gpu = GatTrainer(dg, dc, labels, C, GatConfig(fanouts=fans, batch_size=bs, hidden=hidden,
                                                  heads=4, lr=lr))
    cpu_model = ot.OracleGat(d, hidden, C, len(fans), heads=4)
    cpu_model.load_state_dict(gpu.reference_state())
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
        ot.gat_train_epoch(cpu_model, opt, host.row_offsets, host.col_indices, lab, train, fans,
                           bs, e, decode_rows)
    acc_gpu = gpu.evaluate(val, seed=777)
    acc_cpu = ot.gat_evaluate(cpu_model, host.row_offsets, host.col_indices, lab, val, fans, bs,
                              777, decode_rows)
    assert acc_cpu > 0.3
    assert abs(acc_gpu - acc_cpu) <= 0.005 + 1e-12, (acc_gpu, acc_cpu)
    gpu.sampler.check_errors()


def test_gat_graphed_training_learns():
    dg, labels, dc, train, val = _small_world(n=20_000, d=64, classes=8, seed=0)
    t = GatTrainer(dg, dc, labels, 8, GatConfig(fanouts=(15, 10, 5), batch_size=256,
                                                hidden=128, heads=4))
    losses = []
    for e in range(2):
        nb = t.begin_epoch(train, e)
        if t.graph is None:
            t.capture(warmup_batches=2)
        losses += [float(t.step(b).item()) for b in range(nb)]
    assert np.isfinite(losses).all() and np.mean(losses[-5:]) < losses[0]
    assert t.evaluate(val) > 0.3


@pytest.mark.parametrize("codec_kind,decoded", [("sq8", True), ("sq4", True), ("vq", True),
                                                ("sq8", False), ("sq4", False), ("vq", False)])
def test_gat_gradients_match_cpu_oracle_model(codec_kind, decoded):
    """One batch, same weights: the GPU GAT (input layer straight from the
    code rows, bf16 autocast) and the CPU fp32 oracle GAT on the oracle's
    decodes give the same loss and the same gradient for EVERY parameter --
    including layer 0's attention vectors (round 1's head projection dropped
    dA, so they received none) -- for both input forms: decoded bf16 pick
    rows and the code-reading kernels (fg_gat_code_*)."""
    from paper_2207_14696_b200.gat import PickSource
    from paper_2207_14696_b200.synth import build_vq_codec
    from oracle.sampler import sample_batches_oracle
    n, d, C = 6000, 40, 5
    dg, labels = generate_graph(n, 12.0, C, seed=3)
    if codec_kind == "vq":
        dc, _ = build_vq_codec(n, d, 4, 256, labels=labels, num_classes=C, seed=3, max_iters=3,
                               restarts=1)
        codes = dc.rows[:, :dc.num_parts].cpu().numpy().astype(np.int32)

        def decode_rows(rows):
            return oc.vq_decode(codes, dc.books_host, d, 4, rows)
    else:
        k = 8 if codec_kind == "sq8" else 4
        dc = build_sq_codec(n, d, k, labels=labels, num_classes=C, seed=3)
        c = dc.to_codec()

        def decode_rows(rows):
            return oc.sq_dequant_rows(c.payload, n, d, k, c.params.e_min, c.params.e_max, rows)
    train, _ = split_ids(n, n // 4, n // 10, 3)
    fans, bs = (10, 5), 256
    t = GatTrainer(dg, dc, labels, C, GatConfig(fanouts=fans, batch_size=bs, hidden=64, heads=4,
                                                use_graph=False))
    t.begin_epoch(train, 0)
    t.sampler.load_seeds(0)
    sb = t.sampler.sample_loaded()
    L = len(fans)
    # decoded=False: the input layer's kernels read the code rows directly
    src = PickSource(dc, sb.picks[L - 1], sb.n_picks[L - 1], t.pick_cap, decoded=decoded)
    assert (src.x is None) == (not decoded)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        logits = t.model(src, sb, t.caps, t.pick_cap)
    nd = int(sb.n_nodes[0].item())
    y = labels[sb.nodes[0][:nd].long()].long()
    loss = F.cross_entropy(logits[:nd, :C].float(), y)
    t.model.zero_grad()
    loss.backward()
    # the oracle on the same batch (reference sampler restatement)
    host = dg.to_host()
    ref, _ = sample_batches_oracle(host.row_offsets, host.col_indices, train, fans, bs, 0,
                                   max_batches=1)
    cpu_model = ot.OracleGat(d, 64, C, L, heads=4)
    cpu_model.load_state_dict(t.reference_state())
    x, blocks = ot.gat_batch_tensors(ref[0], decode_rows)
    lab = labels.cpu().numpy()
    loss_c = F.cross_entropy(cpu_model(x, blocks), torch.from_numpy(lab[ref[0].seeds]).long())
    loss_c.backward()
    assert abs(float(loss) - float(loss_c)) < 2e-2 * abs(float(loss_c)), (float(loss), float(loss_c))
    gpu_grads = dict(t.model.named_parameters())
    for name, p in cpu_model.named_parameters():
        g_ref = p.grad
        g = gpu_grads[name].grad.float().cpu()
        assert g_ref is not None and g_ref.norm() > 0, name
        rel = ((g - g_ref).norm() / g_ref.norm()).item()
        assert rel < 1e-1, (name, rel)  # bf16 autocast vs fp32
    # the trainer's explicit step (no autograd) on the same batch: same loss,
    # same gradient for every parameter, written into flat_grad; decoded=False
    # runs it with the fused input kernels reading SQ8 code rows in place
    if decoded or codec_kind == "sq8":
        t._direct = not decoded
        t.flat_grad.fill_(float("nan"))   # every element must be written
        t.forward_backward(sb)
        torch.cuda.synchronize()
        assert abs(float(t.loss_buf) - float(loss_c)) < 2e-2 * abs(float(loss_c))
        assert torch.isfinite(t.flat_grad).all()
        for name, p in cpu_model.named_parameters():
            q = gpu_grads[name]
            off = (q.data_ptr() - t.flat_param.data_ptr()) // 4
            g = t.flat_grad[off:off + q.numel()].view(q.shape).cpu()
            rel = ((g - p.grad).norm() / p.grad.norm()).item()
            assert rel < 5e-2, ("explicit", name, rel)


@pytest.mark.parametrize("in_f32", [0, 1])
def test_gat_elu_kernels_match_torch(in_f32):
    """fg_gat_elu_fwd (bias + ELU -> bf16) and fg_gat_elu_bwd (ELU' from the
    output) against torch on the same values."""
    from paper_2207_14696_b200 import _native as N
    dev = "cuda"
    rows, cols = 1000, 264
    o = torch.randn(rows, cols, device=dev) * 3
    o = o if in_f32 else o.to(torch.bfloat16)
    b = torch.randn(cols, device=dev)
    h = torch.empty((rows, cols), dtype=torch.bfloat16, device=dev)
    s = N.stream_handle()
    N.call("fg_gat_elu_fwd", N.ptr(o), in_f32, cols, N.ptr(b), rows, cols, N.ptr(h), s)
    ref = F.elu(o.float() + b).to(torch.bfloat16)
    torch.cuda.synchronize()
    assert (h.float() - ref.float()).abs().max().item() <= 1e-2
    dh = torch.randn(rows, cols, device=dev).to(torch.bfloat16)
    out = torch.empty((rows, cols), dtype=torch.float32 if in_f32 else torch.bfloat16, device=dev)
    N.call("fg_gat_elu_bwd", N.ptr(dh), N.ptr(h), dh.numel(), N.ptr(out), in_f32, s)
    hf = h.float()
    want = torch.where(hf > 0, dh.float(), dh.float() * (hf + 1))
    torch.cuda.synchronize()
    assert (out.float() - want).abs().max().item() <= (0 if in_f32 else 2e-2)


@pytest.mark.parametrize("heads,hf", [(4, 256), (1, 48), (2, 64)])
def test_gat_gather_backward_matches_atomic(heads, hf):
    """fg_gat_agg_bwd_t over the sampler-style transpose with edge ids
    (fg_block_transpose_ex) == the atomic fg_gat_agg_bwd: dz (bf16 vs fp32)
    and dalpha, live and padded rows."""
    from paper_2207_14696_b200 import _native as N
    rng = np.random.default_rng(hf + heads)
    n_src, n_dst, max_dst, fan = 3000, 700, 760, 9
    counts = rng.integers(0, fan + 1, n_dst)
    indptr = np.zeros(max_dst + 1, np.int32)
    indptr[1:n_dst + 1] = np.cumsum(counts)
    indptr[n_dst + 1:] = indptr[n_dst]
    E = int(indptr[n_dst])
    local = rng.integers(0, n_src - 50, E).astype(np.int32)   # the last 50 sources unused
    dev = "cuda"
    cap_e, cap_src = E + 40, n_src + 24                       # padded capacities
    lc = torch.zeros(cap_e, dtype=torch.int32, device=dev)
    lc[:E] = torch.from_numpy(local).to(dev)
    ip = torch.from_numpy(indptr).to(dev)
    ne, nd, ns = (torch.tensor([x], device=dev) for x in (E, n_dst, n_src))
    t_indptr = torch.zeros(n_src + 1, dtype=torch.int32, device=dev)
    t_dst = torch.zeros(cap_e, dtype=torch.int32, device=dev)
    t_w = torch.zeros(cap_e, dtype=torch.float32, device=dev)
    t_eid = torch.zeros(cap_e, dtype=torch.int32, device=dev)
    scratch = torch.zeros(N.lib().fg_block_transpose_scratch_bytes(n_src), dtype=torch.uint8,
                          device=dev)
    s = N.stream_handle()
    N.call("fg_block_transpose_ex", N.ptr(lc), N.ptr(ne), cap_e, N.ptr(ip), N.ptr(nd), max_dst,
           fan, n_src, N.ptr(t_indptr), N.ptr(t_dst), N.ptr(t_w), N.ptr(t_eid), None,
           N.ptr(scratch), scratch.numel(), s)
    z = torch.randn(cap_src, hf, device=dev).to(torch.bfloat16)
    alpha = torch.rand(cap_e, heads, device=dev)
    dout = torch.randn(max_dst, hf, device=dev)
    dz_a = torch.zeros(cap_src, hf, device=dev)
    da_a = torch.zeros(cap_e, heads, device=dev)
    N.call("fg_gat_agg_bwd", N.ptr(z), hf, heads, N.ptr(alpha), N.ptr(ip), N.ptr(lc), max_dst,
           N.ptr(nd), N.ptr(dout), N.ptr(dz_a), N.ptr(da_a), s)
    assert N.lib().fg_gat_agg_bwd_t_supported(hf, heads)
    dz_t = torch.full((cap_src, hf), 9.0, device=dev).to(torch.bfloat16)
    da_t = torch.zeros(cap_e, heads, device=dev)
    N.call("fg_gat_agg_bwd_t", N.ptr(z), hf, heads, N.ptr(alpha), N.ptr(t_indptr), N.ptr(t_dst),
           N.ptr(t_eid), N.ptr(ns), cap_src, N.ptr(dout), N.ptr(dz_t), N.ptr(da_t), s)
    torch.cuda.synchronize()
    assert (dz_t.float() - dz_a.to(torch.bfloat16).float()).abs().max().item() <= \
        2e-2 * dz_a.abs().max().item()
    assert (dz_t[n_src:] == 0).all()
    assert torch.allclose(da_t[:E], da_a[:E], rtol=1e-4, atol=1e-4)
