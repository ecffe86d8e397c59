"""Fused gather-dequantize-mean (the north-star hot path) and the hidden block
mean against the float64 oracle: |gpu - ref| <= tol * mean|x| + 1e-30 with
tol 1e-5 (fp32 out) / 1e-2 (bf16 out), SURVEY.md §8c."""

import numpy as np
import pytest
import torch

import paper_2207_14696_b200 as fg
from paper_2207_14696_b200 import _native as N
from paper_2207_14696_b200.aggregate import block_mean, gather_dequant_mean
from oracle import codecs as oc
from oracle.aggregate import block_mean as oracle_mean
from oracle.aggregate import mean_tolerance_ok

pytestmark = pytest.mark.gpu


def _block(n_src, n_dst, max_dst, fan, rng, zero_frac=0.1):
    counts = rng.integers(1, fan + 1, n_dst)
    counts[rng.random(n_dst) < zero_frac] = 0
    indptr = np.zeros(max_dst + 1, np.int32)
    indptr[1:n_dst + 1] = np.cumsum(counts)
    indptr[n_dst + 1:] = indptr[n_dst]
    src = rng.integers(0, n_src, int(counts.sum())).astype(np.int32)
    return counts, indptr, src


def _run(dc, counts, indptr, src, n_dst, max_dst, dtype, pitch=None):
    dev = "cuda"
    pitch = pitch or dc.d
    out = torch.full((max_dst, pitch), 7.0, dtype=dtype, device=dev)  # sentinel
    gather_dequant_mean(dc, torch.from_numpy(indptr).to(dev), torch.from_numpy(src).to(dev),
                        torch.tensor([n_dst], device=dev), max_dst, out=out)
    o = out.float().cpu().numpy()
    # rows past the live count and columns past d are never written
    assert (o[n_dst:] == 7.0).all() and (o[:, dc.d:] == 7.0).all()
    return o[:, :dc.d]


# fan 7: tiles staged in shared memory by TMA row copies; fan 40 and d 768:
# tiles overflowing the row buffer take the direct-load fallback
@pytest.mark.parametrize("k,d,fan", [(8, 128, 7), (4, 128, 7), (8, 100, 7), (3, 100, 7),
                                     (1, 64, 7), (2, 37, 7), (5, 16, 7), (6, 24, 7), (7, 40, 7),
                                     (4, 128, 40), (8, 128, 12), (4, 768, 7), (8, 1000, 3)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_fused_sq_mean(k, d, fan, dtype):
    rng = np.random.default_rng(k * 100 + d)
    n = 5000
    x = (np.exp(rng.normal(0, 1, (n, d))) * rng.choice([-1, 1], (n, d))).astype(np.float32)
    f = fg.FeatureMatrix(x)
    c = fg.quantize_sq(f, fg.fit_sq(f, k))
    dc = fg.DeviceSqCodec.from_codec(c)
    n_dst, max_dst = 3000, 3200
    counts, indptr, src = _block(n, n_dst, max_dst, fan, rng)
    pitch = (d + 15) // 16 * 16 + (16 if d % 2 else 0)
    got = _run(dc, counts, indptr, src, n_dst, max_dst, dtype, pitch)
    dec = oc.sq_dequant_rows(c.payload, n, d, k, c.params.e_min, c.params.e_max, src)
    ref = oracle_mean(dec, counts)
    tol = 1e-5 if dtype == torch.float32 else 1e-2
    ok, worst = mean_tolerance_ok(got[:n_dst], ref, dec, counts, tol)
    assert ok, worst
    assert (got[:n_dst][counts == 0] == 0).all()
    got2 = _run(dc, counts, indptr, src, n_dst, max_dst, dtype)   # unpadded pitch
    assert np.array_equal(got2[:n_dst], got[:n_dst])


def _vq_codec(n, d, w, L, rng, metric="cosine"):
    x = rng.standard_normal((n, d)).astype(np.float32)
    books = tuple(rng.standard_normal((L, min(w, d - lo))).astype(np.float32)
                  for lo in range(0, d, w))
    p = fg.VqParams(w, L, metric=metric)
    c = fg.encode_vq(fg.FeatureMatrix(x), fg.VqCodec(p, d, books))
    return c


@pytest.mark.parametrize("w,L,d", [(4, 256, 100), (8, 256, 100), (8, 256, 128), (16, 2048, 96),
                                   (2, 16, 10), (1, 4, 5), (1, 256, 70), (2, 256, 33),
                                   (16, 256, 40), (8, 256, 768), (4, 300, 30),
                                   (4, 256, 402), (8, 256, 260)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_fused_vq_mean(w, L, d, dtype):
    rng = np.random.default_rng(w * 1000 + L + d)
    n = 4000
    c = _vq_codec(n, d, w, L, rng)
    dc = fg.DeviceVqCodec.from_codec(c)
    n_dst, max_dst = 2500, 2600
    counts, indptr, src = _block(n, n_dst, max_dst, 6, rng)
    got = _run(dc, counts, indptr, src, n_dst, max_dst, dtype, (d + 15) // 16 * 16)
    dec = oc.vq_decode(c.codes, c.codebooks, d, w, src)
    ref = oracle_mean(dec, counts)
    tol = 1e-5 if dtype == torch.float32 else 1e-2
    ok, worst = mean_tolerance_ok(got[:n_dst], ref, dec, counts, tol)
    assert ok, worst
    got2 = _run(dc, counts, indptr, src, n_dst, max_dst, dtype)
    assert np.array_equal(got2[:n_dst], got[:n_dst])


def test_vq_gather_decode_nonbyte_codes():
    rng = np.random.default_rng(5)
    c = _vq_codec(3000, 45, 3, 300, rng, metric="euclidean")   # 9-bit codes
    rows = rng.integers(0, 3000, 777)
    assert np.array_equal(fg.decode_vq(c, rows).values,
                          oc.vq_decode(c.codes, c.codebooks, 45, 3, rows))


def test_hidden_block_mean_fwd_bwd():
    rng = np.random.default_rng(3)
    n_src, n_dst, max_dst, H = 4000, 900, 1000, 256
    counts, indptr, src = _block(n_src, n_dst, max_dst, 10, rng)
    dev = "cuda"
    h = torch.randn(n_src, H, device=dev).to(torch.bfloat16).requires_grad_(True)
    ip = torch.from_numpy(indptr).to(dev)
    sl = torch.from_numpy(src).to(dev)
    out = block_mean(h, ip, sl, torch.tensor([n_dst], device=dev), max_dst)
    # torch fp32 reference of the same op
    hf = h.detach().float().requires_grad_(True)
    seg = torch.repeat_interleave(torch.arange(n_dst, device=dev),
                                  torch.from_numpy(counts).to(dev))
    ref = torch.zeros(max_dst, H, device=dev).index_add_(0, seg, hf[sl.long()])
    cnt = torch.zeros(max_dst, device=dev)
    cnt[:n_dst] = torch.from_numpy(counts).float().to(dev)
    ref = ref / cnt.clamp_min(1)[:, None]
    assert torch.allclose(out.float(), ref, atol=2e-2, rtol=1e-2)
    g = torch.randn(max_dst, H, device=dev)
    g[n_dst:] = 0
    out.backward(g.to(torch.bfloat16))
    ref.backward(g.to(torch.bfloat16).float())
    assert torch.allclose(h.grad.float(), hf.grad, atol=2e-2, rtol=1e-2)


def test_hidden_block_mean_fused_relu():
    rng = np.random.default_rng(4)
    n_src, n_dst, max_dst, H = 3000, 700, 800, 128
    counts, indptr, src = _block(n_src, n_dst, max_dst, 8, rng)
    dev = "cuda"
    h = torch.randn(n_src, H, device=dev).to(torch.bfloat16).requires_grad_(True)
    ip, sl = torch.from_numpy(indptr).to(dev), torch.from_numpy(src).to(dev)
    out = block_mean(h, ip, sl, torch.tensor([n_dst], device=dev), max_dst, relu=True)
    hf = h.detach().float().requires_grad_(True)
    seg = torch.repeat_interleave(torch.arange(n_dst, device=dev), torch.from_numpy(counts).to(dev))
    ref = torch.zeros(max_dst, H, device=dev).index_add_(0, seg, torch.relu(hf)[sl.long()])
    cnt = torch.zeros(max_dst, device=dev)
    cnt[:n_dst] = torch.from_numpy(counts).float().to(dev)
    ref = ref / cnt.clamp_min(1)[:, None]
    assert torch.allclose(out.float(), ref, atol=2e-2, rtol=1e-2)
    g = torch.randn(max_dst, H, device=dev)
    g[n_dst:] = 0
    out.backward(g.to(torch.bfloat16))
    ref.backward(g.to(torch.bfloat16).float())
    assert torch.allclose(h.grad.float(), hf.grad, atol=2e-2, rtol=1e-2)


def _transpose_np(indptr, src, n_dst, n_src):
    e = np.arange(src.size)
    cnt = np.diff(indptr[:n_dst + 1])
    dst = np.repeat(np.arange(n_dst), cnt)
    order = np.lexsort((e, src))
    t_indptr = np.zeros(n_src + 1, np.int32)
    np.add.at(t_indptr, src + 1, 1)
    w = (1.0 / np.maximum(cnt, 1)).astype(np.float32)[dst]
    return np.cumsum(t_indptr).astype(np.int32), dst[order].astype(np.int32), w[order]


@pytest.mark.parametrize("relu", [False, True])
def test_hidden_block_mean_gather_backward(relu):
    rng = np.random.default_rng(5)
    n_src, n_dst, max_dst, H = 2500, 600, 700, 64
    counts, indptr, src = _block(n_src, n_dst, max_dst, 9, rng)
    ti, td, tw = _transpose_np(indptr, src, n_dst, n_src)
    dev = "cuda"
    h = torch.randn(n_src, H, device=dev).to(torch.bfloat16).requires_grad_(True)
    ip, sl = torch.from_numpy(indptr).to(dev), torch.from_numpy(src).to(dev)
    trans = (torch.from_numpy(ti).to(dev), torch.from_numpy(td).to(dev),
             torch.from_numpy(tw).to(dev), torch.tensor([n_src], device=dev))
    out = block_mean(h, ip, sl, torch.tensor([n_dst], device=dev), max_dst, relu=relu, trans=trans)
    hf = h.detach().float().requires_grad_(True)
    seg = torch.repeat_interleave(torch.arange(n_dst, device=dev), torch.from_numpy(counts).to(dev))
    act = torch.relu(hf) if relu else hf
    ref = torch.zeros(max_dst, H, device=dev).index_add_(0, seg, act[sl.long()])
    cnt = torch.zeros(max_dst, device=dev)
    cnt[:n_dst] = torch.from_numpy(counts).float().to(dev)
    ref = ref / cnt.clamp_min(1)[:, None]
    g = torch.randn(max_dst, H, device=dev)
    g[n_dst:] = 0
    out.backward(g.to(torch.bfloat16))
    ref.backward(g.to(torch.bfloat16).float())
    assert torch.allclose(h.grad.float(), hf.grad, atol=2e-2, rtol=1e-2)


@pytest.mark.parametrize("H", [64, 256])
def test_block_mean_bwd_t_relu_bits_matches_h_mask(H):
    """fg_block_mean_bwd_t_bits (packed ReLU bits, the MAG GEMM path's dh0)
    equals fg_block_mean_bwd_t with the bf16 h rows as the mask, bit for bit."""
    from paper_2207_14696_b200 import _native as N
    from paper_2207_14696_b200.aggregate import relu_mask_bits
    rng = np.random.default_rng(H)
    n_src, n_dst, max_dst = 4000, 900, 1000
    counts, indptr, src = _block(n_src, n_dst, max_dst, 9, rng)
    ti, td, tw = _transpose_np(indptr, src, n_dst, n_src)
    dev = "cuda"
    h = torch.randn(n_src, H, device=dev).to(torch.bfloat16)
    g = torch.randn(max_dst, H, device=dev).to(torch.bfloat16)
    bits = relu_mask_bits(h)
    t = [torch.from_numpy(x).to(dev) for x in (ti, td, tw)]
    ns = torch.tensor([n_src - 7], device=dev)   # padded rows past the live sources
    a = torch.full((n_src, H), 7.0, device=dev).to(torch.bfloat16)
    b = torch.full_like(a, -7.0)
    s = N.stream_handle()
    N.call("fg_block_mean_bwd_t", N.ptr(g), H, H, N.ptr(t[0]), N.ptr(t[1]), N.ptr(t[2]),
           N.ptr(ns), n_src, N.ptr(h), N.ptr(a), s)
    N.call("fg_block_mean_bwd_t_bits", N.ptr(g), H, H, N.ptr(t[0]), N.ptr(t[1]), N.ptr(t[2]),
           N.ptr(ns), n_src, N.ptr(bits), N.ptr(b), s)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    assert (a[n_src - 7:] == 0).all()


def test_block_transpose_kernel():
    from paper_2207_14696_b200 import _native as N
    rng = np.random.default_rng(8)
    n_src, n_dst, max_dst = 5000, 1200, 1300
    counts, indptr, src = _block(n_src, n_dst, max_dst, 10, rng)
    dev = "cuda"
    E = src.size
    cap_e = E + 100
    local = torch.zeros(cap_e, dtype=torch.int32, device=dev)
    local[:E] = torch.from_numpy(src).to(dev)
    t_indptr = torch.zeros(n_src + 1, dtype=torch.int32, device=dev)
    t_dst = torch.zeros(cap_e, dtype=torch.int32, device=dev)
    t_w = torch.zeros(cap_e, dtype=torch.float32, device=dev)
    scratch = torch.zeros(N.lib().fg_block_transpose_scratch_bytes(n_src), dtype=torch.uint8,
                          device=dev)
    ne_t, nd_t = torch.tensor([E], device=dev), torch.tensor([n_dst], device=dev)
    ip_t = torch.from_numpy(indptr).to(dev)  # keep every buffer alive until sync
    N.call("fg_block_transpose", N.ptr(local), N.ptr(ne_t), cap_e, N.ptr(ip_t), N.ptr(nd_t),
           max_dst, 10, n_src, N.ptr(t_indptr), N.ptr(t_dst), N.ptr(t_w), None, N.ptr(scratch),
           scratch.numel(), N.stream_handle())
    torch.cuda.synchronize()
    ti, td, tw = _transpose_np(indptr, src, n_dst, n_src)
    assert np.array_equal(t_indptr.cpu().numpy(), ti)
    got = t_dst[:E].cpu().numpy()
    for r in range(0, n_src, 7):  # same multiset of dsts per source
        assert np.array_equal(np.sort(got[ti[r]:ti[r + 1]]), np.sort(td[ti[r]:ti[r + 1]]))


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("pad", [0, 1])
def test_fused_softmax_ce_matches_torch(dtype, pad):
    """pad: logits carry one padded class column (ld 48 for 47 classes) whose
    gradient must come back zero; the loss is reduced by the kernel's last
    CTA (run twice to check the completion counter re-arms)."""
    from paper_2207_14696_b200.aggregate import softmax_ce
    dev = "cuda"
    rows, C, nv = 3000, 47, 2570
    ld = C + pad
    x = (torch.randn(rows, ld, device=dev) * 3).to(dtype).float()  # exact in both dtypes
    labels = torch.randint(0, C, (5000,), device=dev, dtype=torch.int32)
    node = torch.randint(0, 5000, (rows,), device=dev, dtype=torch.int32)
    lf = x[:nv, :C].clone().requires_grad_(True)
    ref = torch.nn.functional.cross_entropy(lf, labels[node[:nv].long()].long())
    ref.backward()
    for _ in range(2):
        logits = x.to(dtype).clone().requires_grad_(True)
        loss = softmax_ce(logits, labels, node, torch.tensor([nv], device=dev), C)
        loss.backward()
        assert abs(float(loss.detach()) - float(ref)) < 1e-4 * max(1.0, abs(float(ref)))
        tol = 1e-6 if dtype == torch.float32 else 1e-2 / nv
        assert torch.allclose(logits.grad[:nv, :C].float(), lf.grad, atol=tol, rtol=1e-2)
        assert (logits.grad[nv:] == 0).all()
        assert (logits.grad[:, C:] == 0).all()


# fan 40 over 290 sources: ~100 edges per source row (hub rows); n_src 100:
# fewer edges than one 128-edge tile per CTA
@pytest.mark.parametrize("H,P,relu,fan,n_src", [(256, 112, True, 10, 2900), (256, 144, True, 5, 2900),
                                                (128, 64, False, 15, 2900), (256, 160, True, 3, 2900),
                                                (128, 48, True, 40, 290), (256, 112, True, 10, 100),
                                                (128, 80, True, 10, 2900), (256, 16, True, 2, 50),
                                                (256, 112, True, -3, 2900)])
def test_block_mean_wgrad_tcgen05(H, P, relu, fan, n_src):
    """Edge-tiled fused tcgen05 dW against torch fp32 on the same bf16
    per-edge terms."""
    from paper_2207_14696_b200.aggregate import block_mean_wgrad, wgrad_supported
    assert wgrad_supported(H, P)
    rng = np.random.default_rng(H + P + abs(fan))
    cap_src, n_dst, max_dst = n_src + 200, 700, 760
    # fan < 0: 97 % of destinations without edges, so one 128-edge tile spans
    # more destinations than the kernel's indptr window (slow-path search)
    zf = 0.97 if fan < 0 else 0.1
    fan = abs(fan)
    if zf > 0.5:
        n_dst, max_dst = 20000, 20100
    counts, indptr, src = _block(n_src, n_dst, max_dst, fan, rng, zero_frac=zf)
    dev = "cuda"
    ip = torch.from_numpy(indptr).to(dev)
    local = torch.full((max_dst * fan,), -7, dtype=torch.int32, device=dev)  # capacity > live
    local[:src.size] = torch.from_numpy(src).to(dev)
    g = torch.randn(max_dst, H + 8, device=dev).to(torch.bfloat16)
    h = torch.randn(cap_src, H, device=dev).to(torch.bfloat16)
    x = torch.randn(cap_src, P, device=dev).to(torch.bfloat16)
    x[n_src:] = float("nan")  # rows past the live count must never be read
    dw = block_mean_wgrad(g, ip, local, torch.tensor([n_dst], device=dev), max_dst,
                          h if relu else None, x, H=H)
    torch.cuda.synchronize()
    # reference: per-edge terms bf16-rounded as in the kernel, fp32 GEMM
    dst = torch.repeat_interleave(torch.arange(n_dst, device=dev),
                                  torch.from_numpy(counts).long().to(dev))
    l = torch.from_numpy(src).long().to(dev)
    w = 1.0 / torch.from_numpy(counts).float().to(dev)[dst]
    term = g[dst, :H].float() * w[:, None]
    if relu:
        term = term * (h[l].float() > 0)
    ref = term.to(torch.bfloat16).float().t() @ x[l].float()
    err = (dw - ref).abs().max().item()
    assert err <= 1e-3 * ref.abs().max().item() + 1e-4, err
    assert torch.isfinite(dw).all()
    if relu:  # packed ReLU bits give the identical result
        from paper_2207_14696_b200.aggregate import relu_mask_bits
        bits = relu_mask_bits(h)
        assert bits.shape == (cap_src, H // 8)
        hb = (h[:5].float() > 0).cpu().numpy()
        want = np.packbits(hb.reshape(5, H // 8, 8), axis=2, bitorder="little")[..., 0]
        assert np.array_equal(bits[:5].cpu().numpy(), want)
        dw2 = block_mean_wgrad(g, ip, local, torch.tensor([n_dst], device=dev), max_dst, bits,
                               x, H=H)
        assert torch.equal(dw, dw2)


def test_block_mean_wgrad_empty_block():
    from paper_2207_14696_b200.aggregate import block_mean_wgrad
    dev = "cuda"
    ip = torch.zeros(11, dtype=torch.int32, device=dev)
    local = torch.zeros(40, dtype=torch.int32, device=dev)
    x = torch.randn(30, 48, device=dev).to(torch.bfloat16)
    g = torch.randn(10, 136, device=dev).to(torch.bfloat16)
    dw = block_mean_wgrad(g, ip, local, torch.tensor([0], device=dev), 10, None, x, H=128)
    assert (dw == 0).all()


def test_input_block_mean_autograd_matches_unfused():
    from paper_2207_14696_b200.aggregate import input_block_mean
    rng = np.random.default_rng(11)
    n_src, n_dst, max_dst, H, P = 2500, 600, 700, 256, 112
    counts, indptr, src = _block(n_src, n_dst, max_dst, 10, rng)
    ti, td, tw = _transpose_np(indptr, src, n_dst, n_src)
    dev = "cuda"
    ip, sl = torch.from_numpy(indptr).to(dev), torch.from_numpy(src).to(dev)
    nd = torch.tensor([n_dst], device=dev)
    trans = (torch.from_numpy(ti).to(dev), torch.from_numpy(td).to(dev),
             torch.from_numpy(tw).to(dev), torch.tensor([n_src], device=dev))
    x = torch.randn(n_src, P, device=dev).to(torch.bfloat16)
    w1 = (torch.randn(H, P, device=dev) * 0.1).requires_grad_(True)
    w2 = w1.detach().clone().requires_grad_(True)
    a1 = input_block_mean(x, w1, ip, sl, nd, max_dst)
    h2 = torch.mm(x, w2.to(torch.bfloat16).t())
    a2 = block_mean(h2, ip, sl, nd, max_dst, relu=True, trans=trans, bias_col=True)
    assert torch.equal(a1, a2)
    gout = torch.randn_like(a1.float()).to(torch.bfloat16)
    a1.backward(gout)
    a2.backward(gout)
    rel = ((w1.grad - w2.grad).norm() / w2.grad.norm()).item()
    assert rel < 1e-2, rel


# ----------------------------------------------------- aggregator variants
def _run_wsum(dc, indptr, src, w, n_dst, max_dst, dtype, pitch):
    dev = "cuda"
    out = torch.full((max_dst, pitch), 7.0, dtype=dtype, device=dev)
    gather_dequant_mean(dc, torch.from_numpy(indptr).to(dev), torch.from_numpy(src).to(dev),
                        torch.tensor([n_dst], device=dev), max_dst, out=out,
                        edge_w=torch.from_numpy(w.astype(np.float32)).to(dev))
    o = out.float().cpu().numpy()
    assert (o[n_dst:] == 7.0).all()
    return o[:, :dc.d]


@pytest.mark.parametrize("codec,fan", [(("sq", 8, 100), 7), (("sq", 4, 128), 7),
                                       (("sq", 8, 128), 40), (("sq", 3, 100), 5),
                                       (("vq", 4, 256, 100), 6), (("vq", 8, 256, 768), 5),
                                       (("vq", 2, 256, 33), 6)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_fused_weighted_sum_matches_oracle(codec, fan, dtype):
    """fg_gather_dequant_wsum (GCN path through the fused kernels) against the
    float64 oracle sum_e w_e x_e with random positive weights."""
    from oracle.aggregate import block_wsum, wsum_tolerance_ok
    rng = np.random.default_rng(fan + codec[1] + codec[-1])
    n = 4000
    if codec[0] == "sq":
        k, d = codec[1], codec[2]
        x = (np.exp(rng.normal(0, 1, (n, d))) * rng.choice([-1, 1], (n, d))).astype(np.float32)
        f = fg.FeatureMatrix(x)
        c = fg.quantize_sq(f, fg.fit_sq(f, k))
        dc = fg.DeviceSqCodec.from_codec(c)
    else:
        w_, L, d = codec[1], codec[2], codec[3]
        c = _vq_codec(n, d, w_, L, rng)
        dc = fg.DeviceVqCodec.from_codec(c)
    n_dst, max_dst = 2500, 2600
    counts, indptr, src = _block(n, n_dst, max_dst, fan, rng)
    wts = rng.uniform(0.05, 2.0, src.size)
    got = _run_wsum(dc, indptr, src, wts, n_dst, max_dst, dtype, (d + 15) // 16 * 16)
    if codec[0] == "sq":
        dec = oc.sq_dequant_rows(c.payload, n, d, codec[1], c.params.e_min, c.params.e_max, src)
    else:
        dec = oc.vq_decode(c.codes, c.codebooks, d, codec[1], src)
    ref = block_wsum(dec, counts, wts.astype(np.float32))
    tol = 1e-5 if dtype == torch.float32 else 1e-2
    ok, worst = wsum_tolerance_ok(got[:n_dst], ref, dec, counts, wts, tol)
    assert ok, worst


def test_block_edge_weights_gcn_and_mean():
    from oracle.aggregate import gcn_weights
    from paper_2207_14696_b200.aggregate import edge_weights
    from paper_2207_14696_b200.synth import generate_graph
    dg, _ = generate_graph(5000, 12.0, 4, seed=3)
    host = dg.to_host()
    rng = np.random.default_rng(1)
    n_dst, max_dst = 700, 800
    dst_nodes = np.sort(rng.choice(5000, n_dst, replace=False)).astype(np.int32)
    counts, indptr, src = _block(5000, n_dst, max_dst, 9, rng)
    dev = "cuda"
    dn = torch.zeros(max_dst, dtype=torch.int32, device=dev)
    dn[:n_dst] = torch.from_numpy(dst_nodes).to(dev)
    args = (dg, dn, torch.from_numpy(indptr).to(dev), torch.from_numpy(src).to(dev),
            torch.tensor([n_dst], device=dev), max_dst)
    w = torch.zeros(src.size, dtype=torch.float32, device=dev)
    edge_weights("gcn", *args, w)
    want = gcn_weights(host.row_offsets, dst_nodes, counts, src)
    np.testing.assert_allclose(w.cpu().numpy(), want, rtol=2e-6)
    edge_weights("mean", *args, w)
    np.testing.assert_allclose(w.cpu().numpy(), 1.0 / np.repeat(counts, counts), rtol=1e-7)


def test_hidden_block_weighted_fwd_bwd_and_wgrad():
    """Edge-weighted hidden block: forward (fg_block_mean_fwd with weights),
    gather backward over a weighted transpose, and the edge-tiled wgrad with
    weights, against torch fp32."""
    from paper_2207_14696_b200.aggregate import block_mean_wgrad
    rng = np.random.default_rng(21)
    n_src, n_dst, max_dst, H, P = 3000, 800, 850, 256, 112
    counts, indptr, src = _block(n_src, n_dst, max_dst, 10, rng)
    wts = rng.uniform(0.1, 1.5, src.size).astype(np.float32)
    dev = "cuda"
    ip, sl = torch.from_numpy(indptr).to(dev), torch.from_numpy(src).to(dev)
    nd = torch.tensor([n_dst], device=dev)
    ew = torch.from_numpy(wts).to(dev)
    # weighted transpose
    cap_e = src.size
    t_indptr = torch.zeros(n_src + 1, dtype=torch.int32, device=dev)
    t_dst = torch.zeros(cap_e, dtype=torch.int32, device=dev)
    t_w = torch.zeros(cap_e, dtype=torch.float32, device=dev)
    scratch = torch.zeros(N.lib().fg_block_transpose_scratch_bytes(n_src), dtype=torch.uint8,
                          device=dev)
    ne_t = torch.tensor([cap_e], device=dev)
    N.call("fg_block_transpose", N.ptr(sl), N.ptr(ne_t), cap_e, N.ptr(ip), N.ptr(nd), max_dst,
           10, n_src, N.ptr(t_indptr), N.ptr(t_dst), N.ptr(t_w), N.ptr(ew), N.ptr(scratch),
           scratch.numel(), N.stream_handle())
    trans = (t_indptr, t_dst, t_w, torch.tensor([n_src], device=dev))
    h = torch.randn(n_src, H, device=dev).to(torch.bfloat16).requires_grad_(True)
    a = block_mean(h, ip, sl, nd, max_dst, relu=True, trans=trans, bias_col=True, edge_w=ew)
    seg = torch.repeat_interleave(torch.arange(n_dst, device=dev),
                                  torch.from_numpy(counts).long().to(dev))
    hf = h.detach().float().requires_grad_(True)
    ref = torch.zeros(n_dst, H, device=dev).index_add_(0, seg, torch.relu(hf[sl.long()]) *
                                                       ew[:, None])
    assert torch.allclose(a[:n_dst, :H].float(), ref, atol=2e-2, rtol=1e-2)
    g = torch.randn(max_dst, H + 8, device=dev).to(torch.bfloat16)
    a.backward(g)
    ref.backward(g[:n_dst, :H].float())
    assert torch.allclose(h.grad.float(), hf.grad, atol=2e-2, rtol=2e-2)
    # weighted wgrad: dW = sum_e (relu'(h[l_e]) * w_e g[v_e])^T x[l_e]
    x = torch.randn(n_src, P, device=dev).to(torch.bfloat16)
    dw = block_mean_wgrad(g, ip, sl, nd, max_dst, h.detach(), x, H=H, edge_w=ew)
    term = g[seg, :H].float() * ew[:, None] * (h.detach()[sl.long()].float() > 0)
    want = term.to(torch.bfloat16).float().t() @ x[sl.long()].float()
    assert (dw - want).abs().max().item() <= 1e-3 * want.abs().max().item() + 1e-4


@pytest.mark.parametrize("weighted", [False, True])
def test_block_mean_fwd_emits_relu_bits(weighted):
    """fg_block_mean_fwd_bits: same output as fg_block_mean_fwd(relu), and the
    packed ReLU mask of every source the block reads equals relu_mask_bits."""
    from paper_2207_14696_b200 import _native as N
    from paper_2207_14696_b200.aggregate import relu_mask_bits
    rng = np.random.default_rng(11 + weighted)
    H, n_src, n_dst, max_dst, fan = 256, 3000, 900, 950, 7
    counts, indptr, src = _block(n_src, n_dst, max_dst, fan, rng, zero_frac=0.1)
    dev = "cuda"
    ip = torch.from_numpy(indptr).to(dev)
    local = torch.from_numpy(src).to(dev)
    nd = torch.tensor([n_dst], device=dev)
    h = torch.randn(n_src, H, device=dev).to(torch.bfloat16)
    ew = torch.rand(max(src.size, 1), device=dev) if weighted else None
    a = torch.empty((max_dst, H + 8), dtype=torch.bfloat16, device=dev)
    b = torch.empty_like(a)
    bits = torch.zeros((n_src, H // 8), dtype=torch.uint8, device=dev)
    s = N.stream_handle()
    N.call("fg_block_mean_fwd", N.ptr(h), H, N.ptr(ip), N.ptr(local), N.ptr(nd), max_dst,
           N.ptr(a), H + 8, 1, N.ptr(ew), s)
    N.call("fg_block_mean_fwd_bits", N.ptr(h), H, N.ptr(ip), N.ptr(local), N.ptr(nd), max_dst,
           N.ptr(b), H + 8, N.ptr(ew), N.ptr(bits), s)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    used = torch.unique(local.long())
    assert torch.equal(bits[used], relu_mask_bits(h)[used])


@pytest.mark.parametrize("H,P,fan,weighted,n_dst", [(256, 112, 10, False, 700),
                                                    (256, 144, 15, True, 700),
                                                    (128, 48, 5, False, 700),
                                                    (256, 112, 1, False, 700),
                                                    (128, 256, 40, True, 700),
                                                    (256, 112, 10, False, 20000),
                                                    (256, 112, 10, True, 20000)])
def test_input_block_mean_fwd_tcgen05(H, P, fan, weighted, n_dst):
    """Fused h0 = x W0^T + ReLU block mean (tcgen05) against torch fp32 on the
    same bf16 operands; ReLU bits against the fp32 signs (away from 0); dead
    rows get zeros + the bias column."""
    from paper_2207_14696_b200 import _native as N
    assert N.lib().fg_input_block_mean_supported(H, P, fan)
    rng = np.random.default_rng(H + P + fan)
    n_src, max_dst = 3000, n_dst + 60   # n_dst 20000: several tiles per CTA
    counts, indptr, src = _block(n_src, n_dst, max_dst, fan, rng, zero_frac=0.1)
    dev = "cuda"
    ip = torch.from_numpy(indptr).to(dev)
    local = torch.from_numpy(src).to(dev)
    x = torch.randn(n_src, P, device=dev).to(torch.bfloat16)
    w0 = (torch.randn(H, P, device=dev) / P ** 0.5).to(torch.bfloat16)
    ew = torch.rand(max(src.size, 1), device=dev) if weighted else None
    out = torch.full((max_dst, H + 8), float("nan"), dtype=torch.bfloat16, device=dev)
    bits = torch.zeros((n_src, H // 8), dtype=torch.uint8, device=dev)
    N.call("fg_input_block_mean_fwd", N.ptr(x), P, N.ptr(w0), H, N.ptr(ip), N.ptr(local),
           N.ptr(torch.tensor([n_dst], device=dev)), max_dst, fan, N.ptr(ew), N.ptr(out), H + 8,
           N.ptr(bits), N.stream_handle())
    torch.cuda.synchronize()
    h = x.float() @ w0.float().t()
    dst = torch.repeat_interleave(torch.arange(n_dst, device=dev),
                                  torch.from_numpy(counts).long().to(dev))
    l = local.long()
    w = ew[:src.size] if weighted else 1.0 / torch.from_numpy(counts).float().to(dev)[dst]
    ref = torch.zeros(max_dst, H, device=dev).index_add_(0, dst, h[l].clamp_min(0) * w[:, None])
    got = out[:, :H].float()
    assert torch.allclose(got, ref, atol=2e-2, rtol=1e-2), (got - ref).abs().max()
    assert (got[n_dst:] == 0).all()
    assert (out[:, H].float() == 1).all() and (out[:, H + 1:] == 0).all()
    used = torch.unique(l)
    hb = h[used] > 0
    sh = torch.arange(8, device=dev, dtype=torch.uint8)
    gbits = ((bits[used][..., None] >> sh) & 1).view(-1, H).bool()
    clear = h[used].abs() > 1e-3
    assert torch.equal(gbits[clear], hb[clear])


@pytest.mark.parametrize("K,M,N,chunks", [(153600, 256, 784, 16), (70001, 256, 112, 32),
                                          (40000, 48, 264, None)])
def test_kgemm_matches_fp32_reference(K, M, N, chunks):
    """kgemm (the K-sliced weight-gradient GEMM: MAG's GEMM-path dW0 with 16
    slices, GAT's K-GEMMs, a K % chunks tail) against an fp32 GEMM of the
    same bf16 operands; fp32 partials summed, so within fp32 rounding of a
    K-long dot product."""
    from paper_2207_14696_b200.aggregate import kgemm
    g = torch.Generator(device="cuda").manual_seed(K)
    a = torch.randn(K, M, device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randn(K, N, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.full((M, N), float("nan"), device="cuda")
    kgemm(a, b, out, chunks=chunks)
    ref = a.double().t() @ b.double()
    err = (out.double() - ref).abs().max().item()
    assert err <= 1e-4 * K ** 0.5, err
