"""Diagnostic: the input layer's forward on a real products batch -- cuBLAS
h0 GEMM + block mean (with ReLU bits) vs the fused tcgen05 kernel
(fg_input_block_mean_fwd) -- each alone in a CUDA graph, and the max
abs difference of the outputs.  Not a bench line."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2207_14696_b200 import _native as N  # noqa: E402
from paper_2207_14696_b200.sage import SageTrainer, TrainConfig  # noqa: E402
from tools.chain_timing import timed  # noqa: E402


def main():
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "products"
    dev = torch.device("cuda", 0)
    sg, dc, desc, fanouts, bs, hidden = bench.build_workload(cfg_name, dev)
    tr = SageTrainer(sg.graph, dc, sg.labels, sg.num_classes,
                     TrainConfig(fanouts=fanouts, batch_size=bs, hidden=hidden,
                                 aggregator=bench.aggregator_of(cfg_name)))
    tr.begin_epoch(sg.train_ids, 0)
    tr.capture(3)
    for b in range(3):
        tr.step(b)
    torch.cuda.synchronize()
    sb = tr.samplers[0].batch_view()
    L = len(fanouts)
    l = L - 2
    W0 = tr.w_bf16[0]
    H = W0.shape[0]
    caps = tr.caps
    ew = sb.ew[l] if sb.ew else None
    a1 = torch.empty((caps[l], H + 8), dtype=torch.bfloat16, device=dev)
    a2 = torch.empty_like(a1)
    bits = tr.relu_bits

    def unfused():
        s = N.stream_handle()  # the capture stream inside torch.cuda.graph
        h = torch.mm(tr.agg, W0.t())
        N.call("fg_block_mean_fwd_bits", N.ptr(h), H, N.ptr(sb.indptr[l]), N.ptr(sb.local[l]),
               N.ptr(sb.n_nodes[l]), caps[l], N.ptr(a1), H + 8, N.ptr(ew), N.ptr(bits), s)

    def fused():
        s = N.stream_handle()
        N.call("fg_input_block_mean_fwd", N.ptr(tr.agg), tr.agg.shape[1], N.ptr(W0), H,
               N.ptr(sb.indptr[l]), N.ptr(sb.local[l]), N.ptr(sb.n_nodes[l]), caps[l],
               fanouts[l], N.ptr(ew), N.ptr(a2), H + 8, N.ptr(bits), s)
    for f in (unfused, fused):
        f()
    torch.cuda.synchronize()
    gs = []
    for f in (unfused, fused):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f()
        gs.append(g)
    torch.cuda.synchronize()
    nd = int(sb.n_nodes[l].item())
    ne = int(sb.indptr[l][nd].item())
    # fp32 reference from the same operands
    ip = sb.indptr[l][:nd + 1].long()
    cnt = ip[1:] - ip[:-1]
    dst = torch.repeat_interleave(torch.arange(nd, device=dev), cnt)
    src = sb.local[l][int(ip[0]):int(ip[-1])].long()
    h = tr.agg.float() @ W0.float().t()
    w = ew[int(ip[0]):int(ip[-1])] if ew is not None else 1.0 / cnt.float()[dst]
    ref = torch.zeros(nd, H, device=dev).index_add_(0, dst, h[src].clamp_min(0) * w[:, None])
    for name, a in (("unfused", a1), ("fused", a2)):
        err = (a[:nd, :H].float() - ref).abs()
        bad = (err > 1e-2 + 1e-2 * ref.abs()).any(1).nonzero().flatten()
        print(f"{name}: rel-norm vs fp32 {(err.norm() / ref.norm()).item():.3g}, bad rows "
              f"{bad.numel()} first {bad[:8].tolist()} ip0 {int(ip[0])} max cnt {int(cnt.max())} "
              f"src max {int(src.max())} agg rows {tr.agg.shape[0]}")
    print(f"{desc}: block {l}: {nd} dst, {ne} edges, x rows {tr.agg.shape}; "
          f"unfused {timed(gs[0].replay):.1f} us, fused {timed(gs[1].replay):.1f} us, "
          f"max |diff| {(a1.float() - a2.float()).abs().max().item():.3g} "
          f"(max |a| {a1.float().abs().max().item():.3g}, rel-norm "
          f"{((a1.float() - a2.float()).norm() / a1.float().norm()).item():.3g})")


if __name__ == "__main__":
    main()
