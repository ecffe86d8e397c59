"""Diagnostic: fg_block_mean_wgrad alone on a products-shaped input block
(15 360 destinations x 10 picks over 104 K source rows, H=256, P=112)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2207_14696_b200.aggregate import block_mean_wgrad, wgrad_scratch  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    n_src, n_dst, fan, H, P = 104_000, 15_360, 10, 256, int(sys.argv[1]) if len(sys.argv) > 1 else 112
    counts = np.full(n_dst, fan)
    indptr = np.zeros(n_dst + 1, np.int32)
    indptr[1:] = np.cumsum(counts)
    # power-law-ish sources (hubs), like a real sampled block
    src = np.minimum((rng.pareto(1.2, indptr[-1]) * 2000).astype(np.int64), n_src - 1)
    dev = "cuda"
    ip = torch.from_numpy(indptr).to(dev)
    sl = torch.from_numpy(src.astype(np.int32)).to(dev)
    nd = torch.tensor([n_dst], device=dev)
    g = torch.randn(n_dst, H, device=dev).to(torch.bfloat16)
    h = torch.randn(n_src, H, device=dev).to(torch.bfloat16)
    x = torch.randn(n_src, P, device=dev).to(torch.bfloat16)
    scratch = wgrad_scratch(H, P, dev)
    dw = torch.empty(H, P, device=dev)
    flush = torch.empty(128 * 1024 * 1024, device=dev)
    ts = []
    for i in range(30):
        flush.add_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        block_mean_wgrad(g, ip, sl, nd, n_dst, h, x, dw=dw, scratch=scratch, H=H)
        e.record()
        ts.append((s, e))
    torch.cuda.synchronize()
    print(f"wgrad (kernel + reduce): median {statistics.median(a.elapsed_time(b) for a, b in ts) * 1e3:.1f} us "
          f"for {indptr[-1]} edges, P={P}, v2={os.environ.get('FG_WGRAD_V2', '1')}")


if __name__ == "__main__":
    main()
