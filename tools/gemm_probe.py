"""Diagnostic: device time of the weight-gradient GEMM shapes of the SAGE
step under different cuBLAS formulations (each variant CUDA-graph captured
and replayed, so host launch overhead is excluded)."""
import statistics
import sys

import torch


def timed_graph(fn, reps=30):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) for x, y in ts) * 1e3


def main():
    dev = "cuda"
    shapes = [(256, 60000, 784), (256, 104000, 112), (256, 15360, 264), (48, 1024, 264)]
    for M, K, N in shapes:
        dh = torch.randn(K, M, device=dev).bfloat16()
        x = torch.randn(K, N, device=dev).bfloat16()
        o32 = torch.empty(M, N, device=dev)
        o32t = torch.empty(N, M, device=dev)
        o16 = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        r = {
            "dhT@x fp32": timed_graph(lambda: torch.mm(dh.t(), x, out_dtype=torch.float32, out=o32)),
            "dhT@x bf16": timed_graph(lambda: torch.mm(dh.t(), x, out=o16)),
            "xT@dh fp32": timed_graph(lambda: torch.mm(x.t(), dh, out_dtype=torch.float32, out=o32t)),
        }
        flop = 2.0 * M * K * N
        print(f"M{M} K{K} N{N}: " + ", ".join(f"{k} {v:.1f}us ({flop / v / 1e6:.0f} TF/s)"
                                                for k, v in r.items()))
    # MAG240M-shape layer 1 (GEMM path, P = 784): dW0 and h0 formulations
    sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(
        __import__("os").path.abspath(__file__))))
    from paper_2207_14696_b200.aggregate import kgemm
    for K in (96000, 150000):
        dh = torch.randn(K, 256, device=dev).bfloat16()
        x = torch.randn(K, 784, device=dev).bfloat16()
        o32 = torch.empty(256, 784, device=dev)
        o32t = torch.empty(784, 256, device=dev)
        w = torch.randn(256, 784, device=dev).bfloat16()
        h = torch.empty(K, 256, device=dev, dtype=torch.bfloat16)
        flop = 2.0 * 256 * K * 784
        r = {"dhT@x": timed_graph(lambda: torch.mm(dh.t(), x, out_dtype=torch.float32, out=o32)),
             "xT@dh": timed_graph(lambda: torch.mm(x.t(), dh, out_dtype=torch.float32, out=o32t)),
             "h0=x@wT": timed_graph(lambda: torch.mm(x, w.t(), out=h))}
        for c in (8, 16, 32, 64):
            r[f"kgemm{c}"] = timed_graph(lambda: kgemm(dh, x, o32, chunks=c))
        print(f"MAG K{K}: " + ", ".join(f"{k} {v:.1f}us ({flop / v / 1e6:.0f} TF/s)"
                                        for k, v in r.items()))
    x = torch.randn(60000, 784, device=dev).bfloat16()
    w = torch.randn(256, 784, device=dev).bfloat16()
    print(f"h0 = agg W0^T (60000x784x256): {timed_graph(lambda: torch.mm(x, w.t())):.1f}us")


if __name__ == "__main__":
    sys.exit(main())
