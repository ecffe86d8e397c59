"""Diagnostic: device time of the training chain alone, the sampling chain
alone, and the pipelined step (both overlapped) — each captured in a CUDA
graph and replayed back to back.  Not a bench line; bench.py is."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2207_14696_b200.sage import SageTrainer, TrainConfig  # noqa: E402


def timed(fn, reps=40):
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        ts.append((s, e))
    torch.cuda.synchronize()
    return statistics.median(s.elapsed_time(e) for s, e in ts) * 1e3


def main():
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "products"
    dev = torch.device("cuda", 0)
    sg, dc, desc, fanouts, bs, hidden = bench.build_workload(cfg_name, dev)
    tr = SageTrainer(sg.graph, dc, sg.labels, sg.num_classes,
                     TrainConfig(fanouts=fanouts, batch_size=bs, hidden=hidden,
                                 aggregator=bench.aggregator_of(cfg_name)))
    tr.begin_epoch(sg.train_ids, 0)
    tr.capture(3)
    for b in range(5):
        tr.step(b)
    torch.cuda.synchronize()
    smp = tr.samplers[1]
    sb = tr.samplers[0].batch_view()
    g_train, g_sample = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_train):
        tr._train(sb)
    with torch.cuda.graph(g_sample):
        smp.sample_loaded()
    torch.cuda.synchronize()
    b = [10]

    def step():
        tr.prepare(b[0])
        tr.replay(b[0])
        b[0] += 1
    print(f"{desc}: train chain {timed(g_train.replay):.1f} us, sample chain "
          f"{timed(g_sample.replay):.1f} us, pipelined step {timed(step):.1f} us (median)")


if __name__ == "__main__":
    main()
