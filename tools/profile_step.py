"""Run a few eager training steps of the bench workload inside an NVTX range
"step" (for `ncu --nvtx --nvtx-include step/ ...` launch lists and focused
captures).  Not a benchmark: numbers printed under a profiler are not
measurements."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2207_14696_b200.sage import SageTrainer, TrainConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="products")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    # run backward on this thread so its kernels fall inside the NVTX range
    torch.autograd.set_multithreading_enabled(False)
    sg, dc, desc, fanouts, bs, hidden = bench.build_workload(a.config, dev, scale=a.scale)
    if bench.aggregator_of(a.config) == "gat":
        from paper_2207_14696_b200.gat import GatConfig, GatTrainer
        tr = GatTrainer(sg.graph, dc, sg.labels, sg.num_classes,
                        GatConfig(fanouts=fanouts, batch_size=bs, hidden=hidden))
    else:
        tr = SageTrainer(sg.graph, dc, sg.labels, sg.num_classes,
                         TrainConfig(fanouts=fanouts, batch_size=bs, hidden=hidden,
                                     aggregator=bench.aggregator_of(a.config)))
    tr.begin_epoch(sg.train_ids, 0)
    for b in range(3):
        tr.step(b)
    torch.cuda.synchronize()
    for i in range(a.steps):
        b = 3 + i
        tr.prepare(b)  # seeds of the batch this step samples (outside the range)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("step")
        tr._body(b % len(tr.samplers))
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
    print("profiled", a.steps, "steps of", desc)


if __name__ == "__main__":
    main()
