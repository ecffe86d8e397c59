"""Diagnostic: per-step device time of the captured training step under
different host patterns (back-to-back replays, L2 flush between steps, host
sync per step).  Not a benchmark line; bench.py is."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2207_14696_b200.sage import SageTrainer, TrainConfig  # noqa: E402


def main():
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "products"
    pipe = (sys.argv[2] != "serial") if len(sys.argv) > 2 else True
    dev = torch.device("cuda", 0)
    sg, dc, desc, fanouts, bs, hidden = bench.build_workload(cfg_name, dev)
    tr = SageTrainer(sg.graph, dc, sg.labels, sg.num_classes,
                     TrainConfig(fanouts=fanouts, batch_size=bs, hidden=hidden, pipeline=pipe))
    tr.begin_epoch(sg.train_ids, 0)
    tr.capture(3)
    flush = torch.zeros(128 * 1024 * 1024, dtype=torch.float32, device=dev)
    b = 0
    for b in range(5):
        tr.step(b)
    torch.cuda.synchronize()
    for mode in ("b2b", "flush", "flush+sync", "b2b"):
        ts = []
        for i in range(40):
            b += 1
            if "flush" in mode:
                flush.add_(1)
            tr.prepare(b)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            tr.replay(b)
            e.record()
            if "sync" in mode:
                e.synchronize()
            ts.append((s, e))
        torch.cuda.synchronize()
        ms = [s.elapsed_time(e) for s, e in ts]
        print(f"{desc} pipeline={pipe} {mode:11s} median {statistics.median(ms) * 1e3:.1f} us "
              f"mean {statistics.mean(ms) * 1e3:.1f} min {min(ms) * 1e3:.1f} max {max(ms) * 1e3:.1f}")


if __name__ == "__main__":
    main()
