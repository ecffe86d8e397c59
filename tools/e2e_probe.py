"""Diagnostic: where the end-to-end step (public API, seeds from pinned host
memory, loss read back) spends its time beyond the device-resident step.
Per-step CUDA-event windows like bench.py, L2 flushed between steps."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2207_14696_b200.sage import SageTrainer, TrainConfig  # noqa: E402


def main():
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "papers100m"
    dev = torch.device("cuda", 0)
    sg, dc, desc, fanouts, bs, hidden = bench.build_workload(cfg_name, dev)
    tr = SageTrainer(sg.graph, dc, sg.labels, sg.num_classes,
                     TrainConfig(fanouts=fanouts, batch_size=bs, hidden=hidden,
                                 aggregator=bench.aggregator_of(cfg_name)))
    tr.begin_epoch(sg.train_ids, 0)
    tr.capture(3)
    flush = torch.zeros(128 * 1024 * 1024, dtype=torch.float32, device=dev)
    perm = tr.sampler.perm_host
    K = 30
    pinned = [torch.from_numpy(perm[(b + 1) * bs:(b + 2) * bs].astype(np.int32)).pin_memory()
              for b in range(200)]
    loss_host = torch.zeros(200, dtype=torch.float32).pin_memory()

    import time

    def run(mode, b0):
        evs = []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(K):
            b = b0 + i
            bench.flush_l2(flush)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if mode == "device":
                tr.prepare(b)
                s.record()
                tr.replay(b)
            elif mode == "device+prep":
                s.record()
                tr.prepare(b)
                tr.replay(b)
            elif mode == "h2d":
                s.record()
                tr.step(b, seeds_host=pinned[i])
            else:  # h2d+d2h
                s.record()
                loss = tr.step(b, seeds_host=pinned[i])
                loss_host[i].copy_(loss, non_blocking=True)
            e.record()
            evs.append((s, e))
        host_us = (time.perf_counter() - t0) / K * 1e6  # enqueue rate (no sync in the loop)
        torch.cuda.synchronize()
        return statistics.median(s.elapsed_time(e) for s, e in evs) * 1e3, host_us

    b = 10
    for mode in ["device", "device+prep", "h2d", "h2d+d2h", "device", "h2d+d2h"]:
        dev_us, host_us = run(mode, b)
        print(f"{desc}: {mode:12s} {dev_us:.1f} us/step device (median of {K}), "
              f"host enqueue {host_us:.1f} us/step", flush=True)
        b += K + 2


if __name__ == "__main__":
    main()
