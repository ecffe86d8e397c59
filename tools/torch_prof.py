"""Map device kernels of one eager training step to the torch ops that
launched them (torch.profiler, shapes recorded).  Diagnostic only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2207_14696_b200.sage import SageTrainer, TrainConfig  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "products"
    dev = torch.device("cuda", 0)
    sg, dc, desc, fanouts, bs, hidden = bench.build_workload(cfg, dev)
    tr = SageTrainer(sg.graph, dc, sg.labels, sg.num_classes,
                     TrainConfig(fanouts=fanouts, batch_size=bs, hidden=hidden,
                                 pipeline=False))
    tr.begin_epoch(sg.train_ids, 0)
    for b in range(3):
        tr.sampler.load_seeds(b)
        tr._body()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], record_shapes=True) as p:
        tr.sampler.load_seeds(3)
        tr._body()
        torch.cuda.synchronize()
    print(p.key_averages(group_by_input_shape=True).table(sort_by="cuda_time_total", row_limit=40,
                                                           max_name_column_width=60,
                                                           max_shapes_column_width=80))


if __name__ == "__main__":
    main()
