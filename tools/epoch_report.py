"""Paper-style epoch breakdown (cf. the reference's simulate_epoch /
compare_reports, pipeline.py:300-383) with MEASURED B200 stage times for the
products-shape workloads: VQ (config B) vs SQ k=8 vs GCN-SQ8, same sampling
plan.  Writes the text table and the JSON reports."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2207_14696_b200.measure import compare_reports, measure_epoch, render_text  # noqa: E402
from paper_2207_14696_b200.sage import SageTrainer, TrainConfig  # noqa: E402


def main():
    out_dir = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
    dev = torch.device("cuda", 0)
    reports = []
    for cfg_name in ("products-sq8", "products", "products-gcn"):
        sg, dc, desc, fanouts, bs, hidden = bench.build_workload(cfg_name, dev)
        tr = SageTrainer(sg.graph, dc, sg.labels, sg.num_classes,
                         TrainConfig(fanouts=fanouts, batch_size=bs, hidden=hidden,
                                     aggregator=bench.aggregator_of(cfg_name)))
        label = f"{cfg_name}: {desc}"
        reports.append(measure_epoch(tr, sg.train_ids, label, batches=30))
        del tr, sg, dc
        torch.cuda.empty_cache()
    # the GCN row runs a different model on the same plan: compare SQ vs VQ only
    out = compare_reports(reports[0], reports[1:2]) + [reports[2]]
    text = render_text(out)
    print(text)
    with open(os.path.join(out_dir, "epoch_report.txt"), "w") as fh:
        fh.write(text + "\n")
    with open(os.path.join(out_dir, "epoch_report.json"), "w") as fh:
        json.dump([r.to_dict() for r in out], fh, indent=1)


if __name__ == "__main__":
    main()
