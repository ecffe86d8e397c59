"""Per-phase GPU time of one training step, each phase captured in its own
CUDA graph and timed with CUDA events (L2 flushed before each replay).
Phases: sample (3 layers + uniques), aggregate (fused gather-dequant-mean),
model (SAGE fwd + loss + bwd + Adam)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

import bench  # noqa: E402
from paper_2207_14696_b200.aggregate import gather_dequant_mean  # noqa: E402
from paper_2207_14696_b200.sage import SageTrainer, TrainConfig  # noqa: E402


def timed(g, n, flush):
    ts = []
    for _ in range(n):
        if flush is not None:
            flush.add_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return sum(ts) / len(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="products")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    sg, dc, desc, fanouts, bs, hidden = bench.build_workload(a.config, dev)
    tr = SageTrainer(sg.graph, dc, sg.labels, sg.num_classes,
                     TrainConfig(fanouts=fanouts, batch_size=bs, hidden=hidden,
                                 pipeline=False))
    tr.begin_epoch(sg.train_ids, 0)
    L = len(fanouts)
    flush = torch.zeros(128 * 1024 * 1024, device=dev)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for b in range(3):
            tr.sampler.load_seeds(b)
            tr._body()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    tr.sampler.load_seeds(5)
    gs, ga, gm, gfull = (torch.cuda.CUDAGraph() for _ in range(4))
    with torch.cuda.graph(gs):
        sb = tr.sampler.sample_loaded()
    with torch.cuda.graph(ga):
        gather_dequant_mean(dc, sb.indptr[L - 1], sb.picks[L - 1], sb.n_nodes[L - 1],
                            tr.caps[L - 1], out=tr.agg)

    def fwd_part():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            logits = tr.model(tr.agg, sb, tr.caps)
        from paper_2207_14696_b200.aggregate import softmax_ce
        return softmax_ce(logits, tr.labels, sb.nodes[0], sb.n_nodes[0], tr.model.num_classes)

    gf, gfb, go = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(gf):
        fwd_part()
    with torch.cuda.graph(gfb):
        tr.flat_grad.zero_()
        fwd_part().backward()
    with torch.cuda.graph(go):
        tr.opt.step()

    def model_part():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            logits = tr.model(tr.agg, sb, tr.caps)
        from paper_2207_14696_b200.aggregate import softmax_ce
        loss = softmax_ce(logits, tr.labels, sb.nodes[0], sb.n_nodes[0], tr.model.num_classes)
        tr.flat_grad.zero_()
        loss.backward()
        tr.opt.step()
    with torch.cuda.graph(gm):
        model_part()
    with torch.cuda.graph(gfull):
        tr._body()
    torch.cuda.synchronize()
    out = {"config": desc}
    for name, g in [("sample", gs), ("aggregate", ga), ("model", gm), ("fwd", gf),
                    ("fwd_bwd", gfb), ("adam", go), ("full_step", gfull)]:
        out[name + "_us"] = round(timed(g, a.reps, flush), 1)
        out[name + "_warm_us"] = round(timed(g, a.reps, None), 1)
    out["live"] = [int(x.item()) for x in sb.n_nodes] + [int(sb.n_picks[-1].item())]
    out["caps"] = tr.caps
    print(json.dumps(out))


if __name__ == "__main__":
    main()
