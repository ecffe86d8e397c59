"""Time the fused gather-dequant-mean kernel alone on a bench workload's real
sampled blocks (CUDA events, L2 flushed before every launch), and report
achieved algorithmic GB/s.  Kernel variants are chosen by the environment
(FG_VQ_LANE=0/1, ...), so A/B runs are separate processes:

    python tools/fused_bench.py --config mag240m --iters 20
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2207_14696_b200.aggregate import alloc_aggregate, gather_dequant_mean  # noqa: E402
from paper_2207_14696_b200.sampler import DeviceSampler  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mag240m")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--check", action="store_true", help="compare against FG_VQ_LANE=0 output "
                    "computed in this process (fp32 kernel as reference)")
    ap.add_argument("--probe", default="", help="comma list of FG_FUSED_PROBE diagnostic "
                    "variants to sweep in this process (1 no gather, 2 no decode, 4 no store)")
    ap.add_argument("--flush", default="write", help="comma list of L2 flush modes to sweep: "
                    "write (512 MB write) | write+read (then a 256 MB read, so the flush's "
                    "dirty lines are written back before the timed launch)")
    ap.add_argument("--pitch", type=int, default=0, help="output row pitch in elements "
                    "(default: aggregate.padded_dim(d))")
    ap.add_argument("--l2", default="", help="comma list of L2 fetch granularities (bytes) "
                    "to sweep in this process (fg_set_l2_fetch_granularity); default: as is")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    sg, dc, desc, fanouts, bs, hidden = bench.build_workload(a.config, dev)
    smp = DeviceSampler(sg.graph, fanouts, bs, need_local=True)
    smp.begin_epoch(sg.train_ids, 0)
    L = len(fanouts)
    out = alloc_aggregate(smp.caps[L - 1], dc.d, torch.bfloat16, dev)
    if a.pitch:
        out = torch.zeros((smp.caps[L - 1], a.pitch), dtype=torch.bfloat16, device=dev)
    flush = torch.zeros(128 * 1024 * 1024, dtype=torch.float32, device=dev)
    rflush = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    sink = torch.zeros(1, dtype=torch.float32, device=dev)
    row_bytes = dc.num_parts * dc.bits / 8 if hasattr(dc, "num_parts") else dc.d * dc.params.k / 8
    from paper_2207_14696_b200 import _native as N
    grans = [int(x) for x in a.l2.split(",") if x] or [0]
    base = smp.rng.clone()
    probes = [x for x in a.probe.split(",") if x] or [os.environ.get("FG_FUSED_PROBE", "0")]
    for g in grans:
        if g:
            N.call("fg_set_l2_fetch_granularity", g)
        for pr in probes:
            for fm in a.flush.split(","):
                os.environ["FG_FUSED_PROBE"] = pr
                smp.rng.copy_(base)
                fl = (lambda: flush.add_(1)) if fm == "write" else \
                    (lambda: (flush.add_(1), torch.sum(rflush, dim=0, keepdim=True, out=sink)))
                run(a, dc, smp, out, fl, row_bytes, L, N.l2_fetch_granularity(), fm)


def run(a, dc, smp, out, flush, row_bytes, L, gran, fm="write"):
    ts, bts = [], []
    for i in range(a.iters + 3):
        sb = smp.sample(i)
        torch.cuda.synchronize()
        E = int(sb.n_picks[L - 1].item())
        nd = int(sb.n_nodes[L - 1].item())
        flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        gather_dequant_mean(dc, sb.indptr[L - 1], sb.picks[L - 1], sb.n_nodes[L - 1],
                            smp.caps[L - 1], out=out)
        e.record()
        e.synchronize()
        if i >= 3:
            ts.append(s.elapsed_time(e))
            bts.append(E * (row_bytes + 4) + nd * (4 + dc.d * 2))
        if a.check and i == 3:
            ref = gather_dequant_mean(dc, sb.indptr[L - 1], sb.picks[L - 1], sb.n_nodes[L - 1],
                                      smp.caps[L - 1], out_dtype=torch.float32)
            diff = (out[:nd, :dc.d].float() - ref[:nd, :dc.d]).abs()
            scale = ref[:nd, :dc.d].abs().mean().item()
            print(f"check: max |bf16 - fp32| = {diff.max().item():.3g} "
                  f"(mean |x| {scale:.3g})", file=sys.stderr)
    us = sum(ts) / len(ts) * 1e3
    gbs = sum(bts) / len(bts) / (us * 1e-6) / 1e9
    peak, _ = bench.load_peaks()
    print(json.dumps({"config": a.config, "lane": os.environ.get("FG_VQ_LANE", "0"),
                      "l2_fetch": gran, "flush": fm, "pitch": out.shape[1], "probe": os.environ.get("FG_FUSED_PROBE", "0"),
                      "avg_us": round(us, 2), "min_us": round(min(ts) * 1e3, 2),
                      "alg_bytes": int(sum(bts) / len(bts)), "GBps": round(gbs, 1),
                      "frac": round(gbs / peak, 4)}))


if __name__ == "__main__":
    main()
