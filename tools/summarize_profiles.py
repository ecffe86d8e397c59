"""Condense ncu artefacts from gpurun_out/ into profiles/<round>/ (tracked).

    python tools/summarize_profiles.py --round round1 --launches gpurun_out/launchesN.csv \
        --report gpurun_out/prof_vqN.ncu-rep [--bench gpurun_out/bench.log]
"""
import argparse
import collections
import csv
import json
import os
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_bytes.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, mi, ii = (h.index(x) for x in ("Kernel Name", "Metric Value", "Metric Name", "ID"))
    per = collections.OrderedDict()
    for r in data:
        if len(r) <= vi:
            continue
        d = per.setdefault(r[ii], {"kernel": r[ki]})
        d[r[mi]] = r[vi]
    items = list(per.values())
    step = items[len(items) // 2:]  # second profiled step (warm)
    out = []
    for d in step:
        us = float(d["gpu__time_duration.sum"].replace(",", "")) / 1e3
        out.append({"kernel": d["kernel"].split("(")[0], "us": round(us, 2),
                    "grid": d.get("launch__grid_size"), "block": d.get("launch__block_size")})
    return out


def report_metrics(path):
    if path.endswith(".csv"):  # `ncu -i rep --page raw --csv` output saved on the GPU box
        text = open(path).read()
    else:
        text = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                              capture_output=True, text=True).stdout
    rows = list(csv.reader(text.splitlines()))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        res.append({k: (v[h.index(k)], u[h.index(k)]) for k in KEYS if k in h} |
                   {"kernel": v[h.index("Kernel Name")].split("(")[0]})
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="round1")
    ap.add_argument("--launches")
    ap.add_argument("--report", action="append", default=[])
    ap.add_argument("--bench")
    ap.add_argument("--breakdown")
    a = ap.parse_args()
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        a.round)
    os.makedirs(root, exist_ok=True)
    if a.launches:
        ls = launches(a.launches)
        tot = sum(x["us"] for x in ls)
        agg = collections.defaultdict(float)
        for x in ls:
            agg[x["kernel"]] += x["us"]
        with open(os.path.join(root, "step_launches.json"), "w") as fh:
            json.dump({"note": "ncu --metrics gpu__time_duration.sum --clock-control none, one "
                               "eager training step (tools/profile_step.py), cold-cache "
                               "serialised: compare shares, not absolutes",
                       "total_us": round(tot, 1), "launches": ls}, fh, indent=1)
        with open(os.path.join(root, "step_launches.md"), "w") as fh:
            fh.write(f"# One training step, per-kernel device time (ncu, serialised)\n\n"
                     f"total {tot:.1f} us over {len(ls)} launches\n\n| us | share | kernel |\n"
                     f"|---:|---:|---|\n")
            for k, v in sorted(agg.items(), key=lambda x: -x[1]):
                fh.write(f"| {v:.1f} | {v / tot * 100:.1f}% | `{k}` |\n")
    for rep in a.report:
        m = report_metrics(rep)
        name = os.path.splitext(os.path.basename(rep))[0].removesuffix("_raw")
        with open(os.path.join(root, f"{name}_summary.json"), "w") as fh:
            json.dump({"source": f"ncu --set full --clock-control none --import-source on "
                                 f"({os.path.basename(rep)})", "kernels": m}, fh, indent=1)
    if a.bench:
        lines = [l for l in open(a.bench) if l.startswith("{")]
        if lines:
            with open(os.path.join(root, "bench_line.json"), "w") as fh:
                fh.write(lines[-1])
    if a.breakdown:
        lines = [l for l in open(a.breakdown) if l.startswith("{")]
        if lines:
            with open(os.path.join(root, "phase_breakdown.json"), "w") as fh:
                fh.write(lines[-1])


if __name__ == "__main__":
    main()
