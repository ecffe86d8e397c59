"""Copy one validation run's artefacts (gpurun_out/<dir>/, produced by
tools/gpu/r4a.sh-style scripts) into profiles/round2/: bench lines, test and
smoke logs, fused-kernel ncu summaries and briefs, per-step launch lists.

    python tools/refresh_round2.py gpurun_out/r4a
"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DST = os.path.join(ROOT, "profiles", "round2")


def step_launches(path, cfg):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Value", "ID"))
    per = collections.OrderedDict()
    for r in data:
        if len(r) > vi:
            per[r[ii]] = (r[ki], float(r[vi].replace(",", "")) / 1e3)
    items = list(per.values())
    step = items[len(items) // 2:]  # the second (warm) profiled step
    tot = sum(u for _, u in step)
    ks = sorted(({"name": n[:120], "us": round(u, 2), "share": round(u / tot, 4)} for n, u in step),
                key=lambda x: -x["us"])
    return {"config": cfg, "source": "ncu --nvtx --nvtx-include step/ --metrics "
            "gpu__time_duration.sum --clock-control none, tools/profile_step.py (eager step 2 "
            "of 2; serialized, cold per-launch)", "step_total_us": round(tot, 1), "kernels": ks}


def main():
    src = sys.argv[1]
    for f in os.listdir(src):
        p = os.path.join(src, f)
        if f.startswith("bench_") and f.endswith(".json"):
            name = f[len("bench_"):-len(".json")]
            shutil.copy(p, os.path.join(DST, f"bench_line_{name}.json"))
        elif f.endswith("_brief.txt"):
            shutil.copy(p, os.path.join(DST, f))
        elif f.endswith("_raw.csv"):
            subprocess.run([sys.executable, os.path.join(ROOT, "tools", "summarize_profiles.py"),
                            "--round", "round2", "--report", p], check=True)
        elif f.startswith("launches_") and f.endswith("_step.csv"):
            cfg = f[len("launches_"):-len("_step.csv")]
            with open(os.path.join(DST, f"step_launches_{cfg}.json"), "w") as fh:
                json.dump(step_launches(p, cfg), fh, indent=1)
        elif f == "launches_bench_default.csv":
            shutil.copy(p, os.path.join(DST, f))
        elif f == "t_gpu_all.log":
            shutil.copy(p, os.path.join(DST, "gpu_tests.log"))
        elif f == "smoke.log":
            shutil.copy(p, os.path.join(DST, "smoke.log"))


if __name__ == "__main__":
    main()
