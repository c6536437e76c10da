"""Turn the exports of profiles/capture_all.sh (gpurun_out/) into the
committed per-round summaries under profiles/ and profiles/traffic.json
(the per-launch DRAM bytes and fp64 flop that bench.py reports).

usage: python profiles/make_profiles.py r1
"""
import csv
import json
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from summarize import summarize  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "gpurun_out")


def launch_means(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[i]
    kn, mv = h.index("Kernel Name"), h.index("Metric Value")
    t = {}
    for r in rows[i + 1:]:
        if len(r) > mv:
            t.setdefault(r[kn].split("(")[0], []).append(float(r[mv].replace(",", "")) / 1e3)
    return {k: {"n": len(v), "mean_us": sum(v) / len(v)} for k, v in t.items()}


def main(r, workloads=None):
    try:
        traffic = json.load(open(os.path.join(HERE, "traffic.json")))
    except (OSError, ValueError):
        traffic = {}
    for w in workloads or ["config1", "config2_p1", "config2_p2", "config2_p3", "config2_p4",
                           "config1_seams"]:
        tag = f"{r}_{w}"
        raw = os.path.join(OUT, f"raw_{tag}.csv")
        if not os.path.exists(raw):
            print("missing", raw)
            continue
        s = summarize(raw)
        # r2b / r2c captures live with the round's other files in profiles/r2/
        rd = r if os.path.isdir(os.path.join(HERE, r)) else r[:2]
        dst = os.path.join(HERE, rd) if os.path.isdir(os.path.join(HERE, rd)) else HERE
        with open(os.path.join(dst, f"{tag}_ncu_summary.json"), "w") as f:
            json.dump(s, f, indent=1)
        det = os.path.join(OUT, f"details_{tag}.txt")
        if os.path.exists(det):
            shutil.copy(det, os.path.join(dst, f"{tag}_ncu_details.txt"))
        lc = os.path.join(OUT, f"launches_{tag}.csv")
        if os.path.exists(lc):
            shutil.copy(lc, os.path.join(dst, f"{tag}_launches.csv"))
            with open(os.path.join(dst, f"{tag}_launches_summary.json"), "w") as f:
                json.dump(launch_means(lc), f, indent=1)
        if not w.endswith("_seams"):
            traffic[w] = {k: s[k] for k in ("kernel", "dram_bytes", "duration_us", "fp64_pipe_pct",
                                            "issue_active_pct", "fp64_flop",
                                            "fp64_peak_flop_per_cycle") if k in s}
            rel = os.path.relpath(dst, os.path.dirname(HERE))
            traffic[w]["source"] = (f"{rel}/{tag}_ncu_summary.json (ncu --set full "
                                    f"--clock-control none, one launch)")
        print(tag, {k: s.get(k) for k in ("kernel", "duration_us", "dram_bytes", "fp64_pipe_pct")})
    with open(os.path.join(HERE, "traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1", sys.argv[2:] or None)
