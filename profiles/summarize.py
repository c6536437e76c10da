"""Summarise an ncu --set full capture exported by run_prof.sh (raw page
CSV) into the numbers DESIGN.md and bench.py quote.

usage: python profiles/summarize.py gpurun_out/raw_<tag>.csv [--json out.json]
"""
import csv
import json
import sys

KEYS = [
    ("duration_us", "gpu__time_duration.sum", 1e-3),
    ("dram_read_bytes", "dram__bytes_read.sum", 1.0),
    ("dram_write_bytes", "dram__bytes_write.sum", 1.0),
    ("fp64_pipe_pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1.0),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    ("registers", "launch__registers_per_thread", 1.0),
    ("block", "launch__block_size", 1.0),
    ("grid", "launch__grid_size", 1.0),
    ("dyn_smem_bytes", "launch__shared_mem_per_block_dynamic", 1.0),
    ("inst_executed", "smsp__inst_executed.sum", 1.0),
]


def units(v):
    v = v.replace(",", "")
    try:
        return float(v)
    except ValueError:
        return None


def summarize(path):
    rows = list(csv.reader(open(path)))
    hdr, unit_row, data = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, data))
    u = dict(zip(hdr, unit_row))
    out = {"kernel": d.get("Kernel Name", "")}
    for name, key, scale in KEYS:
        if key in d and units(d[key]) is not None:
            val = units(d[key])
            unit = u.get(key, "")
            if key == "gpu__time_duration.sum":
                val *= {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
            else:
                base = unit.split("/")[0]
                val *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(base, 1.0)
            out[name] = val
    stalls = []
    for k in hdr:
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            v = units(d[k])
            if v:
                stalls.append((v, k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
    tot = sum(v for v, _ in stalls) or 1.0
    out["stall_top"] = {k: round(v / tot, 3) for v, k in sorted(stalls, reverse=True)[:8]}
    if "dram_read_bytes" in out and "dram_write_bytes" in out:
        out["dram_bytes"] = out["dram_read_bytes"] + out["dram_write_bytes"]
    # fp64 work of the launch: thread-level DFMA (2 flop), DMUL, DADD per
    # elapsed SMSP cycle summed over SMSPs, times the elapsed SM cycles
    fma = units(d.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed", ""))
    mul = units(d.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed", ""))
    add = units(d.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed", ""))
    cyc = units(d.get("sm__cycles_elapsed.avg", ""))
    peak = units(d.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum.peak_sustained", ""))
    if None not in (fma, mul, add, cyc):
        out["fp64_flop"] = (2.0 * fma + mul + add) * cyc
    if peak is not None:
        out["fp64_peak_flop_per_cycle"] = 2.0 * peak  # DFMA lanes x 2, whole GPU
    return out


if __name__ == "__main__":
    s = summarize(sys.argv[1])
    if "--json" in sys.argv:
        json.dump(s, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
    for k, v in s.items():
        print(f"{k:20s} {v}")
