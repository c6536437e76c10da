"""Summarise an ncu `--page source --csv --print-source cuda,sass` export:
warp-level instructions executed per opcode and per source line, and
stall samples per source line (profiling aid, not product code)."""
import csv
import re
import sys
from collections import Counter, defaultdict


def main(path, top=40):
    op = Counter()
    line_inst = Counter()
    line_samp = Counter()
    line_src = {}
    fname = "?"
    cur = None
    total = 0
    with open(path) as f:
        for row in csv.reader(f):
            if not row:
                continue
            if row[0] == "File Path":
                fname = row[1].split("/")[-1]
                continue
            if row[0] in ("Function Name", "Line No"):
                continue
            if row[0]:
                cur = (fname, int(row[0]))
                line_src[cur] = row[1].strip()[:90]
                try:
                    line_samp[cur] += int(row[4])
                except ValueError:
                    pass
                continue
            if row[2] in ("...", "-") or cur is None:
                continue
            try:
                n = int(row[7])
            except ValueError:
                continue
            m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", row[3])
            if not m:
                continue
            op[m.group(2)] += n
            line_inst[cur] += n
            total += n
    print(f"total warp instructions {total}")
    for k, v in op.most_common(top):
        print(f"{k:10s} {v:12d} {v / total:6.1%}")
    print("--- per source line (inst, stall samples)")
    for k, v in line_inst.most_common(top):
        print(f"{k[0]}:{k[1]:<5d} {v:11d} {v / total:6.1%} samp {line_samp[k]:6d}  {line_src[k]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
