"""Per-source-line stall-reason breakdown from an ncu `--page source --csv
--print-source cuda,sass` export (profiling aid): for the lines with the most
stall samples, the samples by reason."""
import csv
import sys
from collections import Counter, defaultdict


def main(path, top=30):
    hdr = None
    fname = "?"
    per = defaultdict(Counter)
    src = {}
    tot = Counter()
    with open(path) as f:
        for row in csv.reader(f):
            if not row:
                continue
            if row[0] == "File Path":
                fname = row[1].split("/")[-1]
                continue
            if row[0] == "Line No":
                hdr = row
                cols = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
                continue
            if row[0] in ("Function Name",) or hdr is None or not row[0]:
                continue
            key = (fname, int(row[0]))
            src[key] = row[1].strip()[:70]
            for i, name in cols:
                try:
                    v = int(row[i])
                except ValueError:
                    continue
                per[key][name] += v
                tot[name] += v
    n = sum(tot.values())
    print("total samples", n, {k: round(v / n, 3) for k, v in tot.most_common(9)})
    for key, c in sorted(per.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
        s = sum(c.values())
        print(f"{key[0]}:{key[1]:<4d} {s:6d} {s / n:5.1%} " +
              " ".join(f"{k}={v}" for k, v in c.most_common(4)) + "  | " + src[key])


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
