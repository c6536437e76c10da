"""Static dependency distances of the fp64 instructions of a SASS listing
(cuobjdump -sass -fun <kernel>): for every DFMA / DMUL / DADD, the number of
instructions back to the nearest producer of one of its source registers.
Short distances are issue stalls that only other warps can fill."""
import collections
import re
import sys


def main(path):
    ins = []
    for line in open(path):
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", line)
        if m:
            ins.append(m.group(2).strip())
    fp = ("DFMA", "DMUL", "DADD")
    nowrite = ("STS", "STG", "BRA", "BAR", "ISETP", "DSETP", "STL", "EXIT", "BSSY", "BSYNC",
               "LDGSTS", "ATOMS", "RED", "FSETP", "PLOP3", "WARPSYNC", "MEMBAR", "NOP")
    last = {}
    dist = []
    for i, t in enumerate(ins):
        t2 = re.sub(r"^@!?U?P\d+\s+", "", t)
        op = t2.split()[0]
        regs = re.findall(r"\bR(\d+)\b", t2)
        if not regs:
            continue
        base = op.split(".")[0]
        if base in fp:
            d = 10 ** 9
            for s in regs[1:]:
                for r in (int(s), int(s) + 1):
                    if r in last:
                        d = min(d, i - last[r])
            dist.append(d)
        if base in nowrite:
            continue
        wide = base in fp or "WIDE" in op or ".64" in op or ".128" in op
        for r in ([int(regs[0]), int(regs[0]) + 1] if wide else [int(regs[0])]):
            last[r] = i
    c = collections.Counter(min(d, 12) for d in dist)
    tot = sum(c.values())
    print(len(ins), "instructions,", tot, "fp64")
    acc = 0
    for k in sorted(c):
        acc += c[k]
        print(f"{'>=12' if k == 12 else k:>4} {c[k]:5d} {c[k] / tot:6.1%}  cum {acc / tot:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
