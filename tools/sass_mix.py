"""Per-opcode instruction and stall-sample mix of one kernel from an .ncu-rep source page.

    python tools/sass_mix.py <rep> <kernel-regex> [top]
"""
import csv
import subprocess
import sys
from collections import Counter


def main(rep, kern, top=25):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", "regex:" + kern], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    data = []
    for r in rows:
        if len(r) > 6 and r[0].startswith("0x"):
            data.append(r)
        elif "Instructions Executed" in r:
            hdr = r
    ie, src, smp = hdr.index("Instructions Executed"), hdr.index("Source"), \
        hdr.index("Warp Stall Sampling (All Samples)")
    data = [(r[0], r[src].strip(), int(r[ie] or 0), int(r[smp] or 0)) for r in data]
    tot = sum(d[2] for d in data)
    ts = sum(d[3] for d in data) or 1
    print(f"total instructions {tot}, stall samples {ts}")
    c, s = Counter(), Counter()
    for _, t, n, m in data:
        toks = t.split()
        op = toks[1] if toks[0].startswith("@") else toks[0]
        c[op.split(".")[0]] += n
        s[op.split(".")[0]] += m
    for k, v in c.most_common(top):
        print(f"{k:12s} {v:12d} {v / tot * 100:5.1f}%  samples {s[k] / ts * 100:5.1f}%")
    print("--- hottest by stall samples")
    for a, t, n, m in sorted(data, key=lambda d: -d[3])[:top]:
        print(a[-5:], f"{t[:64]:64s}", n, m)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
