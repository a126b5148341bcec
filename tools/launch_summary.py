"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv --log-file X`).

    python tools/launch_summary.py gpurun_out/launches.csv "<command line>" > profiles/rN_launches.txt

Prints, per kernel name, the mean per-launch duration and its share of the per-step sum of
this library's kernels (namespace cl::), then the torch kernels (input generation,
outside the timed region).  ncu times are cold-cache and serialised: compare shares.
"""
import collections
import csv
import sys


def main(path, cmd):
    hdr, data = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        v = float(d["Metric Value"].replace(",", "")) / 1e3  # ns -> us
        agg.setdefault(d["Kernel Name"], []).append(v)
    ours = {k: v for k, v in agg.items() if "cl::" in k}
    step = sum(sum(v) / len(v) for v in ours.values())
    print(f"# ncu launch list: `ncu --metrics gpu__time_duration.sum --clock-control none {cmd}`")
    print("# (cold-cache, serialised per-launch times; compare SHARES of the step, not absolutes)")
    print(f"# per-step sum of our kernels (mean over launches): {step:.1f} us")
    for k, v in ours.items():
        m = sum(v) / len(v)
        print(f"  {m:9.1f} us  {100 * m / step:5.1f}%  n={len(v):2d}  {k[:110]}")
    print("# torch kernels (input generation, outside the timed region):")
    for k, v in agg.items():
        if k not in ours:
            print(f"  {sum(v) / len(v):9.1f} us  n={len(v):2d}  {k[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
