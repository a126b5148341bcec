"""DRAM traffic of the dominant kernel (the scan) for bench.py's roofline.traffic, keyed to
the library build it was measured on.

On a GPU box:
    python tools/scan_traffic.py --run C3 > gpurun_out/plain.log &&
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none -k regex:"rowpair_ws|lookback_ws" -c 1 --csv \
        --log-file gpurun_out/traffic_C3.csv python tools/scan_traffic.py --run C3
Here (or there):
    python tools/scan_traffic.py --record gpurun_out/traffic_C3.csv C3
appends / replaces the record {config, kernel, kernel_family, lib_sha256, dram bytes} in
profiles/scan_traffic.json.  lib_sha256 is the build fingerprint (sha256 of the library's
sources, headers and nvcc flags: paper_2604_10597_b200.build.fingerprint -- nvcc's output
bytes differ from build to build).  bench.py uses a record only when config, kernel family
and the fingerprint all match (else traffic = null).
"""
import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "profiles", "scan_traffic.json")


def run(config):
    import torch
    import bench
    import paper_2604_10597_b200 as cl
    from paper_2604_10597_b200.mamba1 import Prefill
    batch, dim, L, N, _ = bench.CONFIGS[config]
    dev = torch.device("cuda", 0)
    x = bench.make_inputs(torch, dev, batch, dim, L, N, 1234)
    out = torch.empty_like(x["u"])
    pf = Prefill(cl.HistogramSpec(), None, cl.ChunkBounds(32, 512), device=dev)
    pf(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"], x["delta_bias"], True,
       out=out, return_last_state=True)
    torch.cuda.synchronize()
    print("chunk", pf.decision().decision.chunk)


def record(csv_path, config):
    import bench
    rows = [r for r in csv.reader(open(csv_path)) if r]
    hdr = next(r for r in rows if "Metric Name" in r)
    vals, name = {}, None
    for r in rows[rows.index(hdr) + 1:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3,
                 "ms": 1e6}.get(unit, 1)
        vals[d["Metric Name"]] = v * scale
    batch, dim, L, N, _ = bench.CONFIGS[config]
    rec = {
        "config": config,
        "kernel": name[:120],
        "kernel_family": "lookback_ws_kernel" if "lookback" in name else "rowpair_ws_kernel",
        "lib_sha256": bench.library_sha256(),
        "dram_read_bytes": vals.get("dram__bytes_read.sum"),
        "dram_write_bytes": vals.get("dram__bytes_write.sum"),
        "dram_bytes_per_launch": vals.get("dram__bytes_read.sum", 0) +
                                 vals.get("dram__bytes_write.sum", 0),
        "duration_ns_under_ncu": vals.get("gpu__time_duration.sum"),
        "algorithmic_bytes_per_launch": bench.algorithmic_bytes(batch, dim, L, N)["scan"],
        "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (tools/scan_traffic.py)",
    }
    recs = []
    if os.path.exists(OUT):
        old = json.load(open(OUT))
        recs = old if isinstance(old, list) else []
    recs = [r for r in recs if r.get("config") != config] + [rec]
    json.dump(recs, open(OUT, "w"), indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--run")
    ap.add_argument("--record", nargs=2, metavar=("CSV", "CONFIG"))
    a = ap.parse_args()
    if a.run:
        run(a.run)
    if a.record:
        record(*a.record)
