"""BASELINE.json configs[1] and [4] on the B200 kernels (device time, CUDA events).

  python tools/chunk_sweep.py sweep [--config C2]   # configs[1]: static chunk 64..2048 vs the rule
  python tools/chunk_sweep.py mix                   # configs[4]: serving mix, L = 512..32768

sweep: scan time per static chunk (the paper's static-oracle sweep), the chunk the calibrated
       rule picks, and the full prefill (entropy + decision + scan) with the rule vs with the
       best static chunk (Static policy: no entropy pass).
mix:   one prefill per sequence length of the mix under three policies -- the
       sequence-length-keyed table, Guarded{FullHistogram, safe 512}, Static-512 -- total time.
Prints one JSON object.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_10597_b200 as cl  # noqa: E402
from paper_2604_10597_b200.mamba1 import Prefill, selective_scan_fn  # noqa: E402

BUCKETS = [64, 128, 256, 512, 1024, 2048]


_L2BUF = []


def flush_l2():
    """Write 256 MB (twice the 126 MB L2) so no rep reads the previous rep's lines."""
    if not _L2BUF:
        _L2BUF.append(torch.empty(256 << 20, dtype=torch.uint8, device="cuda"))
    _L2BUF[0].zero_()


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        flush_l2()  # outside the events
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


def args_of(x):
    return (x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"], x["delta_bias"], True)


def sweep(cfg, reps, variant="auto"):
    batch, dim, L, N, desc = bench.CONFIGS[cfg]
    dev = torch.device("cuda", 0)
    x = bench.make_inputs(torch, dev, batch, dim, L, N, 1)
    out = torch.empty_like(x["u"])
    scan_ms = {}
    for c in BUCKETS:
        scan_ms[c] = timed(lambda: selective_scan_fn(*args_of(x), chunk_size=c, out=out,
                                                     variant=variant), reps)
    best = min(scan_ms, key=scan_ms.get)
    bounds, cal = cl.ChunkBounds(64, 2048), cl.CalibrationRef.log_k(256)
    rule_pol = cl.SchedulerPolicy(cl.FullHistogramPolicy(), BUCKETS)
    pf_rule = Prefill(cl.HistogramSpec(), rule_pol, bounds, cal)
    pf_rule.scan_variant = variant
    rule_ms = timed(lambda: pf_rule(*args_of(x), out=out), reps)
    rule_chunk = pf_rule.decision().decision.chunk
    pf_static = Prefill(cl.HistogramSpec(), cl.SchedulerPolicy(cl.StaticPolicy(best), BUCKETS),
                        bounds, cal)
    pf_static.scan_variant = variant
    static_ms = timed(lambda: pf_static(*args_of(x), out=out), reps)
    return {"mode": "sweep", "config": f"{cfg}: {desc}", "scan_variant": variant,
            "scan_ms_by_chunk": scan_ms,
            "static_oracle_chunk": best, "rule_chunk": rule_chunk,
            "prefill_ms_rule": rule_ms, "prefill_ms_static_oracle": static_ms,
            "rule_vs_oracle": rule_ms / static_ms}


def mix(reps, variant="auto"):
    dev = torch.device("cuda", 0)
    dim, N = 2048, 16
    lengths = [512, 2048, 8192, 32768]
    bounds, cal = cl.ChunkBounds(64, 2048), cl.CalibrationRef.log_k(256)
    policies = {
        "seq_len_table": cl.SchedulerPolicy(cl.LearnedTablePolicy(4096, 256, 1024), BUCKETS),
        "guarded_entropy": cl.SchedulerPolicy(
            cl.GuardedPolicy(cl.SchedulerPolicy(cl.FullHistogramPolicy(), BUCKETS), 512, 2),
            BUCKETS),
        "static512": cl.SchedulerPolicy(cl.StaticPolicy(512), BUCKETS),
    }
    inputs = {L: bench.make_inputs(torch, dev, 1, dim, L, N, L) for L in lengths}
    res = {}
    for name, pol in policies.items():
        pf = Prefill(cl.HistogramSpec(), pol, bounds, cal)
        pf.scan_variant = variant
        per_len, chunks = {}, {}
        for L in lengths:
            x = inputs[L]
            out = torch.empty_like(x["u"])
            per_len[L] = timed(lambda: pf(*args_of(x), out=out), reps)
            chunks[L] = pf.decision().decision.chunk
        res[name] = {"total_ms": sum(per_len.values()), "ms_by_len": per_len, "chunk_by_len": chunks}
    return {"mode": "mix", "scan_variant": variant,
            "workload": f"B=1 d_inner={dim} N={N}, one prefill per L in {lengths}",
            "policies": res}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["sweep", "mix"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--variant", default="auto",
                    help="scan kernel family: auto (by shape) or chained (the chunk is the "
                         "scan's segment length on every shape)")
    a = ap.parse_args()
    print(json.dumps(sweep(a.config, a.reps, a.variant) if a.mode == "sweep"
                     else mix(a.reps, a.variant)))


if __name__ == "__main__":
    main()
