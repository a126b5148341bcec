"""Run each prefill stage on a BASELINE config a few times (for ncu / timing).

    python tools/profile_stages.py [--config C3] [--reps 2] [--variant auto]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_10597_b200 as cl  # noqa: E402
from paper_2604_10597_b200.mamba1 import Prefill  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--variant", default="auto")
    ap.add_argument("--median", action="store_true")
    ap.add_argument("--chunk", type=int, default=0, help="fixed chunk (0 = device rule)")
    ap.add_argument("--no-softplus", action="store_true")
    ap.add_argument("--no-z", action="store_true")
    args = ap.parse_args()
    batch, dim, L, N, _ = bench.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    x = bench.make_inputs(torch, dev, batch, dim, L, N, 1)
    out = torch.empty_like(x["u"])
    pf = Prefill(cl.HistogramSpec(), device=dev)
    uf = x["u"].reshape(-1)
    times = {"minmax": [], "hist": [], "decide": [], "scan": []}
    for _ in range(args.reps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record()
        pf.stage_minmax(uf)
        ev[1].record()
        pf.stage_histogram(uf)
        ev[2].record()
        pf.stage_decide(pf.n_samples(uf.numel()), L)
        ev[3].record()
        sp = not args.no_softplus
        zz = None if args.no_z else x["z"]
        if args.chunk or args.no_softplus or args.no_z:
            from paper_2604_10597_b200.mamba1 import selective_scan_fn
            selective_scan_fn(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], zz,
                              x["delta_bias"], sp, False, args.chunk or 512,
                              variant=args.variant, out=out)
        else:
            pf.stage_scan(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"],
                          x["delta_bias"], True, out, False, variant=args.variant)
        ev[4].record()
        torch.cuda.synchronize()
        for i, k in enumerate(times):
            times[k].append(ev[i].elapsed_time(ev[i + 1]))
    if args.median:
        import statistics
        print(f"cfg={os.environ.get('CL_SCAN_CFG', 'default')} chunk={args.chunk} "
              + " ".join(f"{k}={statistics.median(v[1:]):.4f}" for k, v in times.items()))
    else:
        print({k: [round(t, 4) for t in v] for k, v in times.items()})
    print("decision", pf.decision().decision)


if __name__ == "__main__":
    main()
