"""Per-stage device times of token_entropy on a BASELINE config's u (C3 by default).

    python tools/profile_token.py [--config C3] [--reps 10]
"""
import argparse
import ctypes as C
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_10597_b200 as cl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    batch, dim, L, N, _ = bench.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    u = torch.randn(batch, dim, L, device=dev)
    ch = batch * dim
    ctx = cl.Context.get(0)
    spec = cl.HistogramSpec().to_c()
    k = spec.bin_count
    trange = torch.empty(2 * L + 1, dtype=torch.float64, device=dev)
    counts = torch.zeros(L * k, dtype=torch.int32, device=dev)
    out = torch.zeros(4, dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream(dev).cuda_stream
    stages = {
        "range_init": lambda: ctx.call("cl_token_range_init", trange.data_ptr(), L, s),
        "minmax": lambda: ctx.call("cl_token_minmax_f32", u.data_ptr(), ch, L, 0, 1,
                                   trange.data_ptr(), s),
        "zero": lambda: counts.zero_(),
        "histogram": lambda: ctx.call("cl_token_histogram_f32", u.data_ptr(), ch, L, 0,
                                      C.byref(spec), trange.data_ptr(), counts.data_ptr(), s),
        "entropy+finalize": lambda: ctx.call("cl_token_entropy_counts", counts.data_ptr(),
                                             trange.data_ptr(), L, ch, C.byref(spec),
                                             out.data_ptr(), s),
        "one_call": lambda: ctx.call("cl_token_entropy_f32", u.data_ptr(), ch, L, C.byref(spec),
                                     out.data_ptr(), s),
    }
    times = {k_: [] for k_ in stages}
    for _ in range(args.reps):
        for name, fn in stages.items():
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            times[name].append(a.elapsed_time(b))
    print({k_: round(statistics.median(v[1:]), 4) for k_, v in times.items()},
          "raw", float(out[0]))


if __name__ == "__main__":
    main()
