"""C3: standalone device time of the lean entropy stages, the regular ones and the scan, and
the overlap of lean entropy (stream 2) with a scan (stream 1) -- does the entropy of call i+1
actually run under call i's scan?"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2604_10597_b200 as cl  # noqa: E402
from paper_2604_10597_b200.mamba1 import Prefill  # noqa: E402

dev = torch.device("cuda", 0)
B, D, L, N, _ = bench.CONFIGS["C3"]
x = bench.make_inputs(torch, dev, B, D, L, N, 1)
u2 = torch.randn(B * D * L, device=dev)
out = torch.empty_like(x["u"])
pa, pb = Prefill(cl.HistogramSpec(), device=dev), Prefill(cl.HistogramSpec(), device=dev)
uf = x["u"].reshape(-1)


def timed(fn, reps=5, stream=None):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(e))
    return statistics.median(ts)


def regular():
    pb.stage_init()
    pb.stage_minmax(u2, init=False)
    pb.stage_histogram_decide(u2, L, zero=False)


pa(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"], x["delta_bias"], True, out=out)
scan = lambda: pa.stage_scan(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"],  # noqa: E731
                             x["delta_bias"], True, out)
lean = lambda: pb.stage_entropy_lean(u2, L)  # noqa: E731
print("scan", timed(scan), "lean entropy", timed(lean), "regular entropy", timed(regular))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both(first_lean):
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    if first_lean:
        with torch.cuda.stream(s2):
            lean()
        with torch.cuda.stream(s1):
            scan()
    else:
        with torch.cuda.stream(s1):
            scan()
        with torch.cuda.stream(s2):
            lean()
    cur.wait_stream(s1)
    cur.wait_stream(s2)


print("scan || lean (lean enqueued first)", timed(lambda: both(True)))
print("scan || lean (scan enqueued first)", timed(lambda: both(False)))
