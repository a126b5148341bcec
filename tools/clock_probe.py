"""Run one prefill stage back-to-back for ~N seconds and sample SM clock / power during it."""
import argparse
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_10597_b200 as cl  # noqa: E402
from paper_2604_10597_b200.mamba1 import Prefill  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--stage", default="scan")
ap.add_argument("--seconds", type=float, default=3.0)
ap.add_argument("--config", default="C3")
args = ap.parse_args()
batch, dim, L, N, _ = bench.CONFIGS[args.config]
dev = torch.device("cuda", 0)
x = bench.make_inputs(torch, dev, batch, dim, L, N, 1)
out = torch.empty_like(x["u"])
pf = Prefill(cl.HistogramSpec(), device=dev)
uf = x["u"].reshape(-1)
pf.stage_minmax(uf)
pf.stage_histogram(uf)
pf.stage_decide(pf.n_samples(uf.numel()), L)


def run_once():
    if args.stage == "scan":
        pf.stage_scan(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"],
                      x["delta_bias"], True, out)
    elif args.stage == "hist":
        pf.stage_histogram(uf)
    else:
        pf.stage_minmax(uf)


for _ in range(3):
    run_once()
torch.cuda.synchronize()
lines = []
proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                         "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE,
                        text=True)
th = threading.Thread(target=lambda: [lines.append((time.time(), l.strip())) for l in proc.stdout],
                      daemon=True)
th.start()
time.sleep(0.5)
t0 = time.time()
n = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < args.seconds:
    for _ in range(20):
        run_once()
    n += 20
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
t1 = time.time()
proc.terminate()
ms = e0.elapsed_time(e1) / n
samp = [l for ts, l in lines if t0 + 0.2 <= ts <= t1]
clk = sorted(float(l.split(",")[0]) for l in samp)
pw = sorted(float(l.split(",")[1]) for l in samp)
reasons = sorted(set(l.split(",")[2].strip() for l in samp))
print(f"{args.stage}: {ms:.4f} ms/iter over {n} iters; SM clock median {clk[len(clk)//2]:.0f} MHz "
      f"(min {clk[0]:.0f}, max {clk[-1]:.0f}); power median {pw[len(pw)//2]:.0f} W max {pw[-1]:.0f} W; "
      f"reasons {reasons}")
