"""Small-shape driver for compute-sanitizer (memcheck / racecheck / synccheck), one tool per run:

    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py

Exercises every hand-rolled synchronisation of the library on shapes small enough for the
tools: the chained warp-specialised scan (rowpair_ws_kernel: mbarrier rings, producer /
consumer hand-off, tagged carry words, self-resetting ticket) with >= 2 segments per tile,
the L-parallel scan (lookback_ws_kernel: aggregate words, in-order fold), the row kernel,
the register-fed histogram with its arrival-ticket decision (hist_f32_reg_kernel<1>), the
TMA-ring histogram (strided / fixed range), the token-entropy kernels, the fused conv1d
producer, the fp64 scan and the decode step.  Exits 0 after checking a few results (the
sanitizer's own report is the evidence)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_10597_b200 as cl  # noqa: E402
from paper_2604_10597_b200.mamba1 import (Prefill, causal_conv1d_fn, selective_scan_fn,  # noqa: E402
                                          selective_state_update)
from tests._helpers import mamba_inputs  # noqa: E402

dev = torch.device("cuda", 0)


def t(x):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in x.items()}


x = t(mamba_inputs(1, 2, 48, 16, 512))
args = (x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"], x["delta_bias"], True)
# chained kernels: several configurations, 8 segments per tile, h0
h0 = torch.randn(2, 48, 16, device=dev)
y_ref, _ = selective_scan_fn(*args, return_last_state=True, chunk_size=64, variant="cfg:0", h0=h0)
for v in ("cfg:11", "cfg:12", "cfg:1"):
    y, _ = selective_scan_fn(*args, return_last_state=True, chunk_size=64, variant=v, h0=h0)
    assert torch.equal(y, y_ref), v
# the L-parallel kernel (every table row), 16 segments
for r in range(6):
    selective_scan_fn(*args, return_last_state=True, variant=f"lb:{r}", h0=h0)
# prefill: min/max + register-fed histogram whose last CTA decides + scan
pf = Prefill(cl.HistogramSpec(), device=dev)
res = pf(*args, return_last_state=True)
print("prefill chunk", res.decision().decision.chunk)
# TMA-ring histogram paths (stride 8, fixed range) + separate decide
for spec in (cl.HistogramSpec(sample_stride=8),
             cl.HistogramSpec(range_mode=cl.RangeMode.Fixed, fixed_lo=-2.0, fixed_hi=2.0)):
    p2 = Prefill(spec, device=dev)
    p2(*args)
    p2.decision()
# token entropy (TokenHistogram policy)
pt = Prefill(cl.HistogramSpec(), cl.SchedulerPolicy(cl.TokenHistogramPolicy(), [128, 256, 512]),
             cl.ChunkBounds(128, 512), device=dev)
pt(*args)
print("token chunk", pt.decision().decision.chunk)
# producer fusion
w = torch.randn(48, 4, device=dev)
u2 = causal_conv1d_fn(x["u"], w, None, "silu")
pf.from_conv(x["u"], w, None, x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"], x["delta_bias"])
# decode step
st = torch.randn(2, 48, 16, device=dev)
selective_state_update(st, x["u"][..., 0].contiguous(), x["delta"][..., 0].contiguous(), x["A"],
                       x["B"][..., 0].contiguous(), x["C"][..., 0].contiguous(), x["D"],
                       x["z"][..., 0].contiguous(), x["delta_bias"], True)
# fp64 reference-mode scan through the host path
p = cl.random_scan_params(3, 8, 4, 100, True) if hasattr(cl, "random_scan_params") else None
if p is not None:
    cl.scan_chunked(p, cl.ScanState(), 7)
torch.cuda.synchronize()
print("sanitize smoke done")
