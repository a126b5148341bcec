"""A/B scan kernel configurations on given shapes (device time, median of 15):
    python tools/cfg_ab.py 4x2048x4096,1x8192x4096 auto,cfg:6,cfg:12
Each call (B/C transpose + scan) is captured into a CUDA graph and replayed, so the
events time the device alone (an eager selective_scan_fn call on a few-row shape is
host-bound: ~0.07 ms of Python + ctypes + tensor-map encoding per call)."""
import sys, torch, statistics
sys.path.insert(0, '.')
from paper_2604_10597_b200.mamba1 import selective_scan_fn
from tests._helpers import mamba_inputs
import numpy as np
shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1].split(",")] if len(sys.argv) > 1 else [(4, 2048, 4096)]
cfgs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["auto"]
l2buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for (b, d, L) in shapes:
    x = mamba_inputs(1, b, d, 16, L)
    t = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in x.items() if v is not None}
    res = []
    for cfg in cfgs:
        call = lambda: selective_scan_fn(t["u"], t["delta"], t["A"], t["B"], t["C"], t["D"], t["z"], t["delta_bias"], True, True, chunk_size=512, variant=cfg)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            call()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            call()
        f = g.replay
        f(); torch.cuda.synchronize()
        ts = []
        for _ in range(15):
            l2buf.zero_()  # L2 flushed before every timed replay (as bench.py does)
            a, e = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record(); f(); e.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(e))
        res.append(f"{cfg}={statistics.median(ts):.4f}")
    print((b, d, L), "tiles", b * d // 16, " ".join(res), flush=True)
