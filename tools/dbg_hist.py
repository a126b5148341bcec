import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2604_10597_b200 as cl
from paper_2604_10597_b200.mamba1 import Prefill
from oracle import oracle as O
port = O.Port()
v = port.generate(O.DIST_UNIFORM, 10**6, 8).astype(np.float32)
dev = torch.device('cuda', 0)
t = torch.from_numpy(v).to(dev)
oc, lo, hi, n = port.histogram(v, 256)
bad = 0
for rep in range(30):
    pf = Prefill(cl.HistogramSpec(), device=dev)
    pf.stage_minmax(t); pf.stage_histogram(t); torch.cuda.synchronize()
    d = pf.counts.cpu().numpy() - oc.astype(np.int64)
    bad += int(np.abs(d).sum() != 0)
print(os.environ.get("CHUNKLAB_LIB", "default"), "runs with wrong counts:", bad, "/ 30")
