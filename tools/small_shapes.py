"""Few-row prefill timing: eager launches vs CUDA-graph replay, and the host's own
enqueue time per step (a step whose host submission is slower than its device work is
host-bound, whatever the kernels do).

    python tools/small_shapes.py [C1,C2] [auto,chained]

Per config and scan variant: eager step (per-step CUDA events, L2 flushed between
steps), graph step (the same step captured once, replayed; events around each replay),
host enqueue (perf_counter around the eager step's launch calls, no sync), and the
per-stage device times inside the graph (events captured into it)."""
import json
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2604_10597_b200 as cl  # noqa: E402
from paper_2604_10597_b200.mamba1 import Prefill  # noqa: E402

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C1", "C2"]
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["auto", "chained"]
dev = torch.device("cuda", 0)
l2buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
out_rows = []
for cfg in cfgs:
    batch, dim, L, N, _ = bench.CONFIGS[cfg]
    x = bench.make_inputs(torch, dev, batch, dim, L, N, 1234)
    out = torch.empty_like(x["u"])
    h_last = torch.empty(batch, dim, N, device=dev)
    uf = x["u"].reshape(-1)
    for variant in variants:
        pf = Prefill(cl.HistogramSpec(), None, cl.ChunkBounds(32, 512), device=dev)

        def step():
            pf.stage_minmax(uf)
            pf.stage_histogram_decide(uf, L)
            pf.stage_scan(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"],
                          x["delta_bias"], True, out, True, variant=variant)

        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(5):
                step()
            torch.cuda.synchronize()
            # eager, L2 flushed between steps, per-step events
            eager = []
            host = []
            for _ in range(30):
                l2buf.zero_()
                a, b = torch.cuda.Event(True), torch.cuda.Event(True)
                a.record()
                t0 = time.perf_counter()
                step()
                host.append((time.perf_counter() - t0) * 1e3)
                b.record()
                torch.cuda.synchronize()
                eager.append(a.elapsed_time(b))
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        graph = []
        for _ in range(30):
            l2buf.zero_()
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            graph.append(a.elapsed_time(b))
        row = {"config": cfg, "variant": variant,
               "eager_ms": statistics.median(eager), "graph_ms": statistics.median(graph),
               "host_enqueue_ms": statistics.median(host), "chunk": pf.decision().decision.chunk}
        print(json.dumps(row), flush=True)
        out_rows.append(row)
