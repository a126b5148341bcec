"""GPU: repetition stress of the hand-rolled synchronisation (compute-sanitizer is closed on
this pool, see profiles/r2e_sanitizer.txt).  A race in a producer/consumer ring, the tagged
carry words, the aggregate words, the self-resetting work ticket or the histogram's arrival
ticket shows up as run-to-run differences or a hang; every path here must reproduce its
first run bit for bit, many times, including back-to-back launches of DIFFERENT kernels on
one stream (a ticket left dirty by one kernel would skip items of the next).  Run it with
CHUNKLAB_LIB=build/variants/checked.so (-DCL_DEVICE_CHECKS=1) to also trap on the device
invariants (ticket start/end values, tag monotonicity, item and store bounds)."""
import numpy as np
import pytest
import torch

import paper_2604_10597_b200 as cl
from paper_2604_10597_b200.mamba1 import Prefill, selective_scan_fn
from tests._helpers import mamba_inputs

pytestmark = pytest.mark.gpu

REPS = 25


def to_dev(x, cuda):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).to(cuda) for k, v in x.items()}


@pytest.mark.parametrize("shape", [(2, 48, 1024), (1, 1536, 2048), (4, 256, 512)])
def test_interleaved_kernels_reproduce(cuda, shape):
    batch, dim, L = shape
    x = to_dev(mamba_inputs(3, batch, dim, 16, L), cuda)
    args = (x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"], x["delta_bias"], True)
    plan = [("cfg:0", 32), ("lb:0", 512), ("cfg:11", 64), ("lookback", 64), ("cfg:13", 128),
            ("lb:3", 32), ("cfg:1", 256), ("chained", 2048), ("lb:5", 512)]
    first = {}
    for rep in range(REPS):
        for v, chunk in plan:
            y, h = selective_scan_fn(*args, return_last_state=True, chunk_size=chunk, variant=v)
            key = v
            if key not in first:
                first[key] = (y.clone(), h.clone())
            else:
                assert torch.equal(y, first[key][0]) and torch.equal(h, first[key][1]), (rep, v)
    torch.cuda.synchronize()


def test_prefill_fused_decision_reproduces(cuda):
    x = to_dev(mamba_inputs(4, 1, 512, 16, 2048), cuda)
    args = (x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"], x["delta_bias"], True)
    pfs = [Prefill(cl.HistogramSpec(), device=cuda),
           Prefill(cl.HistogramSpec(sample_stride=8), device=cuda)]
    ref = [(p(*args).out.clone(), p.counts.clone(), p.decision_buf.clone()) for p in pfs]
    for rep in range(REPS):
        for p, (y0, c0, d0) in zip(pfs, ref):
            res = p(*args)
            assert torch.equal(res.out, y0) and torch.equal(p.counts, c0), rep
            assert torch.equal(p.decision_buf, d0), rep


def test_token_entropy_reproduces(cuda):
    x = to_dev(mamba_inputs(5, 2, 256, 16, 512), cuda)
    args = (x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"], x["delta_bias"], True)
    pt = Prefill(cl.HistogramSpec(), cl.SchedulerPolicy(cl.TokenHistogramPolicy(), [128, 256, 512]),
                 cl.ChunkBounds(128, 512), device=cuda)
    y0 = pt(*args).out.clone()
    t0 = pt.token_buf.clone()
    for rep in range(REPS):
        assert torch.equal(pt(*args).out, y0) and torch.equal(pt.token_buf, t0), rep


def test_two_streams_concurrent_reproduce(cuda):
    """Two prefills in flight on two streams of one context, REPS times."""
    xa = to_dev(mamba_inputs(6, 1, 768, 16, 2048), cuda)
    xb = to_dev(mamba_inputs(7, 4, 1024, 16, 1024), cuda)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    pa, pb = Prefill(cl.HistogramSpec(), device=cuda), Prefill(cl.HistogramSpec(), device=cuda)
    ya = torch.empty_like(xa["u"])
    yb = torch.empty_like(xb["u"])

    def go():
        with torch.cuda.stream(sa):
            pa(xa["u"], xa["delta"], xa["A"], xa["B"], xa["C"], xa["D"], xa["z"],
               xa["delta_bias"], True, out=ya)
        with torch.cuda.stream(sb):
            pb(xb["u"], xb["delta"], xb["A"], xb["B"], xb["C"], xb["D"], xb["z"],
               xb["delta_bias"], True, out=yb)
        torch.cuda.synchronize()

    go()
    ra, rb = ya.clone(), yb.clone()
    for rep in range(REPS):
        ya.zero_()
        yb.zero_()
        go()
        assert torch.equal(ya, ra) and torch.equal(yb, rb), rep
