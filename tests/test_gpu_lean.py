"""GPU: the lean entropy kernels (cl_entropy_lean_f32: one CTA per SM, 4 warps, <= 64
registers, ~66 KB of shared memory, cp.async.bulk rings) that let call i+1's entropy run on
the SMs of call i's scan.  Counts, range and the decision record must equal the regular
stages' (cl_prefill_init + cl_minmax_f32 + cl_histogram_decide_f32) bit for bit, alone and
while a scan runs on another stream."""
import numpy as np
import pytest
import torch

import paper_2604_10597_b200 as cl
from paper_2604_10597_b200.mamba1 import Prefill
from tests._helpers import mamba_inputs

pytestmark = pytest.mark.gpu


def regular(pf, uf, L):
    pf.stage_init()
    pf.stage_minmax(uf, init=False)
    pf.stage_histogram_decide(uf, L, zero=False)


@pytest.mark.parametrize("n,offset,dist", [(1 << 20, 0, "normal"), (3 * 1536 * 2048 + 4321, 3, "normal"),
                                           (16 << 20, 1, "laplace"), (9000, 0, "uniform"),
                                           (5000, 2, "normal")])
def test_lean_equals_regular(cuda, n, offset, dist):
    rng = np.random.default_rng(n % 1000)
    v = {"normal": rng.standard_normal, "uniform": rng.random,
         "laplace": lambda m: rng.laplace(size=m)}[dist](n + offset).astype(np.float32)
    buf = torch.from_numpy(v).to(cuda)
    uf = buf[offset:]  # offset elements: an unaligned start exercises the head path
    a, b = Prefill(cl.HistogramSpec(), device=cuda), Prefill(cl.HistogramSpec(), device=cuda)
    regular(a, uf, 2048)
    b.stage_entropy_lean(uf, 2048)
    torch.cuda.synchronize()
    assert torch.equal(a.counts, b.counts)
    assert torch.equal(a.range, b.range)
    assert torch.equal(a.decision_buf, b.decision_buf)
    assert int(a.counts.sum()) == n


def test_lean_falls_back_for_other_configs(cuda):
    v = torch.randn(1 << 20, device=cuda)
    for spec in (cl.HistogramSpec(sample_stride=8),
                 cl.HistogramSpec(range_mode=cl.RangeMode.Fixed, fixed_lo=-1.0, fixed_hi=1.0),
                 cl.HistogramSpec(bin_count=512)):
        a, b = Prefill(spec, device=cuda), Prefill(spec, device=cuda)
        regular(a, v, 512)
        b.stage_entropy_lean(v, 512)
        torch.cuda.synchronize()
        assert torch.equal(a.counts, b.counts) and torch.equal(a.decision_buf, b.decision_buf)


def test_lean_under_a_running_scan(cuda):
    """Entropy of batch B (lean, stream 2) while batch A's scan runs (stream 1), repeated:
    both results equal their serial values."""
    xa = {k: torch.from_numpy(np.ascontiguousarray(v)).to(cuda)
          for k, v in mamba_inputs(9, 4, 1024, 16, 2048).items()}
    ub = torch.randn(4 * 1024 * 2048, device=cuda)
    pa = Prefill(cl.HistogramSpec(), device=cuda)
    ya = pa(xa["u"], xa["delta"], xa["A"], xa["B"], xa["C"], xa["D"], xa["z"], xa["delta_bias"],
            True).out.clone()
    pref = Prefill(cl.HistogramSpec(), device=cuda)
    regular(pref, ub, 2048)
    pb = Prefill(cl.HistogramSpec(), device=cuda)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = torch.empty_like(ya)
    torch.cuda.synchronize()
    for _ in range(5):
        with torch.cuda.stream(s1):
            pa.stage_scan(xa["u"], xa["delta"], xa["A"], xa["B"], xa["C"], xa["D"], xa["z"],
                          xa["delta_bias"], True, out)
        with torch.cuda.stream(s2):
            pb.stage_entropy_lean(ub, 2048)
        torch.cuda.synchronize()
        assert torch.equal(out, ya)
        assert torch.equal(pb.counts, pref.counts) and torch.equal(pb.decision_buf, pref.decision_buf)
