"""GPU: parity at BASELINE.json's full single-GPU size, C3 (B=8, L=8192, d_inner=4096, N=16).

The oracle restatement is C, so the entropy stage is checked against it directly on the
whole 268M-element tensor (a few seconds of CPU).  The scan is checked through
size-independent properties -- bitwise chunk invariance, per-row agreement with the fp64
oracle on sampled rows -- and the multi-GPU protocol through additivity of row shards
(MAX of ranges, SUM of counts) on one device."""
import ctypes as C
import math

import numpy as np
import pytest
import torch

import bench
import paper_2604_10597_b200 as cl
from paper_2604_10597_b200.mamba1 import Prefill, selective_scan_fn
from tests._helpers import assert_close_normwise

pytestmark = pytest.mark.gpu

B, D, L, N = bench.CONFIGS["C3"][:4]


@pytest.fixture(scope="module")
def c3(cuda):
    x = bench.make_inputs(torch, cuda, B, D, L, N, 1)
    yield x
    del x
    torch.cuda.empty_cache()


def test_c3_entropy_counts_and_decision_vs_oracle(cuda, c3, port):
    pf = Prefill(cl.HistogramSpec(), device=cuda)
    uf = c3["u"].reshape(-1)
    pf.stage_minmax(uf)
    pf.stage_histogram(uf)
    pf.stage_decide(pf.n_samples(uf.numel()), L)
    rec = pf.decision()
    counts = pf.counts.cpu().numpy().astype(np.uint64)
    ref_counts, lo, hi, n = port.histogram(uf.cpu().numpy(), 256, 1e-8, 1)
    assert n == B * D * L and int(counts.sum()) == n
    assert (counts == ref_counts).all()
    assert (rec.lo, rec.hi) == (lo, hi)
    raw, _ = port.entropy(ref_counts.astype(np.float64) * (1.0 / n))
    assert rec.entropy.raw_nats == pytest.approx(raw, rel=1e-13)
    chunk, _ = port.select_chunk(raw, 32, 512, math.log(256))
    assert rec.decision.chunk == chunk


@pytest.mark.parametrize("stride", [1, 8])
def test_c3_row_shards_are_additive(cuda, c3, stride):
    """Two row shards (the multi-GPU plan at world 2) with global offsets: MAX of their
    ranges and SUM of their counts equal the single-pass range and counts, bit for bit."""
    spec = cl.HistogramSpec(sample_stride=stride)
    uf = c3["u"].reshape(-1)
    full = Prefill(spec, device=cuda)
    full.stage_minmax(uf)
    full.stage_histogram(uf)
    half = uf.numel() // 2
    parts = [Prefill(spec, device=cuda) for _ in range(2)]
    for p, off in zip(parts, (0, half)):
        p.stage_minmax(uf[off:off + half], off)
    rng = torch.maximum(parts[0].range, parts[1].range)
    for p in parts:
        p.range.copy_(rng)
    for p, off in zip(parts, (0, half)):
        p.stage_histogram(uf[off:off + half], off)
    assert torch.equal(rng, full.range)
    assert torch.equal(parts[0].counts + parts[1].counts, full.counts)


def test_c3_scan_chunk_invariance_and_sampled_rows(cuda, c3, port):
    args = (c3["u"], c3["delta"], c3["A"], c3["B"], c3["C"], c3["D"], c3["z"], c3["delta_bias"],
            True)
    y512, h512 = selective_scan_fn(*args, return_last_state=True, chunk_size=512)
    y2048, h2048 = selective_scan_fn(*args, return_last_state=True, chunk_size=2048)
    assert torch.equal(y512, y2048) and torch.equal(h512, h2048)
    assert torch.isfinite(y512).all()
    # fp64 oracle on 48 rows spread over batches and channels
    rows = [(b, d) for b in (0, 3, 7) for d in (0, 1, 15, 16, 1023, 2048, 2049, 3000, 4080,
                                                4094, 4095, 511, 777, 1500, 2500, 3333)]
    xs = {k: v.cpu().numpy() for k, v in c3.items()}
    for b, d in rows:
        yr, hr = port.mamba1(xs["u"][b:b + 1, d:d + 1], xs["delta"][b:b + 1, d:d + 1],
                             xs["A"][d:d + 1], xs["B"][b:b + 1], xs["C"][b:b + 1],
                             xs["D"][d:d + 1], xs["z"][b:b + 1, d:d + 1],
                             xs["delta_bias"][d:d + 1], True)
        assert_close_normwise(y512[b, d].cpu().numpy()[None], yr, 1e-5, f"y[{b},{d}]")
        assert_close_normwise(h512[b, d].cpu().numpy()[None], hr, 1e-5, f"h[{b},{d}]")


def test_c3_producer_fusion_epilogue(cuda, c3):
    from paper_2604_10597_b200.mamba1 import causal_conv1d_fn
    g = torch.Generator(device=cuda)
    g.manual_seed(3)
    w = torch.randn(D, 4, generator=g, device=cuda).mul_(0.5)
    bias = torch.randn(D, generator=g, device=cuda).mul_(0.1)
    ctx = cl.Context.get(cuda.index)
    s = torch.cuda.current_stream(cuda).cuda_stream
    r = torch.zeros(4, dtype=torch.float64, device=cuda)
    ctx.call("cl_range_init", r.data_ptr(), s)
    u = causal_conv1d_fn(c3["u"], w, bias, "silu", None, r)
    r2 = torch.zeros(4, dtype=torch.float64, device=cuda)
    ctx.call("cl_range_init", r2.data_ptr(), s)
    ctx.call("cl_minmax_f32", u.data_ptr(), u.numel(), 0, 1, r2.data_ptr(), s)
    assert torch.equal(r, r2) and r[2].item() == 0.0
    del u
