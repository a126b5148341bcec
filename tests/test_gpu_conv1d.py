"""GPU: producer fusion -- causal depthwise conv1d + SiLU emitting u
with the entropy stage-1 (min/max + finite check) folded into its epilogue.

The conv itself is parity-unpinned (the reference has no convolution): it is checked
against the fp64 restatement oracle.causal_conv1d_f64.  The fused epilogue must equal
cl_minmax_f32 over the same u bit for bit, so the fused prefill's decision is
identical to the unfused one."""
import numpy as np
import pytest
import torch

import paper_2604_10597_b200 as cl
from oracle.oracle import causal_conv1d_f64
from paper_2604_10597_b200.mamba1 import Prefill, causal_conv1d_fn
from tests._helpers import assert_close_normwise, mamba_inputs

pytestmark = pytest.mark.gpu


def t(a, cuda):
    return torch.from_numpy(np.ascontiguousarray(a)).to(cuda)


def conv_inputs(seed, batch, dim, L, width):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((batch, dim, L)).astype(np.float32)
    w = (rng.standard_normal((dim, width)) / np.sqrt(width)).astype(np.float32)
    b = (0.1 * rng.standard_normal(dim)).astype(np.float32)
    return x, w, b


def minmax_range(u, cuda, g0=0, stride=1):
    ctx = cl.Context.get(cuda.index)
    r = torch.zeros(4, dtype=torch.float64, device=cuda)
    s = torch.cuda.current_stream(cuda).cuda_stream
    ctx.call("cl_range_init", r.data_ptr(), s)
    ctx.call("cl_minmax_f32", u.data_ptr(), u.numel(), g0, stride, r.data_ptr(), s)
    return r


@pytest.mark.parametrize("width", [1, 2, 3, 4])
@pytest.mark.parametrize("L", [64, 37, 384, 1152])  # float4 runs / scalar (L % 4 != 0) /
# warp-coalesced (L % 128 == 0: 3 blocks per row, 2 runs + a 1-block tail)
def test_conv_matches_fp64(cuda, width, L):
    x, w, b = conv_inputs(width, 2, 24, L, width)
    for silu in (True, False):
        u = causal_conv1d_fn(t(x, cuda), t(w, cuda), t(b, cuda), "silu" if silu else None)
        ref = causal_conv1d_f64(x, w, b, silu)
        assert_close_normwise(u.cpu().numpy().reshape(-1, L), ref.reshape(-1, L), 2e-6, "u")
    u = causal_conv1d_fn(t(x, cuda), t(w, cuda), None, "silu")
    assert_close_normwise(u.cpu().numpy().reshape(-1, L),
                          causal_conv1d_f64(x, w, None, True).reshape(-1, L), 2e-6, "u")


def test_conv_is_causal(cuda):
    """Changing x at t0 leaves every output before t0 unchanged (bitwise)."""
    x, w, b = conv_inputs(5, 1, 8, 128, 4)
    u0 = causal_conv1d_fn(t(x, cuda), t(w, cuda), t(b, cuda)).cpu().numpy()
    x2 = x.copy()
    x2[:, :, 77:] += 1.0
    u1 = causal_conv1d_fn(t(x2, cuda), t(w, cuda), t(b, cuda)).cpu().numpy()
    assert (u0[:, :, :77] == u1[:, :, :77]).all()
    assert (u0[:, :, 77:] != u1[:, :, 77:]).any()


@pytest.mark.parametrize("stride,g0", [(1, 0), (3, 0), (8, 5), (5, 1000003)])
def test_fused_range_equals_minmax(cuda, stride, g0):
    x, w, b = conv_inputs(11, 3, 40, 256, 4)
    r = torch.zeros(4, dtype=torch.float64, device=cuda)
    ctx = cl.Context.get(cuda.index)
    ctx.call("cl_range_init", r.data_ptr(), torch.cuda.current_stream(cuda).cuda_stream)
    u = causal_conv1d_fn(t(x, cuda), t(w, cuda), t(b, cuda), "silu", None, r, g0, stride)
    r_ref = minmax_range(u, cuda, g0, stride)
    assert torch.equal(r, r_ref)
    assert r[2].item() == 0.0


def test_fused_range_flags_nonfinite(cuda):
    x, w, b = conv_inputs(12, 1, 16, 64, 4)
    x[0, 3, 10] = np.inf
    r = torch.zeros(4, dtype=torch.float64, device=cuda)
    cl.Context.get(cuda.index).call("cl_range_init", r.data_ptr(),
                                    torch.cuda.current_stream(cuda).cuda_stream)
    causal_conv1d_fn(t(x, cuda), t(w, cuda), t(b, cuda), "silu", None, r)
    assert r[2].item() == 1.0


FROM_CONV_CASES = {
    # name: (spec, L, width, policy)
    "dynamic": (dict(), 512, 4, None),
    "dynamic-stride8": (dict(sample_stride=8), 512, 4, None),
    "fixed-fused": (dict(range_mode=cl.RangeMode.Fixed, fixed_lo=-1.5, fixed_hi=2.5), 1024, 4,
                    None),  # the conv + histogram epilogue kernel (clipped outliers too)
    "fixed-fused-w3-k64": (dict(range_mode=cl.RangeMode.Fixed, fixed_lo=-3.0, fixed_hi=3.0,
                                bin_count=64), 1152, 3, None),  # tail units (1152/4/32 = 9)
    "fixed-fallback": (dict(range_mode=cl.RangeMode.Fixed, fixed_lo=-1.5, fixed_hi=2.5), 516, 4,
                       None),  # L % 128 != 0: conv + separate histogram
    "fixed-stride3": (dict(range_mode=cl.RangeMode.Fixed, fixed_lo=-1.5, fixed_hi=2.5,
                           sample_stride=3), 512, 2, None),
    "token": (dict(), 512, 4, "token"),
}


@pytest.mark.parametrize("case", sorted(FROM_CONV_CASES))
def test_prefill_from_conv_equals_unfused(cuda, case):
    """cl_prefill_from_conv_f32 (producer fused: min/max or the whole Fixed-range histogram
    in the conv epilogue) gives the same u, counts, decision and scan output, bit for bit,
    as the conv followed by the unfused prefill on the same u."""
    kw, L, width, pol = FROM_CONV_CASES[case]
    m = mamba_inputs(21, 2, 64, 16, L)
    x, w, b = conv_inputs(22, 2, 64, L, width)
    d = {k: t(v, cuda) for k, v in m.items()}
    spec = cl.HistogramSpec(**kw)
    policy = bounds = None
    if pol == "token":
        policy = cl.SchedulerPolicy(cl.TokenHistogramPolicy(), [128, 256, 512])
        bounds = cl.ChunkBounds(128, 512)
    pf_fused = Prefill(spec, policy, bounds, device=cuda)
    res_f, u = pf_fused.from_conv(t(x, cuda), t(w, cuda), t(b, cuda), d["delta"], d["A"],
                                  d["B"], d["C"], d["D"], d["z"], d["delta_bias"], True,
                                  return_last_state=True)
    rec_f = res_f.decision()
    u_ref = causal_conv1d_fn(t(x, cuda), t(w, cuda), t(b, cuda), "silu")
    assert torch.equal(u, u_ref)
    pf = Prefill(spec, policy, bounds, device=cuda)
    res = pf(u_ref, d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"], True,
             return_last_state=True)
    rec = res.decision()
    assert torch.equal(pf_fused.decision_buf, pf.decision_buf)
    if pol is None:
        assert torch.equal(pf_fused.counts, pf.counts)
    assert rec_f.decision.chunk == rec.decision.chunk
    assert rec_f.entropy.raw_nats == rec.entropy.raw_nats
    assert (rec_f.lo, rec_f.hi) == (rec.lo, rec.hi)
    assert torch.equal(res_f.out, res.out) and torch.equal(res_f.h_last, res.h_last)


def test_prefill_from_conv_fixed_counts_vs_oracle(cuda, port):
    """The conv + Fixed-range histogram epilogue's counts against the C oracle's
    compute_histogram (Fixed mode, entropy.hpp:116-119) of the produced u."""
    x, w, b = conv_inputs(23, 2, 96, 2048, 4)
    m = mamba_inputs(24, 2, 96, 16, 2048)
    d = {k: t(v, cuda) for k, v in m.items()}
    spec = cl.HistogramSpec(range_mode=cl.RangeMode.Fixed, fixed_lo=-0.5, fixed_hi=1.0)
    pf = Prefill(spec, device=cuda)
    _, u = pf.from_conv(t(x, cuda), t(w, cuda), t(b, cuda), d["delta"], d["A"], d["B"], d["C"],
                        d["D"], d["z"], d["delta_bias"], True)
    ref, *_ = port.histogram(u.cpu().numpy().reshape(-1), 256, 1e-8, 1, fixed=(-0.5, 1.0))
    assert (pf.counts.cpu().numpy().astype(np.uint64) == ref).all()


def test_prefill_from_conv_nonfinite_defers_error(cuda):
    x, w, b = conv_inputs(25, 1, 64, 512, 4)
    x[0, 5, 100] = np.nan
    m = mamba_inputs(26, 1, 64, 16, 512)
    d = {k: t(v, cuda) for k, v in m.items()}
    for kw in (dict(), dict(range_mode=cl.RangeMode.Fixed, fixed_lo=-1.0, fixed_hi=1.0)):
        pf = Prefill(cl.HistogramSpec(**kw), device=cuda)
        out = torch.full_like(d["u"], 3.0)
        res, _ = pf.from_conv(t(x, cuda), t(w, cuda), t(b, cuda), d["delta"], d["A"], d["B"],
                              d["C"], d["D"], d["z"], d["delta_bias"], True, out=out)
        with pytest.raises(cl.InvalidInput, match="non-finite input"):
            res.decision()
        assert bool((out == 3.0).all())


def test_conv_validation(cuda):
    x, w, b = conv_inputs(1, 1, 4, 16, 4)
    w5 = np.zeros((4, 5), np.float32)
    with pytest.raises(cl.InvalidInput, match=r"conv width must lie in \[1, 4\]"):
        causal_conv1d_fn(t(x, cuda), t(w5, cuda), t(b, cuda))
    with pytest.raises(cl.InvalidInput, match="shape mismatch"):
        causal_conv1d_fn(t(x, cuda), t(w[:3], cuda), t(b, cuda))
