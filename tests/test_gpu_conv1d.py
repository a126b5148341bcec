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


@pytest.mark.parametrize("stride", [1, 8])
def test_prefill_from_conv_equals_unfused(cuda, stride):
    """Fused producer -> histogram -> decide -> scan gives the same decision, entropy
    and output (bitwise) as conv, then the unfused prefill on the same u."""
    m = mamba_inputs(21, 2, 64, 16, 512)
    x, w, b = conv_inputs(22, 2, 64, 512, 4)
    d = {k: t(v, cuda) for k, v in m.items()}
    spec = cl.HistogramSpec(sample_stride=stride)
    pf_fused = Prefill(spec, device=cuda)
    res_f, u = pf_fused.from_conv(t(x, cuda), t(w, cuda), t(b, cuda), d["delta"], d["A"],
                                  d["B"], d["C"], d["D"], d["z"], d["delta_bias"], True)
    rec_f = res_f.decision()
    pf = Prefill(spec, device=cuda)
    res = pf(u, d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"], True)
    rec = res.decision()
    assert rec_f.decision.chunk == rec.decision.chunk
    assert rec_f.entropy.raw_nats == rec.entropy.raw_nats
    assert (rec_f.lo, rec_f.hi) == (rec.lo, rec.hi)
    assert torch.equal(res_f.out, res.out)


def test_conv_validation(cuda):
    x, w, b = conv_inputs(1, 1, 4, 16, 4)
    w5 = np.zeros((4, 5), np.float32)
    with pytest.raises(cl.InvalidInput, match=r"conv width must lie in \[1, 4\]"):
        causal_conv1d_fn(t(x, cuda), t(w5, cuda), t(b, cuda))
    with pytest.raises(cl.InvalidInput, match="shape mismatch"):
        causal_conv1d_fn(t(x, cuda), t(w[:3], cuda), t(b, cuda))
