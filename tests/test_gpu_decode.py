"""GPU: decode step (mamba_ssm selective_state_update semantics) and the
passive-vs-routed equivalence the paper claims (bitwise output equality).

All Mamba-1 paths share one elementwise math and (N = 16) one C.h order, so:
  * prefill(L) followed by k decode steps == prefill(L + k), bit for bit, for the chained
    kernels (the L-parallel kernel, which AUTO picks for few rows, folds segment
    aggregates into its carry-ins: there the equality holds to rounding,
    tests/test_gpu_lookback.py);
  * the generic scan == the chained TMA scan, bit for bit;
  * any chunk policy (passive Static or routed by entropy) gives the same output bits,
    for every kernel AUTO can pick (the L-parallel split is tied to the shape)."""
import numpy as np
import pytest
import torch

import paper_2604_10597_b200 as cl
from paper_2604_10597_b200.mamba1 import Prefill, selective_scan_fn, selective_state_update
from tests._helpers import assert_close_normwise, mamba_inputs

pytestmark = pytest.mark.gpu


def dev(x, cuda):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).to(cuda) for k, v in x.items()}


@pytest.mark.parametrize("with_z,with_bias", [(True, True), (False, False)])
def test_prefill_then_decode_equals_longer_prefill(cuda, with_z, with_bias):
    L0, k = 256, 4
    x = mamba_inputs(31, 2, 48, 16, L0 + k)
    d = dev(x, cuda)
    z = d["z"] if with_z else None
    bias = d["delta_bias"] if with_bias else None
    full, h_full = selective_scan_fn(d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], z, bias,
                                     True, return_last_state=True, chunk_size=64,
                                     variant="chained")
    part, h = selective_scan_fn(d["u"][..., :L0].contiguous(), d["delta"][..., :L0].contiguous(),
                                d["A"], d["B"][..., :L0].contiguous(),
                                d["C"][..., :L0].contiguous(), d["D"],
                                None if z is None else z[..., :L0].contiguous(), bias, True,
                                return_last_state=True, chunk_size=128, variant="chained")
    assert torch.equal(part, full[..., :L0])
    state = h.clone()
    for t in range(L0, L0 + k):
        y = selective_state_update(state, d["u"][..., t].contiguous(),
                                   d["delta"][..., t].contiguous(), d["A"],
                                   d["B"][..., t].contiguous(), d["C"][..., t].contiguous(),
                                   d["D"], None if z is None else z[..., t].contiguous(), bias,
                                   dt_softplus=True)
        assert torch.equal(y, full[..., t]), t
    assert torch.equal(state, h_full)


def test_generic_equals_tma(cuda):
    x = mamba_inputs(32, 2, 40, 16, 512)
    d = dev(x, cuda)
    args = (d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"], True)
    y_t, h_t = selective_scan_fn(*args, return_last_state=True, chunk_size=256, variant="chained")
    y_g, h_g = selective_scan_fn(*args, return_last_state=True, chunk_size=256, variant="generic")
    assert torch.equal(y_t, y_g) and torch.equal(h_t, h_g)


def test_passive_vs_routed_bitwise(cuda):
    """The paper's quality-preservation claim: the output does not depend on the chunk the
    policy picks -- passive Static{c} for every c vs the entropy-routed rule."""
    x = mamba_inputs(33, 1, 64, 16, 1024)
    d = dev(x, cuda)
    args = (d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"], True)
    routed = Prefill(cl.HistogramSpec(), device=cuda)(*args)
    ref = routed.out.clone()
    for c in (32, 64, 128, 256, 512):
        pol = cl.SchedulerPolicy(cl.StaticPolicy(c), [32, 64, 128, 256, 512])
        res = Prefill(cl.HistogramSpec(), pol, cl.ChunkBounds(32, 512), device=cuda)(*args)
        assert res.decision().decision.chunk == c
        assert torch.equal(res.out, ref), c


def test_decode_vs_oracle(cuda, port):
    """One decode step against the fp64 restatement (a 1-token scan from h0)."""
    x = mamba_inputs(34, 2, 32, 16, 1)
    rng = np.random.default_rng(35)
    h0 = rng.standard_normal((2, 32, 16)).astype(np.float32)
    d = dev(x, cuda)
    state = torch.from_numpy(h0).to(cuda)
    y = selective_state_update(state, d["u"][..., 0].contiguous(), d["delta"][..., 0].contiguous(),
                               d["A"], d["B"][..., 0].contiguous(), d["C"][..., 0].contiguous(),
                               d["D"], d["z"][..., 0].contiguous(), d["delta_bias"], True)
    f64 = {k: v.astype(np.float64) for k, v in x.items()}  # exact widening
    yr, hr = port.mamba1(f64["u"], f64["delta"], f64["A"], f64["B"], f64["C"], f64["D"], f64["z"],
                         f64["delta_bias"], True, h0=h0.astype(np.float64))
    # one token per row: normwise over the whole decode output (a single element has no
    # normwise meaning), per row for the states
    assert_close_normwise(y.cpu().numpy().reshape(1, -1), yr.reshape(1, -1), 1e-5)
    assert_close_normwise(state.cpu().numpy().reshape(-1, 16), hr.reshape(-1, 16), 1e-5)


def test_decode_general_state_dim(cuda, port):
    x = mamba_inputs(36, 1, 16, 8, 1)
    d = dev(x, cuda)
    state = torch.zeros(1, 16, 8, device=cuda)
    y = selective_state_update(state, d["u"][..., 0].contiguous(), d["delta"][..., 0].contiguous(),
                               d["A"], d["B"][..., 0].contiguous(), d["C"][..., 0].contiguous(),
                               d["D"], None, d["delta_bias"], True)
    yr, hr = port.mamba1(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], None,
                         x["delta_bias"], True)
    assert_close_normwise(y.cpu().numpy().reshape(1, -1), yr.reshape(1, -1), 1e-5)


def test_decode_validation(cuda):
    s = torch.zeros(1, 4, 16, device=cuda)
    v = torch.zeros(1, 4, device=cuda)
    A = torch.zeros(4, 16, device=cuda)
    B = torch.zeros(1, 16, device=cuda)
    with pytest.raises(cl.InvalidInput, match="shape mismatch"):
        selective_state_update(s, v, v, A[:3], B, B)
    with pytest.raises(cl.InvalidInput, match="float32"):
        selective_state_update(s, v.double(), v, A, B, B)
