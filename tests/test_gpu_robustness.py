"""GPU: inputs the product must refuse before any launch, and histogram semantics when a
caller-supplied Dynamic range does not cover the data."""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2604_10597_b200 as cl
from paper_2604_10597_b200 import _lib
from paper_2604_10597_b200.mamba1 import Prefill, selective_scan_fn
from tests._helpers import mamba_inputs

pytestmark = pytest.mark.gpu


def dev(x, cuda):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).to(cuda) for k, v in x.items()}


@pytest.mark.parametrize("bad", ["bf16", "cpu", "noncontig", "shape"])
def test_prefill_rejects_bad_inputs_before_any_launch(cuda, bad):
    x = dev(mamba_inputs(1, 1, 64, 16, 256), cuda)
    if bad == "bf16":
        x["u"] = x["u"].to(torch.bfloat16)
    elif bad == "cpu":
        x["u"] = x["u"].cpu()
    elif bad == "noncontig":
        x["delta"] = x["delta"].transpose(1, 2).contiguous().transpose(1, 2)
    else:
        x["z"] = x["z"][:, :, :128].contiguous()
    pf = Prefill(cl.HistogramSpec(), device=cuda)
    before = pf.ctx.launches
    for call in (
        lambda: pf(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"], x["delta_bias"]),
        lambda: selective_scan_fn(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"],
                                  x["delta_bias"], True),
    ):
        with pytest.raises(cl.InvalidInput):
            call()
    assert pf.ctx.launches == before
    torch.cuda.synchronize()  # the context is healthy: nothing illegal was queued


def test_from_conv_rejects_bad_weights_before_any_launch(cuda):
    x = dev(mamba_inputs(1, 1, 64, 16, 256), cuda)
    pf = Prefill(cl.HistogramSpec(), device=cuda)
    before = pf.ctx.launches
    w = torch.randn(64, 4, device=cuda).to(torch.bfloat16)
    with pytest.raises(cl.InvalidInput):
        pf.from_conv(x["u"], w, None, x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"],
                     x["delta_bias"])
    assert pf.ctx.launches == before


def test_device_without_index_is_the_current_device(cuda):
    pf = Prefill(cl.HistogramSpec(), device="cuda")
    assert pf.device == torch.device("cuda", torch.cuda.current_device())


@pytest.mark.parametrize("n", [1 << 20, 3000])
def test_uncovered_dynamic_range_clamps_like_the_reference(cuda, port, n):
    """A d_range narrower than the data (e.g. a missing MAX-allreduce) must bin exactly as
    detail::bin_index does with that range: out-of-range samples clip to the edge bins
    (entropy.hpp:87-94) -- never wrap into bin n mod 256."""
    rng = np.random.default_rng(2)
    v = rng.standard_normal(n).astype(np.float32)
    lo, hi = float(np.float32(-1.0)), float(np.float32(1.25))
    d = torch.from_numpy(v).to(cuda)
    ctx = cl.Context.get(cuda.index)
    s = torch.cuda.current_stream(cuda).cuda_stream
    for k in (256, 64, 100):  # power-of-two K: the one-LOP3 range check; 100: the compare
        spec = cl.HistogramSpec(bin_count=k)
        cs = spec.to_c()
        rng_buf = torch.tensor([-lo, hi, 0.0, 0.0], dtype=torch.float64, device=cuda)
        counts = torch.zeros(k, dtype=torch.int64, device=cuda)
        ctx.call("cl_histogram_f32", d.data_ptr(), n, 0, C.byref(cs), rng_buf.data_ptr(),
                 counts.data_ptr(), s)
        ref, *_ = port.histogram(v, k, 1e-8, 1, fixed=(lo, hi))
        assert (counts.cpu().numpy().astype(np.uint64) == ref).all(), k
        # and through the fused histogram -> decision launch
        counts.zero_()
        dec = torch.zeros(C.sizeof(_lib.cl_decision), dtype=torch.uint8, device=cuda)
        from paper_2604_10597_b200.chunklab import rule_spec
        rule = rule_spec(None, cl.ChunkBounds(32, 512), cl.CalibrationRef.log_k(k))
        ctx.call("cl_histogram_decide_f32", d.data_ptr(), n, C.byref(cs), rng_buf.data_ptr(),
                 counts.data_ptr(), C.byref(rule), 1, dec.data_ptr(), s)
        assert (counts.cpu().numpy().astype(np.uint64) == ref).all(), k
