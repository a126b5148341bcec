"""GPU: the L-parallel scan (scan_lookback.cu) -- VERDICT round 1 "missing #1".

Each 16-row tile's L is split into segments by the SHAPE (never by the decided chunk);
every segment but the last publishes its aggregate (local end state from h = 0, sum of
the discretised steps), and every segment but the first folds its predecessors'
aggregates, in segment order, into its carry-in.  Checked here:
  * <= 1e-5 normwise against the fp64 oracle for every kernel-table row,
    with and without h0 / z / D / softplus, partial tiles, L not a multiple of the box;
  * agreement with the chained kernel within the same 1e-5;
  * bit-identical output for every decided chunk, and run to run (a fixed fold order);
  * deferred device errors write nothing;
  * AUTO picks it exactly for few-row shapes (cl_scan_plan_f32)."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2604_10597_b200 import _lib
from paper_2604_10597_b200.mamba1 import scan_plan, selective_scan_fn, selective_state_update
from tests._helpers import assert_close_normwise, mamba_inputs, rel_err_rows

pytestmark = pytest.mark.gpu

LB_CFGS = [0, 1, 2, 3]


def to_dev(x, cuda):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).to(cuda) for k, v in x.items()}


def oracle64(port, x, h0=None, softplus=True, use_z=True, use_D=True):
    """fp64 restatement on the fp32 inputs (widened), optionally from h0."""
    w = {k: np.asarray(v, dtype=np.float64) for k, v in x.items()}
    return port.mamba1(w["u"], w["delta"], w["A"], w["B"], w["C"], w["D"] if use_D else None,
                       w["z"] if use_z else None, w["delta_bias"], softplus,
                       h0=None if h0 is None else np.asarray(h0, dtype=np.float64))


SHAPES = [  # batch, dim, L
    (1, 48, 2048),   # 3 tiles, many segments
    (2, 40, 1000),   # partial tile, L % 32 != 0
    (1, 16, 4096),   # one tile: the fold crosses up to ~148 segments
    (3, 96, 516),
    (1, 8, 4),       # tiny: one segment
]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("cfg", LB_CFGS)
def test_lookback_matches_oracle(cuda, port, shape, cfg):
    batch, dim, L = shape
    x = mamba_inputs(hash((shape, "lb")) % 1000, batch, dim, 16, L)
    d = to_dev(x, cuda)
    h0 = np.random.default_rng(3).standard_normal((batch, dim, 16)).astype(np.float32)
    for use_h0 in (False, True):
        h0d = torch.from_numpy(h0).to(cuda) if use_h0 else None
        y, h = selective_scan_fn(d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"],
                                 d["delta_bias"], True, True, h0=h0d, variant=f"lb:{cfg}")
        yr, hr = oracle64(port, x, h0 if use_h0 else None)
        assert_close_normwise(y.cpu().numpy().reshape(-1, L), yr, 1e-5, f"y h0={use_h0}")
        assert_close_normwise(h.cpu().numpy().reshape(-1, 16), hr, 1e-5, f"h h0={use_h0}")


@pytest.mark.parametrize("flags", [(False, False, False), (True, False, True),
                                   (False, True, False)])
def test_lookback_optional_terms(cuda, port, flags):
    softplus, use_z, use_D = flags
    batch, dim, L = 2, 32, 1536
    x = mamba_inputs(91, batch, dim, 16, L)
    if not softplus:  # raw delta must stay positive
        x["delta"] = np.abs(x["delta"]) * 0.1
        x["delta_bias"] = np.abs(x["delta_bias"]) * 0.01
    d = to_dev(x, cuda)
    y, h = selective_scan_fn(d["u"], d["delta"], d["A"], d["B"], d["C"],
                             d["D"] if use_D else None, d["z"] if use_z else None,
                             d["delta_bias"], softplus, True, variant="lookback")
    yr, hr = oracle64(port, x, None, softplus, use_z, use_D)
    assert_close_normwise(y.cpu().numpy().reshape(-1, L), yr, 1e-5)
    assert_close_normwise(h.cpu().numpy().reshape(-1, 16), hr, 1e-5, "h")


@pytest.mark.parametrize("shape", [(1, 1536, 2048), (1, 2048, 4096), (1, 64, 8192)])
def test_lookback_vs_chained_and_chunk_invariance(cuda, shape):
    batch, dim, L = shape
    x = to_dev(mamba_inputs(5, batch, dim, 16, L), cuda)
    args = (x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"], x["delta_bias"], True)
    yc, hc = selective_scan_fn(*args, return_last_state=True, variant="chained")
    ys = {}
    for chunk in (32, 512, 2048):
        ys[chunk] = selective_scan_fn(*args, return_last_state=True, chunk_size=chunk,
                                      variant="lookback")
    y, h = ys[512]
    for chunk, (y2, h2) in ys.items():
        assert torch.equal(y2, y) and torch.equal(h2, h), chunk
    again = selective_scan_fn(*args, return_last_state=True, chunk_size=512, variant="lookback")
    assert torch.equal(again[0], y) and torch.equal(again[1], h)
    r = rel_err_rows(y.cpu().numpy().reshape(-1, L), yc.cpu().numpy().reshape(-1, L).astype(np.float64))
    assert r.max() <= 1e-5, r.max()  # each is within ~2e-7 of the fp64 oracle
    rh = rel_err_rows(h.cpu().numpy().reshape(-1, 16), hc.cpu().numpy().reshape(-1, 16).astype(np.float64))
    assert rh.max() <= 1e-5, rh.max()


def test_lookback_deferred_error_writes_nothing(cuda):
    x = to_dev(mamba_inputs(6, 1, 64, 16, 1024), cuda)
    dec = torch.zeros(C.sizeof(_lib.cl_decision), dtype=torch.uint8, device=cuda)
    dec.view(torch.int32)[0] = 1  # CL_DEV_NON_FINITE, as the entropy stage would write
    dec.view(torch.int32)[1] = 512
    out = torch.full_like(x["u"], 7.0)
    selective_scan_fn(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"], x["delta_bias"],
                      True, variant="lookback", decision=dec, out=out)
    torch.cuda.synchronize()
    assert bool((out == 7.0).all())


def test_lookback_prefill_then_decode_close_to_longer_prefill(cuda):
    L0, k = 2048, 4  # both lengths % 4 == 0 (TMA path)
    x = to_dev(mamba_inputs(8, 1, 64, 16, L0 + k), cuda)
    full, _ = selective_scan_fn(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"],
                                x["delta_bias"], True, True, variant="lookback")
    cut = lambda t: t[..., :L0].contiguous()  # noqa: E731
    _, h = selective_scan_fn(cut(x["u"]), cut(x["delta"]), x["A"], cut(x["B"]), cut(x["C"]),
                             x["D"], cut(x["z"]), x["delta_bias"], True, True, variant="lookback")
    state = h.clone()
    for t in range(L0, L0 + k):
        y = selective_state_update(state, x["u"][..., t].contiguous(), x["delta"][..., t].contiguous(),
                                   x["A"], x["B"][..., t].contiguous(), x["C"][..., t].contiguous(),
                                   x["D"], x["z"][..., t].contiguous(), x["delta_bias"], True)
        ref = full[..., t].cpu().numpy().astype(np.float64)
        err = np.linalg.norm(y.cpu().numpy() - ref) / np.linalg.norm(ref)
        assert err <= 1e-6, (t, err)


def test_auto_picks_lookback_for_few_rows(cuda):
    def plan(batch, dim, L):
        x = to_dev(mamba_inputs(1, batch, dim, 16, 8), cuda)  # shapes only matter
        u = torch.empty(batch, dim, L, device=cuda)
        B = torch.empty(batch, 16, L, device=cuda)
        return scan_plan(u, u, x["A"], B, B)

    c1 = plan(1, 1536, 2048)
    assert c1["kernel"] == "lookback_ws_kernel" and c1["n_seg"] > 1
    assert c1["n_seg"] * 96 <= 148 * c1["warps"]  # one wave of items
    c3 = plan(8, 4096, 256)  # C3's row count: the chained kernel fills the GPU
    assert c3["kernel"] == "rowpair_ws_kernel" and c3["n_seg"] == -1
