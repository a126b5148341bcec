"""GPU: parity at every BASELINE.json shape beyond C3 (test_gpu_fullsize.py), through the
prefill a caller uses (Prefill: min/max -> histogram -> device policy -> CL_SCAN_AUTO scan).

  configs[0] C1  B=1 L=2048  d_inner=1536   calibrated rule, every row vs the fp64 oracle
  configs[1] C2  B=1 L=4096  d_inner=2048   calibrated rule, every row vs the fp64 oracle
  configs[3] C4  B=16 L=16384 d_inner=5120  Guarded{Sampled stride 8, safe 512, min_delta 2}
                                            with bounds [128, 2048] (chunk.hpp:344-358):
                                            whole-tensor counts + decision bit-exact, 64 rows
  configs[4] serving mix, B=1 d_inner=2048, the L = 32768 request: guarded entropy policy

Counts and the chunk are bit-exact against the C oracle (which is pinned to the reference
build, tests/test_oracle.py); scan rows are <= 1e-5 normwise against the fp64 Mamba-1
oracle."""
import math

import numpy as np
import pytest
import torch

import bench
import paper_2604_10597_b200 as cl
from oracle import oracle as O
from paper_2604_10597_b200.mamba1 import Prefill, selective_scan_fn
from tests._helpers import assert_close_normwise

pytestmark = pytest.mark.gpu

BUCKETS = [128, 256, 512, 1024, 2048]


def guarded_stride8():
    inner = cl.SchedulerPolicy(cl.SampledHistogramPolicy(8), BUCKETS)
    return cl.SchedulerPolicy(cl.GuardedPolicy(inner, 512, 2), BUCKETS)


def oracle_guarded_chunk(port, raw, bounds):
    p = O.Policy()
    p.kind, p.inner_kind, p.safe_chunk, p.min_delta_buckets = 5, 3, 512, 2
    p.n_buckets = len(BUCKETS)
    for i, b in enumerate(BUCKETS):
        p.buckets[i] = b
    f = O.Features(0, 0.0, 1, raw, 0, 0)
    c, *_ = port.schedule(p, f, bounds[0], bounds[1], math.log(256))
    return c


def run_prefill(x, pf):
    res = pf(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"], x["delta_bias"], True,
             return_last_state=True)
    return res, res.decision()


def check_rows(port, x, res, rows):
    """fp64 oracle on (b, d) rows; inputs sliced on the device, copied per row."""
    A = x["A"].cpu().numpy()
    D = x["D"].cpu().numpy()
    bias = x["delta_bias"].cpu().numpy()
    worst = 0.0
    by_batch = {}
    for b, d in rows:
        by_batch.setdefault(b, []).append(d)
    for b, ds in by_batch.items():
        Bb = x["B"][b:b + 1].cpu().numpy()
        Cb = x["C"][b:b + 1].cpu().numpy()
        for d in ds:
            sl = (slice(b, b + 1), slice(d, d + 1))
            yr, hr = port.mamba1(x["u"][sl].cpu().numpy(), x["delta"][sl].cpu().numpy(),
                                 A[d:d + 1], Bb, Cb, D[d:d + 1], x["z"][sl].cpu().numpy(),
                                 bias[d:d + 1], True)
            r, _, _ = assert_close_normwise(res.out[b, d].cpu().numpy()[None], yr, 1e-5,
                                            f"y[{b},{d}]")
            assert_close_normwise(res.h_last[b, d].cpu().numpy()[None], hr, 1e-5, f"h[{b},{d}]")
            worst = max(worst, r)
    return worst


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_few_row_configs_every_row_through_auto(cuda, port, cfg):
    batch, dim, L, N, _ = bench.CONFIGS[cfg]
    x = bench.make_inputs(torch, cuda, batch, dim, L, N, 7)
    pf = Prefill(cl.HistogramSpec(), None, cl.ChunkBounds(32, 512), device=cuda)
    res, rec = run_prefill(x, pf)
    xs = {k: v.cpu().numpy() for k, v in x.items()}
    counts, lo, hi, n = port.histogram(xs["u"].reshape(-1), 256, 1e-8, 1)
    assert (pf.counts.cpu().numpy().astype(np.uint64) == counts).all()
    raw, _ = port.entropy(counts.astype(np.float64) * (1.0 / n))
    assert rec.decision.chunk == port.select_chunk(raw, 32, 512, math.log(256))[0]
    yr, hr = port.mamba1(xs["u"], xs["delta"], xs["A"], xs["B"], xs["C"], xs["D"], xs["z"],
                         xs["delta_bias"], True)
    assert_close_normwise(res.out.cpu().numpy().reshape(-1, L), yr, 1e-5)
    assert_close_normwise(res.h_last.cpu().numpy().reshape(-1, N), hr, 1e-5, "h_last")
    # the scan's output does not depend on the decided chunk (the L-split of the few-row
    # kernel is tied to the shape, the chained kernel's carry order to nothing)
    args = (x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"], x["delta_bias"], True)
    for chunk in (64, 2048):
        y2, h2 = selective_scan_fn(*args, return_last_state=True, chunk_size=chunk)
        assert torch.equal(y2, res.out) and torch.equal(h2, res.h_last), chunk


@pytest.fixture(scope="module")
def c4(cuda):
    batch, dim, L, N, _ = bench.CONFIGS["C4"]
    x = bench.make_inputs(torch, cuda, batch, dim, L, N, 11)
    yield x
    del x
    torch.cuda.empty_cache()


def test_c4_guarded_stride8_counts_decision_and_rows(cuda, port, c4):
    batch, dim, L, N, _ = bench.CONFIGS["C4"]
    bounds = (128, 2048)
    pf = Prefill(cl.HistogramSpec(sample_stride=8), guarded_stride8(),
                 cl.ChunkBounds(*bounds), cl.CalibrationRef.log_k(256), device=cuda)
    res, rec = run_prefill(c4, pf)
    # whole-tensor histogram at stride 8: 1.34e9 values, 168M samples (the oracle reads
    # the host copy of u with the same global-index sampling)
    u_host = c4["u"].cpu().numpy().reshape(-1)
    counts, lo, hi, n = port.histogram(u_host, 256, 1e-8, 8)
    del u_host
    assert n == (batch * dim * L + 7) // 8
    assert (pf.counts.cpu().numpy().astype(np.uint64) == counts).all()
    assert (rec.lo, rec.hi) == (lo, hi)
    raw, _ = port.entropy(counts.astype(np.float64) * (1.0 / n))
    assert rec.entropy.raw_nats == pytest.approx(raw, rel=1e-13, abs=0)
    expect = oracle_guarded_chunk(port, raw, bounds)
    assert rec.decision.chunk == expect
    # standard-normal u: the rule gives 2048 and the guard keeps it (SURVEY finding 8)
    assert expect == 2048 and rec.decision.source_policy.startswith("guarded")
    rng = np.random.default_rng(5)
    rows = [(int(b), int(d)) for b, d in zip(rng.integers(0, batch, 60), rng.integers(0, dim, 60))]
    rows += [(0, 0), (batch - 1, dim - 1), (3, 15), (9, 16)]
    worst = check_rows(port, c4, res, rows)
    print(f"C4: 64 rows at L={L}, worst row rel err {worst:.2e}")


def test_c4_chunk_invariance(cuda, c4):
    args = (c4["u"], c4["delta"], c4["A"], c4["B"], c4["C"], c4["D"], c4["z"],
            c4["delta_bias"], True)
    y512, h512 = selective_scan_fn(*args, return_last_state=True, chunk_size=512)
    y2048, h2048 = selective_scan_fn(*args, return_last_state=True, chunk_size=2048)
    assert torch.equal(y512, y2048) and torch.equal(h512, h2048)
    assert torch.isfinite(y512).all()


def test_serving_mix_long_request_l32768(cuda, port):
    """BASELINE configs[4]'s longest request: B=1, d_inner=2048, L=32768, guarded entropy."""
    dim, L, N = 2048, 32768, 16
    x = bench.make_inputs(torch, cuda, 1, dim, L, N, 13)
    bounds = (128, 2048)
    inner = cl.SchedulerPolicy(cl.FullHistogramPolicy(), BUCKETS)
    pol = cl.SchedulerPolicy(cl.GuardedPolicy(inner, 512, 2), BUCKETS)
    pf = Prefill(cl.HistogramSpec(), pol, cl.ChunkBounds(*bounds), device=cuda)
    res, rec = run_prefill(x, pf)
    u_host = x["u"].cpu().numpy().reshape(-1)
    counts, lo, hi, n = port.histogram(u_host, 256, 1e-8, 1)
    assert (pf.counts.cpu().numpy().astype(np.uint64) == counts).all()
    raw, _ = port.entropy(counts.astype(np.float64) * (1.0 / n))
    p = O.Policy()
    p.kind, p.inner_kind, p.safe_chunk, p.min_delta_buckets = 5, 2, 512, 2
    p.n_buckets = len(BUCKETS)
    for i, b in enumerate(BUCKETS):
        p.buckets[i] = b
    c, *_ = port.schedule(p, O.Features(1, raw, 0, 0.0, 0, 0), bounds[0], bounds[1],
                          math.log(256))
    assert rec.decision.chunk == c
    rng = np.random.default_rng(6)
    rows = [(0, int(d)) for d in rng.integers(0, dim, 48)] + [(0, 0), (0, dim - 1)]
    worst = check_rows(port, x, res, rows)
    print(f"L=32768: 50 rows, worst row rel err {worst:.2e}")
