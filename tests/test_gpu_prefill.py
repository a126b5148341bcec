"""GPU: the whole prefill hot path (entropy -> rule -> scan) with no host sync,
vs the oracle; deferred device errors; guarded / learned-table policies."""
import numpy as np
import pytest
import torch

import paper_2604_10597_b200 as cl
from paper_2604_10597_b200.mamba1 import Prefill
from tests._helpers import assert_close_normwise, mamba_inputs

pytestmark = pytest.mark.gpu


def dev(x, cuda):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).to(cuda) for k, v in x.items()}


def expected_chunk(port, u32, k, stride, bounds, h_ref):
    counts, lo, hi, n = port.histogram(u32.reshape(-1), k, 1e-8, stride)
    raw, _ = port.entropy(counts.astype(np.float64) * (1.0 / n))
    return port.select_chunk(raw, bounds[0], bounds[1], h_ref)[0], raw


def test_prefill_rule_and_scan(cuda, port):
    x = mamba_inputs(1, 2, 128, 16, 512)
    d = dev(x, cuda)
    pf = Prefill(cl.HistogramSpec(), device=cuda)
    res = pf(d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"], True,
             return_last_state=True)
    rec = res.decision()
    chunk, raw = expected_chunk(port, x["u"], 256, 1, (32, 512), np.log(256))
    assert rec.decision.chunk == chunk and rec.decision.source_policy == "rule"
    assert rec.entropy.raw_nats == pytest.approx(raw, rel=1e-13, abs=0)
    yr, hr = port.mamba1(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"],
                         x["delta_bias"], True)
    assert_close_normwise(res.out.cpu().numpy().reshape(-1, 512), yr, 1e-5)
    assert_close_normwise(res.h_last.cpu().numpy().reshape(-1, 16), hr, 1e-5)


@pytest.mark.parametrize("dist", ["uniform", "sparse"])
def test_prefill_decision_follows_distribution(cuda, port, dist):
    """Perturbation sweep (fixtures.hpp:40-47): the device rule picks the chunk the
    reference rule picks for uniform / sparse activations."""
    x = mamba_inputs(2, 1, 256, 16, 1024)
    rng = np.random.default_rng(4)
    if dist == "uniform":
        x["u"] = rng.uniform(0, 1, x["u"].shape).astype(np.float32)
    else:
        x["u"] = np.where(rng.uniform(size=x["u"].shape) < 0.02, x["u"], 0).astype(np.float32)
    d = dev(x, cuda)
    pf = Prefill(cl.HistogramSpec(), None, cl.ChunkBounds(32, 512), cl.CalibrationRef.legacy(),
                 device=cuda)
    pf(d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"], True)
    rec = pf.decision()
    chunk, _ = expected_chunk(port, x["u"], 256, 1, (32, 512), 8.0)
    assert rec.decision.chunk == chunk


def test_guarded_sampled_policy(cuda, port):
    """C4 policy: Guarded{inner = sampled histogram stride 8, safe 512, min_delta 2}."""
    x = mamba_inputs(3, 1, 256, 16, 1024)
    d = dev(x, cuda)
    inner = cl.SchedulerPolicy(cl.SampledHistogramPolicy(8), [128, 256, 512, 1024, 2048])
    policy = cl.SchedulerPolicy(cl.GuardedPolicy(inner, 512, 2), [128, 256, 512, 1024, 2048])
    for bounds, expect in [(cl.ChunkBounds(128, 2048), None), (cl.ChunkBounds(32, 512), 512)]:
        pf = Prefill(cl.HistogramSpec(sample_stride=8), policy, bounds,
                     cl.CalibrationRef.log_k(256), device=cuda)
        res = pf(d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"])
        rec = res.decision()
        counts, lo, hi, n = port.histogram(x["u"].reshape(-1), 256, 1e-8, 8)
        raw, _ = port.entropy(counts.astype(np.float64) * (1.0 / n))
        from oracle import oracle as O
        p = O.Policy()
        p.kind, p.inner_kind, p.safe_chunk, p.min_delta_buckets = 5, 3, 512, 2
        p.n_buckets = 5
        for i, b in enumerate([128, 256, 512, 1024, 2048]):
            p.buckets[i] = b
        f = O.Features(0, 0.0, 1, raw, 0, 0)
        c, *_ = port.schedule(p, f, bounds.c_min, bounds.c_max, np.log(256))
        assert rec.decision.chunk == c
        if expect is not None:
            assert c == expect
        yr, _ = port.mamba1(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"],
                            x["delta_bias"], True, rows=(0, 8))
        assert_close_normwise(res.out.cpu().numpy().reshape(-1, 1024)[:8], yr, 1e-5)


def test_learned_table_policy(cuda):
    x = mamba_inputs(4, 1, 64, 16, 256)
    d = dev(x, cuda)
    pol = cl.SchedulerPolicy(cl.LearnedTablePolicy(50, 128, 512), [128, 256, 512])
    pf = Prefill(cl.HistogramSpec(), pol, cl.ChunkBounds(128, 512), device=cuda)
    pf(d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"])
    rec = pf.decision()
    assert rec.decision.chunk == 512 and rec.decision.source_policy == "learned_table"


def test_constant_activation_defers_signal_error(cuda):
    """SURVEY.md finding 7: constant u -> H = -log(1+eps) < 0 -> 'signal must be >= 0',
    raised at the decision sync point; the scan kernel writes nothing."""
    x = mamba_inputs(5, 1, 32, 16, 64)
    x["u"] = np.full_like(x["u"], 3.0)
    d = dev(x, cuda)
    out = torch.full_like(d["u"], 7.0)
    pf = Prefill(cl.HistogramSpec(), device=cuda)
    pf(d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"], out=out)
    with pytest.raises(cl.InvalidInput, match="^signal must be >= 0$"):
        pf.decision()
    assert (out == 7.0).all()


def test_nonfinite_activation_defers_error(cuda):
    x = mamba_inputs(6, 1, 32, 16, 64)
    x["u"][0, 3, 17] = np.nan
    d = dev(x, cuda)
    pf = Prefill(cl.HistogramSpec(), device=cuda)
    pf(d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"])
    with pytest.raises(cl.InvalidInput, match="^non-finite input$"):
        pf.decision()


def test_no_host_sync_in_prefill(cuda):
    """The prefill path is capturable in a CUDA graph (proves no host sync / no
    host-side decision between entropy and scan)."""
    x = mamba_inputs(7, 1, 64, 16, 256)
    d = dev(x, cuda)
    pf = Prefill(cl.HistogramSpec(), device=cuda)
    out = torch.empty_like(d["u"])
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        pf(d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"], out=out)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    ref = out.clone()
    g = torch.cuda.CUDAGraph()
    out.zero_()
    with torch.cuda.graph(g):
        pf(d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"], out=out)
    # the graph owns its scratch (a capture-keyed workspace): every replay, including ones
    # after eager prefills on other streams, reproduces the eager bits
    for it in range(5):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, ref), it
        pf(d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"])


def test_several_graphs_share_the_captured_workspace(cuda):
    """Graphs captured on one stream share that stream's captured workspace (torch's
    graphs all capture on one side stream).  Replayed interleaved -- A B A A C B C ... --
    each reproduces its eager bits: the L-parallel aggregate tags come from a device-side
    launch counter (never repeated across graphs), the chained carry words are zeroed
    in-graph, and the work ticket is 0 again at the end of every launch (the row kernel's
    graph restores it in-graph)."""
    cases = [((1, 48, 2048), "lookback"), ((2, 64, 512), "chained"), ((1, 32, 4096), "lookback"),
             ((4, 64, 256), "auto"), ((2, 64, 512), "cfg:1")]  # cfg:1: the row kernel
    runs = []
    for i, (shape, variant) in enumerate(cases):
        d = dev(mamba_inputs(40 + i, *shape[:2], 16, shape[2]), cuda)
        pf = Prefill(cl.HistogramSpec(), device=cuda)
        pf.scan_variant = variant
        out = torch.empty_like(d["u"])
        args = (d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"])
        pf(*args, out=out)
        torch.cuda.synchronize()
        runs.append([pf, args, out, out.clone(), None])
    for r in runs:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            r[0](*r[1], out=r[2])
        r[4] = g
    for it, k in enumerate([0, 1, 0, 0, 2, 1, 2, 3, 0, 2, 2, 3, 1, 0, 4, 1, 4, 0, 4, 3]):
        pf, args, out, ref, g = runs[k]
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, ref), (it, k)


@pytest.mark.parametrize("case", ["default", "repeat", "stride8", "fixed", "k512", "small",
                                  "nonfinite", "guarded", "ragged"])
def test_histogram_decide_fused_equals_separate(cuda, case):
    """cl_histogram_decide_f32 (the histogram's last CTA decides, where the register-fed
    kernel applies) writes the same counts and the same cl_decision bytes as
    cl_histogram_f32 + cl_decide, on the fused path and on every fallback."""
    n = {"small": 3000, "ragged": 1_000_003}.get(case, 1 << 20)
    g = torch.Generator().manual_seed(11)
    u = torch.randn(n, generator=g).to(cuda)
    if case == "nonfinite":
        u[12345] = float("nan")
    spec = cl.HistogramSpec()
    policy = None
    bounds = cl.ChunkBounds(32, 512)
    if case == "stride8":
        spec = cl.HistogramSpec(sample_stride=8)
    elif case == "fixed":
        spec = cl.HistogramSpec(range_mode=cl.RangeMode.Fixed, fixed_lo=-2.0, fixed_hi=2.0)
    elif case == "k512":
        spec = cl.HistogramSpec(bin_count=512)
    elif case == "guarded":
        inner = cl.SchedulerPolicy(cl.FullHistogramPolicy(), [128, 256, 512, 1024, 2048])
        policy = cl.SchedulerPolicy(cl.GuardedPolicy(inner, 512, 2), [128, 256, 512, 1024, 2048])
        bounds = cl.ChunkBounds(128, 2048)
    a = Prefill(spec, policy, bounds, cl.CalibrationRef.log_k(spec.bin_count), device=cuda)
    b = Prefill(spec, policy, bounds, cl.CalibrationRef.log_k(spec.bin_count), device=cuda)
    reps = 3 if case == "repeat" else 1
    for _ in range(reps):  # the arrival ticket must be back at 0 after every call
        a.stage_minmax(u)
        a.stage_histogram_decide(u, 4096)
        b.stage_minmax(u)
        b.stage_histogram(u)
        b.stage_decide(b.n_samples(n), 4096)
        torch.cuda.synchronize()
        assert torch.equal(a.counts, b.counts)
        assert torch.equal(a.decision_buf, b.decision_buf)
        assert torch.equal(a.range, b.range)


@pytest.mark.parametrize("stride", [4, 5, 8, 16])
@pytest.mark.parametrize("n,offset", [(1 << 20, 0), (3 * 1000 * 997 + 13, 3), (4099, 1)])
@pytest.mark.parametrize("kind", ["dynamic", "fixed", "k100"])
def test_gathered_strided_entropy_equals_full_read(cuda, stride, n, offset, kind):
    """For sample_stride >= CL_GATHER_MIN_STRIDE the single-GPU prefill gathers the sampled
    values during min/max (cl_minmax_gather_f32) and histograms only those: range, counts
    and the decision record equal the all-elements strided path bit for bit (Dynamic and
    Fixed range, power-of-two and other K)."""
    g = torch.Generator().manual_seed(n % 97 + stride)
    buf = torch.randn(n + offset, generator=g).to(cuda)
    uf = buf[offset:]
    spec = {"dynamic": cl.HistogramSpec(sample_stride=stride),
            "fixed": cl.HistogramSpec(sample_stride=stride, range_mode=cl.RangeMode.Fixed,
                                      fixed_lo=-1.5, fixed_hi=2.0),
            "k100": cl.HistogramSpec(sample_stride=stride, bin_count=100)}[kind]
    a, b = Prefill(spec, device=cuda), Prefill(spec, device=cuda)
    a.stage_init()
    a.stage_minmax(uf, init=False)
    a.stage_histogram_decide(uf, 2048, zero=False)
    b.stage_init()
    b.stage_entropy(uf, 2048)
    torch.cuda.synchronize()
    assert torch.equal(a.range, b.range)
    assert torch.equal(a.counts, b.counts)
    assert torch.equal(a.decision_buf, b.decision_buf)
    assert int(b.counts.sum()) == (n + stride - 1) // stride


def test_gathered_prefill_matches_oracle_decision(cuda, port):
    """The whole strided prefill (gathered entropy -> decision -> scan) against the C
    oracle's strided histogram and rule."""
    x = mamba_inputs(31, 2, 64, 16, 1024)
    d = dev(x, cuda)
    spec = cl.HistogramSpec(sample_stride=8)
    pf = Prefill(spec, device=cuda)
    pf(d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"])
    torch.cuda.synchronize()
    ref, *_ = port.histogram(x["u"].reshape(-1), 256, 1e-8, 8)
    assert (pf.counts.cpu().numpy().astype(np.uint64) == ref).all()


def test_bc_relayout_handoff_is_per_capture(cuda):
    """The init launch's B / C re-layout (cl_prefill_init_prepare_f32) is consumed by the
    scan only within one capture: a scan graph captured separately from its init graph
    re-lays B / C itself, so replaying another prefill's graph in between cannot leave it
    reading a stale re-layout."""
    xa = dev(mamba_inputs(50, 2, 64, 16, 1024), cuda)
    xb = dev(mamba_inputs(51, 2, 64, 16, 1024), cuda)
    pa, pb = Prefill(cl.HistogramSpec(), device=cuda), Prefill(cl.HistogramSpec(), device=cuda)
    pa.scan_variant = pb.scan_variant = "chained"
    args_a = (xa["u"], xa["delta"], xa["A"], xa["B"], xa["C"], xa["D"], xa["z"], xa["delta_bias"])
    args_b = (xb["u"], xb["delta"], xb["A"], xb["B"], xb["C"], xb["D"], xb["z"], xb["delta_bias"])
    ref_a = pa(*args_a).out.clone()
    ref_b = pb(*args_b).out.clone()
    torch.cuda.synchronize()
    out_a, out_b = torch.empty_like(ref_a), torch.empty_like(ref_b)
    g_init, g_scan, g_b = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_init):
        pa.stage_init(args_a[:5])
        pa.stage_entropy(xa["u"].reshape(-1), 1024)
    with torch.cuda.graph(g_scan):
        pa.stage_scan(*args_a, True, out_a, variant="chained")
    with torch.cuda.graph(g_b):
        pb(*args_b, out=out_b)
    for _ in range(3):
        g_init.replay()
        g_b.replay()      # another prefill's re-layout lands in the shared captured scratch
        g_scan.replay()
        torch.cuda.synchronize()
        assert torch.equal(out_a, ref_a)
        assert torch.equal(out_b, ref_b)
