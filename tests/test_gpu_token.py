"""GPU: token_entropy (entropy.hpp:180-210) and the TokenHistogram policy on the device
(SURVEY.md 8(f) #2).

Pinned to the reference build: tests/golden token cases (make_golden.py runs the
reference's own token_entropy), the reference unit test test_entropy.cpp:267-288, and the
oracle port on random shapes.  Per-position entropies use the device's fp64 log, so
raw_nats agrees to ~1e-15 relative; sample counts and decisions are exact."""
import math

import numpy as np
import pytest
import torch

import paper_2604_10597_b200 as cl
from oracle import oracle as O
from paper_2604_10597_b200.mamba1 import Prefill
from tests._helpers import mamba_inputs

pytestmark = pytest.mark.gpu

ROUTED = [128, 256, 512, 1024, 2048]


def spec_of(k, stride=1, fixed=None, eps=1e-8):
    if fixed:
        return cl.HistogramSpec(k, eps, cl.RangeMode.Fixed, fixed[0], fixed[1], stride)
    return cl.HistogramSpec(k, eps, cl.RangeMode.Dynamic, 0.0, 0.0, stride)


def golden_values(port, m):
    return port.generate(m["dist"], m["channels"] * m["length"], m["seed"],
                         **m["kwargs"]).reshape(m["channels"], m["length"])


def expected_chunk(port, raw, c_min, c_max, h_ref, buckets=ROUTED):
    """TokenHistogram = from_rule(token raw) (chunk.hpp:311-315), i.e. Full's rule + snap."""
    p = O.Policy()
    p.kind = O.POL_FULL
    p.n_buckets = len(buckets)
    for i, b in enumerate(buckets):
        p.buckets[i] = b
    f = O.Features(1, raw, 0, 0.0, 0, 0)
    return port.schedule(p, f, c_min, c_max, h_ref)[0]


def test_golden_host_path(cuda, golden, port):
    meta, _ = golden
    for name, m in meta["token"].items():
        v = golden_values(port, m)
        assert port.fnv1a64(v.reshape(-1)) == m["values_fnv"], name
        e = cl.token_entropy(cl.ActivationTensor(v.reshape(-1), list(v.shape)),
                             spec_of(m["k"], m["stride"], m["fixed"]))
        assert e.sample_count == m["sample_count"], name
        assert e.raw_nats == pytest.approx(m["raw_nats"], rel=1e-13, abs=1e-15), name
        assert e.normalized == pytest.approx(m["normalized"], rel=1e-13, abs=1e-15), name


def test_golden_device_f32_prefill(cuda, golden, port):
    """The prefill with a TokenHistogram policy on fp32 u of shape (1, channels, L)."""
    meta, _ = golden
    for name, m in meta["token"].items():
        v32 = golden_values(port, m).astype(np.float32)
        ch, L = v32.shape
        x = mamba_inputs(5, 1, ch, 16, L)
        d = {k: torch.from_numpy(np.ascontiguousarray(a)).to(cuda) for k, a in x.items()}
        u = torch.from_numpy(v32.reshape(1, ch, L)).to(cuda)
        policy = cl.SchedulerPolicy(cl.TokenHistogramPolicy(), ROUTED)
        pf = Prefill(spec_of(m["k"], m["stride"], m["fixed"]), policy, cl.ChunkBounds(128, 2048),
                     cl.CalibrationRef.log_k(m["k"]), device=cuda)
        pf(u, d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"], True)
        rec = pf.decision()
        assert rec.entropy.raw_nats == pytest.approx(m["raw_nats_f32"], rel=1e-13), name
        assert rec.entropy.sample_count == m["sample_count"], name
        assert rec.decision.source_policy == "token_histogram"
        assert rec.decision.chunk == expected_chunk(port, rec.entropy.raw_nats, 128, 2048,
                                                    math.log(m["k"]))


@pytest.mark.parametrize("ch,L,k,stride,fixed", [(33, 1, 256, 1, None), (65, 19, 64, 2, None),
                                                  (1000, 9, 4096, 7, None), (7, 130, 16, 1, (0., .5)),
                                                  (2048, 8, 256, 1, None),
                                                  # fp32 lane-per-position kernels (L % 4 == 0,
                                                  # K <= 256): ragged position tiles, strides,
                                                  # fixed range, many channel splits
                                                  (4096, 100, 256, 3, None),
                                                  (3000, 36, 64, 1, (-1.0, 1.0)),
                                                  (20000, 44, 256, 8, None),
                                                  (513, 1028, 128, 1, None)])
def test_random_shapes_vs_port(cuda, port, ch, L, k, stride, fixed):
    v = np.random.default_rng(ch * L).standard_normal((ch, L))
    raw, norm, n = port.token_entropy(v, k, 1e-8, stride, fixed)
    e = cl.token_entropy(cl.ActivationTensor(v.reshape(-1), [ch, L]), spec_of(k, stride, fixed))
    assert e.sample_count == n
    assert e.raw_nats == pytest.approx(raw, rel=1e-13, abs=1e-15)
    # the device f32 path sees the same values rounded to fp32
    v32 = v.astype(np.float32)
    raw32, _, _ = port.token_entropy(v32.astype(np.float64), k, 1e-8, stride, fixed)
    out = torch.zeros(4, dtype=torch.float64, device=cuda)
    ctx = cl.Context.get(cuda.index)
    import ctypes as C
    cs = spec_of(k, stride, fixed).to_c()
    ctx.call("cl_token_entropy_f32", torch.from_numpy(v32).to(cuda).data_ptr(), ch, L,
             C.byref(cs), out.data_ptr(), torch.cuda.current_stream(cuda).cuda_stream)
    o = out.cpu().numpy()
    assert o[0] == pytest.approx(raw32, rel=1e-13, abs=1e-15) and o[2] == n and o[3] == 0.0


def test_reference_unit_test(cuda):
    """test_entropy.cpp:267-288."""
    s = spec_of(16, eps=1e-12)
    e = cl.token_entropy(cl.ActivationTensor(np.array([1., 2., 3., 1., 2., 3.]), [2, 3]), s)
    assert abs(e.raw_nats) <= 1e-9
    m = cl.token_entropy(cl.ActivationTensor(np.array([0., 5., 1., 5.]), [2, 2]), s)
    assert m.raw_nats == pytest.approx(0.5 * math.log(2.0), abs=1e-6)
    with pytest.raises(cl.InvalidInput, match="token entropy needs a"):
        cl.token_entropy(cl.ActivationTensor(np.array([1., 2.]), [2]), s)


def test_errors_and_precedence(cuda):
    v = np.arange(12, dtype=np.float64)
    v[5] = np.nan
    t = cl.ActivationTensor(v, [3, 4])
    # validate_tensor (finite check) precedes the spec check (entropy.hpp:182-183)
    with pytest.raises(cl.InvalidInput, match="non-finite input"):
        cl.token_entropy(t, spec_of(1))
    with pytest.raises(cl.InvalidInput, match="non-finite input"):
        cl.compute_histogram(t, spec_of(1))
    # the span overload only visits sampled values (entropy.hpp:108-111)
    h = cl.compute_histogram(v, spec_of(8, stride=2))
    assert h.sample_count == 6
    with pytest.raises(cl.InvalidInput, match="non-finite input"):
        cl.compute_histogram(v, spec_of(8, stride=1))
    ok = cl.ActivationTensor(np.arange(12, dtype=np.float64), [3, 4])
    with pytest.raises(cl.InvalidInput, match="degenerate spec"):
        cl.token_entropy(ok, spec_of(1))
    with pytest.raises(cl.InvalidInput, match="bin_count <= 4096"):
        cl.token_entropy(ok, spec_of(8192))


def test_device_deferred_errors(cuda):
    x = mamba_inputs(6, 1, 32, 16, 64)
    d = {k: torch.from_numpy(np.ascontiguousarray(a)).to(cuda) for k, a in x.items()}
    policy = cl.SchedulerPolicy(cl.TokenHistogramPolicy(), ROUTED)
    pf = Prefill(cl.HistogramSpec(), policy, cl.ChunkBounds(128, 2048), device=cuda)
    u = d["u"].clone()
    u[0, 3, 7] = float("inf")
    pf(u, d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"], True)
    with pytest.raises(cl.InvalidInput, match="non-finite input"):
        pf.decision()
    # constant channels per position -> raw = -eps-level < 0 (Finding 7): rule rejects it
    u = torch.ones_like(d["u"])
    pf(u, d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"], True)
    with pytest.raises(cl.InvalidInput, match="signal must be >= 0"):
        pf.decision()


def test_guarded_token_policy(cuda, port):
    x = mamba_inputs(7, 2, 96, 16, 256)
    d = {k: torch.from_numpy(np.ascontiguousarray(a)).to(cuda) for k, a in x.items()}
    inner = cl.SchedulerPolicy(cl.TokenHistogramPolicy(), ROUTED)
    policy = cl.SchedulerPolicy(cl.GuardedPolicy(inner, 512, 2), ROUTED)
    pf = Prefill(cl.HistogramSpec(), policy, cl.ChunkBounds(128, 2048), device=cuda)
    pf(d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"], True)
    rec = pf.decision()
    raw, _, _ = port.token_entropy(x["u"].reshape(-1, 256).astype(np.float64))
    c_inner = expected_chunk(port, raw, 128, 2048, math.log(256))
    delta = abs(int(math.log2(c_inner)) - int(math.log2(512)))
    assert rec.decision.chunk == (c_inner if delta >= 2 else 512)
    assert rec.decision.source_policy in ("guarded[token_histogram]", "guarded[fallback]")


def test_host_schedule_token_feature(cuda):
    """Scheduler::decide for TokenHistogram needs ScheduleFeatures::token_entropy."""
    policy = cl.SchedulerPolicy(cl.TokenHistogramPolicy(), ROUTED)
    bounds, cal = cl.ChunkBounds(128, 2048), cl.CalibrationRef.log_k(256)
    with pytest.raises(cl.InvalidInput, match="missing feature: token_entropy"):
        cl.schedule(policy, cl.ScheduleFeatures(), bounds, cal)
    d = cl.schedule(policy, cl.ScheduleFeatures(token_entropy=cl.EntropyEstimate(5.0)), bounds,
                    cal)
    assert d.chunk == 2048 and d.source_policy == "token_histogram"


def test_sharded_stages_world1_equal_one_call(cuda):
    """The staged token path behind ShardedPrefill (the multi-GPU protocol's device
    stages, collectives skipped at world 1) equals the one-call path exactly."""
    from paper_2604_10597_b200.sharded import ShardedPrefill, plan_rows
    x = mamba_inputs(8, 2, 160, 16, 96)
    d = {k: torch.from_numpy(np.ascontiguousarray(a)).to(cuda) for k, a in x.items()}
    policy = cl.SchedulerPolicy(cl.TokenHistogramPolicy(), ROUTED)
    for stride in (1, 3):
        spec = cl.HistogramSpec(sample_stride=stride)
        pf1 = Prefill(spec, policy, cl.ChunkBounds(128, 2048), device=cuda)
        sp = ShardedPrefill(pf1, plan_rows(2, 160, 96, 0, 1))
        out1 = sp(d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"])
        r1 = pf1.decision()
        pf2 = Prefill(spec, policy, cl.ChunkBounds(128, 2048), device=cuda)
        res2 = pf2(d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"])
        r2 = pf2.decision()
        assert r1.entropy.raw_nats == r2.entropy.raw_nats
        assert r1.entropy.sample_count == r2.entropy.sample_count
        assert r1.decision.chunk == r2.decision.chunk
        assert torch.equal(out1, res2.out)
