"""GPU: K-bin histogram + entropy (entropy.hpp) through the C-ABI vs the reference.

Counts must be bit-exact (fp64 drop-in path and fp32 device path); entropy is
computed on the device in fp64 in bin order, so raw_nats may differ from glibc's
log only in the last ulps (checked at 1e-13 relative).  Re-expresses
test_entropy.cpp cases (cited per test) against the drop-in API.
"""
import math

import numpy as np
import pytest
import torch

import paper_2604_10597_b200 as cl
from paper_2604_10597_b200.mamba1 import Prefill

pytestmark = pytest.mark.gpu

HIST_CASES = ["uniform", "normal", "normal_s8", "laplace", "sparse10", "sparse02", "normal_k64",
              "normal_c1", "uniform_k512", "normal_s3"]


def _gen(port, m):
    return port.generate(m["dist"], m["n"], m["seed"], **m["kwargs"])


def _device_counts(cuda, v32, k, stride, g0=0):
    """fp32 device path: minmax -> histogram stages (the prefill hot path)."""
    spec = cl.HistogramSpec(bin_count=k, sample_stride=stride)
    pf = Prefill(spec, device=cuda)
    t = torch.from_numpy(np.ascontiguousarray(v32)).to(cuda)
    pf.stage_minmax(t, g0)
    pf.stage_histogram(t, g0)
    torch.cuda.synchronize()
    rng = pf.range.cpu().numpy()
    return pf.counts.cpu().numpy().astype(np.uint64), -rng[0], rng[1], rng[2]


@pytest.mark.parametrize("name", HIST_CASES)
def test_dropin_histogram_golden(cuda, port, golden, name):
    meta, arrays = golden
    m = meta["hist"][name]
    v = _gen(port, m)
    spec = cl.HistogramSpec(bin_count=m["k"], sample_stride=m["stride"])
    h = cl.compute_histogram(cl.ActivationTensor(v, [v.size]), spec)
    assert (h.counts == arrays[f"{name}_counts"]).all()
    assert h.lo == m["lo"] and h.hi == m["hi"] and h.sample_count == m["sample_count"]
    e = cl.estimate_entropy(h, 1e-8)
    assert e.raw_nats == pytest.approx(m["raw_nats"], rel=1e-13, abs=0)
    assert e.normalized == pytest.approx(m["normalized"], rel=1e-13, abs=0)


@pytest.mark.parametrize("name", HIST_CASES)
def test_device_f32_histogram_golden(cuda, port, golden, name):
    meta, arrays = golden
    m = meta["hist"][name]
    v32 = _gen(port, m).astype(np.float32)
    counts, lo, hi, bad = _device_counts(cuda, v32, m["k"], m["stride"])
    assert bad == 0.0
    assert (counts == arrays[f"{name}_counts_f32"]).all()
    assert lo == m["lo_f32"] and hi == m["hi_f32"]


@pytest.mark.parametrize("name", HIST_CASES)
def test_device_decision_golden(cuda, port, golden, name):
    """minmax -> hist -> device entropy -> rule: chunk bit-exact vs the reference."""
    meta, _ = golden
    m = meta["hist"][name]
    v32 = torch.from_numpy(_gen(port, m).astype(np.float32)).to(cuda)
    k = m["k"]
    for key, (bounds, cal) in {
            "logk_32_512": (cl.ChunkBounds(32, 512), cl.CalibrationRef.log_k(k)),
            "legacy8_32_512": (cl.ChunkBounds(32, 512), cl.CalibrationRef.legacy()),
            "logk_128_2048": (cl.ChunkBounds(128, 2048), cl.CalibrationRef.log_k(k))}.items():
        pf = Prefill(cl.HistogramSpec(bin_count=k, sample_stride=m["stride"]), None, bounds, cal,
                     device=cuda)
        pf.stage_minmax(v32)
        pf.stage_histogram(v32)
        pf.stage_decide(pf.n_samples(v32.numel()), 4096)
        rec = pf.decision()
        assert rec.entropy.raw_nats == pytest.approx(m["raw_nats_f32"], rel=1e-13, abs=0)
        if rec.decision.margin > 1e-9:  # knife-edge rule (hard part 6)
            assert rec.decision.chunk == m["chunks_f32"][key], key
        assert rec.lo == m["lo_f32"] and rec.hi == m["hi_f32"]
        assert rec.entropy.sample_count == m["sample_count"]


def test_degenerate_range_bin0(cuda):
    """test_entropy.cpp:51-58."""
    h = cl.compute_histogram(cl.ActivationTensor(np.full(1000, 3.0), [1000]),
                             cl.HistogramSpec(bin_count=256))
    assert h.masses[0] == 1.0 and (h.masses[1:] == 0).all() and h.sample_count == 1000
    counts, *_ = _device_counts(cuda, np.full(5000, 3.0, np.float32), 256, 1)
    assert counts[0] == 5000 and counts[1:].sum() == 0


def test_two_point_symmetry(cuda):
    """test_entropy.cpp:60-66."""
    h = cl.compute_histogram(cl.ActivationTensor(np.array([0.0, 1.0]), [2]),
                             cl.HistogramSpec(bin_count=2))
    assert list(h.masses) == [0.5, 0.5]


def test_error_paths(cuda):
    """test_entropy.cpp:86-99 + validate_spec messages."""
    spec = cl.HistogramSpec()
    with pytest.raises(cl.InvalidInput, match="^no samples$"):
        cl.compute_histogram(cl.ActivationTensor(np.array([]), [0 + 0]), spec)
    with pytest.raises(cl.InvalidInput, match="^non-finite input$"):
        cl.compute_histogram(cl.ActivationTensor(np.array([1.0, np.nan]), [2]), spec)
    with pytest.raises(cl.InvalidInput, match="^degenerate spec$"):
        cl.compute_histogram(cl.ActivationTensor(np.array([1.0]), [1]),
                             cl.HistogramSpec(bin_count=1))
    with pytest.raises(cl.InvalidInput, match="^epsilon must be positive$"):
        cl.compute_histogram(np.array([1.0]), cl.HistogramSpec(epsilon=0.0))
    with pytest.raises(cl.InvalidInput, match="^fixed range requires lo < hi$"):
        cl.compute_histogram(np.array([1.0]), cl.HistogramSpec(range_mode=cl.RangeMode.Fixed,
                                                               fixed_lo=1.0, fixed_hi=1.0))
    with pytest.raises(cl.InvalidInput, match="^stride must be >= 1$"):
        cl.compute_histogram(np.array([1.0]), cl.HistogramSpec(sample_stride=0))
    h = cl.compute_histogram(cl.ActivationTensor(np.array([5.0, 1.0, 2.0]), [3]),
                             cl.HistogramSpec(sample_stride=10))
    assert h.sample_count == 1
    with pytest.raises(cl.InvalidInput, match="^shape/value count mismatch$"):
        cl.compute_histogram(cl.ActivationTensor(np.array([1.0, 2.0]), [3]), spec)
    # non-finite on the fp32 device path is a deferred device error
    v = np.random.default_rng(0).standard_normal(10000).astype(np.float32)
    v[7777] = np.inf
    _, _, _, bad = _device_counts(cuda, v, 256, 1)
    assert bad == 1.0


def test_single_bin_entropy(cuda):
    """test_entropy.cpp:101-109."""
    m = np.zeros(256)
    m[0] = 1.0
    e = cl.estimate_entropy(cl.Histogram(masses=m, sample_count=1000), 1e-8)
    assert abs(e.raw_nats) <= 1e-7 and abs(e.normalized) <= 1e-7
    with pytest.raises(cl.InvalidInput, match="^degenerate spec$"):
        cl.estimate_entropy(cl.Histogram(masses=np.array([1.0]), sample_count=10), 1e-8)


def test_mass_conservation_random_specs(cuda, port):
    """test_entropy.cpp:174-195, with bit-exact counts vs the oracle on both paths."""
    rng = np.random.default_rng(77)
    for _ in range(50):
        n = int(rng.integers(1, 5001))
        v = rng.laplace(0.0, 2.0, n)
        k = int(rng.integers(2, 512))
        spec = cl.HistogramSpec(bin_count=k)
        h = cl.compute_histogram(cl.ActivationTensor(v, [n]), spec)
        oc, olo, ohi, on = port.histogram(v, k)
        assert (h.counts == oc).all() and h.lo == olo and h.hi == ohi
        assert abs(h.masses.sum() - 1.0) <= 1e-12
        e = cl.estimate_entropy(h, 1e-8)
        assert e.raw_nats <= math.log(k) + k * 1e-8 and e.raw_nats >= -k * 1e-8
        v32 = v.astype(np.float32)
        dc, dlo, dhi, _ = _device_counts(cuda, v32, k, 1)
        oc32, olo32, ohi32, _ = port.histogram(v32, k)
        assert (dc == oc32).all() and dlo == olo32 and dhi == ohi32


def test_stride_semantics(cuda, port):
    """test_entropy.cpp:197-223: stride s == manual subsample, bit-exact; plus the
    global-offset convention used by the sharded path."""
    rng = np.random.default_rng(99)
    values = rng.standard_normal(4097)
    for s in (2, 3, 8):
        a = cl.compute_histogram(cl.ActivationTensor(values, [4097]),
                                 cl.HistogramSpec(bin_count=64, sample_stride=s))
        b = cl.compute_histogram(cl.ActivationTensor(values[::s].copy(), [len(values[::s])]),
                                 cl.HistogramSpec(bin_count=64))
        assert (a.masses == b.masses).all() and a.lo == b.lo and a.hi == b.hi
        assert a.sample_count == b.sample_count
    v32 = rng.standard_normal(1 << 20).astype(np.float32)
    for s in (1, 3, 8):
        full, *_ = _device_counts(cuda, v32, 256, s)
        oc, *_ = port.histogram(v32, 256, 1e-8, s)
        assert (full == oc).all()


def test_permutation_invariance(cuda, port):
    """test_entropy.cpp:225-240 (Student-t draws)."""
    r = port  # noqa: F841
    rng = np.random.default_rng(123)
    values = rng.standard_t(3, 2048)
    before = cl.compute_histogram(values, cl.HistogramSpec(bin_count=128))
    after = cl.compute_histogram(rng.permutation(values), cl.HistogramSpec(bin_count=128))
    assert (before.masses == after.masses).all()
    assert cl.estimate_entropy(before, 1e-8).raw_nats == cl.estimate_entropy(after, 1e-8).raw_nats


def test_fixed_range_clips(cuda, port):
    """test_entropy.cpp:256-265 + extreme outliers (x86 int-conversion semantics)."""
    spec = cl.HistogramSpec(bin_count=4, range_mode=cl.RangeMode.Fixed, fixed_lo=0.0,
                            fixed_hi=4.0)
    h = cl.compute_histogram(np.array([-1.0, 0.5, 3.9, 99.0]), spec)
    assert h.masses[0] == 0.5 and h.masses[3] == 0.5
    v = np.array([-1.0, 0.5, 3.9, 99.0, 1e12, -1e12, 4.0, 0.0])
    h = cl.compute_histogram(v, spec)
    oc, *_ = port.histogram(v, 4, 1e-8, 1, fixed=(0.0, 4.0))
    assert (h.counts == oc).all()
    v32 = np.concatenate([v, np.random.default_rng(1).uniform(-2, 6, 10000)]).astype(np.float32)
    pf = Prefill(spec, device=cuda)
    t = torch.from_numpy(v32).to(cuda)
    pf.stage_minmax(t)
    pf.stage_histogram(t)
    oc, *_ = port.histogram(v32, 4, 1e-8, 1, fixed=(0.0, 4.0))
    assert (pf.counts.cpu().numpy().astype(np.uint64) == oc).all()


def test_adversarial_bin_boundaries(cuda, port):
    """fp32 values within a few ulps of every bin threshold must bin exactly as the
    reference's fp64 formula (SURVEY.md finding 5)."""
    rng = np.random.default_rng(5)
    base = rng.standard_normal(1 << 16).astype(np.float32)
    lo, hi = float(base.min()), float(base.max())
    k = 256
    edges = lo + (hi - lo) * np.arange(1, k) / k
    e32 = edges.astype(np.float32)
    neigh = [e32]
    for d in range(1, 4):
        neigh.append(np.nextafter(e32, np.float32(np.inf)))
        neigh.append(np.nextafter(e32, np.float32(-np.inf)))
        e32 = neigh[-2]
    v = np.concatenate([base] + neigh).astype(np.float32)
    rng.shuffle(v)
    for k2 in (256, 64, 200):
        dc, *_ = _device_counts(cuda, v, k2, 1)
        oc, *_ = port.histogram(v, k2)
        assert (dc == oc).all(), k2


def test_unaligned_and_tiny_inputs(cuda, port):
    """Head/tail handling of the TMA bulk-copy histogram and the vector min/max."""
    rng = np.random.default_rng(2)
    big = torch.from_numpy(rng.standard_normal(100003).astype(np.float32)).to(cuda)
    for off in (0, 1, 2, 3):
        for n in (1, 3, 4097, 100003 - off):
            t = big[off:off + n]
            spec = cl.HistogramSpec(bin_count=256)
            pf = Prefill(spec, device=cuda)
            pf.stage_minmax(t)
            pf.stage_histogram(t)
            oc, olo, ohi, _ = port.histogram(t.cpu().numpy(), 256)
            assert (pf.counts.cpu().numpy().astype(np.uint64) == oc).all(), (off, n)
            r = pf.range.cpu().numpy()
            assert -r[0] == olo and r[1] == ohi


def test_repeated_runs_deterministic(cuda, port, golden):
    """Counts must be identical over repeated launches (catches cross-warp counter races,
    e.g. padding samples of a partial chunk addressing another warp's rows)."""
    meta, arrays = golden
    m = meta["hist"]["uniform"]
    v32 = _gen(port, m).astype(np.float32)
    ref = arrays["uniform_counts_f32"]
    for _ in range(20):
        counts, *_ = _device_counts(cuda, v32, 256, 1)
        assert (counts == ref).all()


def test_strided_unsampled_outliers(cuda, port):
    """Unsampled elements far outside the sampled range must not touch any counter."""
    rng = np.random.default_rng(9)
    v = rng.standard_normal(1 << 18).astype(np.float32)
    for s in (2, 3, 8):
        w = v.copy()
        idx = np.arange(w.size)
        w[idx % s != 0] *= 1e6  # only unsampled positions get huge magnitudes
        for _ in range(3):
            counts, lo, hi, _ = _device_counts(cuda, w, 256, s)
            oc, olo, ohi, _ = port.histogram(w, 256, 1e-8, s)
            assert (counts == oc).all() and lo == olo and hi == ohi


@pytest.mark.parametrize("stride", [1, 3, 8])
def test_counter_flush_no_overflow(cuda, port, stride):
    """Lane counters are narrow (8-bit, flushed every 15 chunks): inputs large enough for
    many flushes per CTA, with almost every sample in one bin, must still count exactly
    (full-chunk hot path at stride 1, the general / sparse paths at strides 3 and 8)."""
    n = (1 << 26) + 12345  # ~55 chunks per CTA at the default geometry, ragged tail
    v = np.full(n, 0.25, np.float32)
    rng = np.random.default_rng(stride)
    idx = rng.integers(0, n, 4096)
    v[idx] = rng.uniform(-1.0, 1.0, idx.size).astype(np.float32)
    counts, lo, hi, _ = _device_counts(cuda, v, 256, stride)
    oc, olo, ohi, on = port.histogram(v, 256, 1e-8, stride)
    assert lo == olo and hi == ohi
    assert (counts == oc).all() and int(counts.sum()) == on


def test_counter_flush_degenerate_range(cuda):
    """Constant input (degenerate range, everything in bin 0) at 64M samples."""
    n = 1 << 26
    counts, *_ = _device_counts(cuda, np.full(n, -2.5, np.float32), 256, 1)
    assert counts[0] == n and counts[1:].sum() == 0
