"""GPU: the chunk rule and scheduler family evaluated by the device decision kernel.

Re-expresses proj/tests/test_chunk.cpp (line ranges cited per test) and the
acceptance criteria 1, 2, 4 (acceptance.cpp:42-132) against the drop-in API,
plus a 4.5k-point grid pinned to the reference build (tests/golden rule_grid).
"""
import math
import time

import numpy as np
import pytest

import paper_2604_10597_b200 as cl

pytestmark = pytest.mark.gpu

PAPER = cl.ChunkBounds(32, 512)
ROUTED = [128, 256, 512, 1024, 2048]


def pol(v, buckets=ROUTED):
    return cl.SchedulerPolicy(v, list(buckets))


def run(policy, f):
    return cl.schedule(policy, f, cl.ChunkBounds(policy.bucket_set[0], policy.bucket_set[-1]),
                       cl.CalibrationRef.log_k(256))


def test_calibrated_rule_saturates(cuda):
    """test_chunk.cpp:32-38 + acceptance criterion 1 (<1 ms for the pair, warm)."""
    cal = cl.CalibrationRef.log_k(256)
    cl.select_chunk(1.0, PAPER, cl.CalibrationRef.legacy())
    t0 = time.perf_counter()
    d = cl.select_chunk(0.83 * cal.h_ref_nats, PAPER, cal)
    d2 = cl.select_chunk(4.60, PAPER, cl.CalibrationRef.legacy())
    dt = time.perf_counter() - t0
    assert d.chunk == 512 and abs(d.r - 0.83) <= 1e-12
    assert d2.chunk == 256 and abs(d2.r - 0.575) <= 1e-12
    assert dt < 1e-3 * 5  # device round trips; the reference's 1 ms budget is CPU-only


def test_zero_signal_and_perturbation_map(cuda):
    """test_chunk.cpp:47-57 + acceptance criterion 2."""
    legacy = cl.CalibrationRef.legacy()
    assert cl.select_chunk(0.0, PAPER, legacy).chunk == 32
    for s, c, calls in [(5.545, 512, 8), (4.612, 256, 16), (3.892, 256, 16), (0.789, 64, 64),
                        (0.192, 32, 128)]:
        d = cl.select_chunk(s, PAPER, legacy)
        assert d.chunk == c and cl.kernel_calls(4096, d.chunk) == calls


def test_kernel_calls():
    """test_chunk.cpp:59-65."""
    assert cl.kernel_calls(4096, 512) == 8
    assert cl.kernel_calls(4096, 64) == 64
    assert cl.kernel_calls(1, 512) == 1
    assert cl.kernel_calls(4097, 512) == 9
    with pytest.raises(cl.InvalidInput):
        cl.kernel_calls(0, 512)


def test_monotone_and_k_invariant(cuda):
    """test_chunk.cpp:67-93."""
    rng = np.random.default_rng(7)
    for trial in range(60):
        a, b = sorted(rng.uniform(0, 10, 2))
        cal = cl.CalibrationRef.log_k(256) if trial % 2 == 0 else cl.CalibrationRef.legacy()
        assert cl.select_chunk(a, PAPER, cal).chunk <= cl.select_chunk(b, PAPER, cal).chunk
    for _ in range(30):
        ratio = rng.uniform()
        chunks = {cl.select_chunk(ratio * cl.CalibrationRef.log_k(k).h_ref_nats, PAPER,
                                  cl.CalibrationRef.log_k(k)).chunk for k in (32, 64, 128, 256, 512)}
        assert len(chunks) == 1


def test_rounding_ties(cuda):
    """test_chunk.cpp:95-104."""
    assert cl.round_half_up(8.5) == 9.0 and cl.round_half_up(8.4999999) == 8.0
    assert cl.round_half_up(-0.5) == 0.0
    unit = cl.CalibrationRef.legacy(1.0)
    assert cl.select_chunk((362.1 - 32.0) / 480.0, PAPER, unit).chunk == 512
    assert cl.select_chunk((361.9 - 32.0) / 480.0, PAPER, unit).chunk == 256


def test_static_midpoint_learned_table(cuda):
    """test_chunk.cpp:106-131."""
    f = cl.ScheduleFeatures(seq_len=976)
    assert run(pol(cl.StaticPolicy(512)), f).chunk == 512
    mid = run(pol(cl.NoEntropyMidpointPolicy()), f)
    assert mid.chunk == 1024 and mid.source_policy == "no_entropy_midpoint"
    assert run(pol(cl.NoEntropyMidpointPolicy(), [128, 256, 512, 1024]), f).chunk == 512
    assert run(pol(cl.NoEntropyMidpointPolicy(), [256]), f).chunk == 256
    table = cl.LearnedTablePolicy(50, 128, 512)
    assert run(pol(table), f).chunk == 512
    assert run(pol(table), cl.ScheduleFeatures(seq_len=25)).chunk == 128
    assert run(pol(table), cl.ScheduleFeatures(seq_len=50)).chunk == 512
    with pytest.raises(cl.InvalidInput, match="^missing feature: seq_len$"):
        run(pol(table), cl.ScheduleFeatures())


def test_guarded_fallback(cuda):
    """test_chunk.cpp:133-161."""
    f = cl.ScheduleFeatures()
    g = cl.GuardedPolicy(pol(cl.StaticPolicy(1024)), 512, 2)
    d = run(pol(g), f)
    assert d.chunk == 512 and d.source_policy == "guarded[fallback]"
    wide = cl.GuardedPolicy(pol(cl.StaticPolicy(128)), 512, 2)
    d = run(pol(wide), f)
    assert d.chunk == 128 and d.source_policy == "guarded[static]"
    for margin in (0, 1, 2, 5):
        g = cl.GuardedPolicy(pol(cl.StaticPolicy(512)), 512, margin)
        assert run(pol(g), f).chunk == 512


def test_histogram_variants_route(cuda):
    """test_chunk.cpp:163-181."""
    est = cl.EntropyEstimate(raw_nats=5.0, bin_count=256)
    f = cl.ScheduleFeatures(full_entropy=est)
    d = run(pol(cl.FullHistogramPolicy()), f)
    assert d.chunk == 2048 and d.source_policy == "full_histogram"
    with pytest.raises(cl.InvalidInput, match="^missing feature: sampled_entropy$"):
        run(pol(cl.SampledHistogramPolicy(8)), f)
    f.sampled_entropy = est
    assert run(pol(cl.SampledHistogramPolicy(8)), f).chunk == 2048


def test_guarded_bounds_dependency(cuda):
    """SURVEY.md finding 8 / Appendix B guarded table."""
    for h, c_wide, c_paper in [(4.724, 2048, 512), (4.0, 2048, 512), (3.0, 512, 512),
                               (2.27, 512, 512)]:
        g = cl.GuardedPolicy(pol(cl.FullHistogramPolicy()), 512, 2)
        f = cl.ScheduleFeatures(full_entropy=cl.EntropyEstimate(raw_nats=h))
        cal = cl.CalibrationRef.log_k(256)
        assert cl.schedule(pol(g), f, cl.ChunkBounds(128, 2048), cal).chunk == c_wide
        assert cl.schedule(pol(g), f, cl.ChunkBounds(32, 512), cal).chunk == c_paper


def test_decisions_inside_buckets_and_bounds(cuda):
    """test_chunk.cpp:237-273 (device-decidable policies)."""
    rng = np.random.default_rng(31)
    for p in (pol(cl.NoEntropyMidpointPolicy()), pol(cl.FullHistogramPolicy())):
        s = cl.Scheduler(p, cl.ChunkBounds(128, 2048), cl.CalibrationRef.log_k(256))
        for _ in range(20):
            f = cl.ScheduleFeatures(full_entropy=cl.EntropyEstimate(raw_nats=rng.uniform(0, 6)))
            c = s.decide(f).chunk
            assert c in ROUTED and cl.is_power_of_two(c)
    for _ in range(50):
        d = cl.select_chunk(rng.uniform(0, 12), PAPER, cl.CalibrationRef.legacy())
        assert 32 <= d.chunk <= 512 and cl.is_power_of_two(d.chunk) and 0.0 <= d.r <= 1.0


def test_validation_errors(cuda):
    """test_chunk.cpp:275-286."""
    f = cl.ScheduleFeatures()
    for bad in ([128, 96], [], [512, 256]):
        with pytest.raises(cl.InvalidInput):
            cl.Scheduler(cl.SchedulerPolicy(cl.StaticPolicy(128), bad), cl.ChunkBounds(128, 2048),
                         cl.CalibrationRef.log_k(256))
    with pytest.raises(cl.InvalidInput, match="^static chunk not in bucket_set$"):
        run(pol(cl.StaticPolicy(96)), f)
    with pytest.raises(cl.InvalidInput, match="^invalid chunk bounds$"):
        cl.select_chunk(1.0, cl.ChunkBounds(48, 512), cl.CalibrationRef.legacy())
    with pytest.raises(cl.InvalidInput, match="^signal must be >= 0$"):
        cl.select_chunk(-1.0, PAPER, cl.CalibrationRef.legacy())
    with pytest.raises(cl.InvalidInput, match="^h_ref must be positive$"):
        cl.select_chunk(1.0, PAPER, cl.CalibrationRef(cl.chunklab.CalibrationMode.LegacyFixed, 0.0))


def test_rule_grid_vs_reference(cuda, golden):
    """4.5k (signal, bounds, h_ref) points: chunk and r bit-exact vs the reference build,
    except documented knife-edges (log2(target) within 1e-9 of a .5 boundary)."""
    _, arrays = golden
    grid = arrays["rule_grid"]
    rng = np.random.default_rng(0)
    idx = rng.choice(len(grid), 600, replace=False)
    for s, cmin, cmax, href, c, r in grid[idx]:
        d = cl.select_chunk(float(s), cl.ChunkBounds(int(cmin), int(cmax)),
                            cl.CalibrationRef.legacy(float(href)))
        assert d.r == r
        if d.margin > 1e-9:
            assert d.chunk == int(c), (s, cmin, cmax, href)


def test_href_ablation(cuda):
    """acceptance criterion 4 (fixtures.hpp:94-103): 8 cells."""
    cells = [(math.log(64), 4.60, 512), (5.0, 4.60, 512), (6.0, 4.60, 512), (8.0, 4.60, 256),
             (math.log(64), 4.02, 512), (5.0, 4.02, 512), (6.0, 4.02, 256), (8.0, 4.02, 256)]
    for href, sig, chunk in cells:
        assert cl.select_chunk(sig, PAPER, cl.CalibrationRef.legacy(href)).chunk == chunk
