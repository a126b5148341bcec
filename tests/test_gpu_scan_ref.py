"""GPU: fp64 reference-mode recurrence (scan.hpp) must be BIT-IDENTICAL to the
reference.  Re-expresses proj/tests/test_scan.cpp and acceptance criterion 5."""
import time

import numpy as np
import pytest

import paper_2604_10597_b200 as cl

pytestmark = pytest.mark.gpu


def params(port, seed, D, N, L, tv=True):
    p = port.random_scan_params(seed, D, N, L, tv)
    return cl.ScanParams(D, N, L, p["a"], p["b"], p["c"], p["d"], p["x"])


@pytest.mark.parametrize("key", ["scan_2026_64_16_4096_1", "scan_42_16_8_1000_1",
                                 "scan_9_8_4_64_0", "scan_1_8_4_64_1", "scan_7_4_4_128_1"])
def test_golden_bit_exact(cuda, port, golden, key):
    meta, arrays = golden
    m = meta["scan"][key]
    p = params(port, m["seed"], m["D"], m["N"], m["L"], m["tv"])
    out, st = cl.scan_sequential(p, cl.ScanState())
    assert port.fnv1a64(out.y) == m["y_fnv"]
    assert port.fnv1a64(st.h) == m["h_fnv"]
    assert (st.h == arrays[key + "_h"]).all()


def test_memoryless_limit(cuda):
    """test_scan.cpp:42-62."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal(15)
    p = cl.ScanParams(3, 2, 5, np.zeros(6), np.array([0.5, -1.5]), np.array([2.0, 1.0]),
                      np.zeros(3), x)
    out, _ = cl.scan_sequential(p, cl.ScanState())
    gain = 2.0 * 0.5 + 1.0 * -1.5
    assert np.allclose(out.y, gain * x, atol=1e-15, rtol=0)


def test_prefix_sum_identity(cuda):
    """test_scan.cpp:64-80."""
    p = cl.ScanParams(2, 1, 16, np.ones(2), np.array([1.0]), np.array([1.0]), np.zeros(2),
                      np.ones(32))
    out, st = cl.scan_sequential(p, cl.ScanState())
    assert (out.y.reshape(2, 16) == np.arange(1, 17)).all()
    assert st.h[0] == 16.0


def test_chunked_bit_identical(cuda, port):
    """test_scan.cpp:98-118 + acceptance criterion 5 (<5 s)."""
    p = params(port, 42, 16, 8, 1000)
    ref, ref_state = cl.scan_sequential(p, cl.ScanState())
    for chunk in (4096, 1, 3, 32, 64, 128, 333):
        out, st = cl.scan_chunked(p, cl.ScanState(), chunk)
        assert (out.y == ref.y).all() and (st.h == ref_state.h).all()
    t0 = time.perf_counter()
    p = params(port, 2026, 64, 16, 4096)
    ref, ref_state = cl.scan_sequential(p, cl.ScanState())
    for chunk in (1, 32, 64, 128, 256, 512, 4096):
        out, st = cl.scan_chunked(p, cl.ScanState(), chunk)
        assert (out.y == ref.y).all() and (st.h == ref_state.h).all()
    assert time.perf_counter() - t0 < 5.0


def test_state_handoff(cuda, port):
    """test_scan.cpp:120-166."""
    p = params(port, 7, 4, 4, 128)
    ref, ref_state = cl.scan_sequential(p, cl.ScanState())
    ch, n, L = 4, 4, 128
    X = p.x.reshape(ch, L)
    for split in (1, 17, 64, 127):
        first = cl.ScanParams(ch, n, split, p.a[: split * ch * n], p.b[: split * n],
                              p.c[: split * n], p.d, X[:, :split].reshape(-1).copy())
        second = cl.ScanParams(ch, n, L - split, p.a[split * ch * n:], p.b[split * n:],
                               p.c[split * n:], p.d, X[:, split:].reshape(-1).copy())
        y1, h1 = cl.scan_sequential(first, cl.ScanState())
        y2, h2 = cl.scan_sequential(second, h1)
        assert (h2.h == ref_state.h).all()
        R = ref.y.reshape(ch, L)
        assert (y1.y.reshape(ch, split) == R[:, :split]).all()
        assert (y2.y.reshape(ch, L - split) == R[:, split:]).all()


def test_matches_oracle_random(cuda, port):
    """Independent naive loop (test_scan.cpp:82-96) via the oracle, incl. h0 and odd N."""
    rng = np.random.default_rng(11)
    for seed in (1, 2, 3):
        for N in (1, 3, 4, 16, 20):
            p = port.random_scan_params(seed, 8, N, 64, True)
            h0 = rng.standard_normal(8 * N)
            y, h = port.scan(p, h0=h0)
            out, st = cl.scan_sequential(cl.ScanParams(8, N, 64, p["a"], p["b"], p["c"], p["d"],
                                                       p["x"]), cl.ScanState(h0))
            assert (out.y == y).all() and (st.h == h).all()


def test_error_paths(cuda, port):
    """test_scan.cpp:178-191."""
    p = params(port, 1, 4, 2, 8)
    with pytest.raises(cl.InvalidInput, match="^chunk must be >= 1$"):
        cl.scan_chunked(p, cl.ScanState(), 0)
    bad = cl.ScanParams(p.channels, p.state_dim, p.seq_len, p.a, p.b, p.c, p.d, p.x[:-1])
    with pytest.raises(cl.InvalidInput, match="^shape mismatch$"):
        cl.scan_sequential(bad, cl.ScanState())
    x = p.x.copy()
    x[0] = np.inf
    nonfinite = cl.ScanParams(p.channels, p.state_dim, p.seq_len, p.a, p.b, p.c, p.d, x)
    with pytest.raises(cl.InvalidInput, match="^non-finite input$"):
        cl.scan_sequential(nonfinite, cl.ScanState())
    with pytest.raises(cl.InvalidInput, match="^shape mismatch$"):
        cl.scan_sequential(p, cl.ScanState(np.zeros(3)))
