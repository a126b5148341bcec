"""CPU: pin the oracle restatement (oracle/chunklab_oracle.c) against the reference.

Two independent pins:
  * committed golden fixtures generated from the reference build (tests/golden/), and
  * the reference headers compiled in place (oracle/_ref), when present.
Plus the SURVEY.md Appendix B known-answer scalars, and the exact reduction of the
Mamba-1 recurrence onto chunklab::scan_sequential (SURVEY.md finding 1).
"""
import math

import numpy as np
import pytest

from oracle import oracle as O

APPENDIX_B = {  # SURVEY.md Appendix B (derived from the reference)
    "uniform": (1.9164223760137489e-06, 0.99999992654726755, 5.5450415873139685, 512, 512, 2048),
    "normal": (-4.8771367084113306, 4.5233459468636132, 4.7242405006726766, 512, 256, 2048),
    "normal_s8": (-4.3061552027768659, 4.3582541610515433, 4.8098015627194055, 512, 256, 2048),
    "laplace": (-12.471903275379212, 15.733476552934212, 3.8993669161470006, 512, 256, 2048),
    "sparse10": (-4.4090355758873407, 4.1807362716613383, 0.79880792088178321, 128, 64, 512),
    "sparse02": (-4.0092330290819653, 4.1424502846483042, 0.19539834398694728, 64, 32, 256),
    "normal_k64": (-4.8771367084113306, 4.5233459468636132, 3.338883199120124, 512, 256, 2048),
    "normal_c1": (-5.0765715060991967, 5.0914895678136194, 4.6450975951853648, 512, 256, 2048),
}


def _gen(P, m):
    return P.generate(m["dist"], m["n"], m["seed"], **m["kwargs"])


@pytest.mark.parametrize("name", sorted(APPENDIX_B))
def test_histogram_appendix_b_and_golden(port, golden, name):
    meta, arrays = golden
    m = meta["hist"][name]
    v = _gen(port, m)
    assert port.fnv1a64(v) == m["values_fnv"]  # generator reproduces the reference stream
    counts, lo, hi, n = port.histogram(v, m["k"], 1e-8, m["stride"])
    assert (counts == arrays[f"{name}_counts"]).all()
    masses = counts.astype(np.float64) * (1.0 / n)
    raw, norm = port.entropy(masses)
    lo_b, hi_b, raw_b, c1, c2, c3 = APPENDIX_B[name]
    assert (lo, hi, raw) == (lo_b, hi_b, raw_b) == (m["lo"], m["hi"], m["raw_nats"])
    assert norm == m["normalized"] and n == m["sample_count"]
    k = m["k"]
    assert port.select_chunk(raw, 32, 512, math.log(k))[0] == c1
    assert port.select_chunk(raw, 32, 512, 8.0)[0] == c2
    assert port.select_chunk(raw, 128, 2048, math.log(k))[0] == c3


@pytest.mark.parametrize("name", ["uniform", "normal", "normal_s8", "laplace", "uniform_k512",
                                  "normal_s3", "normal_c1"])
def test_histogram_f32_widened_golden(port, golden, name):
    meta, arrays = golden
    m = meta["hist"][name]
    v32 = _gen(port, m).astype(np.float32)
    counts, lo, hi, n = port.histogram(v32, m["k"], 1e-8, m["stride"])
    assert (counts == arrays[f"{name}_counts_f32"]).all()
    assert (lo, hi) == (m["lo_f32"], m["hi_f32"])
    raw, _ = port.entropy(counts.astype(np.float64) * (1.0 / n))
    assert raw == m["raw_nats_f32"]


def test_rule_grid_golden(port, golden):
    _, arrays = golden
    for s, cmin, cmax, href, c, r in arrays["rule_grid"]:
        cc, rr = port.select_chunk(s, int(cmin), int(cmax), href)
        assert cc == int(c) and rr == r


@pytest.mark.parametrize("key", ["scan_2026_64_16_4096_1", "scan_42_16_8_1000_1",
                                 "scan_9_8_4_64_0", "scan_1_8_4_64_1", "scan_7_4_4_128_1"])
def test_scan_golden(port, golden, key):
    meta, arrays = golden
    m = meta["scan"][key]
    p = port.random_scan_params(m["seed"], m["D"], m["N"], m["L"], m["tv"])
    for k in "abcdx":
        assert port.fnv1a64(p[k]) == m["params_fnv"][k]
    y, h = port.scan(p)
    assert port.fnv1a64(y) == m["y_fnv"] and port.fnv1a64(h) == m["h_fnv"]
    assert (h == arrays[key + "_h"]).all()
    # chunked == sequential, bit-identical (test_scan.cpp:98-118)
    for chunk in (1, 3, 32, 333, 4096):
        yc, hc = port.scan(p, chunk=chunk)
        assert (yc == y).all() and (hc == h).all()


def test_scan_appendix_b_values(port):
    p = port.random_scan_params(2026, 64, 16, 4096, True)
    y, _ = port.scan(p)
    assert y[0] == -0.1159263058640267 and y[-1] == -0.76929978661735932
    p = port.random_scan_params(42, 16, 8, 1000, True)
    y, _ = port.scan(p)
    assert y[0] == -0.22994792022377944 and y[-1] == 1.0664813778300974


def test_oracle_matches_reference_build(port, ref):
    rng = np.random.default_rng(0)
    for trial in range(20):
        n = int(rng.integers(1, 5000))
        v = rng.laplace(0, 2.0, n)
        k = int(rng.integers(2, 600))
        st = int(rng.integers(1, 9))
        counts, lo, hi, ns = port.histogram(v, k, 1e-8, st)
        mr, lor, hir, nr = ref.histogram_masses(v, k, 1e-8, st)
        assert (counts.astype(np.float64) * (1.0 / ns) == mr).all()
        assert (lo, hi, ns) == (lor, hir, nr)
    # fixed range with out-of-range values (test_entropy.cpp:256-265)
    v = np.array([-1.0, 0.5, 3.9, 99.0, 1e12, -1e12])
    c, *_ = port.histogram(v, 4, 1e-8, 1, fixed=(0.0, 4.0))
    mr, *_ = ref.histogram_masses(v, 4, 1e-8, 1, fixed=(0.0, 4.0))
    assert (c.astype(np.float64) * (1.0 / 6) == mr).all()


def test_mamba1_reduces_to_reference_scan(port, golden):
    """SURVEY.md finding 1: Mamba-1 (fp64 restatement) == scan_sequential with
    a = exp(delta'A), x = delta'u, b/c = B/C, d = 0, then + D*u and the gate, bit-exact."""
    meta, arrays = golden
    for key, m in meta["mamba1"].items():
        x = {k: arrays[f"{key}_in_{k}"] for k in ("u", "delta", "A", "B", "C", "D", "z",
                                                   "delta_bias")}
        y, h = port.mamba1(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"],
                           x["delta_bias"], True)
        yr = arrays[f"{key}_y"].reshape(y.shape)
        hr = arrays[f"{key}_h"].reshape(h.shape)
        assert (y == yr).all()
        assert (h == hr).all()


def test_oracle_error_strings(port):
    with pytest.raises(O.OracleError, match="^degenerate spec$"):
        port.histogram(np.array([1.0]), 1)
    with pytest.raises(O.OracleError, match="^non-finite input$"):
        port.histogram(np.array([1.0, np.nan]), 256)
    with pytest.raises(O.OracleError, match="^signal must be >= 0$"):
        port.select_chunk(-1e-8, 32, 512, 8.0)
    with pytest.raises(O.OracleError, match="^invalid chunk bounds$"):
        port.select_chunk(1.0, 48, 512, 8.0)
    # constant tensor -> H = -log(1+eps) < 0 -> the rule throws (SURVEY.md finding 7)
    c, lo, hi, n = port.histogram(np.full(1000, 3.0), 256)
    raw, _ = port.entropy(c.astype(np.float64) / n)
    assert raw == -9.9999998892252911e-09


def test_token_entropy_port_golden(port, golden):
    """The port's token_entropy (entropy.hpp:180-210) equals the reference build's on the
    golden token cases, bit for bit (same glibc log, -ffp-contract=off)."""
    meta, _ = golden
    for name, m in meta["token"].items():
        v = port.generate(m["dist"], m["channels"] * m["length"], m["seed"], **m["kwargs"])
        v = v.reshape(m["channels"], m["length"])
        assert port.fnv1a64(v.reshape(-1)) == m["values_fnv"], name
        fixed = tuple(m["fixed"]) if m["fixed"] else None
        raw, norm, n = port.token_entropy(v, m["k"], 1e-8, m["stride"], fixed)
        assert (raw, norm, n) == (m["raw_nats"], m["normalized"], m["sample_count"]), name
        if O.reference_available():
            assert O.Reference().token_entropy(v, m["k"], 1e-8, m["stride"], fixed) == (raw, norm, n)


def test_ema_host_mirror():
    """test_entropy.cpp:144-172 against the Python mirror (a host scalar recurrence)."""
    import paper_2604_10597_b200 as cl
    nx = cl.update_ema(cl.EmaState(4.0, 0.85, 3), 5.0)
    assert abs(nx.current - 4.15) <= 1e-12 and nx.update_count == 4
    assert cl.update_ema(cl.EmaState(123.0, 0.0), 7.5).current == 7.5
    with pytest.raises(cl.InvalidInput, match=r"ema decay must lie in \[0,1\)"):
        cl.update_ema(cl.EmaState(0.0, 1.0), 1.0)
    s = cl.EmaState(0.0, 0.85)
    for _ in range(7):
        s = cl.update_ema(s, 5.0)
    assert abs(s.current - 5.0 * (1.0 - 0.85 ** 7)) <= 1e-12
