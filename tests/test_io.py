"""CPU: reference file formats against files written by the reference's
own functions (tests/golden/io, from oracle/ref_fixtures.cpp): read them, reproduce them
byte for byte; error strings as io.hpp / serialization.hpp.  One GPU test runs the
loaded fixture through the device fp64 scan against the oracle."""
import os

import numpy as np
import pytest

import paper_2604_10597_b200 as cl
from paper_2604_10597_b200 import io as clio

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")
VALUES = [0.0, 0.25, 0.5, 0.75, -1.5, 1e-3, 3.141592653589793, -0.0]


def _bytes(path):
    with open(path, "rb") as f:
        return f.read()


@pytest.mark.parametrize("stem,args", [("scan_123_8_4_100", (123, 8, 4, 100, True)),
                                       ("scan_9_3_2_17_const", (9, 3, 2, 17, False))])
def test_scan_fixture_roundtrip_bytes(tmp_path, port, stem, args):
    p = clio.load_scan_params(os.path.join(GOLD, stem))
    ref = port.random_scan_params(*args)
    for k in "abcdx":
        assert np.array_equal(getattr(p, k), np.asarray(ref[k])), k  # bit-exact f64
    assert (p.channels, p.state_dim, p.seq_len) == args[1:4]
    clio.save_scan_params(tmp_path / stem, p)
    for ext in (".bin", ".json"):
        assert _bytes(tmp_path / (stem + ext)) == _bytes(os.path.join(GOLD, stem + ext)), ext


def test_flat_arrays(tmp_path):
    assert np.array_equal(clio.read_flat_array(os.path.join(GOLD, "flat_f64.bin"), "f64"), VALUES)
    f32 = clio.read_flat_array(os.path.join(GOLD, "flat_f32.bin"), "f32")
    assert np.array_equal(f32, np.asarray(VALUES, np.float32).astype(np.float64))
    for dt in ("f32", "f64"):
        clio.write_flat_array(tmp_path / f"v.{dt}", VALUES, dt)
        assert _bytes(tmp_path / f"v.{dt}") == _bytes(os.path.join(GOLD, f"flat_{dt}.bin"))
    # test_cli.cpp:222-230: quarter steps survive f32 exactly
    clio.write_flat_array(tmp_path / "q.bin", [0.0, 0.25, 0.5, 0.75], "f32")
    assert list(clio.read_flat_array(tmp_path / "q.bin", "f32")) == [0.0, 0.25, 0.5, 0.75]


def test_errors(tmp_path):
    (tmp_path / "odd.bin").write_bytes(b"\0" * 6)
    with pytest.raises(cl.InvalidInput, match="f32 payload size not a multiple of 4"):
        clio.read_flat_array(tmp_path / "odd.bin", "f32")
    with pytest.raises(cl.InvalidInput, match="f64 payload size not a multiple of 8"):
        clio.read_flat_array(tmp_path / "odd.bin", "f64")
    with pytest.raises(cl.InvalidInput, match="dtype must be f32 or f64"):
        clio.read_flat_array(tmp_path / "odd.bin", "f16")
    with pytest.raises(RuntimeError, match="cannot open"):
        clio.read_flat_array(tmp_path / "missing.bin", "f32")
    # truncated blob
    stem = os.path.join(GOLD, "scan_9_3_2_17_const")
    (tmp_path / "t.json").write_bytes(_bytes(stem + ".json"))
    (tmp_path / "t.bin").write_bytes(_bytes(stem + ".bin")[:-8])
    with pytest.raises(cl.InvalidInput, match="scan fixture truncated"):
        clio.load_scan_params(tmp_path / "t")


def test_format_double():
    lines = clio.read_text_file(os.path.join(GOLD, "format_double.txt")).splitlines()
    xs = [0.0, -0.0, 1.0 / 3.0, 1e-300, 6.02214076e23, 123456789.123456789, -2.5e-7,
          5.545041587313968]
    assert lines == [clio.format_double(x) + " " + clio.format_double(x, 4) for x in xs]


@pytest.mark.gpu
def test_loaded_fixture_scans_on_device(cuda, port):
    """Interchange end to end: the reference-written fixture through the device fp64 scan
    equals the oracle's scan bit for bit (scan.hpp:113-121)."""
    p = clio.load_scan_params(os.path.join(GOLD, "scan_123_8_4_100"))
    out, st = cl.scan_sequential(p)
    yr, hr = port.scan(port.random_scan_params(123, 8, 4, 100, True))
    assert np.array_equal(out.y, yr) and np.array_equal(st.h, hr)
