"""Reference file formats: flat little-endian f32/f64 arrays and the
scan-parameter fixture (an f64 blob + a JSON manifest), so captured activations and
goldens interchange with the reference's CLI and tests.

Host-side file plumbing only, no compute.  Mirrors, byte for byte:
  io.hpp:19-44       read_flat_array (f32 widened to f64)
  io.hpp:46-62       write_flat_array
  io.hpp:64-78       write_text_file / read_text_file (binary mode)
  io.hpp:80-84       format_double ("%.*g")
  serialization.hpp:138-156  save_scan_params (nlohmann dump(2) + "\\n" manifest)
  serialization.hpp:158-184  load_scan_params (validated like validate_scan_params)
tests/golden/io holds files written by the reference's own functions
(oracle/ref_fixtures.cpp) that these must read and reproduce exactly.
"""
from __future__ import annotations

import json
import os
from typing import Sequence, Union

import numpy as np

from ._lib import InvalidInput
from .chunklab import ScanParams

PathLike = Union[str, os.PathLike]


def read_flat_array(path: PathLike, dtype: str) -> np.ndarray:
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError:
        raise RuntimeError(f"cannot open {os.fspath(path)}") from None
    if dtype == "f32":
        if len(raw) % 4:
            raise InvalidInput("f32 payload size not a multiple of 4")
        return np.frombuffer(raw, dtype="<f4").astype(np.float64)
    if dtype == "f64":
        if len(raw) % 8:
            raise InvalidInput("f64 payload size not a multiple of 8")
        return np.frombuffer(raw, dtype="<f8").astype(np.float64)
    raise InvalidInput("dtype must be f32 or f64")


def write_flat_array(path: PathLike, values: Sequence[float], dtype: str) -> None:
    if dtype not in ("f32", "f64"):
        raise InvalidInput("dtype must be f32 or f64")
    v = np.asarray(values, dtype=np.float64)
    data = v.astype("<f4") if dtype == "f32" else v.astype("<f8")
    try:
        with open(path, "wb") as f:
            f.write(data.tobytes())
    except OSError:
        raise RuntimeError(f"cannot open {os.fspath(path)}") from None


def write_text_file(path: PathLike, text: str) -> None:
    with open(path, "wb") as f:  # binary: no newline rewriting (io.hpp:64-69)
        f.write(text.encode())


def read_text_file(path: PathLike) -> str:
    with open(path, "rb") as f:
        return f.read().decode()


def format_double(v: float, digits: int = 10) -> str:
    """snprintf("%.*g", digits, v): locale-independent CSV cell."""
    return "%.*g" % (digits, float(v))


_ARRAYS = ("a", "b", "c", "d", "x")


def save_scan_params(stem: PathLike, p: ScanParams) -> None:
    stem = os.fspath(stem)
    arrs = [np.asarray(getattr(p, k), dtype=np.float64).reshape(-1) for k in _ARRAYS]
    write_flat_array(stem + ".bin", np.concatenate(arrs) if arrs else [], "f64")
    # nlohmann::json objects keep keys sorted; dump(2) == json.dumps(indent=2, sort_keys)
    manifest = {"channels": int(p.channels), "state_dim": int(p.state_dim),
                "seq_len": int(p.seq_len),
                "arrays": [{"name": k, "size": int(a.size)} for k, a in zip(_ARRAYS, arrs)],
                "dtype": "f64"}
    write_text_file(stem + ".json", json.dumps(manifest, indent=2, sort_keys=True) + "\n")


def load_scan_params(stem: PathLike) -> ScanParams:
    stem = os.fspath(stem)
    manifest = json.loads(read_text_file(stem + ".json"))
    blob = read_flat_array(stem + ".bin", "f64")
    p = ScanParams(channels=int(manifest["channels"]), state_dim=int(manifest["state_dim"]),
                   seq_len=int(manifest["seq_len"]))
    off = 0
    for arr in manifest["arrays"]:
        name, size = arr["name"], int(arr["size"])
        if off + size > blob.size:
            raise InvalidInput("scan fixture truncated")
        if name not in _ARRAYS:
            raise InvalidInput("unknown scan array: " + name)
        setattr(p, name, blob[off:off + size].copy())
        off += size
    _validate_loaded(p)
    return p


def _validate_loaded(p: ScanParams) -> None:
    """validate_scan_params (scan.hpp:54-69) on a just-loaded fixture (file plumbing)."""
    from .chunklab import _validate_scan_shapes
    _validate_scan_shapes(p)
    if not all(np.isfinite(np.asarray(getattr(p, k))).all() for k in _ARRAYS):
        raise InvalidInput("non-finite input")
