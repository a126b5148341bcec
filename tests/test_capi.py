"""CPU: the C-ABI library loads and exports every symbol include/*.h declares; the
Python binding types every one of them; no compute call is made (no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2604_10597_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "chunklab_capi.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cl_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_abi():
    names = declared_functions()
    assert "cl_prefill_f32" in names and "cl_scan_f64_host" in names
    assert len(names) >= 20


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2604_10597_b200 import build
        build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (cl_\w+)", out))
    assert set(declared_functions()) <= exported


def test_binding_types_every_symbol():
    assert set(_lib.SIGNATURES) == set(declared_functions())
    lib = _lib.load_library()
    assert lib.cl_abi_version() == 1


def test_no_gpu_fails_loudly():
    """Without a device the context refuses to start: there is no CPU fallback."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(_lib.DeviceError, match="no CPU fallback"):
        _lib.Context(0)


def test_kernels_are_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_enum_constants_match_the_header():
    """The Python constants mirror the header's enums (a drift would silently select the
    wrong kernel or policy)."""
    src = open(HEADER).read()
    for name in ("CL_SCAN_AUTO", "CL_SCAN_ROWSEQ_TMA", "CL_SCAN_GENERIC", "CL_SCAN_LOOKBACK",
                 "CL_SCAN_CHAINED", "CL_SCAN_CONFIG_BASE", "CL_SCAN_LOOKBACK_BASE",
                 "CL_KERNEL_GENERIC", "CL_KERNEL_CHAINED", "CL_KERNEL_ROWSEQ",
                 "CL_KERNEL_LOOKBACK"):
        m = re.search(rf"\b{name}\s*=\s*(\d+)", src)
        assert m, name
        assert getattr(_lib, name) == int(m.group(1)), name
    m = re.search(r"#define\s+CL_GATHER_MIN_STRIDE\s+(\d+)", src)
    assert m and _lib.CL_GATHER_MIN_STRIDE == int(m.group(1))


def test_scan_variant_codes():
    from paper_2604_10597_b200.mamba1 import _variant_code
    assert _variant_code("auto") == _lib.CL_SCAN_AUTO
    assert _variant_code("generic") == _lib.CL_SCAN_GENERIC
    assert _variant_code("cfg:11") == _lib.CL_SCAN_CONFIG_BASE + 11
    assert _variant_code("lookback") == _lib.CL_SCAN_LOOKBACK
    assert _variant_code("chained") == _lib.CL_SCAN_CHAINED
    assert _variant_code("lb:2") == _lib.CL_SCAN_LOOKBACK_BASE + 2
    with pytest.raises(KeyError):
        _variant_code("nope")


def test_samples_in_counts_multiples():
    """cl_samples_in (pure host function): the number of global indices in
    [offset, offset + n) that are multiples of stride."""
    lib = _lib.load_library()
    for off in (0, 1, 7, 8, 1000003):
        for n in (0, 1, 5, 8, 999):
            for st in (1, 3, 4, 8, 16):
                want = sum(1 for g in range(off, off + n) if g % st == 0)
                assert lib.cl_samples_in(off, n, st) == want, (off, n, st)
    assert lib.cl_samples_in(5, 10, 0) == 0
