"""The reference's C++ API (include/chunklab/*.hpp drop-in) compiled with g++ against
libchunklab_b200.so; the GPU test runs the re-expressed reference test cases."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
PKG = os.path.join(ROOT, "paper_2604_10597_b200")
CUDA_INC = "/usr/local/cuda/include"
CUDA_LIB = "/usr/local/cuda/lib64"


THREADS_SRC = os.path.join(ROOT, "tests", "cpp", "test_threads.cpp")
SHARDED_SRC = os.path.join(ROOT, "tests", "cpp", "test_sharded.cpp")


def build(out, src=SRC, extra=()):
    from paper_2604_10597_b200 import build as b
    b.build()
    cmd = ["g++", "-std=c++20", "-O2", "-pthread", "-I" + os.path.join(ROOT, "include"),
           "-I" + CUDA_INC, src, "-L" + PKG, "-lchunklab_b200", "-Wl,-rpath," + PKG,
           "-L" + CUDA_LIB, "-lcudart", "-Wl,-rpath," + CUDA_LIB, *extra, "-o", out]
    subprocess.run(cmd, check=True)
    return out


def test_dropin_headers_compile(tmp_path):
    exe = build(str(tmp_path / "test_dropin"))
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_dropin_reference_cases(tmp_path, cuda):
    exe = build(str(tmp_path / "test_dropin"))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout


def test_threads_program_compiles(tmp_path):
    assert os.path.exists(build(str(tmp_path / "test_threads"), THREADS_SRC))


@pytest.mark.gpu
def test_dropin_threads_and_streams(tmp_path, cuda):
    """SPEC.md:86 (pure, shareable across threads): 4 host threads through the drop-in's
    one process-wide context, and two prefills in flight on two streams of it, give the
    bits each gives alone."""
    exe = build(str(tmp_path / "test_threads"), THREADS_SRC)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "threads ok" in r.stdout


def test_sharded_program_compiles(tmp_path):
    assert os.path.exists(build(str(tmp_path / "test_sharded"), SHARDED_SRC, ["-lnccl"]))


@pytest.mark.gpu
def test_sharded_prefill_cpp_world2_and_nccl(tmp_path, cuda):
    """The C/C++ multi-GPU entry point (cl_prefill_sharded_f32 / chunklab::ShardedPrefill):
    device stages on every rank, host-staged allreduces between rank threads (world 2 and
    4; batch and d_inner splits; rule, guarded stride 8, token policies): range, counts and
    decision bit-identical to the single-GPU call; then world 1 over real NCCL."""
    exe = build(str(tmp_path / "test_sharded"), SHARDED_SRC, ["-lnccl"])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "sharded ok" in r.stdout
