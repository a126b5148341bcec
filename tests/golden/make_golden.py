"""Generate tests/golden/*.npz|json from the REFERENCE itself (oracle/_ref).

    python tests/golden/make_golden.py

oracle/_ref/libchunklab_ref.so is the reference's own headers
(/root/reference/proj/include/chunklab) compiled in place by oracle/Makefile.
Every fixture below is an output of the reference's functions; nothing is
computed by this repo's code.  The fixtures are small and committed so the
tests can pin the oracle restatement and the GPU path on machines (the GPU box)
where /root/reference does not exist.

Cases (SURVEY.md Appendix B + the reference tests' seeds):
  hist_*     generate_activations -> compute_histogram -> estimate_entropy ->
             select_chunk under 3 calibrations (test_entropy.cpp:111-135,
             acceptance.cpp:80-118, fixtures.hpp:40-47)
  scan_*     random_scan_params -> scan_sequential (test_scan.cpp:82-118,
             acceptance.cpp:134-145)
  mamba1_*   Mamba-1 expressed through scan_sequential (SURVEY.md finding 1)
  rule       select_chunk / schedule over a grid of signals and policies
"""
from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

HIST_CASES = [
    # name, dist, seed, n, K, stride, kwargs
    ("uniform", O.DIST_UNIFORM, 8, 10**6, 256, 1, {}),
    ("normal", O.DIST_NORMAL, 8, 10**6, 256, 1, {}),
    ("normal_s8", O.DIST_NORMAL, 8, 10**6, 256, 8, {}),
    ("laplace", O.DIST_LAPLACE, 8, 10**6, 256, 1, {}),
    ("sparse10", O.DIST_SPARSE, 8, 10**6, 256, 1, {"nonzero_fraction": 0.10}),
    ("sparse02", O.DIST_SPARSE, 8, 10**6, 256, 1, {"nonzero_fraction": 0.02}),
    ("normal_k64", O.DIST_NORMAL, 8, 10**6, 64, 1, {}),
    ("normal_c1", O.DIST_NORMAL, 0, 1536 * 2048, 256, 1, {}),
    ("uniform_k512", O.DIST_UNIFORM, 8, 10**6, 512, 1, {}),
    ("normal_s3", O.DIST_NORMAL, 5, 100003, 128, 3, {}),
]

TOKEN_CASES = [
    # name, dist, seed, channels, length, K, stride, fixed, kwargs
    ("tok_normal", O.DIST_NORMAL, 8, 96, 50, 256, 1, None, {}),
    ("tok_normal_s3_k64", O.DIST_NORMAL, 9, 200, 33, 64, 3, None, {}),
    ("tok_uniform_fixed", O.DIST_UNIFORM, 10, 64, 17, 16, 1, (-0.5, 1.5), {}),
    ("tok_laplace", O.DIST_LAPLACE, 11, 1024, 24, 256, 1, None, {}),
    ("tok_sparse_s8", O.DIST_SPARSE, 12, 777, 40, 128, 8, None, {"nonzero_fraction": 0.1}),
]

SCAN_CASES = [  # seed, D, N, L, time_varying
    (2026, 64, 16, 4096, True),
    (42, 16, 8, 1000, True),
    (9, 8, 4, 64, False),
    (1, 8, 4, 64, True),
    (7, 4, 4, 128, True),
]


def hist_fixtures(R: O.Reference, P: O.Port):
    out = {}
    meta = {}
    for name, dist, seed, n, k, stride, kw in HIST_CASES:
        v = R.generate(dist, n, seed, **kw)
        v32 = v.astype(np.float32)
        masses, lo, hi, ns = R.histogram_masses(v, k, 1e-8, stride)
        raw, norm = R.entropy(masses)
        masses32, lo32, hi32, ns32 = R.histogram_masses(v32, k, 1e-8, stride)
        raw32, norm32 = R.entropy(masses32)
        # counts are recovered exactly from the masses: count = round(mass * n)
        counts = np.rint(masses * ns).astype(np.uint64)
        counts32 = np.rint(masses32 * ns32).astype(np.uint64)
        assert (counts.astype(np.float64) * (1.0 / ns) == masses).all()
        assert (counts32.astype(np.float64) * (1.0 / ns32) == masses32).all()
        chunks = {
            "logk_32_512": R.select_chunk(raw, 32, 512, math.log(k))[0],
            "legacy8_32_512": R.select_chunk(raw, 32, 512, 8.0)[0],
            "logk_128_2048": R.select_chunk(raw, 128, 2048, math.log(k))[0],
        }
        chunks32 = {
            "logk_32_512": R.select_chunk(raw32, 32, 512, math.log(k))[0],
            "legacy8_32_512": R.select_chunk(raw32, 32, 512, 8.0)[0],
            "logk_128_2048": R.select_chunk(raw32, 128, 2048, math.log(k))[0],
        }
        out[f"{name}_counts"] = counts
        out[f"{name}_counts_f32"] = counts32
        meta[name] = dict(dist=dist, seed=seed, n=n, k=k, stride=stride, kwargs=kw,
                          lo=lo, hi=hi, sample_count=ns, raw_nats=raw, normalized=norm,
                          chunks=chunks, lo_f32=lo32, hi_f32=hi32, raw_nats_f32=raw32,
                          normalized_f32=norm32, chunks_f32=chunks32,
                          values_fnv=P.fnv1a64(v), values_f32_fnv=P.fnv1a64(v32))
    return out, meta


def token_fixtures(R: O.Reference, P: O.Port):
    """token_entropy (entropy.hpp:180-210) of generated (channels, length) tensors, fp64
    and fp32-rounded values; the tests regenerate the values with the same generator."""
    meta = {}
    for name, dist, seed, ch, L, k, stride, fixed, kw in TOKEN_CASES:
        v = R.generate(dist, ch * L, seed, **kw).reshape(ch, L)
        v32 = v.astype(np.float32).astype(np.float64)
        raw, norm, n = R.token_entropy(v, k, 1e-8, stride, fixed)
        raw32, norm32, n32 = R.token_entropy(v32, k, 1e-8, stride, fixed)
        meta[name] = dict(dist=dist, seed=seed, channels=ch, length=L, k=k, stride=stride,
                          fixed=list(fixed) if fixed else None, kwargs=kw, raw_nats=raw,
                          normalized=norm, sample_count=n, raw_nats_f32=raw32,
                          normalized_f32=norm32, values_fnv=P.fnv1a64(v.reshape(-1)))
    return meta


def scan_fixtures(R: O.Reference, P: O.Port):
    out, meta = {}, {}
    for seed, D, N, L, tv in SCAN_CASES:
        p = R.random_scan_params(seed, D, N, L, tv)
        y, h = R.scan(p)
        key = f"scan_{seed}_{D}_{N}_{L}_{int(tv)}"
        meta[key] = dict(seed=seed, D=D, N=N, L=L, tv=tv, y_fnv=P.fnv1a64(y),
                         h_fnv=P.fnv1a64(h), y0=float(y[0]), ylast=float(y[-1]),
                         params_fnv={k: P.fnv1a64(p[k]) for k in "abcdx"})
        if y.size <= 20000:
            out[key + "_y"] = y
            out[key + "_h"] = h
        else:
            out[key + "_h"] = h
            out[key + "_y_rows0"] = y[: 2 * L]
    return out, meta


def mamba_inputs(seed, batch, dim, N, L):
    rng = np.random.default_rng(seed)
    u = rng.standard_normal((batch, dim, L)).astype(np.float32)
    delta = (0.1 * rng.standard_normal((batch, dim, L))).astype(np.float32)
    dt = np.exp(rng.uniform(np.log(1e-3), np.log(1e-1), dim))
    bias = np.log(np.expm1(dt)).astype(np.float32)
    A = (-(np.arange(1, N + 1)[None, :]) * (1 + 0.1 * rng.uniform(-1, 1, (dim, N)))).astype(np.float32)
    B = rng.standard_normal((batch, N, L)).astype(np.float32)
    C = rng.standard_normal((batch, N, L)).astype(np.float32)
    D = (1 + 0.1 * rng.standard_normal(dim)).astype(np.float32)
    z = rng.standard_normal((batch, dim, L)).astype(np.float32)
    return dict(u=u, delta=delta, A=A, B=B, C=C, D=D, z=z, delta_bias=bias)


MAMBA_CASES = [  # seed, batch, dim, N, L
    (11, 2, 40, 16, 96),
    (12, 1, 8, 4, 50),
]


def mamba_fixtures(R: O.Reference):
    out, meta = {}, {}
    for seed, batch, dim, N, L in MAMBA_CASES:
        x = mamba_inputs(seed, batch, dim, N, L)
        ys, hs = [], []
        for b in range(batch):
            y, h = R.mamba1_f32(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"],
                                x["delta_bias"], True, rows=(b * dim, (b + 1) * dim))
            ys.append(y)
            hs.append(h)
        key = f"mamba1_{seed}_{batch}_{dim}_{N}_{L}"
        for k, v in x.items():
            out[f"{key}_in_{k}"] = v
        out[f"{key}_y"] = np.concatenate(ys).reshape(batch, dim, L)
        out[f"{key}_h"] = np.concatenate(hs).reshape(batch, dim, N)
        meta[key] = dict(seed=seed, batch=batch, dim=dim, N=N, L=L)
    return out, meta


def rule_fixtures(R: O.Reference):
    rng = np.random.default_rng(3)
    signals = np.concatenate([np.linspace(0, 12, 241), rng.uniform(0, 10, 200),
                              [(362.1 - 32.0) / 480.0, (361.9 - 32.0) / 480.0, 4.60, 5.545,
                               4.612, 3.892, 0.789, 0.192, 5.0, 4.02]])
    rows = []
    for s in signals:
        for (cmin, cmax) in [(32, 512), (128, 2048), (64, 1024)]:
            for href in [math.log(256), 8.0, 1.0, math.log(64), 5.0, 6.0]:
                c, r = R.select_chunk(float(s), cmin, cmax, href)
                rows.append([float(s), cmin, cmax, href, c, r])
    return np.array(rows, dtype=np.float64)


def main():
    if not O.reference_available():
        O.build()
    R = O.Reference()
    P = O.Port()
    arrays, meta = {}, {}
    a, m = hist_fixtures(R, P)
    arrays.update(a)
    meta["hist"] = m
    meta["token"] = token_fixtures(R, P)
    a, m = scan_fixtures(R, P)
    arrays.update(a)
    meta["scan"] = m
    a, m = mamba_fixtures(R)
    arrays.update(a)
    meta["mamba1"] = m
    arrays["rule_grid"] = rule_fixtures(R)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True, default=lambda o: int(o))
    print("wrote", os.path.join(HERE, "golden.npz"), os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
