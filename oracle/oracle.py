"""ctypes bindings for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Two libraries, same C signatures:
  * ``port``      -- oracle/liboracle.so, the plain-C restatement (chunklab_oracle.c)
  * ``reference`` -- oracle/_ref/libchunklab_ref.so, the reference's own headers
                     compiled in place (present only where /root/reference was
                     available at build time; the built .so travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libchunklab_ref.so")

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_u64p = C.POINTER(C.c_uint64)


class HistSpec(C.Structure):
    _fields_ = [("bin_count", C.c_int), ("epsilon", C.c_double), ("range_mode", C.c_int),
                ("fixed_lo", C.c_double), ("fixed_hi", C.c_double),
                ("sample_stride", C.c_uint64)]


class Policy(C.Structure):
    _fields_ = [("kind", C.c_int), ("static_chunk", C.c_int), ("inner_kind", C.c_int),
                ("inner_static_chunk", C.c_int), ("safe_chunk", C.c_int),
                ("min_delta_buckets", C.c_int), ("threshold_tokens", C.c_uint64),
                ("short_chunk", C.c_int), ("long_chunk", C.c_int), ("n_buckets", C.c_int),
                ("buckets", C.c_int * 16)]


class Features(C.Structure):
    _fields_ = [("has_full_entropy", C.c_int), ("full_entropy_nats", C.c_double),
                ("has_sampled_entropy", C.c_int), ("sampled_entropy_nats", C.c_double),
                ("has_seq_len", C.c_int), ("seq_len", C.c_uint64)]


POL_STATIC, POL_MIDPOINT, POL_FULL, POL_SAMPLED, POL_TABLE, POL_GUARDED = range(6)
DIST_UNIFORM, DIST_NORMAL, DIST_LAPLACE, DIST_SPARSE = range(4)


def build():
    """Build liboracle.so (and oracle/_ref when the reference tree exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a, ty):
    return a.ctypes.data_as(ty) if a is not None else None


class OracleError(ValueError):
    pass


class _Lib:
    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        self.lib = C.CDLL(path)


class Port(_Lib):
    """The C restatement."""

    def __init__(self, path=PORT_SO):
        if not os.path.exists(path):
            build()
        super().__init__(path)
        L = self.lib
        L.or_error_string.restype = C.c_char_p
        L.or_fnv1a64.restype = C.c_uint64
        L.or_derive_seed.restype = C.c_uint64

    def err(self, code):
        return self.lib.or_error_string(code).decode()

    def _check(self, rc):
        if rc:
            raise OracleError(self.err(rc))

    def generate(self, dist, n, seed, laplace_scale=1.0, nonzero_fraction=1.0):
        out = np.empty(n, dtype=np.float64)
        self._check(self.lib.or_generate_activations(
            C.c_int(dist), C.c_double(laplace_scale), C.c_double(nonzero_fraction),
            C.c_uint64(seed), C.c_size_t(n), _ptr(out, _dp)))
        return out

    def histogram(self, values, bin_count=256, epsilon=1e-8, stride=1, fixed=None):
        values = np.ascontiguousarray(values)
        spec = HistSpec(bin_count, epsilon, 1 if fixed else 0,
                        fixed[0] if fixed else 0.0, fixed[1] if fixed else 0.0, stride)
        counts = np.zeros(max(bin_count, 1), dtype=np.uint64)
        lo, hi, n = C.c_double(), C.c_double(), C.c_uint64()
        if values.dtype == np.float32:
            rc = self.lib.or_compute_histogram_f32(
                _ptr(values, _fp), C.c_size_t(values.size), C.byref(spec),
                _ptr(counts, _u64p), C.byref(lo), C.byref(hi), C.byref(n))
        else:
            values = values.astype(np.float64, copy=False)
            masses = np.zeros(max(bin_count, 1), dtype=np.float64)
            rc = self.lib.or_compute_histogram(
                _ptr(values, _dp), C.c_size_t(values.size), C.byref(spec),
                _ptr(counts, _u64p), _ptr(masses, _dp), C.byref(lo), C.byref(hi), C.byref(n))
        self._check(rc)
        return counts, lo.value, hi.value, n.value

    def token_entropy(self, values, bin_count=256, epsilon=1e-8, stride=1, fixed=None):
        """values (channels, length) -> (raw_nats, normalized, sample_count)."""
        values = np.ascontiguousarray(values, dtype=np.float64)
        channels, length = values.shape
        spec = HistSpec(bin_count, epsilon, 1 if fixed else 0,
                        fixed[0] if fixed else 0.0, fixed[1] if fixed else 0.0, stride)
        raw, norm, n = C.c_double(), C.c_double(), C.c_uint64()
        self._check(self.lib.or_token_entropy(_ptr(values, _dp), C.c_size_t(channels), C.c_size_t(length),
                                       C.byref(spec), C.byref(raw), C.byref(norm), C.byref(n)))
        return raw.value, norm.value, n.value

    def entropy(self, masses, epsilon=1e-8):
        masses = np.ascontiguousarray(masses, dtype=np.float64)
        raw, norm = C.c_double(), C.c_double()
        self._check(self.lib.or_estimate_entropy(_ptr(masses, _dp), C.c_int(masses.size),
                                                 C.c_double(epsilon), C.byref(raw),
                                                 C.byref(norm)))
        return raw.value, norm.value

    def select_chunk(self, signal, c_min, c_max, h_ref):
        chunk, r = C.c_int(), C.c_double()
        self._check(self.lib.or_select_chunk(C.c_double(signal), C.c_int(c_min),
                                             C.c_int(c_max), C.c_double(h_ref),
                                             C.byref(chunk), C.byref(r)))
        return chunk.value, r.value

    def schedule(self, policy, features, c_min, c_max, h_ref):
        chunk, r, sig, src = C.c_int(), C.c_double(), C.c_double(), C.c_int()
        self._check(self.lib.or_schedule(C.byref(policy), C.byref(features), C.c_int(c_min),
                                         C.c_int(c_max), C.c_double(h_ref), C.byref(chunk),
                                         C.byref(r), C.byref(sig), C.byref(src)))
        return chunk.value, r.value, sig.value, src.value

    def random_scan_params(self, seed, channels, state_dim, seq_len, tv=True):
        a_n = seq_len * channels * state_dim if tv else channels * state_dim
        bc_n = seq_len * state_dim if tv else state_dim
        a, b, c = np.empty(a_n), np.empty(bc_n), np.empty(bc_n)
        d, x = np.empty(channels), np.empty(channels * seq_len)
        self.lib.or_random_scan_params(C.c_uint64(seed), C.c_size_t(channels),
                                       C.c_size_t(state_dim), C.c_size_t(seq_len),
                                       C.c_int(int(tv)), _ptr(a, _dp), _ptr(b, _dp),
                                       _ptr(c, _dp), _ptr(d, _dp), _ptr(x, _dp))
        return dict(channels=channels, state_dim=state_dim, seq_len=seq_len, a=a, b=b, c=c,
                    d=d, x=x)

    def scan(self, p, h0=None, chunk=0):
        class SP(C.Structure):
            _fields_ = [("channels", C.c_size_t), ("state_dim", C.c_size_t),
                        ("seq_len", C.c_size_t), ("a", _dp), ("b", _dp), ("c", _dp),
                        ("d", _dp), ("x", _dp), ("a_len", C.c_size_t), ("b_len", C.c_size_t),
                        ("c_len", C.c_size_t), ("d_len", C.c_size_t), ("x_len", C.c_size_t)]
        arrs = {k: np.ascontiguousarray(p[k], dtype=np.float64) for k in "abcdx"}
        sp = SP(p["channels"], p["state_dim"], p["seq_len"],
                *[_ptr(arrs[k], _dp) for k in "abcdx"], *[arrs[k].size for k in "abcdx"])
        y = np.empty(p["channels"] * p["seq_len"])
        h = np.empty(p["channels"] * p["state_dim"])
        h0a = None if h0 is None else np.ascontiguousarray(h0, dtype=np.float64)
        self._check(self.lib.or_scan_chunked(C.byref(sp), _ptr(h0a, _dp), C.c_size_t(chunk),
                                             _ptr(y, _dp), _ptr(h, _dp)))
        return y, h

    def mamba1(self, u, delta, A, B, C_, D=None, z=None, delta_bias=None, delta_softplus=True,
               rows=None, h0=None):
        """u, delta, z: (batch, dim, L); A (dim, N); B, C (batch, N, L).  fp64 result."""
        batch, dim, L = u.shape
        N = A.shape[1]
        r0, r1 = rows if rows is not None else (0, batch * dim)
        y = np.empty((r1 - r0) * L)
        h = np.empty((r1 - r0) * N)
        f32 = u.dtype == np.float32
        ty = _fp if f32 else _dp
        dt = np.float32 if f32 else np.float64
        cv = lambda a: None if a is None else np.ascontiguousarray(a, dtype=dt)  # noqa: E731
        args = [cv(u), cv(delta), cv(A), cv(B), cv(C_), cv(D), cv(z), cv(delta_bias)]
        keep = args  # noqa: F841  keep buffers alive through the call
        if f32:
            assert h0 is None
            rc = self.lib.or_mamba1_scan_rows_f32(
                *[_ptr(a, ty) for a in args], C.c_int(int(delta_softplus)), C.c_size_t(batch),
                C.c_size_t(dim), C.c_size_t(N), C.c_size_t(L), C.c_size_t(r0), C.c_size_t(r1),
                _ptr(y, _dp), _ptr(h, _dp))
        else:
            h0a = None if h0 is None else np.ascontiguousarray(h0, dtype=np.float64)
            rc = self.lib.or_mamba1_scan_rows(
                *[_ptr(a, ty) for a in args], C.c_int(int(delta_softplus)), C.c_size_t(batch),
                C.c_size_t(dim), C.c_size_t(N), C.c_size_t(L), C.c_size_t(r0), C.c_size_t(r1),
                _ptr(h0a, _dp), _ptr(y, _dp), _ptr(h, _dp))
        self._check(rc)
        return y.reshape(r1 - r0, L), h.reshape(r1 - r0, N)

    def fnv1a64(self, arr):
        arr = np.ascontiguousarray(arr)
        return int(self.lib.or_fnv1a64(arr.ctypes.data_as(C.c_void_p), C.c_size_t(arr.nbytes)))


class Reference(_Lib):
    """The reference's own headers compiled in place (oracle/_ref)."""

    def __init__(self, path=REF_SO):
        super().__init__(path)
        self.lib.ref_last_error.restype = C.c_char_p

    def _check(self, rc):
        if rc:
            raise OracleError(self.lib.ref_last_error().decode())

    def generate(self, dist, n, seed, laplace_scale=1.0, nonzero_fraction=1.0):
        out = np.empty(n, dtype=np.float64)
        self._check(self.lib.ref_generate_activations(
            C.c_int(dist), C.c_double(laplace_scale), C.c_double(nonzero_fraction),
            C.c_uint64(seed), C.c_uint64(n), _ptr(out, _dp)))
        return out

    def histogram_masses(self, values, bin_count=256, epsilon=1e-8, stride=1, fixed=None):
        values = np.ascontiguousarray(values)
        spec = HistSpec(bin_count, epsilon, 1 if fixed else 0,
                        fixed[0] if fixed else 0.0, fixed[1] if fixed else 0.0, stride)
        masses = np.zeros(max(bin_count, 1), dtype=np.float64)
        lo, hi, n = C.c_double(), C.c_double(), C.c_uint64()
        if values.dtype == np.float32:
            rc = self.lib.ref_compute_histogram_f32(_ptr(values, _fp), C.c_uint64(values.size),
                                                    C.byref(spec), _ptr(masses, _dp),
                                                    C.byref(lo), C.byref(hi), C.byref(n))
        else:
            values = values.astype(np.float64, copy=False)
            rc = self.lib.ref_compute_histogram(_ptr(values, _dp), C.c_uint64(values.size),
                                                C.byref(spec), _ptr(masses, _dp), C.byref(lo),
                                                C.byref(hi), C.byref(n))
        self._check(rc)
        return masses, lo.value, hi.value, n.value

    def token_entropy(self, values, bin_count=256, epsilon=1e-8, stride=1, fixed=None):
        """values (channels, length) -> (raw_nats, normalized, sample_count)."""
        values = np.ascontiguousarray(values, dtype=np.float64)
        channels, length = values.shape
        spec = HistSpec(bin_count, epsilon, 1 if fixed else 0,
                        fixed[0] if fixed else 0.0, fixed[1] if fixed else 0.0, stride)
        raw, norm, n = C.c_double(), C.c_double(), C.c_uint64()
        self._check(self.lib.ref_token_entropy(_ptr(values, _dp), C.c_uint64(channels), C.c_uint64(length),
                                       C.byref(spec), C.byref(raw), C.byref(norm), C.byref(n)))
        return raw.value, norm.value, n.value

    def entropy(self, masses, epsilon=1e-8):
        masses = np.ascontiguousarray(masses, dtype=np.float64)
        raw, norm = C.c_double(), C.c_double()
        self._check(self.lib.ref_estimate_entropy(_ptr(masses, _dp), C.c_int(masses.size),
                                                  C.c_double(epsilon), C.byref(raw),
                                                  C.byref(norm)))
        return raw.value, norm.value

    def select_chunk(self, signal, c_min, c_max, h_ref):
        chunk, r = C.c_int(), C.c_double()
        self._check(self.lib.ref_select_chunk(C.c_double(signal), C.c_int(c_min),
                                              C.c_int(c_max), C.c_double(h_ref),
                                              C.byref(chunk), C.byref(r)))
        return chunk.value, r.value

    def schedule(self, policy, features, c_min, c_max, h_ref):
        chunk, r, sig, src = C.c_int(), C.c_double(), C.c_double(), C.c_int()
        self._check(self.lib.ref_schedule(C.byref(policy), C.byref(features), C.c_int(c_min),
                                          C.c_int(c_max), C.c_double(h_ref), C.byref(chunk),
                                          C.byref(r), C.byref(sig), C.byref(src)))
        return chunk.value, r.value, sig.value, src.value

    def random_scan_params(self, seed, channels, state_dim, seq_len, tv=True):
        a_n = seq_len * channels * state_dim if tv else channels * state_dim
        bc_n = seq_len * state_dim if tv else state_dim
        a, b, c = np.empty(a_n), np.empty(bc_n), np.empty(bc_n)
        d, x = np.empty(channels), np.empty(channels * seq_len)
        self._check(self.lib.ref_random_scan_params(
            C.c_uint64(seed), C.c_uint64(channels), C.c_uint64(state_dim), C.c_uint64(seq_len),
            C.c_int(int(tv)), _ptr(a, _dp), _ptr(b, _dp), _ptr(c, _dp), _ptr(d, _dp),
            _ptr(x, _dp)))
        return dict(channels=channels, state_dim=state_dim, seq_len=seq_len, a=a, b=b, c=c,
                    d=d, x=x)

    def scan(self, p, h0=None, chunk=0):
        arrs = {k: np.ascontiguousarray(p[k], dtype=np.float64) for k in "abcdx"}
        y = np.empty(p["channels"] * p["seq_len"])
        h = np.empty(p["channels"] * p["state_dim"])
        h0a = None if h0 is None else np.ascontiguousarray(h0, dtype=np.float64)
        args = []
        for k in "abcdx":
            args += [_ptr(arrs[k], _dp), C.c_uint64(arrs[k].size)]
        self._check(self.lib.ref_scan(C.c_uint64(p["channels"]), C.c_uint64(p["state_dim"]),
                                      C.c_uint64(p["seq_len"]), *args, _ptr(h0a, _dp),
                                      C.c_uint64(chunk), _ptr(y, _dp), _ptr(h, _dp)))
        return y, h

    def mamba1_f32(self, u, delta, A, B, C_, D=None, z=None, delta_bias=None,
                   delta_softplus=True, rows=None, threads=1):
        batch, dim, L = u.shape
        N = A.shape[1]
        r0, r1 = rows if rows is not None else (0, dim)
        y = np.empty((r1 - r0) * L)
        h = np.empty((r1 - r0) * N)
        cv = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float32)  # noqa
        args = [cv(u), cv(delta), cv(A), cv(B), cv(C_), cv(D), cv(z), cv(delta_bias)]
        self._check(self.lib.ref_mamba1_rows_f32(
            *[_ptr(a, _fp) for a in args], C.c_int(int(delta_softplus)), C.c_uint64(batch),
            C.c_uint64(dim), C.c_uint64(N), C.c_uint64(L), C.c_uint64(r0), C.c_uint64(r1),
            C.c_int(threads), _ptr(y, _dp), _ptr(h, _dp)))
        return y.reshape(r1 - r0, L), h.reshape(r1 - r0, N)


def causal_conv1d_f64(x, weight, bias=None, silu=True):
    """fp64 restatement of causal_conv1d_fn(x, weight, bias, activation) -- the producer
    of u in the paper's MambaMixer.  PARITY UNPINNED: the reference has
    no convolution; this restates the package's published formula
        u[b,d,t] = act(bias[d] + sum_k weight[d,k] * x[b,d,t-W+1+k]),  x[<0] = 0.
    x (batch, dim, L), weight (dim, W), bias (dim,)."""
    x = np.asarray(x, dtype=np.float64)
    w = np.asarray(weight, dtype=np.float64)
    W = w.shape[1]
    L = x.shape[-1]
    xp = np.concatenate([np.zeros(x.shape[:-1] + (W - 1,)), x], axis=-1)
    out = np.zeros_like(x) + (0.0 if bias is None else np.asarray(bias, np.float64)[:, None])
    for k in range(W):
        out = out + w[None, :, k:k + 1] * xp[..., k:k + L]
    if silu:
        out = out / (1.0 + np.exp(-out))
    return out


def reference_available():
    return os.path.exists(REF_SO)
