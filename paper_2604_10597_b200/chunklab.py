"""Python mirror of the reference's chunklab hot-path API, running on the B200.

Names, argument meaning and error strings follow
/root/reference/proj/include/chunklab/{entropy,chunk,scan}.hpp so that parity
tests read like the reference's own Catch2 tests.  Every computation goes
through libchunklab_b200.so (include/chunklab_capi.h) on the GPU:

  compute_histogram / estimate_entropy      entropy.hpp:101-174   -> cl_compute_histogram_host,
                                                                     cl_estimate_entropy_host
  select_chunk / Scheduler / schedule       chunk.hpp:68-385      -> cl_schedule_host (device rule)
  scan_sequential / scan_chunked            scan.hpp:113-136      -> cl_scan_f64_host (fp64, bit-exact)
  selective_scan_fn (Mamba-1, fp32)         PAPER.md:811, :1340   -> cl_selective_scan_f32
  prefill (entropy -> rule -> scan)         PAPER.md:810-812      -> cl_range_init .. cl_selective_scan_f32

Host-side scalar logic kept here is limited to struct marshalling and
validation that must raise before any device work (same order as the reference).
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence, Union

import numpy as np

from . import _lib
from ._lib import Context, InvalidInput

__all__ = [
    "InvalidInput", "RangeMode", "HistogramSpec", "ActivationTensor", "Histogram",
    "EntropyEstimate", "compute_histogram", "estimate_entropy", "estimate_tensor_entropy",
    "token_entropy", "EmaState", "update_ema", "TokenHistogramPolicy",
    "ChunkBounds", "CalibrationRef", "ChunkDecision", "select_chunk", "kernel_calls",
    "StaticPolicy", "NoEntropyMidpointPolicy", "FullHistogramPolicy", "SampledHistogramPolicy",
    "GuardedPolicy", "LearnedTablePolicy", "SchedulerPolicy", "ScheduleFeatures", "Scheduler",
    "schedule", "ScanParams", "ScanState", "ScanOutput", "scan_sequential", "scan_chunked",
    "is_power_of_two", "log2_exact", "round_half_up", "ceil_div",
]


# ---------------------------------------------------------------- common.hpp
def is_power_of_two(v: int) -> bool:
    return v != 0 and (v & (v - 1)) == 0


def log2_exact(v: int) -> int:
    return int(v).bit_length() - 1 if v >= 1 else 0


def round_half_up(x: float) -> float:
    return math.floor(x + 0.5)


def ceil_div(num: int, den: int) -> int:
    return (num + den - 1) // den


# ---------------------------------------------------------------- entropy.hpp
class RangeMode(enum.IntEnum):
    Dynamic = _lib.CL_RANGE_DYNAMIC
    Fixed = _lib.CL_RANGE_FIXED


@dataclass
class HistogramSpec:
    """entropy.hpp:47-54."""
    bin_count: int = 256
    epsilon: float = 1e-8
    range_mode: RangeMode = RangeMode.Dynamic
    fixed_lo: float = 0.0
    fixed_hi: float = 0.0
    sample_stride: int = 1

    def to_c(self) -> _lib.cl_hist_spec:
        if self.sample_stride < 1:
            # size_t in the reference cannot be negative; 0 is the only invalid value.
            stride = 0
        else:
            stride = int(self.sample_stride)
        return _lib.cl_hist_spec(int(self.bin_count), float(self.epsilon), int(self.range_mode),
                                 float(self.fixed_lo), float(self.fixed_hi), stride)


@dataclass
class ActivationTensor:
    """entropy.hpp:27-32: flat values (row-major in shape) plus a shape."""
    values: np.ndarray
    shape: Sequence[int]

    def size(self) -> int:
        return int(np.asarray(self.values).size)


@dataclass
class Histogram:
    """entropy.hpp:64-71 (+ the raw counts the device produced)."""
    masses: np.ndarray
    lo: float = 0.0
    hi: float = 0.0
    sample_count: int = 0
    counts: Optional[np.ndarray] = None

    def bin_count(self) -> int:
        return int(len(self.masses))


@dataclass
class EntropyEstimate:
    """entropy.hpp:73-80."""
    raw_nats: float = 0.0
    normalized: float = 0.0
    bin_count: int = 0
    epsilon: float = 0.0
    sample_stride: int = 1
    sample_count: int = 0


def validate_tensor(t: ActivationTensor) -> None:
    """entropy.hpp:34-43 (shape part; the finite check runs on the device)."""
    if len(t.shape) == 0:
        raise InvalidInput("empty shape")
    n = 1
    for e in t.shape:
        if e == 0:
            raise InvalidInput("zero shape extent")
        n *= int(e)
    if n != t.size():
        raise InvalidInput("shape/value count mismatch")


def _as_f64(values) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(values, dtype=np.float64).reshape(-1))


def _require_all_finite(v: np.ndarray, ctx: Context) -> None:
    """validate_tensor's value check (entropy.hpp:42) over every value, on the device."""
    ok = C.c_int()
    ctx.call("cl_all_finite_host", v.ctypes.data_as(C.c_void_p), v.size, C.byref(ok))
    if not ok.value:
        raise InvalidInput("non-finite input")


def compute_histogram(values: Union[ActivationTensor, Sequence[float], np.ndarray],
                      spec: HistogramSpec, ctx: Optional[Context] = None) -> Histogram:
    """compute_histogram (entropy.hpp:101-145) on the GPU; counts bit-exact."""
    ctx = ctx or Context.get()
    if isinstance(values, ActivationTensor):
        if values.size() == 0:
            raise InvalidInput("no samples")
        validate_tensor(values)
        v = _as_f64(values.values)
        _require_all_finite(v, ctx)
    else:
        v = _as_f64(values)
    cspec = spec.to_c()
    ctx.call("cl_validate_hist_spec", C.byref(cspec))
    if v.size == 0:
        raise InvalidInput("no samples")
    k = int(spec.bin_count)
    counts = np.zeros(k, dtype=np.uint64)
    masses = np.zeros(k, dtype=np.float64)
    lo, hi, n = C.c_double(), C.c_double(), C.c_uint64()
    ctx.call("cl_compute_histogram_host", v.ctypes.data_as(C.c_void_p), v.size, C.byref(cspec),
             counts.ctypes.data_as(C.c_void_p), masses.ctypes.data_as(C.c_void_p), C.byref(lo),
             C.byref(hi), C.byref(n))
    return Histogram(masses=masses, lo=lo.value, hi=hi.value, sample_count=int(n.value),
                     counts=counts)


def estimate_entropy(hist: Histogram, epsilon: float, ctx: Optional[Context] = None
                     ) -> EntropyEstimate:
    """estimate_entropy (entropy.hpp:149-164) on the GPU."""
    ctx = ctx or Context.get()
    m = _as_f64(hist.masses)
    raw, norm = C.c_double(), C.c_double()
    ctx.call("cl_estimate_entropy_host", m.ctypes.data_as(C.c_void_p), int(m.size),
             float(epsilon), C.byref(raw), C.byref(norm))
    return EntropyEstimate(raw_nats=raw.value, normalized=norm.value, bin_count=int(m.size),
                           epsilon=float(epsilon), sample_count=int(hist.sample_count))


def token_entropy(tensor: ActivationTensor, spec: HistogramSpec,
                  ctx: Optional[Context] = None) -> EntropyEstimate:
    """token_entropy (entropy.hpp:180-210) on the GPU: one histogram per position of the
    last axis over that position's channel values, raw entropies averaged."""
    ctx = ctx or Context.get()
    if tensor.size() == 0:
        raise InvalidInput("no samples")
    validate_tensor(tensor)
    v = _as_f64(tensor.values)
    _require_all_finite(v, ctx)
    cspec = spec.to_c()
    ctx.call("cl_validate_hist_spec", C.byref(cspec))
    if len(tensor.shape) < 2:
        raise InvalidInput("token entropy needs a (channels, length) tensor")
    length = int(tensor.shape[-1])
    channels = v.size // length
    raw, norm, n = C.c_double(), C.c_double(), C.c_uint64()
    ctx.call("cl_token_entropy_host", v.ctypes.data_as(C.c_void_p), channels, length,
             C.byref(cspec), C.byref(raw), C.byref(norm), C.byref(n))
    return EntropyEstimate(raw_nats=raw.value, normalized=norm.value,
                           bin_count=int(spec.bin_count), epsilon=float(spec.epsilon),
                           sample_stride=int(spec.sample_stride), sample_count=int(n.value))


@dataclass
class EmaState:
    """entropy.hpp:214-218."""
    current: float = 0.0
    decay: float = 0.85
    update_count: int = 0


def update_ema(state: EmaState, new_h: float) -> EmaState:
    """entropy.hpp:220-227: H_t = decay * H_{t-1} + (1 - decay) * H_new (a host scalar)."""
    if not (0.0 <= state.decay < 1.0):
        raise InvalidInput("ema decay must lie in [0,1)")
    return EmaState(state.decay * state.current + (1.0 - state.decay) * float(new_h),
                    state.decay, state.update_count + 1)


def estimate_tensor_entropy(tensor: ActivationTensor, spec: HistogramSpec,
                            ctx: Optional[Context] = None) -> EntropyEstimate:
    """entropy.hpp:168-174."""
    e = estimate_entropy(compute_histogram(tensor, spec, ctx), spec.epsilon, ctx)
    e.sample_stride = int(spec.sample_stride)
    return e


# ---------------------------------------------------------------- chunk.hpp
@dataclass
class ChunkBounds:
    """chunk.hpp:29-32."""
    c_min: int = 32
    c_max: int = 512


def validate_bounds(b: ChunkBounds) -> None:
    if (b.c_min <= 0 or b.c_max <= 0 or not is_power_of_two(b.c_min)
            or not is_power_of_two(b.c_max) or b.c_min > b.c_max):
        raise InvalidInput("invalid chunk bounds")


class CalibrationMode(enum.IntEnum):
    LogK = 0
    LegacyFixed = 1


@dataclass
class CalibrationRef:
    """chunk.hpp:42-59."""
    mode: CalibrationMode = CalibrationMode.LogK
    h_ref_nats: float = 0.0

    @staticmethod
    def log_k(bin_count: int) -> "CalibrationRef":
        if bin_count < 2:
            raise InvalidInput("degenerate spec")
        return CalibrationRef(CalibrationMode.LogK, math.log(float(bin_count)))

    @staticmethod
    def legacy(h_ref_nats: float = 8.0) -> "CalibrationRef":
        if not (h_ref_nats > 0.0):
            raise InvalidInput("h_ref must be positive")
        return CalibrationRef(CalibrationMode.LegacyFixed, float(h_ref_nats))


@dataclass
class ChunkDecision:
    """chunk.hpp:61-66 (+ device diagnostics)."""
    chunk: int = 0
    r: float = 0.0
    source_policy: str = ""
    signal_nats: float = 0.0
    margin: float = 1.0


def kernel_calls(seq_len: int, chunk: int) -> int:
    """chunk.hpp:92-95."""
    if seq_len == 0 or chunk == 0:
        raise InvalidInput("seq_len and chunk must be positive")
    return ceil_div(seq_len, chunk)


@dataclass
class StaticPolicy:
    chunk: int = 512


@dataclass
class NoEntropyMidpointPolicy:
    pass


@dataclass
class FullHistogramPolicy:
    pass


@dataclass
class SampledHistogramPolicy:
    stride: int = 8


@dataclass
class TokenHistogramPolicy:
    """chunk.hpp:119 / :311-315: the rule on token_entropy."""


@dataclass
class LearnedTablePolicy:
    threshold_tokens: int = 50
    short_chunk: int = 128
    long_chunk: int = 512


@dataclass
class GuardedPolicy:
    inner: Optional["SchedulerPolicy"] = None
    safe_chunk: int = 512
    min_delta_buckets: int = 2


@dataclass
class SchedulerPolicy:
    variant: object = field(default_factory=FullHistogramPolicy)
    bucket_set: Sequence[int] = field(default_factory=lambda: [128, 256, 512, 1024, 2048])


@dataclass
class ScheduleFeatures:
    """chunk.hpp:185-193 (the device-decidable subset)."""
    full_entropy: Optional[EntropyEstimate] = None
    sampled_entropy: Optional[EntropyEstimate] = None
    seq_len: Optional[int] = None
    token_entropy: Optional[EntropyEstimate] = None


_KIND = {StaticPolicy: _lib.CL_POL_STATIC, NoEntropyMidpointPolicy: _lib.CL_POL_MIDPOINT,
         FullHistogramPolicy: _lib.CL_POL_FULL_HIST,
         SampledHistogramPolicy: _lib.CL_POL_SAMPLED_HIST,
         LearnedTablePolicy: _lib.CL_POL_LEARNED_TABLE, GuardedPolicy: _lib.CL_POL_GUARDED,
         TokenHistogramPolicy: _lib.CL_POL_TOKEN_HIST}


def _fill_simple(spec: _lib.cl_rule_spec, v, inner: bool):
    kind = _KIND.get(type(v))
    if kind is None:
        raise InvalidInput("unsupported policy on the device path: " + type(v).__name__)
    if inner:
        spec.inner_kind = kind
        if isinstance(v, StaticPolicy):
            spec.inner_static_chunk = int(v.chunk)
    else:
        spec.kind = kind
        if isinstance(v, StaticPolicy):
            spec.static_chunk = int(v.chunk)
    if isinstance(v, LearnedTablePolicy):
        spec.threshold_tokens = int(v.threshold_tokens)
        spec.short_chunk = int(v.short_chunk)
        spec.long_chunk = int(v.long_chunk)


def rule_spec(policy: Optional[SchedulerPolicy], bounds: ChunkBounds, cal: CalibrationRef
              ) -> _lib.cl_rule_spec:
    """Flatten a SchedulerPolicy (chunk.hpp:144-147) into the C-ABI rule struct.
    policy None -> the bare select_chunk rule (chunk.hpp:68-89)."""
    s = _lib.cl_rule_spec()
    s.c_min, s.c_max = int(bounds.c_min), int(bounds.c_max)
    s.h_ref_nats = float(cal.h_ref_nats)
    if policy is None:
        s.kind = _lib.CL_POL_RULE
        return s
    buckets = list(policy.bucket_set)
    s.n_buckets = len(buckets)
    if len(buckets) > 16:
        raise InvalidInput("bucket_set too large")
    for i, b in enumerate(buckets):
        s.buckets[i] = int(b)
    v = policy.variant
    if isinstance(v, GuardedPolicy):
        if v.inner is None:
            raise InvalidInput("guarded policy needs an inner policy")
        s.kind = _lib.CL_POL_GUARDED
        s.safe_chunk = int(v.safe_chunk)
        s.min_delta_buckets = int(v.min_delta_buckets)
        if isinstance(v.inner.variant, GuardedPolicy):
            raise InvalidInput("nested guarded policies are not supported on the device path")
        _fill_simple(s, v.inner.variant, inner=True)
    else:
        _fill_simple(s, v, inner=False)
    return s


def _decision_from_c(d: _lib.cl_decision) -> ChunkDecision:
    return ChunkDecision(chunk=int(d.chunk), r=float(d.r), source_policy=_lib.source_tag(d.source),
                         signal_nats=float(d.signal_nats), margin=float(d.margin))


def select_chunk(signal_nats: float, bounds: ChunkBounds, cal: CalibrationRef,
                 ctx: Optional[Context] = None) -> ChunkDecision:
    """select_chunk (chunk.hpp:68-89), evaluated by the device rule kernel."""
    ctx = ctx or Context.get()
    s = rule_spec(None, bounds, cal)
    f = _lib.cl_features(1, float(signal_nats), 0, 0.0, 0, 0)
    out = _lib.cl_decision()
    ctx.call("cl_schedule_host", C.byref(s), C.byref(f), C.byref(out))
    return _decision_from_c(out)


class Scheduler:
    """Scheduler (chunk.hpp:225-375) for the device policy subset."""

    def __init__(self, policy: SchedulerPolicy, bounds: ChunkBounds, cal: CalibrationRef,
                 ctx: Optional[Context] = None):
        self.ctx = ctx or Context.get()
        self._policy = policy
        self._spec = rule_spec(policy, bounds, cal)
        self.ctx.call("cl_validate_rule", C.byref(self._spec))

    def policy(self) -> SchedulerPolicy:
        return self._policy

    def rule(self) -> _lib.cl_rule_spec:
        return self._spec

    def decide(self, features: ScheduleFeatures) -> ChunkDecision:
        f = _lib.cl_features()
        if features.full_entropy is not None:
            f.has_full_entropy = 1
            f.full_entropy_nats = float(features.full_entropy.raw_nats)
        if features.sampled_entropy is not None:
            f.has_sampled_entropy = 1
            f.sampled_entropy_nats = float(features.sampled_entropy.raw_nats)
        if features.seq_len is not None:
            f.has_seq_len = 1
            f.seq_len = int(features.seq_len)
        if features.token_entropy is not None:
            f.has_token_entropy = 1
            f.token_entropy_nats = float(features.token_entropy.raw_nats)
        out = _lib.cl_decision()
        self.ctx.call("cl_schedule_host", C.byref(self._spec), C.byref(f), C.byref(out))
        return _decision_from_c(out)


def schedule(policy: SchedulerPolicy, features: ScheduleFeatures, bounds: ChunkBounds,
             cal: CalibrationRef) -> ChunkDecision:
    """chunk.hpp:379-385."""
    return Scheduler(policy, bounds, cal).decide(features)


# ---------------------------------------------------------------- scan.hpp
@dataclass
class ScanParams:
    """scan.hpp:24-44."""
    channels: int = 0
    state_dim: int = 0
    seq_len: int = 0
    a: np.ndarray = field(default_factory=lambda: np.zeros(0))
    b: np.ndarray = field(default_factory=lambda: np.zeros(0))
    c: np.ndarray = field(default_factory=lambda: np.zeros(0))
    d: np.ndarray = field(default_factory=lambda: np.zeros(0))
    x: np.ndarray = field(default_factory=lambda: np.zeros(0))


@dataclass
class ScanState:
    h: np.ndarray = field(default_factory=lambda: np.zeros(0))


@dataclass
class ScanOutput:
    y: np.ndarray = field(default_factory=lambda: np.zeros(0))


def _validate_scan_shapes(p: ScanParams) -> None:
    """validate_scan_params (scan.hpp:54-69), shape part; finiteness is checked on the GPU."""
    if p.channels == 0 or p.state_dim == 0 or p.seq_len == 0:
        raise InvalidInput("shape mismatch")
    cs = p.channels * p.state_dim
    sz = {k: np.asarray(getattr(p, k)).size for k in "abcdx"}
    if sz["a"] not in (cs, p.seq_len * cs):
        raise InvalidInput("shape mismatch")
    if sz["b"] not in (p.state_dim, p.seq_len * p.state_dim):
        raise InvalidInput("shape mismatch")
    if sz["c"] not in (p.state_dim, p.seq_len * p.state_dim):
        raise InvalidInput("shape mismatch")
    if sz["d"] != p.channels or sz["x"] != p.channels * p.seq_len:
        raise InvalidInput("shape mismatch")


def _scan(p: ScanParams, h0: ScanState, chunk: int, ctx: Optional[Context]):
    ctx = ctx or Context.get()
    _validate_scan_shapes(p)
    arrs = [_as_f64(getattr(p, k)) for k in "abcdx"]
    q = _lib.cl_scan_params_f64(int(p.channels), int(p.state_dim), int(p.seq_len),
                                *[a.ctypes.data for a in arrs], *[a.size for a in arrs])
    cs = int(p.channels) * int(p.state_dim)
    h0a = None
    if h0 is not None and np.asarray(h0.h).size:
        h0a = _as_f64(h0.h)
        if h0a.size != cs:
            raise InvalidInput("shape mismatch")
    y = np.empty(max(int(p.channels) * int(p.seq_len), 1))
    h = np.empty(max(cs, 1))
    ctx.call("cl_scan_f64_host", C.byref(q), None if h0a is None else h0a.ctypes.data,
             int(chunk), y.ctypes.data, h.ctypes.data)
    return ScanOutput(y[: int(p.channels) * int(p.seq_len)]), ScanState(h[:cs])


def scan_sequential(p: ScanParams, h0: ScanState = None, ctx: Optional[Context] = None):
    """scan.hpp:113-121 (fp64 on the GPU, bit-identical)."""
    return _scan(p, h0, 0, ctx)


def scan_chunked(p: ScanParams, h0: ScanState, chunk: int, ctx: Optional[Context] = None):
    """scan.hpp:123-136: validate, then reject chunk < 1, then run windows."""
    _validate_scan_shapes(p)
    if chunk < 1:
        raise InvalidInput("chunk must be >= 1")
    return _scan(p, h0, chunk, ctx)
