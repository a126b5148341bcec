"""Device path of the COREY prefill: entropy -> rule -> fused Mamba-1 scan on the B200.

Tensors are torch CUDA tensors (torch is used for device memory, streams and
torch.distributed only).  Every stage is a kernel in libchunklab_b200.so launched on
torch's current stream; no stage synchronises with the host, so the chunk chosen by
the device rule flows into the scan through device memory (the host sync of the
paper's Python hook, is gone).

  selective_scan_fn   mamba_ssm's public interface + chunk_size
  Prefill             entropy (K-bin, entropy.hpp) -> policy (chunk.hpp) -> scan
  ShardedPrefill      the same over torch.distributed ranks: rows of (batch*dim) are
                      sharded, MAX-allreduce of the range and SUM-allreduce of the
                      K counts are the only collectives
"""
from __future__ import annotations

import copy as _copy
import ctypes as C
from dataclasses import dataclass
from typing import Optional

import torch

from . import _lib
from ._lib import Context, InvalidInput
from .chunklab import (CalibrationRef, ChunkBounds, ChunkDecision, EntropyEstimate,
                       HistogramSpec, SchedulerPolicy, rule_spec)

_VARIANTS = {"auto": _lib.CL_SCAN_AUTO, "rowseq_tma": _lib.CL_SCAN_ROWSEQ_TMA,
             "generic": _lib.CL_SCAN_GENERIC, "lookback": _lib.CL_SCAN_LOOKBACK,
             "chained": _lib.CL_SCAN_CHAINED}


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _check_f32(name, t, device):
    if t is None:
        return
    if not t.is_cuda or t.device != device:
        raise InvalidInput(f"{name} must be a CUDA tensor on {device}")
    if t.dtype != torch.float32:
        raise InvalidInput(f"{name} must be float32")
    if not t.is_contiguous():
        raise InvalidInput(f"{name} must be contiguous")


def check_scan_inputs(u, delta, A, B, C_, D=None, z=None, delta_bias=None, h0=None, out=None,
                      h_last=None, device=None):
    """Every tensor a contiguous float32 CUDA tensor on one device, shapes consistent.
    Runs before ANY kernel is queued: a bf16 or host tensor must never reach a launch
    (the kernels would read past the allocation or dereference a host pointer)."""
    if not isinstance(u, torch.Tensor) or u.dim() != 3:
        raise InvalidInput("u must be a (batch, dim, L) tensor")
    dev = u.device if device is None else device
    for name, t in (("u", u), ("delta", delta), ("A", A), ("B", B), ("C", C_), ("D", D),
                    ("z", z), ("delta_bias", delta_bias), ("h0", h0), ("out", out),
                    ("h_last", h_last)):
        _check_f32(name, t, dev)
    batch, dim, L = u.shape
    if A.dim() != 2:
        raise InvalidInput("shape mismatch")
    N = A.shape[1]
    if tuple(delta.shape) != (batch, dim, L) or (z is not None and tuple(z.shape) != (batch, dim, L)):
        raise InvalidInput("shape mismatch")
    if tuple(A.shape) != (dim, N) or tuple(B.shape) != (batch, N, L) or tuple(C_.shape) != (batch, N, L):
        raise InvalidInput("shape mismatch")
    for t in (D, delta_bias):
        if t is not None and t.numel() != dim:
            raise InvalidInput("shape mismatch")
    if out is not None and tuple(out.shape) != (batch, dim, L):
        raise InvalidInput("shape mismatch")
    for t in (h0, h_last):
        if t is not None and t.numel() != batch * dim * N:
            raise InvalidInput("shape mismatch")


def _mamba_args(u, delta, A, B, C_, D, z, delta_bias, h0, out, h_last, delta_softplus):
    check_scan_inputs(u, delta, A, B, C_, D, z, delta_bias, h0, out, h_last)
    batch, dim, L = u.shape
    N = A.shape[1]
    a = _lib.cl_mamba1_args()
    a.u, a.delta, a.A, a.B, a.C = _ptr(u), _ptr(delta), _ptr(A), _ptr(B), _ptr(C_)
    a.D, a.z, a.delta_bias, a.h0 = _ptr(D), _ptr(z), _ptr(delta_bias), _ptr(h0)
    a.out, a.h_last = _ptr(out), _ptr(h_last)
    a.batch, a.dim, a.seq_len, a.d_state = batch, dim, L, N
    a.delta_softplus = int(bool(delta_softplus))
    return a


def selective_scan_fn(u, delta, A, B, C, D=None, z=None, delta_bias=None, delta_softplus=False,
                      return_last_state=False, chunk_size: int = 512, h0=None,
                      variant: str = "auto", decision: Optional[torch.Tensor] = None,
                      out: Optional[torch.Tensor] = None):
    """mamba_ssm.selective_scan_fn semantics, fp32, on the fused sm_100a kernel.

    u, delta, z: (batch, dim, L); A: (dim, N); B, C: (batch, N, L); D, delta_bias: (dim,).
    chunk_size: L-segment length of the scan's work decomposition (the paper's runtime
    chunk).  `decision` (a device cl_decision buffer from Prefill) makes
    the kernel read the chunk from device memory instead.
    """
    check_scan_inputs(u, delta, A, B, C, D, z, delta_bias, h0, out)
    ctx = Context.get(u.device.index)
    if out is None:
        out = torch.empty_like(u)
    h_last = None
    if return_last_state:
        h_last = torch.empty(u.shape[0], u.shape[1], A.shape[1], device=u.device,
                             dtype=torch.float32)
    a = _mamba_args(u, delta, A, B, C, D, z, delta_bias, h0, out, h_last, delta_softplus)
    ctx.call("cl_selective_scan_f32", C_byref(a), _ptr(decision), int(chunk_size),
             _variant_code(variant), _stream_ptr(u.device))
    return (out, h_last) if return_last_state else out


def _variant_code(variant: str) -> int:
    """"auto" / "chained" / "lookback" / "rowseq_tma" / "generic", "cfg:<i>" for row i of
    the chained kernel table, "lb:<i>" for row i of the L-parallel kernel table."""
    if variant.startswith("cfg:"):
        return _lib.CL_SCAN_CONFIG_BASE + int(variant[4:])
    if variant.startswith("lb:"):
        return _lib.CL_SCAN_LOOKBACK_BASE + int(variant[3:])
    return _VARIANTS[variant]


def scan_plan(u, delta, A, B, C, D=None, z=None, delta_bias=None, delta_softplus=True,
              variant: str = "auto", h0=None, out=None, return_last_state=False) -> dict:
    """The kernel selective_scan_fn would run (cl_scan_plan_f32; no launch)."""
    check_scan_inputs(u, delta, A, B, C, D, z, delta_bias, h0, out)
    out = torch.empty_like(u) if out is None else out
    h_last = (torch.empty(u.shape[0], u.shape[1], A.shape[1], device=u.device)
              if return_last_state else None)
    a = _mamba_args(u, delta, A, B, C, D, z, delta_bias, h0, out, h_last, delta_softplus)
    p = _lib.cl_scan_plan()
    Context.get(u.device.index).call("cl_scan_plan_f32", C_byref(a), _variant_code(variant),
                                     C_byref(p))
    return {"kernel": _lib.KERNEL_NAMES[p.kernel], "config": p.config, "box": p.box,
            "warps": p.warps, "stages": p.stages, "n_seg": p.n_seg, "seg_len": p.seg_len}


def selective_state_update(state, x, dt, A, B, C, D=None, z=None, dt_bias=None,
                           dt_softplus=False, out: Optional[torch.Tensor] = None):
    """mamba_ssm.selective_state_update semantics (decode: one token), fp32, state updated
    in place.  state (batch, dim, N); x, dt, z (batch, dim); A (dim, N); B, C (batch, N).
    Bitwise consistent with selective_scan_fn: prefill(L) + k steps == prefill(L + k)."""
    dev = state.device
    batch, dim, N = state.shape
    for name, t in (("state", state), ("x", x), ("dt", dt), ("A", A), ("B", B), ("C", C),
                    ("D", D), ("z", z), ("dt_bias", dt_bias), ("out", out)):
        _check_f32(name, t, dev)
    if tuple(x.shape) != (batch, dim) or tuple(dt.shape) != (batch, dim):
        raise InvalidInput("shape mismatch")
    if tuple(A.shape) != (dim, N) or tuple(B.shape) != (batch, N) or tuple(C.shape) != (batch, N):
        raise InvalidInput("shape mismatch")
    if z is not None and tuple(z.shape) != (batch, dim):
        raise InvalidInput("shape mismatch")
    for t in (D, dt_bias):
        if t is not None and t.numel() != dim:
            raise InvalidInput("shape mismatch")
    out = torch.empty_like(x) if out is None else out
    a = _lib.cl_state_update_args()
    a.state, a.x, a.dt, a.A, a.B, a.C = (state.data_ptr(), x.data_ptr(), dt.data_ptr(),
                                         A.data_ptr(), B.data_ptr(), C.data_ptr())
    a.D, a.z, a.dt_bias, a.out = _ptr(D), _ptr(z), _ptr(dt_bias), out.data_ptr()
    a.batch, a.dim, a.d_state, a.dt_softplus = batch, dim, N, int(bool(dt_softplus))
    # (the parameter C shadows the ctypes module here: C_byref is module level)
    Context.get(dev.index).call("cl_selective_state_update_f32", C_byref(a), _stream_ptr(dev))
    return out


def causal_conv1d_fn(x, weight, bias=None, activation: Optional[str] = "silu",
                     out: Optional[torch.Tensor] = None, range_buf: Optional[torch.Tensor] = None,
                     global_offset: int = 0, stride: int = 1):
    """causal_conv1d_fn(x, weight, bias, activation) semantics (fp32) on the sm_100a kernel.

    x (batch, dim, L), weight (dim, width <= 4), bias (dim,).  With range_buf (4 fp64,
    initialised by cl_range_init) the kernel also runs the entropy stage-1 min/max over
    the u it produces (producer fusion)."""
    dev = x.device
    _check_f32("x", x, dev)
    _check_f32("weight", weight, dev)
    _check_f32("bias", bias, dev)
    if activation not in (None, "silu", "swish"):
        raise InvalidInput("activation must be None, 'silu' or 'swish'")
    batch, dim, L = x.shape
    if weight.dim() != 2 or weight.shape[0] != dim or (bias is not None and bias.numel() != dim):
        raise InvalidInput("shape mismatch")
    out = torch.empty_like(x) if out is None else out
    _check_f32("out", out, dev)
    ctx = Context.get(dev.index)
    ctx.call("cl_conv1d_f32", x.data_ptr(), weight.data_ptr(), _ptr(bias), out.data_ptr(),
             batch, dim, L, int(weight.shape[1]), int(activation is not None), int(global_offset),
             int(stride), _ptr(range_buf), _stream_ptr(dev))
    return out


def C_byref(x):
    return C.byref(x)


@dataclass
class PrefillResult:
    out: torch.Tensor
    h_last: Optional[torch.Tensor]
    decision_buf: torch.Tensor  # raw cl_decision bytes on the device

    def decision(self) -> "DecisionRecord":
        """Sync point: copy the device decision back; raise deferred device errors."""
        return read_decision(self.decision_buf)


@dataclass
class DecisionRecord:
    decision: ChunkDecision
    entropy: EntropyEstimate
    lo: float
    hi: float


def read_decision(buf: torch.Tensor) -> DecisionRecord:
    ctx = Context.get(buf.device.index)
    d = _lib.cl_decision()
    ctx.call("cl_decision_check", buf.data_ptr(), C.byref(d), _stream_ptr(buf.device))
    dec = ChunkDecision(chunk=int(d.chunk), r=float(d.r), source_policy=_lib.source_tag(d.source),
                        signal_nats=float(d.signal_nats), margin=float(d.margin))
    ent = EntropyEstimate(raw_nats=float(d.raw_nats), normalized=float(d.normalized),
                          bin_count=int(d.bin_count), sample_count=int(d.sample_count))
    return DecisionRecord(dec, ent, float(d.lo), float(d.hi))


class Prefill:
    """One Mamba-1 layer's COREY prefill on one GPU:
    K-bin entropy of u -> scheduler policy -> chunked fused scan, stream-ordered.

    policy=None uses the bare calibrated rule (select_chunk); otherwise any device
    policy (Static / FullHistogram / SampledHistogram / Guarded / LearnedTable).
    """

    def __init__(self, spec: HistogramSpec = None, policy: Optional[SchedulerPolicy] = None,
                 bounds: ChunkBounds = None, cal: CalibrationRef = None, device=None):
        self.spec = spec or HistogramSpec()
        self.bounds = bounds or ChunkBounds()
        self.cal = cal or CalibrationRef.log_k(self.spec.bin_count)
        self.policy = policy
        idx = None if device is None else torch.device(device).index
        # 'cuda' without an index means the current device, as everywhere in torch
        self.device = torch.device("cuda", torch.cuda.current_device() if idx is None else idx)
        self.ctx = Context.get(self.device.index)
        self.cspec = self.spec.to_c()
        self.rule = rule_spec(policy, self.bounds, self.cal)
        self.ctx.call("cl_validate_hist_spec", C.byref(self.cspec))
        self.ctx.call("cl_validate_rule", C.byref(self.rule))
        k = self.spec.bin_count
        self.counts = torch.zeros(k, dtype=torch.int64, device=self.device)
        self.range = torch.zeros(4, dtype=torch.float64, device=self.device)
        self.decision_buf = torch.zeros(C.sizeof(_lib.cl_decision), dtype=torch.uint8,
                                        device=self.device)
        # TokenHistogram (or Guarded{inner TokenHistogram}): per-position entropy instead
        kind = self.rule.inner_kind if self.rule.kind == _lib.CL_POL_GUARDED else self.rule.kind
        self.token = kind == _lib.CL_POL_TOKEN_HIST
        self.token_buf = torch.zeros(4, dtype=torch.float64, device=self.device)
        # scan kernel family for __call__ / from_conv-free paths ("auto": by shape; "chained"
        # makes the decided chunk the scan's segment length on every shape -- chunk sweeps)
        self.scan_variant = "auto"
        # strided sampling: the gathered samples and the stride-1 spec that bins them
        self.samples = None
        spec1 = _copy.copy(self.spec)
        spec1.sample_stride = 1
        self.cspec1 = spec1.to_c()

    # -- stages (exposed for the sharded path and for per-stage timing) --
    def stage_init(self, scan_inputs=None):
        """range_init + counts zero in one launch (cl_prefill_init); with scan_inputs
        (u, delta, A, B, C) the same launch also re-lays B / C for the following scan
        (cl_prefill_init_prepare_f32)."""
        if scan_inputs is None:
            self.ctx.call("cl_prefill_init", self.range.data_ptr(), self.counts.data_ptr(),
                          int(self.spec.bin_count), _stream_ptr(self.device))
            return
        u, delta, A, B, C_ = scan_inputs
        a = _lib.cl_mamba1_args()
        a.u, a.delta, a.A, a.B, a.C = u.data_ptr(), delta.data_ptr(), A.data_ptr(), B.data_ptr(), \
            C_.data_ptr()
        a.batch, a.dim, a.seq_len, a.d_state = u.shape[0], u.shape[1], u.shape[2], A.shape[1]
        self.ctx.call("cl_prefill_init_prepare_f32", self.range.data_ptr(), self.counts.data_ptr(),
                      int(self.spec.bin_count), C.byref(a), _stream_ptr(self.device))

    def stage_minmax(self, u_flat: torch.Tensor, global_offset: int = 0, init: bool = True):
        s = _stream_ptr(self.device)
        if init:
            self.ctx.call("cl_range_init", self.range.data_ptr(), s)
        self.ctx.call("cl_minmax_f32", u_flat.data_ptr(), u_flat.numel(), int(global_offset),
                      int(self.spec.sample_stride), self.range.data_ptr(), s)

    def stage_conv(self, x, weight, bias=None, activation="silu", out=None,
                   global_offset: int = 0, init: bool = True):
        """Producer fusion: u = causal_conv1d(x) (+ SiLU) with stage 1 in its epilogue."""
        if init:
            self.ctx.call("cl_range_init", self.range.data_ptr(), _stream_ptr(self.device))
        return causal_conv1d_fn(x, weight, bias, activation, out, self.range, global_offset,
                                int(self.spec.sample_stride))

    def stage_histogram(self, u_flat: torch.Tensor, global_offset: int = 0, zero: bool = True):
        s = _stream_ptr(self.device)
        if zero:
            self.ctx.call("cl_counts_zero", self.counts.data_ptr(), int(self.spec.bin_count), s)
        self.ctx.call("cl_histogram_f32", u_flat.data_ptr(), u_flat.numel(), int(global_offset),
                      C.byref(self.cspec), self.range.data_ptr(), self.counts.data_ptr(), s)

    def stage_token(self, u: torch.Tensor):
        """token_entropy over u viewed as (channels = B*D, length = L)."""
        L = u.shape[-1]
        self.ctx.call("cl_token_entropy_f32", u.data_ptr(), u.numel() // L, L,
                      C.byref(self.cspec), self.token_buf.data_ptr(), _stream_ptr(self.device))

    def stage_decide_token(self, seq_len: int):
        self.ctx.call("cl_decide_token", self.token_buf.data_ptr(), C.byref(self.cspec),
                      C.byref(self.rule), int(seq_len), self.decision_buf.data_ptr(),
                      _stream_ptr(self.device))

    def stage_entropy_lean(self, u_flat: torch.Tensor, seq_len: int):
        """init + min/max + histogram + decision in the lean, co-schedulable kernels
        (cl_entropy_lean_f32): for running this call's entropy under another call's scan."""
        self.ctx.call("cl_entropy_lean_f32", u_flat.data_ptr(), u_flat.numel(), C.byref(self.cspec),
                      C.byref(self.rule), int(seq_len), self.counts.data_ptr(),
                      self.range.data_ptr(), self.decision_buf.data_ptr(),
                      _stream_ptr(self.device))

    def stage_histogram_decide(self, u_flat: torch.Tensor, seq_len: int, zero: bool = True):
        """Single-GPU stages 2+3 in one launch (the histogram's last CTA decides);
        needs this call's stage_minmax (range_init) before it."""
        s = _stream_ptr(self.device)
        if zero:
            self.ctx.call("cl_counts_zero", self.counts.data_ptr(), int(self.spec.bin_count), s)
        self.ctx.call("cl_histogram_decide_f32", u_flat.data_ptr(), u_flat.numel(),
                      C.byref(self.cspec), self.range.data_ptr(), self.counts.data_ptr(),
                      C.byref(self.rule), int(seq_len), self.decision_buf.data_ptr(), s)

    def stage_entropy(self, u_flat: torch.Tensor, seq_len: int):
        """The single-GPU entropy stages after stage_init, as cl_prefill_f32 runs them:
        min/max, then histogram + decision in one launch; for sample_stride >=
        CL_GATHER_MIN_STRIDE the min/max also gathers the sampled values
        (cl_minmax_gather_f32) and the histogram reads only those."""
        self.stage_entropy_minmax(u_flat)
        self.stage_entropy_histogram(u_flat, seq_len)

    def _gathers(self) -> bool:
        return int(self.spec.sample_stride) >= _lib.CL_GATHER_MIN_STRIDE

    def stage_entropy_minmax(self, u_flat: torch.Tensor):
        """First half of stage_entropy (after stage_init)."""
        if not self._gathers():
            self.stage_minmax(u_flat, init=False)
            return
        st = int(self.spec.sample_stride)
        m = int(self.ctx.lib.cl_samples_in(0, u_flat.numel(), st))
        if self.samples is None or self.samples.numel() < m:
            self.samples = torch.empty(max(m, 1), dtype=torch.float32, device=self.device)
        self.ctx.call("cl_minmax_gather_f32", u_flat.data_ptr(), u_flat.numel(), 0, st,
                      self.range.data_ptr(), self.samples.data_ptr(), _stream_ptr(self.device))

    def stage_entropy_histogram(self, u_flat: torch.Tensor, seq_len: int):
        """Second half of stage_entropy: histogram + decision (of the gathered samples
        when stage_entropy_minmax gathered them)."""
        if not self._gathers():
            self.stage_histogram_decide(u_flat, seq_len, zero=False)
            return
        m = int(self.ctx.lib.cl_samples_in(0, u_flat.numel(), int(self.spec.sample_stride)))
        self.ctx.call("cl_histogram_decide_f32", self.samples.data_ptr(), m,
                      C.byref(self.cspec1), self.range.data_ptr(), self.counts.data_ptr(),
                      C.byref(self.rule), int(seq_len), self.decision_buf.data_ptr(),
                      _stream_ptr(self.device))

    def stage_decide(self, n_samples_total: int, seq_len: int):
        self.ctx.call("cl_decide", self.counts.data_ptr(), self.range.data_ptr(),
                      C.byref(self.cspec), int(n_samples_total), C.byref(self.rule),
                      int(seq_len), self.decision_buf.data_ptr(), _stream_ptr(self.device))

    def stage_scan(self, u, delta, A, B, C, D=None, z=None, delta_bias=None,
                   delta_softplus=True, out=None, return_last_state=False, h0=None,
                   variant="auto"):
        return selective_scan_fn(u, delta, A, B, C, D, z, delta_bias, delta_softplus,
                                 return_last_state, 0, h0, variant, self.decision_buf, out)

    def n_samples(self, n_values: int) -> int:
        st = int(self.spec.sample_stride)
        return (n_values + st - 1) // st

    def __call__(self, u, delta, A, B, C, D=None, z=None, delta_bias=None, delta_softplus=True,
                 out=None, return_last_state=False, h0=None) -> PrefillResult:
        check_scan_inputs(u, delta, A, B, C, D, z, delta_bias, h0, out, device=self.device)
        if u.numel() == 0:
            raise InvalidInput("no samples")
        if self.token:
            self.stage_token(u)
            self.stage_decide_token(u.shape[-1])
        else:
            uf = u.reshape(-1)
            self.stage_init((u, delta, A, B, C))
            self.stage_entropy(uf, u.shape[-1])
        res = self.stage_scan(u, delta, A, B, C, D, z, delta_bias, delta_softplus, out,
                              return_last_state, h0, variant=self.scan_variant)
        if return_last_state:
            o, h = res
        else:
            o, h = res, None
        return PrefillResult(o, h, self.decision_buf)

    def from_conv(self, x, conv_weight, conv_bias, delta, A, B, C, D=None, z=None,
                  delta_bias=None, delta_softplus=True, out=None, return_last_state=False,
                  h0=None, activation="silu", u=None):
        """The prefill with its producer fused (cl_prefill_from_conv_f32): u =
        act(causal_conv1d(x)) is produced with the entropy stage riding on it -- the
        min/max epilogue (Dynamic range) or the whole histogram epilogue (Fixed range) --
        then decide -> scan.  Returns (PrefillResult, u)."""
        # x stands in for u (same shape) until the conv has produced it
        check_scan_inputs(x, delta, A, B, C, D, z, delta_bias, h0, out, device=self.device)
        for name, t in (("conv_weight", conv_weight), ("conv_bias", conv_bias), ("u", u)):
            _check_f32(name, t, self.device)
        if activation not in (None, "silu", "swish"):
            raise InvalidInput("activation must be None, 'silu' or 'swish'")
        if x.numel() == 0:
            raise InvalidInput("no samples")
        if conv_weight.dim() != 2 or conv_weight.shape[0] != x.shape[1] or (
                conv_bias is not None and conv_bias.numel() != x.shape[1]):
            raise InvalidInput("shape mismatch")
        u = torch.empty_like(x) if u is None else u
        out = torch.empty_like(x) if out is None else out
        h_last = (torch.empty(x.shape[0], x.shape[1], A.shape[1], device=x.device)
                  if return_last_state else None)
        a = _mamba_args(u, delta, A, B, C, D, z, delta_bias, h0, out, h_last, delta_softplus)
        cv = _lib.cl_conv_args()  # noqa: F841
        cv.x, cv.weight, cv.bias = x.data_ptr(), conv_weight.data_ptr(), _ptr(conv_bias)
        cv.width, cv.silu = int(conv_weight.shape[1]), int(activation is not None)
        buf = self.token_buf if self.token else self.range
        # (the parameter C shadows the ctypes module here: C_byref is module level)
        self.ctx.call("cl_prefill_from_conv_f32", C_byref(cv), C_byref(a), C_byref(self.cspec),
                      C_byref(self.rule), self.counts.data_ptr(), buf.data_ptr(),
                      self.decision_buf.data_ptr(), _stream_ptr(self.device))
        return PrefillResult(out, h_last, self.decision_buf), u

    def decision(self) -> DecisionRecord:
        return read_decision(self.decision_buf)
