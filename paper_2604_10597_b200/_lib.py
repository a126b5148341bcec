"""ctypes binding of libchunklab_b200.so (include/chunklab_capi.h).

The library is the product; this module only marshals arguments.  Loading fails
loudly when the .so is missing or no sm_100 device is present: there is no CPU
fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CHUNKLAB_LIB", os.path.join(PKG, "libchunklab_b200.so"))

CL_OK, CL_E_INVALID, CL_E_CUDA, CL_E_DEVICE, CL_E_NOMEM = range(5)
CL_RANGE_DYNAMIC, CL_RANGE_FIXED = 0, 1
(CL_POL_STATIC, CL_POL_MIDPOINT, CL_POL_FULL_HIST, CL_POL_SAMPLED_HIST, CL_POL_LEARNED_TABLE,
 CL_POL_GUARDED, CL_POL_RULE, CL_POL_TOKEN_HIST) = range(8)
CL_SRC_GUARDED, CL_SRC_GUARDED_FALLBACK = 16, 32
CL_SCAN_AUTO, CL_SCAN_ROWSEQ_TMA, CL_SCAN_GENERIC, CL_SCAN_LOOKBACK, CL_SCAN_CHAINED = range(5)
CL_SCAN_CONFIG_BASE, CL_SCAN_LOOKBACK_BASE = 16, 64
CL_GATHER_MIN_STRIDE = 4  # cl_prefill_f32 gathers the samples for sample_stride >= this
CL_KERNEL_GENERIC, CL_KERNEL_CHAINED, CL_KERNEL_ROWSEQ, CL_KERNEL_LOOKBACK = range(4)
KERNEL_NAMES = {0: "generic_kernel", 1: "rowpair_ws_kernel", 2: "rowseq_tma_kernel",
                3: "lookback_ws_kernel"}

SOURCE_NAMES = {0: "static", 1: "no_entropy_midpoint", 2: "full_histogram",
                3: "sampled_histogram", 4: "learned_table", 6: "rule", 7: "token_histogram"}


def source_tag(code: int) -> str:
    if code == CL_SRC_GUARDED_FALLBACK:
        return "guarded[fallback]"
    if code >= CL_SRC_GUARDED:
        return "guarded[" + SOURCE_NAMES[code - CL_SRC_GUARDED] + "]"
    return SOURCE_NAMES[code]


class cl_hist_spec(C.Structure):
    _fields_ = [("bin_count", C.c_int), ("epsilon", C.c_double), ("range_mode", C.c_int),
                ("fixed_lo", C.c_double), ("fixed_hi", C.c_double),
                ("sample_stride", C.c_uint64)]


class cl_rule_spec(C.Structure):
    _fields_ = [("kind", C.c_int), ("static_chunk", C.c_int), ("inner_kind", C.c_int),
                ("inner_static_chunk", C.c_int), ("safe_chunk", C.c_int),
                ("min_delta_buckets", C.c_int), ("threshold_tokens", C.c_uint64),
                ("short_chunk", C.c_int), ("long_chunk", C.c_int), ("n_buckets", C.c_int),
                ("buckets", C.c_int * 16), ("c_min", C.c_int), ("c_max", C.c_int),
                ("h_ref_nats", C.c_double)]


class cl_decision(C.Structure):
    _fields_ = [("status", C.c_int32), ("chunk", C.c_int32), ("source", C.c_int32),
                ("bin_count", C.c_int32), ("r", C.c_double), ("signal_nats", C.c_double),
                ("raw_nats", C.c_double), ("normalized", C.c_double), ("lo", C.c_double),
                ("hi", C.c_double), ("sample_count", C.c_uint64), ("margin", C.c_double)]


class cl_features(C.Structure):
    _fields_ = [("has_full_entropy", C.c_int), ("full_entropy_nats", C.c_double),
                ("has_sampled_entropy", C.c_int), ("sampled_entropy_nats", C.c_double),
                ("has_seq_len", C.c_int), ("seq_len", C.c_uint64),
                ("has_token_entropy", C.c_int), ("token_entropy_nats", C.c_double)]


class cl_mamba1_args(C.Structure):
    _fields_ = [("u", C.c_void_p), ("delta", C.c_void_p), ("A", C.c_void_p), ("B", C.c_void_p),
                ("C", C.c_void_p), ("D", C.c_void_p), ("z", C.c_void_p),
                ("delta_bias", C.c_void_p), ("h0", C.c_void_p), ("out", C.c_void_p),
                ("h_last", C.c_void_p), ("batch", C.c_uint64), ("dim", C.c_uint64),
                ("seq_len", C.c_uint64), ("d_state", C.c_uint64), ("delta_softplus", C.c_int)]


class cl_state_update_args(C.Structure):
    _fields_ = [("state", C.c_void_p), ("x", C.c_void_p), ("dt", C.c_void_p), ("A", C.c_void_p),
                ("B", C.c_void_p), ("C", C.c_void_p), ("D", C.c_void_p), ("z", C.c_void_p),
                ("dt_bias", C.c_void_p), ("out", C.c_void_p), ("batch", C.c_uint64),
                ("dim", C.c_uint64), ("d_state", C.c_uint64), ("dt_softplus", C.c_int)]


class cl_scan_plan(C.Structure):
    _fields_ = [("kernel", C.c_int), ("config", C.c_int), ("box", C.c_int), ("warps", C.c_int),
                ("stages", C.c_int), ("n_seg", C.c_int), ("seg_len", C.c_int)]


class cl_conv_args(C.Structure):
    _fields_ = [("x", C.c_void_p), ("weight", C.c_void_p), ("bias", C.c_void_p),
                ("width", C.c_int), ("silu", C.c_int)]


class cl_shard(C.Structure):
    _fields_ = [("global_batch", C.c_uint64), ("global_dim", C.c_uint64), ("b0", C.c_uint64),
                ("b1", C.c_uint64), ("d0", C.c_uint64), ("d1", C.c_uint64)]


_MAXF64 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
_SUMU64 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
_SUMU32 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class cl_collectives(C.Structure):
    _fields_ = [("allreduce_max_f64", _MAXF64), ("allreduce_sum_u64", _SUMU64),
                ("allreduce_sum_u32", _SUMU32), ("user", C.c_void_p)]


class cl_scan_params_f64(C.Structure):
    _fields_ = [("channels", C.c_uint64), ("state_dim", C.c_uint64), ("seq_len", C.c_uint64),
                ("a", C.c_void_p), ("b", C.c_void_p), ("c", C.c_void_p), ("d", C.c_void_p),
                ("x", C.c_void_p), ("a_len", C.c_uint64), ("b_len", C.c_uint64),
                ("c_len", C.c_uint64), ("d_len", C.c_uint64), ("x_len", C.c_uint64)]


_P = C.c_void_p
_u64 = C.c_uint64

# name -> (restype, argtypes); the list IS the exported surface of include/chunklab_capi.h.
SIGNATURES = {
    "cl_abi_version": (C.c_int, []),
    "cl_ctx_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "cl_ctx_destroy": (C.c_int, [_P]),
    "cl_last_error": (C.c_char_p, [_P]),
    "cl_launch_count": (C.c_uint64, [_P]),
    "cl_validate_hist_spec": (C.c_int, [_P, C.POINTER(cl_hist_spec)]),
    "cl_validate_rule": (C.c_int, [_P, C.POINTER(cl_rule_spec)]),
    "cl_range_init": (C.c_int, [_P, _P, _P]),
    "cl_minmax_f32": (C.c_int, [_P, _P, _u64, _u64, _u64, _P, _P]),
    "cl_minmax_gather_f32": (C.c_int, [_P, _P, _u64, _u64, _u64, _P, _P, _P]),
    "cl_samples_in": (_u64, [_u64, _u64, _u64]),
    "cl_minmax_f64": (C.c_int, [_P, _P, _u64, _u64, _u64, _P, _P]),
    "cl_conv1d_f32": (C.c_int, [_P, _P, _P, _P, _P, _u64, _u64, _u64, C.c_int, C.c_int, _u64,
                                _u64, _P, _P]),
    "cl_counts_zero": (C.c_int, [_P, _P, C.c_int, _P]),
    "cl_prefill_init": (C.c_int, [_P, _P, _P, C.c_int, _P]),
    "cl_prefill_init_prepare_f32": (C.c_int, [_P, _P, _P, C.c_int, C.POINTER(cl_mamba1_args), _P]),
    "cl_histogram_f32": (C.c_int, [_P, _P, _u64, _u64, C.POINTER(cl_hist_spec), _P, _P, _P]),
    "cl_histogram_f64": (C.c_int, [_P, _P, _u64, _u64, C.POINTER(cl_hist_spec), _P, _P, _P]),
    "cl_entropy_lean_f32": (C.c_int, [_P, _P, _u64, C.POINTER(cl_hist_spec),
                                      C.POINTER(cl_rule_spec), _u64, _P, _P, _P, _P]),
    "cl_decide": (C.c_int, [_P, _P, _P, C.POINTER(cl_hist_spec), _u64, C.POINTER(cl_rule_spec),
                            _u64, _P, _P]),
    "cl_histogram_decide_f32": (C.c_int, [_P, _P, _u64, C.POINTER(cl_hist_spec), _P, _P,
                                          C.POINTER(cl_rule_spec), _u64, _P, _P]),
    "cl_token_entropy_f32": (C.c_int, [_P, _P, _u64, _u64, C.POINTER(cl_hist_spec), _P, _P]),
    "cl_token_range_init": (C.c_int, [_P, _P, _u64, _P]),
    "cl_token_minmax_f32": (C.c_int, [_P, _P, _u64, _u64, _u64, _u64, _P, _P]),
    "cl_token_histogram_f32": (C.c_int, [_P, _P, _u64, _u64, _u64, C.POINTER(cl_hist_spec), _P,
                                         _P, _P]),
    "cl_token_entropy_counts": (C.c_int, [_P, _P, _P, _u64, _u64, C.POINTER(cl_hist_spec), _P,
                                          _P]),
    "cl_decide_token": (C.c_int, [_P, _P, C.POINTER(cl_hist_spec), C.POINTER(cl_rule_spec), _u64,
                                  _P, _P]),
    "cl_selective_scan_f32": (C.c_int, [_P, C.POINTER(cl_mamba1_args), _P, C.c_int, C.c_int,
                                        _P]),
    "cl_selective_state_update_f32": (C.c_int, [_P, C.POINTER(cl_state_update_args), _P]),
    "cl_scan_plan_f32": (C.c_int, [_P, C.POINTER(cl_mamba1_args), C.c_int, C.POINTER(cl_scan_plan)]),
    "cl_prefill_f32": (C.c_int, [_P, C.POINTER(cl_mamba1_args), C.POINTER(cl_hist_spec),
                                 C.POINTER(cl_rule_spec), _P, _P, _P, _P]),
    "cl_decision_check": (C.c_int, [_P, _P, C.POINTER(cl_decision), _P]),
    "cl_collectives_nccl": (C.c_int, [_P, C.POINTER(cl_collectives)]),
    "cl_prefill_from_conv_f32": (C.c_int, [_P, C.POINTER(cl_conv_args), C.POINTER(cl_mamba1_args),
                                           C.POINTER(cl_hist_spec), C.POINTER(cl_rule_spec),
                                           _P, _P, _P, _P]),
    "cl_prefill_sharded_f32": (C.c_int, [_P, C.POINTER(cl_mamba1_args), C.POINTER(cl_shard),
                                         C.POINTER(cl_hist_spec), C.POINTER(cl_rule_spec),
                                         C.POINTER(cl_collectives), _P, _P, _P, _P]),
    "cl_scan_f64": (C.c_int, [_P, C.POINTER(cl_scan_params_f64), _P, _u64, _P, _P, _P]),
    "cl_all_finite_host": (C.c_int, [_P, _P, _u64, C.POINTER(C.c_int)]),
    "cl_compute_histogram_host": (C.c_int, [_P, _P, _u64, C.POINTER(cl_hist_spec), _P, _P,
                                            C.POINTER(C.c_double), C.POINTER(C.c_double),
                                            C.POINTER(C.c_uint64)]),
    "cl_token_entropy_host": (C.c_int, [_P, _P, _u64, _u64, C.POINTER(cl_hist_spec),
                                        C.POINTER(C.c_double), C.POINTER(C.c_double),
                                        C.POINTER(C.c_uint64)]),
    "cl_estimate_entropy_host": (C.c_int, [_P, _P, C.c_int, C.c_double, C.POINTER(C.c_double),
                                           C.POINTER(C.c_double)]),
    "cl_schedule_host": (C.c_int, [_P, C.POINTER(cl_rule_spec), C.POINTER(cl_features),
                                   C.POINTER(cl_decision)]),
    "cl_scan_f64_host": (C.c_int, [_P, C.POINTER(cl_scan_params_f64), _P, _u64, _P, _P]),
}

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load (once) and type the C-ABI library.  Raises if it is missing."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build it with `python -m paper_2604_10597_b200.build` "
                "(nvcc, sm_100a).  There is no CPU fallback.")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class InvalidInput(ValueError):
    """Mirror of chunklab::invalid_input (common.hpp:15-18); message is verbatim."""


class DeviceError(RuntimeError):
    pass


class Context:
    """Owns one cl_ctx per CUDA device."""

    _per_device: dict = {}
    _lock = threading.Lock()

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        rc = self.lib.cl_ctx_create(device, C.byref(h))
        if rc != CL_OK:
            raise DeviceError(self.lib.cl_last_error(None).decode())
        self.handle = h
        self.device = device

    @classmethod
    def get(cls, device: int | None = None) -> "Context":
        if device is None:
            import torch
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        with cls._lock:
            ctx = cls._per_device.get(device)
            if ctx is None:
                ctx = cls(device)
                cls._per_device[device] = ctx
            return ctx

    def check(self, rc: int):
        if rc == CL_OK:
            return
        msg = self.lib.cl_last_error(self.handle).decode()
        if rc == CL_E_INVALID:
            raise InvalidInput(msg)
        if rc == CL_E_DEVICE:
            raise InvalidInput(msg)
        raise DeviceError(msg)

    def call(self, name, *args):
        self.check(getattr(self.lib, name)(self.handle, *args))

    @property
    def launches(self) -> int:
        return int(self.lib.cl_launch_count(self.handle))

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.lib.cl_ctx_destroy(self.handle)
        except Exception:
            pass
