"""Multi-GPU COREY prefill: rows of the (batch*d_inner, L) flattening sharded over
torch.distributed ranks (one process per GPU, NCCL over NVLink on the B200 box).

SURVEY.md 8(e).  The scan needs no communication (rows are independent).  The
entropy estimate is global and needs exactly two tiny collectives per layer call:

  1. MAX-allreduce of the 4-double range buffer {-lo, hi, nonfinite, 0} after each
     rank's strided min/max over its rows (Dynamic range must be global before any
     sample is binned -- the north star names only the count allreduce; this one is
     required for bit-exact global counts);
  2. SUM-allreduce of the K uint64 counts (carried as int64: counts < 2^63).

Every rank then runs the identical device decision on identical inputs, so every
rank derives the identical chunk with no broadcast.  Stride sampling uses each
row's GLOBAL flat index, so sharded counts equal single-GPU counts bit for bit.

The TokenHistogram policy (token_entropy, entropy.hpp:180-210: one histogram per
position over all channels) has the same two-collective shape with per-position
buffers: MAX-allreduce of the [2L+1] per-position range {-lo[L], hi[L], nonfinite},
then SUM-allreduce of the [L][K] counts (uint32, carried as int32: counts per
position are at most the total channel count, < 2^31).  Channels are sampled by
GLOBAL row index.

The protocol is written against a small stage interface so that the same host
logic runs with the B200 kernels (`DeviceStages`) and, in the CPU tests, with a
test-only implementation over gloo.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Protocol, Sequence

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Segment:
    """A contiguous run of rows of one batch owned by this rank.

    local_offset / global_offset are flat element offsets (row * L)."""
    batch: int
    d0: int
    d1: int
    local_offset: int
    global_offset: int
    numel: int


@dataclass(frozen=True)
class ShardPlan:
    rank: int
    world: int
    batch: int
    dim: int
    seq_len: int
    b0: int        # first batch owned (batch split) or 0 (dim split)
    b1: int
    d0: int        # channel range owned
    d1: int
    segments: Sequence[Segment]

    @property
    def local_batch(self) -> int:
        return self.b1 - self.b0

    @property
    def local_dim(self) -> int:
        return self.d1 - self.d0

    @property
    def global_numel(self) -> int:
        return self.batch * self.dim * self.seq_len


def plan_rows(batch: int, dim: int, seq_len: int, rank: int, world: int) -> ShardPlan:
    """Whole batches per rank when world divides batch (C3/C4), otherwise a
    contiguous d_inner range of every batch (C1/C2; B and C replicated)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    L = seq_len
    if batch % world == 0:
        per = batch // world
        b0, b1 = rank * per, (rank + 1) * per
        seg = Segment(b0, 0, dim, 0, b0 * dim * L, per * dim * L)
        return ShardPlan(rank, world, batch, dim, L, b0, b1, 0, dim, [seg])
    if dim % world != 0:
        raise ValueError("neither batch nor d_inner divisible by world size")
    per = dim // world
    d0, d1 = rank * per, (rank + 1) * per
    segs: List[Segment] = []
    for b in range(batch):
        segs.append(Segment(b, d0, d1, b * per * L, (b * dim + d0) * L, per * L))
    return ShardPlan(rank, world, batch, dim, L, 0, batch, d0, d1, segs)


class Stages(Protocol):
    """Per-rank stage kernels (device path: DeviceStages)."""
    range: torch.Tensor   # float64[4]
    counts: torch.Tensor  # int64[K]

    def range_init(self) -> None: ...
    def minmax(self, flat: torch.Tensor, global_offset: int) -> None: ...
    def counts_zero(self) -> None: ...
    def histogram(self, flat: torch.Tensor, global_offset: int) -> None: ...
    def decide(self, n_samples_total: int, seq_len: int) -> None: ...


def n_samples(numel: int, stride: int) -> int:
    return (numel + stride - 1) // stride


def sharded_entropy_decision(stages: Stages, u_local_flat: torch.Tensor, plan: ShardPlan,
                             stride: int, group=None) -> None:
    """Run the global entropy estimate + decision over the ranks of `group`.
    Afterwards every rank holds the identical decision in its stage buffers."""
    stages.range_init()
    for s in plan.segments:
        stages.minmax(u_local_flat[s.local_offset:s.local_offset + s.numel], s.global_offset)
    if plan.world > 1:
        dist.all_reduce(stages.range, op=dist.ReduceOp.MAX, group=group)
    stages.counts_zero()
    for s in plan.segments:
        stages.histogram(u_local_flat[s.local_offset:s.local_offset + s.numel], s.global_offset)
    if plan.world > 1:
        dist.all_reduce(stages.counts, op=dist.ReduceOp.SUM, group=group)
    stages.decide(n_samples(plan.global_numel, stride), plan.seq_len)


class TokenStages(Protocol):
    """Per-rank token_entropy stage kernels (device path: DeviceStages)."""
    trange: torch.Tensor   # float64[2L + 1]
    tcounts: torch.Tensor  # int32[L * K]

    def token_range_init(self) -> None: ...
    def token_minmax(self, flat: torch.Tensor, channels: int, channel_offset: int) -> None: ...
    def token_counts_zero(self) -> None: ...
    def token_histogram(self, flat: torch.Tensor, channels: int, channel_offset: int) -> None: ...
    def token_decide(self, samples_per_position: int, seq_len: int) -> None: ...


def sharded_token_decision(stages: TokenStages, u_local_flat: torch.Tensor, plan: ShardPlan,
                           stride: int, group=None) -> None:
    """token_entropy over the ranks of `group` (channels = rows of (batch*d_inner), sampled
    by GLOBAL row index) + the identical device decision on every rank."""
    L = plan.seq_len
    stages.token_range_init()
    for s in plan.segments:
        stages.token_minmax(u_local_flat[s.local_offset:s.local_offset + s.numel], s.numel // L,
                            s.global_offset // L)
    if plan.world > 1:
        dist.all_reduce(stages.trange, op=dist.ReduceOp.MAX, group=group)
    stages.token_counts_zero()
    for s in plan.segments:
        stages.token_histogram(u_local_flat[s.local_offset:s.local_offset + s.numel],
                               s.numel // L, s.global_offset // L)
    if plan.world > 1:
        dist.all_reduce(stages.tcounts, op=dist.ReduceOp.SUM, group=group)
    stages.token_decide(n_samples(plan.batch * plan.dim, stride), L)


class DeviceStages:
    """The B200 kernels behind the Stages / TokenStages interfaces (wraps mamba1.Prefill)."""

    def __init__(self, prefill):
        self.pf = prefill
        self.range = prefill.range
        self.counts = prefill.counts

    def range_init(self):
        from ._lib import Context  # noqa: F401
        self.pf.ctx.call("cl_range_init", self.pf.range.data_ptr(),
                         torch.cuda.current_stream(self.pf.device).cuda_stream)

    def minmax(self, flat, global_offset):
        self.pf.stage_minmax(flat, global_offset, init=False)

    def counts_zero(self):
        self.pf.ctx.call("cl_counts_zero", self.pf.counts.data_ptr(),
                         int(self.pf.spec.bin_count),
                         torch.cuda.current_stream(self.pf.device).cuda_stream)

    def histogram(self, flat, global_offset):
        self.pf.stage_histogram(flat, global_offset, zero=False)

    def decide(self, n_samples_total, seq_len):
        self.pf.stage_decide(n_samples_total, seq_len)

    # -- token_entropy stages (buffers sized on first use for this seq_len) --
    def _token_buffers(self, L):
        k = int(self.pf.spec.bin_count)
        if getattr(self, "trange", None) is None or self.trange.numel() != 2 * L + 1:
            self.trange = torch.empty(2 * L + 1, dtype=torch.float64, device=self.pf.device)
            self.tcounts = torch.zeros(L * k, dtype=torch.int32, device=self.pf.device)
            self._L = L

    def _s(self):
        return torch.cuda.current_stream(self.pf.device).cuda_stream

    def token_range_init(self):
        self.pf.ctx.call("cl_token_range_init", self.trange.data_ptr(), self._L, self._s())

    def token_minmax(self, flat, channels, channel_offset):
        self.pf.ctx.call("cl_token_minmax_f32", flat.data_ptr(), int(channels), self._L,
                         int(channel_offset), int(self.pf.spec.sample_stride),
                         self.trange.data_ptr(), self._s())

    def token_counts_zero(self):
        self.tcounts.zero_()

    def token_histogram(self, flat, channels, channel_offset):
        import ctypes as C
        self.pf.ctx.call("cl_token_histogram_f32", flat.data_ptr(), int(channels), self._L,
                         int(channel_offset), C.byref(self.pf.cspec), self.trange.data_ptr(),
                         self.tcounts.data_ptr(), self._s())

    def token_decide(self, samples_per_position, seq_len):
        import ctypes as C
        self.pf.ctx.call("cl_token_entropy_counts", self.tcounts.data_ptr(),
                         self.trange.data_ptr(), self._L, int(samples_per_position),
                         C.byref(self.pf.cspec), self.pf.token_buf.data_ptr(), self._s())
        self.pf.stage_decide_token(seq_len)


class ShardedPrefill:
    """One layer's prefill over all ranks: global entropy -> identical decision ->
    local scan of this rank's rows.

    Inputs are this rank's shard: u, delta, z: (local_batch, local_dim, L);
    A, D, delta_bias: the local_dim rows; B, C: (local_batch, N, L)."""

    def __init__(self, prefill, plan: ShardPlan, group=None):
        self.pf = prefill
        self.plan = plan
        self.group = group
        self.stages = DeviceStages(prefill)

    def __call__(self, u, delta, A, B, C, D=None, z=None, delta_bias=None, delta_softplus=True,
                 out=None, return_last_state=False):
        from .mamba1 import check_scan_inputs
        check_scan_inputs(u, delta, A, B, C, D, z, delta_bias, None, out, device=self.pf.device)
        if tuple(u.shape) != (self.plan.local_batch, self.plan.local_dim, self.plan.seq_len):
            raise ValueError("u does not match the shard plan")
        if self.pf.token:
            self.stages._token_buffers(self.plan.seq_len)
            sharded_token_decision(self.stages, u.reshape(-1), self.plan,
                                   int(self.pf.spec.sample_stride), self.group)
        else:
            sharded_entropy_decision(self.stages, u.reshape(-1), self.plan,
                                     int(self.pf.spec.sample_stride), self.group)
        return self.pf.stage_scan(u, delta, A, B, C, D, z, delta_bias, delta_softplus, out,
                                  return_last_state)
