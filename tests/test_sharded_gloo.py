"""CPU, world_size 2 over gloo: the multi-GPU host protocol (paper_2604_10597_b200/sharded.py).

The per-rank stage computations are replaced by a test-only oracle-backed Stages
implementation; the protocol itself (row sharding, global-offset stride sampling,
MAX-allreduce of the range, SUM-allreduce of counts, identical decision on every
rank) is the product code.  Sharded counts must equal the single-process
reference counts bit for bit, for batch-split and d_inner-split plans and strides.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_10597_b200.sharded import (n_samples, plan_rows, sharded_entropy_decision,
                                           sharded_token_decision)


class OracleStages:
    """Test-only stage implementation over the CPU oracle."""

    def __init__(self, port, k, stride):
        self.port, self.k, self.stride = port, k, stride
        self.range = torch.zeros(4, dtype=torch.float64)
        self.counts = torch.zeros(k, dtype=torch.int64)
        self.chunk = None

    def range_init(self):
        self.range[:] = torch.tensor([-math.inf, -math.inf, 0.0, 0.0], dtype=torch.float64)

    def _sampled(self, flat, g0):
        idx = np.arange(flat.numel()) + g0
        return flat.numpy()[idx % self.stride == 0]

    def minmax(self, flat, g0):
        v = self._sampled(flat, g0).astype(np.float64)
        bad = 0.0 if np.isfinite(flat.numpy()).all() else 1.0
        cur = self.range.numpy()
        if v.size:
            cur[0] = max(cur[0], -v.min())
            cur[1] = max(cur[1], v.max())
        cur[2] = max(cur[2], bad)

    def counts_zero(self):
        self.counts.zero_()

    def histogram(self, flat, g0):
        v = self._sampled(flat, g0).astype(np.float64)
        if not v.size:
            return
        lo, hi = -float(self.range[0]), float(self.range[1])
        if hi > lo:
            c, *_ = self.port.histogram(v, self.k, 1e-8, 1, fixed=(lo, hi))
        else:
            c = np.zeros(self.k, dtype=np.uint64)
            c[0] = v.size
        self.counts += torch.from_numpy(c.astype(np.int64))

    def decide(self, n_total, seq_len):
        masses = self.counts.numpy().astype(np.float64) * (1.0 / n_total)
        raw, _ = self.port.entropy(masses)
        self.raw = raw
        self.chunk, _ = self.port.select_chunk(raw, 32, 512, math.log(self.k))


class OracleTokenStages:
    """Test-only token_entropy stages over the CPU oracle (per-position histograms)."""

    def __init__(self, port, k, stride, L):
        self.port, self.k, self.stride, self.L = port, k, stride, L
        self.trange = torch.zeros(2 * L + 1, dtype=torch.float64)
        self.tcounts = torch.zeros(L * k, dtype=torch.int32)
        self.raw = None

    def _rows(self, flat, channels, off):
        v = flat.numpy().reshape(channels, self.L).astype(np.float64)
        keep = (np.arange(channels) + off) % self.stride == 0
        return v, v[keep]

    def token_range_init(self):
        self.trange[:2 * self.L] = -math.inf
        self.trange[2 * self.L] = 0.0

    def token_minmax(self, flat, channels, off):
        v, samp = self._rows(flat, channels, off)
        t = self.trange.numpy()
        if not np.isfinite(v).all():
            t[2 * self.L] = 1.0
        if samp.shape[0]:
            t[:self.L] = np.maximum(t[:self.L], -samp.min(axis=0))
            t[self.L:2 * self.L] = np.maximum(t[self.L:2 * self.L], samp.max(axis=0))

    def token_counts_zero(self):
        self.tcounts.zero_()

    def token_histogram(self, flat, channels, off):
        _, samp = self._rows(flat, channels, off)
        if not samp.shape[0]:
            return
        t = self.trange.numpy()
        c = self.tcounts.numpy().reshape(self.L, self.k)
        for p in range(self.L):
            lo, hi = -t[p], t[self.L + p]
            if hi > lo:
                h, *_ = self.port.histogram(np.ascontiguousarray(samp[:, p]), self.k, 1e-8, 1,
                                            fixed=(lo, hi))
            else:
                h = np.zeros(self.k, dtype=np.uint64)
                h[0] = samp.shape[0]
            c[p] += h.astype(np.int32)

    def token_decide(self, samples_per_position, seq_len):
        c = self.tcounts.numpy().reshape(self.L, self.k)
        raw_sum = 0.0
        for p in range(self.L):
            raw, _ = self.port.entropy(c[p].astype(np.float64) * (1.0 / samples_per_position))
            raw_sum += raw
        self.raw = raw_sum / self.L


def _token_worker(rank, world, port_no, batch, dim, L, stride, k, seed, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    port = O.Port()
    rng = np.random.default_rng(seed)
    u = rng.standard_normal((batch, dim, L)).astype(np.float32)
    plan = plan_rows(batch, dim, L, rank, world)
    local = u[plan.b0:plan.b1, plan.d0:plan.d1, :].copy()
    st = OracleTokenStages(port, k, stride, L)
    sharded_token_decision(st, torch.from_numpy(local).reshape(-1), plan, stride)
    out_q.put((rank, st.tcounts.numpy().copy(), st.raw))
    dist.destroy_process_group()


def _worker(rank, world, port_no, batch, dim, L, stride, k, seed, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    port = O.Port()
    rng = np.random.default_rng(seed)
    u = rng.standard_normal((batch, dim, L)).astype(np.float32)
    plan = plan_rows(batch, dim, L, rank, world)
    local = u[plan.b0:plan.b1, plan.d0:plan.d1, :].copy()
    st = OracleStages(port, k, stride)
    sharded_entropy_decision(st, torch.from_numpy(local).reshape(-1), plan, stride)
    out_q.put((rank, st.counts.numpy().copy(), st.range.numpy().copy(), st.chunk, st.raw))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("batch,dim,L,stride", [(4, 8, 100, 1), (2, 6, 37, 3), (1, 16, 64, 8),
                                                 (1, 8, 33, 5)])
def test_two_rank_counts_equal_single(port, batch, dim, L, stride):
    world, k, seed = 2, 256, 11
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pn = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, pn, batch, dim, L, stride, k, seed, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(seed)
    u = rng.standard_normal((batch, dim, L)).astype(np.float32)
    ref_counts, lo, hi, n = port.histogram(u.reshape(-1), k, 1e-8, stride)
    assert n == n_samples(u.size, stride)
    raw, _ = port.entropy(ref_counts.astype(np.float64) * (1.0 / n))
    chunk, _ = port.select_chunk(raw, 32, 512, math.log(k))
    for rank, counts, rng_buf, c, r in res:
        assert (counts.astype(np.uint64) == ref_counts).all(), rank
        assert -rng_buf[0] == lo and rng_buf[1] == hi
        assert c == chunk and r == raw


def test_plan_rows_covers_every_row_once():
    for batch, dim, world in [(8, 4096, 8), (16, 5120, 8), (1, 1536, 8), (2, 2048, 4), (8, 64, 2)]:
        seen = np.zeros(batch * dim, dtype=int)
        L = 3
        for r in range(world):
            plan = plan_rows(batch, dim, L, r, world)
            for s in plan.segments:
                rows = np.arange(s.global_offset // L, (s.global_offset + s.numel) // L)
                seen[rows] += 1
                assert s.numel % ((s.d1 - s.d0) * L) == 0
        assert (seen == 1).all()


@pytest.mark.parametrize("batch,dim,L,stride", [(2, 12, 9, 1), (1, 16, 7, 3), (3, 8, 5, 4)])
def test_two_rank_token_entropy_equals_single(port, batch, dim, L, stride):
    """token_entropy sharded over 2 ranks (rows of batch*d_inner) equals the oracle's
    token_entropy of the whole (batch*d_inner, L) tensor bit for bit."""
    world, k, seed = 2, 64, 17
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pn = _free_port()
    procs = [ctx.Process(target=_token_worker,
                         args=(r, world, pn, batch, dim, L, stride, k, seed, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(seed)
    u = rng.standard_normal((batch, dim, L)).astype(np.float32)
    raw, _, n = port.token_entropy(u.reshape(batch * dim, L).astype(np.float64), k, 1e-8, stride)
    assert n == L * ((batch * dim + stride - 1) // stride)
    counts0 = res[0][1]
    for rank, counts, r in res:
        assert (counts == counts0).all(), rank
        assert r == raw, (rank, r, raw)
