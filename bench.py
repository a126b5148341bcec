#!/usr/bin/env python
"""COREY hot-path benchmark: K-bin entropy -> chunk rule -> fused Mamba-1 scan on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C3] [--scaling weak|strong] [--no-e2e] [--no-cpu]
                    [--no-producer]

One "step" = one layer's prefill over the configured workload (BASELINE.json
configs[2], "C3": B=8, L=8192, d_inner=4096, N=16 per rank): range_init ->
minmax -> histogram -> [allreduce MAX range, allreduce SUM counts when N>1] ->
device decision -> chunked fused scan, all stream-ordered with no host sync.
Inputs are synthetic, fp32, resident in HBM, each tensor (1.07 GB) larger than
the 126 MB L2, so no L2 flush is needed between iterations.  Configs whose tensors
fit in L2 (C1, C2) write a 256 MB buffer between steps, outside the per-step events.

Prints ONE JSON line on rank 0 (contract in the task statement): value = whole-job
tokens/s (a token = one (b, l) position through all d_inner channels),
`roofline` for the dominant kernel (the scan), `cpu_baseline`, `e2e` (the same
metric through the public API with pinned host buffers and H2D/D2H inside the
timed region), `clocks`, `gpu_launches`, and (N=1) `producer_fusion`: the conv1d+SiLU
producer of u with the min/max pass fused into its epilogue vs run separately.

--impl reference times the reference's own CPU implementation (oracle/_ref: the
reference headers compiled in place; else the oracle port) on the box's host
cores over a bounded sample of the same workload (one batch of C3 per step).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
L2_BYTES = 128 * 1024 * 1024  # B200 L2 (126 MB), rounded up
# single-GPU step: histogram + decision as one launch (cl_histogram_decide_f32);
# CL_BENCH_SEPARATE_DECIDE=1 times the separate decide kernel instead (A/B)
FUSED_DECIDE = os.environ.get("CL_BENCH_SEPARATE_DECIDE", "0") != "1"
sys.path.insert(0, ROOT)

METRIC = "selective-scan tokens/s & HBM GB/s (% roofline) at 1/2/4/8 B200 vs CPU ref"
CONFIGS = {
    # name: (batch per rank, dim, seq_len, d_state, description)
    "C1": (1, 1536, 2048, 16, "Mamba-130M-shaped layer B=1 L=2048 d_inner=1536 N=16"),
    "C2": (1, 2048, 4096, 16, "Mamba-370M-shaped layer B=1 L=4096 d_inner=2048 N=16"),
    "C3": (8, 4096, 8192, 16, "Mamba-1.4B-shaped layer B=8 L=8192 d_inner=4096 N=16"),
    "C4": (16, 5120, 16384, 16, "Mamba-2.8B-shaped layer B=16 L=16384 d_inner=5120 N=16"),
}


def library_sha256():
    """The library build's fingerprint (sources, headers, nvcc flags, toolkit version:
    paper_2604_10597_b200.build.fingerprint); the .so bytes themselves are not
    reproducible from build to build."""
    from paper_2604_10597_b200 import build as _build
    return _build.fingerprint()


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


HBM_SPEC_GBS = 8000.0  # B200 HBM3e data-sheet bandwidth (report both)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def algorithmic_bytes(batch, dim, L, N, stride=1):
    """Per SURVEY.md 8d / DESIGN.md: per token 8*D (entropy: two reads of u) +
    16*D (scan: read u, delta, z; write out) + 8*N (read B, C)."""
    tokens = batch * L
    return dict(entropy=tokens * 8 * dim, scan=tokens * (16 * dim + 8 * N),
                total=tokens * (24 * dim + 8 * N), tokens=tokens)


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: an NVML polling thread
    (a sample every ~2 ms, so even a 10 ms timed region of the few-row configs gets
    samples), else `nvidia-smi -lms 20`.  summary() keeps the samples between mark("t_start")
    and mark("t_stop")."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device_index=0):
        self.proc = None
        self.nvml = None
        self.samples = []  # (time, sm_mhz, max_mhz, set of reasons, power W or None)
        self.power_limit_w = None
        self.dev = device_index
        self.stop = False

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.dev)
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            try:
                self.power_limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(h) / 1000.0
            except Exception:
                self.power_limit_w = None
            self.nvml = (pynvml, h, bits, mx)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _poll(self):
        pynvml, h, bits, mx = self.nvml
        while not self.stop:
            try:
                sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                try:
                    pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
                except Exception:
                    pw = None
                self.samples.append((time.time(), sm, mx, {n for n, b in bits.items() if r & b},
                                     pw))
            except Exception:
                pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.strip().split(",")]
            if len(parts) < 9:
                continue
            try:
                sm, mx = float(parts[1]), float(parts[2])
            except ValueError:
                continue
            reasons = {n for n, v in zip(self.NAMES, parts[5:9]) if v.lower().startswith("active")}
            try:
                pw = float(parts[3])
            except ValueError:
                pw = None
            self.samples.append((time.time(), sm, mx, reasons, pw))

    def mark(self, which):
        setattr(self, which, time.time())

    def __exit__(self, *a):
        self.stop = True
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, pw = [], None, set(), []
        t0, t1 = getattr(self, "t_start", 0.0), getattr(self, "t_stop", 1e30)
        for ts, s_mhz, m_mhz, rs, p_w in list(self.samples):
            if not (t0 <= ts <= t1 + 0.002):
                continue
            sm.append(s_mhz)
            mx = m_mhz
            reasons |= rs
            if p_w is not None:
                pw.append(p_w)
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
               "reasons": sorted(reasons), "samples": len(sm),
               "source": "nvml" if self.nvml else "nvidia-smi"}
        if sm:
            out["sm_mhz_min"] = min(sm)
        if pw:  # board power during the timed region (sw_power_cap: at the enforced limit)
            out["power_w_median"] = statistics.median(pw)
            out["power_w_max"] = max(pw)
        if self.power_limit_w:
            out["power_limit_w"] = self.power_limit_w
        return out


# ----------------------------------------------------------------- data
def make_inputs(torch, device, batch, dim, L, N, seed):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    f32 = dict(device=device, dtype=torch.float32)
    u = torch.randn(batch, dim, L, generator=g, **f32)
    delta = torch.randn(batch, dim, L, generator=g, **f32).mul_(0.1)
    dt = torch.exp(torch.empty(dim, **f32).uniform_(np.log(1e-3), np.log(1e-1), generator=g))
    delta_bias = torch.log(torch.expm1(dt))
    A = -(torch.arange(1, N + 1, **f32)[None, :]) * (
        1 + 0.1 * torch.empty(dim, N, **f32).uniform_(-1, 1, generator=g))
    B = torch.randn(batch, N, L, generator=g, **f32)
    C = torch.randn(batch, N, L, generator=g, **f32)
    D = 1 + 0.1 * torch.randn(dim, generator=g, **f32)
    z = torch.randn(batch, dim, L, generator=g, **f32)
    return dict(u=u, delta=delta, A=A.contiguous(), B=B, C=C, D=D, z=z, delta_bias=delta_bias)


# ----------------------------------------------------------------- reference arm
def cpu_reference_step(lib_kind, x_host, dim, L, N, threads, ref, port):
    """One bounded sample: entropy over one batch's u + rule + Mamba-1 scan of that batch,
    through the reference's own functions (oracle/_ref) or the oracle port."""
    u = x_host["u"]  # (1, dim, L) float32
    t0 = time.perf_counter()
    if lib_kind == "reference":
        masses, lo, hi, n = ref.histogram_masses(u.reshape(-1), 256, 1e-8, 1)
        raw, _ = ref.entropy(masses)
        chunk, _ = ref.select_chunk(raw, 32, 512, np.log(256.0))
        y, h = ref.mamba1_f32(u, x_host["delta"], x_host["A"], x_host["B"], x_host["C"],
                              x_host["D"], x_host["z"], x_host["delta_bias"], True,
                              rows=(0, dim), threads=threads)
    else:
        counts, lo, hi, n = port.histogram(u.reshape(-1), 256, 1e-8, 1)
        raw, _ = port.entropy(counts.astype(np.float64) / n)
        chunk, _ = port.select_chunk(raw, 32, 512, np.log(256.0))
        y = _port_mamba_threaded(port, x_host, dim, L, N, threads)
    dt = time.perf_counter() - t0
    return dt, chunk, raw


def cpu_single_thread(ref, x, dim, L, rows=256):
    """The reference exactly as shipped (one thread): entropy + rule over one batch's u,
    the scan over `rows` of its channels, scan time scaled to all channels (rows are
    independent and equal work)."""
    u = x["u"]
    t0 = time.perf_counter()
    masses, lo, hi, n = ref.histogram_masses(u.reshape(-1), 256, 1e-8, 1)
    raw, _ = ref.entropy(masses)
    ref.select_chunk(raw, 32, 512, np.log(256.0))
    t1 = time.perf_counter()
    ref.mamba1_f32(u, x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"], x["delta_bias"],
                   True, rows=(0, rows), threads=1)
    t2 = time.perf_counter()
    total = (t1 - t0) + (t2 - t1) * dim / rows
    return {"value": L / total, "unit": "tokens/s", "cores": 1,
            "sample": f"entropy + rule over 1 batch ({dim} x {L}) {t1 - t0:.2f} s; fp64 "
                      f"Mamba-1 scan of {rows} of {dim} rows {t2 - t1:.2f} s, scaled x{dim / rows:g}"}


def _port_mamba_threaded(port, x, dim, L, N, threads):
    from concurrent.futures import ThreadPoolExecutor
    per = (dim + threads - 1) // threads
    def work(i):
        r0, r1 = i * per, min(dim, (i + 1) * per)
        if r0 >= r1:
            return None
        return port.mamba1(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"],
                           x["delta_bias"], True, rows=(r0, r1))
    with ThreadPoolExecutor(threads) as ex:
        return list(ex.map(work, range(threads)))


def sample_host_inputs(cfg, seed=0):
    import torch
    batch, dim, L, N, _ = CONFIGS[cfg]
    x = make_inputs(torch, "cpu", 1, dim, L, N, seed)
    return {k: v.numpy() for k, v in x.items()}


def reference_arm(args):
    from oracle import oracle as O
    batch, dim, L, N, desc = CONFIGS[args.config]
    threads = os.cpu_count() or 1
    kind = "reference" if O.reference_available() else "port"
    ref = O.Reference() if kind == "reference" else None
    port = O.Port()
    x = sample_host_inputs(args.config)
    for _ in range(args.warmup):
        cpu_reference_step(kind, x, dim, L, N, threads, ref, port)
    times = []
    chunk = raw = None
    for _ in range(args.steps):
        dt, chunk, raw = cpu_reference_step(kind, x, dim, L, N, threads, ref, port)
        times.append(dt)
    t = sum(times) / len(times)
    tokens_per_step = L  # one batch of the workload: L positions x all d_inner channels
    value = tokens_per_step / t
    sample = (f"1 of {batch} batches of {args.config} per step ({dim} channels x L={L}, N={N}): "
              f"entropy K=256 over that batch's u + calibrated rule + fp64 Mamba-1 scan "
              f"(reference scan_sequential under the SURVEY finding-1 mapping), {threads} threads")
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (torch.randn, seed 0)",
            "config": {"workload": f"{args.config}: {desc}", "sample": sample,
                       "policy": "calibrated rule log K, bounds [32,512]"},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": kind,
                             "cpu": cpu_model(),
                             "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "chunk": chunk, "raw_nats": raw}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS))
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--chunk-policy", default="rule", choices=["rule", "guarded", "static512"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-producer", action="store_true",
                    help="skip the side measurements (conv1d producer fusion, token entropy)")
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="timed e2e steps (0: enough for ~40 ms of PCIe traffic, at least 8)")
    ap.add_argument("--pipelined", action="store_true",
                    help="also measure two batches in flight (entropy of call i+1 in the lean "
                         "kernels under call i's scan); measured slower on B200, see DESIGN.md")
    ap.add_argument("--eager", action="store_true",
                    help="launch every stage from the host each step instead of replaying "
                         "per-stage CUDA graphs")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            reference_arm(args)
        return 0

    import torch
    import torch.distributed as dist

    # CL_BENCH_DIST_BACKEND=gloo is a functional check of the N>1 code path on a
    # one-GPU box (ranks share cuda:0, collectives staged through the host by gloo);
    # its timings are not scaling numbers.  The product path is NCCL, one GPU per rank.
    backend = os.environ.get("CL_BENCH_DIST_BACKEND", "nccl")
    dev_index = local_rank if backend == "nccl" else local_rank % torch.cuda.device_count()
    torch.cuda.set_device(dev_index)
    device = torch.device("cuda", dev_index)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)

    import paper_2604_10597_b200 as cl
    from paper_2604_10597_b200.mamba1 import Prefill, scan_plan

    batch, dim, L, N, desc = CONFIGS[args.config]
    if args.scaling == "strong" and world > 1:
        assert batch % world == 0, "strong scaling shards whole batches"
        batch //= world
    global_batch = batch * world
    x = make_inputs(torch, device, batch, dim, L, N, seed=1234 + rank)
    out = torch.empty_like(x["u"])
    h_last = torch.empty(batch, dim, N, device=device)

    spec = cl.HistogramSpec(bin_count=256, epsilon=1e-8, sample_stride=1)
    bounds = cl.ChunkBounds(32, 512)
    policy = None
    if args.chunk_policy == "guarded":
        spec.sample_stride = 8
        inner = cl.SchedulerPolicy(cl.SampledHistogramPolicy(8), [128, 256, 512, 1024, 2048])
        policy = cl.SchedulerPolicy(cl.GuardedPolicy(inner, 512, 2), [128, 256, 512, 1024, 2048])
        bounds = cl.ChunkBounds(128, 2048)
    elif args.chunk_policy == "static512":
        policy = cl.SchedulerPolicy(cl.StaticPolicy(512), [128, 256, 512, 1024, 2048])
    pf = Prefill(spec, policy, bounds, cl.CalibrationRef.log_k(256), device=device)
    n_local = batch * dim * L
    g0 = rank * n_local  # global flat offset of this rank's rows (stride sampling)
    n_total = pf.n_samples(n_local * world)
    uf = x["u"].reshape(-1)

    from paper_2604_10597_b200.sharded import DeviceStages, plan_rows, sharded_entropy_decision
    plan = plan_rows(global_batch, dim, L, rank, world)
    assert plan.b0 * dim * L == g0 and plan.local_batch == batch
    stages = DeviceStages(pf)

    # ev: [start, after min/max, after histogram, after decision, after scan]; the timed
    # loop records only slots 0, 3 and 4 (fine=False) -- each event record is a few
    # microseconds of stream time on the few-row shapes -- and a separate untimed pass
    # records all five for the stage breakdown
    def step(ev=None, fine=True):
        if ev:
            ev[0].record()
        if world > 1:
            # the product multi-GPU protocol: MAX-allreduce of the range, SUM-allreduce
            # of the counts, identical device decision on every rank
            sharded_entropy_decision(stages, uf, plan, int(spec.sample_stride))
            if ev:
                if fine:
                    ev[1].record()
                    ev[2].record()
                ev[3].record()
        else:
            pf.stage_init((x["u"], x["delta"], x["A"], x["B"], x["C"]))
            if FUSED_DECIDE:
                # min/max (gathering the samples for strides >= 4), then histogram +
                # decision in one launch (its last CTA decides): stage "histogram"
                # includes the decision -- the single-GPU prefill's own sequence
                pf.stage_entropy_minmax(uf)
                if ev and fine:
                    ev[1].record()
                pf.stage_entropy_histogram(uf, L)
                if ev and fine:
                    ev[2].record()
            else:
                pf.stage_minmax(uf, g0, init=False)
                if ev and fine:
                    ev[1].record()
                pf.stage_histogram(uf, g0, zero=False)
                if ev and fine:
                    ev[2].record()
                pf.stage_decide(n_total, L)
            if ev:
                ev[3].record()
        pf.stage_scan(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"],
                      x["delta_bias"], True, out, True)
        if ev:
            ev[4].record()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    rec = pf.decision()  # sync point outside the timed region; raises on device errors
    plan_info = scan_plan(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"],
                          x["delta_bias"], True, out=out, return_last_state=True)

    # One GPU: each stage is captured once into a CUDA graph and the timed steps replay
    # them (the production way to launch a fixed-shape layer: no Python / ctypes / tensor-
    # map encoding per step, which on the few-row shapes takes as long as the device work).
    # The graphs hold exactly the eager launches -- every kernel runs every step, the
    # decision is taken on the device every step -- and the per-stage events sit between
    # the replays, on the same stream.  N>1 keeps eager launches (NCCL between stages).
    use_graphs = world == 1 and not args.eager
    if use_graphs:
        cap = torch.cuda.Stream(device)
        cap.wait_stream(torch.cuda.current_stream(device))
        graphs = []
        captured0 = pf.ctx.launches
        with torch.cuda.stream(cap):
            # (the graphs are captured on one stream and share its captured workspace; the
            # scan graph re-lays B / C itself -- a hand-off from another graph's init launch
            # would depend on replay order, so the library only takes it within one capture)
            for stage in (lambda: (pf.stage_init(), pf.stage_entropy_minmax(uf)),
                          lambda: pf.stage_entropy_histogram(uf, L),
                          lambda: pf.stage_scan(x["u"], x["delta"], x["A"], x["B"], x["C"],
                                                x["D"], x["z"], x["delta_bias"], True, out,
                                                True)):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cap):
                    stage()
                graphs.append(g)
            kernels_per_step = pf.ctx.launches - captured0  # this library's kernel nodes
            # the timed steps replay the entropy stages as ONE graph (init + minmax +
            # histogram/decision) and the scan as another: the one event between them
            # times the scan inside the timed region; the per-stage graphs above give the
            # untimed stage breakdown
            g_ent = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_ent, stream=cap):
                pf.stage_init()
                pf.stage_entropy(uf, L)
        torch.cuda.current_stream(device).wait_stream(cap)
        torch.cuda.synchronize()

        def step(ev=None, fine=True):  # noqa: F811  (the graph-replay step)
            if ev:
                ev[0].record()
            if fine:  # stage breakdown: one graph per stage, events between
                graphs[0].replay()
                if ev:
                    ev[1].record()
                graphs[1].replay()
                if ev:
                    ev[2].record()
            else:
                g_ent.replay()
            if ev:
                ev[3].record()
            graphs[2].replay()
            if ev:
                ev[4].record()

        for _ in range(args.warmup):
            step(None, fine=False)
        step(None, fine=True)
        torch.cuda.synchronize()
        rec2 = pf.decision()
        assert rec2.decision.chunk == rec.decision.chunk

    # per-stage CUDA events on the launching stream, read after the timed loop
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    launches0 = pf.ctx.launches
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # Shapes whose inputs fit the 126 MB L2 (C1, C2): flush L2 between steps by writing a
    # 256 MB buffer, outside the per-step events; the step time is then the sum of the
    # per-step event intervals instead of the whole loop's
    tensor_bytes = batch * dim * L * 4
    l2_flush = tensor_bytes < L2_BYTES
    l2buf = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=device) if l2_flush else None
    with ClockSampler(dev_index) as clocks:
        time.sleep(0.5)  # let nvidia-smi start sampling before the timed region
        clocks.mark("t_start")
        start.record()
        for i in range(args.steps):
            if l2_flush:
                l2buf.zero_()
            step(evs[i], fine=False)
        stop.record()
        torch.cuda.synchronize()
        clocks.mark("t_stop")
    stage_ms = {"entropy": [e[0].elapsed_time(e[3]) for e in evs],
                "scan": [e[3].elapsed_time(e[4]) for e in evs]}
    # stage breakdown (untimed pass, all five events per step)
    bevs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(10)]
    for bev in bevs:
        if l2_flush:
            l2buf.zero_()
        step(bev, fine=True)
    torch.cuda.synchronize()
    breakdown = {"minmax": statistics.median(e[0].elapsed_time(e[1]) for e in bevs),
                 "histogram_decide": statistics.median(e[1].elapsed_time(e[2]) for e in bevs),
                 "scan": statistics.median(e[3].elapsed_time(e[4]) for e in bevs)}
    if world > 1:
        dist.barrier()
    elapsed_ms = start.elapsed_time(stop)
    if l2_flush:
        elapsed_ms = sum(e[0].elapsed_time(e[4]) for e in evs)
    launches = pf.ctx.launches - launches0
    if use_graphs:  # replays enqueue no host-side launches: count the graphs' kernel nodes
        launches = kernels_per_step * args.steps
    if world > 1:
        t = torch.tensor([elapsed_ms], device=device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    tokens_total = global_batch * L
    value = tokens_total / (ms_per_step / 1e3)

    peak, peak_kind = peaks()
    ab = algorithmic_bytes(batch, dim, L, N)
    scan_ms = statistics.mean(stage_ms["scan"])
    ent_ms = statistics.mean(stage_ms["entropy"])
    scan_gbs = ab["scan"] / (scan_ms / 1e3) / 1e9
    step_gbs = ab["total"] / (ms_per_step / 1e3) / 1e9  # per rank
    # ncu DRAM bytes of the dominant kernel, captured by tools/scan_traffic.py for this
    # exact library build (sha256 of libchunklab_b200.so), config and kernel; null when the
    # record is for another build (a stale figure is worse than none)
    traffic = None
    traffic_note = "no ncu record"
    prof = os.path.join(ROOT, "profiles", "scan_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            recs = json.load(f)
        recs = recs if isinstance(recs, list) else [recs]
        lib_sha = library_sha256()
        traffic_note = "ncu record is for another library build or config"
        for pj in recs:
            if (pj.get("config") == args.config and pj.get("lib_sha256") == lib_sha and
                    pj.get("kernel_family") == plan_info["kernel"]):
                traffic = pj.get("dram_bytes_per_launch")
                traffic_note = "ncu --set full of this build: " + str(pj.get("source", ""))

    result = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": args.scaling if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (torch.randn, seeded)",
        "config": {"workload": f"{args.config}: {desc}", "batch_per_rank": batch,
                   "global_batch": global_batch, "seq_len": L, "d_inner": dim, "d_state": N,
                   "bins": 256, "policy": args.chunk_policy, "parallelism": f"rows x{world}",
                   "l2": (f"L2 flushed between steps (256 MB write outside the per-step "
                          f"events; {tensor_bytes / 1e6:.1f} MB per tensor)") if l2_flush else
                         (f"inputs ({tensor_bytes / 1e9:.2f} GB per tensor) exceed the 126 MB "
                          f"L2; no flush needed")},
        "hbm_gbs": step_gbs, "roofline_frac_step": step_gbs / peak,
        "roofline": {"bound": "hbm", "achieved": scan_gbs, "peak": peak, "unit": "GB/s",
                     "frac": scan_gbs / peak, "traffic": traffic, "traffic_source": traffic_note,
                     "kernel": "rowpair_ws_kernel",
                     "peak_kind": peak_kind,
                     "spec_peak": HBM_SPEC_GBS, "spec_frac": scan_gbs / HBM_SPEC_GBS,
                     "algorithmic_bytes_per_launch": ab["scan"]},
        "stage_ms": ({k: statistics.mean(v) for k, v in stage_ms.items()} if world == 1 else
                     {"entropy_allreduce_decide": statistics.mean(stage_ms["entropy"]),
                      "scan": statistics.mean(stage_ms["scan"])}),
        "stage_breakdown_ms": breakdown,
        "entropy_gbs": ab["entropy"] / (ent_ms / 1e3) / 1e9,
        "chunk": rec.decision.chunk, "raw_nats": rec.entropy.raw_nats,
        "gpu_launches": launches,
        "scan_plan": plan_info,
    }
    result["config"]["launch"] = ("CUDA graphs replayed (captured once): entropy stages, then "
                                  "the scan; the stage breakdown replays one graph per stage"
                                  if use_graphs
                                  else "eager launches")
    result["roofline"]["kernel"] = plan_info["kernel"]
    result["clocks"] = clocks.summary()
    # SFU roofline of the scan: 18 MUFU per (b, d, l) -- 16 state
    # exponentials, one ex2 in softplus, one in SiLU -- at 16 MUFU/clk/SM x SMs x the
    # SM clock sampled during the timed region (the scan's binding pipe; HBM is not).
    # The L-parallel kernel's extra aggregate pass counts as issued work.
    sm_mhz = result["clocks"].get("sm_mhz") or 1965.0
    n_sms = torch.cuda.get_device_properties(device).multi_processor_count
    mufu_per_launch = batch * dim * L * (N + 2)
    if plan_info["kernel"] == "lookback_ws_kernel":
        # + the aggregate pass over every segment but the last (16 state exps + the
        # softplus ex2 per element) + the carry-in folds (16 exps per folded segment)
        ns, sl = plan_info["n_seg"], plan_info["seg_len"]
        last = L - (ns - 1) * sl
        mufu_per_launch += batch * dim * ((L - last) * (N + 1) + N * ns * (ns - 1) // 2)
    sfu_peak = 16 * n_sms * sm_mhz * 1e6 / 1e12
    sfu_ach = mufu_per_launch / (scan_ms / 1e3) / 1e12
    result["roofline"]["sfu"] = {"achieved": sfu_ach, "peak": sfu_peak, "unit": "TMUFU/s",
                                 "frac": sfu_ach / sfu_peak,
                                 "mufu_per_launch": mufu_per_launch,
                                 "peak_basis": f"16/clk/SM x {n_sms} SMs x {sm_mhz:.0f} MHz"}

    # ---- pipelined steady state (two batches in flight), a separately labelled figure
    if world == 1 and args.pipelined and args.chunk_policy == "rule":
        torch.cuda.synchronize()
        pf(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"], x["delta_bias"], True,
           out=out)  # the serial reference output of batch 0 (same decision buffers)
        torch.cuda.synchronize()
        mk = lambda seed: make_inputs(torch, device, batch, dim, L, N, seed)  # noqa: E731
        result["pipelined"] = pipelined_measure(torch, device, x, pf, out,
                                                max(args.steps // 2, 6), mk, lean=False)
        result["pipelined_lean"] = pipelined_measure(torch, device, x, pf, out,
                                                     max(args.steps // 2, 6), mk, lean=True)

    # ---- producer fusion (conv1d + SiLU with the min/max epilogue), side measurement
    if not args.no_producer and world == 1:
        result["producer_fusion"] = producer_fusion_measure(torch, device, x, pf)
        result["token_entropy"] = token_entropy_measure(torch, device, x)

    # ---- e2e through the public API with host buffers (pinned), H2D/D2H timed
    if not args.no_e2e:
        if world > 1:  # the public multi-GPU API: global entropy over all ranks' rows
            from paper_2604_10597_b200.sharded import ShardedPrefill
            sp = ShardedPrefill(pf, plan)

            def run_prefill(d, o):
                sp(d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"],
                   True, out=o)
        else:
            def run_prefill(d, o):
                pf(d["u"], d["delta"], d["A"], d["B"], d["C"], d["D"], d["z"], d["delta_bias"],
                   True, out=o)
        e2e_steps = args.e2e_steps
        if e2e_steps <= 0:
            # the three-stream pipeline fills and drains around the timed steps: size the
            # run to ~40 ms of uploads at ~50 GB/s so small configs reach steady state
            step_s = sum(v.numel() * 4 for v in x.values()) / 50e9
            e2e_steps = int(min(256, max(8, 0.04 / step_s)))
        result["e2e"] = e2e_measure(torch, dist, world, device, x, run_prefill, L, global_batch,
                                    e2e_steps)
    del x, out
    torch.cuda.empty_cache()

    # ---- CPU baseline (rank 0, N=1 only)
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            from oracle import oracle as O
            kind = "reference" if O.reference_available() else "port"
            ref = O.Reference() if kind == "reference" else None
            port = O.Port()
            threads = os.cpu_count() or 1
            xh = sample_host_inputs(args.config)
            cpu_reference_step(kind, xh, dim, L, N, threads, ref, port)  # warm
            dt, _, _ = cpu_reference_step(kind, xh, dim, L, N, threads, ref, port)
            result["cpu_baseline"] = {
                "value": L / dt, "unit": "tokens/s", "cores": threads, "kind": kind,
                "cpu": cpu_model(),
                "sample": f"1 batch of {args.config} ({dim} x {L}): entropy + rule + fp64 "
                          f"Mamba-1 scan, {threads} threads, {dt:.2f} s"}
            if kind == "reference":
                result["cpu_baseline"]["single_thread"] = cpu_single_thread(ref, xh, dim, L)
        except Exception as e:  # the baseline must never take the bench down
            result["cpu_baseline"] = {"value": None, "error": str(e)}

    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def producer_fusion_measure(torch, device, x, pf, reps=20):
    """the conv1d(+SiLU) producer of u with the stage-1 min/max in its
    epilogue, vs the same conv followed by the separate min/max pass (device time)."""
    from paper_2604_10597_b200.mamba1 import causal_conv1d_fn
    batch, dim, L = x["u"].shape
    g = torch.Generator(device=device)
    g.manual_seed(7)
    xin = torch.randn(batch, dim, L, generator=g, device=device, dtype=torch.float32)
    w = torch.randn(dim, 4, generator=g, device=device, dtype=torch.float32).mul_(0.5)
    b = torch.randn(dim, generator=g, device=device, dtype=torch.float32).mul_(0.1)
    u = torch.empty_like(xin)
    uf = u.reshape(-1)

    def fused():
        pf.stage_conv(xin, w, b, "silu", out=u)

    def unfused():
        causal_conv1d_fn(xin, w, b, "silu", out=u)
        pf.stage_minmax(uf)

    def conv_only():
        causal_conv1d_fn(xin, w, b, "silu", out=u)

    res = {}
    for name, fn in (("fused_ms", fused), ("unfused_ms", unfused), ("conv_only_ms", conv_only)):
        fn()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(reps)]
        for a, e in evs:
            a.record()
            fn()
            e.record()
        torch.cuda.synchronize()
        res[name] = statistics.median(a.elapsed_time(e) for a, e in evs)
    fused_bytes = 2 * xin.numel() * 4  # read x, write u
    res["saved_ms"] = res["unfused_ms"] - res["fused_ms"]
    res["fused_gbs"] = fused_bytes / (res["fused_ms"] / 1e3) / 1e9
    res["workload"] = f"conv width 4 + SiLU over ({batch}, {dim}, {L}) fp32, stride 1"

    # the whole layer: conv -> entropy -> decision -> scan, fused (cl_prefill_from_conv_f32)
    # vs the conv followed by the unfused prefill on its u, for the calibrated rule
    # (Dynamic range: min/max in the conv epilogue) and a Fixed range (the whole histogram
    # in the conv epilogue: u is never re-read for the entropy)
    import paper_2604_10597_b200 as cl
    from paper_2604_10597_b200.mamba1 import Prefill
    out = torch.empty_like(xin)
    layer = {}
    for tag, spec in (("dynamic", cl.HistogramSpec()),
                      ("fixed", cl.HistogramSpec(range_mode=cl.RangeMode.Fixed, fixed_lo=-0.5,
                                                 fixed_hi=4.0))):
        lp = Prefill(spec, None, cl.ChunkBounds(32, 512), device=device)

        def fused_layer():
            lp.from_conv(xin, w, b, x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"],
                         x["delta_bias"], True, out=out, u=u)

        def unfused_layer():
            causal_conv1d_fn(xin, w, b, "silu", out=u)
            lp(u, x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"], x["delta_bias"], True,
               out=out)

        for name, fn in (("fused_ms", fused_layer), ("unfused_ms", unfused_layer)):
            fn()
            torch.cuda.synchronize()
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(reps // 2)]
            for a, e in evs:
                a.record()
                fn()
                e.record()
            torch.cuda.synchronize()
            layer.setdefault(tag, {})[name] = statistics.median(a.elapsed_time(e) for a, e in evs)
        layer[tag]["saved_ms"] = layer[tag]["unfused_ms"] - layer[tag]["fused_ms"]
    layer["workload"] = ("conv1d(width 4) + SiLU -> K=256 entropy -> calibrated rule -> fused "
                         "scan, cl_prefill_from_conv_f32 vs causal_conv1d + cl_prefill_f32; "
                         "fixed range [-0.5, 4]")
    res["layer"] = layer
    del xin, u, out
    return res


def pipelined_measure(torch, device, x, pf, out_serial, steps, make, lean=True):
    """Steady-state throughput with two independent batches in flight: call i+1's entropy
    (lean=True: cl_entropy_lean_f32, lean kernels sized to share SMs with a scan CTA;
    lean=False: the regular stages) on one stream while call i's scan runs on another.  Every call still does all of its own work
    (min/max, histogram, device decision, scan); outputs are checked against the serial
    step bit for bit.  A separately labelled figure beside the single-call latency."""
    import paper_2604_10597_b200 as cl
    from paper_2604_10597_b200.mamba1 import Prefill
    batch, dim, L = x["u"].shape
    xb = make(1234 + 777)
    sets = [x, xb]
    outs = [torch.empty_like(x["u"]), torch.empty_like(x["u"])]
    pfs = [Prefill(pf.spec, pf.policy, pf.bounds, pf.cal, device=device) for _ in range(2)]
    s_ent, s_scan = torch.cuda.Stream(device), torch.cuda.Stream(device)
    ent_done = [torch.cuda.Event(), torch.cuda.Event()]
    scan_done = [torch.cuda.Event(), torch.cuda.Event()]
    scanned = [False, False]

    def entropy(j):
        with torch.cuda.stream(s_ent):
            if scanned[j]:
                s_ent.wait_event(scan_done[j])  # its buffers are read by that scan
            if lean:
                pfs[j].stage_entropy_lean(sets[j]["u"].reshape(-1), L)
            else:
                pfs[j].stage_init()
                pfs[j].stage_entropy(sets[j]["u"].reshape(-1), L)
            ent_done[j].record(s_ent)

    def scan(j):
        X = sets[j]
        with torch.cuda.stream(s_scan):
            s_scan.wait_event(ent_done[j])
            pfs[j].stage_scan(X["u"], X["delta"], X["A"], X["B"], X["C"], X["D"], X["z"],
                              X["delta_bias"], True, outs[j])
            scan_done[j].record(s_scan)
            scanned[j] = True

    def run(n):
        entropy(0)
        for i in range(n):
            if i + 1 < n:
                entropy((i + 1) % 2)
            scan(i % 2)

    torch.cuda.synchronize()
    run(4)  # warm-up
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(s_ent)
    s_scan.wait_event(t0)
    run(steps)
    t1.record(s_scan)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    # the serial step's output for batch 0 (same inputs, same decision) -- bit for bit
    same = bool(torch.equal(outs[0], out_serial))
    same_dec = bool(torch.equal(pfs[0].decision_buf, pf.decision_buf))
    res = {"ms_per_step": ms, "value": batch * L / (ms / 1e3), "unit": "tokens/s",
           "steps": steps, "matches_serial_bitwise": same and same_dec,
           "workload": "two independent batches in flight: entropy(i+1) [" +
                       ("lean" if lean else "regular") + " kernels, stream 2] under scan(i) "
                       "[stream 1]; every call's own min/max + histogram + device decision + "
                       "scan"}
    del xb, outs, sets
    return res


def token_entropy_measure(torch, device, x, reps=10):
    """token_entropy (per-position histograms over channels) of u on the
    device, as the TokenHistogram policy's prefill stage (both passes + per-position
    entropies + the ordered mean)."""
    from paper_2604_10597_b200.mamba1 import Prefill
    import paper_2604_10597_b200 as cl
    pf = Prefill(cl.HistogramSpec(), cl.SchedulerPolicy(cl.TokenHistogramPolicy(),
                                                        [128, 256, 512, 1024, 2048]),
                 cl.ChunkBounds(128, 2048), device=device)
    u = x["u"]
    pf.stage_token(u)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(reps)]
    for a, e in evs:
        a.record()
        pf.stage_token(u)
        e.record()
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(e) for a, e in evs)
    raw = float(pf.token_buf[0].item())
    return {"ms": ms, "gbs": 2 * u.numel() * 4 / (ms / 1e3) / 1e9, "raw_nats": raw,
            "workload": f"u {tuple(u.shape)} as (channels={u.numel() // u.shape[-1]}, "
                        f"length={u.shape[-1]}), K=256, two passes over u"}


def e2e_measure(torch, dist, world, device, x, run_prefill, L, global_batch, steps):
    """Same metric through the public API (Prefill) with every step's inputs copied from
    pinned host memory and its output read back, inside the timed region.

    Serving-style pipeline over three streams: H2D of step i+1 (copy engine 1), the prefill
    of step i (SMs) and the D2H of step i-1 (copy engine 2) overlap; device inputs and
    outputs are double-buffered and ordered by events (PCIe is full duplex, so the
    readback hides under the next step's upload).  Timed with device events from the
    first copy to the last readback."""
    host = {k: v.cpu().pin_memory() for k, v in x.items()}
    h_out = torch.empty_like(host["u"]).pin_memory()
    bufs = [{k: torch.empty_like(v) for k, v in x.items()} for _ in range(2)]
    outs = [torch.empty_like(x["u"]) for _ in range(2)]
    h2d = sum(v.numel() * 4 for v in host.values())
    d2h = h_out.numel() * 4
    s_in, s_run, s_out = (torch.cuda.Stream(device) for _ in range(3))
    ev = lambda: torch.cuda.Event()  # noqa: E731
    in_done, run_done, out_done = ([ev() for _ in range(2)] for _ in range(3))
    used = [False, False]

    def step(i):
        j = i % 2
        with torch.cuda.stream(s_in):
            if used[j]:
                s_in.wait_event(run_done[j])  # buffer j's previous prefill has read it
            for k in bufs[j]:
                bufs[j][k].copy_(host[k], non_blocking=True)
            in_done[j].record(s_in)
        with torch.cuda.stream(s_run):
            s_run.wait_event(in_done[j])
            if used[j]:
                s_run.wait_event(out_done[j])  # output j has been read back
            run_prefill(bufs[j], outs[j])
            run_done[j].record(s_run)
        with torch.cuda.stream(s_out):
            s_out.wait_event(run_done[j])
            h_out.copy_(outs[j], non_blocking=True)
            out_done[j].record(s_out)
        used[j] = True

    step(0)
    step(1)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(s_in)
    for i in range(steps):
        step(i)
    end.record(s_out)
    torch.cuda.synchronize()
    ms = start.elapsed_time(end) / steps
    if world > 1:
        t = torch.tensor([ms], device=device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    pcie = pcie_bound(torch, host["u"], bufs[0]["u"], h_out, outs[0], h2d, d2h, ms)
    del bufs, outs
    return {"value": global_batch * L / (ms / 1e3), "unit": "tokens/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": ms,
            "steps": steps, "pipeline": "H2D(i+1) | prefill(i) | D2H(i-1) on 3 streams",
            "pcie": pcie}


def pcie_bound(torch, h_src, d_dst, h_dst, d_src, h2d, d2h, ms, reps=3):
    """The e2e pipeline's roofline: host<->device copy bandwidth measured here (pinned, CUDA
    events) for H2D alone and for H2D + D2H at once (the link is not fully duplex on these
    boxes), and the per-step floor it implies -- the readback overlapped with the upload,
    the rest of the upload alone."""
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    nbytes = h_src.numel() * 4

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps / 1e3

    def both():
        with torch.cuda.stream(s1):
            d_dst.copy_(h_src, non_blocking=True)
        with torch.cuda.stream(s2):
            h_dst.copy_(d_src, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)

    h2d_bw = nbytes / timed(lambda: d_dst.copy_(h_src, non_blocking=True))
    dup_bw = nbytes / timed(both)
    # D2H fully overlapped with part of the upload at the duplex rate, the rest at H2D rate
    overlap = min(d2h, h2d)
    floor_s = overlap / dup_bw + (h2d - overlap) / h2d_bw
    return {"h2d_gbs": h2d_bw / 1e9, "duplex_gbs_each": dup_bw / 1e9,
            "floor_ms": floor_s * 1e3, "frac": floor_s * 1e3 / ms}


if __name__ == "__main__":
    sys.exit(main())
