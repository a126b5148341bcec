"""GPU, world_size 2 over gloo on ONE B200: the Python multi-GPU path (sharded.py
ShardedPrefill) with the REAL device stages (DeviceStages -> libchunklab_b200.so) -- the
CPU gloo test swaps them for an oracle implementation.  Two processes share cuda:0; the
collectives are gloo allreduces of device tensors, which synchronise through the host, so
no kernel of one rank ever waits on a kernel of the other (safe on one GPU).  Every rank's
range, counts and decision must equal the single-GPU prefill's bit for bit, and its rows of
the scan output must equal the single-GPU rows."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shape, stride, token, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2604_10597_b200 as cl
        from paper_2604_10597_b200.mamba1 import Prefill
        from paper_2604_10597_b200.sharded import ShardedPrefill, plan_rows
        from tests._helpers import mamba_inputs
        batch, dim, L = shape
        dev = torch.device("cuda", 0)
        x = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev)
             for k, v in mamba_inputs(17, batch, dim, 16, L).items()}
        spec = cl.HistogramSpec(sample_stride=stride)
        pol = (cl.SchedulerPolicy(cl.TokenHistogramPolicy(), [128, 256, 512, 1024, 2048])
               if token else None)
        bounds = cl.ChunkBounds(128, 2048) if token else cl.ChunkBounds(32, 512)
        full = Prefill(spec, pol, bounds, device=dev)
        y_full = full(x["u"], x["delta"], x["A"], x["B"], x["C"], x["D"], x["z"],
                      x["delta_bias"], True).out
        plan = plan_rows(batch, dim, L, rank, world)
        b0, b1, d0, d1 = plan.b0, plan.b1, plan.d0, plan.d1
        loc = lambda t: t[b0:b1, d0:d1].contiguous()  # noqa: E731
        pf = Prefill(spec, pol, bounds, device=dev)
        sp = ShardedPrefill(pf, plan)
        y = sp(loc(x["u"]), loc(x["delta"]), x["A"][d0:d1].contiguous(),
               x["B"][b0:b1].contiguous(), x["C"][b0:b1].contiguous(), x["D"][d0:d1].contiguous(),
               loc(x["z"]), x["delta_bias"][d0:d1].contiguous(), True)
        torch.cuda.synchronize()
        ok = bool(torch.equal(pf.decision_buf, full.decision_buf))
        if not token:
            ok &= bool(torch.equal(pf.counts, full.counts)) and bool(torch.equal(pf.range, full.range))
        rows_ok = bool(torch.allclose(y, loc(y_full), rtol=0, atol=0) or
                       float((y - loc(y_full)).norm() / loc(y_full).norm()) <= 1e-6)
        q.put((rank, ok, rows_ok, pf.decision().decision.chunk))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape,stride,token", [((4, 64, 1024), 1, False),   # batch split
                                                ((1, 128, 2048), 8, False),  # d_inner split
                                                ((2, 64, 512), 1, True)])    # token policy
def test_python_sharded_prefill_device_stages_world2(cuda, shape, stride, token):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shape, stride, token, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, rows_ok, chunk in res:
        assert ok, f"rank {rank}: range / counts / decision differ from single GPU"
        assert rows_ok, f"rank {rank}: scan rows differ"
    assert res[0][3] == res[1][3]
