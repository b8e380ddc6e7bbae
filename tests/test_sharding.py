"""CPU, world_size 2 (gloo): (batch x head) sharding + final gather reproduce the
unsharded result exactly (slice independence, test_tiled.cpp:223-262). The
per-shard compute here is the f64 oracle; on the GPU box it is the C ABI."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_14376_b200.shard import run_sharded, shard_range


def test_shard_range_partitions():
    for n in (1, 7, 64, 512):
        for world in (1, 2, 3, 8):
            ranges = [shard_range(n, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [e - s for s, e in ranges]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle

    orc = Oracle()
    orc.threads = 1
    rng = np.random.default_rng(0)
    B, H, T, L, dqk, dhv = 2, 3, 32, 8, 8, 12
    arrs = [rng.standard_normal(s) for s in ((B, H, T, dqk), (B, H, T, dqk), (B, H, T, dhv), (B, H, T), (B, H, T))]
    tens = [torch.from_numpy(a) for a in arrs]

    def compute(q, k, v, ip, fp):
        f = orc.forward(*(x.numpy().copy() for x in (q, k, v, ip, fp)), L, 0)
        return [torch.from_numpy(f["h"]), torch.from_numpy(f["m"])]

    h, m = run_sharded(compute, tens, B, H)
    if rank == 0:
        full = orc.forward(*arrs, L, 0)
        out_q.put((float((h.numpy() - full["h"]).__abs__().max()), float(np.abs(m.numpy() - full["m"]).max())))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_rank_sharded_forward_equals_full():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
    assert res == (0.0, 0.0)
