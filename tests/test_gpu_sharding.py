"""Multi-rank (batch x head) sharding through the C-ABI library on the GPU
(slice independence, test_tiled.cpp:223-262).

Two ranks (gloo, both on cuda:0 -- the GPU box has one GPU for these tests)
each run tfla_chunkwise_forward + tfla_chunkwise_backward on their contiguous
range of the flattened (b*NH + h) slices, and the final all-gather rebuilds
every output. The result must be bit-identical to one rank running the whole
batch: a wrong slice pointer, a shared workspace or stream between ranks, or
any cross-slice dependence shows up as a mismatch.

Also drives bench.py under torchrun with two ranks sharing the GPU
(TFLA_BENCH_SHARE_GPU=1): the weak-scaling default and the strong-scaling
BASELINE config 5 mode (--B-total), whose JSON line must account for every
slice exactly once.
"""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
SHAPE = (2, 3, 512, 128, 128, 256)  # B, NH, T, L, dqk, dhv (6 slices over 2 ranks)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _compute_factory(variant, T, L, dqk, dhv):
    import torch

    from paper_2503_14376_b200 import Dims, SequenceInputs, Variant, chunkwise_backward, chunkwise_forward

    def compute(q, k, v, ip, fp, dh):
        n = q.shape[1]
        dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=n, n_batch=1)
        dev = lambda x: x.to("cuda:0").contiguous()
        inp = SequenceInputs(dev(q), dev(k), dev(v), dev(ip), dev(fp))
        out = chunkwise_forward(inp, dims, Variant(variant))
        g = chunkwise_backward(inp, dims, Variant(variant), dev(dh), out.states, out.stats, out.saved_states)
        torch.cuda.synchronize()
        # gloo gathers host tensors
        return [x.cpu() for x in (out.h_tilde, out.C_final, out.stats.m_combine, out.stats.h_denom,
                                  g.dq, g.dk, g.dv, g.d_fpre, g.d_ipre)]

    return compute


def _inputs(variant):
    import torch

    B, H, T, L, dqk, dhv = SHAPE
    g = torch.Generator().manual_seed(31 + variant)
    bf = lambda *s: torch.randn(*s, generator=g).to(torch.bfloat16)
    return [bf(B, H, T, dqk), bf(B, H, T, dqk), bf(B, H, T, dhv), torch.randn(B, H, T, generator=g),
            torch.randn(B, H, T, generator=g) + 1.0, bf(B, H, T, dhv)]


def _worker(rank, world, port, variant, out_q):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, str(ROOT))
    from paper_2503_14376_b200.shard import run_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B, H, T, L, dqk, dhv = SHAPE
    outs = run_sharded(_compute_factory(variant, T, L, dqk, dhv), _inputs(variant), B, H)
    if rank == 0:
        out_q.put([o.numpy() if o.dtype != torch.bfloat16 else o.float().numpy() for o in outs])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_two_rank_sharded_c_abi_equals_one_rank(variant):
    import torch
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, variant, q)) for r in range(2)]
    for p in procs:
        p.start()
    sharded = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    B, H, T, L, dqk, dhv = SHAPE
    full = _compute_factory(variant, T, L, dqk, dhv)(*[x.reshape(1, B * H, *x.shape[2:]) for x in _inputs(variant)])
    names = ("h", "C_final", "m_combine", "h_denom", "dq", "dk", "dv", "d_fpre", "d_ipre")
    for name, a, f in zip(names, sharded, full):
        f = f.float().numpy() if f.dtype == torch.bfloat16 else f.numpy()
        assert np.array_equal(a.reshape(f.shape), f), name


def _bench(nproc, *extra):
    env = dict(os.environ, TFLA_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"),
           "--gpus", str(nproc), "--steps", "2", "--warmup", "3", "--S", "1024", "--no-cpu-baseline",
           "--no-e2e", "--no-sweep", *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_two_ranks_weak_scaling():
    line = _bench(2)
    assert line["n_gpus"] == 2 and line["scaling"] == "weak"
    assert line["value"] > 0 and line["config"]["finite"]
    assert line["gather"] is not None and line["gather"]["backend"].startswith("gloo")


@pytest.mark.gpu
def test_bench_two_ranks_strong_scaling_config5():
    line = _bench(2, "--B-total", "4", "--NH", "3")  # 12 slices: 6 per rank
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["slices_per_rank"] == [6, 6]
    assert line["value"] > 0 and line["config"]["finite"]
