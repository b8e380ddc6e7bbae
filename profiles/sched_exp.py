"""Step-schedule experiment (7B shape, L=128): the same fwd+bwd work over the
(b,h) slices issued as sub-steps in different stream schedules, each captured
in a CUDA graph and timed with CUDA events. Prints ms/step per schedule.

  alt-N   : N sub-steps, sub-step i (fwd then bwd) on stream i % 2 (bench.py --splits N)
  pipe-N  : N sub-steps; one stream runs the forwards in order, a second the
            backwards, backward i waiting for forward i (software pipeline)
  pipe3-N : as pipe-N with the backwards alternating over two streams
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
os.environ.setdefault("TFLA_FORCE_FUSED_FWD", "1")

import torch  # noqa: E402

from paper_2503_14376_b200 import _ffi  # noqa: E402


def main():
    B, NH, T, L, dqk, dhv = 8, 8, 8192, 128, 256, 512
    steps = int(os.environ.get("STEPS", "20"))
    dev = torch.device("cuda", 0)
    lib = _ffi.lib()
    variant = 0
    BH, NC = B * NH, T // L
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    bf = dict(dtype=torch.bfloat16, device=dev)
    f32 = dict(dtype=torch.float32, device=dev)
    q = torch.randn(BH, T, dqk, generator=g, device=dev).to(torch.bfloat16)
    k = torch.randn(BH, T, dqk, generator=g, device=dev).to(torch.bfloat16)
    v = torch.randn(BH, T, dhv, generator=g, device=dev).to(torch.bfloat16)
    ip = torch.randn(BH, T, generator=g, device=dev)
    fp = torch.randn(BH, T, generator=g, device=dev)
    dh = torch.randn(BH, T, dhv, generator=g, device=dev).to(torch.bfloat16)
    h = torch.empty(BH, T, dhv, **bf)
    m_states = torch.empty(BH, NC + 1, **f32)
    m_comb = torch.empty(BH, T, **f32)
    h_denom = torch.empty(BH, T, **f32)
    c_final = torch.empty(BH, dqk, dhv, **f32)
    n_final = torch.empty(BH, dqk, **f32)
    m_final = torch.empty(BH, **f32)
    saved = torch.empty(BH, NC, dqk, dhv, **bf)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    dfp, dip = torch.empty_like(fp), torch.empty_like(ip)

    def make_subs(parts):
        subs, off = [], 0
        for n_i in parts:
            P = lambda t: t[off:off + n_i].data_ptr()  # noqa: E731
            sdm = _ffi.tfla_dims(T, L, dqk, dhv, n_i, 1)
            subs.append(dict(
                dims=sdm,
                inp=_ffi.tfla_inputs(P(q), P(k), P(v), P(ip), P(fp)),
                out=_ffi.tfla_fwd_out(P(h), None, None, P(m_states), P(m_comb), P(h_denom), P(c_final),
                                      P(n_final), P(m_final), P(saved)),
                bin=_ffi.tfla_bwd_in(P(dh), P(saved), None, P(m_states), P(m_comb), P(h_denom)),
                gr=_ffi.tfla_grads(P(dq), P(dk), P(dv), P(dfp), P(dip)),
                wf=torch.empty(lib.tfla_workspace_bytes(ctypes.byref(sdm), variant, 0), dtype=torch.uint8, device=dev),
                wb=torch.empty(lib.tfla_workspace_bytes(ctypes.byref(sdm), variant, 1), dtype=torch.uint8, device=dev)))
            off += n_i
        return subs

    def fwd(u, s):
        if lib.tfla_chunkwise_forward(ctypes.byref(u["dims"]), variant, ctypes.byref(u["inp"]),
                                      ctypes.byref(u["out"]), u["wf"].data_ptr(), u["wf"].numel(),
                                      ctypes.c_void_p(s.cuda_stream)):
            raise RuntimeError(_ffi.last_error())

    def bwd(u, s):
        if lib.tfla_chunkwise_backward(ctypes.byref(u["dims"]), variant, ctypes.byref(u["inp"]),
                                       ctypes.byref(u["bin"]), ctypes.byref(u["gr"]), u["wb"].data_ptr(),
                                       u["wb"].numel(), ctypes.c_void_p(s.cuda_stream)):
            raise RuntimeError(_ffi.last_error())

    sides = [torch.cuda.Stream(dev) for _ in range(3)]

    def sched_alt(subs):
        main = torch.cuda.current_stream(dev)
        e = torch.cuda.Event()
        e.record(main)
        ss = [main, sides[0]]
        ss[1].wait_event(e)
        for i, u in enumerate(subs):
            fwd(u, ss[i % 2])
            bwd(u, ss[i % 2])
        j = torch.cuda.Event()
        j.record(ss[1])
        main.wait_event(j)

    def sched_pipe(subs, nb):
        main = torch.cuda.current_stream(dev)
        e = torch.cuda.Event()
        e.record(main)
        bs = sides[:nb]
        for s in bs:
            s.wait_event(e)
        for i, u in enumerate(subs):
            fwd(u, main)
            ev = torch.cuda.Event()
            ev.record(main)
            bs[i % nb].wait_event(ev)
            bwd(u, bs[i % nb])
        for s in bs:
            j = torch.cuda.Event()
            j.record(s)
            main.wait_event(j)

    def time_sched(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        gr_ = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(gr_, stream=cap):
            fn()
        torch.cuda.synchronize()
        for _ in range(3):
            gr_.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            gr_.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    specs = os.environ.get("SCHEDS", "alt-1,alt-2,alt-4,pipe-2,pipe-4,pipe-8,pipe3-4,pipe3-8").split(",")
    for spec in specs:
        kind, n = spec.split("-")
        parts = [int(x) for x in n.split("/")] if "/" in n else [BH // int(n)] * int(n)
        subs = make_subs(parts)
        if kind == "alt":
            fn = lambda: sched_alt(subs)  # noqa: E731
        elif kind == "pipe":
            fn = lambda: sched_pipe(subs, 1)  # noqa: E731
        else:
            fn = lambda: sched_pipe(subs, 2)  # noqa: E731
        ms = time_sched(fn)
        print(f"{spec:12s} {ms:.3f} ms/step  ({B * T / ms * 1e3 / 1e6:.2f} M tok/s)", flush=True)


if __name__ == "__main__":
    main()
