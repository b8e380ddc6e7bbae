"""Host <-> device copy rates on this box (pinned host memory, 1 GiB buffers,
CUDA events): H2D alone, D2H alone, and both at once on two streams -- the
ceiling of bench.py's e2e leg (1.61 GB each way per step)."""
import torch

n = 1 << 30
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=5):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_event(e0)
    s2.wait_event(e0)
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d_a.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_b, non_blocking=True)
    ev1, ev2 = torch.cuda.Event(), torch.cuda.Event()
    ev1.record(s1)
    ev2.record(s2)
    torch.cuda.current_stream().wait_event(ev1)
    torch.cuda.current_stream().wait_event(ev2)
    e1.record()
    torch.cuda.synchronize()
    return reps * n / (e0.elapsed_time(e1) / 1e3) / 1e9


run(True, True, 1)
print(f"H2D alone      {run(True, False):.1f} GB/s")
print(f"D2H alone      {run(False, True):.1f} GB/s")
print(f"H2D + D2H      {run(True, True):.1f} GB/s per direction")
