import torch
n = 1 << 30
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
def run(ns, reps=4):
    ss = [torch.cuda.Stream() for _ in range(2 * ns)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in ss: s.wait_event(e0)
    part = n // ns
    for _ in range(reps):
        for i in range(ns):
            with torch.cuda.stream(ss[i]):
                d_a[i*part:(i+1)*part].copy_(h_in[i*part:(i+1)*part], non_blocking=True)
            with torch.cuda.stream(ss[ns+i]):
                h_out[i*part:(i+1)*part].copy_(d_b[i*part:(i+1)*part], non_blocking=True)
    for s in ss:
        ev = torch.cuda.Event(); ev.record(s); torch.cuda.current_stream().wait_event(ev)
    e1.record(); torch.cuda.synchronize()
    return reps * n / (e0.elapsed_time(e1) / 1e3) / 1e9
run(1, 1)
for ns in (1, 2, 4):
    print(f"{ns} stream(s) per direction: {run(ns):.1f} GB/s per direction (bidirectional)")
