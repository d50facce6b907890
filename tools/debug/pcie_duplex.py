"""Achievable PCIe bandwidth on this box: H2D alone, D2H alone, and both at once (pinned, 64 MiB chunks)."""
import torch, json
n = 64 << 20
reps = 32
h_in = torch.empty(n * reps, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n * reps, dtype=torch.uint8, pin_memory=True)
d = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(2)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d[0].copy_(h_in[i * n:(i + 1) * n], non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out[i * n:(i + 1) * n].copy_(d[1], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return n * reps / (e0.elapsed_time(e1) / 1e3) / 1e9
run(1, 1)
print(json.dumps({"h2d_GBps": run(1, 0), "d2h_GBps": run(0, 1), "duplex_each_GBps": run(1, 1)}))
