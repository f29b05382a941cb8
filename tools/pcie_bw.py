"""Pinned host<->device copy bandwidth, alone and concurrent (1 GiB each)."""
import torch

n = 1 << 27  # 1 GiB of f64
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def both():
    e = torch.cuda.current_stream().record_event()
    s1.wait_event(e)
    s2.wait_event(e)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


gb = n * 8 / 1e9
t = timed(lambda: d_in.copy_(h_in, non_blocking=True))
print(f"H2D {gb / t * 1e3:.1f} GB/s")
t = timed(lambda: h_out.copy_(d_out, non_blocking=True))
print(f"D2H {gb / t * 1e3:.1f} GB/s")
t = timed(both)
print(f"H2D+D2H concurrent: {2 * gb / t * 1e3:.1f} GB/s aggregate")
