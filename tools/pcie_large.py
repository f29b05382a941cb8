"""D2H bandwidth into large pinned buffers: one copy vs split across two copy streams."""
import torch

for gib in (1, 4, 8):
    n = gib << 27
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
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

    def split():
        e = torch.cuda.current_stream().record_event()
        for s, (lo, hi) in ((s1, (0, n // 2)), (s2, (n // 2, n))):
            s.wait_event(e)
            with torch.cuda.stream(s):
                h[lo:hi].copy_(d[lo:hi], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)

    def chunks():
        for lo in range(0, n, 1 << 24):
            h[lo:lo + (1 << 24)].copy_(d[lo:lo + (1 << 24)], non_blocking=True)

    gb = n * 8 / 1e9
    print(f"{gib} GiB: D2H one copy {gb / timed(lambda: h.copy_(d, non_blocking=True)) * 1e3:.1f} GB/s, "
          f"two streams {gb / timed(split) * 1e3:.1f} GB/s, 128 MiB chunks {gb / timed(chunks) * 1e3:.1f} GB/s",
          flush=True)
    del h, d
