"""Host-link probe (development tool): pinned H2D alone, D2H alone, and both at once on two
streams, 4 GiB each, timed with CUDA events."""
import torch

n = 4 << 30
h_src = torch.empty(n, dtype=torch.uint8).pin_memory()
h_dst = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(up, down):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_event(e0); s2.wait_event(e0)
    if up:
        with torch.cuda.stream(s1):
            d_a.copy_(h_src, non_blocking=True)
    if down:
        with torch.cuda.stream(s2):
            h_dst.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return ms, (n * (up + down)) / (ms * 1e-3) / 1e9


for _ in range(2):
    for up, down in ((1, 0), (0, 1), (1, 1)):
        ms, gbs = run(up, down)
        print(f"up={up} down={down}: {ms:.1f} ms, {gbs:.1f} GB/s aggregate")
