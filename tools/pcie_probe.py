"""Host<->device copy ceiling on this box (pinned memory, CUDA events): H2D alone, D2H
alone, and both directions at once -- the bound of bench.py's e2e pipeline."""
import torch

n = 1 << 28  # 1 GiB of fp32
h = torch.empty(n, dtype=torch.float32).pin_memory()
h2 = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


gb = n * 4 / 1e9
t = timed(lambda: d.copy_(h, non_blocking=True))
print(f"H2D {gb / (t / 1e3):.1f} GB/s")
t = timed(lambda: h2.copy_(d2, non_blocking=True))
print(f"D2H {gb / (t / 1e3):.1f} GB/s")
t = timed(both)
print(f"both directions: {gb / (t / 1e3):.1f} GB/s each")
