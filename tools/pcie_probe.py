"""PCIe copy rates for the e2e path: 8 MiB H2D, D2H, and both concurrently (pinned)."""
import torch
n = 1 << 20
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=50):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t_h2d = timeit(lambda: d1.copy_(h1, non_blocking=True))
t_d2h = timeit(lambda: h2.copy_(d2, non_blocking=True))
t_both = timeit(both)
print(f"H2D 8 MiB {t_h2d:.1f} us ({8 * n / t_h2d / 1e3:.1f} GB/s); D2H {t_d2h:.1f} us ({8 * n / t_d2h / 1e3:.1f} GB/s); "
      f"both concurrently {t_both:.1f} us")
