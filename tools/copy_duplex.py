"""H2D and D2H concurrency on separate streams (pinned host memory)."""
import torch

n = 128 * 1024 * 1024  # 1 GiB of doubles
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.ones(n, dtype=torch.float64, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for _ in range(2):
    t_h2d = timed(lambda: d_a.copy_(h_in, non_blocking=True))
    t_d2h = timed(lambda: h_out.copy_(d_b, non_blocking=True))

    def both():
        with torch.cuda.stream(sa):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(sb):
            h_out.copy_(d_b, non_blocking=True)

    t_both = timed(both)
print(f"H2D 1 GiB {t_h2d:.2f} ms ({8 * n / t_h2d / 1e6:.1f} GB/s), D2H {t_d2h:.2f} ms ({8 * n / t_d2h / 1e6:.1f} GB/s), "
      f"both on two streams {t_both:.2f} ms")
