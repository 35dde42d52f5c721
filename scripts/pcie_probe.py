"""Host<->device copy rates (pinned): H2D alone, D2H alone, both directions concurrently."""
import time
import torch

n_x, n_y = 4096 * 440, 4096 * 2048
hx = torch.empty(n_x, dtype=torch.float32).pin_memory()
hy = torch.empty(n_y, dtype=torch.float32).pin_memory()
dx = torch.empty(n_x, dtype=torch.float32, device="cuda")
dy = torch.empty(n_y, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def h2d():
    with torch.cuda.stream(s1):
        dx.copy_(hx, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        hy.copy_(dy, non_blocking=True)


def both():
    h2d()
    d2h()


th, td, tb = timeit(h2d), timeit(d2h), timeit(both)
print(f"H2D {n_x * 4 / th / 1e9:.1f} GB/s ({th * 1e3:.3f} ms), D2H {n_y * 4 / td / 1e9:.1f} GB/s "
      f"({td * 1e3:.3f} ms), both {tb * 1e3:.3f} ms")
