"""H2D / D2H bandwidth alone and concurrently (pinned host memory)."""
import torch, time
n = 64 << 20  # 256 MB
h1 = torch.empty(n, dtype=torch.int32).pin_memory()
h2 = torch.empty(n, dtype=torch.int32).pin_memory()
d1 = torch.empty(n, dtype=torch.int32, device="cuda")
d2 = torch.empty(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
b = 4 * n / 1e9
print("H2D GB/s", b / t(h2d)); print("D2H GB/s", b / t(d2h)); print("both (per direction) GB/s", b / t(both))
