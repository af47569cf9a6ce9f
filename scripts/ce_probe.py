"""Copy-engine probes at cfg2 sizes: per-call overhead of chunked copies,
both directions concurrently, and a chunked H2D -> D2H pipeline."""
import torch
B, z1, z2 = 4096, 1500, 2100
n = z1 + z2 - 1
a = torch.randint(0, 1 << 30, (B, z1 + z2), dtype=torch.int32).pin_memory()
c = torch.empty((B, n), dtype=torch.int32).pin_memory()
da = torch.empty((B, z1 + z2), dtype=torch.int32, device="cuda")
dc = torch.randint(0, 1 << 30, (B, n), dtype=torch.int32, device="cuda")
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
main = torch.cuda.current_stream()
mb_in, mb_out = a.numel() * 4 / 1e6, c.numel() * 4 / 1e6


def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(reps):
        fn()
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d(nch):
    rows = B // nch
    def fn():
        s_in.wait_stream(main)
        with torch.cuda.stream(s_in):
            for i in range(nch):
                da[i * rows:(i + 1) * rows].copy_(a[i * rows:(i + 1) * rows], non_blocking=True)
        main.wait_stream(s_in)
    return fn


def d2h(nch):
    rows = B // nch
    def fn():
        s_out.wait_stream(main)
        with torch.cuda.stream(s_out):
            for i in range(nch):
                c[i * rows:(i + 1) * rows].copy_(dc[i * rows:(i + 1) * rows], non_blocking=True)
        main.wait_stream(s_out)
    return fn


def both(nch):
    f1, f2 = h2d(nch), d2h(nch)
    def fn():
        s_in.wait_stream(main); s_out.wait_stream(main)
        rows = B // nch
        for i in range(nch):
            with torch.cuda.stream(s_in):
                da[i * rows:(i + 1) * rows].copy_(a[i * rows:(i + 1) * rows], non_blocking=True)
            with torch.cuda.stream(s_out):
                c[i * rows:(i + 1) * rows].copy_(dc[i * rows:(i + 1) * rows], non_blocking=True)
        main.wait_stream(s_in); main.wait_stream(s_out)
    return fn


def pipe(nch):
    rows = B // nch
    evs = [torch.cuda.Event() for _ in range(nch)]
    def fn():
        s_in.wait_stream(main); s_out.wait_stream(main)
        for i in range(nch):
            r = slice(i * rows, (i + 1) * rows)
            with torch.cuda.stream(s_in):
                da[r].copy_(a[r], non_blocking=True)
                evs[i].record(s_in)
            s_out.wait_event(evs[i])
            with torch.cuda.stream(s_out):
                c[r].copy_(dc[r], non_blocking=True)
        main.wait_stream(s_out)
    return fn


for nch in (1, 8, 32, 128):
    t = timeit(h2d(nch)); print(f"H2D  {nch:3d} chunks {t:.3f} ms {mb_in / t:.1f} GB/s")
for nch in (1, 8, 32, 128):
    t = timeit(d2h(nch)); print(f"D2H  {nch:3d} chunks {t:.3f} ms {mb_out / t:.1f} GB/s")
for nch in (1, 8, 32, 128):
    t = timeit(both(nch)); print(f"BOTH {nch:3d} chunks {t:.3f} ms {(mb_in + mb_out) / t:.1f} GB/s total")
for nch in (4, 16, 32, 64, 128):
    t = timeit(pipe(nch)); print(f"PIPE {nch:3d} chunks {t:.3f} ms {(mb_in + mb_out) / t:.1f} GB/s total")
