"""Copy-only probes of the e2e pipeline shape (cfg2 sizes): where does the
time go between the PCIe bound and the measured e2e step?"""
import torch
B, z1, z2 = 4096, 1500, 2100
n = z1 + z2 - 1
a = torch.randint(0, 1 << 30, (B, z1), dtype=torch.int32).pin_memory()
b = torch.randint(0, 1 << 30, (B, z2), dtype=torch.int32).pin_memory()
c = torch.empty((B, n), dtype=torch.int32).pin_memory()
da = torch.empty((B, z1), dtype=torch.int32, device="cuda")
db = torch.empty((B, z2), dtype=torch.int32, device="cuda")
dc = torch.randint(0, 1 << 30, (B, n), dtype=torch.int32, device="cuda")
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
main = torch.cuda.current_stream()

def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(reps):
        fn()
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

def h2d_all():
    s_in.wait_stream(main)
    with torch.cuda.stream(s_in):
        da.copy_(a, non_blocking=True); db.copy_(b, non_blocking=True)
    main.wait_stream(s_in)

def d2h_all():
    s_out.wait_stream(main)
    with torch.cuda.stream(s_out):
        c.copy_(dc, non_blocking=True)
    main.wait_stream(s_out)

def both_all():
    s_in.wait_stream(main); s_out.wait_stream(main)
    with torch.cuda.stream(s_in):
        da.copy_(a, non_blocking=True); db.copy_(b, non_blocking=True)
    with torch.cuda.stream(s_out):
        c.copy_(dc, non_blocking=True)
    main.wait_stream(s_in); main.wait_stream(s_out)

def chunked(nch):
    rows = B // nch
    evs = [torch.cuda.Event() for _ in range(nch)]
    def fn():
        s_in.wait_stream(main)
        for i in range(nch):
            r = slice(i * rows, (i + 1) * rows)
            with torch.cuda.stream(s_in):
                da[r].copy_(a[r], non_blocking=True); db[r].copy_(b[r], non_blocking=True)
                evs[i].record(s_in)
            s_out.wait_event(evs[i])
            with torch.cuda.stream(s_out):
                c[r].copy_(dc[r], non_blocking=True)
        main.wait_stream(s_out)
    return fn

mb_in, mb_out = 4 * B * (z1 + z2) / 1e6, 4 * B * n / 1e6
t = timeit(h2d_all); print(f"H2D only      {t:.3f} ms  {mb_in / t:.1f} GB/s")
t = timeit(d2h_all); print(f"D2H only      {t:.3f} ms  {mb_out / t:.1f} GB/s")
t = timeit(both_all); print(f"H2D||D2H      {t:.3f} ms  {(mb_in + mb_out) / t:.1f} GB/s total")
for nch in (2, 4, 8, 16):
    t = timeit(chunked(nch)); print(f"chunked {nch:2d}    {t:.3f} ms  {(mb_in + mb_out) / t:.1f} GB/s total")
